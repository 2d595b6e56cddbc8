"""Real-domain emulated DGEMM / SGEMM throughput vs cuBLAS native (run on the GPU box).

    python tools/real_bench.py [--shape M N K] [--moduli N] [--precision double|single]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2512_08321_b200 as crt  # noqa: E402
from paper_2512_08321_b200 import _native as nat  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", type=int, nargs=3, default=[16384, 16384, 16384])
    ap.add_argument("--moduli", type=int, nargs="+", default=[14, 16])
    ap.add_argument("--precision", default="double")
    a = ap.parse_args()
    m, n, k = a.shape
    dt = torch.float64 if a.precision == "double" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(0)
    A = (torch.rand(m, k, generator=g, device="cuda", dtype=torch.float64) - 0.5).to(dt)
    B = (torch.rand(k, n, generator=g, device="cuda", dtype=torch.float64) - 0.5).to(dt)
    native = timed(lambda: A @ B)
    rows = []
    for N in a.moduli:
        cfg = crt.EmuConfig(precision=a.precision, domain="real", mode="fast", num_moduli=N)
        nat.profile_enable(True)
        ms = timed(lambda: crt.emulate_gemm_real(A, B, cfg))
        st, cnt = nat.profile_read()
        nat.profile_enable(False)
        reps = 6
        rows.append({"N": N, "ms": ms, "tflops": 2 * m * n * k / (ms * 1e-3) / 1e12,
                     "native_ms": native, "speedup": native / ms,
                     "stage_ms": {s: v / reps for s, v in st.items()}})
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
