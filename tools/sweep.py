"""Throughput over the BASELINE.json configs (device-resident synthetic inputs,
CUDA-event timing, cuBLAS native on the same inputs).

    python tools/sweep.py > profiles/rNN_configs.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2512_08321_b200 as crt  # noqa: E402
from bench import synth  # noqa: E402

CONFIGS = [
    # cfg1: ZGEMM 1024^3 N=14 (the reference's CPU-runnable case)
    ("zgemm", 1024, 1024, 1024, 14, "fast", 0.5),
    ("zgemm", 1024, 1024, 1024, 14, "accurate", 0.5),
    # cfg2: CGEMM 8192^3, N 6..10, fast
    *[("cgemm", 8192, 8192, 8192, N, "fast", 1.0) for N in (6, 7, 8, 9, 10)],
    ("cgemm", 8192, 8192, 8192, 7, "accurate", 1.0),
    # cfg3: ZGEMM 16384^3, N 12..20, fast vs accurate
    *[("zgemm", 16384, 16384, 16384, N, "fast", 0.5) for N in (12, 14, 15, 16, 18, 20)],
    *[("zgemm", 16384, 16384, 16384, N, "accurate", 0.5) for N in (13, 15, 17)],
    # cfg4: skinny ZGEMM m=n=4096, k=65536, wide exponent range
    *[("zgemm", 4096, 4096, 65536, N, "fast", 4.0) for N in (14, 17, 20)],
    ("zgemm", 4096, 4096, 65536, 16, "accurate", 2.0),
    # CGEMM at the headline shape
    ("cgemm", 16384, 16384, 16384, 8, "fast", 1.0),
]


def time_fn(fn, reps=3, warm=2):
    for _ in range(warm):
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
    dev = torch.device("cuda", 0)
    out = []
    native_cache = {}
    for kind, m, n, k, N, mode, phi in CONFIGS:
        cdt = torch.complex128 if kind == "zgemm" else torch.complex64
        A = synth(torch, m, k, phi, 1, cdt, dev)
        B = synth(torch, k, n, phi, 2, cdt, dev)
        cfg = crt.EmuConfig(precision="double" if kind == "zgemm" else "single", domain="complex",
                            mode=mode, num_moduli=N)
        C = torch.empty((m, n), dtype=cdt, device=dev)
        ms = time_fn(lambda: crt.run_complex(A, B, cfg, sync_check=False, out=C))
        key = (kind, m, n, k)
        if key not in native_cache:
            native_cache[key] = time_fn(lambda: torch.matmul(A, B, out=C), reps=2, warm=1)
        nat = native_cache[key]
        fl = 8.0 * m * n * k
        rec = {"kind": kind, "m": m, "n": n, "k": k, "N": N, "mode": mode, "phi": phi,
               "ms": ms, "tflops": fl / ms / 1e9, "native_ms": nat,
               "native_tflops": fl / nat / 1e9, "speedup": nat / ms,
               "int8_tops": 6 * (N + (mode == "accurate")) * m * n * k / ms / 1e9}
        out.append(rec)
        print(json.dumps(rec), file=sys.stderr, flush=True)
        del A, B, C
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
