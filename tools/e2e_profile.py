"""Where the end-to-end (host-buffer) call spends its time (run on the GPU box).

Times crtg_gemm_complex_host through the public API on pinned host tensors and
reports the wall time next to the GPU time of each stage (CUDA events inside
the library), so wall - sum(stages) is the time the GPU waited for PCIe.

    python tools/e2e_profile.py [--shape M N K] [--moduli N] [--reps R]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2512_08321_b200 as crt  # noqa: E402
from paper_2512_08321_b200 import _native as nat  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", type=int, nargs=3, default=[16384, 16384, 16384])
    ap.add_argument("--moduli", type=int, default=15)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n-block", type=int, default=8192)
    a = ap.parse_args()
    m, n, k = a.shape
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(m, k, dtype=torch.complex128, device="cuda", generator=g)
    B = torch.randn(k, n, dtype=torch.complex128, device="cuda", generator=g)
    hA, hB = A.cpu().pin_memory(), B.cpu().pin_memory()
    # PCIe: one contiguous 4 GiB H2D, and B's 2048-column blocks as 2-D copies
    dA = torch.empty_like(A)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pcie = {}
    for name, fn in (("h2d_contig", lambda: dA.copy_(hA, non_blocking=True)),
                     ("h2d_cols2048", lambda: [dA[:, j:j + 2048].copy_(hB[:, j:j + 2048],
                                                                      non_blocking=True)
                                               for j in range(0, n, 2048)]),
                     ("d2h_contig", lambda: hA.copy_(dA, non_blocking=True))):
        fn()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        pcie[name] = round(A.numel() * 16 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
    del A, B, dA
    cfg = crt.EmuConfig(precision="double", domain="complex", mode="fast", num_moduli=a.moduli,
                        n_block=a.n_block)
    crt.emulate_gemm_complex(hA, hB, cfg)
    torch.cuda.synchronize()
    nat.load()
    nat.profile_enable(True)
    t0 = time.perf_counter()
    for _ in range(a.reps):
        crt.emulate_gemm_complex(hA, hB, cfg)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / a.reps * 1e3
    st, cnt = nat.profile_read()
    nat.profile_enable(False)
    stages = {s: v / a.reps for s, v in st.items()}
    print(json.dumps({"shape": a.shape, "moduli": a.moduli, "wall_ms": wall, "pcie_GBps": pcie,
                      "stage_ms": stages, "stage_launches": {s: c / a.reps for s, c in cnt.items()},
                      "gpu_busy_ms": sum(stages.values()),
                      "tflops": 8 * m * n * k / (wall * 1e-3) / 1e12}))


if __name__ == "__main__":
    main()
