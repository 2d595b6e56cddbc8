"""Per-call wall time of the device path for small products (host overhead +
GPU work), e.g. python tools/small_latency.py 256 1024"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_08321_b200 as crt  # noqa: E402

for s in (int(x) for x in (sys.argv[1:] or ["256", "1024"])):
    A = torch.randn(s, s, dtype=torch.complex128, device="cuda")
    B = torch.randn(s, s, dtype=torch.complex128, device="cuda")
    cfg = crt.EmuConfig(domain="complex", num_moduli=14)
    for _ in range(5):
        crt.emulate_gemm_complex(A, B, cfg)
    torch.cuda.synchronize()
    reps = 200
    t0 = time.perf_counter()
    for _ in range(reps):
        crt.emulate_gemm_complex(A, B, cfg)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        crt.emulate_gemm_complex(A, B, cfg)
    e1.record()
    torch.cuda.synchronize()
    print(f"{s}^3 N=14: {dt * 1e6:.0f} us wall per call, {e0.elapsed_time(e1) / reps * 1e3:.0f} us "
          f"GPU-timeline per call", flush=True)
