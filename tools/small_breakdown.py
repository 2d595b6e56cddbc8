"""Where the time of a small emulated product goes (run on the GPU box):
public API per call (synchronous, like the reference), the device entry without
the synchronous domain check, the GPU time alone (CUDA events around a loop of
graph replays), and cuBLAS native on the same operands.

    python tools/small_breakdown.py [size ...]   -> one JSON line per size
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_08321_b200 as crt  # noqa: E402
from bench import synth  # noqa: E402


def wall(fn, reps):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


def device(fn, reps):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    dev = torch.device("cuda", 0)
    for s in (int(x) for x in (sys.argv[1:] or ["256", "1024", "2048"])):
        A = synth(torch, s, s, 0.5, 1, torch.complex128, dev)
        B = synth(torch, s, s, 0.5, 2, torch.complex128, dev)
        C = torch.empty((s, s), dtype=torch.complex128, device=dev)
        reps = 200 if s <= 1024 else 50
        rec = {"size": s, "N": 14, "mode": "fast"}
        for mode in ("fast", "accurate"):
            cfg = crt.EmuConfig(domain="complex", mode=mode, num_moduli=14)
            rec[mode] = {
                "public_api_us": wall(lambda: crt.emulate_gemm_complex(A, B, cfg), reps),
                "device_entry_nosync_us": wall(
                    lambda: crt.run_complex(A, B, cfg, sync_check=False, out=C), reps),
                "gpu_timeline_us": device(
                    lambda: crt.run_complex(A, B, cfg, sync_check=False, out=C), reps),
            }
        rec["native_cublas_us"] = device(lambda: torch.matmul(A, B, out=C), reps)
        rec["speedup_public_fast"] = rec["native_cublas_us"] / rec["fast"]["public_api_us"]
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
