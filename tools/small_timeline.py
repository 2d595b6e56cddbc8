"""Kernel timeline of one small emulation (latency analysis), run on the GPU box:

    python tools/small_timeline.py [m n k N mode]
"""
import sys
import time

import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_08321_b200 as crt
from bench import synth

m, n, k, N = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (1024, 1024, 1024, 14)))
mode = sys.argv[5] if len(sys.argv) > 5 else "fast"
dev = torch.device("cuda:0")
A = synth(torch, m, k, 0.5, 1, torch.complex128, dev)
B = synth(torch, k, n, 0.5, 2, torch.complex128, dev)
C = torch.empty(m, n, dtype=torch.complex128, device=dev)
cfg = crt.EmuConfig(domain="complex", mode=mode, num_moduli=N)
for _ in range(5):
    crt.run_complex(A, B, cfg, sync_check=False, out=C)
torch.cuda.synchronize()
reps = 50
t0 = time.perf_counter()
for _ in range(reps):
    crt.run_complex(A, B, cfg, sync_check=False, out=C)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / reps
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    crt.run_complex(A, B, cfg, sync_check=False, out=C)
e1.record()
torch.cuda.synchronize()
print(f"wall/call {wall*1e3:.3f} ms, device/call {e0.elapsed_time(e1)/reps:.3f} ms")
t0 = time.perf_counter()
for _ in range(reps):
    crt.run_complex(A, B, cfg, sync_check=False, out=C)
host = (time.perf_counter() - t0) / reps
torch.cuda.synchronize()
print(f"host enqueue/call {host*1e3:.3f} ms")
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        crt.run_complex(A, B, cfg, sync_check=False, out=C)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
last = None
for e in evs[-40:]:
    gap = (e.time_range.start - last) if last is not None else 0
    print(f"{e.name[:60]:60s} start+{gap:8.1f}us dur {e.time_range.elapsed_us():8.1f}us")
    last = e.time_range.end
