"""Per-call device time and output hash for one m x n x k shape, e.g.
    CRTG_GEMM=one python tools/shape_ab.py 4096 4096 65536 14 fast"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_08321_b200 as crt  # noqa: E402
from bench import synth  # noqa: E402

m, n, k, N = (int(x) for x in sys.argv[1:5])
mode = sys.argv[5] if len(sys.argv) > 5 else "fast"
A = synth(torch, m, k, 0.5, 1, torch.complex128, torch.device("cuda"))
B = synth(torch, k, n, 0.5, 2, torch.complex128, torch.device("cuda"))
cfg = crt.EmuConfig(domain="complex", mode=mode, num_moduli=N)
C = crt.emulate_gemm_complex(A, B, cfg)
h = hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()[:12]
for _ in range(3):
    crt.emulate_gemm_complex(A, B, cfg)
reps = max(3, min(100, int(2e12 // (m * n * k))))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(reps):
    crt.emulate_gemm_complex(A, B, cfg)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"shape": [m, n, k], "N": N, "mode": mode,
                  "env": {kk: v for kk, v in os.environ.items() if kk.startswith("CRTG_")},
                  "us": round(e0.elapsed_time(e1) / reps * 1e3, 1), "hash": h}), flush=True)
