"""Host-side profile of the public call on a small product (run on the GPU box):
where the Python / ctypes time of one emulate_gemm_complex goes.

    python tools/small_pyprof.py [size]
"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_08321_b200 as crt  # noqa: E402
from bench import synth  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dev = torch.device("cuda", 0)
A = synth(torch, s, s, 0.5, 1, torch.complex128, dev)
B = synth(torch, s, s, 0.5, 2, torch.complex128, dev)
cfg = crt.EmuConfig(domain="complex", num_moduli=14)
for _ in range(20):
    crt.emulate_gemm_complex(A, B, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(500):
    crt.emulate_gemm_complex(A, B, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
