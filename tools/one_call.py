"""A few synchronous emulated products of one size (run on the GPU box), e.g.
as the target of an ncu capture of the small-product kernels:

    CRTG_GRAPHS=0 ncu --set full -k regex:k_ -s 7 -c 7 -o prof python tools/one_call.py 1024 3
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_08321_b200 as crt
from bench import synth
s = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
A = synth(torch, s, s, 0.5, 1, torch.complex128, dev)
B = synth(torch, s, s, 0.5, 2, torch.complex128, dev)
C = torch.empty((s, s), dtype=torch.complex128, device=dev)
cfg = crt.EmuConfig(domain="complex", num_moduli=14)
for _ in range(reps):
    crt.run_complex(A, B, cfg, sync_check=True, out=C)
torch.cuda.synchronize()
