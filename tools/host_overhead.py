"""Host-side cost of one synchronous small product (run on the GPU box): the
public call, the device entry with its synchronous check, and the bare C-ABI
call with prebuilt arguments -- the differences are Python wrapper time.

    python tools/host_overhead.py [size]
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_08321_b200 as crt  # noqa: E402
from paper_2512_08321_b200 import _native as nat  # noqa: E402
from paper_2512_08321_b200.moduli import device_constants  # noqa: E402
from bench import synth  # noqa: E402


def wall(fn, reps=400):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


s = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dev = torch.device("cuda", 0)
A = synth(torch, s, s, 0.5, 1, torch.complex128, dev)
B = synth(torch, s, s, 0.5, 2, torch.complex128, dev)
C = torch.empty((s, s), dtype=torch.complex128, device=dev)
cfg = crt.EmuConfig(domain="complex", num_moduli=14)
lib = nat.load()
need = lib.crtg_workspace_size(0, 0, s, s, s, 14, cfg.n_block)
ws = torch.empty(need, dtype=torch.uint8, device=dev)
dg = torch.empty(nat.DIAG_LEN, dtype=torch.int64, device=dev)
K = ctypes.byref(device_constants(14))
stream = torch.cuda.current_stream(dev).cuda_stream
args = (0, 0, s, s, s, A.data_ptr(), s, B.data_ptr(), s, C.data_ptr(), s, K, cfg.n_block,
        ws.data_ptr(), ws.numel(), None, None, dg.data_ptr(), 1, stream)
f = lib.crtg_gemm_complex
rec = {
    "size": s,
    "public_us": wall(lambda: crt.emulate_gemm_complex(A, B, cfg)),
    "run_complex_sync_us": wall(lambda: crt.run_complex(A, B, cfg, sync_check=True, out=C, ws=ws)),
    "c_abi_sync_us": wall(lambda: f(*args)),
    "c_abi_nosync_us": wall(lambda: f(*(args[:18] + (0, stream)))),
}
print(json.dumps(rec))
