"""Wall time of emulate_gemm_complex on plain numpy operands (the CLI's path):
staircase streaming through pinned staging rings, result in plain numpy memory.

    python tools/numpy_e2e.py [m n k N]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_08321_b200 as crt  # noqa: E402

m, n, k, N = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (16384, 16384, 16384, 15)))
rng = np.random.default_rng(0)
t0 = time.perf_counter()
a = rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))
b = rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))
print(f"inputs generated in {time.perf_counter() - t0:.1f} s", flush=True)
cfg = crt.EmuConfig(domain="complex", num_moduli=N)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c = crt.emulate_gemm_complex(a, b, cfg)
    dt = time.perf_counter() - t0
    print(f"call {it}: {dt * 1e3:.1f} ms wall, {8 * m * n * k / dt * 1e-12:.1f} TFLOPS "
          f"(numpy in, numpy out {type(c).__name__} {c.dtype})", flush=True)
