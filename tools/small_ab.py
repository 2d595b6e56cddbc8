"""Small-size A/B of env knobs: per-call device time and an output hash, e.g.
    CRTG_GEMM=one python tools/small_ab.py 1024 2048
Compare the hashes across runs for bitwise equality."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_08321_b200 as crt  # noqa: E402
from bench import synth  # noqa: E402

for s in (int(x) for x in (sys.argv[1:] or ["1024"])):
    A = synth(torch, s, s, 0.5, 1, torch.complex128, torch.device("cuda"))
    B = synth(torch, s, s, 0.5, 2, torch.complex128, torch.device("cuda"))
    for mode in os.environ.get("SAB_MODES", "fast,accurate").split(","):
        cfg = crt.EmuConfig(domain="complex", mode=mode, num_moduli=14)
        C = crt.emulate_gemm_complex(A, B, cfg)
        h = hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()[:12]
        for _ in range(5):
            crt.emulate_gemm_complex(A, B, cfg)
        reps = max(3, min(100, int(2e12 // s**3)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            crt.emulate_gemm_complex(A, B, cfg)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"size": s, "mode": mode, "env": {k: v for k, v in os.environ.items()
                                                           if k.startswith("CRTG_")},
                          "us": round(e0.elapsed_time(e1) / reps * 1e3, 1), "hash": h}), flush=True)
