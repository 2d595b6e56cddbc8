"""GPU: every launch-configuration variant of the library computes the same
bytes (reference contract: the result depends only on the inputs and the
modulus count / mode -- SPEC.md:306, tests/test_emulate.py:90-96).

The kernel variants are chosen per call from the problem size and a few
process-wide switches that the library reads once (environment).  Each variant
set below runs in its own process on the same seeded inputs; the SHA-256 of
every result must agree with the default configuration's:
  * the residue kernel's rolled (small launches) / unrolled modulus loop
    (CRTG_RES_ROLLED_TILES), the CRT's two / four columns per thread
    (CRTG_CRT_Q2_THREADS), the 128 x 256 / 256 x 256 GEMM (CRTG_GEMM);
  * programmatic dependent launch (CRTG_PDL), the forked B chain (CRTG_FORK)
    and CUDA-graph replay (CRTG_GRAPHS)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, json, sys
sys.path.insert(0, %(root)r)
import numpy as np
import torch
import paper_2512_08321_b200 as crt
from oracle import ozaki2 as orc

CASES = [
    # (m, k, n, N, mode, precision, phi, seed)
    (1000, 700, 900, 14, "fast", "double", 1.0, 3),
    (384, 2048, 512, 15, "accurate", "double", 0.5, 5),
    (300, 500, 400, 8, "fast", "single", 1.0, 7),
    (2048, 1024, 2048, 14, "fast", "double", 0.5, 9),
]
out = {}
for (m, k, n, N, mode, prec, phi, seed) in CASES:
    a = np.ascontiguousarray(orc.gen_matrix(m, k, phi, seed, prec))
    b = np.ascontiguousarray(orc.gen_matrix(k, n, phi, seed + 1, prec))
    A = torch.from_numpy(a).cuda()
    B = torch.from_numpy(b).cuda()
    cfg = crt.EmuConfig(precision=prec, domain="complex", mode=mode, num_moduli=N)
    digests = []
    for _ in range(3):  # eager, capture, replay (graphs on)
        c = crt.emulate_gemm_complex(A, B, cfg)
        torch.cuda.synchronize()
        digests.append(hashlib.sha256(c.cpu().numpy().tobytes()).hexdigest())
    out[f"{m}x{k}x{n}_{N}_{mode}_{prec}"] = digests
print("RESULT " + json.dumps(out))
"""

VARIANTS = {
    "default": {},
    "unrolled_q4_nopdl": {"CRTG_RES_ROLLED_TILES": "0", "CRTG_CRT_Q2_THREADS": "0",
                          "CRTG_PDL": "0", "CRTG_FORK": "0", "CRTG_GRAPHS": "0"},
    "rolled_q2_wide": {"CRTG_RES_ROLLED_TILES": "100000000",
                       "CRTG_CRT_Q2_THREADS": "100000000000", "CRTG_GEMM": "wide"},
    "one_gemm": {"CRTG_GEMM": "one", "CRTG_GRAPHS": "0"},
}


def _run(env_extra):
    env = dict(os.environ)
    for key in ("CRTG_RES_ROLLED_TILES", "CRTG_CRT_Q2_THREADS", "CRTG_PDL", "CRTG_FORK",
                "CRTG_GRAPHS", "CRTG_GEMM"):
        env.pop(key, None)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")][-1]
    return json.loads(line[len("RESULT "):])


def test_variants_bitwise_identical():
    results = {name: _run(env) for name, env in VARIANTS.items()}
    base = results["default"]
    for case, digests in base.items():
        assert len(set(digests)) == 1, (case, "eager / capture / replay differ")
    for name, res in results.items():
        for case, digests in res.items():
            assert set(digests) == {base[case][0]}, (name, case)
