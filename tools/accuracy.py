"""Per-moduli-count accuracy of the B200 emulation against an exact product.

For each (precision, mode, N, phi): max relative error (the reference's metric,
oracle.py:131-169) over a random sample of output entries, each computed exactly
(Dekker-split products + math.fsum, oracle.exact_entries), next to cuBLAS native
(torch.matmul) on the same inputs.  Inputs: the reference generator (Philox +
ndtri) at m = n = 1024, k = 16384 (the paper's accuracy shape).

    python tools/accuracy.py [--m 1024 --n 1024 --k 16384 --samples 256] > profiles/accuracy.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_08321_b200 as crt  # noqa: E402
from oracle import ozaki2 as orc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1024)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--k", type=int, default=16384)
    ap.add_argument("--samples", type=int, default=256)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    rows = rng.integers(0, a.m, a.samples)
    cols = rng.integers(0, a.n, a.samples)
    sweeps = [("single", (0.0, 0.5, 1.0, 1.5), {"fast": range(6, 11), "accurate": range(6, 10)}),
              ("double", (0.5, 1.0, 2.0, 4.0), {"fast": range(12, 21), "accurate": range(12, 20)})]
    out = {"shape": [a.m, a.n, a.k], "samples": a.samples, "results": []}
    for prec, phis, modes in sweeps:
        for phi in phis:
            t0 = time.time()
            A = orc.gen_matrix(a.m, a.k, phi, 1, prec)
            B = orc.gen_matrix(a.k, a.n, phi, 2, prec)
            hi, lo = orc.exact_entries(A, B, rows, cols)
            ta = torch.from_numpy(np.ascontiguousarray(A)).cuda()
            tb = torch.from_numpy(np.ascontiguousarray(B)).cuda()
            native = torch.matmul(ta, tb).cpu().numpy()
            e_nat = orc.max_relative_error(native[rows, cols], hi, lo)
            for mode, Ns in modes.items():
                for N in Ns:
                    cfg = crt.EmuConfig(precision=prec, domain="complex", mode=mode, num_moduli=N)
                    c = crt.emulate_gemm_complex(ta, tb, cfg).cpu().numpy()
                    e = orc.max_relative_error(c[rows, cols], hi, lo)
                    out["results"].append({"precision": prec, "phi": phi, "mode": mode, "N": N,
                                           "max_rel_err": e, "native_max_rel_err": e_nat})
            print(f"{prec} phi={phi} done in {time.time() - t0:.1f}s", file=sys.stderr)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
