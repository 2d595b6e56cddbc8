"""Per-moduli-count accuracy on the FULL product (every entry), via the GPU
double-double reference (bit-identical to the reference's reference_gemm_dd).

    python tools/accuracy_full.py [--n 16384] [--phis 0.5 4] > profiles/rNN_accuracy_full.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2512_08321_b200 as crt  # noqa: E402
from bench import synth  # noqa: E402
from paper_2512_08321_b200 import accuracy as acc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--phis", type=float, nargs="+", default=[0.5, 4.0])
    ap.add_argument("--kind", choices=("zgemm", "cgemm"), default="zgemm")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = a.n
    cdt = torch.complex128 if a.kind == "zgemm" else torch.complex64
    prec = "double" if a.kind == "zgemm" else "single"
    sweeps = ({"fast": range(12, 21), "accurate": range(13, 20)} if prec == "double"
              else {"fast": range(6, 11), "accurate": range(6, 10)})
    out = {"kind": a.kind, "shape": [n, n, n], "results": []}
    for phi in a.phis:
        A = synth(torch, n, n, phi, 1, cdt, dev)
        B = synth(torch, n, n, phi, 2, cdt, dev)
        torch.cuda.synchronize()
        t0 = time.time()
        ref = acc.reference_gemm_dd(A.to(torch.complex128), B.to(torch.complex128))
        torch.cuda.synchronize()
        t_dd = time.time() - t0
        nat = torch.matmul(A, B)
        e_nat = acc.max_relative_error(nat, ref)
        del nat
        rec = {"phi": phi, "dd_seconds": t_dd, "native_max_rel_err": e_nat, "emulated": []}
        for mode, Ns in sweeps.items():
            for N in Ns:
                cfg = crt.EmuConfig(precision=prec, domain="complex", mode=mode, num_moduli=N)
                c = crt.emulate_gemm_complex(A, B, cfg)
                e = acc.max_relative_error(c, ref)
                del c
                rec["emulated"].append({"mode": mode, "N": N, "max_rel_err": e})
                print(f"phi={phi} {mode} N={N}: {e:.3e} (native {e_nat:.3e})", file=sys.stderr,
                      flush=True)
        out["results"].append(rec)
        del A, B, ref
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
