"""Golden vectors for the stage-level drop-in API (paper_2512_08321_b200/stages.py),
generated from the UNMODIFIED reference package.

Run in the build container only (the reference tree does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_stage_golden.py

Every output below is the reference's own function applied to seeded inputs
(the inputs are stored too: they are small).  Functions covered:
`quantize` (scaling.py:277-293), `symmetric_mod_int` (crt.py:136-151),
`residue_decompose` (crt.py:199-218), `crt_accumulate` (crt.py:221-243),
`crt_reduce` (crt.py:246-258), `symmetric_mod_wide` (crt.py:154-184),
`inverse_scale` (emulate.py:135-144), `crt_integer_gemm` (emulate.py:120-132).
"""

from __future__ import annotations

import os

import numpy as np

import crtgemm as ref  # noqa: E402  (reference, read-only, via PYTHONPATH)

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(20260)
    fx = {}

    # quantize: per-row and per-column exponents, incl. wide results (2^80)
    a = ref.gen_matrix(ref.GenSpec(23, 41, 2.0, 70, "double", "complex"))
    ms14 = ref.select_moduli(14)
    sc14 = ref.ScalingConstants.from_product(ms14.product)
    b = ref.gen_matrix(ref.GenSpec(41, 41, 2.0, 71, "double", "complex"))
    sv = ref.fast_scaling(a, b, ms14, sc14)
    x = np.ascontiguousarray(a.real)
    fx["q_x"] = x
    fx["q_mu"] = sv.mu_exp
    fx["q_rows"] = ref.quantize(x, sv.mu_exp, 0)
    fx["q_nu"] = sv.nu_exp
    fx["q_cols"] = ref.quantize(x, sv.nu_exp, 1)
    wide_e = rng.integers(60, 80, size=23).astype(np.int64)
    fx["q_wide_e"] = wide_e
    fx["q_wide"] = ref.quantize(x, wide_e, 0)

    # symmetric_mod_int: int64 (|x| < 2^61), integer-valued float64 (|x| < 2^90)
    xi = rng.integers(-(2 ** 60), 2 ** 60, size=3000, dtype=np.int64)
    xi[:8] = [0, 1, -1, 127, -128, 2 ** 60 - 1, -(2 ** 60), 255]
    xf = np.trunc(rng.uniform(-1, 1, size=3000) * 2.0 ** rng.integers(0, 90, size=3000))
    xf[:6] = [0.0, -0.0, 2.0 ** 89, -(2.0 ** 89), 2.0 ** 63, -(2.0 ** 31)]
    fx["smi_xi"] = xi
    fx["smi_xf"] = xf
    plist = [2, 3, 127, 128, 173, 199, 241, 255, 256]
    fx["smi_p"] = np.array(plist, np.int64)
    for p in plist:
        fx[f"smi_i_{p}"] = ref.symmetric_mod_int(xi, p)
        fx[f"smi_f_{p}"] = ref.symmetric_mod_int(xf, p)
    fx["smi_scalar"] = np.array([[v, p, ref.symmetric_mod_int(v, p)]
                                 for v in (0, 5, -5, 128, -129, 10 ** 15, -(10 ** 15))
                                 for p in (7, 128, 256)], np.int64)

    # residue_decompose of the wide quantized matrix at N=20
    ms20 = ref.select_moduli(20)
    fx["rd_20"] = ref.residue_decompose(fx["q_wide"], ms20).entries

    # crt_accumulate / crt_reduce / inverse_scale on a small product's e-planes
    for N, prec in ((15, "double"), (8, "single"), (20, "double"), (1, "double")):
        ms = ref.select_moduli(N)
        e = np.stack([rng.integers(-(p // 2), (p + 1) // 2, size=(19, 33)).astype(np.int8)
                      for p in ms.moduli])
        st = ref.ResidueStack(e, ms)
        fx[f"ca_{N}_e"] = e
        acc = ref.crt_accumulate(st, ms, prec)
        if prec == "double":
            fx[f"ca_{N}_s1"], fx[f"ca_{N}_s2"] = acc
        else:
            fx[f"ca_{N}_s"] = acc
        red = ref.crt_reduce(acc, ms)
        fx[f"ca_{N}_red"] = red
        mu = rng.integers(-40, 80, size=19).astype(np.int64)
        nu = rng.integers(-40, 80, size=33).astype(np.int64)
        svx = ref.ScalingVectors(mu_exp=mu, nu_exp=nu)
        fx[f"ca_{N}_mu"], fx[f"ca_{N}_nu"] = mu, nu
        fx[f"ca_{N}_inv64"] = ref.inverse_scale(red, svx, np.float64)
        fx[f"ca_{N}_inv32"] = ref.inverse_scale(red, svx, np.float32)

    # symmetric_mod_wide on arbitrary accumulators (both paths)
    for N in (6, 14, 20):
        P = ref.select_moduli(N).product
        hi = rng.uniform(-1, 1, size=500) * float(P) * 8.0
        lo = rng.uniform(-1, 1, size=500) * 2.0 ** 20
        hi[:4] = [0.0, float(P) / 2, -float(P) / 2, float(P) * 1.5]
        fx[f"smw_{N}_hi"], fx[f"smw_{N}_lo"] = hi, lo
        fx[f"smw_{N}_dd"] = ref.symmetric_mod_wide((hi, lo), P, use_dd=True)
        fx[f"smw_{N}_plain"] = ref.symmetric_mod_wide(hi, P, use_dd=False)
        fx[f"smw_{N}_P"] = np.array(str(P))

    # crt_integer_gemm: exact integer products (and one beyond the uniqueness bound)
    for tag, N, bits, m, k, n in (("cig_a", 8, 20, 17, 50, 13), ("cig_b", 14, 40, 9, 300, 11),
                                  ("cig_c", 3, 12, 6, 40, 7)):
        ms = ref.select_moduli(N)
        ai = rng.integers(-(2 ** bits), 2 ** bits, size=(m, k)).astype(np.float64)
        bi = rng.integers(-(2 ** bits), 2 ** bits, size=(k, n)).astype(np.float64)
        fx[f"{tag}_a"], fx[f"{tag}_b"], fx[f"{tag}_N"] = ai, bi, np.array(N)
        fx[f"{tag}_d"] = ref.crt_integer_gemm(ai, bi, ms, "double")
        fx[f"{tag}_s"] = ref.crt_integer_gemm(ai, bi, ms, "single", n_block=4)

    np.savez_compressed(os.path.join(HERE, "golden_stages.npz"), **fx)


if __name__ == "__main__":
    main()
