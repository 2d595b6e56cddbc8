"""Generate the golden fixtures from the UNMODIFIED reference package.

Run in the build container only (the reference tree does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Everything it writes is produced by the reference's public API
(`crtgemm.select_moduli`, `ScalingConstants.from_product`, `log2_upper`,
`fast_scaling`, `accurate_scaling`, `quantize`, `residue_decompose`,
`complex_gemm_mod`, `crt_accumulate`, `crt_reduce`, `emulate_gemm_complex`,
`gen_matrix`).  Inputs are NOT stored: they are regenerated from
(rows, cols, phi, seed) with the Philox generator the oracle restates, and the
fixture stores a sha256 of the reference-generated input so a drift is caught.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import crtgemm as ref  # noqa: E402  (reference, read-only, via PYTHONPATH)

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def moduli_fixture():
    out = {}
    for n in range(1, 21):
        ms = ref.select_moduli(n)
        sc = ref.ScalingConstants.from_product(ms.product)
        out[f"moduli_{n}"] = np.array(ms.moduli, np.int64)
        out[f"coeff_hi_{n}"] = ms.coeff_hi
        out[f"coeff_lo_{n}"] = ms.coeff_lo
        out[f"consts_{n}"] = np.array([sc.p_fast, sc.p_accu, sc.delta], np.float32)
        out[f"P_{n}"] = np.array(str(ms.product))
    return out


def log2_fixture():
    rng = np.random.default_rng(7)
    x = np.concatenate([
        np.exp(rng.uniform(-700, 700, 4000)),
        rng.uniform(1, 2, 2000),
        2.0 ** np.arange(-1074, 1024, 7, dtype=np.float64),
        np.array([1.0, 2.0, 3.0, 1e-310, 5e-324, 1.7976931348623157e308]),
    ])
    return {"log2_x": x, "log2_y": ref.log2_upper(x)}


# (tag, m, n, k, phi, seed, precision, mode, N)
SMALL_CASES = [
    ("z_fast_14", 37, 29, 53, 0.5, 0, "double", "fast", 14),
    ("z_fast_20", 40, 33, 150, 4.0, 3, "double", "fast", 20),
    ("z_accu_15", 35, 41, 67, 1.0, 5, "double", "accurate", 15),
    ("z_accu_13", 16, 18, 300, 2.0, 11, "double", "accurate", 13),
    ("c_fast_8", 31, 27, 45, 0.5, 2, "single", "fast", 8),
    ("c_fast_6", 30, 20, 260, 1.5, 9, "single", "fast", 6),
    ("c_accu_7", 25, 26, 70, 1.0, 4, "single", "accurate", 7),
    ("z_fast_1", 8, 9, 10, 0.0, 1, "double", "fast", 1),
    ("z_fast_3", 5, 7, 3, 0.5, 6, "double", "fast", 3),
    ("z_wide_k", 4, 6, 1000, 4.0, 12, "double", "fast", 16),
    ("z_tiny", 1, 1, 1, 0.5, 13, "double", "fast", 14),
]


def small_case(tag, m, n, k, phi, seed, precision, mode, N):
    a = ref.gen_matrix(ref.GenSpec(m, k, phi, seed, precision, "complex"))
    b = ref.gen_matrix(ref.GenSpec(k, n, phi, seed + 1, precision, "complex"))
    cfg = ref.EmuConfig(precision=precision, domain="complex", mode=mode, num_moduli=N)
    diag = {}
    c = ref.emulate_gemm_complex(a, b, cfg, diag)
    ms = ref.select_moduli(N)
    sc = ref.ScalingConstants.from_product(ms.product)
    a_c = a.astype(np.complex128)
    b_c = b.astype(np.complex128)
    if mode == "fast":
        sv = ref.fast_scaling(a_c, b_c, ms, sc)
    else:
        sv = ref.accurate_scaling(a_c, b_c, ms, sc)
    ar = ref.quantize(np.ascontiguousarray(a_c.real), sv.mu_exp, 0)
    ai = ref.quantize(np.ascontiguousarray(a_c.imag), sv.mu_exp, 0)
    br = ref.quantize(np.ascontiguousarray(b_c.real), sv.nu_exp, 1)
    bi = ref.quantize(np.ascontiguousarray(b_c.imag), sv.nu_exp, 1)
    st = [ref.residue_decompose(x, ms).entries for x in (ar, ai, br, bi)]
    er = np.empty((N, m, n), np.int8)
    ei = np.empty((N, m, n), np.int8)
    for idx, p in enumerate(ms.moduli):
        er[idx], ei[idx] = ref.complex_gemm_mod(st[0][idx], st[1][idx], st[2][idx],
                                                st[3][idx], p)
    p_ = f"{tag}__"
    return {
        p_ + "meta": np.array([m, n, k, seed, N, precision == "double", mode == "fast"],
                              np.int64),
        p_ + "phi": np.array(phi),
        p_ + "a_sha": np.array(sha(a)),
        p_ + "b_sha": np.array(sha(b)),
        p_ + "mu": sv.mu_exp, p_ + "nu": sv.nu_exp,
        p_ + "ar": st[0], p_ + "ai": st[1], p_ + "br": st[2], p_ + "bi": st[3],
        p_ + "er": er, p_ + "ei": ei, p_ + "c": c,
        p_ + "diag": np.array([diag.get("clamped_mu", 0), diag.get("clamped_nu", 0)]),
    }


# larger configs: only exponents and hashes are stored
HASH_CASES = [
    ("cfg1_z1024_fast14", 1024, 1024, 1024, 0.5, 0, "double", "fast", 14),
    ("cfg1_z1024_accu14", 1024, 1024, 1024, 0.5, 0, "double", "accurate", 14),
    ("z512_fast20_phi4", 512, 512, 512, 4.0, 21, "double", "fast", 20),
    ("z384_accu17_phi2", 384, 320, 448, 2.0, 22, "double", "accurate", 17),
    ("c512_fast6_phi0", 512, 512, 512, 0.0, 23, "single", "fast", 6),
    ("c512_fast10_phi1", 512, 512, 512, 1.0, 24, "single", "fast", 10),
    ("c512_accu8_phi1", 512, 512, 512, 1.0, 25, "single", "accurate", 8),
    ("z_skinny_fast14", 128, 96, 8192, 2.0, 26, "double", "fast", 14),
    ("z_ragged_fast13", 300, 200, 1000, 1.0, 27, "double", "fast", 13),
]


def hash_case(tag, m, n, k, phi, seed, precision, mode, N):
    a = ref.gen_matrix(ref.GenSpec(m, k, phi, seed, precision, "complex"))
    b = ref.gen_matrix(ref.GenSpec(k, n, phi, seed + 1, precision, "complex"))
    cfg = ref.EmuConfig(precision=precision, domain="complex", mode=mode, num_moduli=N)
    c = ref.emulate_gemm_complex(a, b, cfg)
    ms = ref.select_moduli(N)
    sc = ref.ScalingConstants.from_product(ms.product)
    a_c, b_c = a.astype(np.complex128), b.astype(np.complex128)
    sv = (ref.fast_scaling if mode == "fast" else ref.accurate_scaling)(a_c, b_c, ms, sc)
    return {
        "m": m, "n": n, "k": k, "phi": phi, "seed": seed, "precision": precision,
        "mode": mode, "N": N, "a_sha": sha(a), "b_sha": sha(b), "c_sha": sha(c),
        "mu": sv.mu_exp.tolist(), "nu": sv.nu_exp.tolist(),
        # a few raw values for a readable diff on failure
        "c_head": [[float(v.real), float(v.imag)] for v in c.reshape(-1)[:4]],
    }


# real domain (emulate_gemm_real, emulate.py:169-190)
REAL_CASES = [
    ("r_fast_15", 37, 29, 53, 0.5, 40, "double", "fast", 15),
    ("r_fast_20", 33, 40, 150, 4.0, 41, "double", "fast", 20),
    ("r_accu_15", 35, 41, 67, 1.0, 42, "double", "accurate", 15),
    ("r_fast_8s", 31, 27, 45, 0.5, 43, "single", "fast", 8),
    ("r_accu_7s", 25, 26, 70, 1.0, 44, "single", "accurate", 7),
    ("r_fast_2", 4, 5, 6, 0.0, 45, "double", "fast", 2),
    ("r_tiny", 1, 1, 1, 0.5, 46, "double", "fast", 15),
]


def real_case(tag, m, n, k, phi, seed, precision, mode, N):
    a = ref.gen_matrix(ref.GenSpec(m, k, phi, seed, precision, "real"))
    b = ref.gen_matrix(ref.GenSpec(k, n, phi, seed + 1, precision, "real"))
    cfg = ref.EmuConfig(precision=precision, domain="real", mode=mode, num_moduli=N)
    diag = {}
    c = ref.emulate_gemm_real(a, b, cfg, diag)
    ms = ref.select_moduli(N)
    sc = ref.ScalingConstants.from_product(ms.product)
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    sv = (ref.fast_scaling if mode == "fast" else ref.accurate_scaling)(a64, b64, ms, sc)
    ai = ref.quantize(a64, sv.mu_exp, 0)
    bi = ref.quantize(b64, sv.nu_exp, 1)
    ra = ref.residue_decompose(ai, ms).entries
    rb = ref.residue_decompose(bi, ms).entries
    e = np.stack([ref.symmetric_mod_int(ref.gemm_i8_i32(ra[i], rb[i]).astype(np.int64), p)
                  for i, p in enumerate(ms.moduli)]).astype(np.int8)
    p_ = f"{tag}__"
    return {
        p_ + "rmeta": np.array([m, n, k, seed, N, precision == "double", mode == "fast"],
                               np.int64),
        p_ + "phi": np.array(phi), p_ + "a_sha": np.array(sha(a)), p_ + "b_sha": np.array(sha(b)),
        p_ + "mu": sv.mu_exp, p_ + "nu": sv.nu_exp, p_ + "ra": ra, p_ + "rb": rb, p_ + "e": e,
        p_ + "c": c,
        p_ + "diag": np.array([diag.get("clamped_mu", 0), diag.get("clamped_nu", 0)]),
    }


REAL_HASH_CASES = [
    ("real512_fast15", 512, 512, 512, 1.0, 50, "double", "fast", 15),
    ("real384_accu15", 384, 320, 448, 2.0, 51, "double", "accurate", 15),
    ("real512_fast8s", 512, 512, 512, 1.0, 52, "single", "fast", 8),
    ("real_k2pow17_fast", 8, 6, 131072, 1.0, 53, "double", "fast", 15),
]


def real_hash_case(tag, m, n, k, phi, seed, precision, mode, N):
    a = ref.gen_matrix(ref.GenSpec(m, k, phi, seed, precision, "real"))
    b = ref.gen_matrix(ref.GenSpec(k, n, phi, seed + 1, precision, "real"))
    cfg = ref.EmuConfig(precision=precision, domain="real", mode=mode, num_moduli=N)
    c = ref.emulate_gemm_real(a, b, cfg)
    return {"m": m, "n": n, "k": k, "phi": phi, "seed": seed, "precision": precision,
            "mode": mode, "N": N, "domain": "real", "a_sha": sha(a), "b_sha": sha(b),
            "c_sha": sha(c), "c_head": [float(v) for v in c.reshape(-1)[:4]]}


# double-double reference products (oracle.py:60-128), the accuracy harness's target
DD_CASES = [
    ("dd_c1", 20, 30, 40, 0.5, 60, "complex"),
    ("dd_c2", 7, 5, 300, 4.0, 61, "complex"),
    ("dd_c3", 33, 17, 129, 2.0, 62, "complex"),
    ("dd_r1", 19, 23, 77, 1.0, 63, "real"),
]


def dd_case(tag, m, n, k, phi, seed, domain):
    a = ref.gen_matrix(ref.GenSpec(m, k, phi, seed, "double", domain))
    b = ref.gen_matrix(ref.GenSpec(k, n, phi, seed + 1, "double", domain))
    dd = ref.reference_gemm_dd(a, b)
    approx = a.astype(np.complex64 if domain == "complex" else np.float32) @ \
        b.astype(np.complex64 if domain == "complex" else np.float32)
    err, zeros = ref.max_relative_error(approx, dd, return_zero_count=True)
    p_ = f"{tag}__"
    return {p_ + "ddmeta": np.array([m, n, k, seed, domain == "complex"], np.int64),
            p_ + "phi": np.array(phi), p_ + "hi": dd.hi, p_ + "lo": dd.lo,
            p_ + "approx": approx, p_ + "err": np.array([err, zeros])}


def main():
    fx = {}
    fx.update(moduli_fixture())
    fx.update(log2_fixture())
    for case in SMALL_CASES:
        fx.update(small_case(*case))
    for case in REAL_CASES:
        fx.update(real_case(*case))
    for case in DD_CASES:
        fx.update(dd_case(*case))
    # exponents with long pairwise rows (k > 128 blocks, ragged tails)
    for k in (7, 127, 129, 1000, 4100, 70001):
        a = ref.gen_matrix(ref.GenSpec(3, k, 4.0, 100 + k, "double", "complex"))
        b = ref.gen_matrix(ref.GenSpec(k, 2, 4.0, 200 + k, "double", "complex"))
        ms = ref.select_moduli(14)
        sc = ref.ScalingConstants.from_product(ms.product)
        sv = ref.fast_scaling(a, b, ms, sc)
        fx[f"pw_{k}__mu"] = sv.mu_exp
        fx[f"pw_{k}__nu"] = sv.nu_exp
    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **fx)
    hashes = {}
    for case in HASH_CASES:
        hashes[case[0]] = hash_case(*case)
        print("hashed", case[0], file=sys.stderr)
    for case in REAL_HASH_CASES:
        hashes[case[0]] = real_hash_case(*case)
        print("hashed", case[0], file=sys.stderr)
    with open(os.path.join(HERE, "golden_hashes.json"), "w") as f:
        json.dump(hashes, f, indent=1)


if __name__ == "__main__":
    main()
