"""GPU parity: every stage of the CUDA path against the reference's golden vectors
and the CPU oracle (bit-exact; integer stages and final results alike).

All tests here need a B200 and the built libcrtg.so (marker `gpu`)."""

import hashlib

import numpy as np
import pytest

from oracle import ozaki2 as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def crt():
    import paper_2512_08321_b200 as crt
    from paper_2512_08321_b200 import _native
    _native.load()
    return crt


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _cases(golden):
    return sorted({k.split("__")[0] for k in golden.files if k.endswith("__meta")})


def _case_inputs(golden, tag):
    g = lambda s: golden[f"{tag}__{s}"]  # noqa: E731
    m, n, k, seed, N, dbl, fast = g("meta").tolist()
    prec = "double" if dbl else "single"
    mode = "fast" if fast else "accurate"
    a = orc.gen_matrix(m, k, float(g("phi")), seed, prec)
    b = orc.gen_matrix(k, n, float(g("phi")), seed + 1, prec)
    return a, b, N, prec, mode, g


# ---------------------------------------------------------------- K3: int8 GEMM
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (37, 29, 53), (128, 256, 128), (300, 500, 1000),
                                   (129, 257, 4096), (64, 1000, 130)])
def test_gemm_i8_i32_random(crt, m, n, k):
    rng = np.random.default_rng(m * 7 + n * 11 + k)
    a = rng.integers(-128, 128, (m, k), dtype=np.int8)
    b = rng.integers(-128, 128, (k, n), dtype=np.int8)
    c = crt.gemm_i8_i32(a, b)
    assert c.dtype == np.int32
    assert np.array_equal(c, orc.i8_product(a, b))


def test_gemm_i8_i32_extremes(crt):
    # all -128 with k = 4096 (reference tests/test_kernel.py:34-39)
    a = np.full((130, 4096), -128, np.int8)
    b = np.full((4096, 300), -128, np.int8)
    c = crt.gemm_i8_i32(a, b)
    assert np.all(c == 4096 * 16384)
    # the k cap and the int32 accumulator bound
    with pytest.raises(crt.DimensionError):
        crt.gemm_i8_i32(np.zeros((1, 2 ** 17 + 1), np.int8), np.zeros((2 ** 17 + 1, 1), np.int8))


def test_gemm_i8_i32_max_k(crt):
    rng = np.random.default_rng(5)
    a = rng.integers(-128, 128, (4, 2 ** 16), dtype=np.int8)
    b = rng.integers(-128, 128, (2 ** 16, 256), dtype=np.int8)
    assert np.array_equal(crt.gemm_i8_i32(a, b), orc.i8_product(a, b))


# ------------------------------------------------------- K3: Karatsuba mod product
# 241, 233, 197, 173 have a square root of -1: the split (2-product) form
@pytest.mark.parametrize("p", [256, 255, 251, 241, 239, 233, 199, 197, 173])
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (40, 33, 70), (256, 512, 384), (131, 260, 1000)])
def test_complex_gemm_mod(crt, p, m, n, k):
    rng = np.random.default_rng(p + m + n + k)
    lo, hi = (-(p // 2), p - 1 - p // 2) if p % 2 == 0 else (-((p - 1) // 2), (p - 1) // 2)
    ar, ai = (rng.integers(lo, hi + 1, (m, k)).astype(np.int8) for _ in range(2))
    br, bi = (rng.integers(lo, hi + 1, (k, n)).astype(np.int8) for _ in range(2))
    er, ei = crt.complex_gemm_mod(ar, ai, br, bi, p)
    xr, xi = orc.karatsuba_mod(ar, ai, br, bi, p)
    assert np.array_equal(er, xr) and np.array_equal(ei, xi)


def test_complex_gemm_mod_hand_case(crt):
    # (1+2i)(3+4i) = -5+10i (reference tests/test_kernel.py:58-66)
    er, ei = crt.complex_gemm_mod([[1]], [[2]], [[3]], [[4]], 251)
    assert int(er[0, 0]) == -5 and int(ei[0, 0]) == 10


def test_complex_gemm_mod_split_hand_case(crt):
    # split modulus 241 (j = 64): (1+2i)(3+4i) = -5+10i, and a sum over k
    er, ei = crt.complex_gemm_mod([[1]], [[2]], [[3]], [[4]], 241)
    assert int(er[0, 0]) == -5 and int(ei[0, 0]) == 10
    ar, ai = np.array([[120, -120]], np.int8), np.array([[-120, 7]], np.int8)
    br, bi = np.array([[120], [-3]], np.int8), np.array([[120], [-120]], np.int8)
    er, ei = crt.complex_gemm_mod(ar, ai, br, bi, 241)
    xr, xi = orc.karatsuba_mod(ar, ai, br, bi, 241)
    assert np.array_equal(er, xr) and np.array_equal(ei, xi)


def test_split_moduli_equal_karatsuba_form(crt, tmp_path):
    """The split (2-product) form for moduli with sqrt(-1) and the 3-product
    Karatsuba form give bit-identical results (CRTG_SPLIT=0 forces the latter)."""
    import subprocess
    import sys
    code = (
        "import numpy as np, hashlib, sys\n"
        "sys.path.insert(0, '.')\n"
        "import paper_2512_08321_b200 as crt\n"
        "from oracle import ozaki2 as orc\n"
        "out = []\n"
        "for prec, N, mode in (('double', 20, 'fast'), ('double', 16, 'accurate'), ('single', 8, 'fast')):\n"
        "    a = orc.gen_matrix(300, 700, 1.0, 3, prec); b = orc.gen_matrix(700, 520, 1.0, 4, prec)\n"
        "    cfg = crt.EmuConfig(precision=prec, domain='complex', mode=mode, num_moduli=N)\n"
        "    out.append(hashlib.sha256(crt.emulate_gemm_complex(a, b, cfg).tobytes()).hexdigest())\n"
        "print(' '.join(out))\n")
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("0", "1"):
        env = dict(os.environ, CRTG_SPLIT=flag)
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        res[flag] = r.stdout.strip().split()[-3:]
    assert res["0"] == res["1"]


@pytest.mark.parametrize("knob,values", [("CRTG_FORK", ("0", "1")),
                                         ("CRTG_GEMM", ("one", "wide"))])
def test_launch_knobs_bitwise_neutral(crt, knob, values):
    """Schedule choices are bitwise neutral: the forked B chain for small
    products (CRTG_FORK) and the 128x256 vs 256x256 K3 kernels (CRTG_GEMM),
    on shapes where the default picks the fork / the 128x256 kernel and one
    with k >= 8192 where it picks the wide kernel."""
    import os
    import subprocess
    import sys
    code = (
        "import hashlib, sys\n"
        "sys.path.insert(0, '.')\n"
        "import paper_2512_08321_b200 as crt\n"
        "from oracle import ozaki2 as orc\n"
        "out = []\n"
        "for m, k, n, N, mode in ((1024, 1024, 1100, 14, 'fast'), (1024, 1024, 1100, 14, 'accurate'),\n"
        "                         (256, 8192, 512, 15, 'fast')):\n"
        "    a = orc.gen_matrix(m, k, 0.5, 5, 'double'); b = orc.gen_matrix(k, n, 0.5, 6, 'double')\n"
        "    cfg = crt.EmuConfig(domain='complex', mode=mode, num_moduli=N)\n"
        "    out.append(hashlib.sha256(crt.emulate_gemm_complex(a, b, cfg).tobytes()).hexdigest())\n"
        "print(' '.join(out))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for v in values:
        env = dict(os.environ, **{knob: v})
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        res[v] = r.stdout.strip().split()[-3:]
    assert res[values[0]] == res[values[1]]


def test_complex_gemm_mod_full_range_k_cap(crt):
    # extreme residues at the complex k cap: int32 D-E would overflow without
    # reducing D, E, F first (reference kernel.py:46-50)
    p = 256
    k = 2 ** 16
    ar = np.full((2, k), -128, np.int8)
    ai = np.full((2, k), 127, np.int8)
    br = np.full((k, 256), -128, np.int8)
    bi = np.full((k, 256), -128, np.int8)
    er, ei = crt.complex_gemm_mod(ar, ai, br, bi, p)
    xr, xi = orc.karatsuba_mod(ar, ai, br, bi, p)
    assert np.array_equal(er, xr) and np.array_equal(ei, xi)


@pytest.mark.parametrize("p,j", [(241, 64), (173, 80)])
def test_complex_gemm_mod_split_extreme_k_cap(crt, p, j):
    # split modulus: U = V = -128 everywhere (re = -128 mod p, im = 0) so both
    # products reach k * 128^2 = 2^30 at the k cap
    assert (j * j + 1) % p == 0
    k = 2 ** 16
    v = np.int8(p - 128)
    ar = np.full((3, k), v, np.int8)
    ai = np.zeros((3, k), np.int8)
    br = np.full((k, 260), v, np.int8)
    bi = np.zeros((k, 260), np.int8)
    bi[5, :] = 3  # break the symmetry a little
    er, ei = crt.complex_gemm_mod(ar, ai, br, bi, p)
    xr, xi = orc.karatsuba_mod(ar, ai, br, bi, p)
    assert np.array_equal(er, xr) and np.array_equal(ei, xi)


@pytest.mark.parametrize("N", [15, 20])
def test_offset_residues_extreme_k_cap(crt, N):
    """The pipeline stores residues as ((a' + 128) mod p) - 128, so a' = -128 gives
    -128 in EVERY modulus plane.  With injected exponents 0 and k = 2^16 every
    Karatsuba / split product reaches k * 128^2 = 2^30.  (The CRT is accurate
    relative to P, not exact for such a small product, so the check is against
    the oracle on the same exponents.)"""
    from paper_2512_08321_b200 import dist
    k, m, n = 2 ** 16, 2, 3
    a = np.full((m, k), complex(-128, -128))
    b = np.full((k, n), complex(-128, -127))
    b[7, 1] = complex(-128, 5)
    mu, nu = np.zeros(m, np.int32), np.zeros(n, np.int32)
    dev = torch.device("cuda")
    cfg = crt.EmuConfig(precision="double", domain="complex", mode="fast", num_moduli=N)
    out = dist.tile_with_exponents(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev),
                                   torch.from_numpy(mu).to(dev), torch.from_numpy(nu).to(dev), cfg)
    want = orc.emulate_complex_exps(a, b, mu, nu, N, "double")
    assert out.cpu().numpy().tobytes() == want.tobytes()


# ------------------------------------------------------------------ K1: scaling
def test_scaling_vs_golden(crt, golden):
    for tag in _cases(golden):
        a, b, N, prec, mode, g = _case_inputs(golden, tag)
        ms = crt.select_moduli(N)
        fn = crt.fast_scaling if mode == "fast" else crt.accurate_scaling
        diag = {}
        sv = fn(a, b, ms, None, diag)
        assert np.array_equal(sv.mu_exp, g("mu")), tag
        assert np.array_equal(sv.nu_exp, g("nu")), tag
        assert [diag.get("clamped_mu", 0), diag.get("clamped_nu", 0)] == g("diag").tolist()


@pytest.mark.parametrize("k", [7, 127, 129, 1000, 4100, 70001])
def test_fast_exponents_long_rows(crt, golden, k):
    a = orc.gen_matrix(3, k, 4.0, 100 + k)
    b = orc.gen_matrix(k, 2, 4.0, 200 + k)
    sv = crt.fast_scaling(a, b, crt.select_moduli(14))
    assert np.array_equal(sv.mu_exp, golden[f"pw_{k}__mu"])
    assert np.array_equal(sv.nu_exp, golden[f"pw_{k}__nu"])


def test_fast_exponents_random_rows(crt):
    # pairwise order stress: wide dynamic range, odd lengths
    for k in (9, 136, 250, 1023, 5000, 16384):
        rng = np.random.default_rng(k)
        a = (rng.standard_normal((33, k)) * np.exp(rng.standard_normal((33, k)) * 6)
             + 1j * rng.standard_normal((33, k)) * np.exp(rng.standard_normal((33, k)) * 6))
        b = (rng.standard_normal((k, 7)) * np.exp(rng.standard_normal((k, 7)) * 6)
             + 1j * rng.standard_normal((k, 7)))
        sv = crt.fast_scaling(a, b, crt.select_moduli(17))
        mu, nu = orc.exponents(a, b, 17, "fast")
        assert np.array_equal(sv.mu_exp, mu) and np.array_equal(sv.nu_exp, nu), k


# ------------------------------------------------------------------ K2: residues
def test_residues_vs_golden(crt, golden):
    for tag in _cases(golden):
        a, b, N, prec, mode, g = _case_inputs(golden, tag)
        ms = crt.select_moduli(N)
        ra = crt.quantized_residues(a, g("mu"), ms, axis=0)
        rb = crt.quantized_residues(b, g("nu"), ms, axis=1)
        assert np.array_equal(ra[:, 0], g("ar")) and np.array_equal(ra[:, 1], g("ai")), tag
        assert np.array_equal(rb[:, 0], g("br")) and np.array_equal(rb[:, 1], g("bi")), tag
        for idx, p in enumerate(ms.moduli):
            assert np.array_equal(ra[idx, 2], orc.sym_residue_int(
                g("ar")[idx].astype(np.int64) + g("ai")[idx], p)), tag


def test_residues_wide_values(crt):
    # |a'| up to 2^89 (N = 20 budgets reach 2^77; the reference allows < 2^90)
    rng = np.random.default_rng(1)
    x = (rng.standard_normal((40, 300)) + 1j * rng.standard_normal((40, 300)))
    exps = rng.integers(0, 87, 40)
    ms = crt.select_moduli(20)
    got = crt.quantized_residues(x, exps, ms, axis=0)
    ar = orc.truncate(np.ascontiguousarray(x.real), exps, 0)
    ai = orc.truncate(np.ascontiguousarray(x.imag), exps, 0)
    assert np.array_equal(got[:, 0], orc.residues(ar, orc.pick_moduli(20)))
    assert np.array_equal(got[:, 1], orc.residues(ai, orc.pick_moduli(20)))


def test_residues_overflow_is_domain_error(crt):
    x = np.full((2, 3), 1.5 + 0j)
    with pytest.raises(crt.DomainError):
        crt.quantized_residues(x, np.array([90, 0]), crt.select_moduli(14), axis=0)


# --------------------------------------------------------------------- K4: CRT
def test_crt_vs_golden(crt, golden):
    for tag in _cases(golden):
        a, b, N, prec, mode, g = _case_inputs(golden, tag)
        c = crt.crt_reconstruct(g("er"), g("ei"), g("mu"), g("nu"), crt.select_moduli(N), prec)
        assert c.tobytes() == g("c").tobytes(), tag


# ------------------------------------------------------------ end to end
def test_emulate_small_golden(crt, golden):
    for tag in _cases(golden):
        a, b, N, prec, mode, g = _case_inputs(golden, tag)
        cfg = crt.EmuConfig(precision=prec, domain="complex", mode=mode, num_moduli=N)
        diag = {}
        c = crt.emulate_gemm_complex(a, b, cfg, diag)
        assert c.dtype == g("c").dtype, tag
        assert c.tobytes() == g("c").tobytes(), tag
        assert [diag.get("clamped_mu", 0), diag.get("clamped_nu", 0)] == g("diag").tolist()


@pytest.mark.parametrize("tag", ["cfg1_z1024_fast14", "cfg1_z1024_accu14", "z512_fast20_phi4",
                                 "z384_accu17_phi2", "c512_fast6_phi0", "c512_fast10_phi1",
                                 "c512_accu8_phi1", "z_skinny_fast14", "z_ragged_fast13"])
def test_emulate_hash_golden(crt, golden_hashes, tag):
    h = golden_hashes[tag]
    a = orc.gen_matrix(h["m"], h["k"], h["phi"], h["seed"], h["precision"])
    b = orc.gen_matrix(h["k"], h["n"], h["phi"], h["seed"] + 1, h["precision"])
    assert _sha(a) == h["a_sha"] and _sha(b) == h["b_sha"]
    cfg = crt.EmuConfig(precision=h["precision"], domain="complex", mode=h["mode"],
                        num_moduli=h["N"])
    c = crt.emulate_gemm_complex(a, b, cfg)
    assert _sha(c) == h["c_sha"], (c.reshape(-1)[:4], h["c_head"])


def test_torch_inputs_and_n_block_invariance(crt):
    a = orc.gen_matrix(300, 700, 1.0, 31)
    b = orc.gen_matrix(700, 900, 1.0, 32)
    ref = orc.emulate_complex(a, b, 14)
    ta = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    tb = torch.from_numpy(np.ascontiguousarray(b)).cuda()
    for nb in (1, 256, 300, 8192):
        cfg = crt.EmuConfig(domain="complex", n_block=nb)
        c = crt.emulate_gemm_complex(ta, tb, cfg)
        assert isinstance(c, torch.Tensor) and c.is_cuda
        assert c.cpu().numpy().tobytes() == ref.tobytes(), nb


def test_conjugate_symmetry_and_integer_inputs(crt):
    a = orc.gen_matrix(64, 96, 2.0, 40)
    b = orc.gen_matrix(96, 80, 2.0, 41)
    cfg = crt.EmuConfig(domain="complex")
    c1 = crt.emulate_gemm_complex(a, b, cfg)
    c2 = crt.emulate_gemm_complex(np.conj(a), np.conj(b), cfg)
    assert np.array_equal(c1, np.conj(c2))
    ai = np.round(a * 50)
    bi = np.round(b * 50)
    ci = crt.emulate_gemm_complex(ai, bi, cfg)
    assert np.array_equal(ci, ai @ bi)


def test_errors(crt):
    cfg = crt.EmuConfig(domain="complex")
    a = np.ones((4, 5), complex)
    bad = a.copy()
    bad[1, 2] = np.nan
    with pytest.raises(crt.DomainError):
        crt.emulate_gemm_complex(bad, np.ones((5, 3), complex), cfg)
    with pytest.raises(crt.DomainError):
        crt.emulate_gemm_complex(a, np.full((5, 3), np.inf + 0j), cfg)
    with pytest.raises(crt.DimensionError):
        crt.emulate_gemm_complex(a, np.ones((4, 3), complex), cfg)
    with pytest.raises(crt.DimensionError):
        crt.emulate_gemm_complex(np.ones((1, 2 ** 16 + 1)), np.ones((2 ** 16 + 1, 1)), cfg)
    with pytest.raises(crt.ConfigError):
        crt.emulate_gemm_complex(a, np.ones((5, 3)), crt.EmuConfig(domain="real"))


def test_zero_rows_and_accurate_zero_b(crt):
    a = orc.gen_matrix(20, 30, 1.0, 50)
    b = orc.gen_matrix(30, 10, 1.0, 51)
    a[3] = 0
    b[:, 4] = 0
    for mode in ("fast", "accurate"):
        cfg = crt.EmuConfig(domain="complex", mode=mode)
        c = crt.emulate_gemm_complex(a, b, cfg)
        ref = orc.emulate_complex(a, b, None, mode)
        assert c.tobytes() == ref.tobytes(), mode
    # accurate mode with B == 0 and A != 0: mu = 1023 -> DomainError (reference behaviour)
    with pytest.raises(crt.DomainError):
        crt.emulate_gemm_complex(a, np.zeros((30, 10), complex),
                                 crt.EmuConfig(domain="complex", mode="accurate"))


def test_blas_gemm_colmajor(crt):
    m, n, k = 7, 5, 9
    rng = np.random.default_rng(8)
    lda, ldb, ldc = 10, 12, 8
    a = rng.standard_normal(lda * k) + 1j * rng.standard_normal(lda * k)
    b = rng.standard_normal(ldb * n) + 1j * rng.standard_normal(ldb * n)
    c = np.zeros(ldc * n, complex)
    out = crt.gemm("complex", "double", m, n, k, a, lda, b, ldb, c, ldc)
    av = a[:lda * k].reshape((lda, k), order="F")[:m]
    bv = b[:ldb * n].reshape((ldb, n), order="F")[:k]
    ref = orc.emulate_complex(av, bv, 14)
    assert out is c
    assert np.array_equal(c.reshape((ldc, n), order="F")[:m], ref)
    assert np.all(c.reshape((ldc, n), order="F")[m:] == 0)


# ------------------------------------------------------- full-size properties
def test_subblock_parity_large(crt):
    """Fast mode is row/column local: a block of the 4096^3 product equals the
    emulation of the corresponding slabs, which the oracle can afford."""
    m = n = k = 4096
    a = orc.gen_matrix(m, k, 0.5, 60)
    b = orc.gen_matrix(k, n, 0.5, 61)
    cfg = crt.EmuConfig(domain="complex")
    c = crt.emulate_gemm_complex(a, b, cfg)
    rows = slice(1000, 1064)
    cols = slice(3000, 3048)
    ref = orc.emulate_complex(a[rows], b[:, cols], 14)
    assert c[rows, cols].tobytes() == ref.tobytes()
    # and the last ragged corner
    ref2 = orc.emulate_complex(a[-5:], b[:, -7:], 14)
    assert c[-5:, -7:].tobytes() == ref2.tobytes()


@pytest.mark.parametrize("mode", ["fast", "accurate"])
@pytest.mark.parametrize("shape", [(4352, 4608, 300), (4100, 300, 260), (300, 8300, 129),
                                   (4100, 260, 1100)])  # A = 72 MB: page-locked in place
def test_host_streaming_equals_device_path(crt, mode, shape):
    """crtg_gemm_complex_host (numpy in/out, A row chunks x B column blocks
    streamed in a staircase over the copy engines) is bitwise the device path,
    including ragged last chunks / blocks."""
    m, n, k = shape
    rng = np.random.default_rng(m + n + k)
    a = (rng.standard_normal((m, k)) * np.exp(rng.standard_normal((m, k)))
         + 1j * rng.standard_normal((m, k)))
    b = (rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))
         * np.exp(rng.standard_normal((k, n))))
    cfg = crt.EmuConfig(domain="complex", mode=mode, num_moduli=13)
    host = crt.emulate_gemm_complex(a, b, cfg)  # numpy -> streamed host path
    dev = crt.emulate_gemm_complex(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), cfg)
    assert isinstance(host, np.ndarray)
    assert host.tobytes() == dev.cpu().numpy().tobytes()
    # spot-check a sub-block against the oracle (fast mode is row/column local)
    if mode == "fast":
        want = orc.emulate_complex(a[-37:], b[:, -41:], 13, "fast")
        assert host[-37:, -41:].tobytes() == want.tobytes()


@pytest.mark.parametrize("prec,N", [("single", 8), ("double", 20)])
def test_host_streaming_single_and_wide_moduli(crt, prec, N):
    """Host-streaming entry with complex64 inputs (single precision) and with
    N = 20 (7 split moduli, wide residue limbs at phi = 4), 16-piece staircase
    with ragged last pieces: bitwise the device path."""
    m, n, k = 4100, 4352, 700
    rng = np.random.default_rng(N)
    dt = np.complex64 if prec == "single" else np.complex128
    a = (rng.standard_normal((m, k)) * np.exp(4 * rng.standard_normal((m, k)))
         + 1j * rng.standard_normal((m, k))).astype(dt)
    b = (rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))).astype(dt)
    cfg = crt.EmuConfig(precision=prec, domain="complex", mode="fast", num_moduli=N)
    host = crt.emulate_gemm_complex(a, b, cfg)
    dev = crt.emulate_gemm_complex(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), cfg)
    assert host.dtype == dev.cpu().numpy().dtype
    assert host.tobytes() == dev.cpu().numpy().tobytes()
    want = orc.emulate_complex(a[:33], b[:, -29:], N, "fast", prec)
    assert host[:33, -29:].tobytes() == want.tobytes()


def test_host_pinned_and_staged_paths_agree(crt):
    """The host entry streams pinned (page-locked) operands directly and
    pageable ones through its pinned staging ring: both are bitwise the device
    path (ragged pieces, 16-piece staircase)."""
    m, n, k = 4300, 4200, 500
    rng = np.random.default_rng(11)
    a = rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))
    b = rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))
    cfg = crt.EmuConfig(domain="complex", mode="fast", num_moduli=14)
    staged = crt.emulate_gemm_complex(a, b, cfg)                       # numpy: staged
    ta = torch.from_numpy(a).pin_memory()
    tb = torch.from_numpy(b).pin_memory()
    pinned = crt.emulate_gemm_complex(ta, tb, cfg)                     # pinned: direct
    dev = crt.emulate_gemm_complex(ta.cuda(), tb.cuda(), cfg)
    assert staged.tobytes() == pinned.numpy().tobytes() == dev.cpu().numpy().tobytes()


# ------------------------------------------------------- every modulus count
@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("N", list(range(1, 21)))
def test_every_modulus_count_fast(crt, prec, N):
    """Each N has its own CRT kernel instantiation (k_crt_n<N>, two CTAs per SM
    above 16) and its own mix of Karatsuba / split moduli: all 20 counts, both
    precisions, against the oracle at a shape with ragged rows and K (reference
    emulate.py:193-240)."""
    a = orc.gen_matrix(37, 300, 1.0, 100 + N, prec)
    b = orc.gen_matrix(300, 45, 1.0, 200 + N, prec)
    cfg = crt.EmuConfig(precision=prec, domain="complex", mode="fast", num_moduli=N)
    got = crt.emulate_gemm_complex(a, b, cfg)
    want = orc.emulate_complex(a, b, N, "fast", prec)
    assert got.dtype == want.dtype and got.tobytes() == want.tobytes()


@pytest.mark.parametrize("N", [2, 5, 9, 11, 18, 19])
def test_modulus_counts_accurate_large_tiles(crt, N):
    """Accurate mode and a product large enough for the 256x256-tile GEMM and
    several residue tiles per CTA, for modulus counts the goldens skip."""
    a = orc.gen_matrix(300, 1100, 2.0, 300 + N, "double")
    b = orc.gen_matrix(1100, 260, 2.0, 400 + N, "double")
    for mode in ("fast", "accurate"):
        cfg = crt.EmuConfig(precision="double", domain="complex", mode=mode, num_moduli=N)
        got = crt.emulate_gemm_complex(a, b, cfg)
        want = orc.emulate_complex(a, b, N, mode, "double")
        assert got.tobytes() == want.tobytes(), mode


def _fuzz_cases(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        m, n, k = (int(x) for x in rng.integers(1, 700, 3))
        out.append((i, m, n, k, int(rng.integers(1, 21)), ["fast", "accurate"][i % 2],
                    ["double", "single"][(i // 2) % 2], float(rng.choice([0.5, 1.0, 2.0, 4.0]))))
    return out


@pytest.mark.parametrize("case", _fuzz_cases(24, 2026), ids=lambda c: f"fuzz{c[0]}")
def test_random_shapes_modes_precisions(crt, case):
    """Seeded sweep over ragged shapes (every extent 1..699, so partial residue
    tiles, partial 128/256-row GEMM tiles and odd CRT column counts), modulus
    counts 1..20, both modes, both precisions and exponent spreads phi, each
    compared bit for bit with the oracle (reference emulate.py:193-240)."""
    i, m, n, k, N, mode, prec, phi = case
    a = orc.gen_matrix(m, k, phi, 1000 + i, prec)
    b = orc.gen_matrix(k, n, phi, 2000 + i, prec)
    cfg = crt.EmuConfig(precision=prec, domain="complex", mode=mode, num_moduli=N)
    got = crt.emulate_gemm_complex(a, b, cfg)
    want = orc.emulate_complex(a, b, N, mode, prec)
    assert got.dtype == want.dtype and got.shape == want.shape
    assert got.tobytes() == want.tobytes(), f"{int(np.count_nonzero(got != want))} mismatches"
