"""Pin the CPU oracle (oracle/ozaki2.py) to golden vectors produced by the
unmodified reference (tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import ozaki2 as orc


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_moduli_and_constants(golden):
    for n in range(1, 21):
        ms = orc.pick_moduli(n)
        assert ms.primes == tuple(golden[f"moduli_{n}"].tolist())
        assert np.array_equal(ms.coeff_hi, golden[f"coeff_hi_{n}"])
        assert np.array_equal(ms.coeff_lo, golden[f"coeff_lo_{n}"])
        assert str(ms.P) == str(golden[f"P_{n}"])
        pf, pa, d = orc.scale_thresholds(ms.P)
        assert np.array_equal(np.array([pf, pa, d], np.float32), golden[f"consts_{n}"])


def test_log2_upper(golden):
    y = orc.log2_up(golden["log2_x"])
    assert np.array_equal(y.view(np.int32), golden["log2_y"].view(np.int32))


def _cases(golden):
    return sorted({k.split("__")[0] for k in golden.files if k.endswith("__meta")})


def test_small_cases_every_stage(golden):
    for tag in _cases(golden):
        g = lambda s: golden[f"{tag}__{s}"]  # noqa: E731
        m, n, k, seed, N, dbl, fast = g("meta").tolist()
        phi = float(g("phi"))
        prec = "double" if dbl else "single"
        mode = "fast" if fast else "accurate"
        a = orc.gen_matrix(m, k, phi, seed, prec)
        b = orc.gen_matrix(k, n, phi, seed + 1, prec)
        assert _sha(a) == str(g("a_sha")) and _sha(b) == str(g("b_sha")), tag
        diag = {}
        c, st = orc.emulate_complex(a, b, N, mode, prec, diag, return_stages=True)
        assert np.array_equal(st["mu"], g("mu")), tag
        assert np.array_equal(st["nu"], g("nu")), tag
        for key in ("ar", "ai", "br", "bi", "er", "ei"):
            assert np.array_equal(st[key], g(key)), (tag, key)
        assert c.dtype == g("c").dtype
        assert c.tobytes() == g("c").tobytes(), tag
        assert [diag.get("clamped_mu", 0), diag.get("clamped_nu", 0)] == g("diag").tolist()


@pytest.mark.parametrize("k", [7, 127, 129, 1000, 4100, 70001])
def test_pairwise_row_exponents(golden, k):
    a = orc.gen_matrix(3, k, 4.0, 100 + k)
    b = orc.gen_matrix(k, 2, 4.0, 200 + k)
    mu, nu = orc.exponents(a, b, 14, "fast")
    assert np.array_equal(mu, golden[f"pw_{k}__mu"])
    assert np.array_equal(nu, golden[f"pw_{k}__nu"])


@pytest.mark.parametrize("tag", ["z512_fast20_phi4", "c512_fast6_phi0", "z384_accu17_phi2",
                                 "z_ragged_fast13", "c512_accu8_phi1"])
def test_hash_cases(golden_hashes, tag):
    h = golden_hashes[tag]
    a = orc.gen_matrix(h["m"], h["k"], h["phi"], h["seed"], h["precision"])
    b = orc.gen_matrix(h["k"], h["n"], h["phi"], h["seed"] + 1, h["precision"])
    assert _sha(a) == h["a_sha"] and _sha(b) == h["b_sha"]
    c, st = orc.emulate_complex(a, b, h["N"], h["mode"], h["precision"], return_stages=True)
    assert st["mu"].tolist() == h["mu"] and st["nu"].tolist() == h["nu"]
    assert _sha(c) == h["c_sha"]


def test_pairwise_tree_matches_numpy():
    rng = np.random.default_rng(3)
    for k in (1, 5, 8, 9, 128, 129, 136, 255, 1000, 16384, 65536, 70001):
        x = rng.standard_normal(k) * np.exp(rng.standard_normal(k) * 3)
        leaves = orc.pairwise_tree(k)
        assert sum(l for _, l in leaves) == k

        def leaf(s, ln):
            v = x[s:s + ln]
            if ln < 8:
                r = 0.0
                for t in v:
                    r += t
                return r
            r = list(v[:8])
            full = ln - ln % 8
            for i in range(8, full, 8):
                for j in range(8):
                    r[j] += v[i + j]
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            for i in range(full, ln):
                res += v[i]
            return res

        def rec(s, ln):
            if ln <= 128:
                return leaf(s, ln)
            h = ln // 2
            h -= h % 8
            return rec(s, h) + rec(s + h, ln - h)

        assert 0.0 + rec(0, k) == np.sum(x[None, :], axis=1)[0]


def _real_cases(golden):
    return sorted({k.split("__")[0] for k in golden.files if k.endswith("__rmeta")})


def test_real_small_cases_every_stage(golden):
    for tag in _real_cases(golden):
        g = lambda s: golden[f"{tag}__{s}"]  # noqa: E731
        m, n, k, seed, N, dbl, fast = g("rmeta").tolist()
        prec = "double" if dbl else "single"
        mode = "fast" if fast else "accurate"
        a = orc.gen_matrix(m, k, float(g("phi")), seed, prec, "real")
        b = orc.gen_matrix(k, n, float(g("phi")), seed + 1, prec, "real")
        assert _sha(a) == str(g("a_sha")) and _sha(b) == str(g("b_sha")), tag
        diag = {}
        c, st = orc.emulate_real(a, b, N, mode, prec, diag, return_stages=True)
        assert np.array_equal(st["mu"], g("mu")) and np.array_equal(st["nu"], g("nu")), tag
        for key in ("ra", "rb", "e"):
            assert np.array_equal(st[key], g(key)), (tag, key)
        assert c.dtype == g("c").dtype and c.tobytes() == g("c").tobytes(), tag
        assert [diag.get("clamped_mu", 0), diag.get("clamped_nu", 0)] == g("diag").tolist()


@pytest.mark.parametrize("tag", ["real512_fast15", "real384_accu15", "real512_fast8s",
                                 "real_k2pow17_fast"])
def test_real_hash_cases(golden_hashes, tag):
    h = golden_hashes[tag]
    a = orc.gen_matrix(h["m"], h["k"], h["phi"], h["seed"], h["precision"], "real")
    b = orc.gen_matrix(h["k"], h["n"], h["phi"], h["seed"] + 1, h["precision"], "real")
    assert _sha(a) == h["a_sha"] and _sha(b) == h["b_sha"]
    c = orc.emulate_real(a, b, h["N"], h["mode"], h["precision"])
    assert _sha(c) == h["c_sha"]


def test_dd_gemm_oracle(golden):
    tags = sorted({k.split("__")[0] for k in golden.files if k.endswith("__ddmeta")})
    assert tags
    for tag in tags:
        m, n, k, seed, cplx = golden[f"{tag}__ddmeta"].tolist()
        phi = float(golden[f"{tag}__phi"])
        dom = "complex" if cplx else "real"
        a = orc.gen_matrix(m, k, phi, seed, "double", dom)
        b = orc.gen_matrix(k, n, phi, seed + 1, "double", dom)
        hi, lo = orc.dd_gemm(a, b)
        assert hi.tobytes() == golden[f"{tag}__hi"].tobytes(), tag
        assert lo.tobytes() == golden[f"{tag}__lo"].tobytes(), tag
        err = orc.max_relative_error(golden[f"{tag}__approx"], hi, lo)
        assert err == float(golden[f"{tag}__err"][0]), tag
