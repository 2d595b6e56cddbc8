"""GPU: the real-domain path (emulate_gemm_real, reference emulate.py:169-190;
SURVEY §8f rank 2) — bit-exact against the reference's golden vectors and the
oracle, including numpy's layout-dependent summation order, plus the reference's
own real-emulation tests (tests/test_emulate.py:52-117 there) restated."""

import hashlib

import numpy as np
import pytest

from oracle import ozaki2 as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def crt():
    import paper_2512_08321_b200 as crt
    return crt


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_real_small_golden(crt, golden):
    tags = sorted({k.split("__")[0] for k in golden.files if k.endswith("__rmeta")})
    assert tags
    for tag in tags:
        g = lambda s: golden[f"{tag}__{s}"]  # noqa: E731
        m, n, k, seed, N, dbl, fast = g("rmeta").tolist()
        prec, mode = ("double" if dbl else "single"), ("fast" if fast else "accurate")
        a = orc.gen_matrix(m, k, float(g("phi")), seed, prec, "real")   # Fortran order
        b = orc.gen_matrix(k, n, float(g("phi")), seed + 1, prec, "real")
        diag = {}
        c = crt.emulate_gemm_real(a, b, crt.EmuConfig(precision=prec, mode=mode, num_moduli=N),
                                  diag)
        assert c.dtype == g("c").dtype and c.tobytes() == g("c").tobytes(), tag
        assert [diag.get("clamped_mu", 0), diag.get("clamped_nu", 0)] == g("diag").tolist()


@pytest.mark.parametrize("tag", ["real512_fast15", "real384_accu15", "real512_fast8s",
                                 "real_k2pow17_fast"])
def test_real_hash_golden(crt, golden_hashes, tag):
    h = golden_hashes[tag]
    a = orc.gen_matrix(h["m"], h["k"], h["phi"], h["seed"], h["precision"], "real")
    b = orc.gen_matrix(h["k"], h["n"], h["phi"], h["seed"] + 1, h["precision"], "real")
    c = crt.emulate_gemm_real(a, b, crt.EmuConfig(precision=h["precision"], mode=h["mode"],
                                                  num_moduli=h["N"]))
    assert _sha(c) == h["c_sha"], (c.reshape(-1)[:4], h["c_head"])


@pytest.mark.parametrize("la,lb", [("C", "C"), ("F", "F"), ("C", "F"), ("F", "C")])
@pytest.mark.parametrize("mode", ["fast", "accurate"])
def test_real_layouts_follow_numpy_order(crt, la, lb, mode):
    """Layout decides numpy's reduction order for real operands; both must match."""
    rng = np.random.default_rng(7)
    m, n, k = 70, 90, 3000
    a = np.asarray(rng.standard_normal((m, k)) * np.exp(rng.standard_normal((m, k)) * 5), order=la)
    b = np.asarray(rng.standard_normal((k, n)) * np.exp(rng.standard_normal((k, n)) * 5), order=lb)
    cfg = crt.EmuConfig(mode=mode, num_moduli=16)
    got = crt.emulate_gemm_real(a, b, cfg)
    want = orc.emulate_real(a, b, 16, mode)
    assert got.tobytes() == want.tobytes()
    # strided views too
    a2, b2 = a[::2, 1:], b[1:, ::3]
    assert crt.emulate_gemm_real(a2, b2, cfg).tobytes() == orc.emulate_real(a2, b2, 16, mode).tobytes()


def test_real_vector_shapes(crt):
    rng = np.random.default_rng(3)
    for (m, k, n) in [(1, 500, 7), (6, 500, 1), (1, 300, 1), (5, 1, 4)]:
        a = rng.standard_normal((m, k)) * 3
        b = rng.standard_normal((k, n)) * 3
        for cfg in (crt.EmuConfig(num_moduli=15), crt.EmuConfig(mode="accurate", num_moduli=15)):
            got = crt.emulate_gemm_real(a, b, cfg)
            want = orc.emulate_real(a, b, 15, cfg.mode)
            assert got.tobytes() == want.tobytes(), (m, k, n, cfg.mode)


# ---- restated from the reference's TestRealEmulation ----
@pytest.mark.parametrize("mode", ["fast", "accurate"])
@pytest.mark.parametrize("num_moduli", [2, 8, 15, 20])
def test_identity_exact(crt, mode, num_moduli):
    eye = np.eye(4)
    assert np.array_equal(crt.emulate_gemm_real(eye, eye, crt.EmuConfig(mode=mode,
                                                                          num_moduli=num_moduli)), eye)


@pytest.mark.parametrize("mode", ["fast", "accurate"])
def test_integer_inputs_bitwise_exact(crt, mode):
    rng = np.random.default_rng(2)
    a = rng.integers(-1000, 1000, (9, 31)).astype(np.float64)
    b = rng.integers(-1000, 1000, (31, 7)).astype(np.float64)
    got = crt.emulate_gemm_real(a, b, crt.EmuConfig(mode=mode, num_moduli=8))
    assert np.array_equal(got, a @ b)


def test_single_precision_output(crt):
    a = orc.gen_matrix(16, 64, 0.5, 3, "single", "real")
    b = orc.gen_matrix(64, 12, 0.5, 4, "single", "real")
    cfg = crt.EmuConfig(precision="single", mode="accurate", num_moduli=7)
    got = crt.emulate_gemm_real(a, b, cfg)
    assert got.dtype == np.float32
    assert got.tobytes() == orc.emulate_real(a, b, 7, "accurate", "single").tobytes()


def test_block_width_bitwise_invariant(crt):
    a = orc.gen_matrix(40, 300, 1.0, 5, "double", "real")
    b = orc.gen_matrix(300, 700, 1.0, 6, "double", "real")
    outs = [crt.emulate_gemm_real(a, b, crt.EmuConfig(num_moduli=10, n_block=nb))
            for nb in (1, 256, 8192)]
    assert all(o.tobytes() == outs[0].tobytes() for o in outs)


def test_real_errors(crt):
    with pytest.raises(crt.DomainError):
        crt.emulate_gemm_real(np.array([[np.nan, 1.0], [1.0, 1.0]]), np.ones((2, 2)),
                              crt.EmuConfig(num_moduli=4))
    with pytest.raises(crt.DomainError):
        crt.emulate_gemm_real(np.ones((2, 2), complex), np.ones((2, 2)), crt.EmuConfig(num_moduli=4))
    with pytest.raises(crt.DimensionError):
        crt.emulate_gemm_real(np.ones((2, 3)), np.ones((2, 2)), crt.EmuConfig(num_moduli=4))
    with pytest.raises(crt.ConfigError):
        crt.emulate_gemm_real(np.ones((2, 2)), np.ones((2, 2)), crt.EmuConfig(domain="complex"))
    with pytest.raises(crt.DimensionError):
        crt.emulate_gemm_real(np.ones((1, 2 ** 17 + 1)), np.ones((2 ** 17 + 1, 1)),
                              crt.EmuConfig(num_moduli=4))
    with pytest.raises(crt.DimensionError):
        crt.emulate_gemm_real(np.ones((1, 2 ** 16 + 1)), np.ones((2 ** 16 + 1, 1)),
                              crt.EmuConfig(mode="accurate", num_moduli=4))


def test_blas_gemm_real_leading_dims(crt):
    # reference tests/test_emulate.py:219-235: flat column-major buffers
    rng = np.random.default_rng(4)
    m, n, k, lda, ldb, ldc = 5, 4, 6, 7, 8, 9
    a_buf = rng.standard_normal(lda * k)
    b_buf = rng.standard_normal(ldb * n)
    c_buf = np.zeros(ldc * n)
    out = crt.gemm("real", "double", m, n, k, a_buf, lda, b_buf, ldb, c_buf, ldc,
                   crt.EmuConfig(num_moduli=8))
    a_mat = a_buf.reshape((lda, k), order="F")[:m]
    b_mat = b_buf.reshape((ldb, n), order="F")[:k]
    want = orc.emulate_real(a_mat, b_mat, 8)
    assert out is c_buf
    assert np.array_equal(c_buf.reshape((ldc, n), order="F")[:m], want)


def test_real_torch_inputs(crt):
    a = torch.randn(100, 333, dtype=torch.float64, device="cuda")
    b = torch.randn(333, 77, dtype=torch.float64, device="cuda")
    got = crt.emulate_gemm_real(a, b, crt.EmuConfig())
    assert got.is_cuda and got.dtype == torch.float64
    want = orc.emulate_real(a.cpu().numpy(), b.cpu().numpy(), 15)
    assert got.cpu().numpy().tobytes() == want.tobytes()


def _fuzz_real(count, seed):
    rng = np.random.default_rng(seed)
    return [(i, *(int(x) for x in rng.integers(1, 700, 3)), int(rng.integers(1, 21)),
             ["fast", "accurate"][i % 2], ["double", "single"][(i // 2) % 2],
             float(rng.choice([0.5, 2.0, 4.0]))) for i in range(count)]


@pytest.mark.parametrize("case", _fuzz_real(16, 2027), ids=lambda c: f"fuzz{c[0]}")
def test_real_random_shapes(crt, case):
    """Seeded ragged shapes, modulus counts, modes and precisions for the real
    pipeline (EPI_REAL, reference emulate.py:169-190) against the oracle."""
    i, m, n, k, N, mode, prec, phi = case
    a = orc.gen_matrix(m, k, phi, 3000 + i, prec, domain="real")
    b = orc.gen_matrix(k, n, phi, 4000 + i, prec, domain="real")
    cfg = crt.EmuConfig(precision=prec, domain="real", mode=mode, num_moduli=N)
    got = crt.emulate_gemm_real(a, b, cfg)
    want = orc.emulate_real(a, b, N, mode, prec)
    assert got.dtype == want.dtype and got.tobytes() == want.tobytes()
