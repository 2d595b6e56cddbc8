"""Fast-mode exponents at the edges of the double range (K1 single-pass kernels).

k_row_stats / k_col_stats sum UNSCALED squares in the reference's order and
apply 2^-2fl once, which is bit-exact only while every square stays normal and
no sum overflows; rows / columns outside that range take the two-pass fallback.
These cases put rows and columns on both sides of the boundary — huge (2^600 ..
2^1000), tiny (2^-600 .. 2^-1000), subnormal, a wide dynamic range inside one
row, zero rows — and compare against the oracle (complex exponents through
`fast_scaling`, real results through `emulate_gemm_real` in all four layouts,
which routes each operand through the row or the column kernel).
"""

import numpy as np
import pytest

from oracle import ozaki2 as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def crt():
    import paper_2512_08321_b200 as crt
    return crt


SCALES = [0, 600, -600, 1000, -1000, 40, -40, 500, -511, -512, 480]


def edgy(rows, cols, seed, cplx, axis):
    """Matrix whose lines along `axis` (0 = rows, 1 = columns) span the range."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((rows, cols))
    if cplx:
        x = x + 1j * rng.standard_normal((rows, cols))
    nl = rows if axis == 0 else cols
    sc = np.array([SCALES[i % len(SCALES)] for i in range(nl)], float)
    x = x * (np.exp2(sc)[:, None] if axis == 0 else np.exp2(sc)[None, :])
    # wide dynamic range inside some lines, subnormals, a zero line, a lone value
    line = (lambda i: x[i]) if axis == 0 else (lambda i: x[:, i])
    if nl > 3:
        v = line(1)
        v[::3] *= 2.0 ** -700
        v = line(2)
        v[::5] = 5e-324
        line(3)[:] = 0
    if nl > 5:
        v = line(5)
        v[:] = 0
        v[len(v) // 2] = 2.0 ** -1070
    return x


@pytest.mark.parametrize("k", [5, 129, 1000, 4099])
def test_complex_fast_exponents_extreme(crt, k):
    a = edgy(23, k, k, True, 0)
    b = edgy(k, 19, k + 1, True, 1)
    ms = crt.select_moduli(14)
    diag = {}
    sv = crt.fast_scaling(a, b, ms, None, diag)
    odiag = {}
    mu, nu = orc.exponents(a, b, 14, "fast", odiag)
    assert np.array_equal(sv.mu_exp, mu)
    assert np.array_equal(sv.nu_exp, nu)
    assert diag.get("clamped_mu", 0) == odiag.get("clamped_mu", 0)
    assert diag.get("clamped_nu", 0) == odiag.get("clamped_nu", 0)


def test_complex64_fast_exponents_extreme(crt):
    rng = np.random.default_rng(5)
    a = (rng.standard_normal((17, 300)) * np.exp2(rng.integers(-120, 120, (17, 1)))).astype(np.float32)
    b = (rng.standard_normal((300, 11)) * np.exp2(rng.integers(-120, 120, (1, 11)))).astype(np.float32)
    a = (a + 1j * a[::-1]).astype(np.complex64)
    b = (b + 1j * 1e-45).astype(np.complex64)
    sv = crt.fast_scaling(a, b, crt.select_moduli(7))
    mu, nu = orc.exponents(a.astype(np.complex128), b.astype(np.complex128), 7, "fast")
    assert np.array_equal(sv.mu_exp, mu) and np.array_equal(sv.nu_exp, nu)


@pytest.mark.parametrize("la,lb", [("C", "C"), ("F", "F"), ("C", "F"), ("F", "C")])
def test_real_fast_extreme_all_layouts(crt, la, lb):
    m, n, k = 29, 31, 777
    a = np.asarray(edgy(m, k, 3, False, 0), order=la)
    b = np.asarray(edgy(k, n, 4, False, 1), order=lb)
    cfg = crt.EmuConfig(mode="fast", num_moduli=14)
    got = crt.emulate_gemm_real(a, b, cfg)
    want = orc.emulate_real(a, b, 14, "fast")
    assert got.tobytes() == want.tobytes()


def test_unaligned_leading_dimension_path(crt):
    """complex64 B with an odd leading dimension is not 16-byte aligned per row:
    the two-pass column kernels run instead of the cp.async one."""
    rng = np.random.default_rng(9)
    full = (rng.standard_normal((300, 13)) + 1j * rng.standard_normal((300, 13))).astype(np.complex64)
    bt = torch.from_numpy(full).cuda()[:, :11]  # row stride 13 complex64 = 104 bytes
    a = (rng.standard_normal((9, 300)) + 1j * rng.standard_normal((9, 300))).astype(np.complex64)
    cfg = crt.EmuConfig(precision="single", domain="complex", num_moduli=8)
    got = crt.emulate_gemm_complex(torch.from_numpy(a).cuda(), bt, cfg).cpu().numpy()
    want = orc.emulate_complex(a, full[:, :11], 8, "fast", "single")
    assert got.tobytes() == want.tobytes()


def key_edge_columns(k, n, seed):
    """Columns at the edges of k_col_stats' integer keys (high word of |x|, bit 0
    set for a nonzero low word): equal high words with different low words,
    2^500 exactly and one ulp above, 2^-511 exactly and one ulp below, columns
    whose nonzeros are all below 2^-1042 (key 1: exponent only in the low
    word), a lone NaN-free huge value, and ordinary columns in between."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))
    ulp_up = lambda v: np.nextafter(v, np.inf)  # noqa: E731
    ulp_dn = lambda v: np.nextafter(v, 0.0)  # noqa: E731
    x[:, 0] = 2.0 ** 500
    x[7, 1] = ulp_up(2.0 ** 500)
    x[:, 1] = np.where(np.arange(k) == 7, x[7, 1], 1.0)
    x[:, 2] = 2.0 ** -511
    x[3, 2] = 1.0
    x[:, 3] = 1.0
    x[5, 3] = ulp_dn(2.0 ** -511)
    x[:, 4] = 0.0
    x[::7, 4] = 2.0 ** -1060
    x[1, 4] = 2.0 ** -1065 + 2.0 ** -1070
    x[:, 5] = 0.0
    x[9, 5] = 5e-324 * 3
    x[:, 6] = (1.0 + 2.0 ** -40) * (1 + 1j)  # high words equal, low words differ
    x[11, 6] = 1.0 + 2.0 ** -52
    x[:, 8] = x[:, 8].real * 2.0 ** -1030 + 1j * x[:, 8].imag * 2.0 ** -1010  # subnormal mix
    x[:, 9] = 0.0
    x[0, 9] = 1j * 2.0 ** -1050
    return x


@pytest.mark.parametrize("k,n", [(200, 40), (64, 16), (1000, 33)])
def test_col_stats_key_edges(crt, k, n):
    b = key_edge_columns(k, n, k + n)
    a = np.random.default_rng(1).standard_normal((5, k)) + 0j
    ms = crt.select_moduli(14)
    diag, odiag = {}, {}
    sv = crt.fast_scaling(a, b, ms, None, diag)
    mu, nu = orc.exponents(a, b, 14, "fast", odiag)
    assert np.array_equal(sv.nu_exp, nu)
    assert np.array_equal(sv.mu_exp, mu)
    assert diag.get("clamped_nu", 0) == odiag.get("clamped_nu", 0)
