"""GPU parity at the BENCHMARKED configurations (BASELINE.json configs 2-4), on
the benchmark's own inputs (bench.synth: (u - 0.5) * exp(z * phi) drawn on the
device), bit-exact against the CPU oracle.

The full products run on the GPU at full size; the oracle checks slabs of them:
* fast mode is row/column local (mu_i depends only on row i of A over all k,
  nu_j only on column j of B; reference scaling.py:174-213), so the block
  C[rows, cols] of the full product equals the oracle's emulation of
  A[rows, :] @ B[:, cols] -- a few seconds of CPU per slab;
* accurate mode's exponents are global (scaling.py:260-271): mu for the slab
  rows is checked against the oracle's bound product of those rows with ALL of
  B, nu for the slab columns against ALL of A with those columns, and the C
  slab against the oracle's pipeline with the GPU's (verified) exponents
  injected (emulate.py:213-240 after the scaling).
Slabs sit at the first / last rows and columns (largest plane offsets: int32
index overflows would show there), across the 8192-column n_block boundary
and across raster-group boundaries.

Needs a B200 (~60 GB of device memory at 16384^3) and ~4 GB of host memory
per operand copy."""

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


def _synth(rows, cols, phi, seed, dtype):
    from bench import synth
    return synth(torch, rows, cols, phi, seed, dtype, torch.device("cuda", 0))


# (rows, cols) slabs of an m x n product: corners, the n_block boundary at 8192,
# a raster boundary (2048-row groups) in the middle
def _slabs(m, n):
    s = [(slice(0, 64), slice(0, 48)), (slice(m - 64, m), slice(n - 48, n))]
    if n > 8192:
        s.append((slice(2016, 2080), slice(8168, 8216)))
    else:
        s.append((slice(m // 2 - 32, m // 2 + 32), slice(n // 2 - 24, n // 2 + 24)))
    return s


def _host(t):
    return t.cpu().numpy()


def _run(crt, A, B, N, mode, prec, n_block=8192):
    cfg = crt.EmuConfig(precision=prec, domain="complex", mode=mode, num_moduli=N,
                        n_block=n_block)
    out, mu, nu = crt.run_complex(A, B, cfg, None, A.device, return_exponents=True)
    torch.cuda.synchronize()
    return out, mu.cpu().numpy().astype(np.int64), nu.cpu().numpy().astype(np.int64)


# ------------------------------------------------------------------ cfg3 fast
@pytest.fixture(scope="module")
def cfg3_inputs():
    m = n = k = 16384
    A = _synth(m, k, 0.5, 1000, torch.complex128)  # bench.py's rank-0 seeds
    B = _synth(k, n, 0.5, 2000, torch.complex128)
    yield A, B
    del A, B
    torch.cuda.empty_cache()


@pytest.mark.parametrize("N", [15, 12, 20])
def test_cfg3_zgemm16384_fast(crt, cfg3_inputs, N):
    """The headline (N=15) and the sweep ends of cfg3, fast mode, phi=0.5."""
    A, B = cfg3_inputs
    C, mu, nu = _run(crt, A, B, N, "fast", "double")
    for rows, cols in _slabs(16384, 16384):
        a = _host(A[rows])
        b = _host(B[:, cols])
        want_mu, want_nu = orc.exponents(a, b, N, "fast")
        assert np.array_equal(mu[rows], want_mu) and np.array_equal(nu[cols], want_nu)
        want = orc.emulate_complex(a, b, N, "fast", "double")
        got = _host(C[rows, cols])
        assert got.tobytes() == want.tobytes(), (N, rows, cols)


@pytest.mark.parametrize("N", [15, 13])
def test_cfg3_zgemm16384_accurate(crt, cfg3_inputs, N):
    """cfg3 accurate mode: exponents of slab rows / columns from the oracle's
    bound products against the FULL other operand, then the C slab with those
    exponents injected."""
    A, B = cfg3_inputs
    C, mu, nu = _run(crt, A, B, N, "accurate", "double")
    mods = orc.pick_moduli(N)
    _, pa, delta = orc.scale_thresholds(mods.P)
    a_full = orc._split(_host(A))
    b_full = orc._split(_host(B))
    for rows, cols in _slabs(16384, 16384)[:2]:
        a = _host(A[rows])
        b = _host(B[:, cols])
        mu_rows, _, _ = orc.accurate_exps(orc._split(a), b_full, pa, delta)
        _, nu_cols, _ = orc.accurate_exps(a_full, orc._split(b), pa, delta)
        assert np.array_equal(mu[rows], mu_rows), rows
        assert np.array_equal(nu[cols], nu_cols), cols
        want = orc.emulate_complex_exps(a, b, mu_rows, nu_cols, N, "double")
        assert _host(C[rows, cols]).tobytes() == want.tobytes(), (N, rows, cols)


# ------------------------------------------------------------------ cfg2 CGEMM
@pytest.mark.parametrize("N", [6, 8, 10])
def test_cfg2_cgemm8192_fast(crt, N):
    """cfg2: complex64 inputs, single precision, N = 6..10 (fast)."""
    m = n = k = 8192
    A = _synth(m, k, 1.0, 3000 + N, torch.complex64)
    B = _synth(k, n, 1.0, 4000 + N, torch.complex64)
    C, mu, nu = _run(crt, A, B, N, "fast", "single")
    assert C.dtype == torch.complex64
    for rows, cols in _slabs(m, n):
        a = _host(A[rows])
        b = _host(B[:, cols])
        want = orc.emulate_complex(a, b, N, "fast", "single")
        assert _host(C[rows, cols]).tobytes() == want.tobytes(), (N, rows, cols)
    del A, B, C
    torch.cuda.empty_cache()


def test_cfg2_cgemm8192_accurate(crt):
    """cfg2 accurate (N=7, the single-precision accurate default)."""
    m = n = k = 8192
    N = 7
    A = _synth(m, k, 1.0, 3100, torch.complex64)
    B = _synth(k, n, 1.0, 4100, torch.complex64)
    C, mu, nu = _run(crt, A, B, N, "accurate", "single")
    mods = orc.pick_moduli(N)
    _, pa, delta = orc.scale_thresholds(mods.P)
    a_full = orc._split(_host(A).astype(np.complex128))
    b_full = orc._split(_host(B).astype(np.complex128))
    rows, cols = _slabs(m, n)[1]
    a = _host(A[rows]).astype(np.complex128)
    b = _host(B[:, cols]).astype(np.complex128)
    mu_rows, _, _ = orc.accurate_exps(orc._split(a), b_full, pa, delta)
    _, nu_cols, _ = orc.accurate_exps(a_full, orc._split(b), pa, delta)
    assert np.array_equal(mu[rows], mu_rows) and np.array_equal(nu[cols], nu_cols)
    want = orc.emulate_complex_exps(a, b, mu_rows, nu_cols, N, "single")
    assert _host(C[rows, cols]).tobytes() == want.tobytes()
    del A, B, C
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ cfg4 skinny
@pytest.mark.parametrize("N,phi", [(20, 4.0), (14, 2.0)])
def test_cfg4_zgemm_skinny_k65536(crt, N, phi):
    """cfg4: m = n = 4096, k = 2^16 (the complex k cap), wide exponent range
    (phi = 4: |a'| up to ~2^77 at N = 20, the six-limb residue form)."""
    m = n = 4096
    k = 65536
    A = _synth(m, k, phi, 5000 + N, torch.complex128)
    B = _synth(k, n, phi, 6000 + N, torch.complex128)
    C, mu, nu = _run(crt, A, B, N, "fast", "double")
    for rows, cols in _slabs(m, n)[:2]:
        a = _host(A[rows])
        b = _host(B[:, cols])
        want = orc.emulate_complex(a, b, N, "fast", "double")
        assert _host(C[rows, cols]).tobytes() == want.tobytes(), (N, rows, cols)
    del A, B, C
    torch.cuda.empty_cache()


# ------------------------------------------------ accurate exponents, full size
def test_accurate_exponents_full_4096(crt):
    """mu / nu of an accurate-mode 4096^3 product, every entry, against the
    oracle's full bound product (three 4096^3 exact int8 GEMMs on the CPU)."""
    m = n = k = 4096
    N = 15
    A = _synth(m, k, 2.0, 7000, torch.complex128)
    B = _synth(k, n, 2.0, 7001, torch.complex128)
    C, mu, nu = _run(crt, A, B, N, "accurate", "double")
    a, b = _host(A), _host(B)
    want_mu, want_nu = orc.exponents(a, b, N, "accurate")
    assert np.array_equal(mu, want_mu) and np.array_equal(nu, want_nu)
    rows, cols = slice(4000, 4096), slice(0, 64)
    want = orc.emulate_complex_exps(a[rows], b[:, cols], want_mu[rows], want_nu[cols], N)
    assert _host(C[rows, cols]).tobytes() == want.tobytes()


def test_accurate_bound_saturated_bytes(crt):
    """Every row of A and column of B holds an entry (1 - 2^-10)(1 + 1j): its
    bound operands are R = I = 64, so R + I = 128 -- the one byte value above
    127, which only the unsigned u8 x u8 descriptor of the (R+I)(R'+I') product
    reads correctly -- decides the row / column maxima of the bound."""
    rng = np.random.default_rng(128)
    m, n, k = 300, 520, 700
    a = (rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))) * 0.3
    b = (rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))) * 0.3
    sat = (1.0 - 2.0 ** -10) * (1 + 1j)
    a[np.arange(m), rng.integers(0, k, m)] = sat
    b[rng.integers(0, k, n), np.arange(n)] = sat
    # and a block where the saturated entries meet in the same k
    a[:40, 5] = sat
    b[5, :40] = sat
    for N in (13, 15):
        cfg = crt.EmuConfig(domain="complex", mode="accurate", num_moduli=N)
        at = torch.from_numpy(a).cuda()
        bt = torch.from_numpy(b).cuda()
        out, mu, nu = crt.run_complex(at, bt, cfg, None, at.device, return_exponents=True)
        want_mu, want_nu = orc.exponents(a, b, N, "accurate")
        assert np.array_equal(mu.cpu().numpy(), want_mu)
        assert np.array_equal(nu.cpu().numpy(), want_nu)
        want = orc.emulate_complex(a, b, N, "accurate")
        assert out.cpu().numpy().tobytes() == want.tobytes(), N
