"""CPU: host-side logic of the drop-in API — configuration knobs and errors
(mirroring reference tests/test_emulate.py:13-29), modulus sets and scaling
constants against the reference's golden values, the C constant struct."""

import ctypes
import functools
import os
import subprocess
import tempfile

import numpy as np
import pytest

import paper_2512_08321_b200 as crt
from paper_2512_08321_b200.moduli import CrtgConsts, device_constants


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@functools.lru_cache(maxsize=None)
def c_layout():
    """sizeof/offsetof of crtg_consts as the C compiler lays it out."""
    fields = ("moduli", "coeff_hi", "coeff_lo", "p_hi", "p_lo", "p_fast", "p_accu", "delta")
    src = ('#include <stdio.h>\n#include <stddef.h>\n#include "crtg.h"\nint main(void){'
           'printf("size %zu\\n", sizeof(crtg_consts));'
           + "".join(f'printf("{f} %zu\\n", offsetof(crtg_consts, {f}));' for f in fields)
           + "return 0;}")
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        exe = os.path.join(d, "t")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    return {k: int(v) for k, v in (line.split() for line in out.splitlines())}


class TestEmuConfig:
    def test_defaults_resolve(self):
        assert crt.EmuConfig().resolved_moduli == 15
        assert crt.EmuConfig(domain="complex").resolved_moduli == 14
        assert crt.EmuConfig(domain="complex", mode="accurate").resolved_moduli == 15
        assert crt.EmuConfig(domain="complex", precision="single").resolved_moduli == 8
        assert crt.EmuConfig(domain="complex", precision="single",
                             mode="accurate").resolved_moduli == 7
        assert crt.EmuConfig(domain="complex", num_moduli=20).resolved_moduli == 20
        assert crt.EmuConfig().n_block == 8192 and crt.EmuConfig().strategy == "karatsuba"

    @pytest.mark.parametrize("kw", [dict(precision="half"), dict(domain="quaternion"),
                                    dict(mode="slow"), dict(num_moduli=0), dict(num_moduli=21),
                                    dict(n_block=0), dict(strategy="strassen")])
    def test_validation(self, kw):
        with pytest.raises(crt.ConfigError):
            crt.EmuConfig(**kw)

    def test_errors_are_value_errors(self):
        for e in (crt.ConfigError, crt.DimensionError, crt.DomainError):
            assert issubclass(e, ValueError)

    def test_domain_mismatch_raises_before_device(self):
        with pytest.raises(crt.ConfigError):
            crt.emulate_gemm_complex(np.ones((2, 2)), np.ones((2, 2)), crt.EmuConfig())
        with pytest.raises(crt.ConfigError):
            crt.gemm("complex", "single", 1, 1, 1, [1], 1, [1], 1, [0j], 1,
                     crt.EmuConfig(domain="complex"))


class TestModuli:
    def test_against_golden(self, golden):
        for n in range(1, 21):
            ms = crt.select_moduli(n)
            assert ms.moduli == tuple(golden[f"moduli_{n}"].tolist())
            assert np.array_equal(ms.coeff_hi, golden[f"coeff_hi_{n}"])
            assert np.array_equal(ms.coeff_lo, golden[f"coeff_lo_{n}"])
            assert str(ms.product) == str(golden[f"P_{n}"])
            sc = crt.ScalingConstants.from_product(ms.product)
            assert np.array_equal(np.array([sc.p_fast, sc.p_accu, sc.delta], np.float32),
                                  golden[f"consts_{n}"])

    def test_known_sets(self):
        assert crt.select_moduli(6).moduli == (256, 255, 253, 251, 247, 241)
        assert crt.select_moduli(8).moduli[-2:] == (239, 233)
        assert crt.select_moduli(14).moduli[-1] == 199
        assert crt.select_moduli(20).moduli[-1] == 173

    def test_crt_weights_reconstruct(self):
        ms = crt.select_moduli(9)
        rng = np.random.default_rng(0)
        for x in rng.integers(-(2 ** 60), 2 ** 60, 50).tolist():
            res = [((x % p) + p // 2) % p - p // 2 for p in ms.moduli]
            s = sum(int(h) * r for h, r in zip(ms.coeff_hi, res)) + \
                sum(int(lo) * r for lo, r in zip(ms.coeff_lo, res))
            z = (s + ms.product // 2) // ms.product
            assert s - z * ms.product == x

    def test_invalid_sets(self):
        with pytest.raises(crt.ConfigError):
            crt.ModulusSet.from_moduli([256, 254])
        with pytest.raises(crt.ConfigError):
            crt.ModulusSet.from_moduli([257])
        with pytest.raises(crt.ConfigError):
            crt.select_moduli(0)

    def test_device_struct(self):
        k = device_constants(14)
        assert ctypes.sizeof(CrtgConsts) == c_layout()["size"]
        for f in ("moduli", "coeff_hi", "coeff_lo", "p_hi", "p_lo", "p_fast", "p_accu", "delta"):
            assert getattr(CrtgConsts, f).offset == c_layout()[f], f
        ms = crt.select_moduli(14)
        assert k.num_moduli == 14 and list(k.moduli)[:14] == list(ms.moduli)
        assert k.p_hi == float(ms.product)
        assert int(k.p_hi) + int(k.p_lo) == ms.product or abs(
            (int(k.p_hi) + int(k.p_lo)) - ms.product) < 2 ** 60
        assert np.float32(k.p_fast) == crt.ScalingConstants.from_product(ms.product).p_fast


class TestSplitModuli:
    """Moduli with a square root of -1 take the 2-product (split) form on the GPU."""

    def test_sqrt_minus_one(self):
        from paper_2512_08321_b200.moduli import has_sqrt_minus_one
        # primes 1 mod 4 split, primes 3 mod 4 and even moduli do not
        assert [p for p in (241, 233, 229, 197, 193, 181, 173) if has_sqrt_minus_one(p)] == \
            [241, 233, 229, 197, 193, 181, 173]
        assert not any(has_sqrt_minus_one(p) for p in (256, 255, 253, 251, 247, 239, 227, 223,
                                                       217, 211, 199, 191, 179))
        # composite with every factor 1 mod 4 (5 * 13 = 65, 5 * 17 = 85)
        assert has_sqrt_minus_one(65) and has_sqrt_minus_one(85)
        assert not has_sqrt_minus_one(3 * 5)

    def test_identity_on_residues(self):
        # e_R = (X + Y)/2, e_I = (X - Y)/(2j) with X = U U', Y = V V'  (mod p)
        rng = np.random.default_rng(3)
        for p in (241, 173, 197):
            j = next(x for x in range(1, p) if (x * x + 1) % p == 0)
            ar, ai, br, bi = (rng.integers(-(p // 2), p // 2 + 1, 50) for _ in range(4))
            u, v = (ar + j * ai) % p, (ar - j * ai) % p
            u2, v2 = (br + j * bi) % p, (br - j * bi) % p
            X, Y = int(np.sum(u * u2)), int(np.sum(v * v2))
            inv2, inv2j = pow(2, -1, p), pow(2 * j, -1, p)
            er = int(np.sum(ar * br - ai * bi))
            ei = int(np.sum(ar * bi + ai * br))
            assert (X + Y) * inv2 % p == er % p
            assert (X - Y) * inv2j % p == ei % p

    def test_products_per_modulus(self, monkeypatch):
        from paper_2512_08321_b200.moduli import products_per_modulus
        ms = crt.select_moduli(15)
        monkeypatch.setenv("CRTG_SPLIT", "1")
        assert sum(products_per_modulus(ms)) == 41
        assert sum(products_per_modulus(crt.select_moduli(20))) == 53
        monkeypatch.setenv("CRTG_SPLIT", "0")
        assert sum(products_per_modulus(ms)) == 45


# ---------------------------------------------------------------- empty extents
@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("domain", ["complex", "real"])
def test_empty_rows_or_cols_fast(prec, domain):
    """Reference behaviour (run against crtgemm 0.1.0): fast mode with m = 0 or
    n = 0 returns an empty result of the output dtype; no device work."""
    import numpy as np

    import paper_2512_08321_b200 as crt
    cfg = crt.EmuConfig(precision=prec, domain=domain, mode="fast")
    fn = crt.emulate_gemm_complex if domain == "complex" else crt.emulate_gemm_real
    cplx = domain == "complex"
    want = {("complex", "double"): np.complex128, ("complex", "single"): np.complex64,
            ("real", "double"): np.float64, ("real", "single"): np.float32}[(domain, prec)]
    for sa, sb in (((0, 5), (5, 3)), ((4, 5), (5, 0))):
        a = np.ones(sa, np.complex128 if cplx else np.float64)
        b = np.ones(sb, np.complex128 if cplx else np.float64)
        c = fn(a, b, cfg)
        assert c.shape == (sa[0], sb[1]) and c.dtype == want


@pytest.mark.parametrize("mode", ["fast", "accurate"])
def test_empty_extents_raise_like_reference(mode):
    """Zero k (any mode) and zero m / n in accurate mode fail in the reference's
    max-reduction with a ValueError; DimensionError is a ValueError."""
    import numpy as np

    import paper_2512_08321_b200 as crt
    cfg = crt.EmuConfig(domain="complex", mode=mode)
    cases = [((4, 0), (0, 3)), ((0, 0), (0, 0))]
    if mode == "accurate":
        cases += [((0, 5), (5, 3)), ((4, 5), (5, 0))]
    for sa, sb in cases:
        with pytest.raises(ValueError):
            crt.emulate_gemm_complex(np.ones(sa, complex), np.ones(sb, complex), cfg)
