"""The reference's three complex-product strategies on the GPU (kernel.py:45-120):
Karatsuba (three tcgen05 products) and the expanded formulations (one tcgen05
product on doubled operands, reference `_expand_rows_block` / `_expand_cols_block`),
both through `complex_gemm_mod` and through `emulate_gemm_complex(cfg.strategy)`.

Bar (reference tests/test_emulate.py:151-161, tests/test_kernel.py): every
strategy returns identical residues and identical products, bytes-equal to the
reference-made goldens; the expanded forms raise ArithmeticError exactly where
the reference's int32 guard does (kernel.py:33-34)."""

import numpy as np
import pytest

from oracle import ozaki2 as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

STRATS = ("karatsuba", "expand-rows", "expand-cols")


@pytest.fixture(scope="module")
def crt():
    import paper_2512_08321_b200 as crt
    from paper_2512_08321_b200 import _native
    _native.load()
    return crt


def _cases(golden):
    return sorted({k.split("__")[0] for k in golden.files if k.endswith("__meta")})


@pytest.mark.parametrize("strategy", STRATS)
def test_complex_gemm_mod_vs_golden(crt, golden, strategy):
    # the golden stacks and e-planes come from the reference (make_golden.py)
    for tag in _cases(golden):
        g = lambda s: golden[f"{tag}__{s}"]  # noqa: E731
        N = int(g("meta")[4])
        ms = crt.select_moduli(N)
        for idx, p in enumerate(ms.moduli):
            er, ei = crt.complex_gemm_mod(g("ar")[idx], g("ai")[idx], g("br")[idx], g("bi")[idx],
                                          p, strategy=strategy, n_block=7)
            assert er.tobytes() == g("er")[idx].tobytes(), (tag, p, strategy)
            assert ei.tobytes() == g("ei")[idx].tobytes(), (tag, p, strategy)


@pytest.mark.parametrize("p", [256, 255, 241, 173, 2, 3])
def test_strategies_identical_random(crt, p):
    rng = np.random.default_rng(p)
    lo, hi = -(p // 2) if p % 2 == 0 else -((p - 1) // 2), (p - 1) // 2
    m, k, n = 70, 333, 90
    ops = [rng.integers(lo, hi + 1, size=s).astype(np.int8)
           for s in ((m, k), (m, k), (k, n), (k, n))]
    got = [crt.complex_gemm_mod(*ops, p, strategy=s, n_block=32) for s in STRATS]
    for er, ei in got[1:]:
        assert er.tobytes() == got[0][0].tobytes() and ei.tobytes() == got[0][1].tobytes()
    # against exact integer arithmetic
    ar, ai, br, bi = (x.astype(np.int64) for x in ops)
    want_r = orc.sym_residue_int(ar @ br - ai @ bi, p)
    want_i = orc.sym_residue_int(ar @ bi + ai @ br, p)
    assert got[0][0].tobytes() == want_r.tobytes() and got[0][1].tobytes() == want_i.tobytes()


def test_expand_int32_guard(crt):
    # k = 2^16, p = 256, every residue -128: the doubled inner length gives
    # 2^17 * 2^14 = 2^31 > int32 max -> ArithmeticError for the expanded forms
    # only (the reference behaves the same, kernel.py:33-34)
    k = 65536
    a = np.full((1, k), -128, np.int8)
    b = np.full((k, 1), -128, np.int8)
    er, ei = crt.complex_gemm_mod(a, a, b, b, 256, strategy="karatsuba")
    assert int(er[0, 0]) == 0 and int(ei[0, 0]) == 0
    for s in ("expand-rows", "expand-cols"):
        with pytest.raises(ArithmeticError):
            crt.complex_gemm_mod(a, a, b, b, 256, strategy=s)


@pytest.mark.parametrize("strategy", ["expand-rows", "expand-cols"])
def test_emulate_strategy_vs_golden(crt, golden, strategy):
    for tag in _cases(golden):
        g = lambda s: golden[f"{tag}__{s}"]  # noqa: E731
        m, n, k, seed, N, dbl, fast = g("meta").tolist()
        prec = "double" if dbl else "single"
        mode = "fast" if fast else "accurate"
        a = orc.gen_matrix(m, k, float(g("phi")), seed, prec)
        b = orc.gen_matrix(k, n, float(g("phi")), seed + 1, prec)
        cfg = crt.EmuConfig(precision=prec, domain="complex", mode=mode, num_moduli=N,
                            strategy=strategy, n_block=16)
        diag = {}
        c = crt.emulate_gemm_complex(a, b, cfg, diag)
        assert c.dtype == g("c").dtype and c.tobytes() == g("c").tobytes(), (tag, strategy)
        assert [diag.get("clamped_mu", 0), diag.get("clamped_nu", 0)] == g("diag").tolist()


@pytest.mark.parametrize("strategy", ["expand-rows", "expand-cols"])
def test_emulate_strategy_equals_pipeline_device(crt, strategy):
    a = torch.from_numpy(orc.gen_matrix(300, 700, 1.0, 5, "double")).cuda()
    b = torch.from_numpy(orc.gen_matrix(700, 260, 1.0, 6, "double")).cuda()
    base = crt.emulate_gemm_complex(a, b, crt.EmuConfig(domain="complex", num_moduli=15))
    cfg = crt.EmuConfig(domain="complex", num_moduli=15, strategy=strategy, n_block=100)
    got = crt.emulate_gemm_complex(a, b, cfg)
    assert got.is_cuda and got.dtype == base.dtype
    assert torch.equal(got.view(torch.float64), base.view(torch.float64))
