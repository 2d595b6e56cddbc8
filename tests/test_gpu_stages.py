"""GPU parity of the stage-level drop-in API (paper_2512_08321_b200/stages.py)
against golden vectors produced by the UNMODIFIED reference
(tests/golden/make_stage_golden.py -> golden_stages.npz; log2_upper from
golden_small.npz).  Every comparison is bytes-equal: dtype, shape and bits.

Reference functions: log2_upper scaling.py:62-82, quantize scaling.py:277-293,
symmetric_mod_int crt.py:136-151, residue_decompose crt.py:199-218,
crt_accumulate crt.py:221-243, crt_reduce crt.py:246-258, symmetric_mod_wide
crt.py:154-184, inverse_scale emulate.py:135-144, crt_integer_gemm
emulate.py:120-132."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def crt():
    import paper_2512_08321_b200 as crt
    from paper_2512_08321_b200 import _native
    _native.load()
    return crt


@pytest.fixture(scope="module")
def gs():
    return np.load(os.path.join(HERE, "golden", "golden_stages.npz"))


def same(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.dtype == want.dtype, (got.dtype, want.dtype)
    assert got.shape == want.shape, (got.shape, want.shape)
    if got.tobytes() != want.tobytes():
        u = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[got.itemsize]
        bad = np.flatnonzero(np.ascontiguousarray(got).reshape(-1).view(u)
                             != np.ascontiguousarray(want).reshape(-1).view(u))
        i = bad[0]
        raise AssertionError(f"{bad.size} of {got.size} differ; first at {i}: "
                             f"{got.reshape(-1)[i]!r} vs {want.reshape(-1)[i]!r}")


def test_log2_upper(crt, golden):
    same(crt.log2_upper(golden["log2_x"]), golden["log2_y"])
    # torch in -> torch out, same bits
    t = torch.from_numpy(golden["log2_x"]).cuda()
    out = crt.log2_upper(t)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    same(out.cpu().numpy(), golden["log2_y"])
    # scalar in -> float32 scalar out
    x = float(golden["log2_x"][17])
    assert np.float32(crt.log2_upper(x)) == golden["log2_y"][17]


def test_quantize(crt, gs):
    same(crt.quantize(gs["q_x"], gs["q_mu"], 0), gs["q_rows"])
    same(crt.quantize(gs["q_x"], gs["q_nu"], 1), gs["q_cols"])
    same(crt.quantize(gs["q_x"], gs["q_wide_e"], 0), gs["q_wide"])


def test_quantize_errors(crt, gs):
    with pytest.raises(crt.DimensionError):
        crt.quantize(gs["q_x"], gs["q_mu"][:-1], 0)
    with pytest.raises(crt.ConfigError):
        crt.quantize(gs["q_x"], gs["q_mu"], 2)
    # |a'| >= 2^90 -> DomainError (scaling.py:290-292)
    with pytest.raises(crt.DomainError):
        crt.quantize(np.array([[1.0]]), np.array([90]), 0)


@pytest.mark.parametrize("p", [2, 3, 127, 128, 173, 199, 241, 255, 256])
def test_symmetric_mod_int(crt, gs, p):
    same(crt.symmetric_mod_int(gs["smi_xi"], p), gs[f"smi_i_{p}"])
    same(crt.symmetric_mod_int(gs["smi_xf"], p), gs[f"smi_f_{p}"])


def test_symmetric_mod_int_scalar(crt, gs):
    for v, p, want in gs["smi_scalar"].tolist():
        assert crt.symmetric_mod_int(int(v), int(p)) == want
    with pytest.raises(crt.DomainError):
        crt.symmetric_mod_int(np.array([1, 2]), 1)


def test_residue_decompose(crt, gs):
    ms = crt.select_moduli(20)
    st = crt.residue_decompose(gs["q_wide"], ms)
    assert isinstance(st, crt.ResidueStack) and st.modulus_set is ms
    same(st.entries, gs["rd_20"])
    # non-integer / non-finite / >= 2^90 inputs are rejected like crt.py:203-213
    with pytest.raises(crt.DomainError):
        crt.residue_decompose(np.array([[0.5]]), ms)
    with pytest.raises(crt.DomainError):
        crt.residue_decompose(np.array([[np.inf]]), ms)
    with pytest.raises(crt.DomainError):
        crt.residue_decompose(np.array([[2.0 ** 90]]), ms)


@pytest.mark.parametrize("N,prec", [(15, "double"), (8, "single"), (20, "double"), (1, "double")])
def test_crt_accumulate_reduce_inverse_scale(crt, gs, N, prec):
    ms = crt.select_moduli(N)
    st = crt.ResidueStack(gs[f"ca_{N}_e"], ms)
    acc = crt.crt_accumulate(st, ms, prec)
    if prec == "double":
        same(acc[0], gs[f"ca_{N}_s1"])
        same(acc[1], gs[f"ca_{N}_s2"])
    else:
        same(acc, gs[f"ca_{N}_s"])
    red = crt.crt_reduce(acc, ms)
    same(red, gs[f"ca_{N}_red"])
    sv = crt.ScalingVectors(gs[f"ca_{N}_mu"], gs[f"ca_{N}_nu"])
    same(crt.inverse_scale(red, sv, np.float64), gs[f"ca_{N}_inv64"])
    same(crt.inverse_scale(red, sv, np.float32), gs[f"ca_{N}_inv32"])


def test_crt_accumulate_wrong_set(crt, gs):
    st = crt.ResidueStack(gs["ca_15_e"], crt.select_moduli(15))
    with pytest.raises(crt.ConfigError):
        crt.crt_accumulate(st, crt.select_moduli(15), "half")


@pytest.mark.parametrize("N", [6, 14, 20])
def test_symmetric_mod_wide(crt, gs, N):
    P = int(str(gs[f"smw_{N}_P"]))
    assert P == crt.select_moduli(N).product
    same(crt.symmetric_mod_wide((gs[f"smw_{N}_hi"], gs[f"smw_{N}_lo"]), P, use_dd=True),
         gs[f"smw_{N}_dd"])
    same(crt.symmetric_mod_wide(gs[f"smw_{N}_hi"], P, use_dd=False), gs[f"smw_{N}_plain"])


@pytest.mark.parametrize("tag", ["cig_a", "cig_b", "cig_c"])
def test_crt_integer_gemm(crt, gs, tag):
    ms = crt.select_moduli(int(gs[f"{tag}_N"]))
    same(crt.crt_integer_gemm(gs[f"{tag}_a"], gs[f"{tag}_b"], ms, "double"), gs[f"{tag}_d"])
    same(crt.crt_integer_gemm(gs[f"{tag}_a"], gs[f"{tag}_b"], ms, "single", n_block=4),
         gs[f"{tag}_s"])


def test_complex_matrix(crt):
    re = np.arange(6.0).reshape(2, 3)
    cm = crt.ComplexMatrix(re, -re)
    same(cm.to_complex(), re + 1j * -re)
    with pytest.raises(crt.DimensionError):
        crt.ComplexMatrix(re, re[:1])
