"""GPU accuracy harness: the device double-double product is
bit-identical to the reference's numba oracle (golden vectors from
reference_gemm_dd), and the device max_relative_error equals the reference's."""

import numpy as np
import pytest

from oracle import ozaki2 as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_dd_gemm_golden(golden):
    from paper_2512_08321_b200 import accuracy as acc
    tags = sorted({k.split("__")[0] for k in golden.files if k.endswith("__ddmeta")})
    assert tags
    for tag in tags:
        m, n, k, seed, cplx = golden[f"{tag}__ddmeta"].tolist()
        dom = "complex" if cplx else "real"
        phi = float(golden[f"{tag}__phi"])
        a = orc.gen_matrix(m, k, phi, seed, "double", dom)
        b = orc.gen_matrix(k, n, phi, seed + 1, "double", dom)
        ref = acc.reference_gemm_dd(a, b)
        assert ref.hi.cpu().numpy().tobytes() == golden[f"{tag}__hi"].tobytes(), tag
        assert ref.lo.cpu().numpy().tobytes() == golden[f"{tag}__lo"].tobytes(), tag
        err, zeros = acc.max_relative_error(golden[f"{tag}__approx"], ref, return_zero_count=True)
        want = golden[f"{tag}__err"]
        assert err == float(want[0]) and zeros == int(want[1]), tag


def test_dd_gemm_vs_oracle_medium():
    from paper_2512_08321_b200 import accuracy as acc
    a = orc.gen_matrix(64, 700, 3.0, 90)
    b = orc.gen_matrix(700, 48, 3.0, 91)
    ref = acc.reference_gemm_dd(a, b)
    hi, lo = orc.dd_gemm(a, b)
    assert ref.hi.cpu().numpy().tobytes() == hi.tobytes()
    assert ref.lo.cpu().numpy().tobytes() == lo.tobytes()


def test_emulation_error_per_moduli_monotone():
    import paper_2512_08321_b200 as crt
    from paper_2512_08321_b200 import accuracy as acc
    a = orc.gen_matrix(256, 1024, 1.0, 92)
    b = orc.gen_matrix(1024, 256, 1.0, 93)
    ref = acc.reference_gemm_dd(a, b)
    errs = [acc.max_relative_error(crt.emulate_gemm_complex(
        a, b, crt.EmuConfig(domain="complex", num_moduli=N)), ref) for N in (12, 14, 16, 18)]
    assert errs[0] > errs[1] > errs[2] >= errs[3]
    assert errs[3] < 1e-14
