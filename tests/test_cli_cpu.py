"""OZ2M files, the generator, the perf model and the CLI surface — CPU only.

Fixtures in tests/golden/cli/ come from the unmodified reference
(make_cli_golden.py): its `gen` output files, its `write_matrix` output per
dtype code, and its perf-model numbers / CLI text.  Mirrors the reference's
tests/test_matfile.py, test_perfmodel.py and test_cli.py.
"""

import io
import json
import os
import struct
from contextlib import redirect_stdout

import numpy as np
import pytest

from paper_2512_08321_b200 import (ConfigError, GenSpec, PerfParams, gen_matrix, heatmap_csv,
                                   heatmap_grid, predict_time, predicted_tflops, read_matrix,
                                   write_matrix)
from paper_2512_08321_b200 import perfmodel as pm
from paper_2512_08321_b200.cli import cli_dispatch

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cli")
CASES = json.load(open(os.path.join(GOLD, "cli_cases.json")))


def gold(name):
    return os.path.join(GOLD, name)


def run(*argv):
    return cli_dispatch(list(argv))


# ------------------------------------------------------------------ OZ2M files

@pytest.mark.parametrize("code", range(4))
def test_golden_dtype_files_round_trip_bytes(tmp_path, code):
    x = read_matrix(gold(f"dtype{code}.oz2m"))
    assert x.shape == (3, 5)
    out = tmp_path / "x.oz2m"
    write_matrix(out, x)
    assert out.read_bytes() == open(gold(f"dtype{code}.oz2m"), "rb").read()


@pytest.mark.parametrize("dtype", [np.float32, np.float64, np.complex64, np.complex128])
def test_round_trip(tmp_path, dtype):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((7, 4)).astype(dtype)
    if np.iscomplexobj(x):
        x = (x + 1j * rng.standard_normal((7, 4))).astype(dtype)
    write_matrix(tmp_path / "m.oz2m", x)
    y = read_matrix(tmp_path / "m.oz2m")
    assert y.dtype == x.dtype and np.array_equal(x, y)


def test_header_and_column_major_payload(tmp_path):
    x = np.arange(6, dtype=np.float64).reshape(2, 3)
    write_matrix(tmp_path / "m.oz2m", x)
    raw = (tmp_path / "m.oz2m").read_bytes()
    assert raw[:4] == b"OZ2M"
    assert struct.unpack("<qqB", raw[4:21]) == (2, 3, 1)
    assert np.array_equal(np.frombuffer(raw[21:], "<f8"), [0, 3, 1, 4, 2, 5])


def test_empty_matrix(tmp_path):
    write_matrix(tmp_path / "e.oz2m", np.zeros((0, 3), np.float32))
    assert read_matrix(tmp_path / "e.oz2m").shape == (0, 3)


def test_torch_tensor_input(tmp_path):
    torch = pytest.importorskip("torch")
    t = torch.arange(6, dtype=torch.float64).reshape(3, 2)
    write_matrix(tmp_path / "t.oz2m", t)
    assert np.array_equal(read_matrix(tmp_path / "t.oz2m"), t.numpy())


def test_errors(tmp_path):
    p = tmp_path / "bad.oz2m"
    p.write_bytes(b"NOPE" + bytes(17))
    with pytest.raises(ValueError, match="not an OZ2M"):
        read_matrix(p)
    p.write_bytes(b"OZ2M" + bytes(5))
    with pytest.raises(ValueError, match="truncated header"):
        read_matrix(p)
    p.write_bytes(b"OZ2M" + struct.pack("<qqB", -1, 2, 1))
    with pytest.raises(ValueError, match="negative"):
        read_matrix(p)
    p.write_bytes(b"OZ2M" + struct.pack("<qqB", 1, 2, 9))
    with pytest.raises(ValueError, match="unknown dtype code"):
        read_matrix(p)
    p.write_bytes(b"OZ2M" + struct.pack("<qqB", 2, 2, 1) + bytes(31))
    with pytest.raises(ValueError, match="truncated data"):
        read_matrix(p)
    with pytest.raises(ValueError, match="unsupported"):
        write_matrix(p, np.zeros((2, 2), np.float16))
    with pytest.raises(ValueError, match="2-D"):
        write_matrix(p, np.zeros(3))


# ------------------------------------------------------------------ generator

@pytest.mark.parametrize("case", CASES["emulate"], ids=lambda c: c["name"])
def test_gen_matches_reference_files(tmp_path, case):
    for side in ("a", "b"):
        assert run("gen", *case[f"gen_{side}"], "--out", str(tmp_path / "g.oz2m")) == 0
        want = open(gold(f"{case['name']}_{side}.oz2m"), "rb").read()
        assert (tmp_path / "g.oz2m").read_bytes() == want


def test_gen_matrix_against_oracle():
    from oracle import ozaki2 as oz

    for dom, prec in (("complex", "double"), ("real", "single")):
        got = gen_matrix(GenSpec(11, 6, 0.7, 3, prec, dom))
        want = oz.gen_matrix(11, 6, 0.7, 3, prec, dom)
        assert got.dtype == want.dtype and np.array_equal(got, want)


def test_genspec_validation():
    for bad in (dict(rows=0, cols=1), dict(rows=1, cols=1, phi=-1.0),
                dict(rows=1, cols=1, precision="half"), dict(rows=1, cols=1, domain="quat")):
        with pytest.raises(ConfigError):
            GenSpec(**bad)


# ------------------------------------------------------------------ perf model

@pytest.mark.parametrize("i", range(len(CASES["perf"])))
def test_perfmodel_matches_reference(i):
    c = CASES["perf"][i]
    pp = PerfParams(**c["params"])
    assert predict_time(pp) == c["seconds"]
    assert predicted_tflops(pp) == c["tflops"]


def test_perfmodel_validation_and_default_correction():
    base = dict(bandwidth=1e12, int8_ops=1e15, m=8, n=8, k=8, num_moduli=5)
    assert PerfParams(**base).c == 5.0
    for bad in (dict(bandwidth=0), dict(int8_ops=-1), dict(m=0), dict(num_moduli=0),
                dict(mode="slow"), dict(precision="half"), dict(correction=-1.0)):
        with pytest.raises(ConfigError):
            PerfParams(**{**base, **bad})


def test_heatmap_grid():
    t = PerfParams(1e12, 1e15, 1024, 1024, 1024, 8, "fast")
    rows = heatmap_grid((1e12, 2e12), (1e15, 3e15), (2, 3), t)
    assert [r[:2] for r in rows] == [(1e12, 1e15), (1e12, 2e15), (1e12, 3e15),
                                    (2e12, 1e15), (2e12, 2e15), (2e12, 3e15)]
    assert heatmap_csv(rows).splitlines()[0] == "b,p,tflops"
    with pytest.raises(ConfigError):
        heatmap_grid((2e12, 1e12), (1e15, 2e15), 2, t)
    with pytest.raises(ConfigError):
        heatmap_grid((1e12, 2e12), (1e15, 2e15), 0, t)


def test_fused_model_bounds():
    pp = pm.b200_params(16384, 16384, 16384, 15, "fast")
    t = pm.predict_time_fused(pp)
    gemm_only = 6 * 15 * 16384 ** 3 / pm.B200_INT8_OPS_PER_S
    assert gemm_only < t < predict_time(pp)
    assert pm.fused_bytes(pm.b200_params(64, 64, 64, 4, "accurate")) > \
        pm.fused_bytes(pm.b200_params(64, 64, 64, 4, "fast"))


# ------------------------------------------------------------------ CLI text / usage

@pytest.mark.parametrize("i", range(len(CASES["cli_text"])))
def test_cli_text_matches_reference(i):
    c = CASES["cli_text"][i]
    buf = io.StringIO()
    with redirect_stdout(buf):
        assert cli_dispatch(c["argv"]) == 0
    assert buf.getvalue() == c["stdout"]


def test_usage_errors():
    assert run("frobnicate") == 2
    assert run("gen", "-m", "2", "-n", "2", "--out", "x", "--bogus") == 2
    assert run("gen", "-m", "2") == 2


def test_missing_file_is_runtime_error(tmp_path, capsys):
    assert run("emulate", str(tmp_path / "a.oz2m"), str(tmp_path / "b.oz2m"),
               "--out", str(tmp_path / "c.oz2m")) == 1
    assert "crtgemm: error" in capsys.readouterr().err


def test_gen_config_error_is_exit_1(tmp_path, capsys):
    assert run("gen", "-m", "0", "-n", "2", "--out", str(tmp_path / "x.oz2m")) == 1
    assert "error" in capsys.readouterr().err
