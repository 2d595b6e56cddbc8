"""CLI `emulate` / `accuracy` on the GPU (reference tests/test_cli.py).

`emulate` must write files BYTE-identical to the ones the reference CLI wrote
for the same input files and flags (tests/golden/cli/, make_cli_golden.py):
complex double (fast/accurate), complex single, real double and real single.
"""

import os

import numpy as np
import pytest

from paper_2512_08321_b200 import EmuConfig, emulate_gemm_complex, emulate_gemm_real, read_matrix
from paper_2512_08321_b200.cli import cli_dispatch
from test_cli_cpu import CASES, gold

pytestmark = pytest.mark.gpu


def run(*argv):
    return cli_dispatch([str(a) for a in argv])


@pytest.mark.parametrize("case", CASES["emulate"], ids=lambda c: c["name"])
def test_emulate_file_identical_to_reference(tmp_path, case):
    name = case["name"]
    out = tmp_path / "c.oz2m"
    assert run("emulate", gold(f"{name}_a.oz2m"), gold(f"{name}_b.oz2m"), "--out", out,
               *case["flags"]) == 0
    assert out.read_bytes() == open(gold(f"{name}_c.oz2m"), "rb").read()


def test_gen_then_emulate_matches_library(tmp_path):
    a, b, c = (tmp_path / f"{x}.oz2m" for x in "abc")
    assert run("gen", "-m", 9, "-n", 12, "--phi", 0.5, "--seed", 5, "--domain", "complex",
               "--out", a) == 0
    assert run("gen", "-m", 12, "-n", 7, "--phi", 0.5, "--seed", 6, "--domain", "complex",
               "--out", b) == 0
    assert run("emulate", a, b, "--out", c, "--mode", "accurate", "-N", 10, "--time") == 0
    am, bm, cm = (read_matrix(p) for p in (a, b, c))
    want = emulate_gemm_complex(am, bm, EmuConfig(domain="complex", mode="accurate", num_moduli=10))
    assert np.array_equal(cm, want)


def test_emulate_identity_real(tmp_path):
    from paper_2512_08321_b200 import write_matrix

    a, e, c = (tmp_path / f"{x}.oz2m" for x in "aec")
    run("gen", "-m", 6, "-n", 6, "--phi", 0, "--seed", 1, "--out", a)
    write_matrix(e, np.eye(6))
    assert run("emulate", a, e, "--out", c, "-N", 8) == 0
    want = emulate_gemm_real(read_matrix(a), np.eye(6), EmuConfig(num_moduli=8))
    assert np.array_equal(read_matrix(c), want)


def test_accuracy_single_row(tmp_path):
    out = tmp_path / "acc.csv"
    assert run("accuracy", "-m", 6, "-n", 6, "-k", 12, "-N", 5, "--phi", 0.5, "--seeds", 0,
               "--domain", "complex", "--out", out) == 0
    lines = out.read_text().strip().split("\n")
    assert lines[0] == "N,phi,seed,max_rel_error" and len(lines) == 2
    assert lines[1].startswith("5,0.5,0,")


def test_accuracy_byte_identical_reruns(tmp_path):
    args = ("accuracy", "-m", 5, "-n", 5, "-k", 10, "-N", "4,6", "--phi", "0,1", "--seeds", "0,1",
            "--precision", "single", "--domain", "real", "--mode", "fast")
    o1, o2 = tmp_path / "a1.csv", tmp_path / "a2.csv"
    assert run(*args, "--out", o1) == 0 and run(*args, "--out", o2) == 0
    assert o1.read_bytes() == o2.read_bytes()
    assert len(o1.read_text().strip().split("\n")) == 1 + 2 * 2 * 2


def test_accuracy_sweep_matches_oracle_metric():
    """The device sweep's error equals the oracle's dd metric on the same product."""
    from oracle import ozaki2 as oz
    from paper_2512_08321_b200 import GenSpec, gen_matrix, run_accuracy_sweep

    rows = run_accuracy_sweep((24, 20, 40), [8, 12], [1.0], mode="fast", domain="complex")
    a = gen_matrix(GenSpec(24, 40, 1.0, 0, "double", "complex"))
    b = gen_matrix(GenSpec(40, 20, 1.0, 1, "double", "complex"))
    for count, phi, seed, err in rows:
        c = emulate_gemm_complex(a, b, EmuConfig(domain="complex", num_moduli=count))
        hi, lo = oz.dd_gemm(a, b)
        assert err == oz.max_relative_error(c, hi, lo)
