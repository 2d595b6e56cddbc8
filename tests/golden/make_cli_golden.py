"""Generate the CLI / file-format / perf-model fixtures from the UNMODIFIED reference.

Run in the build container only (the reference tree does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_cli_golden.py

Writes tests/golden/cli/:
  * OZ2M files produced by the reference CLI (`crtgemm.cli.cli_dispatch`: `gen`,
    then `emulate`) — the inputs and the emulated products, byte for byte;
  * `write_matrix` outputs for each dtype code (f32, f64, c32, c64);
  * perfmodel.json: `predict_time` / `predicted_tflops` over a parameter grid,
    and the `perfmodel` / `heatmap` CLI outputs (exact text).
"""

from __future__ import annotations

import io
import json
import os
import sys
from contextlib import redirect_stdout

import numpy as np

import crtgemm as ref  # noqa: E402  (reference, read-only, via PYTHONPATH)
from crtgemm.cli import cli_dispatch  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli")

# (name, gen args for A, gen args for B, emulate flags)
EMULATE_CASES = [
    ("cz_accu10", ["-m", "9", "-n", "12", "--phi", "0.5", "--seed", "5", "--domain", "complex"],
     ["-m", "12", "-n", "7", "--phi", "0.5", "--seed", "6", "--domain", "complex"],
     ["--mode", "accurate", "-N", "10"]),
    ("cz_fast_default", ["-m", "33", "-n", "40", "--phi", "1", "--seed", "2", "--domain", "complex"],
     ["-m", "40", "-n", "17", "--phi", "1", "--seed", "3", "--domain", "complex"],
     []),
    ("cc_single_fast", ["-m", "20", "-n", "31", "--phi", "0.5", "--seed", "7", "--domain", "complex",
                        "--precision", "single"],
     ["-m", "31", "-n", "11", "--phi", "0.5", "--seed", "8", "--domain", "complex",
      "--precision", "single"],
     ["--mode", "fast", "-N", "7", "--block", "4"]),
    ("rd_fast8", ["-m", "6", "-n", "6", "--phi", "0", "--seed", "1"],
     ["-m", "6", "-n", "5", "--phi", "2", "--seed", "4"],
     ["-N", "8"]),
    ("rs_accu", ["-m", "13", "-n", "29", "--phi", "1.5", "--seed", "9", "--precision", "single"],
     ["-m", "29", "-n", "8", "--phi", "1.5", "--seed", "10", "--precision", "single"],
     ["--mode", "accurate"]),
]

PERF_GRID = [
    dict(m=16384, n=16384, k=16384, num_moduli=13, mode="accurate", precision="double",
         correction=13.0, bandwidth=4e12, int8_ops=1.5e15),
    dict(m=16384, n=16384, k=16384, num_moduli=15, mode="fast", precision="double",
         correction=None, bandwidth=6.5364e12, int8_ops=2.7154e15),
    dict(m=8192, n=8192, k=8192, num_moduli=8, mode="fast", precision="single",
         correction=None, bandwidth=6.5364e12, int8_ops=2.7154e15),
    dict(m=4096, n=4096, k=65536, num_moduli=14, mode="accurate", precision="single",
         correction=2.5, bandwidth=3e12, int8_ops=1e15),
    dict(m=1024, n=1024, k=1024, num_moduli=14, mode="fast", precision="double",
         correction=0.0, bandwidth=1e12, int8_ops=2.5e14),
]

CLI_TEXT = [
    ["perfmodel", "-m", "16384", "-n", "16384", "-k", "16384", "-N", "13", "-c", "13", "-b", "4e12",
     "-p", "1.5e15"],
    ["perfmodel", "-N", "15", "--mode", "fast"],
    ["heatmap", "-N", "6", "-c", "6", "--precision", "single", "--mode", "fast"],
    ["heatmap", "-m", "2048", "-n", "4096", "-k", "1024", "-N", "9", "--b-steps", "3",
     "--p-steps", "4"],
]


def main():
    os.makedirs(HERE, exist_ok=True)
    cases = []
    for name, ga, gb, flags in EMULATE_CASES:
        pa, pb, pc = (os.path.join(HERE, f"{name}_{x}.oz2m") for x in "abc")
        assert cli_dispatch(["gen", *ga, "--out", pa]) == 0
        assert cli_dispatch(["gen", *gb, "--out", pb]) == 0
        assert cli_dispatch(["emulate", pa, pb, "--out", pc, *flags]) == 0
        cases.append({"name": name, "gen_a": ga, "gen_b": gb, "flags": flags})
    for code, dt in enumerate([np.float32, np.float64, np.complex64, np.complex128]):
        x = (np.arange(15).reshape(3, 5) * 0.37 - 2).astype(dt)
        if np.iscomplexobj(x):
            x = (x + 1j * (np.arange(15).reshape(3, 5) * -0.11)).astype(dt)
        ref.write_matrix(os.path.join(HERE, f"dtype{code}.oz2m"), x)
    perf = []
    for p in PERF_GRID:
        pp = ref.PerfParams(**p)
        perf.append({"params": p, "seconds": ref.predict_time(pp), "tflops": ref.predicted_tflops(pp)})
    texts = []
    for argv in CLI_TEXT:
        buf = io.StringIO()
        with redirect_stdout(buf):
            assert cli_dispatch(argv) == 0
        texts.append({"argv": argv, "stdout": buf.getvalue()})
    with open(os.path.join(HERE, "cli_cases.json"), "w") as f:
        json.dump({"emulate": cases, "perf": perf, "cli_text": texts}, f, indent=1)
    print("wrote", HERE, file=sys.stderr)


if __name__ == "__main__":
    main()
