"""Command-line interface — the reference's `crtgemm` CLI (pkg/src/crtgemm/cli.py:1-198).

    python -m paper_2512_08321_b200 gen -m 4096 -n 4096 --phi 0.5 --domain complex --out A.oz2m
    python -m paper_2512_08321_b200 emulate A.oz2m B.oz2m --out C.oz2m --mode fast -N 14
    python -m paper_2512_08321_b200 accuracy -m 256 -n 256 -k 4096 -N 12,14,16 --phi 0.5,4
    python -m paper_2512_08321_b200 perfmodel -N 15 --mode fast [--b200]
    python -m paper_2512_08321_b200 heatmap -N 13 --out grid.csv

Same subcommands, flags, defaults, output formats and exit codes (0 ok,
1 runtime/value error with "crtgemm: error: ..." on stderr, 2 usage error).
`emulate` runs on the GPU through `emulate_gemm_complex` / `emulate_gemm_real`
and writes a file byte-identical to the reference's; `accuracy` uses the
device double-double harness.  B200 additions: `perfmodel --b200` evaluates the
fused-pipeline model with the measured B200 bandwidth / INT8 rate, and
`emulate --time` reports the device time of the call on stderr.
"""

from __future__ import annotations

import argparse
import sys

import numpy as np


def _emu_flags(sub):
    sub.add_argument("--mode", choices=["fast", "accurate"], default="fast")
    sub.add_argument("-N", "--num-moduli", type=int, default=None)
    sub.add_argument("--block", type=int, default=8192, help="output-column block width")
    sub.add_argument("--strategy", default="karatsuba",
                     choices=["karatsuba", "expand-rows", "expand-cols"])


def _perf_dims(sub):
    sub.add_argument("-m", type=int, default=16384)
    sub.add_argument("-n", type=int, default=16384)
    sub.add_argument("-k", type=int, default=16384)
    sub.add_argument("-N", "--num-moduli", type=int, default=13)
    sub.add_argument("-c", "--correction", type=float, default=None)
    sub.add_argument("--mode", choices=["fast", "accurate"], default="accurate")
    sub.add_argument("--precision", choices=["single", "double"], default="double")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(
        prog="crtgemm",
        description="GEMM emulation on exact INT8 tensor-core products with CRT "
                    "reconstruction (B200), plus the analytic performance model.")
    subs = ap.add_subparsers(dest="command", required=True)

    g = subs.add_parser("gen", help="generate a matrix file")
    g.add_argument("-m", type=int, required=True, help="rows")
    g.add_argument("-n", type=int, required=True, help="columns")
    g.add_argument("--phi", type=float, default=0.0)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--precision", choices=["single", "double"], default="double")
    g.add_argument("--domain", choices=["real", "complex"], default="real")
    g.add_argument("--out", required=True)

    e = subs.add_parser("emulate", help="multiply two matrix files")
    e.add_argument("a")
    e.add_argument("b")
    e.add_argument("--out", required=True)
    _emu_flags(e)
    e.add_argument("--time", action="store_true", help="report the device time on stderr")

    acc = subs.add_parser("accuracy", help="accuracy sweep over (N, phi, seed)")
    acc.add_argument("-m", type=int, default=256)
    acc.add_argument("-n", type=int, default=256)
    acc.add_argument("-k", type=int, default=4096)
    acc.add_argument("-N", "--num-moduli", default=None, help="comma-separated modulus counts")
    acc.add_argument("--phi", default="0.5", help="comma-separated phi values")
    acc.add_argument("--seeds", default="0", help="comma-separated seeds")
    acc.add_argument("--mode", choices=["fast", "accurate"], default="fast")
    acc.add_argument("--precision", choices=["single", "double"], default="double")
    acc.add_argument("--domain", choices=["real", "complex"], default="complex")
    acc.add_argument("--out", default=None, help="CSV path (default stdout)")

    pm = subs.add_parser("perfmodel", help="single performance prediction")
    _perf_dims(pm)
    pm.add_argument("-b", type=float, default=4.0e12, help="memory bandwidth in B/s")
    pm.add_argument("-p", type=float, default=1.5e15, help="INT8 throughput in ops/s")
    pm.add_argument("--b200", action="store_true",
                    help="fused B200 pipeline with the measured b and p (ignores -b/-p/-c)")
    pm.add_argument("--out", default=None)

    hm = subs.add_parser("heatmap", help="performance-model grid as CSV")
    _perf_dims(hm)
    hm.add_argument("--b-min", type=float, default=1.0e12)
    hm.add_argument("--b-max", type=float, default=5.0e12)
    hm.add_argument("--b-steps", type=int, default=17)
    hm.add_argument("--p-min", type=float, default=2.5e14)
    hm.add_argument("--p-max", type=float, default=2.0e15)
    hm.add_argument("--p-steps", type=int, default=15)
    hm.add_argument("--out", default=None)
    return ap


def _emit(text: str, path) -> None:
    if path is None:
        sys.stdout.write(text)
    else:
        with open(path, "w") as fh:
            fh.write(text)


def _ints(text, cast):
    return [cast(t) for t in str(text).split(",") if t != ""]


def _gen(args) -> int:
    from .gen import GenSpec, gen_matrix
    from .matfile import write_matrix

    spec = GenSpec(args.m, args.n, args.phi, args.seed, args.precision, args.domain)
    write_matrix(args.out, gen_matrix(spec))
    return 0


def _emulate(args) -> int:
    from .config import EmuConfig
    from .emulate import emulate_gemm_complex, emulate_gemm_real
    from .matfile import read_matrix, write_matrix

    a, b = read_matrix(args.a), read_matrix(args.b)
    cplx = np.iscomplexobj(a) or np.iscomplexobj(b)
    single = a.dtype in (np.float32, np.complex64) and b.dtype in (np.float32, np.complex64)
    cfg = EmuConfig(precision="single" if single else "double",
                    domain="complex" if cplx else "real", mode=args.mode,
                    num_moduli=args.num_moduli, n_block=args.block, strategy=args.strategy)
    # the reference widens to complex128 / float64 first (cli.py:120-124); both
    # widenings are exact, so the emulation sees the same values
    if cplx:
        a, b, run = a.astype(np.complex128), b.astype(np.complex128), emulate_gemm_complex
    else:
        a, b, run = a.astype(np.float64), b.astype(np.float64), emulate_gemm_real
    if args.time:
        import time

        import torch
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        c = run(a, b, cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        m, k = a.shape
        flops = (8 if cplx else 2) * m * b.shape[1] * k
        print(f"crtgemm: emulate {m}x{b.shape[1]}x{k} {cfg.domain} {cfg.precision} {cfg.mode} "
              f"N={cfg.resolved_moduli}: {dt * 1e3:.3f} ms, {flops / dt * 1e-12:.3f} TFLOPS "
              "(host in/out)", file=sys.stderr)
    else:
        c = run(a, b, cfg)
    write_matrix(args.out, c)
    return 0


def _accuracy(args) -> int:
    from .accuracy import run_accuracy_sweep, sweep_csv
    from .config import EmuConfig

    if args.num_moduli is None:
        counts = [EmuConfig(precision=args.precision, domain=args.domain,
                            mode=args.mode).resolved_moduli]
    else:
        counts = _ints(args.num_moduli, int)
    rows = run_accuracy_sweep((args.m, args.n, args.k), counts, _ints(args.phi, float), args.mode,
                              args.precision, args.domain, _ints(args.seeds, int))
    _emit(sweep_csv(rows), args.out)
    return 0


def _params(args, b, p):
    from .perfmodel import PerfParams

    return PerfParams(bandwidth=b, int8_ops=p, m=args.m, n=args.n, k=args.k,
                      num_moduli=args.num_moduli, mode=args.mode, precision=args.precision,
                      correction=args.correction)


def _perfmodel(args) -> int:
    from . import perfmodel as pm

    if args.b200:
        pp = pm.b200_params(args.m, args.n, args.k, args.num_moduli, args.mode, args.precision)
        t, tf = pm.predict_time_fused(pp), pm.predicted_tflops_fused(pp)
    else:
        pp = _params(args, args.b, args.p)
        t, tf = pm.predict_time(pp), pm.predicted_tflops(pp)
    _emit(f"seconds,tflops\n{t!r},{tf!r}\n", args.out)
    return 0


def _heatmap(args) -> int:
    from .perfmodel import heatmap_csv, heatmap_grid

    rows = heatmap_grid((args.b_min, args.b_max), (args.p_min, args.p_max),
                        (args.b_steps, args.p_steps), _params(args, args.b_min, args.p_min))
    _emit(heatmap_csv(rows), args.out)
    return 0


_RUN = {"gen": _gen, "emulate": _emulate, "accuracy": _accuracy, "perfmodel": _perfmodel,
        "heatmap": _heatmap}


def cli_dispatch(argv) -> int:
    """One CLI invocation -> exit status (cli.py:179-190)."""
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    from ._native import NativeError

    try:
        return _RUN[args.command](args)
    except (OSError, ValueError, ArithmeticError, NativeError) as exc:
        print(f"crtgemm: error: {exc}", file=sys.stderr)
        return 1


def main() -> None:
    sys.exit(cli_dispatch(sys.argv[1:]))


if __name__ == "__main__":
    main()
