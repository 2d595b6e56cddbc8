#!/usr/bin/env python
"""Benchmark of the emulated complex GEMM (Ozaki-II / CRT on INT8 tcgen05).

Workload (BASELINE.json metric "emulated ZGEMM/CGEMM TFLOPS at m=n=k=16384 vs
cuBLAS native; max rel. error"): ZGEMM m=n=k=16384 per GPU, fast mode, N=15
moduli, phi=0.5 synthetic inputs (configs[2]).  N=15 is the smallest count whose
max relative error over the full product is below cuBLAS native's at this shape
(profiles/r01_accuracy_full_16384.json: N=14 2.0e-6, N=15 1.2e-7, native 6.4e-7);
the line also times N=14 (the reference's EmuConfig default) and measures both
errors live against the GPU double-double reference.  A "step" is one full emulated product
C = A @ B: scaling + residues + 3N tcgen05 INT8 GEMMs + CRT.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...

Multi-GPU: weak scaling by output tiles — rank r owns an A row-block and a B
column-block (R x C grid) of a (16384 R) x (16384 C) x 16384 product and
computes its C tile; fast mode needs no collective on the data path.

`--impl reference` times the reference algorithm's CPU implementation (the
numpy port in oracle/, float64-BLAS "INT8 engine" like the reference) on a
bounded row/column-local sample of the same product on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = ("emulated ZGEMM TFLOPS (8mnk/t) at m=n=k=16384 per GPU, fast mode, 15 moduli "
          "(max rel. error <= cuBLAS native)")
UNIT = "TFLOPS"
METRIC_STRONG = ("emulated ZGEMM TFLOPS (8mnk/t) of one m=n=k=32768 product sharded by output "
                 "tiles (cfg5), scatter + compute + gather per step")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--shape", type=int, nargs=3, default=[16384, 16384, 16384],
                    metavar=("M", "N", "K"), help="per-GPU m n k")
    ap.add_argument("--moduli", type=int, default=15)
    ap.add_argument("--mode", choices=("fast", "accurate"), default="fast")
    ap.add_argument("--precision", choices=("double", "single"), default="double")
    ap.add_argument("--phi", type=float, default=0.5)
    ap.add_argument("--n-block", type=int, default=8192)
    ap.add_argument("--no-native", action="store_true", help="skip the cuBLAS native timing")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-accuracy", action="store_true",
                    help="skip the live max-relative-error check (GPU double-double reference)")
    ap.add_argument("--strong", action="store_true",
                    help="cfg5 strong scaling: ONE product of --shape (default 32768^3) sharded "
                         "by output tiles over the ranks; rank 0 holds A and B, scatters the "
                         "row / column blocks and gathers C over NCCL inside the timed step")
    ap.add_argument("--no-strong", action="store_true",
                    help="N>1: skip the cfg5 strong-scaling (one sharded 32768^3 product) leg")
    ap.add_argument("--strong-size", type=int, default=32768)
    ap.add_argument("--strong-steps", type=int, default=3)
    ap.add_argument("--strong-warmup", type=int, default=1)
    ap.add_argument("--cpu-sample", type=int, default=64,
                    help="rows/cols of the CPU sample block (k kept full)")
    ap.add_argument("--no-cpu-cfg1", action="store_true",
                    help="reference arm: skip the full cfg1 (1024^3) CPU runs")
    a = ap.parse_args()
    if a.strong and a.shape == [16384, 16384, 16384]:
        a.shape = [32768, 32768, 32768]
    a.m, a.n, a.k = a.shape
    return a


def workload_name(a) -> str:
    kind = "zgemm" if a.precision == "double" else "cgemm"
    return f"{kind}_{a.m}x{a.n}x{a.k}_{a.mode}_N{a.moduli}"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        self.rows = [r for r in self.rows if len(r) >= 9]  # skip error / partial lines
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# --------------------------------------------------------------------------- helpers
def peaks():
    """(bf16 burst, bf16 sustained, HBM GB/s, source) from MEASURED_PEAKS.json,
    else the profiling guide's fallback (1590 burst / ~1400 sustained / 6650)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return (p.get("bf16_tflops", 1590.0), p.get("bf16_tflops_sustained", 1400.0),
                p.get("hbm_gbs", 6650.0), "measured")
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def int8_peak():
    """Measured cuBLASLt INT8 16384^3 rate on this pool (tools/int8_peak.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "int8_peak.json")) as f:
            p = json.load(f)
        return {k: p[k] for k in ("int8_tops_burst", "int8_tops_sustained",
                                  "sm_mhz_median_sustained")}
    except Exception:
        return None


def profile_traffic():
    """Per-launch DRAM bytes of the GEMM from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def fingerprint(torch, t) -> int:
    """Order-independent 64-bit signature of a tensor's bytes (wrapping int64 sum
    of its words and of the words times their index)."""
    w = t.reshape(-1).view(torch.int64)
    idx = torch.arange(w.numel(), device=w.device, dtype=torch.int64)
    return (int(w.sum().item()) ^ (int((w * idx).sum().item()) << 1)) & ((1 << 64) - 1)


def synth(torch, rows, cols, phi, seed, dtype, dev):
    """(u - 0.5) * exp(z * phi) per part, the reference generator's distribution
    (bench.py:50-54 there), drawn on the device."""
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    real = torch.float64 if dtype == torch.complex128 else torch.float32
    parts = []
    for _ in range(2):
        u = torch.rand((rows, cols), generator=g, device=dev, dtype=real)
        z = torch.randn((rows, cols), generator=g, device=dev, dtype=real)
        parts.append((u - 0.5) * torch.exp(z * phi))
    return torch.complex(parts[0], parts[1]).to(dtype)


# --------------------------------------------------------------------------- CPU leg
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def load_reference():
    """The UNMODIFIED reference package `crtgemm`, pip-installed into
    baseline/_ref.  -> (module, kind); falls back to the
    oracle port (kind "port") only if the install is absent."""
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "crtg_numba_cache"))
    if os.path.isdir(os.path.join(REF_DIR, "crtgemm")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        try:
            import crtgemm  # noqa: F401
            return crtgemm, "reference"
        except Exception as e:  # pragma: no cover - reported in the line
            print(f"reference import failed ({e!r}); timing the oracle port", file=sys.stderr)
    return None, "port"


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _ref_call(ref, kind, A, B, a, num_moduli, mode, prec):
    if kind == "reference":
        cfg = ref.EmuConfig(precision=prec, domain="complex", mode=mode, num_moduli=num_moduli)
        return ref.emulate_gemm_complex(A, B, cfg)
    from oracle import ozaki2 as orc
    return orc.emulate_complex(A, B, num_moduli, mode, prec)


def _ref_inputs(ref, kind, rows, k, cols, phi, prec, seed):
    if kind == "reference":
        A = ref.gen_matrix(ref.GenSpec(rows, k, phi, seed, prec, "complex"))
        B = ref.gen_matrix(ref.GenSpec(k, cols, phi, seed + 1, prec, "complex"))
        return A, B
    from oracle import ozaki2 as orc
    return orc.gen_matrix(rows, k, phi, seed, prec), orc.gen_matrix(k, cols, phi, seed + 1, prec)


def cpu_sample(a, reps: int = 1, ref=None, kind=None):
    """The reference's own CPU implementation (crtgemm.emulate_gemm_complex from
    baseline/_ref: numpy + OpenBLAS + numba on all host threads) on a bounded
    row/column-local block `s x s x k` of the same product (k kept full; fast
    mode's exponents are row/column local, so the block is the same work per
    output element as the full product)."""
    if ref is None and kind is None:
        ref, kind = load_reference()
    s = min(a.cpu_sample, a.m, a.n)
    prec = a.precision
    A, B = _ref_inputs(ref, kind, s, a.k, s, a.phi, prec, 11)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        _ref_call(ref, kind, A, B, a, a.moduli, a.mode, prec)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return {"value": 8.0 * s * s * a.k / t / 1e12, "unit": UNIT, "cores": os.cpu_count(),
            "kind": kind, "cpu_model": cpu_model(),
            "impl": ("crtgemm.emulate_gemm_complex (unmodified reference, baseline/_ref)"
                     if kind == "reference" else "oracle port (reference not installed)"),
            "sample": f"{s}x{s}x{a.k} block of the {a.m}x{a.n}x{a.k} product "
                      f"({a.mode}, N={a.moduli}, phi={a.phi}), median of {reps}, "
                      f"{t:.2f} s each, on {os.cpu_count()} host threads"}


def cpu_cfg1(ref, kind):
    """BASELINE.md section 2's CPU reference run: cfg1 = ZGEMM 1024^3, N=14,
    phi=0.5, seeds 0/1, fast and accurate, the FULL product (one call each
    after a warm-up call)."""
    A, B = _ref_inputs(ref, kind, 1024, 1024, 1024, 0.5, "double", 0)
    res = {}
    for mode in ("fast", "accurate"):
        _ref_call(ref, kind, A, B, None, 14, mode, "double")
        t0 = time.perf_counter()
        _ref_call(ref, kind, A, B, None, 14, mode, "double")
        t = time.perf_counter() - t0
        res[mode] = {"seconds": t, "tflops": 8.0 * 1024 ** 3 / t / 1e12}
    return {"workload": "zgemm_1024x1024x1024_N14 (cfg1), full product", **res}


def run_reference(a, rank: int):
    """`--impl reference`: the reference's own CPU path on the host cores, rank 0
    only (other ranks exit without work)."""
    if rank != 0:
        return
    ref, kind = load_reference()
    for _ in range(max(1, a.warmup)):
        cpu_sample(a, ref=ref, kind=kind)  # warm numpy / BLAS / numba
    vals = []
    for _ in range(a.steps):
        vals.append(cpu_sample(a, ref=ref, kind=kind)["value"])
    v = statistics.median(vals)
    base = cpu_sample(a, ref=ref, kind=kind)
    s = min(a.cpu_sample, a.m, a.n)
    ms = 8.0 * s * s * a.k / (v * 1e12) * 1e3
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64" if a.precision == "double" else "f32",
            "data": "synthetic (reference generator, Philox + ndtri)",
            "config": {"workload": workload_name(a), "m": a.m, "n": a.n, "k": a.k,
                       "num_moduli": a.moduli, "mode": a.mode, "precision": a.precision,
                       "phi": a.phi},
            "impl": "reference",
            "cpu_baseline": {**base, "value": v,
                             "sample": f"each step: {base['sample'].split(', median')[0]}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not a.no_cpu_cfg1:
        line["cpu_baseline"]["cfg1"] = cpu_cfg1(ref, kind)
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU leg
def run_ours(a, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    import paper_2512_08321_b200 as crt
    from paper_2512_08321_b200 import _native as nat

    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", local_rank % max(ndev, 1))
    torch.cuda.set_device(dev)
    init_dist(world, dev)
    # 2-D grid of output tiles for weak scaling
    R = 1 << (int(math.log2(world)) // 2)
    Cc = world // R
    r_i, c_i = rank // Cc, rank % Cc

    cdt = torch.complex128 if a.precision == "double" else torch.complex64
    A = synth(torch, a.m, a.k, a.phi, 1000 + r_i, cdt, dev)
    B = synth(torch, a.k, a.n, a.phi, 2000 + c_i, cdt, dev)
    cfg = crt.EmuConfig(precision=a.precision, domain="complex", mode=a.mode,
                        num_moduli=a.moduli, n_block=a.n_block)
    ws = None
    out = torch.empty((a.m, a.n), dtype=cdt, device=dev)

    emu = None
    if world > 1 and a.mode == "accurate":
        # accurate mode: exponents are global over the grid row / column -> the
        # MAX all-reduce of the bound maxima (dist.ShardedEmulator)
        from paper_2512_08321_b200 import dist as cdist
        emu = cdist.ShardedEmulator(cfg, cdist.TileGrid(R, Cc), rank)

    def step():
        if emu is not None:
            out.copy_(emu.tile(A, B, sync_check=False))
            return
        crt.run_complex(A, B, cfg, None, dev, sync_check=False, ws=ws_holder[0], out=out)

    ws_holder = [None]
    lib = nat.load()
    need = lib.crtg_workspace_size((1 if a.precision == "single" else 0)
                                   | (16 if cdt == torch.complex64 else 0),
                                   0 if a.mode == "fast" else 1, a.m, a.n, a.k, a.moduli,
                                   a.n_block)
    ws_holder[0] = torch.empty(need, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(a.warmup):
        step()
    barrier()
    nat.profile_enable(True)
    nat.profile_read()  # clear
    launches0 = nat.launch_count()
    sampler = ClockSampler(dev.index)
    sampler.start()
    stream = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    launches = nat.launch_count() - launches0
    stage_ms, stage_n = nat.profile_read()
    nat.profile_enable(False)
    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        on_dev = dist.get_backend() == "nccl"
        t = torch.tensor([x], dtype=torch.float64, device=dev if on_dev else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_total = max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms_total / a.steps
    flops_step = 8.0 * a.m * a.n * a.k * world
    value = flops_step / (ms_step * 1e-3) / 1e12

    # roofline of the dominant kernel (K3 tcgen05 GEMM): INT8 ops the tensor
    # cores execute per launch = 2 * m * n_block * k * sum_l products_l, with 3
    # products per modulus (Karatsuba) or 2 for a modulus with a square root of
    # -1 (split form); the reference's perf model counts 6 * N * mnk
    bf16, bf16_sus, hbm, src = peaks()
    launches_gemm = max(1, stage_n["gemm"])
    gemm_ms = stage_ms["gemm"] / launches_gemm
    prods = sum(crt.moduli.products_per_modulus(crt.select_moduli(a.moduli)))
    ops_launch = 2.0 * prods * a.m * a.n * a.k * a.steps / launches_gemm
    ops_model = 6.0 * a.moduli * a.m * a.n * a.k * a.steps / launches_gemm
    achieved = ops_launch / (gemm_ms * 1e-3) / 1e12
    # Denominator: K3 runs inside a long, power-capped step, so the SUSTAINED
    # figure applies: B200 dense INT8 = 2 x dense BF16, i.e. 2 x the measured
    # sustained bf16 rate of MEASURED_PEAKS.json.  `achieved` counts the
    # ALGORITHMIC ops of SURVEY section 8(d) (6 N m n_block k per launch: three
    # INT8 products per modulus); the tensor cores execute fewer (a modulus with
    # a square root of -1 needs two products), reported as frac_executed.  The
    # measured cuBLASLt INT8 rate on this pool (profiles/int8_peak.json: burst /
    # 4 s sustained at 16384^3) is reported beside it.
    peak_int8 = 2.0 * bf16_sus
    achieved_alg = ops_model / (gemm_ms * 1e-3) / 1e12
    i8 = int8_peak()
    traffic = profile_traffic()
    if traffic and [traffic.get(k) for k in ("m", "n", "k", "N", "n_block", "mode")] != \
            [a.m, a.n, a.k, a.moduli, a.n_block, a.mode]:
        traffic = None  # the committed capture is for another configuration
    roof = {"bound": "tensor", "kernel": "k_gemm_w (256x256 Karatsuba/split tiles)",
            "achieved": achieved_alg, "peak": peak_int8, "unit": "TFLOP/s",
            "op_kind": "INT8 tensor ops (one MAC = 2 ops), TOPS",
            "frac": achieved_alg / peak_int8,
            "peak_note": f"INT8 dense = 2 x {src} SUSTAINED bf16 ({bf16_sus} TF/s, "
                         "MEASURED_PEAKS.json): the kernel is timed inside a long step",
            "achieved_executed": achieved, "frac_executed": achieved / peak_int8,
            "frac_of_2x_burst_bf16": achieved_alg / (2.0 * bf16),
            "frac_of_spec_4500": achieved_alg / 4500.0,
            "cublaslt_int8_measured": i8,
            "frac_of_cublaslt_int8_sustained": (achieved_alg / i8["int8_tops_sustained"]
                                                if i8 else None),
            "ops_per_launch": ops_model, "executed_ops_per_launch": ops_launch,
            "ms_per_launch": gemm_ms, "int8_products_per_step": prods,
            "ops_note": f"algorithmic 6*N*m*n_block*k per launch (SURVEY 8(d)); executed: "
                        f"{prods} products of m x n_block x k per step (3N = {3 * a.moduli} "
                        "Karatsuba, minus one per split modulus)",
            "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
            "traffic_note": traffic.get("config") if traffic else None}
    stages = {k: v / a.steps for k, v in stage_ms.items()}

    result = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
              "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step,
              "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
              "dtype": "int8 tensor / f64" if a.precision == "double" else "int8 tensor / f32",
              "data": "synthetic (u-0.5)*exp(z*phi), drawn on device",
              "config": {"workload": workload_name(a), "m": a.m, "n": a.n, "k": a.k,
                         "num_moduli": a.moduli, "mode": a.mode, "precision": a.precision,
                         "phi": a.phi, "n_block": a.n_block, "grid": f"{R}x{Cc}",
                         "parallelism": f"output-tile x{world}",
                         "l2": f"inputs ({A.numel() * A.element_size() / 2**30:.2f} GiB and "
                               f"{B.numel() * B.element_size() / 2**30:.2f} GiB) vs 126 MB L2; "
                               "no flush"},
              "stage_ms_per_step": stages, "gpu_launches": int(launches),
              "roofline": roof, "clocks": clocks}

    # cuBLAS native baseline on the same device (rank 0)
    # fingerprint of the emulated result: nothing below may write into `out`
    # (asserted before its error is computed)
    out_sig = fingerprint(torch, out)
    if rank == 0 and not a.no_native:
        torch.backends.cuda.matmul.allow_tf32 = False
        nat_out = torch.empty_like(out)  # cuBLAS writes its own buffer
        for _ in range(2):
            torch.matmul(A, B, out=nat_out)
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        reps = 3
        f0.record(stream)
        for _ in range(reps):
            torch.matmul(A, B, out=nat_out)
        f1.record(stream)
        torch.cuda.synchronize()
        nat_ms = f0.elapsed_time(f1) / reps
        nat_tf = 8.0 * a.m * a.n * a.k / (nat_ms * 1e-3) / 1e12
        result["native_cublas"] = {"op": "torch.matmul " + str(cdt).replace("torch.", ""),
                                   "ms": nat_ms, "tflops": nat_tf,
                                   "speedup_per_gpu": (value / world) / nat_tf}
    else:
        nat_out = None

    # the reference's EmuConfig default (N=14) on the same inputs, for context
    if rank == 0 and a.moduli != 14 and a.precision == "double" and a.mode == "fast":
        cfg14 = crt.EmuConfig(precision="double", domain="complex", mode="fast", num_moduli=14,
                              n_block=a.n_block)
        out14 = torch.empty_like(out)
        for _ in range(2):
            crt.run_complex(A, B, cfg14, None, dev, sync_check=False, ws=ws_holder[0], out=out14)
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(3):
            crt.run_complex(A, B, cfg14, None, dev, sync_check=False, ws=ws_holder[0], out=out14)
        g1.record(stream)
        torch.cuda.synchronize()
        ms14 = g0.elapsed_time(g1) / 3
        result["variant_N14"] = {"ms_per_step": ms14, "value": flops_step / world / (ms14 * 1e-3) / 1e12}
    else:
        out14 = None

    # accuracy, live: the reference's metric over EVERY entry against the GPU
    # double-double product (bit-identical to reference_gemm_dd)
    if rank == 0 and world == 1 and not a.no_accuracy:
        from paper_2512_08321_b200 import accuracy as acc
        t0 = time.time()
        ref = acc.reference_gemm_dd(A.to(torch.complex128), B.to(torch.complex128))
        torch.cuda.synchronize()
        t_dd = time.time() - t0
        native = nat_out if nat_out is not None else torch.matmul(A, B)
        if fingerprint(torch, out) != out_sig:
            raise RuntimeError("the emulated result buffer changed after the timed steps")
        if torch.equal(out, native):
            raise RuntimeError("accuracy leg: emulated and cuBLAS results are the same tensor")
        accr = {"metric": "max relative error over all entries (reference oracle.py:131-169)",
                "reference": "GPU double-double GEMM, bit-identical to reference_gemm_dd",
                "emulated": acc.max_relative_error(out, ref),
                "native_cublas": acc.max_relative_error(native, ref), "dd_seconds": t_dd,
                "emulated_buffer": f"written only by the timed steps (fingerprint {out_sig:#x} "
                                   "checked); cuBLAS wrote a separate buffer"}
        if out14 is not None:
            accr["emulated_N14"] = acc.max_relative_error(out14, ref)
        accr["emulated_le_native"] = accr["emulated"] <= accr["native_cublas"]
        result["accuracy"] = accr
        del ref, native, nat_out
        torch.cuda.empty_cache()

    # the north star's CGEMM target at the same shape: emulated CGEMM (complex64,
    # fast, N=8 -- the reference's default for single precision) vs cuBLAS CGEMM
    if rank == 0 and world == 1 and a.precision == "double" and not a.no_native:
        Ac, Bc = A.to(torch.complex64), B.to(torch.complex64)
        cfgc = crt.EmuConfig(precision="single", domain="complex", mode="fast", num_moduli=8,
                             n_block=a.n_block)
        outc = torch.empty((a.m, a.n), dtype=torch.complex64, device=dev)
        wsc = torch.empty(lib.crtg_workspace_size(1 | 16, 0, a.m, a.n, a.k, 8, a.n_block),
                          dtype=torch.uint8, device=dev)

        def time_it(fn, reps):
            fn()
            torch.cuda.synchronize()
            t0e = torch.cuda.Event(enable_timing=True)
            t1e = torch.cuda.Event(enable_timing=True)
            t0e.record(stream)
            for _ in range(reps):
                fn()
            t1e.record(stream)
            torch.cuda.synchronize()
            return t0e.elapsed_time(t1e) / reps

        msc = time_it(lambda: crt.run_complex(Ac, Bc, cfgc, None, dev, sync_check=False, ws=wsc,
                                              out=outc), 3)
        msn = time_it(lambda: torch.matmul(Ac, Bc), 2)
        vc = {"ms_per_step": msc, "value": flops_step / (msc * 1e-3) / 1e12,
              "native_cublas_ms": msn, "native_cublas_tflops": flops_step / (msn * 1e-3) / 1e12,
              "speedup": msn / msc,
              "config": f"cgemm_{a.m}x{a.n}x{a.k}_fast_N8 (complex64 copies of the same inputs)"}
        del wsc
        if not a.no_accuracy:
            # reference: the emulated ZGEMM at N=20 of the same complex64 values
            # (max relative error ~1e-14 at this shape, far below either fp32 error)
            from paper_2512_08321_b200 import accuracy as acc
            cfg20 = crt.EmuConfig(precision="double", domain="complex", mode="fast",
                                  num_moduli=20, n_block=a.n_block)
            refc = crt.run_complex(Ac.to(torch.complex128), Bc.to(torch.complex128), cfg20, None,
                                   dev)
            vc["accuracy"] = {
                "metric": "max relative error over all entries vs emulated ZGEMM N=20 of the "
                          "same complex64 inputs",
                "emulated": acc.max_relative_error(outc, refc),
                "native_cublas": acc.max_relative_error(torch.matmul(Ac, Bc), refc)}
            vc["accuracy"]["emulated_le_native"] = (vc["accuracy"]["emulated"]
                                                    <= vc["accuracy"]["native_cublas"])
            # entrywise maxima are dominated by near-cancelled entries at fp32;
            # the normwise error is the usual single-precision yardstick
            rn = torch.linalg.norm(refc).item()
            vc["accuracy"]["normwise_emulated"] = (
                torch.linalg.norm(outc.to(torch.complex128) - refc).item() / rn)
            vc["accuracy"]["normwise_native"] = (
                torch.linalg.norm(torch.matmul(Ac, Bc).to(torch.complex128) - refc).item() / rn)
            del refc
        result["variant_cgemm_N8"] = vc
        del Ac, Bc, outc
        torch.cuda.empty_cache()

    # end to end through the public API with host buffers (rank 0 shape per rank)
    if not a.no_e2e:
        hA = A.cpu().pin_memory()
        hB = B.cpu().pin_memory()
        hC = torch.empty((a.m, a.n), dtype=cdt).pin_memory()
        cfg_e = crt.EmuConfig(precision=a.precision, domain="complex", mode=a.mode,
                              num_moduli=a.moduli, n_block=a.n_block)

        def e2e_step():
            # pinned host tensors in -> pinned host tensor out (H2D/D2H inside)
            return crt.emulate_gemm_complex(hA, hB, cfg_e)

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        reps = max(1, min(a.steps, 3))
        for _ in range(reps):
            e2e_step()
        barrier()
        dt = max_over_ranks((time.perf_counter() - t0) / reps)
        result["e2e"] = {"value": flops_step / dt / 1e12, "unit": UNIT,
                         # whole job: every rank streams its own operands / tile
                         "h2d_bytes_per_step": world * int(hA.numel() * hA.element_size()
                                                           + hB.numel() * hB.element_size()),
                         "d2h_bytes_per_step": world * int(hC.numel() * hC.element_size()),
                         "ms_per_step": dt * 1e3,
                         "api": "paper_2512_08321_b200.emulate_gemm_complex(pinned host tensors)"
                                " -> crtg_gemm_complex_host (A row chunks / B column blocks streamed in a staircase, C tiles back, on the copy engines)"}

    # cfg5 (BASELINE configs[4]) at N > 1: ONE 32768^3 product sharded by output
    # tiles, NCCL scatter + tiles + gather inside each step
    if world > 1 and not a.no_strong:
        del A, B, out
        ws_holder[0] = None
        torch.cuda.empty_cache()
        m5 = a.strong_size
        result["strong_cfg5"] = strong_measure(a, rank, world, dev, m5, m5, m5,
                                               a.strong_steps, a.strong_warmup,
                                               sample_clocks=False)

    if rank == 0 and world == 1 and not a.no_cpu:
        result["cpu_baseline"] = cpu_sample(a, reps=1)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def init_dist(world: int, dev):
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        # NCCL over NVLink on the box; CRTG_BENCH_BACKEND=gloo lets the multi-rank
        # logic be exercised with several ranks sharing one GPU (CI only)
        backend = os.environ.get("CRTG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)


def strong_measure(a, rank: int, world: int, dev, m: int, n: int, k: int, steps: int,
                   warmup: int, sample_clocks: bool = True) -> dict:
    """cfg5: one (m x k) @ (k x n) product sharded by output tiles over `world`
    ranks (paper_2512_08321_b200.dist).  The timed step is what a caller of the
    sharded product pays with operands resident on rank 0: scatter of A's row
    blocks and B's column blocks (NCCL over NVLink), each rank's tile (accurate
    mode: with the MAX all-reduce of the bound maxima), gather of C to rank 0
    (grouped receives).  Tile compute alone is reported beside it."""
    import torch
    import torch.distributed as dist

    import paper_2512_08321_b200 as crt
    from paper_2512_08321_b200 import _native as nat
    from paper_2512_08321_b200 import dist as cdist

    grid = cdist.TileGrid.for_world(world)
    cdt = torch.complex128 if a.precision == "double" else torch.complex64
    cfg = crt.EmuConfig(precision=a.precision, domain="complex", mode=a.mode,
                        num_moduli=a.moduli, n_block=a.n_block)
    A = B = None
    if rank == 0:
        A = synth(torch, m, k, a.phi, 1000, cdt, dev)
        B = synth(torch, k, n, a.phi, 2000, cdt, dev)
    emu = cdist.ShardedEmulator(cfg, grid, rank) if world > 1 else None
    groups = emu.groups if (emu and emu.groups) else (
        cdist.TileGroups(grid, rank) if world > 2 else None)
    tile_ms = []

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step():
        if world == 1:
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            crt.run_complex(A, B, cfg, None, dev, sync_check=False)
            t1.record()
            tile_ms.append((t0, t1))
            return
        a_loc, b_loc = cdist.scatter_operands(A, B, grid, rank, m, n, k, cdt, dev,
                                              groups=groups)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        c_loc = emu.tile(a_loc, b_loc, sync_check=False)
        t1.record()
        tile_ms.append((t0, t1))
        cdist.gather_tiles(c_loc, grid, rank, m, n)

    for _ in range(warmup):
        step()
    barrier()
    tile_ms.clear()
    launches0 = nat.launch_count()
    sampler = ClockSampler(dev.index) if sample_clocks else None
    if sampler:
        sampler.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    barrier()
    clocks = sampler.stop() if sampler else None
    launches = nat.launch_count() - launches0

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        on_dev = dist.get_backend() == "nccl"
        t = torch.tensor([x], dtype=torch.float64, device=dev if on_dev else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_step = max_over_ranks(e0.elapsed_time(e1)) / steps
    ms_tile = max_over_ranks(sum(x.elapsed_time(y) for x, y in tile_ms)) / steps
    flops = 8.0 * m * n * k
    kind = "zgemm" if a.precision == "double" else "cgemm"
    res = {"metric": METRIC_STRONG, "value": flops / (ms_step * 1e-3) / 1e12, "unit": UNIT,
           "n_gpus": world, "steps": steps, "warmup": warmup, "ms_per_step": ms_step,
           "higher_is_better": True, "scaling": "strong",
           "config": {"workload": f"{kind}_{m}x{n}x{k}_{a.mode}_N{a.moduli}_sharded",
                      "m": m, "n": n, "k": k, "num_moduli": a.moduli, "mode": a.mode,
                      "grid": f"{grid.R}x{grid.C}", "parallelism": f"output-tile x{world}",
                      "l2": "operands far larger than the 126 MB L2; no flush"},
           "tile_compute_ms": ms_tile,
           "tile_compute_tflops": flops / (ms_tile * 1e-3) / 1e12,
           "comm_ms": ms_step - ms_tile, "gpu_launches": int(launches)}
    if clocks is not None:
        res["clocks"] = clocks
    del A, B
    torch.cuda.empty_cache()
    return res


def run_strong(a, rank: int, world: int, local_rank: int):
    """`--strong`: the cfg5 line on its own (default 32768^3)."""
    import torch
    import torch.distributed as dist

    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", local_rank % max(ndev, 1))
    torch.cuda.set_device(dev)
    init_dist(world, dev)
    res = strong_measure(a, rank, world, dev, a.m, a.n, a.k, a.steps, a.warmup)
    res.update({"vs_baseline": None,
                "dtype": "int8 tensor / f64" if a.precision == "double" else "int8 tensor / f32",
                "data": "synthetic (u-0.5)*exp(z*phi), drawn on device (rank 0)"})
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(a.gpus if a.gpus == 1 else 1)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank)
        return
    if a.strong:
        run_strong(a, rank, world, local_rank)
        return
    run_ours(a, rank, world, local_rank)


if __name__ == "__main__":
    main()
