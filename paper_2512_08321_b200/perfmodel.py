"""Analytic time / throughput model (pkg/src/crtgemm/perfmodel.py:1-120), plus its
B200 calibration.

`PerfParams`, `predict_time`, `predicted_tflops`, `heatmap_grid` and
`heatmap_csv` are the reference's model with the same formulas, validation
(`ConfigError`) and CSV text: time = bytes / b + INT8 ops / p, where the
bytes term is the paper's unfused pipeline (INT32 products and int8 residue
stacks round-tripping through memory, c = overhead term, default N) and the
ops term is 6 N m n k (fast) or 6 (N+1) m n k (accurate).

`fused_bytes` is the traffic of THIS implementation: residues
are written once and read by the GEMM, INT32 products never leave TMEM, so the
m n term is 4N (int8 e_re, e_im written and read back) + the output instead
of the paper's 16N.  `b200_params` returns a `PerfParams` whose b and p are the
measured B200 figures (HBM copy bandwidth and in-step INT8 rate under the
board's power cap, MEASURED_PEAKS.json / profiles/), and `predict_time_fused`
evaluates the fused model with them; DESIGN.md compares both against the
measured configs.
"""

from __future__ import annotations

import io
from dataclasses import dataclass, replace

import numpy as np

from .errors import ConfigError

# measured on this pool's B200s (MEASURED_PEAKS.json: HBM copy 6536.4 GB/s; dense
# bf16 1357.7 TF/s sustained -> INT8 2x); the emulation GEMM itself sustains
# 2.2-2.9 POPS inside a long step at the sw_power_cap clock (profiles/)
B200_HBM_BYTES_PER_S = 6.5364e12
B200_INT8_OPS_PER_S = 2.7154e15


@dataclass(frozen=True)
class PerfParams:
    """Inputs of the analytic model (perfmodel.py:17-58)."""

    bandwidth: float
    int8_ops: float
    m: int
    n: int
    k: int
    num_moduli: int
    mode: str = "accurate"
    precision: str = "double"
    correction: float | None = None

    def __post_init__(self):
        if self.bandwidth <= 0 or self.int8_ops <= 0:
            raise ConfigError("bandwidth and int8_ops must be positive")
        if min(self.m, self.n, self.k) <= 0:
            raise ConfigError("dimensions must be positive")
        if self.num_moduli < 1:
            raise ConfigError("num_moduli must be >= 1")
        if self.mode not in ("fast", "accurate"):
            raise ConfigError("mode must be 'fast' or 'accurate'")
        if self.precision not in ("single", "double"):
            raise ConfigError("precision must be 'single' or 'double'")
        if self.correction is not None and self.correction < 0:
            raise ConfigError("correction must be >= 0")

    @property
    def c(self) -> float:
        return float(self.num_moduli) if self.correction is None else float(self.correction)


def _ops(pp: PerfParams) -> int:
    n_eff = pp.num_moduli + (1 if pp.mode == "accurate" else 0)
    return 6 * n_eff * pp.m * pp.n * pp.k


def model_bytes(pp: PerfParams) -> float:
    """Memory traffic of the paper's pipeline (perfmodel.py:63-78)."""
    N, c, m, n, k = pp.num_moduli, pp.c, pp.m, pp.n, pp.k
    dbl = pp.precision == "double"
    if pp.mode == "fast":
        per_k, per_vec = (32 if dbl else 16), 4
        per_mn = 16 * N + (16 if dbl else 8) + 2 * c
    else:
        per_k, per_vec = (35 if dbl else 19), 8
        per_mn = 16 * N + (40 if dbl else 32) + 2 * c
    return ((3 * N + per_k + c) * k + per_vec) * (m + n) + per_mn * m * n


def predict_time(pp: PerfParams) -> float:
    """Predicted seconds (perfmodel.py:61-80)."""
    return model_bytes(pp) / pp.bandwidth + _ops(pp) / pp.int8_ops


def predicted_tflops(pp: PerfParams) -> float:
    """8 m n k / time * 1e-12 (perfmodel.py:83-85)."""
    return 8.0 * pp.m * pp.n * pp.k / predict_time(pp) * 1e-12


def heatmap_grid(b_range, p_range, steps, template: PerfParams):
    """(bandwidth, int8_ops, tflops) rows, bandwidth-major (perfmodel.py:88-111)."""
    b_steps, p_steps = (steps, steps) if isinstance(steps, int) else steps
    if b_steps < 1 or p_steps < 1:
        raise ConfigError("steps must be >= 1")
    (b_lo, b_hi), (p_lo, p_hi) = b_range, p_range
    if b_lo <= 0 or p_lo <= 0 or b_hi < b_lo or p_hi < p_lo:
        raise ConfigError("ranges must be positive and ordered")
    rows = []
    for b in np.linspace(b_lo, b_hi, b_steps):
        for p in np.linspace(p_lo, p_hi, p_steps):
            pp = replace(template, bandwidth=float(b), int8_ops=float(p))
            rows.append((float(b), float(p), predicted_tflops(pp)))
    return rows


def heatmap_csv(rows) -> str:
    """`b,p,tflops` CSV with repr() floats (perfmodel.py:114-120)."""
    out = io.StringIO()
    out.write("b,p,tflops\n")
    for b, p, tf in rows:
        out.write(f"{b!r},{p!r},{tf!r}\n")
    return out.getvalue()


# ---------------------------------------------------------------- B200 fused model

def fused_bytes(pp: PerfParams) -> float:
    """Algorithmic HBM bytes of this implementation.

    s = bytes per complex input element (16 double / 8 single):
      inputs read twice (scaling, residues)      2 s k (m + n)
      int8 residue planes written (re, im, sum)  3 N k (m + n)
      e_re / e_im written by K3, read by the CRT 4 N m n
      output written                             s m n
    (the GEMM's operand reads are charged to its INT8 term: at these tile
    sizes they are L2-served, profiles/r01_gemm_raster_experiment.json)
    accurate mode adds the bound-GEMM operands (ceil-quantised, 3 planes) and
    one more input pass: (s + 3) k (m + n).
    """
    N, m, n, k = pp.num_moduli, pp.m, pp.n, pp.k
    s = 16 if pp.precision == "double" else 8
    b = (2 * s + 3 * N) * k * (m + n) + (4 * N + s) * m * n
    if pp.mode == "accurate":
        b += (s + 3) * k * (m + n)
    return float(b)


def b200_params(m: int, n: int, k: int, num_moduli: int, mode: str = "fast",
                precision: str = "double") -> PerfParams:
    """PerfParams with the measured B200 bandwidth and in-step INT8 rate."""
    return PerfParams(bandwidth=B200_HBM_BYTES_PER_S, int8_ops=B200_INT8_OPS_PER_S, m=m, n=n, k=k,
                      num_moduli=num_moduli, mode=mode, precision=precision)


def predict_time_fused(pp: PerfParams) -> float:
    """Seconds for the fused B200 pipeline: fused bytes / b + INT8 ops / p."""
    return fused_bytes(pp) / pp.bandwidth + _ops(pp) / pp.int8_ops


def predicted_tflops_fused(pp: PerfParams) -> float:
    return 8.0 * pp.m * pp.n * pp.k / predict_time_fused(pp) * 1e-12
