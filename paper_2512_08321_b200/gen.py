"""Deterministic test matrices — the reference generator (pkg/src/crtgemm/bench.py:28-70).

Entry (column-major index e) of each real part is (u - 0.5) * exp(z * phi) with
  u = ((raw >> 11) + 1) * 2^-53            uniform on (0, 1]
  z = ndtri(((raw >> 11) + 0.5) * 2^-53)   standard normal (inverse CDF)
drawn from numpy's Philox(seed) raw 64-bit stream: all uniforms of the real
part, then its normals, then (complex) the imaginary part's uniforms and
normals.  The same (rows, cols, phi, seed, precision, domain) always yields the
same matrix bit for bit, which is what makes the CLI `gen` files and the
accuracy sweeps reproducible against the reference.

This is host-side input generation (numpy + scipy's ndtri), not part of the
emulation path: `exp` and `ndtri` have no bit-exact device equivalent, and the
benchmark draws its large inputs on the device instead (bench.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError


@dataclass(frozen=True)
class GenSpec:
    """Shape, dynamic-range parameter and stream seed of one matrix (bench.py:28-47)."""

    rows: int
    cols: int
    phi: float = 0.0
    seed: int = 0
    precision: str = "double"
    domain: str = "real"

    def __post_init__(self):
        if self.rows < 1 or self.cols < 1:
            raise ConfigError("matrix dimensions must be positive")
        if self.phi < 0:
            raise ConfigError("phi must be >= 0")
        if self.precision not in ("single", "double"):
            raise ConfigError("precision must be 'single' or 'double'")
        if self.domain not in ("real", "complex"):
            raise ConfigError("domain must be 'real' or 'complex'")


def _part(raw_u: np.ndarray, raw_z: np.ndarray, phi: float, shape) -> np.ndarray:
    scale = 2.0 ** -53
    from scipy.special import ndtri

    u = ((raw_u >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * scale
    z = ndtri(((raw_z >> np.uint64(11)).astype(np.float64) + 0.5) * scale)
    return ((u - 0.5) * np.exp(z * phi)).reshape(shape, order="F")


def gen_matrix(gs: GenSpec) -> np.ndarray:
    """The reference's matrix for `gs` (bench.py:57-70), Fortran-ordered."""
    count = gs.rows * gs.cols
    parts = 4 if gs.domain == "complex" else 2
    raw = np.random.Philox(gs.seed).random_raw(parts * count)
    shape = (gs.rows, gs.cols)
    re = _part(raw[:count], raw[count:2 * count], gs.phi, shape)
    if gs.domain == "real":
        return re.astype(np.float32 if gs.precision == "single" else np.float64)
    im = _part(raw[2 * count:3 * count], raw[3 * count:], gs.phi, shape)
    # assembled as re + 1j*im like the reference: real = re + (0*im - 0),
    # imag = 0 + (0 + im) -> identical to complex(re, im) except signed zeros,
    # so keep the same expression
    out = re + 1j * im
    return out.astype(np.complex64 if gs.precision == "single" else np.complex128)
