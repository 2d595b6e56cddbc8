"""Host-side number theory: modulus selection, CRT weights and the scaling
thresholds — exact big-integer arithmetic, done once per modulus count.

Restates reference crt.py:32-110 (`ModulusSet`, `select_moduli`) and
scaling.py:85-115 (`ScalingConstants.from_product`) and packs the result into
the `crtg_consts` struct of include/crtg.h for the device kernels.
"""

from __future__ import annotations

import ctypes
import functools
import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

MAX_MODULI = 20
_RESIDUE_BITS = 7
_DOUBLE_BITS = 53


@dataclass(frozen=True)
class ModulusSet:
    """Pairwise-coprime moduli (descending, <= 256) with CRT weights split into
    an exact high part on a shared 2^shift grid and a nearest-double low part."""

    moduli: tuple
    product: int
    log2_product: float
    inverses: tuple
    coeff_hi: np.ndarray
    coeff_lo: np.ndarray

    @classmethod
    def from_moduli(cls, moduli) -> "ModulusSet":
        moduli = tuple(sorted((int(p) for p in moduli), reverse=True))
        n = len(moduli)
        if not 1 <= n <= MAX_MODULI:
            raise ConfigError(f"need 1..{MAX_MODULI} moduli, got {n}")
        if any(not 2 <= p <= 256 for p in moduli):
            raise ConfigError("moduli must lie in [2, 256]")
        if len(set(moduli)) != n:
            raise ConfigError("moduli must be distinct")
        for i in range(n):
            for j in range(i + 1, n):
                if math.gcd(moduli[i], moduli[j]) != 1:
                    raise ConfigError(f"moduli {moduli[i]} and {moduli[j]} share a factor")
        prod = math.prod(moduli)
        grid = max(0, prod.bit_length() + _RESIDUE_BITS + (n - 1).bit_length() - _DOUBLE_BITS)
        inv, hi, lo = [], np.empty(n), np.empty(n)
        for idx, p in enumerate(moduli):
            cof = prod // p
            q = pow(cof, -1, p)
            inv.append(q)
            w = cof * q
            h = (w >> grid) << grid
            hi[idx], lo[idx] = float(h), float(w - h)
        return cls(moduli, prod, math.log2(prod), tuple(inv), hi, lo)

    def __len__(self) -> int:
        return len(self.moduli)


@functools.lru_cache(maxsize=None)
def select_moduli(num_moduli: int) -> ModulusSet:
    """Greedy descending coprime scan from 256 (reference crt.py:94-110)."""
    if not isinstance(num_moduli, int) or not 1 <= num_moduli <= MAX_MODULI:
        raise ConfigError(f"num_moduli must be in 1..{MAX_MODULI}, got {num_moduli!r}")
    chosen, cand = [256], 255
    while len(chosen) < num_moduli:
        if all(math.gcd(cand, p) == 1 for p in chosen):
            chosen.append(cand)
        cand -= 1
    return ModulusSet.from_moduli(chosen)


def has_sqrt_minus_one(p: int) -> bool:
    """True when some j has j^2 == -1 (mod p): Z[i]/p splits and the library
    forms a complex product mod p from two INT8 products instead of three
    (the e-planes are identical either way)."""
    return p % 2 == 1 and any((j * j + 1) % p == 0 for j in range(1, p))


def products_per_modulus(ms: "ModulusSet") -> list:
    """INT8 products the GPU runs per modulus in the complex pipeline: 2 for a
    split modulus, 3 (Karatsuba) otherwise; CRTG_SPLIT=0 forces 3."""
    import os
    split_on = os.environ.get("CRTG_SPLIT", "1") != "0"
    return [2 if split_on and has_sqrt_minus_one(int(p)) else 3 for p in ms.moduli]


def _f32_down(y: float) -> np.float32:
    r = np.float32(y)
    return np.nextafter(r, np.float32(-np.inf)) if float(r) > y else r


@dataclass(frozen=True)
class ScalingConstants:
    """float32 thresholds log2(P-1)/2 - 1.5 (fast) and - 0.5 (accurate), biased
    down, and delta = 0.5/(1-4u) rounded down (reference scaling.py:100-115)."""

    p_fast: np.float32
    p_accu: np.float32
    delta: np.float32
    u: float = 2.0 ** -24

    @classmethod
    def from_product(cls, product: int) -> "ScalingConstants":
        t = int(product) - 1
        if t < 1:
            raise ConfigError("modulus product must exceed 1")
        if t & (t - 1) == 0:
            half = 0.5 * (t.bit_length() - 1)
            pf, pa = np.float32(half - 1.5), np.float32(half - 0.5)
        else:
            half = 0.5 * math.log2(t)
            pf = _f32_down(half - 1.5 - 2.0 ** -43)
            pa = _f32_down(half - 0.5 - 2.0 ** -43)
        return cls(np.float32(pf), np.float32(pa), _f32_down(0.5 / (1.0 - 4.0 * 2.0 ** -24)))


class CrtgConsts(ctypes.Structure):
    """Mirror of `crtg_consts` (include/crtg.h)."""

    _fields_ = [
        ("num_moduli", ctypes.c_int32),
        ("moduli", ctypes.c_int32 * MAX_MODULI),
        ("coeff_hi", ctypes.c_double * MAX_MODULI),
        ("coeff_lo", ctypes.c_double * MAX_MODULI),
        ("p_hi", ctypes.c_double),
        ("p_lo", ctypes.c_double),
        ("p_fast", ctypes.c_float),
        ("p_accu", ctypes.c_float),
        ("delta", ctypes.c_float),
        ("reserved", ctypes.c_int32),
    ]


@functools.lru_cache(maxsize=None)
def device_constants(num_moduli: int) -> CrtgConsts:
    ms = select_moduli(num_moduli)
    sc = ScalingConstants.from_product(ms.product)
    k = CrtgConsts()
    k.num_moduli = len(ms)
    for i, p in enumerate(ms.moduli):
        k.moduli[i] = p
        k.coeff_hi[i] = float(ms.coeff_hi[i])
        k.coeff_lo[i] = float(ms.coeff_lo[i])
    k.p_hi = float(ms.product)
    k.p_lo = float(ms.product - int(k.p_hi))
    k.p_fast, k.p_accu, k.delta = float(sc.p_fast), float(sc.p_accu), float(sc.delta)
    return k
