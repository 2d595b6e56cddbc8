"""Stage-level drop-in API: the reference's stage functions and types
(crtgemm `__init__.py:10-42`) with its numpy semantics, computed on the GPU by
the stage kernels of libcrtg.so (include/crtg.h "stage-level entry points").

| here | reference |
|---|---|
| `ComplexMatrix` | emulate.py:81-93 |
| `ResidueStack` | crt.py:187-196 |
| `ScaledIntMatrices` | scaling.py:130-136 |
| `log2_upper` | scaling.py:62-82 |
| `quantize` | scaling.py:277-293 |
| `symmetric_mod_int` | crt.py:136-151 |
| `symmetric_mod_wide` | crt.py:154-184 |
| `residue_decompose` | crt.py:199-218 |
| `crt_accumulate` | crt.py:221-243 |
| `crt_reduce` | crt.py:246-258 |
| `inverse_scale` | emulate.py:135-144 |
| `crt_integer_gemm` | emulate.py:120-132 |

numpy arrays in -> numpy arrays out (the reference's behaviour); torch tensors
in -> torch CUDA tensors out.  Python scalars (symmetric_mod_int of an int,
log2_upper / symmetric_mod_wide of a 0-d value) keep the reference's scalar
results.  Every array computation runs on the device; there is no CPU path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .config import DEFAULT_N_BLOCK, MAX_K_REAL
from .errors import ConfigError, DimensionError, DomainError
from .moduli import CrtgConsts, ModulusSet, ScalingConstants

__all__ = [
    "ComplexMatrix", "ResidueStack", "ScaledIntMatrices", "log2_upper", "quantize",
    "symmetric_mod_int", "symmetric_mod_wide", "residue_decompose", "crt_accumulate",
    "crt_reduce", "inverse_scale", "crt_integer_gemm",
]


# ----------------------------------------------------------------------------
# types
# ----------------------------------------------------------------------------
@dataclass
class ComplexMatrix:
    """Explicit real/imaginary pair; convertible to a complex array
    (reference emulate.py:81-93)."""

    re: np.ndarray
    im: np.ndarray

    def __post_init__(self):
        if tuple(self.re.shape) != tuple(self.im.shape):
            raise DimensionError("real/imaginary shapes differ")

    def to_complex(self):
        if isinstance(self.re, torch.Tensor):
            return torch.complex(self.re.to(torch.float64), self.im.to(torch.float64))
        return self.re + 1j * self.im


@dataclass(frozen=True)
class ResidueStack:
    """Per-modulus signed 8-bit residue matrices of one integer matrix
    (reference crt.py:187-196)."""

    entries: np.ndarray  # int8, shape (N, rows, cols)
    modulus_set: ModulusSet

    def __post_init__(self):
        if self.entries.shape[0] != len(self.modulus_set):
            raise ConfigError("stack depth does not match modulus count")


@dataclass
class ScaledIntMatrices:
    """Quantized operands a' = trunc(a * 2^mu_exp) plus their exponents
    (reference scaling.py:130-136)."""

    a_int: np.ndarray
    b_int: np.ndarray
    scaling: object  # ScalingVectors


# ----------------------------------------------------------------------------
# plumbing
# ----------------------------------------------------------------------------
def _dev():
    from .emulate import _device
    return _device()


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _to_dev(x, dtype, dev):
    """-> (contiguous device tensor of `dtype`, was_torch)."""
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=dtype).contiguous(), True
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=_np_of(dtype)))).to(dev), False


def _np_of(dtype):
    return {torch.float64: np.float64, torch.float32: np.float32, torch.int64: np.int64,
            torch.int32: np.int32, torch.int8: np.int8}[dtype]


def _out(t: torch.Tensor, was_torch: bool):
    return t if was_torch else t.cpu().numpy()


def _flags(dev, n=3):
    return torch.empty(n, dtype=torch.int64, device=dev)


def consts_for(ms: ModulusSet) -> CrtgConsts:
    """crtg_consts of an arbitrary modulus set (moduli, CRT weights, P split)."""
    k = CrtgConsts()
    k.num_moduli = len(ms)
    for i, p in enumerate(ms.moduli):
        k.moduli[i] = int(p)
        k.coeff_hi[i] = float(ms.coeff_hi[i])
        k.coeff_lo[i] = float(ms.coeff_lo[i])
    k.p_hi = float(ms.product)
    k.p_lo = float(ms.product - int(k.p_hi))
    if ms.product > 1:
        sc = ScalingConstants.from_product(ms.product)
        k.p_fast, k.p_accu, k.delta = float(sc.p_fast), float(sc.p_accu), float(sc.delta)
    return k


# ----------------------------------------------------------------------------
# scaling stages
# ----------------------------------------------------------------------------
def log2_upper(x):
    """Deterministic float32 upper bound on log2(x) (reference scaling.py:62-82)."""
    scalar = np.isscalar(x) or (not isinstance(x, torch.Tensor) and np.ndim(x) == 0)
    dev = _dev()
    t, was_torch = _to_dev(np.reshape(np.asarray(x, np.float64), -1) if scalar else x,
                           torch.float64, dev)
    out = torch.empty(t.shape, dtype=torch.float32, device=dev)
    nat.call("crtg_log2_upper", t.data_ptr(), t.numel(), out.data_ptr(), _flags(dev).data_ptr(),
             1, _stream(dev))
    if scalar:
        return np.float32(out.cpu().numpy()[0])
    return _out(out, was_torch)


def quantize(mat, exps, axis: int = 0):
    """trunc(mat * 2^exps), exact power-of-two scaling; axis=0 applies exps
    per row, axis=1 per column (reference scaling.py:277-293)."""
    if axis not in (0, 1):
        raise ConfigError("axis must be 0 (rows) or 1 (columns)")
    dev = _dev()
    m, was_torch = _to_dev(mat, torch.float64, dev)
    if m.dim() != 2:
        raise DimensionError("matrix must be 2-D")
    e, _ = _to_dev(exps, torch.int64, dev)
    if e.dim() != 1 or e.shape[0] != m.shape[axis]:
        raise DimensionError("exponent vector does not match matrix")
    rows, cols = m.shape
    out = torch.empty((rows, cols), dtype=torch.float64, device=dev)
    nat.call("crtg_quantize", m.data_ptr(), rows, cols, max(cols, 1), e.data_ptr(), axis,
             out.data_ptr(), max(cols, 1), _flags(dev).data_ptr(), 1, _stream(dev))
    return _out(out, was_torch)


# ----------------------------------------------------------------------------
# residues
# ----------------------------------------------------------------------------
def _kind_of(x):
    """-> (device tensor, kind code, was_torch) for an integer-valued array."""
    dev = _dev()
    if isinstance(x, torch.Tensor):
        if x.is_floating_point():
            return x.to(device=dev, dtype=torch.float64).contiguous(), 0, True
        if x.dtype == torch.int32:
            return x.to(dev).contiguous(), 2, True
        return x.to(device=dev, dtype=torch.int64).contiguous(), 1, True
    arr = np.asarray(x)
    if np.issubdtype(arr.dtype, np.floating):
        return torch.from_numpy(np.ascontiguousarray(arr, np.float64)).to(dev), 0, False
    if arr.dtype == np.int32:
        return torch.from_numpy(np.ascontiguousarray(arr)).to(dev), 2, False
    return torch.from_numpy(np.ascontiguousarray(arr.astype(np.int64))).to(dev), 1, False


STRICT = 8  # residue_decompose's input checks (crt.py:203-213)


def _residues(t: torch.Tensor, kind: int, moduli) -> torch.Tensor:
    dev = t.device
    n = len(moduli)
    out = torch.empty((n,) + tuple(t.shape), dtype=torch.int8, device=dev)
    mods = (ctypes.c_int32 * n)(*[int(p) for p in moduli])
    nat.call("crtg_symmetric_mod", kind, t.data_ptr(), t.numel(), mods, n, out.data_ptr(),
             _flags(dev).data_ptr(), 1, _stream(dev))
    return out


def symmetric_mod_int(x, p: int):
    """Symmetric remainder x - p*round(x/p), half-quotients rounded up
    (reference crt.py:136-151): int8-range residues congruent to x."""
    if p < 2:
        raise DomainError(f"modulus must be >= 2, got {p}")
    if not isinstance(x, (np.ndarray, torch.Tensor)):
        x = int(x)
        return x - p * ((2 * x + p) // (2 * p))
    if p > 256:
        # the reference's formula for moduli beyond int8 (not used by the
        # emulation; the device kernel covers p <= 256)
        raise DomainError("device residues cover moduli up to 256")
    t, kind, was_torch = _kind_of(x)
    r = _residues(t.reshape(-1), kind, (p,))[0].reshape(t.shape)
    # the reference returns int64 (integer input) / int64 (float input) arrays
    return r.to(torch.int64) if was_torch else r.cpu().numpy().astype(np.int64)


def residue_decompose(matrix, ms: ModulusSet) -> ResidueStack:
    """Map an integer-valued matrix to its symmetric residues per modulus
    (reference crt.py:199-218)."""
    t, kind, was_torch = _kind_of(matrix)
    stack = _residues(t.reshape(-1), kind | STRICT, ms.moduli).reshape(
        (len(ms),) + tuple(t.shape))
    return ResidueStack(stack if was_torch else stack.cpu().numpy(), ms)


# ----------------------------------------------------------------------------
# CRT
# ----------------------------------------------------------------------------
def crt_accumulate(stack: ResidueStack, ms: ModulusSet, precision: str = "double"):
    """Weighted sum S = sum_l (P/p_l) q_l E_l in ascending l (reference
    crt.py:221-243): (S1, S2) on the double path, S1 + S2 on the single path."""
    if tuple(stack.modulus_set.moduli) != tuple(ms.moduli):
        raise ConfigError("residue stack was built for a different modulus set")
    if precision not in ("double", "single"):
        raise ConfigError(f"unknown precision path {precision!r}")
    dev = _dev()
    e, was_torch = _to_dev(stack.entries, torch.int8, dev)
    shape = tuple(e.shape[1:])
    count = int(np.prod(shape)) if shape else 1
    s1 = torch.empty(shape, dtype=torch.float64, device=dev)
    s2 = torch.empty(shape, dtype=torch.float64, device=dev)
    nat.call("crtg_crt_accumulate", e.data_ptr(), count, ctypes.byref(consts_for(ms)),
             1 if precision == "single" else 0, s1.data_ptr(), s2.data_ptr(), _stream(dev))
    if precision == "single":
        return _out(s1, was_torch)
    return _out(s1, was_torch), _out(s2, was_torch)


def symmetric_mod_wide(s, product: int, use_dd: bool = True):
    """Symmetric remainder mod a big P, half-quotients rounded down, result in
    (-P/2, P/2] (reference crt.py:154-184)."""
    p_hi = float(product)
    p_lo = float(product - int(p_hi))
    dev = _dev()
    pair = isinstance(s, tuple)
    hi_in = s[0] if pair else s
    was_torch = isinstance(hi_in, torch.Tensor)
    hi, _ = _to_dev(np.asarray(hi_in, np.float64) if not was_torch else hi_in, torch.float64, dev)
    lo = None
    if pair:
        lo, _ = _to_dev(np.asarray(s[1], np.float64) if not isinstance(s[1], torch.Tensor)
                        else s[1], torch.float64, dev)
        hi, lo = torch.broadcast_tensors(hi, lo)
        hi, lo = hi.contiguous(), lo.contiguous()
    out = torch.empty(hi.shape, dtype=torch.float64, device=dev)
    nat.call("crtg_symmetric_mod_wide", hi.data_ptr(), lo.data_ptr() if lo is not None else None,
             hi.numel(), p_hi, p_lo, 1 if use_dd else 0, out.data_ptr(), _stream(dev))
    if out.dim() == 0:
        return float(out.item())
    return _out(out, was_torch)


def crt_reduce(accumulator, ms: ModulusSet):
    """Final reduction mod P of the CRT accumulator (reference crt.py:246-258):
    double-double for an (S1, S2) pair, plain float64 otherwise."""
    if isinstance(accumulator, tuple):
        r = symmetric_mod_wide(accumulator, ms.product, use_dd=True)
    else:
        r = symmetric_mod_wide(accumulator, ms.product, use_dd=False)
    return r if isinstance(r, torch.Tensor) else np.asarray(r)


def inverse_scale(c_prime, sv, out_dtype=np.float64):
    """C = 2^(-mu_i - nu_j) * C' with one final cast (reference emulate.py:135-144)."""
    dev = _dev()
    c, was_torch = _to_dev(c_prime, torch.float64, dev)
    mu, _ = _to_dev(sv.mu_exp, torch.int64, dev)
    nu, _ = _to_dev(sv.nu_exp, torch.int64, dev)
    rows, cols = c.shape
    if mu.numel() != rows or nu.numel() != cols:
        raise DimensionError("scaling vectors do not match the matrix")
    f32 = np.dtype(out_dtype) == np.float32 if not isinstance(out_dtype, torch.dtype) \
        else out_dtype == torch.float32
    if not f32 and not (out_dtype in (np.float64, float, torch.float64)
                        or np.dtype(out_dtype) == np.float64):
        raise ConfigError(f"unsupported output dtype {out_dtype!r}")
    out = torch.empty((rows, cols), dtype=torch.float32 if f32 else torch.float64, device=dev)
    nat.call("crtg_inverse_scale", c.data_ptr(), rows, cols, max(cols, 1), mu.data_ptr(),
             nu.data_ptr(), 1 if f32 else 0, out.data_ptr(), max(cols, 1), _stream(dev))
    return _out(out, was_torch)


def crt_integer_gemm(a_int, b_int, ms: ModulusSet, precision: str = "double",
                     n_block: int = DEFAULT_N_BLOCK):
    """Integer matrix product via residues and CRT (reference
    emulate.py:120-132): residue stacks of both operands, one exact INT8
    product per modulus on the tensor cores reduced back to residues, CRT
    accumulate + reduce.  Exact whenever 2 sum_h |a_ih||b_hj| < P."""
    from .emulate import gemm_i8_i32
    if n_block < 1:
        raise ConfigError("n_block must be >= 1")
    a_st = residue_decompose(a_int, ms)
    b_st = residue_decompose(b_int, ms)
    was_torch = isinstance(a_st.entries, torch.Tensor)
    dev = _dev()
    ae = torch.as_tensor(a_st.entries).to(dev)
    be = torch.as_tensor(b_st.entries).to(dev)
    if ae.dim() != 3 or be.dim() != 3 or ae.shape[2] != be.shape[1]:
        raise DimensionError("inner dimensions differ")
    if ae.shape[2] > MAX_K_REAL:
        raise DimensionError(f"inner dimension {ae.shape[2]} exceeds {MAX_K_REAL}")
    m, n = ae.shape[1], be.shape[2]
    out = torch.empty((len(ms), m, n), dtype=torch.int8, device=dev)
    for idx, p in enumerate(ms.moduli):
        # n_block only bounds the working set: results are bitwise invariant
        for j0 in range(0, n, n_block):
            j1 = min(j0 + n_block, n)
            d = gemm_i8_i32(ae[idx], be[idx][:, j0:j1].contiguous())
            out[idx, :, j0:j1] = _residues(d.reshape(-1), 2, (p,))[0].reshape(d.shape)
    acc = crt_accumulate(ResidueStack(out, ms), ms, precision)
    res = crt_reduce(acc, ms)
    return res if was_torch else res.cpu().numpy() if isinstance(res, torch.Tensor) else res
