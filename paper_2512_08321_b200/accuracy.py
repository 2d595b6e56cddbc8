"""GPU accuracy harness.

`reference_gemm_dd(a, b)` is the reference's double-double product
(oracle.py:108-128 there), computed on the device bit-for-bit (same error-free
transformations, same ascending term order of the stacked real forms);
`max_relative_error(approx, reference)` is the reference's metric
(oracle.py:131-169) evaluated on the device.  Used to report the emulation's
error per moduli count at sizes the CPU oracle cannot reach (16384^3: the numba
oracle needs ~16 h on 8 cores).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .emulate import _device, _stream_ptr
from .errors import DimensionError


@dataclass(frozen=True)
class DDMatrix:
    """Unevaluated sum hi + lo per element (~106-bit), device tensors."""

    hi: torch.Tensor
    lo: torch.Tensor

    def to_array(self):
        return (self.hi + self.lo).cpu().numpy()


def _dev_f64(x, cplx, dev):
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    t = t.to(torch.complex128 if cplx else torch.float64)
    return t.to(dev).contiguous()


def reference_gemm_dd(a, b) -> DDMatrix:
    dev = _device()
    cplx = (a.is_complex() if isinstance(a, torch.Tensor) else np.iscomplexobj(a)) or \
        (b.is_complex() if isinstance(b, torch.Tensor) else np.iscomplexobj(b))
    at, bt = _dev_f64(a, cplx, dev), _dev_f64(b, cplx, dev)
    if at.dim() != 2 or bt.dim() != 2 or at.shape[1] != bt.shape[0]:
        raise DimensionError(f"bad shapes {tuple(at.shape)} x {tuple(bt.shape)}")
    m, k = at.shape
    n = bt.shape[1]
    hi = torch.empty((m, n), dtype=at.dtype, device=dev)
    lo = torch.empty_like(hi)
    nat.call("crtg_dd_gemm", int(cplx), m, n, k, at.data_ptr(), at.stride(0), bt.data_ptr(),
             bt.stride(0), hi.data_ptr(), lo.data_ptr(), hi.stride(0), _stream_ptr(dev))
    return DDMatrix(hi, lo)


def max_relative_error(approx, reference: DDMatrix, return_zero_count: bool = False):
    dev = reference.hi.device
    cplx = reference.hi.is_complex()
    x = approx if isinstance(approx, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(approx))
    if tuple(x.shape) != tuple(reference.hi.shape):
        raise DimensionError("shape mismatch between approximation and reference")
    single = x.dtype in (torch.complex64, torch.float32)
    want = (torch.complex64 if single else torch.complex128) if cplx else \
        (torch.float32 if single else torch.float64)
    x = x.to(want).to(dev).contiguous()
    out = torch.zeros(2, dtype=torch.int64, device=dev)
    nat.call("crtg_max_relative_error", int(cplx), x.shape[0], x.shape[1], x.data_ptr(),
             int(single), x.stride(0), reference.hi.data_ptr(), reference.lo.data_ptr(),
             reference.hi.stride(0), out.data_ptr(), out.data_ptr() + 8, _stream_ptr(dev))
    bits, zeros = out.cpu().tolist()
    worst = float(np.array([bits], np.int64).view(np.float64)[0])
    return (worst, int(zeros)) if return_zero_count else worst
