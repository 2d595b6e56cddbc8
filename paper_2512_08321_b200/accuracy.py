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


def _as_dd(reference, cplx_hint: bool, dev) -> DDMatrix:
    if isinstance(reference, DDMatrix):
        return reference
    # a plain array is a reference with lo = 0 (oracle.py:144-146)
    t = reference if isinstance(reference, torch.Tensor) else \
        torch.from_numpy(np.ascontiguousarray(reference))
    cplx = t.is_complex() or cplx_hint
    hi = t.to(torch.complex128 if cplx else torch.float64).to(dev).contiguous()
    return DDMatrix(hi, torch.zeros_like(hi))


def max_relative_error(approx, reference, return_zero_count: bool = False):
    """Largest componentwise relative error (oracle.py:131-169): |(x - hi) - lo| /
    |hi + lo| over the real and imaginary parts separately, zero references
    excluded (and counted when `return_zero_count`)."""
    x = approx if isinstance(approx, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(approx))
    dev = reference.hi.device if isinstance(reference, DDMatrix) else _device()
    reference = _as_dd(reference, x.is_complex(), dev)
    if tuple(x.shape) != tuple(reference.hi.shape):
        raise DimensionError("shape mismatch between approximation and reference")
    cplx = reference.hi.is_complex() or x.is_complex()
    if cplx and not reference.hi.is_complex():
        reference = DDMatrix(reference.hi.to(torch.complex128), reference.lo.to(torch.complex128))
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


def run_accuracy_sweep(dims, moduli_counts, phis, mode="accurate", precision="double",
                       domain="complex", seeds=(0,)) -> list:
    """(N, phi, seed, max_rel_error) rows ordered by (N, phi, seed) (bench.py:73-104).

    Inputs are the reference's generator (`gen_matrix`, seed and seed+1), the
    double-double reference of each (phi, seed) is computed once on the device
    and shared across moduli counts, and the emulation runs through the public
    `emulate_gemm_complex` / `emulate_gemm_real`.
    """
    from .config import EmuConfig
    from .emulate import emulate_gemm_complex, emulate_gemm_real
    from .gen import GenSpec, gen_matrix

    m, n, k = dims
    refs, inputs = {}, {}
    for phi in phis:
        for seed in seeds:
            a = gen_matrix(GenSpec(m, k, phi, seed, precision, domain))
            b = gen_matrix(GenSpec(k, n, phi, seed + 1, precision, domain))
            inputs[(phi, seed)] = (a, b)
            refs[(phi, seed)] = reference_gemm_dd(a, b)
    rows = []
    for count in moduli_counts:
        cfg = EmuConfig(precision=precision, domain=domain, mode=mode, num_moduli=count)
        for phi in phis:
            for seed in seeds:
                a, b = inputs[(phi, seed)]
                run = emulate_gemm_complex if domain == "complex" else emulate_gemm_real
                err = max_relative_error(run(a, b, cfg), refs[(phi, seed)])
                rows.append((count, float(phi), int(seed), err))
    return rows


def sweep_csv(rows) -> str:
    """`N,phi,seed,max_rel_error` CSV (bench.py:107-113)."""
    lines = ["N,phi,seed,max_rel_error"]
    lines += [f"{count},{phi!r},{seed},{err!r}" for count, phi, seed, err in rows]
    return "\n".join(lines) + "\n"


def exact_gemm_bigint(a, b) -> np.ndarray:
    """Exact product of integer-valued matrices as an object array of Python
    ints (reference oracle.py:32-57; a test-side checker, host arithmetic).
    int64 accumulation when k * max|a| * max|b| < 2^62 cannot overflow, Python
    big ints otherwise."""
    a_arr = np.asarray(a)
    b_arr = np.asarray(b)
    if a_arr.ndim != 2 or b_arr.ndim != 2 or a_arr.shape[1] != b_arr.shape[0]:
        raise DimensionError(f"bad shapes {a_arr.shape} x {b_arr.shape}")
    to_obj = np.frompyfunc(int, 1, 1)
    ao = to_obj(a_arr).astype(object) if a_arr.size else np.empty(a_arr.shape, object)
    bo = to_obj(b_arr).astype(object) if b_arr.size else np.empty(b_arr.shape, object)
    amax = max((abs(v) for v in ao.flat), default=0)
    bmax = max((abs(v) for v in bo.flat), default=0)
    if a_arr.shape[1] * amax * bmax < 2 ** 62:
        c = a_arr.astype(np.int64) @ b_arr.astype(np.int64)
        return to_obj(c).astype(object) if c.size else np.empty(c.shape, object)
    return ao @ bo
