"""Drop-in complex GEMM emulation on B200 (reference emulate.py:193-278).

`emulate_gemm_complex(a, b, cfg=None, diagnostics=None)` and the BLAS-style
`gemm(...)` keep the reference's names, arguments, defaults, error classes and
results (bit-for-bit, see tests/).  Everything below the argument checks runs in
libcrtg.so on the GPU (include/crtg.h); there is no CPU path.

Inputs may be numpy arrays (copied to the device, result returned as numpy —
the reference's behaviour) or torch tensors (CUDA or CPU; if both inputs are
torch tensors the result is a torch CUDA tensor on the same device).

Lower-level GPU parity hooks mirror the reference's stage functions:
`gemm_i8_i32` (kernel.py:20-35), `complex_gemm_mod` (kernel.py:70-120),
`fast_scaling` / `accurate_scaling` (scaling.py:198-274), `quantized_residues`
(quantize + residue_decompose, scaling.py:277-293 + crt.py:199-218) and
`crt_reconstruct` (crt.py:221-258 + emulate.py:135-144).
"""

from __future__ import annotations

import ctypes
import threading
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .config import MAX_K_COMPLEX, MAX_K_REAL, STRATEGIES, EmuConfig
from .errors import ConfigError, DimensionError, DomainError
from .moduli import ModulusSet, ScalingConstants, device_constants, select_moduli

__all__ = [
    "ScalingVectors", "emulate_gemm_complex", "emulate_gemm_real", "gemm", "gemm_i8_i32", "complex_gemm_mod",
    "fast_scaling", "accurate_scaling", "quantized_residues", "crt_reconstruct",
]


@dataclass
class ScalingVectors:
    """mu = 2^mu_exp per row of A, nu = 2^nu_exp per column of B
    (reference scaling.py:118-127)."""

    mu_exp: np.ndarray
    nu_exp: np.ndarray
    bar_mu_exp: np.ndarray | None = None
    bar_nu_exp: np.ndarray | None = None


# ----------------------------------------------------------------------------
# device plumbing
# ----------------------------------------------------------------------------
_cuda_seen = False


def _device() -> torch.device:
    global _cuda_seen
    if not _cuda_seen:
        if not torch.cuda.is_available():
            raise nat.NativeError("no CUDA device: the B200 emulation has no CPU path")
        _cuda_seen = True
    dev = torch.device("cuda", torch.cuda.current_device())
    nat.check_device(dev.index)
    return dev


# the raw handle of the current stream without building a torch Stream object
# (a few microseconds per call on small products)
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_ptr(dev) -> int:
    if _raw_stream is not None:
        return _raw_stream(dev.index)
    return torch.cuda.current_stream(dev).cuda_stream


def _to_device_matrix(x, name: str, dev, complex_out: bool = True):
    """-> (contiguous CUDA tensor, was_torch).  Mirrors _check_complex_input
    (emulate.py:159-166): 2-D, cast to complex (complex64 kept, upcast exactly
    on the device)."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.dim() != 2:
            raise DimensionError(f"{name} must be 2-D")
        if complex_out and not t.is_complex():
            t = t.to(torch.complex128)
        if complex_out and t.dtype not in (torch.complex64, torch.complex128):
            t = t.to(torch.complex128)
        if not (t.is_cuda and t.get_device() == dev.index):
            t = t.to(dev)
        return (t if t.is_contiguous() else t.contiguous()), True
    arr = np.asarray(x)
    if arr.ndim != 2:
        raise DimensionError(f"{name} must be 2-D")
    if complex_out and arr.dtype not in (np.complex64, np.complex128):
        arr = arr.astype(np.complex128)
    # pageable upload (11 GB/s) beats copying into a fresh pinned buffer first
    return torch.from_numpy(np.ascontiguousarray(arr)).to(dev), False


def _workspace(nbytes: int, dev) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)


# Small products reuse one workspace + diagnostics buffer per (thread, device,
# stream): stream order makes reuse safe, it saves two allocations per call and
# keeps the buffer addresses stable, which is what lets the library replay its
# captured CUDA graph (api.cu).  Larger workspaces are allocated per call.
_SMALL_WS_BYTES = 256 << 20
_tls = threading.local()
_ws_size_cache: dict = {}


def _small_buffers(need: int, dev, stream: int):
    cache = getattr(_tls, "bufs", None)
    if cache is None:
        cache = _tls.bufs = {}
    key = (dev.index, stream)
    ent = cache.get(key)
    if ent is None or ent[0].numel() < need:
        ent = (torch.empty(max(need, 1 << 20), dtype=torch.uint8, device=dev),
               torch.empty(nat.DIAG_LEN, dtype=torch.int64, device=dev))
        cache[key] = ent
    return ent


def _workspace_size(lib, prec, mode, m, n, k, nmod, n_block) -> int:
    key = (prec, mode, m, n, k, nmod, n_block)
    v = _ws_size_cache.get(key)
    if v is None:
        if len(_ws_size_cache) > 4096:
            _ws_size_cache.clear()
        v = _ws_size_cache[key] = int(lib.crtg_workspace_size(prec, mode, m, n, k, nmod, n_block))
    return v


# ----------------------------------------------------------------------------
# the hot path
# ----------------------------------------------------------------------------
def _empty_product(a, b, cfg: EmuConfig, complex_out: bool):
    """Zero-extent operands, as the reference behaves (no kernel launched): fast
    mode with m = 0 or n = 0 (k > 0) returns an empty (m, n) result of the
    output dtype; every other zero extent fails in numpy's max-reduction inside
    the reference's scaling (a ValueError) -> DimensionError (a ValueError).
    Returns None when no extent is zero."""
    ash = tuple(a.shape) if isinstance(a, torch.Tensor) else np.shape(a)
    bsh = tuple(b.shape) if isinstance(b, torch.Tensor) else np.shape(b)
    if len(ash) != 2 or len(bsh) != 2 or min(ash + bsh) > 0:
        return None
    if ash[1] != bsh[0]:
        raise DimensionError(f"inner dimensions differ: {ash} x {bsh}")
    m, k = ash
    n = bsh[1]
    if k == 0 or cfg.mode != "fast":
        raise DimensionError("zero-size array to reduction operation maximum which has no identity")
    single = cfg.precision == "single"
    if isinstance(a, torch.Tensor) and isinstance(b, torch.Tensor):
        dt = ((torch.complex64 if single else torch.complex128) if complex_out
              else (torch.float32 if single else torch.float64))
        dev = a.device if a.is_cuda else (b.device if b.is_cuda else _device())
        return torch.empty((m, n), dtype=dt, device=dev)
    dt = (np.complex64 if single else np.complex128) if complex_out else (
        np.float32 if single else np.float64)
    return np.empty((m, n), dtype=dt)


def emulate_gemm_complex(a, b, cfg: EmuConfig | None = None,
                         diagnostics: dict | None = None):
    """Emulated complex matrix product A @ B (reference emulate.py:193-240)."""
    cfg = cfg or EmuConfig(domain="complex")
    if cfg.domain != "complex":
        raise ConfigError("config domain must be 'complex'")
    empty = _empty_product(a, b, cfg, True)
    if empty is not None:
        return empty
    dev = _device()
    on_dev = [isinstance(x, torch.Tensor) and x.is_cuda for x in (a, b)]
    if not any(on_dev) and cfg.strategy == "karatsuba":
        # host operands: stream them through the copy engines (crtg_gemm_complex_host)
        pins = _HostPins()
        try:
            ha, a_torch = _host_matrix(a, "A", pins)
            hb, b_torch = _host_matrix(b, "B", pins)
            _check_shapes(ha, hb)
            # numpy in -> numpy out owning plain memory; torch in -> pinned tensor
            out = run_complex_host(ha, hb, cfg, diagnostics, dev,
                                   pageable_out=not (a_torch and b_torch))  # synchronous
        finally:
            pins.release()
        return out if (a_torch and b_torch) else out.numpy()
    at, a_torch = _to_device_matrix(a, "A", dev)
    bt, b_torch = _to_device_matrix(b, "B", dev)
    _check_shapes(at, bt)
    if cfg.strategy != "karatsuba":
        out = _emulate_complex_stages(at, bt, cfg, diagnostics)
    else:
        out = run_complex(at, bt, cfg, diagnostics, dev)
    if a_torch and b_torch:
        return out
    return out.cpu().numpy()


def _check_shapes(at, bt):
    if at.shape[1] != bt.shape[0]:
        raise DimensionError(f"inner dimensions differ: {tuple(at.shape)} x {tuple(bt.shape)}")
    if at.shape[1] > MAX_K_COMPLEX:
        raise DimensionError(f"inner dimension {at.shape[1]} exceeds {MAX_K_COMPLEX}")


_REGISTER_MIN_BYTES = 32 << 20


class _HostPins:
    """Pageable numpy operands are staged by the library itself (host threads
    gather each piece into a ring of pinned slots that the copy engine streams
    from, crtg_gemm_complex_host), so by default nothing is page-locked here.
    CRTG_HOST_REGISTER=1 instead page-locks the caller's arrays IN PLACE
    (cudaHostRegister, ~0.33 s per 4 GiB plus the unlock) for the call."""

    REGISTER = os.environ.get("CRTG_HOST_REGISTER", "0") == "1"

    def __init__(self):
        self.ptrs = []

    def pin(self, arr: np.ndarray):
        if not self.REGISTER or arr.nbytes < _REGISTER_MIN_BYTES:
            return torch.from_numpy(arr)
        cr = torch.cuda.cudart()
        err = cr.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
        if int(err) == 0:
            self.ptrs.append(arr.ctypes.data)
        # already registered / not registrable: the copies still work (pageable)
        return torch.from_numpy(arr)

    def release(self):
        cr = torch.cuda.cudart()
        for ptr in self.ptrs:
            cr.cudaHostUnregister(ptr)
        self.ptrs.clear()


def _host_matrix(x, name: str, pins: _HostPins):
    """-> (contiguous CPU complex tensor, page-locked while the call runs, was_torch)."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.dim() != 2:
            raise DimensionError(f"{name} must be 2-D")
        if t.dtype not in (torch.complex64, torch.complex128):
            t = t.to(torch.complex128)
        t = t.contiguous()
        if t.is_pinned():
            return t, True
        return pins.pin(t.numpy()), True
    arr = np.asarray(x)
    if arr.ndim != 2:
        raise DimensionError(f"{name} must be 2-D")
    if arr.dtype not in (np.complex64, np.complex128):
        arr = arr.astype(np.complex128)
    return pins.pin(np.ascontiguousarray(arr)), False


def run_complex_host(ha: torch.Tensor, hb: torch.Tensor, cfg: EmuConfig,
                     diagnostics: dict | None = None, dev=None, pageable_out: bool = False):
    """Host operands in, host result out; H2D of B's column blocks and D2H of C's
    blocks overlap the GPU work (crtg_gemm_complex_host).  The result is a
    pinned tensor from torch's caching host allocator, or with pageable_out a
    plain (pageable) tensor that owns its memory (numpy callers: results they
    keep do not hold page-locked memory; the library stages the copy-back
    through its pinned ring)."""
    dev = dev or _device()
    if ha.dtype != hb.dtype:  # mixed complex64 / complex128: widen the narrow one
        ha, hb = ha.to(torch.complex128), hb.to(torch.complex128)
    m, k = ha.shape
    n = hb.shape[1]
    nmod = cfg.resolved_moduli
    prec = nat.SINGLE if cfg.precision == "single" else nat.DOUBLE
    if ha.dtype == torch.complex64:
        prec |= 16
    mode = nat.FAST if cfg.mode == "fast" else nat.ACCURATE
    lib = nat.load()
    ws = _workspace(lib.crtg_host_workspace_size(prec, mode, m, n, k, nmod, cfg.n_block), dev)
    odt = torch.complex64 if cfg.precision == "single" else torch.complex128
    # the result lands in pinned host memory (torch's caching host allocator
    # reuses it across calls: 16384^3 numpy in / numpy out 0.25 s per call in
    # steady state).  A pageable C also works -- the library then stages the
    # copy-back through pinned slots -- but measured 0.45 s per call (fresh pages
    # touched every call) against 1.1 s instead of 2.4 s for the first call.
    out = torch.empty((m, n), dtype=odt, pin_memory=not pageable_out)
    diag = torch.zeros(nat.DIAG_LEN, dtype=torch.int64, device=dev)
    nat.call("crtg_gemm_complex_host", prec, mode, m, n, k, ha.data_ptr(), ha.stride(0),
             hb.data_ptr(), hb.stride(0), out.data_ptr(), out.stride(0),
             ctypes.byref(device_constants(nmod)), cfg.n_block, ws.data_ptr(), ws.numel(),
             diag.data_ptr(), 1, _stream_ptr(dev))
    if diagnostics is not None:
        d = diag.cpu().tolist()
        for key, idx in (("clamped_mu", nat.DIAG_CLAMPED_MU), ("clamped_nu", nat.DIAG_CLAMPED_NU)):
            if d[idx]:
                diagnostics[key] = diagnostics.get(key, 0) + int(d[idx])
    return out


def run_complex(at: torch.Tensor, bt: torch.Tensor, cfg: EmuConfig,
                diagnostics: dict | None = None, dev=None, sync_check: bool = True,
                ws: torch.Tensor | None = None, out: torch.Tensor | None = None,
                return_exponents: bool = False):
    """Device-resident entry: contiguous CUDA complex tensors in, CUDA tensor out.
    Used by the public API, the benchmark and the multi-GPU driver."""
    dev = dev or at.device
    if at.dtype != bt.dtype:  # mixed precision inputs: upcast the narrower one
        at, bt = at.to(torch.complex128), bt.to(torch.complex128)
    m, k = at.shape
    n = bt.shape[1]
    nmod = cfg.resolved_moduli
    consts = device_constants(nmod)
    prec = nat.SINGLE if cfg.precision == "single" else nat.DOUBLE
    if at.dtype == torch.complex64:
        prec |= 16  # CRTG_IN_C64
    mode = nat.FAST if cfg.mode == "fast" else nat.ACCURATE
    lib = nat.load()
    need = _workspace_size(lib, prec, mode, m, n, k, nmod, cfg.n_block)
    stream = _stream_ptr(dev)
    diag = None
    if ws is None or ws.numel() < need:
        if need <= _SMALL_WS_BYTES:
            ws, diag = _small_buffers(need, dev, stream)
        else:
            ws = _workspace(need, dev)
    odt = torch.complex64 if cfg.precision == "single" else torch.complex128
    if out is None:
        out = torch.empty((m, n), dtype=odt, device=dev)
    # crtg_gemm_complex zeroes the counters on the stream itself
    if diag is None:
        diag = torch.empty(nat.DIAG_LEN, dtype=torch.int64, device=dev)
    mu = torch.empty(m, dtype=torch.int32, device=dev) if return_exponents else None
    nu = torch.empty(n, dtype=torch.int32, device=dev) if return_exponents else None
    nat.call("crtg_gemm_complex", prec, mode, m, n, k, at.data_ptr(), at.stride(0),
             bt.data_ptr(), bt.stride(0), out.data_ptr(), out.stride(0),
             ctypes.byref(consts), cfg.n_block, ws.data_ptr(), ws.numel(),
             mu.data_ptr() if mu is not None else None,
             nu.data_ptr() if nu is not None else None,
             diag.data_ptr(), 1 if sync_check else 0, stream)
    if diagnostics is not None:
        d = diag.cpu().tolist()
        for key, idx in (("clamped_mu", nat.DIAG_CLAMPED_MU), ("clamped_nu", nat.DIAG_CLAMPED_NU)):
            if d[idx]:
                diagnostics[key] = diagnostics.get(key, 0) + int(d[idx])
    if return_exponents:
        return out, mu, nu
    return out


# ----------------------------------------------------------------------------
# real domain (reference emulate.py:169-190)
# ----------------------------------------------------------------------------
def _real_operand(x, name: str, dev, reduce_axis: int):
    """-> (device tensor holding the data, colmajor flag, leading dim, was_torch).

    The reference keeps a real operand's memory layout (astype(copy=False)), and
    numpy then sums squares pairwise along the innermost (smallest-stride) axis and
    sequentially along the other.  The operand is shipped in the layout whose
    contiguous axis is numpy's inner axis, so the library reproduces the order.
    """
    was_torch = isinstance(x, torch.Tensor)
    if was_torch:
        if x.dim() != 2:
            raise DimensionError(f"{name} must be 2-D")
        if x.is_complex():
            raise DomainError(f"{name} must be real for real-domain emulation")
        t = x
    else:
        arr = np.asarray(x)
        if arr.ndim != 2:
            raise DimensionError(f"{name} must be 2-D")
        if np.iscomplexobj(arr):
            raise DomainError(f"{name} must be real for real-domain emulation")
    shape = tuple(t.shape) if was_torch else arr.shape
    strides = (tuple(abs(v) for v in t.stride()) if was_torch
               else tuple(abs(v) // max(arr.itemsize, 1) for v in arr.strides))
    other = 1 - reduce_axis
    # numpy's inner loop axis: the non-trivial axis with the smallest stride
    if shape[reduce_axis] <= 1:
        inner = other
    elif shape[other] <= 1:
        inner = reduce_axis
    else:
        inner = 0 if strides[0] < strides[1] else 1
    colmajor = inner == 0  # axis 0 contiguous -> column-major storage
    if was_torch:
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        t = (t.t().contiguous().t() if colmajor else t.contiguous()).to(dev)
        ld = t.stride(1) if colmajor else t.stride(0)
        return t, colmajor, max(int(ld), 1), True
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    arr = np.asfortranarray(arr) if colmajor else np.ascontiguousarray(arr)
    flat = torch.from_numpy(arr.ravel(order="F" if colmajor else "C"))
    t = flat.to(dev)
    ld = arr.shape[0] if colmajor else arr.shape[1]
    return t, colmajor, max(int(ld), 1), False


def emulate_gemm_real(a, b, cfg: EmuConfig | None = None, diagnostics: dict | None = None):
    """Emulated real matrix product A @ B (reference emulate.py:169-190)."""
    cfg = cfg or EmuConfig()
    if cfg.domain != "real":
        raise ConfigError("config domain must be 'real'")
    for x, name in ((a, "A"), (b, "B")):
        if x.is_complex() if isinstance(x, torch.Tensor) else np.iscomplexobj(x):
            raise DomainError(f"{name} must be real for real-domain emulation")
    empty = _empty_product(a, b, cfg, False)
    if empty is not None:
        return empty
    dev = _device()
    ash = tuple(a.shape) if isinstance(a, torch.Tensor) else np.shape(a)
    bsh = tuple(b.shape) if isinstance(b, torch.Tensor) else np.shape(b)
    at, a_col, lda, a_torch = _real_operand(a, "A", dev, 1)
    bt, b_col, ldb, b_torch = _real_operand(b, "B", dev, 0)
    if ash[1] != bsh[0]:
        raise DimensionError(f"inner dimensions differ: {ash} x {bsh}")
    m, k = ash
    n = bsh[1]
    k_cap = MAX_K_REAL if cfg.mode == "fast" else MAX_K_COMPLEX
    if k > k_cap:
        raise DimensionError(f"inner dimension {k} exceeds {k_cap}")
    if at.dtype != bt.dtype:
        at, bt = at.to(torch.float64), bt.to(torch.float64)
    nmod = cfg.resolved_moduli
    prec = nat.SINGLE if cfg.precision == "single" else nat.DOUBLE
    if at.dtype == torch.float32:
        prec |= 16  # CRTG_IN_F32
    mode = nat.FAST if cfg.mode == "fast" else nat.ACCURATE
    lib = nat.load()
    ws = _workspace(lib.crtg_real_workspace_size(prec, mode, m, n, k, nmod, cfg.n_block), dev)
    out = torch.empty((m, n), dtype=torch.float32 if cfg.precision == "single" else torch.float64,
                      device=dev)
    diag = torch.zeros(nat.DIAG_LEN, dtype=torch.int64, device=dev)
    nat.call("crtg_gemm_real", prec, mode, m, n, k, at.data_ptr(), lda, int(a_col),
             bt.data_ptr(), ldb, int(b_col), out.data_ptr(), out.stride(0),
             ctypes.byref(device_constants(nmod)), cfg.n_block, ws.data_ptr(), ws.numel(),
             None, None, diag.data_ptr(), 1, _stream_ptr(dev))
    if diagnostics is not None:
        d = diag.cpu().tolist()
        for key, idx in (("clamped_mu", nat.DIAG_CLAMPED_MU), ("clamped_nu", nat.DIAG_CLAMPED_NU)):
            if d[idx]:
                diagnostics[key] = diagnostics.get(key, 0) + int(d[idx])
    if a_torch and b_torch:
        return out
    return out.cpu().numpy()


def _colmajor_view(buf, ld, rows, cols, name):
    """Column-major view with leading dimension (reference emulate.py:243-253)."""
    if isinstance(buf, torch.Tensor):
        if buf.dim() == 1:
            if buf.numel() < ld * cols:
                raise DimensionError(f"{name} buffer too small for ld={ld}")
            return buf.as_strided((rows, cols), (1, ld))
        if buf.dim() == 2:
            if buf.shape[0] < rows or buf.shape[1] < cols:
                raise DimensionError(f"{name} array smaller than {rows}x{cols}")
            return buf[:rows, :cols]
        raise DimensionError(f"{name} must be 1-D storage or a 2-D array")
    arr = np.asarray(buf)
    if arr.ndim == 1:
        if arr.size < ld * cols:
            raise DimensionError(f"{name} buffer too small for ld={ld}")
        return arr[:ld * cols].reshape((ld, cols), order="F")[:rows, :]
    if arr.ndim == 2:
        if arr.shape[0] < rows or arr.shape[1] < cols:
            raise DimensionError(f"{name} array smaller than {rows}x{cols}")
        return arr[:rows, :cols]
    raise DimensionError(f"{name} must be 1-D storage or a 2-D array")


def gemm(domain: str, precision: str, m: int, n: int, k: int, a, lda: int, b, ldb: int,
         c, ldc: int, cfg: EmuConfig | None = None):
    """GEMM-style entry on column-major buffers with leading dimensions; writes
    the product into ``c`` and returns it (reference emulate.py:256-278)."""
    if cfg is None:
        cfg = EmuConfig(precision=precision, domain=domain)
    if cfg.precision != precision or cfg.domain != domain:
        raise ConfigError("cfg disagrees with the requested domain/precision")
    av = _colmajor_view(a, lda, m, k, "A")
    bv = _colmajor_view(b, ldb, k, n, "B")
    cv = _colmajor_view(c, ldc, m, n, "C")
    if domain == "real":
        result = emulate_gemm_real(av, bv, cfg)
    else:
        result = emulate_gemm_complex(av, bv, cfg)
    if isinstance(cv, torch.Tensor):
        cv.copy_(torch.as_tensor(result).to(cv.device, cv.dtype))
    else:
        cv[...] = result
    return c


# ----------------------------------------------------------------------------
# stage-level parity hooks
# ----------------------------------------------------------------------------
def _i8_device(x, name, dev):
    if isinstance(x, torch.Tensor):
        if x.dim() != 2:
            raise DimensionError("operands must be 2-D")
        if x.dtype != torch.int8:
            raise DimensionError("operands must be int8")
        return x.to(dev).contiguous(), True
    arr = np.asarray(x)
    if arr.ndim != 2:
        raise DimensionError("operands must be 2-D")
    if arr.dtype != np.int8:
        raise DimensionError("operands must be int8")
    return torch.from_numpy(np.ascontiguousarray(arr)).to(dev), False


def _gemm_i8_raw(at, bt, dev):
    m, k = at.shape
    n = bt.shape[1]
    lib = nat.load()
    ws = _workspace(lib.crtg_i8_workspace_size(m, n, k, 1), dev)
    c = torch.empty((m, n), dtype=torch.int32, device=dev)
    nat.call("crtg_gemm_i8_i32", m, n, k, at.data_ptr(), bt.data_ptr(), c.data_ptr(),
             ws.data_ptr(), ws.numel(), _stream_ptr(dev))
    return c


def gemm_i8_i32(a, b):
    """Exact int8 x int8 -> int32 product on tcgen05 (reference kernel.py:20-35)."""
    dev = _device()
    at, ta = _i8_device(a, "A", dev)
    bt, tb = _i8_device(b, "B", dev)
    if at.shape[1] != bt.shape[0]:
        raise DimensionError(f"inner dimensions differ: {tuple(at.shape)} x {tuple(bt.shape)}")
    k = at.shape[1]
    if k > MAX_K_REAL:
        raise DimensionError(f"inner dimension {k} exceeds {MAX_K_REAL}")
    if k <= MAX_K_COMPLEX:
        c = _gemm_i8_raw(at, bt, dev)
    else:
        # |partial| <= 2^30 per half; the reference raises beyond int32 (kernel.py:33-34)
        h = MAX_K_COMPLEX
        c64 = (_gemm_i8_raw(at[:, :h].contiguous(), bt[:h].contiguous(), dev).to(torch.int64)
               + _gemm_i8_raw(at[:, h:].contiguous(), bt[h:].contiguous(), dev))
        if c64.numel() and int(c64.abs().max()) > 2 ** 31 - 1:
            raise ArithmeticError("dot product exceeds the 32-bit accumulator")
        c = c64.to(torch.int32)
    return c if (ta and tb) else c.cpu().numpy()


def _residue_bounds(p):
    lo = -(p // 2) if p % 2 == 0 else -((p - 1) // 2)
    return lo, (p - 1) // 2


def complex_gemm_mod(ar, ai, br, bi, p: int, strategy: str = "karatsuba",
                     n_block: int = 8192):
    """Modular complex product on residue operands (reference kernel.py:70-120):
    Karatsuba (three tcgen05 products, crtg_complex_gemm_mod) or the expanded
    formulations (one product on doubled operands, _expand_gemm_mod)."""
    if strategy not in STRATEGIES:
        raise DimensionError(f"unknown strategy {strategy!r}")
    if n_block < 1:
        raise DimensionError("n_block must be >= 1")
    dev = _device()
    ops = [_i8_device(np.asarray(x, dtype=np.int8) if not isinstance(x, torch.Tensor) else x,
                      nm, dev) for x, nm in ((ar, "ar"), (ai, "ai"), (br, "br"), (bi, "bi"))]
    (art, t0), (ait, _), (brt, _), (bit, _) = ops
    if art.shape != ait.shape or brt.shape != bit.shape:
        raise DimensionError("real/imaginary parts must share shapes")
    if art.shape[1] != brt.shape[0]:
        raise DimensionError(f"inner dimensions differ: {tuple(art.shape)} x {tuple(brt.shape)}")
    m, k = art.shape
    n = brt.shape[1]
    if k > MAX_K_COMPLEX:
        raise DimensionError(f"inner dimension {k} exceeds {MAX_K_COMPLEX} "
                             "for complex modular products")
    lo, hi = _residue_bounds(p)
    for name, t in (("ar", art), ("ai", ait), ("br", brt), ("bi", bit)):
        if t.numel() and (int(t.min()) < lo or int(t.max()) > hi):
            raise DimensionError(f"{name} entries outside residue range of p={p}")
    if strategy == "karatsuba":
        lib = nat.load()
        ws = _workspace(lib.crtg_i8_workspace_size(m, n, k, 3), dev)
        er = torch.empty((m, n), dtype=torch.int8, device=dev)
        ei = torch.empty((m, n), dtype=torch.int8, device=dev)
        nat.call("crtg_complex_gemm_mod", m, n, k, art.data_ptr(), ait.data_ptr(), brt.data_ptr(),
                 bit.data_ptr(), int(p), er.data_ptr(), ei.data_ptr(), ws.data_ptr(), ws.numel(),
                 _stream_ptr(dev))
    else:
        er, ei = _expand_gemm_mod(art, ait, brt, bit, int(p), strategy, n_block)
    if all(isinstance(x, torch.Tensor) for x in (ar, ai, br, bi)):
        return er, ei
    return er.cpu().numpy(), ei.cpu().numpy()


def _sym_i8(t: torch.Tensor, p: int) -> torch.Tensor:
    """Symmetric residues (symmetric_mod_int, crt.py:136-151) of an int32 / int64
    device tensor, as int8, on the residue kernel."""
    from .stages import _residues
    kind = 2 if t.dtype == torch.int32 else 1
    src = t if kind == 2 else t.to(torch.int64)
    return _residues(src.contiguous().reshape(-1), kind, (p,))[0].reshape(t.shape)


def _expand_gemm_mod(art, ait, brt, bit, p: int, strategy: str, n_block: int):
    """The reference's expanded formulations (kernel.py:54-67): ONE integer GEMM
    per column block on doubled operands -- [[ar, -ai], [ai, ar]] @ [br; bi]
    (expand-rows) or [ai, ar] @ [[br, -bi], [bi, br]] (expand-cols) -- on the
    tcgen05 gemm_i8_i32, reduced to symmetric residues.  Inner length 2k: like
    the reference, a dot product beyond int32 raises ArithmeticError
    (kernel.py:33-34) where the Karatsuba form cannot overflow."""
    m, k = art.shape
    n = brt.shape[1]
    er = torch.empty((m, n), dtype=torch.int8, device=art.device)
    ei = torch.empty((m, n), dtype=torch.int8, device=art.device)
    if strategy == "expand-rows":
        neg_ai = _sym_i8(-ait.to(torch.int32), p)
        a_hat = torch.cat([torch.cat([art, neg_ai], 1), torch.cat([ait, art], 1)], 0).contiguous()
        for j0 in range(0, n, n_block):
            j1 = min(j0 + n_block, n)
            b_hat = torch.cat([brt[:, j0:j1], bit[:, j0:j1]], 0).contiguous()
            c = gemm_i8_i32(a_hat, b_hat)
            er[:, j0:j1] = _sym_i8(c[:m], p)
            ei[:, j0:j1] = _sym_i8(c[m:], p)
    else:
        neg_bi = _sym_i8(-bit.to(torch.int32), p)
        a_hat = torch.cat([ait, art], 1).contiguous()
        for j0 in range(0, n, n_block):
            j1 = min(j0 + n_block, n)
            w = j1 - j0
            brb, bib = brt[:, j0:j1], bit[:, j0:j1]
            b_hat = torch.cat([torch.cat([brb, neg_bi[:, j0:j1]], 1), torch.cat([bib, brb], 1)],
                              0).contiguous()
            c = gemm_i8_i32(a_hat, b_hat)
            er[:, j0:j1] = _sym_i8(c[:, w:], p)
            ei[:, j0:j1] = _sym_i8(c[:, :w], p)
    return er, ei


def _emulate_complex_stages(at: torch.Tensor, bt: torch.Tensor, cfg: EmuConfig,
                            diagnostics: dict | None):
    """emulate_gemm_complex for the expand strategies, stage by stage exactly as
    the reference composes it (emulate.py:193-240): device exponents, quantize,
    residue_decompose, one complex_gemm_mod per modulus with cfg.strategy, CRT
    accumulate / reduce, inverse scale, re + 1j*im.  Every stage is a libcrtg
    kernel; the result is bitwise that of the fused Karatsuba pipeline (all
    strategies are identical by contract) unless an expanded dot product
    leaves int32, which raises ArithmeticError as in the reference."""
    from . import stages as stg
    ms = select_moduli(cfg.resolved_moduli)
    if at.dtype != torch.complex128:
        at = at.to(torch.complex128)
    if bt.dtype != torch.complex128:
        bt = bt.to(torch.complex128)
    sv = _scaling(at, bt, ms, nat.FAST if cfg.mode == "fast" else nat.ACCURATE, diagnostics)
    dev = at.device
    mu = torch.from_numpy(sv.mu_exp).to(dev)
    nu = torch.from_numpy(sv.nu_exp).to(dev)
    ar = stg.quantize(at.real.contiguous(), mu, 0)
    ai = stg.quantize(at.imag.contiguous(), mu, 0)
    br = stg.quantize(bt.real.contiguous(), nu, 1)
    bi = stg.quantize(bt.imag.contiguous(), nu, 1)
    st = [stg.residue_decompose(x, ms).entries for x in (ar, ai, br, bi)]
    m, n = ar.shape[0], br.shape[1]
    e_re = torch.empty((len(ms), m, n), dtype=torch.int8, device=dev)
    e_im = torch.empty((len(ms), m, n), dtype=torch.int8, device=dev)
    for idx, p in enumerate(ms.moduli):
        e_re[idx], e_im[idx] = complex_gemm_mod(st[0][idx], st[1][idx], st[2][idx], st[3][idx],
                                                p, strategy=cfg.strategy, n_block=cfg.n_block)
    path = cfg.precision
    c_re = stg.crt_reduce(stg.crt_accumulate(stg.ResidueStack(e_re, ms), ms, path), ms)
    c_im = stg.crt_reduce(stg.crt_accumulate(stg.ResidueStack(e_im, ms), ms, path), ms)
    odt = torch.float64 if cfg.precision == "double" else torch.float32
    re = stg.inverse_scale(c_re, sv, odt)
    im = stg.inverse_scale(c_im, sv, odt)
    # numpy's re + 1j*im: real = re + (0*im - 0), imag = 0 + (0 + im)
    real = re + (0.0 * im - 0.0)
    imag = 0.0 + (0.0 + im)
    return torch.complex(real, imag)


def _scaling(a, b, ms: ModulusSet, mode: int, diagnostics):
    dev = _device()
    at, _ = _to_device_matrix(a, "A", dev)
    bt, _ = _to_device_matrix(b, "B", dev)
    if at.dtype != bt.dtype:
        at, bt = at.to(torch.complex128), bt.to(torch.complex128)
    if at.shape[1] != bt.shape[0]:
        raise DimensionError("inner dimensions differ")
    m, k = at.shape
    n = bt.shape[1]
    if mode == nat.ACCURATE and k > MAX_K_COMPLEX:
        raise DimensionError(f"inner dimension {k} exceeds {MAX_K_COMPLEX} for the bound product")
    consts = device_constants(len(ms))
    prec = 16 if at.dtype == torch.complex64 else 0
    lib = nat.load()
    ws = _workspace(lib.crtg_workspace_size(prec, mode, m, n, k, len(ms), n), dev)
    mu = torch.empty(m, dtype=torch.int32, device=dev)
    nu = torch.empty(n, dtype=torch.int32, device=dev)
    diag = torch.zeros(nat.DIAG_LEN, dtype=torch.int64, device=dev)
    nat.call("crtg_scaling", prec, mode, m, n, k, at.data_ptr(), at.stride(0), bt.data_ptr(),
             bt.stride(0), ctypes.byref(consts), ws.data_ptr(), ws.numel(), mu.data_ptr(),
             nu.data_ptr(), diag.data_ptr(), _stream_ptr(dev))
    d = diag.cpu().tolist()
    if d[2] or d[3]:
        raise DomainError("matrix entries must be finite")
    if diagnostics is not None:
        for key, idx in (("clamped_mu", 0), ("clamped_nu", 1)):
            if d[idx]:
                diagnostics[key] = diagnostics.get(key, 0) + int(d[idx])
    return ScalingVectors(mu.cpu().numpy().astype(np.int64), nu.cpu().numpy().astype(np.int64))


def fast_scaling(a, b, ms: ModulusSet, sc: ScalingConstants | None = None,
                 diagnostics: dict | None = None) -> ScalingVectors:
    """Cauchy-Schwarz exponents on the GPU (reference scaling.py:198-213).
    Complex (or real, treated with a zero imaginary part) operands."""
    return _scaling(a, b, ms, nat.FAST, diagnostics)


def accurate_scaling(a, b, ms: ModulusSet, sc: ScalingConstants | None = None,
                     diagnostics: dict | None = None) -> ScalingVectors:
    """Bound-GEMM exponents on the GPU (reference scaling.py:229-274)."""
    return _scaling(a, b, ms, nat.ACCURATE, diagnostics)


def quantized_residues(mat, exps, ms: ModulusSet, axis: int = 0):
    """trunc(mat * 2^exps) reduced to symmetric residues for every modulus:
    int8 array (N, 3, rows, cols) with planes (re, im, sym(re+im)).  axis=0:
    exps per row (left operand); axis=1: exps per column (right operand).
    (reference quantize scaling.py:277-293 + residue_decompose crt.py:199-218 +
    the Karatsuba sums kernel.py:101-103)."""
    dev = _device()
    xt, was_t = _to_device_matrix(mat, "matrix", dev)
    exps_np = np.asarray(exps, dtype=np.int64)
    if axis not in (0, 1):
        raise ConfigError("axis must be 0 (rows) or 1 (columns)")
    if exps_np.shape[0] != xt.shape[axis]:
        raise DimensionError("exponent vector does not match matrix")
    # np.ldexp semantics outside the kernel's exact-multiply range: 2^e with
    # e > 1023 overflows any nonzero entry (DomainError in quantize), e < -1074
    # flushes every entry to zero
    big = exps_np > 1023
    if big.any():
        xs = xt.abs().amax(dim=1 if axis == 0 else 0).cpu().numpy()
        if np.any(xs[big] != 0):
            raise DomainError("scaled magnitudes exceed the quantization budget")
    et = torch.from_numpy(np.clip(exps_np, -1074, 1023).astype(np.int32)).to(dev)
    rows, kdim = (xt.shape[0], xt.shape[1]) if axis == 0 else (xt.shape[1], xt.shape[0])
    consts = device_constants(len(ms))
    nmod = len(ms)
    r_pad = -(-rows // 256) * 256
    k_pad = -(-kdim // 128) * 128
    ws = _workspace(3 * nmod * r_pad * k_pad, dev)
    out = torch.empty((nmod, 3, rows, kdim), dtype=torch.int8, device=dev)
    diag = torch.zeros(nat.DIAG_LEN, dtype=torch.int64, device=dev)
    prec = 16 if xt.dtype == torch.complex64 else 0
    nat.call("crtg_residues", prec, axis, rows, kdim, xt.data_ptr(), xt.stride(0), et.data_ptr(),
             ctypes.byref(consts), out.data_ptr(), ws.data_ptr(), ws.numel(), diag.data_ptr(),
             _stream_ptr(dev))
    d = diag.cpu().tolist()
    if d[4] or d[5]:
        raise DomainError("scaled magnitudes exceed the quantization budget")
    if axis == 1:
        out = out.transpose(2, 3)  # back to (k, n) orientation
    return out if was_t else out.cpu().numpy()


def crt_reconstruct(e_re, e_im, mu, nu, ms: ModulusSet, precision: str = "double"):
    """CRT accumulate + reduce + inverse scaling of residue stacks (N, m, n)
    (reference crt.py:221-258 + emulate.py:135-144, 234-240)."""
    dev = _device()
    ert = torch.as_tensor(np.asarray(e_re, np.int8) if not isinstance(e_re, torch.Tensor)
                          else e_re).to(dev).contiguous()
    eit = torch.as_tensor(np.asarray(e_im, np.int8) if not isinstance(e_im, torch.Tensor)
                          else e_im).to(dev).contiguous()
    nmod, m, n = ert.shape
    if nmod != len(ms):
        raise ConfigError("stack depth does not match modulus count")
    mut = torch.as_tensor(np.asarray(mu, np.int64).astype(np.int32)).to(dev)
    nut = torch.as_tensor(np.asarray(nu, np.int64).astype(np.int32)).to(dev)
    odt = torch.complex64 if precision == "single" else torch.complex128
    out = torch.empty((m, n), dtype=odt, device=dev)
    nat.call("crtg_crt_reconstruct", nat.SINGLE if precision == "single" else nat.DOUBLE, m, n,
             ert.data_ptr(), eit.data_ptr(), mut.data_ptr(), nut.data_ptr(),
             ctypes.byref(device_constants(len(ms))), out.data_ptr(), out.stride(0),
             _stream_ptr(dev))
    return out.cpu().numpy()
