"""ctypes binding of the C-ABI in include/crtg.h (libcrtg.so, built in-tree).

There is no fallback: if the library is missing or the device is not an
sm_100 part, every entry point raises.  The symbols bound here are exactly the
ones include/crtg.h declares (tests/test_abi.py checks both directions).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigError, DimensionError, DomainError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcrtg.so")

OK, ERR_CONFIG, ERR_DIMENSION, ERR_DOMAIN, ERR_CUDA, ERR_WORKSPACE, ERR_ARITH = range(7)
DOUBLE, SINGLE = 0, 1
FAST, ACCURATE = 0, 1
DIAG_LEN = 8
DIAG_CLAMPED_MU, DIAG_CLAMPED_NU = 0, 1

_c_i64, _c_int, _vp, _sz = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t

# name -> (restype, argtypes)
SIGNATURES = {
    "crtg_version": (ctypes.c_char_p, []),
    "crtg_last_error": (ctypes.c_char_p, []),
    "crtg_device_check": (_c_int, [_c_int]),
    "crtg_workspace_size": (_sz, [_c_int, _c_int, _c_i64, _c_i64, _c_i64, _c_int, _c_i64]),
    "crtg_gemm_complex": (_c_int, [_c_int, _c_int, _c_i64, _c_i64, _c_i64, _vp, _c_i64, _vp,
                                   _c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _sz, _vp, _vp, _vp,
                                   _c_int, _vp]),
    "crtg_scaling": (_c_int, [_c_int, _c_int, _c_i64, _c_i64, _c_i64, _vp, _c_i64, _vp, _c_i64,
                              _vp, _vp, _sz, _vp, _vp, _vp, _vp]),
    "crtg_residues": (_c_int, [_c_int, _c_int, _c_i64, _c_i64, _vp, _c_i64, _vp, _vp, _vp, _vp,
                               _sz, _vp, _vp]),
    "crtg_i8_workspace_size": (_sz, [_c_i64, _c_i64, _c_i64, _c_int]),
    "crtg_gemm_i8_i32": (_c_int, [_c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "crtg_complex_gemm_mod": (_c_int, [_c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _c_int, _vp,
                                       _vp, _vp, _sz, _vp]),
    "crtg_crt_reconstruct": (_c_int, [_c_int, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp,
                                      _c_i64, _vp]),
    "crtg_host_workspace_size": (_sz, [_c_int, _c_int, _c_i64, _c_i64, _c_i64, _c_int, _c_i64]),
    "crtg_gemm_complex_host": (_c_int, [_c_int, _c_int, _c_i64, _c_i64, _c_i64, _vp, _c_i64, _vp,
                                        _c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _sz, _vp, _c_int,
                                        _vp]),
    "crtg_real_workspace_size": (_sz, [_c_int, _c_int, _c_i64, _c_i64, _c_i64, _c_int, _c_i64]),
    "crtg_gemm_real": (_c_int, [_c_int, _c_int, _c_i64, _c_i64, _c_i64, _vp, _c_i64, _c_int, _vp,
                                _c_i64, _c_int, _vp, _c_i64, _vp, _c_i64, _vp, _sz, _vp, _vp,
                                _vp, _c_int, _vp]),
    "crtg_gemm_complex_exps": (_c_int, [_c_int, _c_i64, _c_i64, _c_i64, _vp, _c_i64, _vp,
                                        _c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _vp, _vp, _sz,
                                        _vp, _c_int, _vp]),
    "crtg_accurate_partial": (_c_int, [_c_int, _c_i64, _c_i64, _c_i64, _vp, _c_i64, _vp, _c_i64,
                                       _vp, _vp, _sz, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "crtg_accurate_exponents": (_c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "crtg_dd_gemm": (_c_int, [_c_int, _c_i64, _c_i64, _c_i64, _vp, _c_i64, _vp, _c_i64, _vp,
                              _vp, _c_i64, _vp]),
    "crtg_max_relative_error": (_c_int, [_c_int, _c_i64, _c_i64, _vp, _c_int, _c_i64, _vp, _vp,
                                         _c_i64, _vp, _vp, _vp]),
    "crtg_release_host_staging": (None, []),
    "crtg_log2_upper": (_c_int, [_vp, _c_i64, _vp, _vp, _c_int, _vp]),
    "crtg_quantize": (_c_int, [_vp, _c_i64, _c_i64, _c_i64, _vp, _c_int, _vp, _c_i64, _vp,
                               _c_int, _vp]),
    "crtg_symmetric_mod": (_c_int, [_c_int, _vp, _c_i64, _vp, _c_int, _vp, _vp, _c_int, _vp]),
    "crtg_crt_accumulate": (_c_int, [_vp, _c_i64, _vp, _c_int, _vp, _vp, _vp]),
    "crtg_symmetric_mod_wide": (_c_int, [_vp, _vp, _c_i64, ctypes.c_double, ctypes.c_double,
                                         _c_int, _vp, _vp]),
    "crtg_inverse_scale": (_c_int, [_vp, _c_i64, _c_i64, _c_i64, _vp, _vp, _c_int, _vp, _c_i64,
                                    _vp]),
    "crtg_launch_count": (ctypes.c_uint64, []),
    "crtg_profile_enable": (_c_int, [_c_int]),
    "crtg_profile_read": (_c_int, [_vp, _vp]),
}

STAGES = ("scaling", "residue_a", "residue_b", "gemm", "crt")


def profile_enable(on: bool) -> None:
    raise_for(load().crtg_profile_enable(1 if on else 0))


def profile_read():
    """-> ({stage: device ms}, {stage: launches}); synchronizes the recorded events."""
    ms = (ctypes.c_double * len(STAGES))()
    cnt = (ctypes.c_uint64 * len(STAGES))()
    raise_for(load().crtg_profile_read(ctypes.addressof(ms), ctypes.addressof(cnt)))
    return dict(zip(STAGES, list(ms))), dict(zip(STAGES, list(cnt)))


def launch_count() -> int:
    return int(load().crtg_launch_count())

_lib = None
_lock = threading.Lock()
_checked_devices: set = set()


class NativeError(RuntimeError):
    """CUDA-side failure of the native library (no CPU fallback exists)."""


def load(path: str | None = None) -> ctypes.CDLL:
    """Load libcrtg.so and bind every declared symbol; raises if absent.
    CRTG_LIB=/path/to/libcrtg.so selects another build of the same library
    (A/B timing of kernel variants, tools/ab.py)."""
    global _lib
    if _lib is not None and path is None:  # hot path: no lock once loaded
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = path or os.environ.get("CRTG_LIB") or LIB_PATH
        if not os.path.exists(path):
            raise NativeError(
                f"{path} is missing: build it with `python -m paper_2512_08321_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def raise_for(status: int) -> None:
    if status == OK:
        return
    msg = load().crtg_last_error().decode()
    if status == ERR_CONFIG:
        raise ConfigError(msg)
    if status == ERR_DIMENSION:
        raise DimensionError(msg)
    if status == ERR_DOMAIN:
        raise DomainError(msg)
    if status == ERR_ARITH:
        raise ArithmeticError(msg)
    raise NativeError(msg)


def call(name: str, *args):
    status = getattr(load(), name)(*args)
    raise_for(status)


def check_device(index: int) -> None:
    if index in _checked_devices:
        return
    raise_for(load().crtg_device_check(index))
    _checked_devices.add(index)
