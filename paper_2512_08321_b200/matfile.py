"""OZ2M matrix files — the reference's on-disk format (pkg/src/crtgemm/matfile.py:1-57).

File = b"OZ2M" | int64 rows | int64 cols | uint8 dtype code | payload, all
little-endian; codes 0 = f32, 1 = f64, 2 = c32 (complex64), 3 = c64
(complex128); the payload is the matrix in COLUMN-MAJOR element order.

Differences from the reference are performance only: the payload is streamed
with `ndarray.tofile` / `np.fromfile` (no full in-memory bytes copy, which
matters at 16384^2 complex128 = 4 GiB), and `write_matrix` accepts torch
tensors (CPU or CUDA) as well as anything `np.asarray` takes.  Errors are the
reference's: `ValueError` for a bad magic, truncated header or payload,
negative dimensions, unknown code, unsupported dtype or non-2-D input.
"""

from __future__ import annotations

import os
import struct

import numpy as np

MAGIC = b"OZ2M"
_HDR = struct.Struct("<qqB")
_DTYPES = ("<f4", "<f8", "<c8", "<c16")  # index = dtype code


def dtype_code(dtype) -> int:
    """OZ2M code of a numpy dtype (matfile.py:19-24)."""
    dt = np.dtype(dtype)
    for code, name in enumerate(_DTYPES):
        if dt.kind == np.dtype(name).kind and dt.itemsize == np.dtype(name).itemsize:
            return code
    raise ValueError(f"unsupported matrix dtype {dtype!r}; use f32, f64, c32 or c64")


def _as_numpy(matrix) -> np.ndarray:
    try:
        import torch
        if isinstance(matrix, torch.Tensor):
            return matrix.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(matrix)


def write_matrix(path, matrix) -> None:
    """Write a 2-D matrix as OZ2M (matfile.py:27-36)."""
    arr = _as_numpy(matrix)
    if arr.ndim != 2:
        raise ValueError("only 2-D matrices are supported")
    code = dtype_code(arr.dtype)
    rows, cols = arr.shape
    # column-major payload: the transpose of a Fortran-ordered array is
    # C-contiguous, so tofile() streams it without another copy
    payload = np.asfortranarray(arr.astype(_DTYPES[code], copy=False)).T
    with open(path, "wb") as fh:
        fh.write(MAGIC + _HDR.pack(rows, cols, code))
        if payload.size:
            payload.tofile(fh)


def read_matrix(path) -> np.ndarray:
    """Read an OZ2M file into a native-endian array (matfile.py:39-57)."""
    with open(path, "rb") as fh:
        if fh.read(4) != MAGIC:
            raise ValueError(f"{path}: not an OZ2M matrix file")
        hdr = fh.read(_HDR.size)
        if len(hdr) != _HDR.size:
            raise ValueError(f"{path}: truncated header")
        rows, cols, code = _HDR.unpack(hdr)
        if rows < 0 or cols < 0:
            raise ValueError(f"{path}: negative dimensions")
        if code >= len(_DTYPES):
            raise ValueError(f"{path}: unknown dtype code {code}")
        dt = np.dtype(_DTYPES[code])
        count = rows * cols
        avail = os.fstat(fh.fileno()).st_size - fh.tell()
        if avail < count * dt.itemsize:
            raise ValueError(f"{path}: truncated data section")
        flat = np.fromfile(fh, dtype=dt, count=count) if count else np.empty(0, dt)
    # native-endian copy that keeps the column-major layout, as the reference's
    return flat.reshape((rows, cols), order="F").astype(dt.newbyteorder("="))
