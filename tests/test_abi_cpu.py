"""CPU: the C-ABI library builds, loads and exports exactly what include/crtg.h
declares; the product has no CPU compute path (no GPU here -> it must raise)."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "crtg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(crtg_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2512_08321_b200 import _native, build
    build.build()
    return _native.load()


def test_header_symbols_exported(lib):
    names = _declared()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name


def test_bindings_match_header(lib):
    from paper_2512_08321_b200 import _native
    assert sorted(_native.SIGNATURES) == _declared()


def test_version_and_workspace_queries(lib):
    assert lib.crtg_version().startswith(b"crtg")
    # workspace planning is host-only arithmetic; 16384^3, N=14, two column blocks
    ws = lib.crtg_workspace_size(0, 0, 16384, 16384, 16384, 14, 8192)
    planes = 3 * 14 * 16384 * 16384 + 3 * 14 * 8192 * 16384 + 2 * 14 * 16384 * 8192
    assert planes <= ws < planes + (1 << 24)
    assert lib.crtg_i8_workspace_size(100, 100, 100, 1) > 0


def test_sass_is_tcgen05(lib):
    """The GEMM really is a tcgen05 kernel fed by the TMA engine (UTC*MMA, UBLKCP)."""
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    so = os.path.join(ROOT, "paper_2512_08321_b200", "libcrtg.so")
    out = subprocess.run([cuobjdump, "-sass", so], capture_output=True, text=True).stdout
    assert "UTCIMMA" in out  # tcgen05.mma.kind::i8
    assert "UBLKCP" in out or "UTMALDG" in out
    assert "LDTM" in out
    assert "HMMA" not in out and "IMMA." not in out.replace("UTCIMMA", "")


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2512_08321_b200 as crt
    from paper_2512_08321_b200 import _native
    with pytest.raises(_native.NativeError):
        crt.emulate_gemm_complex(np.ones((2, 2), complex), np.ones((2, 2), complex))
    with pytest.raises(_native.NativeError):
        crt.gemm_i8_i32(np.ones((2, 2), np.int8), np.ones((2, 2), np.int8))
