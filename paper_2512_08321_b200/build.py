"""Build libcrtg.so (sm_100a) in-tree with nvcc.

    python -m paper_2512_08321_b200.build        # or __graft_entry__.build()

Every translation unit is compiled for `-gencode arch=compute_100a,code=sm_100a`
with -lineinfo (ncu source view).  The exactness-critical units (scaling,
residue, crt) additionally get -fmad=false so no FP multiply-add is ever
contracted (numpy never fuses); the GEMM/API units are integer code.
The CUDA runtime is linked statically so the library does not depend on which
libcudart torch happens to load.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libcrtg.so")
BUILD = os.path.join(HERE, "_build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
          "--expt-relaxed-constexpr"]
EXACT = {"scaling.cu", "residue.cu", "crt.cu", "accuracy.cu"}
SOURCES = ["api.cu", "gemm_tc.cu", "scaling.cu", "residue.cu", "crt.cu", "accuracy.cu"]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; cannot build the sm_100a kernels")
    return cand


def _stale(src_files, target) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(f) > t for f in src_files)


def build(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "crtg.h"))
    deps.append(os.path.abspath(__file__))
    if not force and not _stale(deps, OUT):
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    cc = nvcc()

    def compile_one(src):
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        flags = list(COMMON)
        # A/B experiments only: extra -D definitions (e.g. CRTG_NVCC_DEFS="CRTG_EPI_DB=1")
        flags += ["-D" + d for d in os.environ.get("CRTG_NVCC_DEFS", "").split()]
        if src in EXACT:
            flags.append("-fmad=false")
        if src == "api.cu":
            flags += ["-Xcompiler", "-fopenmp"]  # host-side staging copies
        cmd = [cc, *ARCH, *flags, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = OUT + ".tmp"
    cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-Xcompiler", "-fopenmp", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
