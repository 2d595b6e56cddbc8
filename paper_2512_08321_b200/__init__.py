"""B200-native (sm_100a) Ozaki-II / CRT emulation of complex GEMM.

Drop-in for the complex-GEMM path of the reference `crtgemm` package
(arXiv 2512.08321): same entry points (`EmuConfig`, `emulate_gemm_complex`,
`gemm`), knobs (`num_moduli`, fast/accurate `mode`) and errors, computed by
hand-written tcgen05 / TMA kernels in `libcrtg.so` (include/crtg.h).
"""

from .config import DEFAULT_N_BLOCK, MAX_K_COMPLEX, MAX_K_REAL, STRATEGIES, EmuConfig
from .emulate import (ScalingVectors, accurate_scaling, complex_gemm_mod, crt_reconstruct,
                      emulate_gemm_complex, emulate_gemm_real, fast_scaling, gemm, gemm_i8_i32,
                      quantized_residues, run_complex)
from .errors import ConfigError, DimensionError, DomainError
from .moduli import ModulusSet, ScalingConstants, select_moduli

__version__ = "0.1.0"

__all__ = [
    "ConfigError", "DEFAULT_N_BLOCK", "DimensionError", "DomainError", "EmuConfig",
    "MAX_K_COMPLEX", "MAX_K_REAL", "ModulusSet", "STRATEGIES", "ScalingConstants",
    "ScalingVectors", "accurate_scaling", "complex_gemm_mod", "crt_reconstruct",
    "emulate_gemm_complex", "emulate_gemm_real", "fast_scaling", "gemm", "gemm_i8_i32", "quantized_residues",
    "run_complex", "select_moduli",
]
