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
from .gen import GenSpec, gen_matrix
from .matfile import read_matrix, write_matrix
from .moduli import ModulusSet, ScalingConstants, select_moduli
from .perfmodel import PerfParams, heatmap_csv, heatmap_grid, predict_time, predicted_tflops
from .stages import (ComplexMatrix, ResidueStack, ScaledIntMatrices, crt_accumulate,
                     crt_integer_gemm, crt_reduce, inverse_scale, log2_upper, quantize,
                     residue_decompose, symmetric_mod_int, symmetric_mod_wide)


def __getattr__(name):
    # the accuracy harness imports torch-side helpers lazily
    if name in ("DDMatrix", "reference_gemm_dd", "max_relative_error", "run_accuracy_sweep",
                "sweep_csv", "exact_gemm_bigint"):
        from . import accuracy
        return getattr(accuracy, name)
    raise AttributeError(name)

__version__ = "0.1.0"

__all__ = [
    "ComplexMatrix", "ResidueStack", "ScaledIntMatrices", "crt_accumulate", "crt_integer_gemm",
    "crt_reduce", "inverse_scale", "log2_upper", "quantize", "residue_decompose",
    "symmetric_mod_int", "symmetric_mod_wide",
    "ConfigError", "DDMatrix", "exact_gemm_bigint", "DEFAULT_N_BLOCK", "DimensionError", "DomainError", "EmuConfig",
    "GenSpec", "MAX_K_COMPLEX", "MAX_K_REAL", "ModulusSet", "PerfParams", "STRATEGIES",
    "ScalingConstants", "ScalingVectors", "accurate_scaling", "complex_gemm_mod",
    "crt_reconstruct", "emulate_gemm_complex", "emulate_gemm_real", "fast_scaling", "gemm",
    "gemm_i8_i32", "gen_matrix", "heatmap_csv", "heatmap_grid", "max_relative_error",
    "predict_time", "predicted_tflops", "quantized_residues", "read_matrix", "reference_gemm_dd",
    "run_accuracy_sweep", "run_complex", "select_moduli", "sweep_csv", "write_matrix",
]
