// kernels.cuh — launch interfaces of the non-GEMM kernels (scaling, residues, CRT).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace crtg {

// element type of an input matrix
enum Elem { E_C128 = 0, E_C64 = 1, E_F64 = 2, E_F32 = 3 };

// numpy pairwise-sum recursion of one row, flattened: leaves (start, len) in
// order, internal nodes (left slot, right slot) sorted by height; value slot s
// < nleaves is a leaf, else internal node s - nleaves.
struct PwTree {
  int nleaves, nnodes, nlevels;
  const int2* leaves;
  const int2* nodes;
  const int* level_start;  // nlevels + 1 entries into nodes
};

// ---- scaling (scaling.cu) ----
// A rows: absmax (+ non-finite flag) and, in fast mode, the pairwise sum of
// squares and the exponent.  Writes mu[i] (fast) or rowabs[i] (always).
int launch_row_stats(int elem, bool fast, const void* A, int64_t lda, int64_t m, int64_t k,
                     const PwTree& tree, float p_fast, float delta, int32_t* mu, double* rowabs,
                     unsigned long long* diag, cudaStream_t s);
// B columns: absmax per column (atomic max on the bit pattern) + non-finite flag.
int launch_col_absmax(int elem, const void* B, int64_t ldb, int64_t k, int64_t n,
                      double* colabs, unsigned long long* diag, cudaStream_t s);
// B columns: sequential sums of squares (numpy axis-0 order) and the exponent.
// fast-mode column stats: absmax -> colabs, exponents -> nu (one pass)
int launch_col_fast(int elem, const void* B, int64_t ldb, int64_t k, int64_t n,
                    double* colabs, double* colsq, float p_fast, float delta, int32_t* nu,
                    unsigned long long* diag, cudaStream_t s);
// accurate mode: bar = 5 - floor_log2(absmax) (0 for zero rows/cols)
int launch_bar(const double* absval, int64_t count, int32_t* bar, cudaStream_t s);
// accurate mode exponents from the bound maxima (scaling.py:260-271)
int launch_accurate_exps(const int32_t* maxb, const double* absval, const int32_t* bar,
                         int64_t count, float p_accu, float delta, int32_t* out,
                         unsigned long long* clamp_counter, cudaStream_t s);

// ---- residues / operand packing (residue.cu) ----
enum PackKind { PACK_RESIDUE = 0, PACK_BARS = 1 };
// operand 0: rows of A (m x k row-major complex), exps per row;
// operand 1: columns [col0, col0+rows) of B (k x n row-major complex), exps per column.
// Writes planes [N][3] (complex: re, im, re+im) or [N][1] (real) of
// k_pad x rb_count*128 packed bytes.
int launch_pack(int elem, int operand, int kind, const void* X, int64_t ldx, int64_t rows,
                int64_t kdim, int64_t col0, const int32_t* exps, const DevConsts& dc,
                int8_t* out, int64_t plane_bytes, int64_t rb_count,
                unsigned long long* overflow_flag, cudaStream_t s, int max_ctas = 0,
                int64_t row_base = 0, int64_t fill_rows = 0);
// plain int8 matrix -> one packed plane.  trans=0: X is rows x kdim row-major;
// trans=1: X is kdim x rows row-major (a right operand).
int launch_pack_i8(const int8_t* X, int trans, int64_t rows, int64_t kdim, int8_t* out,
                   int64_t rb_count, cudaStream_t s);
// packed plane -> plain int8 rows x kdim
int launch_unpack_i8(const int8_t* packed, int64_t rows, int64_t kdim, int64_t rb_count,
                     int8_t* out, cudaStream_t s);

// ---- CRT reconstruction (crt.cu) ----
// real = true: e_im unused, C is a real f64 / f32 matrix
int launch_crt(bool single, bool real, int64_t m, int64_t n, const int8_t* e_re, const int8_t* e_im,
               int64_t e_plane, int64_t e_ld, const int32_t* mu, const int32_t* nu,
               const DevConsts& dc, void* C, int64_t ldc, cudaStream_t s, int max_ctas = 0);

// ---- accuracy harness (accuracy.cu) ----
int launch_dd_gemm(bool cplx, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                   const double* B, int64_t ldb, double* hi, double* lo, int64_t ldo,
                   cudaStream_t s);
int launch_max_rel_err(bool cplx, int64_t m, int64_t n, const void* approx, bool approx_single,
                       int64_t lda_x, const double* hi, const double* lo, int64_t ldo,
                       unsigned long long* max_bits, unsigned long long* zeros, cudaStream_t s);

// ---- stage-level API (stages.py / crtg_stage_*) ----
struct SymModuli {
  int n;
  int p[CRTG_MAX_MODULI];
};
struct CrtCoeffs {
  double hi[CRTG_MAX_MODULI];
  double lo[CRTG_MAX_MODULI];
};
int launch_log2_upper(const double* x, int64_t n, float* out, unsigned long long* flags,
                      cudaStream_t s);
int launch_quantize(const double* x, int64_t rows, int64_t cols, int64_t ldx, const int64_t* exps,
                    int axis, double* out, int64_t ldo, unsigned long long* flags,
                    cudaStream_t s);
int launch_sym_mod(int kind, const void* x, int64_t count, const SymModuli& mods, int8_t* out,
                   unsigned long long* flags, cudaStream_t s);
int launch_crt_accumulate(const int8_t* e, int nmod, int64_t count, const CrtCoeffs& cf,
                          bool single, double* s1, double* s2, cudaStream_t s);
int launch_sym_mod_wide(const double* s_hi, const double* s_lo, int64_t count, double p_hi,
                        double p_lo, bool use_dd, double* out, cudaStream_t s);
int launch_inverse_scale(const double* c, int64_t rows, int64_t cols, int64_t ldc,
                         const int64_t* mu, const int64_t* nu, bool out_f32, void* out,
                         int64_t ldo, cudaStream_t s);

}  // namespace crtg
