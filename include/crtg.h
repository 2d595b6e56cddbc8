/*
 * crtg.h — C-ABI of the B200 (sm_100a) Ozaki-II / CRT complex GEMM emulation.
 *
 * This is the drop-in boundary for the reference's hot path
 * `crtgemm.emulate_gemm_complex` (/root/reference/pkg/src/crtgemm/emulate.py:193-240)
 * and its BLAS-style wrapper `crtgemm.gemm` (emulate.py:256-278).  The reference
 * is a pure-Python package, so "the reference FFI for this path" is its Python
 * call surface; every entry point below replaces one reference function and is
 * bound with ctypes by `paper_2512_08321_b200/_native.py`.
 *
 * Conventions
 *   - All matrix pointers are DEVICE pointers; `stream` is a cudaStream_t (NULL =
 *     legacy default stream).  Every launch is stream-ordered; scratch comes from
 *     the caller-owned workspace `ws`.  The only memory the library allocates
 *     itself is the small, documented "library-held state" below (a one-time
 *     device tree per (device, k) and, for pageable host operands only, a pinned
 *     staging ring released by crtg_release_host_staging()).
 *   - Complex matrices are interleaved (re, im) pairs, row-major, with a row
 *     stride `ld*` counted in complex elements.  Inputs are complex128, or
 *     complex64 with CRTG_IN_C64 (upcast exactly, emulate.py:159-166); the
 *     result is complex128 (CRTG_DOUBLE) or complex64 (CRTG_SINGLE).
 *   - Return value: CRTG_OK or one of the CRTG_ERR_* codes; crtg_last_error()
 *     returns a thread-local message.  The Python layer maps
 *     CONFIG->ConfigError, DIMENSION->DimensionError, DOMAIN->DomainError
 *     (reference errors.py:4-13).
 *   - Data-dependent domain errors (non-finite input, |a'| >= 2^90 after
 *     scaling) are detected on the device and reported through `diag`
 *     (device uint64[CRTG_DIAG_LEN]); with sync_check != 0 the call synchronizes
 *     the stream and returns CRTG_ERR_DOMAIN itself.
 */
#ifndef CRTG_H
#define CRTG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CRTG_MAX_MODULI 20

enum crtg_status {
  CRTG_OK = 0,
  CRTG_ERR_CONFIG = 1,     /* ConfigError     */
  CRTG_ERR_DIMENSION = 2,  /* DimensionError  */
  CRTG_ERR_DOMAIN = 3,     /* DomainError     */
  CRTG_ERR_CUDA = 4,       /* launch / device failure */
  CRTG_ERR_WORKSPACE = 5,  /* ws too small */
  CRTG_ERR_ARITH = 6       /* ArithmeticError (int32 accumulator bound) */
};

/* precision argument: low bit = result precision (double -> complex128 result
 * and the double-double CRT path; single -> complex64 result and the plain-f64
 * CRT path, crt.py:246-258).  OR in CRTG_IN_C64 when the inputs are complex64
 * (read and upcast exactly on the device); otherwise inputs are complex128. */
enum crtg_precision {
  CRTG_DOUBLE = 0,
  CRTG_SINGLE = 1,
  CRTG_IN_C64 = 16, /* complex entry points: inputs are complex64 */
  CRTG_IN_F32 = 16  /* real entry point: inputs are float32 */
};
enum crtg_mode { CRTG_FAST = 0, CRTG_ACCURATE = 1 };

/* diag[] slots (device uint64) */
enum crtg_diag {
  CRTG_DIAG_CLAMPED_MU = 0,  /* scaling.py:165-171 key "clamped_mu" */
  CRTG_DIAG_CLAMPED_NU = 1,  /* key "clamped_nu" */
  CRTG_DIAG_NONFINITE_A = 2, /* emulate.py:163-165 */
  CRTG_DIAG_NONFINITE_B = 3,
  CRTG_DIAG_OVERFLOW_A = 4,  /* scaling.py:290-292, crt.py:209-210 */
  CRTG_DIAG_OVERFLOW_B = 5,
  CRTG_DIAG_INT32_OVERFLOW = 6, /* kernel.py:33-34 (real path, k > 2^16 only) */
  CRTG_DIAG_LEN = 8
};

/*
 * Modulus-set constants.  Built on the host from exact big-integer arithmetic
 * (reference crt.py:52-110 `ModulusSet.from_moduli`, scaling.py:100-115
 * `ScalingConstants.from_product`) — the Python layer fills it.
 */
typedef struct crtg_consts {
  int32_t num_moduli;                  /* N in 1..20 */
  int32_t moduli[CRTG_MAX_MODULI];     /* descending, pairwise coprime, <= 256 */
  double coeff_hi[CRTG_MAX_MODULI];    /* crt.py:84-86 */
  double coeff_lo[CRTG_MAX_MODULI];
  double p_hi;                         /* float(P)           crt.py:163 */
  double p_lo;                         /* float(P - int(p_hi)) crt.py:164 */
  float p_fast;                        /* ScalingConstants.p_fast */
  float p_accu;                        /* ScalingConstants.p_accu */
  float delta;                         /* ScalingConstants.delta  */
  int32_t reserved;
} crtg_consts;

/* library identity / errors */
const char* crtg_version(void);
const char* crtg_last_error(void);
/* 0 if `device` is an sm_100 part the kernels were built for, else CRTG_ERR_CUDA */
int crtg_device_check(int device);

/*
 * Bytes of scratch `crtg_gemm_complex` needs.  n_block bounds the number of B
 * columns processed per pass (reference kernel.py:15 DEFAULT_N_BLOCK, used here
 * as a working-set bound only — results are bitwise independent of it).
 */
size_t crtg_workspace_size(int precision, int mode, int64_t m, int64_t n, int64_t k,
                           int num_moduli, int64_t n_block);

/*
 * C = A @ B emulated with N moduli (replaces emulate_gemm_complex,
 * emulate.py:193-240).  A: m x k, B: k x n, C: m x n.  mu_out / nu_out
 * (device int32[m] / int32[n], may be NULL) receive the scaling exponents.
 */
int crtg_gemm_complex(int precision, int mode, int64_t m, int64_t n, int64_t k,
                      const void* A, int64_t lda, const void* B, int64_t ldb,
                      void* C, int64_t ldc, const crtg_consts* K, int64_t n_block,
                      void* ws, size_t ws_bytes, int32_t* mu_out, int32_t* nu_out,
                      uint64_t* diag, int sync_check, void* stream);

/*
 * Library-held state (everything else is caller-owned: A, B, C, the workspace
 * and the stream; every kernel is stream-ordered on the caller's stream).
 *  - Immutable per-thread cache of the last 8 modulus-constant tables built
 *    from crtg_consts (host memory, a few KB each).
 *  - Immutable per-(device, k) pairwise-sum tree of the fast-mode row
 *    statistics (numpy's summation order), uploaded once with cudaMalloc and
 *    kept for the process lifetime (16 * (k / 64 + 4) bytes: 16 KB at k = 65536).
 *  - Per-thread, per-device auxiliary streams: one fork stream (highest
 *    priority) for B's chain on small products and two copy-engine streams of
 *    crtg_gemm_complex_host.  They are joined to the caller's stream with
 *    events before the call returns.
 *  - Per-thread 64-byte page-locked buffers that synchronous calls read their
 *    device counters back into (sync_check = 1), right before synchronising:
 *    one filled by a copy, and one device-mapped that the captured graphs of
 *    synchronous small products write from their last kernel.
 *  - Per-thread cache of up to 16 instantiated CUDA graphs of small complex
 *    products (m*n*k <= ~2048^3, one column block), keyed by every argument of
 *    crtg_gemm_complex (pointers included): the second identical call captures
 *    its launch sequence, later ones replay it.  Kept until process exit;
 *    CRTG_GRAPHS=0 disables it.  A replay re-reads the operands, so in-place
 *    updates between calls are seen (tests/test_gpu_graphs.py).
 *  - crtg_gemm_complex_host with PAGEABLE A / B / C only: a per-thread ring of
 *    3 pinned staging slots, each one streamed piece (~1/16 of an operand; 256
 *    MiB at 16384^2 complex128).  Freed at thread exit or by
 *    crtg_release_host_staging() (call with no call in flight on the thread).
 * Concurrent calls from different host threads on different streams are safe
 * and bitwise identical to serial calls (tests/test_gpu_concurrency.py).
 */
void crtg_release_host_staging(void);

/*
 * The same product on HOST buffers (pinned for full overlap): A, B, C are host
 * pointers.  A's row chunks and B's column blocks (~1/16 of each) are copied in
 * interleaved on a copy engine; each landed piece releases a strip of output
 * tiles that is computed (one GEMM + CRT launch) while later pieces are still
 * in flight, and finished strips of C are copied back on a second copy engine.
 * `n_block` is accepted (results are bitwise invariant) but the pieces bound the
 * working set.  `ws` is a DEVICE workspace of crtg_host_workspace_size(...)
 * bytes.  On return (stream-ordered) C is complete once `stream` is synchronized.
 */
size_t crtg_host_workspace_size(int precision, int mode, int64_t m, int64_t n, int64_t k,
                                int num_moduli, int64_t n_block);
int crtg_gemm_complex_host(int precision, int mode, int64_t m, int64_t n, int64_t k,
                           const void* A, int64_t lda, const void* B, int64_t ldb,
                           void* C, int64_t ldc, const crtg_consts* K, int64_t n_block,
                           void* ws, size_t ws_bytes, uint64_t* diag, int sync_check,
                           void* stream);

/*
 * Real domain, C = A @ B with real float64 / float32 inputs (replaces
 * emulate_gemm_real, emulate.py:169-190): one INT8 product
 * per modulus.  a_colmajor / b_colmajor give each operand's storage order
 * (lda / ldb are then the column strides): the reference keeps the caller's
 * layout for real operands, and numpy's summation order for the fast-mode
 * exponents follows it (pairwise along the contiguous axis, sequential along the
 * strided one) — the library reproduces both.  C is row-major (ldc).  Result
 * float64 (CRTG_DOUBLE) or float32 (CRTG_SINGLE); OR CRTG_IN_F32 for float32
 * inputs.  k <= 2^17 (fast) / 2^16 (accurate).
 */
size_t crtg_real_workspace_size(int precision, int mode, int64_t m, int64_t n, int64_t k,
                                int num_moduli, int64_t n_block);
int crtg_gemm_real(int precision, int mode, int64_t m, int64_t n, int64_t k,
                   const void* A, int64_t lda, int a_colmajor, const void* B, int64_t ldb,
                   int b_colmajor, void* C, int64_t ldc, const crtg_consts* K, int64_t n_block,
                   void* ws, size_t ws_bytes, int32_t* mu_out, int32_t* nu_out,
                   uint64_t* diag, int sync_check, void* stream);

/* ---- multi-GPU building blocks (output-tile sharding) ---- */

/* The K2..K4 pipeline with caller-provided exponents (device int32 mu[m],
 * nu[n]), e.g. accurate-mode exponents reduced across ranks. */
int crtg_gemm_complex_exps(int precision, int64_t m, int64_t n, int64_t k,
                           const void* A, int64_t lda, const void* B, int64_t ldb,
                           void* C, int64_t ldc, const crtg_consts* K, int64_t n_block,
                           const int32_t* mu, const int32_t* nu, void* ws, size_t ws_bytes,
                           uint64_t* diag, int sync_check, void* stream);

/* Accurate mode, local half (scaling.py:229-258): bound-product maxima of the
 * local block (row_max int32[m], col_max int32[n]), normalisation exponents
 * (bar_mu int32[m], bar_nu int32[n]) and absmax (row_abs double[m],
 * col_abs double[n]).  Any output pointer may be NULL.  A rank holding
 * A[I,:] and B[:,J] all-reduces row_max (MAX) over the ranks sharing I and
 * col_max over the ranks sharing J, then calls crtg_accurate_exponents. */
int crtg_accurate_partial(int precision, int64_t m, int64_t n, int64_t k,
                          const void* A, int64_t lda, const void* B, int64_t ldb,
                          const crtg_consts* K, void* ws, size_t ws_bytes,
                          int32_t* row_max, int32_t* col_max, int32_t* bar_mu,
                          int32_t* bar_nu, double* row_abs, double* col_abs,
                          uint64_t* diag, void* stream);

/* Accurate-mode exponents from (globally reduced) bound maxima
 * (scaling.py:260-271); clamp events are added to *clamp_counter (device). */
int crtg_accurate_exponents(int64_t count, const int32_t* maxb, const double* absval,
                            const int32_t* bar, const crtg_consts* K, int32_t* out,
                            uint64_t* clamp_counter, void* stream);

/* ---- parity hooks: each reuses the production kernels of one stage ---- */

/* Scaling vectors only (fast_scaling scaling.py:198-213 / accurate_scaling
 * scaling.py:229-274).  Workspace: crtg_workspace_size(...). */
int crtg_scaling(int precision, int mode, int64_t m, int64_t n, int64_t k,
                 const void* A, int64_t lda, const void* B, int64_t ldb,
                 const crtg_consts* K, void* ws, size_t ws_bytes,
                 int32_t* mu_out, int32_t* nu_out, uint64_t* diag, void* stream);

/* quantize (scaling.py:277-293) + residue_decompose (crt.py:199-218) with
 * injected exponents.  operand 0: X is the left operand (rows x kdim, exps per
 * row); operand 1: X is the right operand (kdim x rows, exps per column).
 * out: int8 [N][3][rows][kdim] with planes (re, im, mod(re+im)) — the third is
 * the Karatsuba sum of kernel.py:101-103.  Workspace: packed tiles,
 * 3*N*round_up(rows,256)*round_up(kdim,128) bytes. */
int crtg_residues(int precision, int operand, int64_t rows, int64_t kdim,
                  const void* X, int64_t ldx, const int32_t* exps,
                  const crtg_consts* K, int8_t* out, void* ws, size_t ws_bytes,
                  uint64_t* diag, void* stream);

/* Exact int8 x int8 -> int32 on tcgen05 (replaces gemm_i8_i32,
 * kernel.py:20-35).  A: m x k row-major, B: k x n row-major, C: m x n.
 * k <= 65536, where |C| <= k * 128^2 <= 2^30 cannot overflow (CRTG_ERR_DIMENSION
 * above).  The reference accepts k <= 2^17 and raises ArithmeticError when an
 * entry leaves int32 (kernel.py:30-34); callers split larger k into two calls
 * and check the int64 sum, as paper_2512_08321_b200.gemm_i8_i32 does. */
size_t crtg_i8_workspace_size(int64_t m, int64_t n, int64_t k, int nplanes);
int crtg_gemm_i8_i32(int64_t m, int64_t n, int64_t k, const int8_t* A,
                     const int8_t* B, int32_t* C, void* ws, size_t ws_bytes,
                     void* stream);

/* Modular complex product on residue operands, Karatsuba form (replaces
 * complex_gemm_mod, kernel.py:70-120): e_re = ar br - ai bi, e_im = ar bi +
 * ai br (mod p), symmetric int8.  Inputs row-major: ar, ai m x k; br, bi k x n.
 * Workspace: crtg_i8_workspace_size(m, n, k, 3). */
int crtg_complex_gemm_mod(int64_t m, int64_t n, int64_t k, const int8_t* ar,
                          const int8_t* ai, const int8_t* br, const int8_t* bi,
                          int p, int8_t* e_re, int8_t* e_im, void* ws,
                          size_t ws_bytes, void* stream);

/* CRT accumulate + reduce + inverse scale + complex assembly (crt.py:221-258,
 * emulate.py:135-144, 234-240).  e_re / e_im: int8 [N][m][n]. */
int crtg_crt_reconstruct(int precision, int64_t m, int64_t n, const int8_t* e_re,
                         const int8_t* e_im, const int32_t* mu, const int32_t* nu,
                         const crtg_consts* K, void* C, int64_t ldc, void* stream);

/* ---- stage-level entry points (the reference's stage functions on device
 * arrays; paper_2512_08321_b200/stages.py).  `flags` is a caller-owned DEVICE
 * array of uint64 (1 or 3 entries, zeroed by the call); with sync_check the
 * call synchronizes `stream` and maps the flags to the reference's errors. ---- */

/* log2_upper (scaling.py:62-82): float32 upper bound on log2 x, x > 0 finite
 * (CRTG_ERR_DOMAIN otherwise). */
int crtg_log2_upper(const double* x, int64_t n, float* out, uint64_t* flags, int sync_check,
                    void* stream);

/* quantize (scaling.py:277-293): out = trunc(ldexp(x, e)), e per row (axis 0)
 * or per column (axis 1); |out| >= 2^90 -> CRTG_ERR_DOMAIN.  Row-major. */
int crtg_quantize(const double* x, int64_t rows, int64_t cols, int64_t ldx, const int64_t* exps,
                  int axis, double* out, int64_t ldo, uint64_t* flags, int sync_check,
                  void* stream);

/* symmetric residues (residue_decompose crt.py:199-218 / symmetric_mod_int
 * crt.py:136-151) of `count` integer-valued entries for each of the nmod host
 * moduli: out int8 [nmod][count].  kind 0: float64 (finite and < 2^90, else
 * CRTG_ERR_DOMAIN), 1: int64, 2: int32; kind | 8 = residue_decompose's checks
 * (float64 integer-valued, int64 < 2^61).  flags: 3 entries. */
int crtg_symmetric_mod(int kind, const void* x, int64_t count, const int32_t* moduli, int nmod,
                       int8_t* out, uint64_t* flags, int sync_check, void* stream);

/* crt_accumulate (crt.py:221-243): e int8 [N][count] -> s1 = sum coeff_hi e,
 * s2 = sum coeff_lo e (ascending l, no FMA); single != 0 writes s1 + s2 to s1. */
int crtg_crt_accumulate(const int8_t* e, int64_t count, const crtg_consts* K, int single,
                        double* s1, double* s2, void* stream);

/* symmetric_mod_wide (crt.py:154-184): (s_hi + s_lo) mod P into (-P/2, P/2],
 * P = p_hi + p_lo; s_lo may be NULL; use_dd selects the double-double path
 * (Dekker two_prod exactly as ddarith.py). */
int crtg_symmetric_mod_wide(const double* s_hi, const double* s_lo, int64_t count, double p_hi,
                            double p_lo, int use_dd, double* out, void* stream);

/* inverse_scale (emulate.py:135-144): out = ldexp(c, int32(-mu_i - nu_j)) as
 * float64 or (out_f32) float32.  Row-major. */
int crtg_inverse_scale(const double* c, int64_t rows, int64_t cols, int64_t ldc, const int64_t* mu,
                       const int64_t* nu, int out_f32, void* out, int64_t ldo, void* stream);

/* ---- accuracy harness ---- */

/* Double-double reference product, bit-identical to the reference's
 * reference_gemm_dd (oracle.py:60-128): hi + lo per entry (~106 bits), terms of
 * the stacked real forms in ascending order.  is_complex: A, B, hi, lo are
 * complex128 (interleaved), else float64.  Row-major, strides in elements. */
int crtg_dd_gemm(int is_complex, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                 const void* B, int64_t ldb, void* hi, void* lo, int64_t ldo, void* stream);

/* max_relative_error (oracle.py:131-169) of `approx` (complex128/complex64 or
 * float64/float32 with approx_single) against (hi, lo): *max_bits receives the
 * IEEE bits of the largest componentwise relative error (atomic max; zero it
 * first), *zero_count the number of components with a zero reference. */
int crtg_max_relative_error(int is_complex, int64_t m, int64_t n, const void* approx,
                            int approx_single, int64_t ld_approx, const void* hi, const void* lo,
                            int64_t ldo, uint64_t* max_bits, uint64_t* zero_count, void* stream);

/* ---- instrumentation (bench.py) ---- */
/* total kernels this library has launched in the process */
uint64_t crtg_launch_count(void);
/* stage ids for the per-stage device timers */
enum crtg_stage {
  CRTG_STAGE_SCALING = 0, /* K1 (+ bound GEMM in accurate mode) */
  CRTG_STAGE_RESIDUE_A = 1,
  CRTG_STAGE_RESIDUE_B = 2,
  CRTG_STAGE_GEMM = 3, /* K3 Karatsuba tcgen05 GEMM (all moduli of a block) */
  CRTG_STAGE_CRT = 4,
  CRTG_STAGE_COUNT = 5
};
/* enable (1) / disable (0) CUDA-event timing of every stage launch, recorded
 * on the launching stream */
int crtg_profile_enable(int on);
/* synchronize the recorded events and return, per stage, the summed device
 * milliseconds (ms[CRTG_STAGE_COUNT]) and launch counts; clears the record */
int crtg_profile_read(double* ms, uint64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* CRTG_H */
