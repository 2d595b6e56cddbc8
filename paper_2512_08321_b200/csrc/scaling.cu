// scaling.cu — K1: power-of-two scaling exponents (fast and accurate mode).
//
// Bit-exact restatement on the GPU of reference scaling.py:
//   log2_upper            scaling.py:62-82   (Horner, separate roundings, f32 round-up)
//   _fast_exponents       scaling.py:174-195 (absmax, floor_log2, sum of squares)
//   accurate exponents    scaling.py:260-271
// Bit-exactness rules: every FP op is an explicit __d*_rn intrinsic (no FMA
// contraction; the file is also compiled with -fmad=false), and the sums of
// squares follow numpy's reduction order exactly — np.sum(axis=1) over a
// contiguous row is numpy's pairwise sum (8-accumulator leaves <= 128 elements,
// recursive halving at n/2 rounded down to a multiple of 8, initial value 0);
// np.sum(axis=0) is a sequential column sweep.
#include "common.cuh"
#include "kernels.cuh"

namespace crtg {

namespace {

__constant__ double kLog2Poly[17] = {
    2.2775402178481487e-14, 1.4426950408757782,   -0.7213475191685141,
    0.4808982977587932,     -0.3606727542079527,  0.28852642308593507,
    -0.2403442897663445,    0.2054837442266186,   -0.17769294959119178,
    0.15174988229827802,    -0.1229870201590372,  0.0895501501300455,
    -0.05496910933753177,   0.026522983843890614, -0.009240638947705725,
    0.0020404147534928345,  -0.00021265579458876327,
};

// deterministic float32 upper bound on log2(x), x > 0 finite (scaling.py:62-82)
__device__ float log2_upper(double x) {
  int ex;
  const double fr = frexp(x, &ex);
  const double t = __dsub_rn(__dmul_rn(2.0, fr), 1.0);
  double acc = kLog2Poly[16];
#pragma unroll
  for (int i = 15; i >= 0; --i) acc = __dadd_rn(__dmul_rn(acc, t), kLog2Poly[i]);
  const double y = __dadd_rn(__dadd_rn(double(ex - 1), acc), 0x1p-21);
  return __double2float_ru(y);
}

__device__ int32_t clamp_exp(int64_t e, unsigned long long* counter) {
  if (e > 1023 || e < -1023) {
    atomicAdd(counter, 1ull);
    return e > 1023 ? 1023 : -1023;
  }
  return int32_t(e);
}

// fast-mode exponent from the row/column absmax and sum of squares
// (scaling.py:186-195)
__device__ int32_t fast_exponent(double absmax, double sumsq, float p_fast, float delta,
                                 unsigned long long* counter) {
  if (absmax == 0.0) return 1023;  // zero row/column: upper clamp, not counted
  const int fl = ilogb(absmax);
  const double lb = double(log2_upper(sumsq));
  const double inner = fmax(1.0, __dmul_rn(double(delta), lb));
  const float head = __double2float_rd(__dsub_rn(double(p_fast), inner));
  const int64_t e = int64_t(floorf(head)) - fl;
  return clamp_exp(e, counter);
}

// x * 2^-fl for the normalised sum of squares; direct multiply when 2^-fl is
// representable (np.ldexp is then one correctly rounded multiply)
struct Pow2 {
  double s;
  int e;
  bool direct;
};
__device__ __forceinline__ Pow2 make_pow2(int e) {
  Pow2 p;
  p.e = e;
  p.direct = (e >= -1074 && e <= 1023);
  p.s = p.direct ? (e >= -1022 ? __longlong_as_double(int64_t(e + 1023) << 52)
                               : __longlong_as_double(int64_t(1) << (e + 1074)))
                 : 0.0;
  return p;
}
__device__ __forceinline__ double apply(const Pow2& p, double x) {
  return p.direct ? __dmul_rn(x, p.s) : ldexp(x, p.e);
}
__device__ __forceinline__ double sq(const Pow2& p, double x) {
  const double y = apply(p, x);
  return __dmul_rn(y, y);
}

// element h of a row / column: complex (interleaved pairs) or real (im = 0)
template <typename T, bool REAL>
__device__ __forceinline__ void load_c(const T* base, int64_t h, double& re, double& im) {
  if constexpr (REAL) {
    re = double(base[h]);
    im = 0.0;
  } else if constexpr (sizeof(T) == 8) {
    const double2 v = reinterpret_cast<const double2*>(base)[h];
    re = v.x;
    im = v.y;
  } else {
    const float2 v = reinterpret_cast<const float2*>(base)[h];
    re = double(v.x);
    im = double(v.y);
  }
}

__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  for (int i = 0; i < int(blockDim.x >> 5); ++i) r = fmax(r, red[i]);
  __syncthreads();
  return r;
}

// One CTA per row of A.  Pass 1: absmax over both parts; pass 2 (fast mode): the
// pairwise sums of squares of re and im (numpy order), then the exponent.
template <typename T, bool REAL>
__global__ void __launch_bounds__(256) k_row_stats(const T* __restrict__ A, int64_t lda, int k,
                                                   PwTree tree, float p_fast, float delta,
                                                   int fast, int32_t* __restrict__ mu,
                                                   double* __restrict__ rowabs,
                                                   unsigned long long* __restrict__ diag) {
  extern __shared__ double vals[];  // [2][nleaves + nnodes]
  __shared__ double red[8];
  const int64_t i = blockIdx.x;
  const T* row = A + (REAL ? 1 : 2) * i * lda;

  double mx = 0.0;
  int bad = 0;
  for (int h = threadIdx.x; h < k; h += blockDim.x) {
    double re, im;
    load_c<T, REAL>(row, h, re, im);
    bad |= !(isfinite(re) && isfinite(im));
    mx = fmax(mx, fmax(fabs(re), fabs(im)));
  }
  bad = __syncthreads_or(bad);
  const double absmax = block_max(mx, red);
  if (threadIdx.x == 0) {
    rowabs[i] = absmax;
    if (bad) atomicAdd(diag + CRTG_DIAG_NONFINITE_A, 1ull);
  }
  if (!fast) return;
  const bool zero = absmax == 0.0;
  const Pow2 sc = make_pow2(zero ? 0 : -ilogb(absmax));

  const int nv = tree.nleaves + tree.nnodes;
  const int grp = threadIdx.x >> 3, j = threadIdx.x & 7;
  for (int base = 0; base < tree.nleaves; base += int(blockDim.x >> 3)) {
    const int lf = base + grp;
    const bool active = lf < tree.nleaves;
    const int2 L = active ? tree.leaves[lf] : make_int2(0, 0);
    const int start = L.x, len = L.y;
    double sr = 0.0, si = 0.0;
    if (len >= 8) {
      const int full = len - (len & 7);
      double re, im;
      load_c<T, REAL>(row, start + j, re, im);
      sr = sq(sc, re);
      si = sq(sc, im);
      for (int t = 8 + j; t < full; t += 8) {
        load_c<T, REAL>(row, start + t, re, im);
        sr = __dadd_rn(sr, sq(sc, re));
        si = __dadd_rn(si, sq(sc, im));
      }
    }
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) inside each 8-lane group
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      sr = __dadd_rn(sr, __shfl_xor_sync(0xffffffffu, sr, o));
      si = __dadd_rn(si, __shfl_xor_sync(0xffffffffu, si, o));
    }
    if (active && j == 0) {
      // sequential tail (and whole leaf when len < 8: res = 0; res += a[i])
      for (int t = (len >= 8 ? len - (len & 7) : 0); t < len; ++t) {
        double re, im;
        load_c<T, REAL>(row, start + t, re, im);
        sr = __dadd_rn(sr, sq(sc, re));
        si = __dadd_rn(si, sq(sc, im));
      }
      vals[lf] = sr;
      vals[nv + lf] = si;
    }
  }
  __syncthreads();
  for (int lv = 0; lv < tree.nlevels; ++lv) {
    for (int idx = tree.level_start[lv] + threadIdx.x; idx < tree.level_start[lv + 1];
         idx += blockDim.x) {
      const int2 c = tree.nodes[idx];
      vals[tree.nleaves + idx] = __dadd_rn(vals[c.x], vals[c.y]);
      vals[nv + tree.nleaves + idx] = __dadd_rn(vals[nv + c.x], vals[nv + c.y]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int root = nv - 1;
    double sumsq = __dadd_rn(__dadd_rn(0.0, vals[root]), vals[nv + root]);
    if (zero) sumsq = 1.0;
    mu[i] = fast_exponent(absmax, sumsq, p_fast, delta, diag + CRTG_DIAG_CLAMPED_MU);
  }
}

// Column absmax of B (k x n row-major complex): one thread per column, rows split
// in chunks; order-free max merged with an atomic max on the bit pattern.
template <typename T, bool REAL>
__global__ void __launch_bounds__(128) k_col_absmax(const T* __restrict__ B, int64_t ldb, int k,
                                                    int n, int rows_per_chunk,
                                                    double* __restrict__ colabs,
                                                    unsigned long long* __restrict__ diag) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int h0 = blockIdx.y * rows_per_chunk;
  const int h1 = min(k, h0 + rows_per_chunk);
  double mx = 0.0;
  int bad = 0;
  if (j < n) {
#pragma unroll 8
    for (int h = h0; h < h1; ++h) {
      double re, im;
      load_c<T, REAL>(B + (REAL ? 1 : 2) * int64_t(h) * ldb, j, re, im);
      bad |= !(isfinite(re) && isfinite(im));
      mx = fmax(mx, fmax(fabs(re), fabs(im)));
    }
    atomicMax(reinterpret_cast<unsigned long long*>(colabs) + j,
              (unsigned long long)__double_as_longlong(mx));
  }
  bad = __syncthreads_or(bad);
  if (bad && threadIdx.x == 0) atomicAdd(diag + CRTG_DIAG_NONFINITE_B, 1ull);
}

// Column sums of squares in numpy's axis-0 order: for each column and part a
// sequential chain over k.  Thread t -> (column t/2, part t%2); a warp reads 16
// columns x 16 bytes contiguously.
template <typename T, bool REAL>
__global__ void __launch_bounds__(128) k_col_sumsq(const T* __restrict__ B, int64_t ldb, int k,
                                                   int n, const double* __restrict__ colabs,
                                                   double* __restrict__ colsq) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int j = int(t >> 1), part = int(t & 1);
  if (j >= n) return;
  if (REAL && part == 1) {  // no imaginary part: its sum of squares is 0
    colsq[int64_t(n) + j] = 0.0;
    return;
  }
  const double mx = colabs[j];
  const Pow2 sc = make_pow2(mx == 0.0 ? 0 : -ilogb(mx));
  const T* p = B + (REAL ? 1 : 2) * int64_t(j) + part;
  const int64_t stride = (REAL ? 1 : 2) * ldb;
  double s = 0.0;
  constexpr int U = 16;
  int h = 0;
  for (; h + U <= k; h += U) {
    double x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = double(p[(h + u) * stride]);
#pragma unroll
    for (int u = 0; u < U; ++u) s = __dadd_rn(s, sq(sc, x[u]));
  }
  for (; h < k; ++h) s = __dadd_rn(s, sq(sc, double(p[h * stride])));
  colsq[int64_t(part) * n + j] = s;
}

__global__ void k_col_finalize(int n, const double* __restrict__ colabs,
                               const double* __restrict__ colsq, float p_fast, float delta,
                               int32_t* __restrict__ nu, unsigned long long* __restrict__ diag) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double mx = colabs[j];
  double sumsq = __dadd_rn(__dadd_rn(0.0, colsq[j]), colsq[n + j]);
  if (mx == 0.0) sumsq = 1.0;
  nu[j] = fast_exponent(mx, sumsq, p_fast, delta, diag + CRTG_DIAG_CLAMPED_NU);
}

__global__ void k_bar(const double* __restrict__ absval, int64_t count, int32_t* __restrict__ bar) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double v = absval[i];
  bar[i] = v == 0.0 ? 0 : 5 - ilogb(v);
}

// accurate-mode exponents (scaling.py:260-271)
__global__ void k_accurate_exps(const int32_t* __restrict__ maxb, const double* __restrict__ absval,
                                const int32_t* __restrict__ bar, int64_t count, float p_accu,
                                float delta, int32_t* __restrict__ out,
                                unsigned long long* __restrict__ counter) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double mv = double(maxb[i]);
  const bool dead = (mv <= 0.0) || (absval[i] == 0.0);
  if (dead) {
    out[i] = 1023;
    return;
  }
  const double lb = double(log2_upper(mv));
  const float head = __double2float_rd(__dsub_rn(double(p_accu), __dmul_rn(double(delta), lb)));
  const int64_t e = int64_t(bar[i]) + int64_t(floorf(head));
  out[i] = clamp_exp(e, counter);
}

}  // namespace

#define CRTG_ELEM_DISPATCH(elem, ...)                                                    \
  switch (elem) {                                                                       \
    case E_C128: { using T = double; constexpr bool R = false; __VA_ARGS__; } break;     \
    case E_C64:  { using T = float;  constexpr bool R = false; __VA_ARGS__; } break;     \
    case E_F64:  { using T = double; constexpr bool R = true;  __VA_ARGS__; } break;     \
    default:     { using T = float;  constexpr bool R = true;  __VA_ARGS__; } break;     \
  }

int launch_row_stats(int elem, bool fast, const void* A, int64_t lda, int64_t m, int64_t k,
                     const PwTree& tree, float p_fast, float delta, int32_t* mu, double* rowabs,
                     unsigned long long* diag, cudaStream_t s) {
  if (m <= 0) return 0;
  const size_t smem = fast ? size_t(2) * (tree.nleaves + tree.nnodes) * sizeof(double) : 0;
  CRTG_ELEM_DISPATCH(elem, {
    cudaFuncSetAttribute(k_row_stats<T, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem > 48 * 1024 ? smem : 48 * 1024));
    k_row_stats<T, R><<<unsigned(m), 256, smem, s>>>(static_cast<const T*>(A), lda, int(k), tree,
                                                     p_fast, delta, fast, mu, rowabs, diag);
  })
  return int(cudaGetLastError());
}

int launch_col_absmax(int elem, const void* B, int64_t ldb, int64_t k, int64_t n,
                      double* colabs, unsigned long long* diag, cudaStream_t s) {
  if (n <= 0) return 0;
  const int rows_per_chunk = 1024;
  dim3 grid(unsigned((n + 127) / 128), unsigned((k + rows_per_chunk - 1) / rows_per_chunk));
  CRTG_ELEM_DISPATCH(elem, {
    k_col_absmax<T, R><<<grid, 128, 0, s>>>(static_cast<const T*>(B), ldb, int(k), int(n),
                                            rows_per_chunk, colabs, diag);
  })
  return int(cudaGetLastError());
}

int launch_col_fast(int elem, const void* B, int64_t ldb, int64_t k, int64_t n,
                    const double* colabs, double* colsq, float p_fast, float delta, int32_t* nu,
                    unsigned long long* diag, cudaStream_t s) {
  if (n <= 0) return 0;
  const unsigned grid = unsigned((2 * n + 127) / 128);
  CRTG_ELEM_DISPATCH(elem, {
    k_col_sumsq<T, R><<<grid, 128, 0, s>>>(static_cast<const T*>(B), ldb, int(k), int(n), colabs,
                                           colsq);
  })
  k_col_finalize<<<unsigned((n + 127) / 128), 128, 0, s>>>(int(n), colabs, colsq, p_fast, delta,
                                                            nu, diag);
  return int(cudaGetLastError());
}

int launch_bar(const double* absval, int64_t count, int32_t* bar, cudaStream_t s) {
  if (count <= 0) return 0;
  k_bar<<<unsigned((count + 255) / 256), 256, 0, s>>>(absval, count, bar);
  return int(cudaGetLastError());
}

int launch_accurate_exps(const int32_t* maxb, const double* absval, const int32_t* bar,
                         int64_t count, float p_accu, float delta, int32_t* out,
                         unsigned long long* clamp_counter, cudaStream_t s) {
  if (count <= 0) return 0;
  k_accurate_exps<<<unsigned((count + 255) / 256), 256, 0, s>>>(maxb, absval, bar, count, p_accu,
                                                                 delta, out, clamp_counter);
  return int(cudaGetLastError());
}

}  // namespace crtg
