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
#include <atomic>

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

__device__ __forceinline__ double block_min(double v, double* red) {
  for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double r = INFINITY;
  for (int i = 0; i < int(blockDim.x >> 5); ++i) r = fmin(r, red[i]);
  __syncthreads();
  return r;
}

// Single-pass sums of squares.  The reference squares x * 2^-fl (fl = floor
// log2 absmax), which needs absmax first — a second read of the operand.  But a
// power-of-two scale commutes with every rounding while all values stay
// normal, so sum((x 2^-fl)^2) == 2^-2fl * sum(x^2) bit for bit when
//   every nonzero x^2 and (x 2^-fl)^2 is >= 2^-1022   (min |x| != 0 >= 2^-511,
//                                                     and >= 2^(fl-511))
//   no partial sum overflows                          (absmax <= 2^500, k <= 2^18)
// (nonzero partial sums are >= the smallest nonzero square).  Kernels sum the
// unscaled squares in the reference's order and scale once; when the check
// fails they fall back to the two-pass form.
__device__ __forceinline__ bool unscaled_ok(double absmax, double minnz) {
  if (absmax == 0.0) return true;
  if (!(absmax <= 0x1p500)) return false;  // also rejects inf / nan
  if (minnz == INFINITY) return true;       // no nonzero values besides absmax's
  return minnz >= 0x1p-511 && ilogb(minnz) - ilogb(absmax) >= -511;
}

// 2^-2fl * s as two exact multiplies (2^-2fl itself may not be representable)
__device__ __forceinline__ double unscale_sq(double s, const Pow2& sc) {
  return apply(sc, apply(sc, s));
}

// One CTA per row of A.  Fast mode: ONE pass over the row computes absmax, the
// smallest nonzero |x|, finiteness and the numpy-pairwise leaf sums of the
// UNSCALED squares of re and im; the tree combine and a 2^-2fl scale then give
// the reference's sums (see unscaled_ok), else a second, scaled pass runs.
// Accurate mode: absmax only.
template <typename T, bool REAL>
__device__ void row_leaf_sums(const T* row, const PwTree& tree, double* vals, int nv,
                              const Pow2* sc, double& mx, double& mn, int& bad) {
  const int grp = threadIdx.x >> 3, j = threadIdx.x & 7;
  auto term = [&](double x) -> double {
    if (sc == nullptr) {
      const double ax = fabs(x);
      bad |= !isfinite(x);
      mx = fmax(mx, ax);
      if (ax != 0.0) mn = fmin(mn, ax);
      return __dmul_rn(x, x);
    }
    return sq(*sc, x);
  };
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
      sr = term(re);
      si = term(im);
      for (int t = 8 + j; t < full; t += 8) {
        load_c<T, REAL>(row, start + t, re, im);
        sr = __dadd_rn(sr, term(re));
        si = __dadd_rn(si, term(im));
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
        sr = __dadd_rn(sr, term(re));
        si = __dadd_rn(si, term(im));
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
}

template <typename T, bool REAL>
__global__ void __launch_bounds__(256) k_row_stats(const T* __restrict__ A, int64_t lda, int k,
                                                   PwTree tree, float p_fast, float delta,
                                                   int fast, int32_t* __restrict__ mu,
                                                   double* __restrict__ rowabs,
                                                   unsigned long long* __restrict__ diag) {
  pdl_begin();
  extern __shared__ double vals[];  // [2][nleaves + nnodes]
  __shared__ double red[8];
  const int64_t i = blockIdx.x;
  const T* row = A + (REAL ? 1 : 2) * i * lda;

  double mx = 0.0, mn = INFINITY;
  int bad = 0;
  const int nv = tree.nleaves + tree.nnodes;
  if (!fast) {
    for (int h = threadIdx.x; h < k; h += blockDim.x) {
      double re, im;
      load_c<T, REAL>(row, h, re, im);
      bad |= !(isfinite(re) && isfinite(im));
      mx = fmax(mx, fmax(fabs(re), fabs(im)));
    }
  } else {
    row_leaf_sums<T, REAL>(row, tree, vals, nv, nullptr, mx, mn, bad);
  }
  bad = __syncthreads_or(bad);
  const double absmax = block_max(mx, red);
  if (threadIdx.x == 0) {
    rowabs[i] = absmax;
    if (bad) atomicAdd(diag + CRTG_DIAG_NONFINITE_A, 1ull);
  }
  if (!fast) return;
  const double minnz = block_min(mn, red);
  const bool zero = absmax == 0.0;
  const Pow2 sc = make_pow2(zero ? 0 : -ilogb(absmax));
  const int root = nv - 1;
  double sr, si;
  if (unscaled_ok(absmax, minnz)) {
    sr = unscale_sq(vals[root], sc);
    si = unscale_sq(vals[nv + root], sc);
  } else {
    __syncthreads();  // everyone has read the unscaled root
    row_leaf_sums<T, REAL>(row, tree, vals, nv, &sc, mx, mn, bad);
    sr = vals[root];
    si = vals[nv + root];
  }
  if (threadIdx.x == 0) {
    double sumsq = __dadd_rn(__dadd_rn(0.0, sr), si);
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
  pdl_begin();
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
  pdl_begin();
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

// ---------------------------------------------------------------------------
// Fast-mode column statistics in ONE pass (k_col_stats): per column j of B (and
// per part) the sequential numpy axis-0 chain of UNSCALED squares, the absmax,
// the smallest nonzero |x| and finiteness; then the exponent in-kernel when
// unscaled_ok, else the chain lanes re-run that column's chains scaled from B
// (the reference's two-pass form; no second launch).  Memory-level parallelism comes from a cp.async ring: a CTA
// owns 32 components (16 complex columns x (re, im), or 32 real columns) = one
// 256-byte (128 for float) segment per row of B, and keeps kColS stages of
// kColR rows in flight while warp 0 runs the 32 chains out of shared memory —
// the per-column chains are inherently sequential, so with few columns (n =
// 4096 at k = 65536) a register-only loop cannot cover the DRAM latency.
// ---------------------------------------------------------------------------
// rows per stage x stages of the cp.async ring (64 x 4 = 64 KiB per CTA for
// complex128: 3 CTAs per SM; CRTG_COL_R=32 halves it)
#ifndef CRTG_COL_R
#define CRTG_COL_R 64
#endif
constexpr int kColR = CRTG_COL_R;  // rows per stage
constexpr int kColS = 4;           // stages

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Unsigned key of |x| for the order-free column statistics: float -> the bits of
// |x|; double -> the high word of |x| with bit 0 also set when the low word is
// nonzero.  Zero <-> key 0, inf / nan <-> key >= the exponent mask, and for
// every x with a nonzero key, the double whose high word is the key has x's
// ilogb and the same comparisons against 2^500 / 2^-511 as |x| (so absmax and
// the smallest nonzero |x| derive from max / min keys), except key 1: a nonzero
// |x| < 2^-1042, whose exponent lies in the low word (unscaled_ok rejects it).
template <typename T>
__device__ __forceinline__ uint32_t abs_key(const T* p) {
  if constexpr (sizeof(T) == 8) {
    const uint2 w = *reinterpret_cast<const uint2*>(p);
    return (w.y & 0x7FFFFFFFu) | min(w.x, 1u);
  } else {
    return __float_as_uint(*p) & 0x7FFFFFFFu;
  }
}
template <typename T>
__device__ __forceinline__ double key_value(uint32_t key) {
  if constexpr (sizeof(T) == 8) return __hiloint2double(int(key), 0);
  else return double(__uint_as_float(key));
}

template <typename T, bool REAL>
__global__ void __launch_bounds__(128) k_col_stats(const T* __restrict__ B, int64_t ldb, int k,
                                                   int n, float p_fast, float delta,
                                                   int32_t* __restrict__ nu,
                                                   double* __restrict__ colabs,
                                                   unsigned long long* __restrict__ diag) {
  pdl_begin();
  constexpr int kParts = REAL ? 1 : 2;
  constexpr int kCols = 32 / kParts;            // columns per CTA
  constexpr int kSeg = 32 * int(sizeof(T));     // bytes per row segment
  constexpr int kChunks = kSeg / 16;            // 16-byte chunks per row segment
  extern __shared__ __align__(16) uint8_t ring[];  // [kColS][kColR][kSeg]
  const int j0 = blockIdx.x * kCols;
  const int64_t row_bytes = int64_t(kParts) * ldb * int64_t(sizeof(T));
  const char* base = reinterpret_cast<const char*>(B) + int64_t(j0) * kParts * int64_t(sizeof(T));
  const int valid = min(kCols, n - j0) * kParts * int(sizeof(T));  // bytes of a row segment in range
  const int nst = (k + kColR - 1) / kColR;
  const uint32_t ring_u32 = smem_u32(ring);

  // full stages of full segments (every stage but the last, every CTA but the
  // last column strip): thread t always copies chunk t % kChunks of rows
  // t / kChunks + i * (128 / kChunks), so the addresses advance by constants
  // (~3 instructions per 16-byte copy instead of ~28 for the general form)
  constexpr int kRowStep = 128 / kChunks;  // rows between one thread's copies
  static_assert(128 % kChunks == 0 && kColR % kRowStep == 0, "copy pattern");
  const bool full_seg = valid == kSeg && blockDim.x == 128;
  const int my_q = threadIdx.x % kChunks, my_r = threadIdx.x / kChunks;
  const char* my_src = base + int64_t(my_r) * row_bytes + 16 * my_q;
  const uint32_t my_dst = ring_u32 + my_r * kSeg + 16 * my_q;
  auto issue = [&](int st) {
    if (st < nst && full_seg && (st + 1) * kColR <= k) {
      const char* src = my_src + int64_t(st) * kColR * row_bytes;
      const uint32_t dst = my_dst + (st % kColS) * (kColR * kSeg);
#pragma unroll
      for (int i = 0; i < kColR / kRowStep; ++i)
        cp_async16(dst + i * kRowStep * kSeg, src + int64_t(i) * kRowStep * row_bytes, 16);
    } else if (st < nst) {
      const uint32_t dst0 = ring_u32 + (st % kColS) * (kColR * kSeg);
      for (int c = threadIdx.x; c < kColR * kChunks; c += blockDim.x) {
        const int r = c / kChunks, q = c % kChunks;
        const int h = st * kColR + r;
        const int bytes = h < k ? max(0, min(16, valid - 16 * q)) : 0;
        const char* src = bytes ? base + h * row_bytes + 16 * q : base;
        cp_async16(dst0 + r * kSeg + 16 * q, src, bytes);
      }
    }
    cp_async_commit();  // possibly empty: keeps the group count uniform
  };

#pragma unroll
  for (int st = 0; st < kColS - 1; ++st) issue(st);
  // warp 0 runs the 32 order-dependent sum chains (numpy's sequential axis-0
  // order) and nothing else, so each row costs it one load, one DMUL and the
  // DADD on the chain; warps 1-3 take the order-free statistics (absmax,
  // smallest nonzero, finiteness) of the same stage rows in parallel
  // order-free statistics as unsigned integer keys of |x| (see abs_key):
  // max key -> absmax exponent / finiteness, min of (key - 1) -> smallest nonzero
  __shared__ uint32_t red_mx[3][32], red_mn[3][32];
  double sum = 0.0;
  uint32_t kmx = 0u, kmn = 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  for (int st = 0; st < nst; ++st) {
    issue(st + kColS - 1);
    cp_async_wait<kColS - 1>();
    __syncthreads();
    const T* seg = reinterpret_cast<const T*>(ring + (st % kColS) * (kColR * kSeg));
    const int nr = min(kColR, k - st * kColR);
    if (warp == 0) {
      if (nr == kColR) {
#pragma unroll 16
        for (int r = 0; r < kColR; ++r) {
          const double x = double(seg[r * 32 + lane]);
          sum = __dadd_rn(sum, __dmul_rn(x, x));
        }
      } else {
        for (int r = 0; r < nr; ++r) {
          const double x = double(seg[r * 32 + lane]);
          sum = __dadd_rn(sum, __dmul_rn(x, x));
        }
      }
    } else {
#pragma unroll 4
      for (int r = warp - 1; r < nr; r += 3) {
        const uint32_t key = abs_key(seg + r * 32 + lane);
        kmx = max(kmx, key);
        kmn = min(kmn, key - 1u);  // 0 (zero) wraps to the largest key
      }
    }
    __syncthreads();
  }
  if (warp > 0) {
    red_mx[warp - 1][lane] = kmx;
    red_mn[warp - 1][lane] = kmn;
  }
  __syncthreads();
  if (warp > 0) return;
  kmx = max(max(red_mx[0][lane], red_mx[1][lane]), red_mx[2][lane]);
  kmn = min(min(red_mn[0][lane], red_mn[1][lane]), red_mn[2][lane]);
  const bool bad = kmx >= (sizeof(T) == 8 ? 0x7FF00000u : 0x7F800000u);  // inf / nan
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicAdd(diag + CRTG_DIAG_NONFINITE_B, 1ull);
  double other = 0.0;
  if (!REAL) {  // lanes (2c, 2c+1) = (re, im) of column c
    kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, 1));
    kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, 1));
    other = __shfl_xor_sync(0xffffffffu, sum, 1);
  }
  const int j = j0 + (REAL ? lane : lane >> 1);
  const bool live = j < n;  // both lanes of a column pair agree
  double mx = key_value<T>(kmx);
  const double mn = kmn == 0xFFFFFFFFu ? INFINITY : key_value<T>(kmn + 1u);
  // key 1 (double): every nonzero |x| < 2^-1042, its exponent is not in the key
  const bool inexact = sizeof(T) == 8 && kmx == 1u;
  const bool pend = live && (inexact || !unscaled_ok(mx, mn));
  double s_re = sum, s_im = other;
  if (__any_sync(0xffffffffu, pend)) {
    // rare: the reference's two-pass form for this column, right here (each lane
    // its own part: the exact absmax when the key could not carry it, then the
    // sequential chain of scaled squares re-read from B)
    const T* p = B + int64_t(j) * kParts + (REAL ? 0 : (lane & 1));
    const int64_t stride = int64_t(kParts) * ldb;
    if (pend && inexact) {
      double a = 0.0;
      for (int h = 0; h < k; ++h) a = fmax(a, fabs(double(p[h * stride])));
      mx = a;
    }
    if (!REAL) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    double sc_sum = 0.0;
    if (pend) {
      const Pow2 sc = make_pow2(mx == 0.0 ? 0 : -ilogb(mx));
      for (int h = 0; h < k; ++h) sc_sum = __dadd_rn(sc_sum, sq(sc, double(p[h * stride])));
    }
    const double sc_other = REAL ? 0.0 : __shfl_xor_sync(0xffffffffu, sc_sum, 1);
    if (pend) {
      s_re = sc_sum;
      s_im = sc_other;
    }
  }
  if (!live || (!REAL && (lane & 1))) return;
  colabs[j] = mx;
  const bool zero = mx == 0.0;
  double sumsq;
  if (pend) {
    sumsq = __dadd_rn(__dadd_rn(0.0, s_re), s_im);  // already scaled
  } else {
    const Pow2 sc = make_pow2(zero ? 0 : -ilogb(mx));
    sumsq = __dadd_rn(__dadd_rn(0.0, unscale_sq(s_re, sc)), unscale_sq(s_im, sc));
  }
  if (zero) sumsq = 1.0;
  nu[j] = fast_exponent(mx, sumsq, p_fast, delta, diag + CRTG_DIAG_CLAMPED_NU);
}

__global__ void k_col_finalize(int n, const double* __restrict__ colabs,
                               const double* __restrict__ colsq, float p_fast, float delta,
                               int32_t* __restrict__ nu, unsigned long long* __restrict__ diag) {
  pdl_begin();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double mx = colabs[j];
  double sumsq = __dadd_rn(__dadd_rn(0.0, colsq[j]), colsq[n + j]);
  if (mx == 0.0) sumsq = 1.0;
  nu[j] = fast_exponent(mx, sumsq, p_fast, delta, diag + CRTG_DIAG_CLAMPED_NU);
}

__global__ void k_bar(const double* __restrict__ absval, int64_t count, int32_t* __restrict__ bar) {
  pdl_begin();
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
  pdl_begin();
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

#define CRTG_TRY_L(expr)          \
  do {                            \
    const int _e = int(expr);     \
    if (_e) return _e;            \
  } while (0)

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
    launch_k(k_row_stats<T, R>, unsigned(m), 256, smem, s, static_cast<const T*>(A), lda, int(k), tree,
                                                     p_fast, delta, fast, mu, rowabs, diag);
  })
  return launched(1);
}

int launch_col_absmax(int elem, const void* B, int64_t ldb, int64_t k, int64_t n,
                      double* colabs, unsigned long long* diag, cudaStream_t s) {
  if (n <= 0) return 0;
  // enough row chunks for ~4 CTAs per SM (a narrow B at k = 1024 otherwise ran
  // 8 CTAs of 1024-long chains: 216 us at 1024^3); atomicMax is order-free
  const int64_t xb = (n + 127) / 128;
  const int64_t chunks = std::max<int64_t>(1, (4 * 148 + xb - 1) / xb);
  const int rows_per_chunk =
      int(std::min<int64_t>(1024, std::max<int64_t>(16, round_up((k + chunks - 1) / chunks, 16))));
  dim3 grid(unsigned(xb), unsigned((k + rows_per_chunk - 1) / rows_per_chunk));
  CRTG_ELEM_DISPATCH(elem, {
    launch_k(k_col_absmax<T, R>, grid, 128, 0, s, static_cast<const T*>(B), ldb, int(k), int(n),
                                            rows_per_chunk, colabs, diag);
  })
  return launched(1);
}

// Fast-mode column statistics: writes colabs and nu (colsq is scratch for the
// two-pass path, used when B's rows are not 16-byte aligned for cp.async)
int launch_col_fast(int elem, const void* B, int64_t ldb, int64_t k, int64_t n, double* colabs,
                    double* colsq, float p_fast, float delta, int32_t* nu,
                    unsigned long long* diag, cudaStream_t s) {
  if (n <= 0) return 0;
  const int esz = (elem == E_C128) ? 16 : (elem == E_C64 || elem == E_F64) ? 8 : 4;
  const bool aligned = (reinterpret_cast<uintptr_t>(B) % 16 == 0) && ((ldb * esz) % 16 == 0);
  if (!aligned) {
    CRTG_TRY_L(cudaMemsetAsync(colabs, 0, size_t(n) * sizeof(double), s));
    CRTG_TRY_L(launch_col_absmax(elem, B, ldb, k, n, colabs, diag, s));
    const unsigned grid = unsigned((2 * n + 127) / 128);
    CRTG_ELEM_DISPATCH(elem, {
      launch_k(k_col_sumsq<T, R>, grid, 128, 0, s, static_cast<const T*>(B), ldb, int(k), int(n), colabs,
                                             colsq);
    })
    launch_k(k_col_finalize, unsigned((n + 127) / 128), 128, 0, s, int(n), colabs, colsq, p_fast, delta,
                                                              nu, diag);
    return launched(2);
  }
  CRTG_ELEM_DISPATCH(elem, {
    constexpr int parts = R ? 1 : 2;
    constexpr int cols = 32 / parts;
    const size_t smem = size_t(kColS) * kColR * 32 * sizeof(T);
    // the attribute is per device: set once per (instantiation, device)
    static std::atomic<unsigned long long> attr_set{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_set.load(std::memory_order_relaxed) & bit) &&
        cudaFuncSetAttribute(k_col_stats<T, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem)) == cudaSuccess)
      attr_set.fetch_or(bit, std::memory_order_relaxed);
    launch_k(k_col_stats<T, R>, unsigned((n + cols - 1) / cols), 128, smem, s,
        static_cast<const T*>(B), ldb, int(k), int(n), p_fast, delta, nu, colabs, diag);
  })
  return launched(1);
}

int launch_bar(const double* absval, int64_t count, int32_t* bar, cudaStream_t s) {
  if (count <= 0) return 0;
  launch_k(k_bar, unsigned((count + 255) / 256), 256, 0, s, absval, count, bar);
  return launched(1);
}

int launch_accurate_exps(const int32_t* maxb, const double* absval, const int32_t* bar,
                         int64_t count, float p_accu, float delta, int32_t* out,
                         unsigned long long* clamp_counter, cudaStream_t s) {
  if (count <= 0) return 0;
  launch_k(k_accurate_exps, unsigned((count + 255) / 256), 256, 0, s, maxb, absval, bar, count, p_accu,
                                                                 delta, out, clamp_counter);
  return launched(1);
}

// ---------------------------------------------------------------------------
// stage-level API (stages.py): the reference's log2_upper and quantize on
// device arrays
// ---------------------------------------------------------------------------
namespace {
// flags[0]: non-finite or non-positive input
__global__ void k_log2_upper_arr(const double* __restrict__ x, int64_t n, float* __restrict__ out,
                                 unsigned long long* flags) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double v = x[i];
    if (!(v > 0.0) || !isfinite(v)) {
      atomicAdd(flags, 1ull);
      out[i] = 0.0f;
      continue;
    }
    out[i] = log2_upper(v);
  }
}

// trunc(ldexp(x, e)) with e per row (axis 0) or per column (axis 1)
// (scaling.py:277-293); flags[0]: |scaled| >= 2^90 (DomainError)
__global__ void k_quantize(const double* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                           const int64_t* __restrict__ exps, int axis, double* __restrict__ out,
                           int64_t ldo, unsigned long long* flags) {
  const int64_t total = rows * cols;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = t / cols, j = t % cols;
    int64_t e = exps[axis == 0 ? i : j];
    // np.ldexp with an out-of-range exponent saturates: beyond +-2200 every
    // finite nonzero double has already overflowed / flushed to zero
    e = e > 2200 ? 2200 : (e < -2200 ? -2200 : e);
    const double v = ldexp(x[i * ldx + j], int(e));
    if (fabs(v) >= 0x1p90) atomicAdd(flags, 1ull);
    out[i * ldo + j] = trunc(v);
  }
}
}  // namespace

int launch_log2_upper(const double* x, int64_t n, float* out, unsigned long long* flags,
                      cudaStream_t s) {
  if (n <= 0) return 0;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_log2_upper_arr<<<unsigned(blocks), 256, 0, s>>>(x, n, out, flags);
  return launched(1);
}

int launch_quantize(const double* x, int64_t rows, int64_t cols, int64_t ldx, const int64_t* exps,
                    int axis, double* out, int64_t ldo, unsigned long long* flags,
                    cudaStream_t s) {
  const int64_t total = rows * cols;
  if (total <= 0) return 0;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_quantize<<<unsigned(blocks), 256, 0, s>>>(x, rows, cols, ldx, exps, axis, out, ldo, flags);
  return launched(1);
}

}  // namespace crtg
