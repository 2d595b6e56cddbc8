// crt.cu — K4: CRT accumulate + symmetric reduction mod P + inverse scaling +
// complex assembly, one thread per 4 output elements.
//
// Op-for-op restatement (no FMA; every op an explicit _rn intrinsic) of
//   crt_accumulate   crt.py:221-243  S1 += coeff_hi[l]*e_l, S2 += coeff_lo[l]*e_l, l ascending
//   crt_reduce       crt.py:246-258 -> symmetric_mod_wide crt.py:154-184
//                    (double-double with Dekker two_prod, ddarith.py:15-54, on the
//                     double path; plain float64 on the single path)
//   inverse_scale    emulate.py:135-144   ldexp(C', -mu_i - nu_j), one cast
//   assembly         emulate.py:239-240   (re + 1j*im): real = re + (0*im - 0),
//                                          imag = 0 + (0 + im), in the output type
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

// CTAs per SM the CRT kernel is compiled for (3: 80 registers, no spills)
#ifndef CRTG_CRT_MINB
#define CRTG_CRT_MINB 3
#endif
// moduli whose residue words are loaded ahead of the arithmetic (even)
#ifndef CRTG_CRT_UNROLL
#define CRTG_CRT_UNROLL 0
#endif
// the complex pipeline's CRT specialised on the modulus count (k_crt_n)
#ifndef CRTG_CRT_TEMPLATED
#define CRTG_CRT_TEMPLATED 1
#endif
// CTAs per SM of the two-column form (N <= 16 / N > 16)
#ifndef CRTG_CRT_Q2_MINB
#define CRTG_CRT_Q2_MINB 4
#endif
#ifndef CRTG_CRT_Q2_MINB_WIDE
#define CRTG_CRT_Q2_MINB_WIDE 3
#endif
#ifndef CRTG_CRT_BATCH
#define CRTG_CRT_BATCH 8
#endif

namespace crtg {

namespace {

struct DD {
  double hi, lo;
};

__device__ __forceinline__ DD two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}

__device__ __forceinline__ DD quick_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}

// two_prod(p_hi, z) (ddarith.py:36-44).  Dekker's error term is EXACT here
// (no overflow, |z| < 2^13, p_hi < 2^1000), so it equals the single-rounding
// fma(p_hi, z, -p) bit for bit — signed zeros included (z = +-0 gives +0 both
// ways) — at 2 FP64 ops instead of 13.
__device__ __forceinline__ DD two_prod_p(double a, double b) {
  const double p = __dmul_rn(a, b);
  return {p, __fma_rn(a, b, -p)};
}

__device__ __forceinline__ DD dd_add(double ahi, double alo, double bhi, double blo) {
  DD s = two_sum(ahi, bhi);
  const DD t = two_sum(alo, blo);
  double s2 = __dadd_rn(s.lo, t.hi);
  s = quick_two_sum(s.hi, s2);
  s2 = __dadd_rn(s.lo, t.lo);
  return quick_two_sum(s.hi, s2);
}

// z = ceil(q - 0.5) with q = fl(s / p_hi) (crt.py:166-167).  The quotient is
// formed with the reciprocal; whenever q - 0.5 lies within a few ulps of an
// integer (where the two roundings could disagree) the exact division is used.
// |q| < 2^13 here, so rounding to an integer is the 1.5*2^52 magic-number add
// (two DADDs on the FP64 pipe instead of the slower FRND).
__device__ __forceinline__ double rint_small(double d) {
  return __dsub_rn(__dadd_rn(d, 0x1.8p52), 0x1.8p52);
}

__device__ __forceinline__ double ceil_small(double d) {
  const double r = rint_small(d);
  return r < d ? __dadd_rn(r, 1.0) : r;
}

__device__ __forceinline__ double quotient_z(double s, const DevConsts& dc) {
  const double d = __dsub_rn(__dmul_rn(s, dc.inv_p), 0.5);
  const double r = rint_small(d);
  if (fabs(__dsub_rn(d, r)) > 0x1p-40 * (fabs(d) + 1.0)) return ceil_small(d);
  return ceil(__dsub_rn(__ddiv_rn(s, dc.p_hi), 0.5));
}

// residue byte q of a word whose bytes are e + 128 (word ^ 0x80808080) -> (double)e
// exactly: the bit pattern 0x43300000:(e + 128) is 2^52 + e + 128 (no I2F)
__device__ __forceinline__ double byte_to_f64(uint32_t wx, int q) {
  return __dsub_rn(__hiloint2double(0x43300000, int(__byte_perm(wx, 0, 0x4440 + q))),
                   4503599627370624.0 /* 2^52 + 128 */);
}

// symmetric_mod_wide (crt.py:154-184), double-double path
__device__ __forceinline__ double reduce_double(double s1, double s2, const DevConsts& dc) {
  const double z = quotient_z(__dadd_rn(s1, s2), dc);
  const DD hl = two_sum(s1, s2);
  DD pz = two_prod_p(dc.p_hi, z);
  pz.lo = __dadd_rn(pz.lo, __dmul_rn(dc.p_lo, z));
  pz = quick_two_sum(pz.hi, pz.lo);
  const DD r = dd_add(hl.hi, hl.lo, -pz.hi, -pz.lo);
  return __dadd_rn(r.hi, r.lo);
}

// plain float64 path (single precision results)
__device__ __forceinline__ double reduce_single(double s, const DevConsts& dc) {
  const double z = quotient_z(__dadd_rn(s, 0.0), dc);
  return __dsub_rn(__dsub_rn(s, __dmul_rn(z, dc.p_hi)), __dmul_rn(z, dc.p_lo));
}

// c + a.h0 * b.b0 + a.h1 * b.b1 (lo: bytes 0,1 / hi: bytes 2,3); a unsigned 16-bit
// halves, b signed bytes
__device__ __forceinline__ int32_t dp2a_lo(uint32_t a, uint32_t b, int32_t c) {
  int32_t d;
  asm("dp2a.lo.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ int32_t dp2a_hi(uint32_t a, uint32_t b, int32_t c) {
  int32_t d;
  asm("dp2a.hi.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ uint32_t load_word(const int8_t* p, bool aligned, int64_t j0, int64_t n) {
  if (aligned) return *reinterpret_cast<const uint32_t*>(p);
  uint32_t w = 0;
  for (int q = 0; q < 4 && j0 + q < n; ++q) w |= uint32_t(uint8_t(p[q])) << (8 * q);
  return w;
}

template <bool SINGLE, bool LIMBS, bool REAL>
__global__ void __launch_bounds__(256, CRTG_CRT_MINB) k_crt(int64_t m, int64_t n, const int8_t* __restrict__ e_re,
                                             const int8_t* __restrict__ e_im, int64_t e_plane,
                                             int64_t e_ld, const int32_t* __restrict__ mu,
                                             const int32_t* __restrict__ nu,
                                             const __grid_constant__ DevConsts dc, void* C,
                                             int64_t ldc) {
  pdl_begin();
  // 2-D: x = quads of 4 columns, y strides over rows (no division per element)
  const int64_t nq = (n + 3) >> 2;
  const int64_t jq = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (jq >= nq) return;
  const int64_t j0 = jq * 4;
  for (int64_t i = blockIdx.y; i < m; i += gridDim.y) {
  const int8_t* pr = e_re + i * e_ld + j0;
  const int8_t* pi = e_im + i * e_ld + j0;
  const bool aligned = ((reinterpret_cast<uintptr_t>(pr) |
                         (REAL ? 0 : reinterpret_cast<uintptr_t>(pi)) | uintptr_t(e_plane)) & 3) ==
                            0 &&
                        j0 + 4 <= n;
  // S1 (exact, on a 2^g grid): integer limbs on the INT pipes; S2: the rounded
  // f64 sequence of crt.py:239-240, l ascending, no FMA.
  int32_t tr[3][4] = {}, ti[3][4] = {};
  double s1r[4] = {0, 0, 0, 0}, s1i[4] = {0, 0, 0, 0};
  double s2r[4] = {0, 0, 0, 0}, s2i[4] = {0, 0, 0, 0};
  // residue words are loaded in batches of kB moduli ahead of the arithmetic
  // (latency-bound otherwise); S2 terms are still added in ascending l, and the
  // exact integer S1 limbs take two moduli per dp2a (16-bit limb pair x the
  // residue bytes of both moduli)
  constexpr int kB = CRTG_CRT_BATCH;
#if CRTG_CRT_UNROLL
  // unrolled over the moduli: coeff_lo / limb constants become immediate
  // constant-bank operands instead of per-modulus LDC loads
#pragma unroll
  for (int l0 = 0; l0 < CRTG_MAX_MODULI; l0 += kB) {
    if (l0 >= dc.n) break;
#else
  for (int l0 = 0; l0 < dc.n; l0 += kB) {
#endif
    uint32_t wr[kB], wi[kB];
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      wr[b] = wi[b] = 0;
      if (l0 + b < dc.n) {
        wr[b] = load_word(pr + (l0 + b) * e_plane, aligned, j0, n);
        if (!REAL) wi[b] = load_word(pi + (l0 + b) * e_plane, aligned, j0, n);
      }
    }
    if constexpr (LIMBS) {
#pragma unroll
      for (int b = 0; b < kB; b += 2) {
        if (l0 + b >= dc.n) break;
        // bytes (e_l[q], e_l+1[q]) for q = 0,1 and q = 2,3
        const uint32_t r01 = __byte_perm(wr[b], wr[b + 1], 0x5140);
        const uint32_t r23 = __byte_perm(wr[b], wr[b + 1], 0x7362);
        const uint32_t i01 = __byte_perm(wi[b], wi[b + 1], 0x5140);
        const uint32_t i23 = __byte_perm(wi[b], wi[b + 1], 0x7362);
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const uint32_t hp = dc.limb_pair[(l0 + b) >> 1][t];
          tr[t][0] = dp2a_lo(hp, r01, tr[t][0]);
          tr[t][1] = dp2a_hi(hp, r01, tr[t][1]);
          tr[t][2] = dp2a_lo(hp, r23, tr[t][2]);
          tr[t][3] = dp2a_hi(hp, r23, tr[t][3]);
          if (!REAL) {
            ti[t][0] = dp2a_lo(hp, i01, ti[t][0]);
            ti[t][1] = dp2a_hi(hp, i01, ti[t][1]);
            ti[t][2] = dp2a_lo(hp, i23, ti[t][2]);
            ti[t][3] = dp2a_hi(hp, i23, ti[t][3]);
          }
        }
      }
    }
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const int l = l0 + b;
      if (l >= dc.n) break;
      const double cl = dc.coeff_lo[l];
      const uint32_t xr = wr[b] ^ 0x80808080u, xi = wi[b] ^ 0x80808080u;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double er = byte_to_f64(xr, q);
        const double ei = REAL ? 0.0 : byte_to_f64(xi, q);
        if constexpr (!LIMBS) {
          s1r[q] = __dadd_rn(s1r[q], __dmul_rn(dc.coeff_hi[l], er));
          s1i[q] = __dadd_rn(s1i[q], __dmul_rn(dc.coeff_hi[l], ei));
        }
        s2r[q] = __dadd_rn(s2r[q], __dmul_rn(cl, er));
        if (!REAL) s2i[q] = __dadd_rn(s2i[q], __dmul_rn(cl, ei));
      }
    }
  }
  if constexpr (LIMBS) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t ir = (int64_t(tr[2][q]) << 32) + (int64_t(tr[1][q]) << 16) + tr[0][q];
      const int64_t ii = (int64_t(ti[2][q]) << 32) + (int64_t(ti[1][q]) << 16) + ti[0][q];
      s1r[q] = __dmul_rn(double(ir), dc.hi_scale);  // exact
      s1i[q] = __dmul_rn(double(ii), dc.hi_scale);
    }
  }
  const int32_t mi = mu[i];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t j = j0 + q;
    if (j >= n) break;
    const int ex = -mi - nu[j];
    if (REAL) {
      // emulate_gemm_real: inverse_scale of the reduced real value, one cast
      if (SINGLE) {
        const double cr = reduce_single(__dadd_rn(s1r[q], s2r[q]), dc);
        reinterpret_cast<float*>(C)[i * ldc + j] = __double2float_rn(ldexp_rn(cr, ex));
      } else {
        reinterpret_cast<double*>(C)[i * ldc + j] =
            ldexp_rn(reduce_double(s1r[q], s2r[q], dc), ex);
      }
    } else if (SINGLE) {
      const double cr = reduce_single(__dadd_rn(s1r[q], s2r[q]), dc);
      const double ci = reduce_single(__dadd_rn(s1i[q], s2i[q]), dc);
      const float re = __double2float_rn(ldexp_rn(cr, ex));
      const float im = __double2float_rn(ldexp_rn(ci, ex));
      const float xr = __fsub_rn(__fmul_rn(0.0f, im), 0.0f);
      const float xi = __fadd_rn(0.0f, im);
      float2 o;
      o.x = __fadd_rn(re, xr);
      o.y = __fadd_rn(0.0f, xi);
      reinterpret_cast<float2*>(C)[i * ldc + j] = o;
    } else {
      const double re = ldexp_rn(reduce_double(s1r[q], s2r[q], dc), ex);
      const double im = ldexp_rn(reduce_double(s1i[q], s2i[q], dc), ex);
      const double xr = __dsub_rn(__dmul_rn(0.0, im), 0.0);
      const double xi = __dadd_rn(0.0, im);
      double2 o;
      o.x = __dadd_rn(re, xr);
      o.y = __dadd_rn(0.0, xi);
      reinterpret_cast<double2*>(C)[i * ldc + j] = o;
    }
  }
  }  // grid-stride loop
}

// ---------------------------------------------------------------------------
// k_crt_n: the complex-pipeline CRT with the modulus count N a compile-time
// constant.  Same arithmetic, in the same order, as k_crt<SINGLE, LIMBS=true,
// REAL=false>; what changes is the instruction stream around it:
//  * every modulus loop is fully unrolled, so coeff_lo[l] and the S1 limb pairs
//    are constant-bank operands of the DMUL / IDP (no per-modulus LDC, no loop
//    branches or bounds checks); all 2N residue words are loaded up front;
//  * the quotient z = ceil(fl(fl(S / p_hi) - 0.5)) (crt.py:166-167) is formed as
//    ceil(fl(S * (1/p_hi)) - 0.5) with one round-up add of 1.5 * 2^52 (valid for
//    |d| < 2^51); the two quotients differ by < 2^-39 (|S / p_hi| < 2^13), so
//    whenever the candidate z lies more than 2^-24 inside (d, d + 1) it equals the
//    reference's ceil, and otherwise the exact division runs.  A zero z comes out
//    as +0 where numpy's ceil gives -0: z only enters through p_hi * z and
//    p_lo * z, and with S1 = +0 (integer limbs) every signed zero downstream is
//    the same either way (K4).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double quotient_z_fast(double s, const DevConsts& dc) {
  const double e = __dmul_rn(s, dc.inv_p);
  const double d = __dsub_rn(e, 0.5);
  const double z = __dsub_rn(__dadd_ru(d, 0x1.8p52), 0x1.8p52);  // ceil(d)
  if (fabs(__dsub_rn(z, e)) < 0.5 - 0x1p-24) return z;
  return ceil(__dsub_rn(__ddiv_rn(s, dc.p_hi), 0.5));
}

__device__ __forceinline__ double reduce_double_fast(double s1, double s2, const DevConsts& dc) {
  const DD hl = two_sum(s1, s2);
  const double z = quotient_z_fast(hl.hi, dc);
  DD pz = two_prod_p(dc.p_hi, z);
  pz.lo = __dadd_rn(pz.lo, __dmul_rn(dc.p_lo, z));
  pz = quick_two_sum(pz.hi, pz.lo);
  const DD r = dd_add(hl.hi, hl.lo, -pz.hi, -pz.lo);
  return __dadd_rn(r.hi, r.lo);
}

__device__ __forceinline__ double reduce_single_fast(double s, const DevConsts& dc) {
  const double z = quotient_z_fast(__dadd_rn(s, 0.0), dc);
  return __dsub_rn(__dsub_rn(s, __dmul_rn(z, dc.p_hi)), __dmul_rn(z, dc.p_lo));
}

// residue byte q of a raw e-plane word (signed bytes) -> (double)e:
//  0: 2^52 + (e + 128) built in a register pair, minus 2^52 + 128 (FP64 pipe)
//  1: sign-extending PRMT + I2F.F64.S32 (conversion pipe)
#ifndef CRTG_CRT_CVT
#define CRTG_CRT_CVT 2
#endif
__device__ __forceinline__ double raw_byte_to_f64(uint32_t w, int q) {
#if CRTG_CRT_CVT == 1
  return double(int32_t(__byte_perm(w, 0, 0x8880 + q + 0x0000)));
#elif CRTG_CRT_CVT == 2
  double d;
  asm("cvt.rn.f64.s8 %0, %1;" : "=d"(d) : "h"(static_cast<unsigned short>(w >> (8 * q))));
  return d;
#else
  return byte_to_f64(w ^ 0x80808080u, q);
#endif
}

// numpy's re + 1j*im for finite re, im (emulate.py:239-240):
//   real = re + (0*im - 0), imag = 0 + (0 + im).
// 0*im - 0 is a zero carrying im's sign, so real == re except that re = -0 with
// im's sign bit clear gives +0; imag == im except that -0 gives +0 (= im + 0).
// Integer select + one DADD instead of five FP64-pipe ops.
__device__ __forceinline__ double2 assemble_f64(double re, double im) {
  const long long rb = __double_as_longlong(re), ib = __double_as_longlong(im);
  double2 o;
  o.x = __longlong_as_double((rb == (long long)0x8000000000000000ull && ib >= 0) ? 0ll : rb);
  o.y = __dadd_rn(im, 0.0);
  return o;
}

// Q: output columns per thread (4; 2 for small grids, where 4 left a third of
// a wave as the tail: 1024^2 was 2.3 waves)
template <int N, bool SINGLE, bool REAL, int Q = 4>
__global__ void __launch_bounds__(256, N > 16 ? (Q == 2 ? CRTG_CRT_Q2_MINB_WIDE : 2) : (Q == 2 ? CRTG_CRT_Q2_MINB : CRTG_CRT_MINB))
    k_crt_n(int64_t m, int64_t n, const int8_t* __restrict__ e_re, const int8_t* __restrict__ e_im,
            int64_t e_plane, int64_t e_ld, const int32_t* __restrict__ mu,
            const int32_t* __restrict__ nu, const __grid_constant__ DevConsts dc, void* C,
            int64_t ldc) {
  static_assert(Q == 4 || Q == 2, "4 or 2 columns per thread");
  pdl_begin();
  const int64_t nq = (n + Q - 1) / Q;
  const int64_t jq = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (jq >= nq) return;
  const int64_t j0 = jq * Q;
  for (int64_t i = blockIdx.y; i < m; i += gridDim.y) {
    const int8_t* pr = e_re + i * e_ld + j0;
    const int8_t* pi = REAL ? pr : e_im + i * e_ld + j0;  // no imaginary plane (real path)
    const bool aligned =
        ((reinterpret_cast<uintptr_t>(pr) | reinterpret_cast<uintptr_t>(pi) | uintptr_t(e_plane)) &
         (Q - 1)) == 0 &&
        j0 + Q <= n;
    uint32_t wr[N + (N & 1)], wi[N + (N & 1)];
    if (aligned) {
#pragma unroll
      for (int l = 0; l < N; ++l) {
        if (Q == 4) {
          wr[l] = __ldg(reinterpret_cast<const uint32_t*>(pr + l * e_plane));
          wi[l] = REAL ? 0u : __ldg(reinterpret_cast<const uint32_t*>(pi + l * e_plane));
        } else {
          wr[l] = __ldg(reinterpret_cast<const uint16_t*>(pr + l * e_plane));
          wi[l] = REAL ? 0u : __ldg(reinterpret_cast<const uint16_t*>(pi + l * e_plane));
        }
      }
    } else {
#pragma unroll
      for (int l = 0; l < N; ++l) {
        wr[l] = load_word(pr + l * e_plane, false, j0, Q == 4 ? n : min(n, j0 + Q));
        wi[l] = REAL ? 0u : load_word(pi + l * e_plane, false, j0, Q == 4 ? n : min(n, j0 + Q));
      }
    }
    if (N & 1) wr[N + (N & 1) - 1] = wi[N + (N & 1) - 1] = 0u;
    // per modulus pair: S1 as exact integer limb sums (two moduli per dp2a), then
    // S2 -- the rounded f64 sequence of crt.py:239-240, l ascending, no FMA
    int32_t tr[3][Q] = {}, ti[3][Q] = {};
    double s2r[Q] = {}, s2i[Q] = {};
#pragma unroll
    for (int l = 0; l < N; l += 2) {
      const uint32_t r01 = __byte_perm(wr[l], wr[l + 1], 0x5140);
      const uint32_t i01 = __byte_perm(wi[l], wi[l + 1], 0x5140);
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const uint32_t hp = dc.limb_pair[l >> 1][t];
        tr[t][0] = dp2a_lo(hp, r01, tr[t][0]);
        tr[t][1] = dp2a_hi(hp, r01, tr[t][1]);
        if (!REAL) {
          ti[t][0] = dp2a_lo(hp, i01, ti[t][0]);
          ti[t][1] = dp2a_hi(hp, i01, ti[t][1]);
        }
        if (Q == 4) {
          const uint32_t r23 = __byte_perm(wr[l], wr[l + 1], 0x7362);
          const uint32_t i23 = __byte_perm(wi[l], wi[l + 1], 0x7362);
          tr[t][Q - 2] = dp2a_lo(hp, r23, tr[t][Q - 2]);
          tr[t][Q - 1] = dp2a_hi(hp, r23, tr[t][Q - 1]);
          if (!REAL) {
            ti[t][Q - 2] = dp2a_lo(hp, i23, ti[t][Q - 2]);
            ti[t][Q - 1] = dp2a_hi(hp, i23, ti[t][Q - 1]);
          }
        }
      }
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        if (l + b >= N) break;
        const double cl = dc.coeff_lo[l + b];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          s2r[q] = __dadd_rn(s2r[q], __dmul_rn(cl, raw_byte_to_f64(wr[l + b], q)));
          if (!REAL) s2i[q] = __dadd_rn(s2i[q], __dmul_rn(cl, raw_byte_to_f64(wi[l + b], q)));
        }
      }
    }
    const int32_t mi = mu[i];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int64_t j = j0 + q;
      if (j >= n) break;
      const int64_t ir = (int64_t(tr[2][q]) << 32) + (int64_t(tr[1][q]) << 16) + tr[0][q];
      const int64_t ii = (int64_t(ti[2][q]) << 32) + (int64_t(ti[1][q]) << 16) + ti[0][q];
      const double s1r = __dmul_rn(double(ir), dc.hi_scale);  // exact
      const double s1i = __dmul_rn(double(ii), dc.hi_scale);
      const int ex = -mi - nu[j];
      if (REAL) {
        // emulate_gemm_real: inverse_scale of the reduced real value, one cast
        if (SINGLE)
          reinterpret_cast<float*>(C)[i * ldc + j] =
              __double2float_rn(ldexp_rn(reduce_single_fast(__dadd_rn(s1r, s2r[q]), dc), ex));
        else
          reinterpret_cast<double*>(C)[i * ldc + j] =
              ldexp_rn(reduce_double_fast(s1r, s2r[q], dc), ex);
      } else if (SINGLE) {
        const double cr = reduce_single_fast(__dadd_rn(s1r, s2r[q]), dc);
        const double ci = reduce_single_fast(__dadd_rn(s1i, s2i[q]), dc);
        const float re = __double2float_rn(ldexp_rn(cr, ex));
        const float im = __double2float_rn(ldexp_rn(ci, ex));
        float2 o;
        o.x = __fadd_rn(re, __fsub_rn(__fmul_rn(0.0f, im), 0.0f));
        o.y = __fadd_rn(0.0f, __fadd_rn(0.0f, im));
        reinterpret_cast<float2*>(C)[i * ldc + j] = o;
      } else {
        const double re = ldexp_rn(reduce_double_fast(s1r, s2r[q], dc), ex);
        const double im = ldexp_rn(reduce_double_fast(s1i, s2i[q], dc), ex);
        reinterpret_cast<double2*>(C)[i * ldc + j] = assemble_f64(re, im);
      }
    }
  }
}

}  // namespace

int launch_crt(bool single, bool real, int64_t m, int64_t n, const int8_t* e_re,
               const int8_t* e_im, int64_t e_plane, int64_t e_ld, const int32_t* mu,
               const int32_t* nu, const DevConsts& dc, void* C, int64_t ldc, cudaStream_t s,
               int max_ctas) {
  const bool limbs = dc.hi_scale != 0.0;
  // complex pipeline: two columns per thread at 4 CTAs/SM (3 above 16 moduli),
  // 64 registers, no spills -- twice the resident warps of the 4-column form
  // (80 registers at 3 CTAs/SM) hide the FP64 dependency chains: 16384^3 N=15
  // CRT stage 5.33 -> 5.12 ms per step; small grids (1024^2: ~5 waves instead
  // of ~2.3 with a one-third tail) gain too.  CRTG_CRT_Q2_THREADS caps the
  // 4-column thread count that still takes the 2-column form (0: never).
  static const int64_t q2_max = [] {
    const char* v = std::getenv("CRTG_CRT_Q2_THREADS");
    return v && *v ? int64_t(std::atoll(v)) : INT64_MAX;
  }();
  const bool q2 = CRTG_CRT_TEMPLATED && limbs && !real && max_ctas == 0 &&
                  m * ((n + 3) / 4) <= q2_max;
  const int64_t nq = q2 ? (n + 1) / 2 : (n + 3) / 4;
  if (m <= 0 || nq <= 0) return 0;
  const unsigned gx = unsigned((nq + 255) / 256);
  int64_t gy = std::min<int64_t>(m, 65535);
  // max_ctas (side-stream runs beside the GEMM): cap the total CTA count
  if (max_ctas > 0) gy = std::max<int64_t>(1, std::min<int64_t>(gy, max_ctas / int64_t(gx)));
  const dim3 grid(gx, unsigned(gy));
#if CRTG_CRT_TEMPLATED
  if (limbs && dc.n >= 1 && dc.n <= CRTG_MAX_MODULI) {
#define CRTG_CRT_NR(NN, S, R, Q) \
  launch_k(k_crt_n<NN, S, R, Q>, grid, 256, 0, s, m, n, e_re, e_im, e_plane, e_ld, mu, nu, dc, C, ldc)
#define CRTG_CRT_N(NN)                                                      \
  case NN:                                                              \
    if (real) {                                                         \
      if (single) CRTG_CRT_NR(NN, true, true, 4); else CRTG_CRT_NR(NN, false, true, 4);   \
    } else if (q2) {                                                    \
      if (single) CRTG_CRT_NR(NN, true, false, 2); else CRTG_CRT_NR(NN, false, false, 2); \
    } else {                                                            \
      if (single) CRTG_CRT_NR(NN, true, false, 4); else CRTG_CRT_NR(NN, false, false, 4); \
    }                                                                   \
    break;
    switch (dc.n) {
      CRTG_CRT_N(1) CRTG_CRT_N(2) CRTG_CRT_N(3) CRTG_CRT_N(4) CRTG_CRT_N(5)
      CRTG_CRT_N(6) CRTG_CRT_N(7) CRTG_CRT_N(8) CRTG_CRT_N(9) CRTG_CRT_N(10)
      CRTG_CRT_N(11) CRTG_CRT_N(12) CRTG_CRT_N(13) CRTG_CRT_N(14) CRTG_CRT_N(15)
      CRTG_CRT_N(16) CRTG_CRT_N(17) CRTG_CRT_N(18) CRTG_CRT_N(19) CRTG_CRT_N(20)
    }
#undef CRTG_CRT_N
#undef CRTG_CRT_NR
    return launched(1);
  }
#endif
#define CRTG_CRT(S, L, R) \
  launch_k(k_crt<S, L, R>, grid, 256, 0, s, m, n, e_re, e_im, e_plane, e_ld, mu, nu, dc, C, ldc)
  if (real) {
    if (single) { if (limbs) CRTG_CRT(true, true, true); else CRTG_CRT(true, false, true); }
    else { if (limbs) CRTG_CRT(false, true, true); else CRTG_CRT(false, false, true); }
  } else {
    if (single) { if (limbs) CRTG_CRT(true, true, false); else CRTG_CRT(true, false, false); }
    else { if (limbs) CRTG_CRT(false, true, false); else CRTG_CRT(false, false, false); }
  }
#undef CRTG_CRT
  return launched(1);
}

// ---------------------------------------------------------------------------
// stage-level API (stages.py): crt_accumulate (crt.py:221-243),
// symmetric_mod_wide (crt.py:154-184) with the reference's Dekker two_prod
// literally (ddarith.py:30-44; any double input, not only CRT sums), and
// inverse_scale (emulate.py:135-144)
// ---------------------------------------------------------------------------
namespace {
__global__ void k_crt_accumulate(const int8_t* __restrict__ e, int nmod, int64_t count,
                                 CrtCoeffs cf, int single, double* __restrict__ s1,
                                 double* __restrict__ s2) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    double a = 0.0, b = 0.0;
    for (int l = 0; l < nmod; ++l) {
      const double v = double(e[int64_t(l) * count + i]);
      a = __dadd_rn(a, __dmul_rn(cf.hi[l], v));
      b = __dadd_rn(b, __dmul_rn(cf.lo[l], v));
    }
    if (single) {
      s1[i] = __dadd_rn(a, b);
    } else {
      s1[i] = a;
      s2[i] = b;
    }
  }
}

__device__ __forceinline__ DD dekker_split(double a) {
  const double c = __dmul_rn(134217729.0, a);
  const double hi = __dsub_rn(c, __dsub_rn(c, a));
  return {hi, __dsub_rn(a, hi)};
}

__device__ __forceinline__ DD dekker_two_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  const DD as = dekker_split(a), bs = dekker_split(b);
  const double e = __dadd_rn(__dadd_rn(__dadd_rn(__dsub_rn(__dmul_rn(as.hi, bs.hi), p),
                                                 __dmul_rn(as.hi, bs.lo)),
                                        __dmul_rn(as.lo, bs.hi)),
                             __dmul_rn(as.lo, bs.lo));
  return {p, e};
}

__global__ void k_sym_mod_wide(const double* __restrict__ s_hi, const double* __restrict__ s_lo,
                               int64_t count, double p_hi, double p_lo, int use_dd,
                               double* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double h = s_hi[i];
    const double l = s_lo ? s_lo[i] : 0.0;
    const double z = ceil(__dsub_rn(__ddiv_rn(__dadd_rn(h, l), p_hi), 0.5));
    if (use_dd) {
      const DD hl = two_sum(h, l);
      DD pz = dekker_two_prod(p_hi, z);
      pz.lo = __dadd_rn(pz.lo, __dmul_rn(p_lo, z));
      pz = quick_two_sum(pz.hi, pz.lo);
      const DD r = dd_add(hl.hi, hl.lo, -pz.hi, -pz.lo);
      out[i] = __dadd_rn(r.hi, r.lo);
    } else {
      out[i] = __dsub_rn(__dsub_rn(h, __dmul_rn(z, p_hi)), __dmul_rn(z, p_lo));
    }
  }
}

__global__ void k_inverse_scale(const double* __restrict__ c, int64_t rows, int64_t cols,
                                int64_t ldc, const int64_t* __restrict__ mu,
                                const int64_t* __restrict__ nu, int out_f32,
                                void* __restrict__ out, int64_t ldo) {
  const int64_t total = rows * cols;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = t / cols, j = t % cols;
    const int32_t e = int32_t(-mu[i] - nu[j]);  // .astype(np.int32)
    const double v = ldexp(c[i * ldc + j], e);
    if (out_f32)
      static_cast<float*>(out)[i * ldo + j] = __double2float_rn(v);
    else
      static_cast<double*>(out)[i * ldo + j] = v;
  }
}

int64_t stage_blocks(int64_t n) { return std::min<int64_t>((n + 255) / 256, 148 * 16); }
}  // namespace

int launch_crt_accumulate(const int8_t* e, int nmod, int64_t count, const CrtCoeffs& cf,
                          bool single, double* s1, double* s2, cudaStream_t s) {
  if (count <= 0) return 0;
  k_crt_accumulate<<<unsigned(stage_blocks(count)), 256, 0, s>>>(e, nmod, count, cf,
                                                                 single ? 1 : 0, s1, s2);
  return launched(1);
}

int launch_sym_mod_wide(const double* s_hi, const double* s_lo, int64_t count, double p_hi,
                        double p_lo, bool use_dd, double* out, cudaStream_t s) {
  if (count <= 0) return 0;
  k_sym_mod_wide<<<unsigned(stage_blocks(count)), 256, 0, s>>>(s_hi, s_lo, count, p_hi, p_lo,
                                                               use_dd ? 1 : 0, out);
  return launched(1);
}

int launch_inverse_scale(const double* c, int64_t rows, int64_t cols, int64_t ldc,
                         const int64_t* mu, const int64_t* nu, bool out_f32, void* out,
                         int64_t ldo, cudaStream_t s) {
  if (rows * cols <= 0) return 0;
  k_inverse_scale<<<unsigned(stage_blocks(rows * cols)), 256, 0, s>>>(
      c, rows, cols, ldc, mu, nu, out_f32 ? 1 : 0, out, ldo);
  return launched(1);
}

}  // namespace crtg
