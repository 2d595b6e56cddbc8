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
#include "common.cuh"
#include "kernels.cuh"

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

__device__ __forceinline__ DD split(double a) {
  const double c = __dmul_rn(134217729.0, a);
  const double hi = __dsub_rn(c, __dsub_rn(c, a));
  return {hi, __dsub_rn(a, hi)};
}

__device__ __forceinline__ DD two_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  const DD as = split(a), bs = split(b);
  const double e = __dadd_rn(
      __dadd_rn(__dadd_rn(__dsub_rn(__dmul_rn(as.hi, bs.hi), p), __dmul_rn(as.hi, bs.lo)),
                __dmul_rn(as.lo, bs.hi)),
      __dmul_rn(as.lo, bs.lo));
  return {p, e};
}

__device__ __forceinline__ DD dd_add(double ahi, double alo, double bhi, double blo) {
  DD s = two_sum(ahi, bhi);
  const DD t = two_sum(alo, blo);
  double s2 = __dadd_rn(s.lo, t.hi);
  s = quick_two_sum(s.hi, s2);
  s2 = __dadd_rn(s.lo, t.lo);
  return quick_two_sum(s.hi, s2);
}

// symmetric_mod_wide (crt.py:154-184)
__device__ __forceinline__ double reduce_double(double s1, double s2, double p_hi, double p_lo) {
  const double q = __ddiv_rn(__dadd_rn(s1, s2), p_hi);
  const double z = ceil(__dsub_rn(q, 0.5));
  const DD hl = two_sum(s1, s2);
  DD pz = two_prod(p_hi, z);
  pz.lo = __dadd_rn(pz.lo, __dmul_rn(p_lo, z));
  pz = quick_two_sum(pz.hi, pz.lo);
  const DD r = dd_add(hl.hi, hl.lo, -pz.hi, -pz.lo);
  return __dadd_rn(r.hi, r.lo);
}

__device__ __forceinline__ double reduce_single(double s, double p_hi, double p_lo) {
  const double q = __ddiv_rn(__dadd_rn(s, 0.0), p_hi);
  const double z = ceil(__dsub_rn(q, 0.5));
  return __dsub_rn(__dsub_rn(s, __dmul_rn(z, p_hi)), __dmul_rn(z, p_lo));
}

template <bool SINGLE>
__global__ void __launch_bounds__(256) k_crt(int64_t m, int64_t n, const int8_t* __restrict__ e_re,
                                             const int8_t* __restrict__ e_im, int64_t e_plane,
                                             int64_t e_ld, const int32_t* __restrict__ mu,
                                             const int32_t* __restrict__ nu,
                                             const __grid_constant__ DevConsts dc, void* C,
                                             int64_t ldc) {
  const int64_t nq = (n + 3) >> 2;
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= m * nq) return;
  const int64_t i = t / nq;
  const int64_t j0 = (t - i * nq) * 4;
  double s1r[4] = {0, 0, 0, 0}, s2r[4] = {0, 0, 0, 0}, s1i[4] = {0, 0, 0, 0},
         s2i[4] = {0, 0, 0, 0};
  const int8_t* pr = e_re + i * e_ld + j0;
  const int8_t* pi = e_im + i * e_ld + j0;
  const bool aligned = ((reinterpret_cast<uintptr_t>(pr) | reinterpret_cast<uintptr_t>(pi) |
                         uintptr_t(e_plane)) & 3) == 0 && j0 + 4 <= n;
  for (int l = 0; l < dc.n; ++l) {
    uint32_t wr, wi;
    if (aligned) {
      wr = *reinterpret_cast<const uint32_t*>(pr + l * e_plane);
      wi = *reinterpret_cast<const uint32_t*>(pi + l * e_plane);
    } else {
      wr = wi = 0;
      for (int q = 0; q < 4 && j0 + q < n; ++q) {
        wr |= uint32_t(uint8_t(pr[l * e_plane + q])) << (8 * q);
        wi |= uint32_t(uint8_t(pi[l * e_plane + q])) << (8 * q);
      }
    }
    const double ch = dc.coeff_hi[l], cl = dc.coeff_lo[l];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double er = double(int8_t(wr >> (8 * q)));
      const double ei = double(int8_t(wi >> (8 * q)));
      s1r[q] = __dadd_rn(s1r[q], __dmul_rn(ch, er));
      s2r[q] = __dadd_rn(s2r[q], __dmul_rn(cl, er));
      s1i[q] = __dadd_rn(s1i[q], __dmul_rn(ch, ei));
      s2i[q] = __dadd_rn(s2i[q], __dmul_rn(cl, ei));
    }
  }
  const int32_t mi = mu[i];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t j = j0 + q;
    if (j >= n) break;
    const int ex = -mi - nu[j];
    if (SINGLE) {
      const double cr = reduce_single(__dadd_rn(s1r[q], s2r[q]), dc.p_hi, dc.p_lo);
      const double ci = reduce_single(__dadd_rn(s1i[q], s2i[q]), dc.p_hi, dc.p_lo);
      const float re = __double2float_rn(ldexp_rn(cr, ex));
      const float im = __double2float_rn(ldexp_rn(ci, ex));
      const float xr = __fsub_rn(__fmul_rn(0.0f, im), 0.0f);
      const float xi = __fadd_rn(0.0f, im);
      float2 o;
      o.x = __fadd_rn(re, xr);
      o.y = __fadd_rn(0.0f, xi);
      reinterpret_cast<float2*>(C)[i * ldc + j] = o;
    } else {
      const double re = ldexp_rn(reduce_double(s1r[q], s2r[q], dc.p_hi, dc.p_lo), ex);
      const double im = ldexp_rn(reduce_double(s1i[q], s2i[q], dc.p_hi, dc.p_lo), ex);
      const double xr = __dsub_rn(__dmul_rn(0.0, im), 0.0);
      const double xi = __dadd_rn(0.0, im);
      double2 o;
      o.x = __dadd_rn(re, xr);
      o.y = __dadd_rn(0.0, xi);
      reinterpret_cast<double2*>(C)[i * ldc + j] = o;
    }
  }
}

}  // namespace

int launch_crt(bool single, int64_t m, int64_t n, const int8_t* e_re, const int8_t* e_im,
               int64_t e_plane, int64_t e_ld, const int32_t* mu, const int32_t* nu,
               const DevConsts& dc, void* C, int64_t ldc, cudaStream_t s) {
  const int64_t total = m * ((n + 3) / 4);
  if (total <= 0) return 0;
  const unsigned grid = unsigned((total + 255) / 256);
  if (single)
    k_crt<true><<<grid, 256, 0, s>>>(m, n, e_re, e_im, e_plane, e_ld, mu, nu, dc, C, ldc);
  else
    k_crt<false><<<grid, 256, 0, s>>>(m, n, e_re, e_im, e_plane, e_ld, mu, nu, dc, C, ldc);
  return int(cudaGetLastError());
}

}  // namespace crtg
