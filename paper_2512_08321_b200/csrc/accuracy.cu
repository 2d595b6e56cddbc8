// accuracy.cu — GPU accuracy harness.
//
// k_dd_gemm: the reference's double-double product (oracle.py:60-128,
// _dd_gemm_kernel / reference_gemm_dd), bit for bit: for every output entry the
// terms of the stacked real forms C_R = [A_R, -A_I][B_R; B_I] and
// C_I = [A_R, A_I][B_I; B_R] are taken in ascending order, each product is split
// exactly (Dekker, 2^27+1) and accumulated with the accurate double-double
// addition — every FP op an explicit _rn intrinsic (the file is built with
// -fmad=false).  16x16 output tile per CTA, K staged through shared memory with
// the Dekker splits precomputed once per element (split(-x) = -split(x) exactly,
// so the negated A_I terms reuse them).
// k_max_rel_err: max_relative_error (oracle.py:131-169) of an approximation
// against (hi, lo) — componentwise, zero references excluded and counted.
#include "common.cuh"

namespace crtg {

namespace {

constexpr int kT = 16;   // output tile edge
constexpr int kKT = 32;  // K step staged in shared memory

struct Split {
  double x, hi, lo;
};

__device__ __forceinline__ Split split3(double x) {
  const double c = __dmul_rn(134217729.0, x);
  const double hi = __dsub_rn(c, __dsub_rn(c, x));
  return {x, hi, __dsub_rn(x, hi)};
}

// one term of _dd_gemm_kernel (oracle.py:73-96)
__device__ __forceinline__ void dd_term(double& shi, double& slo, double x, double xhi, double xlo,
                                        double y, double yhi, double ylo) {
  const double p = __dmul_rn(x, y);
  const double e = __dadd_rn(
      __dadd_rn(__dadd_rn(__dsub_rn(__dmul_rn(xhi, yhi), p), __dmul_rn(xhi, ylo)),
                __dmul_rn(xlo, yhi)),
      __dmul_rn(xlo, ylo));
  double s1 = __dadd_rn(shi, p);
  double bb = __dsub_rn(s1, shi);
  double s2 = __dadd_rn(__dsub_rn(shi, __dsub_rn(s1, bb)), __dsub_rn(p, bb));
  const double t1 = __dadd_rn(slo, e);
  bb = __dsub_rn(t1, slo);
  const double t2 = __dadd_rn(__dsub_rn(slo, __dsub_rn(t1, bb)), __dsub_rn(e, bb));
  s2 = __dadd_rn(s2, t1);
  double z = __dadd_rn(s1, s2);
  s2 = __dsub_rn(s2, __dsub_rn(z, s1));
  s1 = z;
  s2 = __dadd_rn(s2, t2);
  z = __dadd_rn(s1, s2);
  slo = __dsub_rn(s2, __dsub_rn(z, s1));
  shi = z;
}

// CPLX: A, B interleaved complex128; otherwise real float64.
template <bool CPLX>
__global__ void __launch_bounds__(kT * kT) k_dd_gemm(const double* __restrict__ A, int64_t lda,
                                                     const double* __restrict__ B, int64_t ldb,
                                                     int m, int n, int k, double* __restrict__ hi,
                                                     double* __restrict__ lo, int64_t ldo) {
  __shared__ Split sa[kT][kKT];       // the A part of this pass (rows of the tile)
  __shared__ Split sb[2][kKT][kT];    // B_R and B_I (columns of the tile)
  const int tx = threadIdx.x % kT, ty = threadIdx.x / kT;
  const int i = blockIdx.y * kT + ty, j = blockIdx.x * kT + tx;
  double rh = 0.0, rl = 0.0, ih = 0.0, il = 0.0;
  const int passes = CPLX ? 2 : 1;
  for (int pass = 0; pass < passes; ++pass) {
    for (int h0 = 0; h0 < k; h0 += kKT) {
      // stage: A part (pass 0: A_R, pass 1: A_I) and both parts of B
      for (int t = threadIdx.x; t < kT * kKT; t += kT * kT) {
        const int r = t / kKT, c = t % kKT;
        const int gi = blockIdx.y * kT + r, gh = h0 + c;
        double v = 0.0;
        if (gi < m && gh < k) v = CPLX ? A[2 * (int64_t(gi) * lda + gh) + pass] : A[int64_t(gi) * lda + gh];
        sa[r][c] = split3(v);
      }
      for (int t = threadIdx.x; t < kKT * kT; t += kT * kT) {
        const int r = t / kT, c = t % kT;
        const int gh = h0 + r, gj = blockIdx.x * kT + c;
        double vr = 0.0, vi = 0.0;
        if (gh < k && gj < n) {
          if (CPLX) {
            vr = B[2 * (int64_t(gh) * ldb + gj)];
            vi = B[2 * (int64_t(gh) * ldb + gj) + 1];
          } else {
            vr = B[int64_t(gh) * ldb + gj];
          }
        }
        sb[0][r][c] = split3(vr);
        if (CPLX) sb[1][r][c] = split3(vi);
      }
      __syncthreads();
      const int hn = min(kKT, k - h0);
      if (i < m && j < n) {
        for (int h = 0; h < hn; ++h) {
          const Split x = sa[ty][h];
          if (!CPLX) {
            const Split y = sb[0][h][tx];
            dd_term(rh, rl, x.x, x.hi, x.lo, y.x, y.hi, y.lo);
          } else if (pass == 0) {
            // C_R += A_R B_R ; C_I += A_R B_I   (first k terms of both stacked forms)
            const Split yr = sb[0][h][tx], yi = sb[1][h][tx];
            dd_term(rh, rl, x.x, x.hi, x.lo, yr.x, yr.hi, yr.lo);
            dd_term(ih, il, x.x, x.hi, x.lo, yi.x, yi.hi, yi.lo);
          } else {
            // C_R += (-A_I) B_I ; C_I += A_I B_R   (last k terms)
            const Split yr = sb[0][h][tx], yi = sb[1][h][tx];
            dd_term(rh, rl, -x.x, -x.hi, -x.lo, yi.x, yi.hi, yi.lo);
            dd_term(ih, il, x.x, x.hi, x.lo, yr.x, yr.hi, yr.lo);
          }
        }
      }
      __syncthreads();
    }
  }
  if (i < m && j < n) {
    if (CPLX) {
      reinterpret_cast<double2*>(hi)[int64_t(i) * ldo + j] = make_double2(rh, ih);
      reinterpret_cast<double2*>(lo)[int64_t(i) * ldo + j] = make_double2(rl, il);
    } else {
      hi[int64_t(i) * ldo + j] = rh;
      lo[int64_t(i) * ldo + j] = rl;
    }
  }
}

// per component: err = |(x - hi) - lo|, ref = |hi + lo|, rel = err / ref (ref != 0)
__global__ void k_max_rel_err(int64_t m, int64_t n, int comps, const void* __restrict__ approx,
                              int approx_single, int64_t lda_x, const double* __restrict__ hi,
                              const double* __restrict__ lo, int64_t ldo,
                              unsigned long long* __restrict__ max_bits,
                              unsigned long long* __restrict__ zeros) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  double worst = 0.0;
  unsigned long long nz = 0;
  if (t < m * n) {
    const int64_t i = t / n, j = t % n;
    for (int c = 0; c < comps; ++c) {
      const double x = approx_single
                           ? double(static_cast<const float*>(approx)[(i * lda_x + j) * comps + c])
                           : static_cast<const double*>(approx)[(i * lda_x + j) * comps + c];
      const double h = hi[(i * ldo + j) * comps + c], l = lo[(i * ldo + j) * comps + c];
      const double err = fabs(__dsub_rn(__dsub_rn(x, h), l));
      const double ref = fabs(__dadd_rn(h, l));
      if (ref == 0.0) {
        ++nz;
      } else {
        worst = fmax(worst, __ddiv_rn(err, ref));
      }
    }
  }
  for (int o = 16; o; o >>= 1) {
    worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
    nz += __shfl_xor_sync(0xffffffffu, nz, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(max_bits, (unsigned long long)__double_as_longlong(worst));
    if (nz) atomicAdd(zeros, nz);
  }
}

}  // namespace

int launch_dd_gemm(bool cplx, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                   const double* B, int64_t ldb, double* hi, double* lo, int64_t ldo,
                   cudaStream_t s) {
  dim3 grid(unsigned((n + kT - 1) / kT), unsigned((m + kT - 1) / kT));
  if (cplx)
    k_dd_gemm<true><<<grid, kT * kT, 0, s>>>(A, lda, B, ldb, int(m), int(n), int(k), hi, lo, ldo);
  else
    k_dd_gemm<false><<<grid, kT * kT, 0, s>>>(A, lda, B, ldb, int(m), int(n), int(k), hi, lo, ldo);
  return launched(1);
}

int launch_max_rel_err(bool cplx, int64_t m, int64_t n, const void* approx, bool approx_single,
                       int64_t lda_x, const double* hi, const double* lo, int64_t ldo,
                       unsigned long long* max_bits, unsigned long long* zeros, cudaStream_t s) {
  const int64_t total = m * n;
  if (total <= 0) return 0;
  k_max_rel_err<<<unsigned((total + 255) / 256), 256, 0, s>>>(
      m, n, cplx ? 2 : 1, approx, approx_single ? 1 : 0, lda_x, hi, lo, ldo, max_bits, zeros);
  return launched(1);
}

}  // namespace crtg
