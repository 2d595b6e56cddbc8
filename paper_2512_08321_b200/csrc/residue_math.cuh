// residue_math.cuh — integer residue arithmetic shared by the register
// residue kernels (residue.cu).
#pragma once
#include <cstdint>

#include "common.cuh"

namespace crtg {
namespace {

// Value representations (one truncating conversion per value):
//  medium (|a'| < 2^63, every warp at N <= 14 and most at N <= 20):
//      v = a' + 2^63 as (lo, hi) words = four 16-bit limbs;
//      u = dp2a.hi(hi, c, dp2a.lo(lo, c, k63)) with c = bytes (1, 2^16, 2^32, 2^48 mod p)
//  wide (some |a'| >= 2^63 in the warp): v = 2^90 + a' as three words = six limbs,
//      one more dp2a against (2^64, 2^80 mod p)
// Both give u == a' + off (mod p), u < 2^27; one magic reduction -> t in [0,p).
struct Val3 {
  uint32_t w0, w1, w2;
};

__device__ __forceinline__ void int_parts(double q, uint64_t& M, int& s) {
  const uint64_t bits = uint64_t(__double_as_longlong(q));
  const int e2 = int((bits >> 52) & 0x7FF) - 1023;
  const uint64_t sig = (bits & 0xFFFFFFFFFFFFFull) | (uint64_t(1) << 52);
  s = 0;
  if (e2 < 0) {
    M = 0;
  } else if (e2 <= 52) {
    M = sig >> (52 - e2);
  } else {
    M = sig;
    s = e2 - 52;
  }
}

// v = 2^90 + q as three 32-bit words for an integer-valued |q| < 2^90:
// q = +-M 2^s with M < 2^53 and s <= 37, so M 2^s = hi 2^64 + lo with hi < 2^26;
// the negative case is the two's-complement difference 2^90 - (hi:lo)
__device__ __forceinline__ Val3 split_wide(double q) {
  uint64_t M;
  int s;
  int_parts(q, M, s);
  const uint64_t lo = M << s;
  const uint32_t hi = s > 11 ? uint32_t(M >> (64 - s)) : 0u;
  const uint64_t nlo = 0ull - lo;
  const uint32_t nhi = (1u << 26) - hi - (lo != 0 ? 1u : 0u);
  const bool neg = q < 0.0;
  const uint64_t w01 = neg ? nlo : lo;
  return {uint32_t(w01), uint32_t(w01 >> 32), neg ? nhi : hi + (1u << 26)};
}

// explicit single-instruction integer ops (keeps ptxas from re-associating the
// chains into forms that need register copies of uniform operands)
__device__ __forceinline__ uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// c + a.h0 * b.byte0 + a.h1 * b.byte1   (lo)   /  ... b.byte2, b.byte3   (hi)
__device__ __forceinline__ uint32_t dp2a_lo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("dp2a.lo.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ uint32_t dp2a_hi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("dp2a.hi.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// u mod p for u < 2^31: q = umulhi(u, magic) >> shift (powers of two: magic =
// 2^(32 - log2 p), shift 0), t = u - q p -- three instructions, no branch
__device__ __forceinline__ uint32_t mod_small(uint32_t u, const ResConst& c) {
  const uint32_t q = __umulhi(u, c.magic) >> c.shift;
  return mad_lo(q, c.neg_p, u);
}

// FORM 1: |a'| < 2^31, v = a' + 2^31 (one word, one dp2a); 2: |a'| < 2^63, four
// limbs (two dp2a); 3: six limbs of 2^90 + a' (three dp2a)
template <int FORM>
__device__ __forceinline__ uint32_t res_t(const Val3& v, const ResConst& c) {
  uint32_t u;
  if (FORM == 3) {
    u = dp2a_lo(v.w0, c.dw0123, c.kw);
    u = dp2a_hi(v.w1, c.dw0123, u);
    u = dp2a_lo(v.w2, c.dw45, u);
  } else if (FORM == 2) {
    u = dp2a_hi(v.w1, c.dw0123, dp2a_lo(v.w0, c.dw0123, c.k63));
  } else {
    u = dp2a_lo(v.w0, c.dw0123, c.k31);
  }
  return mod_small(u, c);  // t = (a' + off) mod p
}

}  // namespace
}  // namespace crtg
