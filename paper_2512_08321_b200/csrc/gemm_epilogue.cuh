// gemm_epilogue.cuh — TMEM -> register epilogues shared by the 1-CTA and the
// CTA-pair tcgen05 GEMMs (gemm_tc.cu, gemm_pair.cu).
//
// One thread owns one TMEM lane = one output row of the tile and 256 columns,
// read in 8 chunks of 32 (tcgen05.ld.32x32b.x32).
//   KARATSUBA phase 0 (D = Ar*Br): keep D mod p in st[] (packed bytes);
//   phase 1 (E = Ai*Bi): write e_R = sym(D - E), keep (D + E) mod p;
//   phase 2 (F = As*Bs): write e_I = sym(F - (D + E))     (kernel.py:45-51).
//   Reducing D, E, F mod p before combining keeps every value in int32 (the
//   reference widens to int64, kernel.py:46-50) and gives the same residue.
//   RAW: store the int32 accumulator (gemm_i8_i32 parity hook).
#pragma once
#include "common.cuh"
#include "gemm_tc.cuh"

// CRTG_EPI_DB=1 double-buffers the TMEM loads of 8-chunk epilogues (chunk c+1
// in flight while chunk c is reduced); the default single buffer keeps the
// 256-column wide-tile epilogue within 168 registers without spills
#ifndef CRTG_EPI_DB
#define CRTG_EPI_DB 0
#endif

namespace crtg {

__device__ __forceinline__ uint32_t ep_pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return (a & 0xFF) | ((b & 0xFF) << 8) | ((c & 0xFF) << 16) | (d << 24);
}

__device__ __forceinline__ uint32_t ep_byte(uint32_t w, int i) { return (w >> (8 * i)) & 0xFF; }

// u mod p for 0 <= u < 2^31 + 2^23 (shift = floor(log2 p) keeps the magic exact
// there), or u mod 2^j for a power-of-two modulus (wrapping u is then harmless)
template <bool POW2>
__device__ __forceinline__ uint32_t ep_red(uint32_t u, const ModConst& c) {
  if (POW2) return u & uint32_t(c.p - 1);
  const uint32_t q = __umulhi(u, c.magic) >> c.shift;
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(q), "r"(c.neg_p), "r"(u));
  return r;
}

__device__ __forceinline__ uint32_t ep_pack_bytes(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// Karatsuba phases (kernel.py:45-51) with every combination folded into ONE
// biased reduction (|D|, |E|, |F| <= k*127^2 < 2^30 for p < 256; bias >= 2^30 is
// a multiple of p, h = floor(p/2)):
//   phase 0 (D):  dm   = (D + bias) mod p                     -> st
//   phase 1 (E):  e_R  = ((dm - E + bias + h) mod p) - h       -> out
//                 keep = (dm + E + bias) mod p                 -> st
//   phase 2 (F):  e_I  = ((F - keep + bias + h) mod p) - h     -> out
// ((x + h) mod p) - h is the symmetric residue in [-floor(p/2), ceil(p/2) - 1].
template <int NCH, bool POW2>
__device__ __forceinline__ void karatsuba_phase(const GemmArgs& g, uint32_t taddr, int s, int l,
                                                int row, bool row_ok, int col_base,
                                                const ModConst& mc, uint32_t (&st)[NCH * 8]) {
  int8_t* dst_base = nullptr;
  if (s == 1) dst_base = g.e_re + (int64_t)l * g.e_plane + (int64_t)row * g.e_ld + col_base;
  if (s == 2) dst_base = g.e_im + (int64_t)l * g.e_plane + (int64_t)row * g.e_ld + col_base;
  const uint32_t bias = uint32_t(mc.bias), bias_h = mc.bias_h, h = mc.h;
  // 8 chunks per thread: chunk c+1's TMEM load is in flight while chunk c is
  // reduced; 4 chunks (16 epilogue warps, register-limited): one buffer
  constexpr int NB = NCH >= 8 && CRTG_EPI_DB ? 2 : 1;
  uint32_t v[NB][32];
  tmem_ld32(taddr, v[0]);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    if (NB == 1 && c > 0) tmem_ld32(taddr + c * 32, v[0]);
    tmem_wait_ld();  // chunk c has landed (the only load in flight)
    if (NB == 2 && c + 1 < NCH) tmem_ld32(taddr + (c + 1) * 32, v[(c + 1) % NB]);
    const uint32_t (&cv)[32] = v[c % NB];
    uint32_t out[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      uint32_t a[4], b[4];
      const uint32_t sw = st[c * 8 + w];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t x = cv[4 * w + j];
        const uint32_t prev = __byte_perm(sw, 0, 0x4440 + j);  // byte j of the state
        if (s == 0) {
          a[j] = ep_red<POW2>(x + bias, mc);
        } else if (s == 1) {
          a[j] = ep_red<POW2>(prev - x + bias_h, mc) - h;
          b[j] = ep_red<POW2>(prev + x + bias, mc);
        } else {
          a[j] = ep_red<POW2>(x - prev + bias_h, mc) - h;
        }
      }
      if (s == 0) {
        st[c * 8 + w] = ep_pack_bytes(a[0], a[1], a[2], a[3]);
      } else {
        out[w] = ep_pack_bytes(a[0], a[1], a[2], a[3]);
        if (s == 1) st[c * 8 + w] = ep_pack_bytes(b[0], b[1], b[2], b[3]);
      }
    }
    if (s != 0 && row_ok) {
      uint4* d4 = reinterpret_cast<uint4*>(dst_base + c * 32);
      d4[0] = make_uint4(out[0], out[1], out[2], out[3]);
      d4[1] = make_uint4(out[4], out[5], out[6], out[7]);
    }
  }
}


// Split modulus (ModConst::nphase == 2, j^2 == -1 mod p):
//   phase 0 (X = U*U'):  xm  = (X + bias) mod p                  -> st
//   phase 1 (Y = V*V'):  ym  = (Y + bias) mod p
//                        e_R = (((xm + ym) inv2 + h) mod p) - h        -> out
//                        e_I = (((xm - ym + p) inv2j + h) mod p) - h   -> out
// X == CR + j CI and Y == CR - j CI (mod p), so e_R, e_I are the same residues
// the three Karatsuba products give.  Operands of the last two reductions are
// below 2p^2 + p < 2^17.
template <int NCH>
__device__ __forceinline__ void split_phase(const GemmArgs& g, uint32_t taddr, int s, int l,
                                            int row, bool row_ok, int col_base,
                                            const ModConst& mc, uint32_t (&st)[NCH * 8]) {
  int8_t* dre = g.e_re + (int64_t)l * g.e_plane + (int64_t)row * g.e_ld + col_base;
  int8_t* dim = g.e_im + (int64_t)l * g.e_plane + (int64_t)row * g.e_ld + col_base;
  const uint32_t bias = uint32_t(mc.bias), h = mc.h, p = uint32_t(mc.p);
  const uint32_t inv2 = mc.inv2, inv2j = mc.inv2j;
  constexpr int NB = NCH >= 8 && CRTG_EPI_DB ? 2 : 1;
  uint32_t v[NB][32];
  tmem_ld32(taddr, v[0]);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    if (NB == 1 && c > 0) tmem_ld32(taddr + c * 32, v[0]);
    tmem_wait_ld();
    if (NB == 2 && c + 1 < NCH) tmem_ld32(taddr + (c + 1) * 32, v[(c + 1) % NB]);
    const uint32_t (&cv)[32] = v[c % NB];
    uint32_t ore[8], oim[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      uint32_t a[4], b[4];
      const uint32_t sw = st[c * 8 + w];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t x = cv[4 * w + j];
        if (s == 0) {
          a[j] = ep_red<false>(x + bias, mc);
        } else {
          const uint32_t xm = __byte_perm(sw, 0, 0x4440 + j);
          const uint32_t ym = ep_red<false>(x + bias, mc);
          a[j] = ep_red<false>((xm + ym) * inv2 + h, mc) - h;
          b[j] = ep_red<false>((xm + p - ym) * inv2j + h, mc) - h;
        }
      }
      if (s == 0) {
        st[c * 8 + w] = ep_pack_bytes(a[0], a[1], a[2], a[3]);
      } else {
        ore[w] = ep_pack_bytes(a[0], a[1], a[2], a[3]);
        oim[w] = ep_pack_bytes(b[0], b[1], b[2], b[3]);
      }
    }
    if (s != 0 && row_ok) {
      uint4* r4 = reinterpret_cast<uint4*>(dre + c * 32);
      r4[0] = make_uint4(ore[0], ore[1], ore[2], ore[3]);
      r4[1] = make_uint4(ore[4], ore[5], ore[6], ore[7]);
      uint4* i4 = reinterpret_cast<uint4*>(dim + c * 32);
      i4[0] = make_uint4(oim[0], oim[1], oim[2], oim[3]);
      i4[1] = make_uint4(oim[4], oim[5], oim[6], oim[7]);
    }
  }
}

// The same two epilogues with the per-column state in SHARED memory (word i of
// this thread at st[i * stride]) so that the chunk loop is NOT unrolled: one
// phase is then ~250 instructions that stay in the instruction cache, where the
// fully unrolled register-state form is ~1000 straight-line instructions per
// phase and variant (10.5K in all) and short-K tiles, whose epilogue is not
// hidden behind long K loops, stalled on instruction fetch (ncu at 1024^3:
// `no_instruction` the top stall reason).  Used by the 128 x 256 kernel.
template <int NCH, bool POW2>
__device__ __forceinline__ void karatsuba_phase_sm(const GemmArgs& g, uint32_t taddr, int s, int l,
                                                   int row, bool row_ok, int col_base,
                                                   const ModConst& mc, uint32_t* st, int stride) {
  int8_t* dst_base = nullptr;
  if (s == 1) dst_base = g.e_re + (int64_t)l * g.e_plane + (int64_t)row * g.e_ld + col_base;
  if (s == 2) dst_base = g.e_im + (int64_t)l * g.e_plane + (int64_t)row * g.e_ld + col_base;
  const uint32_t bias = uint32_t(mc.bias), bias_h = mc.bias_h, h = mc.h;
#pragma unroll 1
  for (int c = 0; c < NCH; ++c) {
    uint32_t cv[32];
    tmem_ld32(taddr + c * 32, cv);
    uint32_t* sc = st + c * 8 * stride;
    uint32_t sw[8];
    if (s != 0) {
#pragma unroll
      for (int w = 0; w < 8; ++w) sw[w] = sc[w * stride];
    }
    tmem_wait_ld();
    uint32_t out[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      uint32_t a[4], b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t x = cv[4 * w + j];
        if (s == 0) {
          a[j] = ep_red<POW2>(x + bias, mc);
        } else {
          const uint32_t prev = __byte_perm(sw[w], 0, 0x4440 + j);
          if (s == 1) {
            a[j] = ep_red<POW2>(prev - x + bias_h, mc) - h;
            b[j] = ep_red<POW2>(prev + x + bias, mc);
          } else {
            a[j] = ep_red<POW2>(x - prev + bias_h, mc) - h;
          }
        }
      }
      if (s == 0) {
        sc[w * stride] = ep_pack_bytes(a[0], a[1], a[2], a[3]);
      } else {
        out[w] = ep_pack_bytes(a[0], a[1], a[2], a[3]);
        if (s == 1) sc[w * stride] = ep_pack_bytes(b[0], b[1], b[2], b[3]);
      }
    }
    if (s != 0 && row_ok) {
      uint4* d4 = reinterpret_cast<uint4*>(dst_base + c * 32);
      d4[0] = make_uint4(out[0], out[1], out[2], out[3]);
      d4[1] = make_uint4(out[4], out[5], out[6], out[7]);
    }
  }
}

template <int NCH>
__device__ __forceinline__ void split_phase_sm(const GemmArgs& g, uint32_t taddr, int s, int l,
                                               int row, bool row_ok, int col_base,
                                               const ModConst& mc, uint32_t* st, int stride) {
  int8_t* dre = g.e_re + (int64_t)l * g.e_plane + (int64_t)row * g.e_ld + col_base;
  int8_t* dim = g.e_im + (int64_t)l * g.e_plane + (int64_t)row * g.e_ld + col_base;
  const uint32_t bias = uint32_t(mc.bias), h = mc.h, p = uint32_t(mc.p);
  const uint32_t inv2 = mc.inv2, inv2j = mc.inv2j;
#pragma unroll 1
  for (int c = 0; c < NCH; ++c) {
    uint32_t cv[32];
    tmem_ld32(taddr + c * 32, cv);
    uint32_t* sc = st + c * 8 * stride;
    uint32_t sw[8];
    if (s != 0) {
#pragma unroll
      for (int w = 0; w < 8; ++w) sw[w] = sc[w * stride];
    }
    tmem_wait_ld();
    uint32_t ore[8], oim[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      uint32_t a[4], b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t x = cv[4 * w + j];
        if (s == 0) {
          a[j] = ep_red<false>(x + bias, mc);
        } else {
          const uint32_t xm = __byte_perm(sw[w], 0, 0x4440 + j);
          const uint32_t ym = ep_red<false>(x + bias, mc);
          a[j] = ep_red<false>((xm + ym) * inv2 + h, mc) - h;
          b[j] = ep_red<false>((xm + p - ym) * inv2j + h, mc) - h;
        }
      }
      if (s == 0) {
        sc[w * stride] = ep_pack_bytes(a[0], a[1], a[2], a[3]);
      } else {
        ore[w] = ep_pack_bytes(a[0], a[1], a[2], a[3]);
        oim[w] = ep_pack_bytes(b[0], b[1], b[2], b[3]);
      }
    }
    if (s != 0 && row_ok) {
      uint4* r4 = reinterpret_cast<uint4*>(dre + c * 32);
      r4[0] = make_uint4(ore[0], ore[1], ore[2], ore[3]);
      r4[1] = make_uint4(ore[4], ore[5], ore[6], ore[7]);
      uint4* i4 = reinterpret_cast<uint4*>(dim + c * 32);
      i4[0] = make_uint4(oim[0], oim[1], oim[2], oim[3]);
      i4[1] = make_uint4(oim[4], oim[5], oim[6], oim[7]);
    }
  }
}

// segments (K loops) of one output tile: the Karatsuba / split count of its
// modulus, or the launch's fixed count (RAW, REAL)
template <int MODE>
__device__ __forceinline__ int tile_segments(const GemmArgs& g, int l) {
  return MODE == EPI_KARATSUBA ? g.mc[l].nphase : g.nphase;
}

// NCH chunks of 32 columns per thread (8 = the whole 256-column tile, 4 = one
// half when two warps share a TMEM lane quarter).  The Karatsuba path double-
// buffers the TMEM loads: chunk c+1 is in flight while chunk c is reduced.
template <int MODE, int NCH>
__device__ __forceinline__ void epilogue_phase(const GemmArgs& g, uint32_t taddr, int s, int l,
                                               int row, bool row_ok, int col_base,
                                               const ModConst& mc, uint32_t (&st)[NCH * 8]) {
  if (MODE == EPI_RAW) {
#pragma unroll 1
    for (int c = 0; c < NCH; ++c) {
      uint32_t v[32];
      tmem_ld32(taddr + c * 32, v);
      tmem_wait_ld();
      if (row_ok) {
        int32_t* dst = g.raw + (int64_t)s * g.raw_plane + (int64_t)row * g.raw_ld + col_base + c * 32;
#pragma unroll
        for (int w = 0; w < 8; ++w)
          reinterpret_cast<uint4*>(dst)[w] = make_uint4(v[4 * w], v[4 * w + 1], v[4 * w + 2], v[4 * w + 3]);
      }
    }
    return;
  }
  if (MODE == EPI_REAL) {
    // one product per modulus (emulate_gemm_real -> crt_integer_gemm, emulate.py:103-132):
    // e = sym(D mod p).  |D| <= k*128^2 with k <= 2^17 can reach 2^31 only for p = 256
    // with every product (-128)^2; the int32 accumulator then wraps to INT32_MIN,
    // which is exactly the reference's ArithmeticError case (kernel.py:33-34).
    int8_t* dst = g.e_re + (int64_t)l * g.e_plane + (int64_t)row * g.e_ld + col_base;
    bool wrapped = false;
#pragma unroll 1
    for (int c = 0; c < NCH; ++c) {
      uint32_t v[32];
      tmem_ld32(taddr + c * 32, v);
      tmem_wait_ld();
      uint32_t out[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          wrapped |= v[4 * w + j] == 0x80000000u;
          o[j] = uint32_t(to_sym(mod_i32(int32_t(v[4 * w + j]), mc), mc));
        }
        out[w] = ep_pack4(o[0], o[1], o[2], o[3] & 0xFF);
      }
      if (row_ok) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
        d4[0] = make_uint4(out[0], out[1], out[2], out[3]);
        d4[1] = make_uint4(out[4], out[5], out[6], out[7]);
      }
    }
    if (wrapped && row_ok && g.overflow) atomicAdd(g.overflow, 1ull);
    return;
  }
#ifdef CRTG_EPI_NOP
  // timing experiment only (results wrong): drain TMEM, skip the math and stores
  if (MODE == EPI_KARATSUBA) {
    uint32_t v[32];
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      tmem_ld32(taddr + c * 32, v);
      tmem_wait_ld();
      acc ^= v[c];
    }
    st[0] ^= acc;
    return;
  }
#endif
  if (mc.nphase == 2)
    split_phase<NCH>(g, taddr, s, l, row, row_ok, col_base, mc, st);
  else if (mc.is_pow2)
    karatsuba_phase<NCH, true>(g, taddr, s, l, row, row_ok, col_base, mc, st);
  else
    karatsuba_phase<NCH, false>(g, taddr, s, l, row, row_ok, col_base, mc, st);
}

template <int NCH>
__device__ __forceinline__ void karatsuba_epilogue_sm(const GemmArgs& g, uint32_t taddr, int s,
                                                      int l, int row, bool row_ok, int col_base,
                                                      const ModConst& mc, uint32_t* st,
                                                      int stride) {
  if (mc.nphase == 2)
    split_phase_sm<NCH>(g, taddr, s, l, row, row_ok, col_base, mc, st, stride);
  else if (mc.is_pow2)
    karatsuba_phase_sm<NCH, true>(g, taddr, s, l, row, row_ok, col_base, mc, st, stride);
  else
    karatsuba_phase_sm<NCH, false>(g, taddr, s, l, row, row_ok, col_base, mc, st, stride);
}

}  // namespace crtg
