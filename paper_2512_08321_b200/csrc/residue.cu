// residue.cu — K2: scale + truncate + symmetric residues, written straight into the
// packed tcgen05 operand image; plus the accurate-mode bound operands (K1a).
//
// Replaces, per element and fused in one HBM pass:
//   quantize           scaling.py:277-293   a' = trunc(ldexp(a, e))
//   residue_decompose  crt.py:199-218       r_l = sym(a' mod p_l) for every modulus
//   Karatsuba sums     kernel.py:101-103    s_l = sym(r_re + r_im mod p_l)
//   _bound_matrices    scaling.py:216-226   ceil(|x| 2^bar): their sum and difference
// Integer residues are exact for |a'| < 2^90: a' = M * 2^s with a 53-bit integer
// significand M; M mod p is folded on 32-bit lanes through 2^32 mod p and
// 2^16 mod p, then multiplied by 2^s mod p.  The congruence class equals the
// reference's 2^31 split (crt.py:123-133), so the symmetric residue is identical.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "residue_math.cuh"

namespace crtg {

namespace {

constexpr int kTileRows = 32;  // operand rows per CTA
constexpr int kThreads = 256;  // 32 rows x 8 sixteen-byte K chunks

// element (row, h) of an operand: complex interleaved or real (im = 0)
template <typename T, bool REAL>
__device__ __forceinline__ void load_c(const T* p, double& re, double& im) {
  if constexpr (REAL) {
    re = double(*p);
    im = 0.0;
  } else if constexpr (sizeof(T) == 8) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    re = v.x;
    im = v.y;
  } else {
    const float2 v = *reinterpret_cast<const float2*>(p);
    re = double(v.x);
    im = double(v.y);
  }
}

template <typename T, int OPERAND, int KIND, bool REAL>
__global__ void __launch_bounds__(kThreads) k_pack(const T* __restrict__ X, int64_t ldx, int rows,
                                                  int kdim, int64_t col0,
                                                  const int32_t* __restrict__ exps,
                                                  const __grid_constant__ DevConsts dc,
                                                  int8_t* __restrict__ out, int64_t plane_bytes,
                                                  int64_t rb_count,
                                                  unsigned long long* __restrict__ overflow) {
  pdl_begin();
  __shared__ __align__(16) uint8_t stage[3][kTileRows * 128];
  const int kb = blockIdx.x;
  const int r0 = blockIdx.y * kTileRows;
  // thread -> (row r, 16-byte K chunk c)
  int r, c;
  if (OPERAND == 0) {  // rows of A: 8 lanes sweep one row's 128 K bytes
    r = threadIdx.x >> 3;
    c = threadIdx.x & 7;
  } else {  // columns of B: a warp covers 32 consecutive columns at one K index
    r = threadIdx.x & 31;
    c = threadIdx.x >> 5;
  }
  const int row = r0 + r;
  const int h0 = kb * 128 + c * 16;
  const bool row_ok = row < rows;
  const int e = row_ok ? exps[row] : 0;

  double re[16], im[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int h = h0 + t;
    re[t] = 0.0;
    im[t] = 0.0;
    if (row_ok && h < kdim) {
      const T* p = (OPERAND == 0) ? X + (REAL ? 1 : 2) * (int64_t(row) * ldx + h)
                                  : X + (REAL ? 1 : 2) * (int64_t(h) * ldx + col0 + row);
      load_c<T, REAL>(p, re[t], im[t]);
    }
  }

  // swizzled position of this thread's 16-byte chunk inside the 4 KiB stage tile
  const int soff = (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4);
  // the CTA's 32 rows are one contiguous 4 KiB run of the packed plane
  const int64_t goff = (int64_t(kb) * rb_count + (r0 >> 7)) * kBlockBytes + (r0 & 127) * 128;

  {
    // bound operands from R = ceil(|re| 2^bar), I = ceil(|im| 2^bar) in [0, 64]:
    // plane 0 the sum R + I in [0, 128] (an unsigned byte), plane 2 the
    // difference R - I in [-64, 64]; plane 1 is not used (the bound GEMM
    // needs the two products (R+I)(R'+I') and (R-I)(R'-I'), gemm_tc.cu)
    uint32_t w[2][4] = {};
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int vr = int(ceil(ldexp_rn(fabs(re[t]), e)));
      const int vi = int(ceil(ldexp_rn(fabs(im[t]), e)));
      w[0][t >> 2] |= uint32_t((vr + vi) & 0xFF) << (8 * (t & 3));
      w[1][t >> 2] |= uint32_t((vr - vi) & 0xFF) << (8 * (t & 3));
    }
#pragma unroll
    for (int q = 0; q < 2; ++q)
      *reinterpret_cast<uint4*>(&stage[q][soff]) = make_uint4(w[q][0], w[q][1], w[q][2], w[q][3]);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q)
      reinterpret_cast<uint4*>(out + 2 * q * plane_bytes + goff)[threadIdx.x] =
          reinterpret_cast<const uint4*>(stage[q])[threadIdx.x];
  }
}

// ---------------------------------------------------------------------------
// Residue kernel.  CTA tile = 16 operand rows x 128 K (one packed K block);
// thread = 8 consecutive K of one row (16 real values).  Each value is
// decomposed once into 16-bit limbs; per modulus a value then costs two (or
// three) dp2a and one magic-number reduction.  A rows store straight to the
// packed plane; B columns go through a 6 KiB smem stage so every global store
// is a coalesced 16-byte write of a contiguous 2 KiB run of the packed plane.
//
// Stored representative.  SYM = true writes the reference's symmetric residue
// (crt.py:136-151; the crtg_residues parity hook, and the real path for
// k > 16384, whose int32 overflow check depends on it).  SYM = false (the
// complex pipeline) writes, for k <= 16384 (DevConsts::uns), the unsigned
// residue t = a' mod p in [0, p) -- the GEMM then runs u8 x u8 products, which
// draw less power, and (p - 1)^2 k < 2^30 keeps every sum inside the
// epilogue's single biased reduction -- and for longer K the signed
// (a' + 128 mod p) - 128 in [-128, p - 129] (byte t ^ 0x80, |value| <= 128
// keeps k 128^2 <= 2^30 up to k = 2^16).  Both are congruent to a', so every
// modular product and e-plane is unchanged.
// ---------------------------------------------------------------------------
constexpr int kResRows = 16;
#ifndef CRTG_RES_MINB
#define CRTG_RES_MINB 4  // CTAs per SM the register residue kernel is built for
#endif
#ifndef CRTG_RES_UNROLL
#define CRTG_RES_UNROLL 1
#endif

// split modulus: t_U = (re + j im + off) mod p (V = 1: p - j) straight from the
// limbs of both values (u < 2 * 6 * 2^16 * 255 + p < 2^28, one reduction)
template <int FORM>
__device__ __forceinline__ uint32_t res_uv(const Val3& vr, const Val3& vi, const ResConst& c,
                                           int V) {
  const uint32_t w = V ? c.vw0123 : c.uw0123;
  uint32_t u;
  if (FORM == 3) {
    u = dp2a_lo(vi.w0, w, V ? c.kvw : c.kuw);
    u = dp2a_hi(vi.w1, w, u);
    u = dp2a_lo(vi.w2, V ? c.vw45 : c.uw45, u);
    u = dp2a_lo(vr.w0, c.dw0123, u);
    u = dp2a_hi(vr.w1, c.dw0123, u);
    u = dp2a_lo(vr.w2, c.dw45, u);
  } else if (FORM == 2) {
    u = dp2a_hi(vi.w1, w, dp2a_lo(vi.w0, w, V ? c.kv63 : c.ku63));
    u = dp2a_hi(vr.w1, c.dw0123, dp2a_lo(vr.w0, c.dw0123, u));
  } else {
    u = dp2a_lo(vr.w0, c.dw0123, dp2a_lo(vi.w0, w, V ? c.kv31 : c.ku31));
  }
  return mod_small(u, c);
}

// 4 values t_i in [0,p) -> packed bytes: SYM, the symmetric t_i - off; else
// the bytes of t_i xor `off` (a per-byte mask: 0x80 -> signed t - 128, 0 -> t)
template <bool SYM>
__device__ __forceinline__ uint32_t pack_t(uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                           uint32_t off) {
  if (SYM) {
    const uint32_t lo = __byte_perm(a - off, b - off, 0x0040);
    const uint32_t hi = __byte_perm(c - off, d - off, 0x0040);
    return __byte_perm(lo, hi, 0x5410);
  }
  // off = 128: (t - 128) mod 256 == t ^ 0x80 for t < 256 (signed bytes); off = 0:
  // t itself (unsigned bytes, mask 0)
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410) ^ off;
}

// planes of one modulus: [re, im, re+im] (Karatsuba), or [U, V] = [re + j im,
// re - j im] for a split modulus (c.split; w[2] is then not written)
template <int FORM, bool SYM>
__device__ __forceinline__ void residue_words(const Val3 (&re)[8], const Val3 (&im)[8],
                                              const ResConst& c, uint32_t (&w)[3][2]) {
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    if (c.split) {
      // U = re + j im, V = re - j im, each one reduction of a limb sum over both
      // values (no separate re / im residues)
      uint32_t tu[4], tv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        tu[j] = res_uv<FORM>(re[4 * half + j], im[4 * half + j], c, 0);
        tv[j] = res_uv<FORM>(re[4 * half + j], im[4 * half + j], c, 1);
      }
      w[0][half] = pack_t<SYM>(tu[0], tu[1], tu[2], tu[3], SYM ? c.off : c.xor_mask);
      w[1][half] = pack_t<SYM>(tv[0], tv[1], tv[2], tv[3], SYM ? c.off : c.xor_mask);
    } else {
      uint32_t tr[4], ti[4], ts[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        tr[j] = res_t<FORM>(re[4 * half + j], c);
        ti[j] = res_t<FORM>(im[4 * half + j], c);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        // (re + im) + off = (tr - off) + (ti - off) + off  (mod p); x < 3p, so two
        // conditional subtractions on the ALU pipe (umin(x, x - p) wraps below p)
        // instead of a magic reduction on the busier FMA-heavy pipe
        const uint32_t x = tr[j] + ti[j] + c.sum_k;
        const uint32_t y = min(x, x + c.neg_p);
        ts[j] = min(y, y + c.neg_p);
      }
      w[0][half] = pack_t<SYM>(tr[0], tr[1], tr[2], tr[3], SYM ? c.off : c.xor_mask);
      w[1][half] = pack_t<SYM>(ti[0], ti[1], ti[2], ti[3], SYM ? c.off : c.xor_mask);
      w[2][half] = pack_t<SYM>(ts[0], ts[1], ts[2], ts[3], SYM ? c.off : c.xor_mask);
    }
  }
}

// the per-modulus loop of one tile (complex operands)
template <int OPERAND, int FORM, bool SYM, bool MSPLIT = false>
__device__ __forceinline__ void store_moduli(const Val3 (&vr)[8], const Val3 (&vi)[8],
                                             const DevConsts& dc, const ResConst* rcs,
                                             int8_t* __restrict__ out, int64_t plane_bytes,
                                             int64_t goff, int soff, int cq, int cs,
                                             uint8_t (*stage)[kResRows * 128]) {
  // large launches: unrolled over the modulus index, so each modulus's
  // constants become immediate constant-bank operands instead of per-iteration
  // LDC loads.  Small launches (MSPLIT): blockIdx.y of gridDim.y CTAs share a
  // tile, each taking the moduli l == blockIdx.y (mod gridDim.y)
  int it = 0;  // moduli processed by this CTA (smem stage buffer parity)
  auto one = [&](int l) {
    const ResConst c = rcs[l];
    uint32_t w[3][2];
    residue_words<FORM, SYM>(vr, vi, c, w);
    if (OPERAND == 0) {
      // A rows: the 16 lanes of a row cover its whole 128-byte line of the plane,
      // so a warp store is already two full lines -- no staging needed
      int8_t* base = out + int64_t(3 * l) * plane_bytes + goff + soff;
      *reinterpret_cast<uint2*>(base) = make_uint2(w[0][0], w[0][1]);
      *reinterpret_cast<uint2*>(base + plane_bytes) = make_uint2(w[1][0], w[1][1]);
      if (!c.split)
        *reinterpret_cast<uint2*>(base + 2 * plane_bytes) = make_uint2(w[2][0], w[2][1]);
    } else {
      // double-buffered stage: modulus l uses buffer l & 1, so one barrier per
      // modulus suffices (a thread writing buffer b again for l + 2 has passed
      // the barrier of l + 1, which every thread reaches only after copying l out)
      uint8_t (*sb)[kResRows * 128] = stage + 3 * ((MSPLIT ? it++ : l) & 1);
      *reinterpret_cast<uint2*>(&sb[0][soff]) = make_uint2(w[0][0], w[0][1]);
      *reinterpret_cast<uint2*>(&sb[1][soff]) = make_uint2(w[1][0], w[1][1]);
      if (!c.split) *reinterpret_cast<uint2*>(&sb[2][soff]) = make_uint2(w[2][0], w[2][1]);
      __syncthreads();
      int8_t* base = out + int64_t(3 * l) * plane_bytes + goff;
      reinterpret_cast<uint4*>(base + cq * plane_bytes)[cs] =
          reinterpret_cast<const uint4*>(sb[cq])[cs];
      if (cq == 0 && !c.split)
        reinterpret_cast<uint4*>(base + 2 * plane_bytes)[cs] =
            reinterpret_cast<const uint4*>(sb[2])[cs];
    }
  };
  if constexpr (MSPLIT) {
    // small operands (and the moduli-split launches): a rolled loop, constants
    // by uniform loads -- the unrolled form is ~20K instructions and latency-bound
    // small launches stalled on instruction fetch (ncu at 1024^2: no_instruction
    // the top stall); large launches keep the unrolled loop (rolled: A 5.4 -> 5.8 ms)
#pragma unroll 1
    for (int l = int(blockIdx.y); l < dc.n; l += int(gridDim.y)) one(l);
  } else {
#if CRTG_RES_UNROLL
#pragma unroll
    for (int l = 0; l < CRTG_MAX_MODULI; ++l) {
      if (l >= dc.n) break;
      one(l);
    }
#else
    for (int l = 0; l < dc.n; ++l) one(l);
#endif
  }
  if (OPERAND != 0) __syncthreads();  // the next tile reuses the buffers
}

template <int FORM>
__device__ __forceinline__ uint32_t pack_real(const Val3 (&v)[8], int i0, const ResConst& c) {
  return pack_t<true>(res_t<FORM>(v[i0], c), res_t<FORM>(v[i0 + 1], c), res_t<FORM>(v[i0 + 2], c),
                      res_t<FORM>(v[i0 + 3], c), c.off);
}

// MS: the moduli are split over gridDim.y CTAs per tile (small operands); a
// separate instantiation so the large-operand kernel does not carry the extra
// register pressure
template <typename T, int OPERAND, bool REAL, bool SYM, bool MS = false>
__global__ void __launch_bounds__(256, CRTG_RES_MINB) k_residues(const T* __restrict__ X, int64_t ldx, int rows,
                                                  int kdim, int64_t col0,
                                                  const int32_t* __restrict__ exps,
                                                  const __grid_constant__ DevConsts dc,
                                                  int8_t* __restrict__ out, int64_t plane_bytes,
                                                  int64_t rb_count,
                                                  unsigned long long* __restrict__ overflow,
                                                  int n_kb, int n_rt, int row_base) {
  pdl_begin();
  // B of the complex pipeline (TIN): the tile's 128 K x 16 columns of B are
  // transposed on the way IN (coalesced 256-byte rows into a swizzled shared
  // tile, then each thread reads its column's 8 consecutive K), so its planes
  // are stored like A's -- straight from registers, whole 128-byte lines, no
  // per-modulus barrier.  Other B launches stage the planes on the way out.
  constexpr bool TIN = OPERAND == 1 && !REAL;
  constexpr int kStageBytes = TIN ? 128 * 16 * 2 * int(sizeof(T)) : 6 * kResRows * 128;
  __shared__ __align__(16) uint8_t smem_buf[kStageBytes];
  uint8_t (*stage)[kResRows * 128] = reinterpret_cast<uint8_t (*)[kResRows * 128]>(smem_buf);
  // representative of the stored residues: the symmetric (rc) or the pipeline's
  // unsigned / 128-offset (rx) tables
  const ResConst* rcs = SYM ? dc.rc : dc.rx;
  // grid-stride over (K block, 16-row tile): a full grid when launched alone, one
  // CTA per SM when it runs beside the persistent GEMM (side stream)
  for (int tile = blockIdx.x; tile < n_kb * n_rt; tile += gridDim.x) {
  // A: consecutive tiles walk along a row (contiguous K); B: along the columns
  const int kb = OPERAND == 0 ? tile % n_kb : tile / n_rt;
  const int r0 = (OPERAND == 0 ? tile / n_kb : tile % n_rt) * kResRows;
  int r, seg;  // row within the tile, 8-element K segment (0..15)
  if (OPERAND == 0 || TIN) {
    r = threadIdx.x >> 4;
    seg = threadIdx.x & 15;
  } else {
    r = threadIdx.x & 15;
    seg = threadIdx.x >> 4;
  }
  const int row = r0 + r;
  const int h0 = kb * 128 + seg * 8;
  const bool row_ok = row < rows;
  const int e = row_ok ? exps[row] : 0;
  if constexpr (TIN) {
    // rows h of the tile: 16 columns x (re, im) = 16 x 2 sizeof(T) bytes, slot of
    // column c at c ^ (h / 8) (the reads below are then bank-conflict free)
    constexpr int kEl = 2 * int(sizeof(T));
    __syncthreads();  // the previous tile's reads are done
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = i * 256 + int(threadIdx.x);
      const int hl = idx >> 4, c = idx & 15;
      const int h = kb * 128 + hl;
      const int col = r0 + c;
      uint8_t* dst = smem_buf + hl * (16 * kEl) + ((c ^ ((hl >> 3) & 15)) * kEl);
      if (h < kdim && col < rows) {
        if constexpr (sizeof(T) == 8)
          *reinterpret_cast<double2*>(dst) =
              *reinterpret_cast<const double2*>(X + 2 * (int64_t(h) * ldx + col0 + col));
        else
          *reinterpret_cast<float2*>(dst) =
              *reinterpret_cast<const float2*>(X + 2 * (int64_t(h) * ldx + col0 + col));
      } else {
        if constexpr (sizeof(T) == 8)
          *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
        else
          *reinterpret_cast<float2*>(dst) = make_float2(0.f, 0.f);
      }
    }
    __syncthreads();
  }
  // 2^e for e in [-1023, 1023] is representable (2^-1023 subnormal): one
  // correctly rounded multiply == np.ldexp
  const double scale = __longlong_as_double(e >= -1022 ? int64_t(e + 1023) << 52
                                                       : int64_t(1) << (e + 1074));

  // q = x * 2^e exactly (quantize, scaling.py:277-293); a' = trunc(q)
  double qr[8], qi[8];
  int bad = 0;
  bool huge = false, medium = false;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int h = h0 + t;
    double re = 0.0, im = 0.0;
    if constexpr (TIN) {
      constexpr int kEl = 2 * int(sizeof(T));
      const int hl = seg * 8 + t;
      load_c<T, false>(reinterpret_cast<const T*>(smem_buf + hl * (16 * kEl) +
                                                  ((r ^ seg) * kEl)), re, im);
    } else if (row_ok && h < kdim) {
      const T* p = (OPERAND == 0) ? X + (REAL ? 1 : 2) * (int64_t(row) * ldx + h)
                                  : X + (REAL ? 1 : 2) * (int64_t(h) * ldx + col0 + row);
      load_c<T, REAL>(p, re, im);
    }
    qr[t] = __dmul_rn(re, scale);
    qi[t] = __dmul_rn(im, scale);
    if (!(fabs(qr[t]) < 0x1p90)) { bad = 1; qr[t] = 0.0; }
    if (!(fabs(qi[t]) < 0x1p90)) { bad = 1; qi[t] = 0.0; }
    const double mq = fmax(fabs(qr[t]), fabs(qi[t]));
    huge |= mq >= 0x1p63;
    medium |= mq >= 0x1p31;
  }
  // warp-uniform representation (a wider form is valid for every value): a
  // warp that mixed forms would execute several per-modulus paths
  huge = __any_sync(0xffffffffu, huge);
  medium = __any_sync(0xffffffffu, medium);
  Val3 vr[8], vi[8];
  if (!medium) {
    // |a'| < 2^31 (single precision at N <= 8): a' + 2^31 in one word
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      vr[t] = {uint32_t(__double2int_rz(qr[t])) ^ 0x80000000u, 0u, 0u};
      vi[t] = {uint32_t(__double2int_rz(qi[t])) ^ 0x80000000u, 0u, 0u};
    }
  } else if (!huge) {
    // |a'| < 2^63: one truncating conversion gives a' as int64; a' + 2^63 flips the sign bit
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const long long ar = __double2ll_rz(qr[t]), ai = __double2ll_rz(qi[t]);
      vr[t] = {uint32_t(ar), uint32_t(uint64_t(ar) >> 32) ^ 0x80000000u, 0u};
      vi[t] = {uint32_t(ai), uint32_t(uint64_t(ai) >> 32) ^ 0x80000000u, 0u};
    }
  } else {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      vr[t] = split_wide(trunc(qr[t]));
      vi[t] = split_wide(trunc(qi[t]));
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(overflow, 1ull);

  // swizzled byte offset of this thread's 8 bytes inside the 2 KiB stage tile
  const int chunk = seg >> 1;
  const int soff = (r >> 3) * 1024 + (r & 7) * 128 + ((chunk ^ (r & 7)) << 4) + (seg & 1) * 8;
  // the tile's 16 rows form one contiguous 2 KiB run of each packed plane
  const int gr0 = r0 + row_base;  // row of this tile inside the packed plane
  const int64_t goff = (int64_t(kb) * rb_count + (gr0 >> 7)) * kBlockBytes + (gr0 & 127) * 128;
  const int cq = threadIdx.x >> 7;       // copy-out: plane handled by this half
  const int cs = threadIdx.x & 127;      // 16-byte slot within the 2 KiB run

  if constexpr (REAL) {
    // one plane per modulus (emulate_gemm_real: no imaginary part / Karatsuba sum)
    for (int l = 0; l < dc.n; ++l) {
      if (MS && l % int(gridDim.y) != int(blockIdx.y)) continue;
      // symmetric residues, or (dc.uns, k <= 16384) t in [0, p): rx has off = 0,
      // so pack_t<true> stores the bytes of t
      const ResConst c = dc.uns ? dc.rx[l] : dc.rc[l];
      uint32_t w0, w1;
      if (huge) {
        w0 = pack_real<3>(vr, 0, c);
        w1 = pack_real<3>(vr, 4, c);
      } else if (medium) {
        w0 = pack_real<2>(vr, 0, c);
        w1 = pack_real<2>(vr, 4, c);
      } else {
        w0 = pack_real<1>(vr, 0, c);
        w1 = pack_real<1>(vr, 4, c);
      }
      if (OPERAND == 0) {
        *reinterpret_cast<uint2*>(out + int64_t(l) * plane_bytes + goff + soff) = make_uint2(w0, w1);
      } else {
        *reinterpret_cast<uint2*>(&stage[0][soff]) = make_uint2(w0, w1);
        __syncthreads();
        if (cq == 0)
          reinterpret_cast<uint4*>(out + int64_t(l) * plane_bytes + goff)[cs] =
              reinterpret_cast<const uint4*>(stage[0])[cs];
        __syncthreads();
      }
    }
  } else if (huge) {  // MS: this CTA's share of the moduli
    store_moduli<TIN ? 0 : OPERAND, 3, SYM, MS>(vr, vi, dc, rcs, out, plane_bytes, goff, soff, cq,
                                                cs, stage);
  } else if (medium) {
    store_moduli<TIN ? 0 : OPERAND, 2, SYM, MS>(vr, vi, dc, rcs, out, plane_bytes, goff, soff, cq,
                                                cs, stage);
  } else {
    store_moduli<TIN ? 0 : OPERAND, 1, SYM, MS>(vr, vi, dc, rcs, out, plane_bytes, goff, soff, cq,
                                                cs, stage);
  }
  }  // tile loop
}

// plain int8 -> packed plane (test hooks); one thread per 16-byte chunk
__global__ void k_pack_i8(const int8_t* __restrict__ X, int trans, int64_t rows, int64_t kdim,
                          int64_t kpad, int8_t* __restrict__ out, int64_t rb_count,
                          int64_t total_chunks) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= total_chunks) return;
  const int64_t chunks_per_row = kpad / 16;
  const int64_t r = t / chunks_per_row;
  const int64_t c = t % chunks_per_row;
  uint32_t w[4] = {0, 0, 0, 0};
  for (int b = 0; b < 16; ++b) {
    const int64_t h = c * 16 + b;
    int8_t v = 0;
    if (r < rows && h < kdim) v = trans ? X[h * rows + r] : X[r * kdim + h];
    w[b >> 2] |= uint32_t(uint8_t(v)) << (8 * (b & 3));
  }
  *reinterpret_cast<uint4*>(out + pack_offset(r, c * 16, rb_count)) = make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void k_unpack_i8(const int8_t* __restrict__ packed, int64_t rows, int64_t kdim,
                            int64_t rb_count, int8_t* __restrict__ out) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * kdim) return;
  const int64_t r = t / kdim, h = t % kdim;
  out[t] = packed[pack_offset(r, h, rb_count)];
}

template <typename T, int OP, int KIND, bool REAL>
void launch_one(const void* X, int64_t ldx, int64_t rows, int64_t kdim, int64_t col0,
                const int32_t* exps, const DevConsts& dc, int8_t* out, int64_t plane_bytes,
                int64_t rb_count, unsigned long long* overflow, cudaStream_t s, int max_ctas,
                int64_t row_base, int64_t fill_rows) {
  if constexpr (KIND == PACK_RESIDUE) {
    // tiles cover the plane from row_base up to fill_rows (the zero padding of
    // the last chunk included)
    const int64_t extent = fill_rows > 0 ? fill_rows : rb_count * 128 - row_base;
    const int n_kb = int((kdim + 127) / 128), n_rt = int((extent + kResRows - 1) / kResRows);
    const int64_t tiles = int64_t(n_kb) * n_rt;
    const unsigned grid1 = unsigned(max_ctas > 0 && max_ctas < tiles ? max_ctas : tiles);
    // few tiles (small operands): split the moduli over gridDim.y CTAs per tile
    static int nsm_r = [] {
      int d = 0, v = 148;
      cudaGetDevice(&d);
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
      return v;
    }();
    const int msplit = (max_ctas > 0 || tiles >= 2 * nsm_r)
                           ? 1
                           : int(std::min<int64_t>(dc.n, (2 * nsm_r + tiles - 1) / tiles));
    // small launches take the rolled-loop instantiation (MS): up to 2048^2
    // operands (<= 4096 tiles; 1024^3 N=14 136 vs 151 us per product, 2048^3
    // -3%, 4096^3 and up neutral to slower; CRTG_RES_ROLLED_TILES overrides)
    static const int64_t rolled_tiles = [] {
      const char* v = std::getenv("CRTG_RES_ROLLED_TILES");
      return v && *v ? int64_t(std::atoll(v)) : int64_t(4096);
    }();
    const bool ms = msplit > 1 || (max_ctas == 0 && tiles <= rolled_tiles);
    const dim3 grid(grid1, unsigned(std::max(1, msplit)));
    // symmetric residues for the real path and the parity hook (dc.sym), the
    // unsigned (k <= 16384) or 128-offset representative in the complex pipeline
#define CRTG_RES_LAUNCH(R, S, M)                                                              \
  launch_k(k_residues<T, OP, R, S, M>, grid, 256, 0, s, static_cast<const T*>(X), ldx, int(rows),      \
                                                  int(kdim), col0, exps, dc, out, plane_bytes,   \
                                                  rb_count, overflow, n_kb, n_rt, int(row_base))
    if (REAL || dc.sym) {
      if (ms) CRTG_RES_LAUNCH(REAL, true, true); else CRTG_RES_LAUNCH(REAL, true, false);
    } else if (ms) {
      CRTG_RES_LAUNCH(false, false, true);
    } else {
      CRTG_RES_LAUNCH(false, false, false);
    }
#undef CRTG_RES_LAUNCH
  } else {
  // cover every padded row of the plane so the GEMM reads zeros there
  dim3 grid(unsigned((kdim + 127) / 128), unsigned(rb_count * 128 / kTileRows));
  launch_k(k_pack<T, OP, KIND, REAL>, grid, kThreads, 0, s, static_cast<const T*>(X), ldx, int(rows),
                                                int(kdim), col0, exps, dc, out, plane_bytes,
                                                rb_count, overflow);
  }
}

}  // namespace

int launch_pack(int elem, int operand, int kind, const void* X, int64_t ldx, int64_t rows,
                int64_t kdim, int64_t col0, const int32_t* exps, const DevConsts& dc,
                int8_t* out, int64_t plane_bytes, int64_t rb_count,
                unsigned long long* overflow, cudaStream_t s, int max_ctas, int64_t row_base,
                int64_t fill_rows) {
  if (rows <= 0 || kdim <= 0) return 0;
#define CRTG_PACK(T, OP, KIND, R) \
  launch_one<T, OP, KIND, R>(X, ldx, rows, kdim, col0, exps, dc, out, plane_bytes, rb_count, \
                             overflow, s, max_ctas, row_base, fill_rows)
#define CRTG_PACK_KIND(T, OP, R) \
  if (kind == PACK_BARS) CRTG_PACK(T, OP, PACK_BARS, R); else CRTG_PACK(T, OP, PACK_RESIDUE, R);
#define CRTG_PACK_OP(T, R) \
  if (operand == 0) { CRTG_PACK_KIND(T, 0, R) } else { CRTG_PACK_KIND(T, 1, R) }
  switch (elem) {
    case E_C128: CRTG_PACK_OP(double, false) break;
    case E_C64: CRTG_PACK_OP(float, false) break;
    case E_F64: CRTG_PACK_OP(double, true) break;
    default: CRTG_PACK_OP(float, true) break;
  }
#undef CRTG_PACK_OP
#undef CRTG_PACK_KIND
#undef CRTG_PACK
  return launched(1);
}

int launch_pack_i8(const int8_t* X, int trans, int64_t rows, int64_t kdim, int8_t* out,
                   int64_t rb_count, cudaStream_t s) {
  const int64_t kpad = round_up(kdim, 128);
  const int64_t rpad = rb_count * 128;
  const int64_t total = rpad * (kpad / 16);
  if (total <= 0) return 0;
  k_pack_i8<<<unsigned((total + 255) / 256), 256, 0, s>>>(X, trans, rows, kdim, kpad, out, rb_count,
                                                          total);
  return launched(1);
}

int launch_unpack_i8(const int8_t* packed, int64_t rows, int64_t kdim, int64_t rb_count,
                     int8_t* out, cudaStream_t s) {
  const int64_t total = rows * kdim;
  if (total <= 0) return 0;
  k_unpack_i8<<<unsigned((total + 255) / 256), 256, 0, s>>>(packed, rows, kdim, rb_count, out);
  return launched(1);
}

// ---------------------------------------------------------------------------
// stage-level API (stages.py): symmetric residues of integer-valued arrays for
// every modulus (residue_decompose crt.py:199-218, symmetric_mod_int :136-151)
// ---------------------------------------------------------------------------
namespace {
__device__ __forceinline__ int8_t sym_of(int64_t r, int p) {
  // r in [0, p): the symmetric representative x - p * floor((2x + p) / 2p)
  return int8_t(r - p * ((2 * r + p) / (2 * p)));
}

// kind & 3: 0 float64, 1 int64, 2 int32; kind & 8 (strict, residue_decompose):
// float64 must be integer-valued, int64 below 2^61.  float64 is always checked
// finite and below 2^90.  flags: [0] non-finite, [1] |x| >= bound, [2] not
// integer-valued.  x = hi * 2^31 + lo with hi = floor(x / 2^31) (crt.py:123-133:
// a non-integer float keeps trunc(lo), as the reference's astype(int64) does).
__global__ void k_sym_mod(int kind, const void* __restrict__ x, int64_t count,
                          SymModuli mods, int8_t* __restrict__ out,
                          unsigned long long* flags) {
  const bool strict = (kind & 8) != 0;
  kind &= 3;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t hi = 0, lo = 0;  // x = hi * 2^31 + lo, 0 <= lo < 2^31
    if (kind == 0) {
      const double v = static_cast<const double*>(x)[i];
      if (!isfinite(v)) { atomicAdd(flags, 1ull); continue; }
      if (fabs(v) >= 0x1p90) { atomicAdd(flags + 1, 1ull); continue; }
      if (strict && trunc(v) != v) { atomicAdd(flags + 2, 1ull); continue; }
      const double h = floor(v * 0x1p-31);
      hi = int64_t(h);
      lo = int64_t(v - h * 0x1p31);
    } else {
      const int64_t v = kind == 1 ? static_cast<const int64_t*>(x)[i]
                                  : int64_t(static_cast<const int32_t*>(x)[i]);
      if (strict && kind == 1 && (v >= (int64_t(1) << 61) || v <= -(int64_t(1) << 61))) {
        atomicAdd(flags + 1, 1ull);
        continue;
      }
      hi = v >> 31;  // arithmetic shift: floor(v / 2^31)
      lo = v - hi * (int64_t(1) << 31);
    }
    for (int l = 0; l < mods.n; ++l) {
      const int p = mods.p[l];
      const int64_t hm = ((hi % p) + p) % p;
      const int64_t r = (hm * ((int64_t(1) << 31) % p) + lo) % p;
      out[int64_t(l) * count + i] = sym_of(r, p);
    }
  }
}
}  // namespace

int launch_sym_mod(int kind, const void* x, int64_t count, const SymModuli& mods, int8_t* out,
                   unsigned long long* flags, cudaStream_t s) {
  if (count <= 0) return 0;
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 16);
  k_sym_mod<<<unsigned(blocks), 256, 0, s>>>(kind, x, count, mods, out, flags);
  return launched(1);
}

}  // namespace crtg
