// common.cuh — shared device helpers for the sm_100a Ozaki-II / CRT kernels.
//
// Operand tile image ("packed") layout used by every producer kernel and read by
// the tcgen05 GEMM with plain 1-D bulk copies (TMA engine, no tensor map):
//   one plane  = residue (or bound) matrix of R rows x K bytes, K-major,
//                R padded to 256, K padded to 128;
//   block      = 128 rows x 128 K-bytes = 16 KiB, stored as the exact
//                SWIZZLE_128B shared-memory image UMMA expects
//                (8-row groups of 1 KiB; 16-byte chunk c of row r lands at chunk
//                c ^ (r & 7));
//   block order = [kb][rb] so one 128-byte K step of a 256-row B tile is one
//                contiguous 32 KiB copy.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/crtg.h"

namespace crtg {

// kernel-launch accounting for crtg_launch_count (defined in api.cu); every
// launcher reports the kernels it enqueued
void note_launches(int n);
inline int launched(int n) {
  note_launches(n);
  return int(cudaGetLastError());
}

// Programmatic dependent launch.  The pipeline kernels (statistics, residues,
// GEMM, CRT) are launched with launch_k, which lets the next kernel of the
// stream be scheduled while this one still runs; every such kernel starts with
// pdl_begin(): griddepcontrol.wait returns once the grids it depends on have
// completed and their memory is visible (a no-op for a normal launch), so no
// global load or store of the kernel can overtake its predecessor, and the
// trigger then lets its own successor launch and park at that wait.  What is
// saved is the launch latency between dependent kernels (small products run
// ~6 of them back to back).  CRTG_PDL=0 launches normally.
bool pdl_enabled();

template <typename... K, typename... A>
inline cudaError_t launch_k(void (*kern)(K...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  unsigned na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  // carry the stream's priority into the launch (and so into a captured graph
  // node: the small-product graphs run B's longer chain on a high-priority fork)
  int prio = 0;
  if (cudaStreamGetPriority(s, &prio) == cudaSuccess && prio != 0) {
    attr[na].id = cudaLaunchAttributePriority;
    attr[na++].val.priority = prio;
  }
  cfg.attrs = na ? attr : nullptr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<A&&>(args)...);
}

#ifndef CRTG_PDL_TRIGGER
#define CRTG_PDL_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if CRTG_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

constexpr int kBlockRows = 128;
constexpr int kBlockK = 128;                    // bytes
constexpr int kBlockBytes = kBlockRows * kBlockK;  // 16 KiB
constexpr int kRowPad = 256;                    // rows padded to the GEMM N tile

__host__ __device__ inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// byte offset of element (r, kbyte) inside one packed plane with `rb_count`
// 128-row blocks.
__host__ __device__ inline int64_t pack_offset(int64_t r, int64_t kbyte, int64_t rb_count) {
  const int64_t kb = kbyte >> 7, rb = r >> 7;
  const int rr = int(r & 127), kin = int(kbyte & 127);
  return (kb * rb_count + rb) * kBlockBytes + (rr >> 3) * 1024 + (rr & 7) * 128 +
         ((((kin >> 4) ^ (rr & 7)) << 4) | (kin & 15));
}

// Per-modulus integer constants for exact residue arithmetic on 32-bit lanes.
//   mod(u) = u - p * (umulhi(u, magic) >> shift)  exact for u < 2^31 when p is
//   not a power of two (shift = floor(log2 p), magic = ceil(2^(32+shift)/p));
//   p == 256 uses a mask.
struct ModConst {
  int32_t p;
  uint32_t magic;
  int32_t shift;
  int32_t half;      // (p + 1) / 2 : symmetric residue r >= half -> r - p
  uint32_t c16;      // 2^16 mod p
  uint32_t c32;      // 2^32 mod p
  int32_t bias;      // p * ceil(2^30 / p): makes |x| <= 2^30 non-negative
  int32_t is_pow2;
  uint32_t neg_p;    // (uint32)(-p): u - q*p as one IMAD
  uint32_t bias_h;   // bias + floor(p/2): sym(x) = ((x + bias_h) mod p) - floor(p/2)
  uint32_t h;        // floor(p/2)
  // Karatsuba epilogue: 3 phases (D = Ar*Br, E = Ai*Bi, F = As*Bs).  Split
  // moduli (some j with j^2 == -1 mod p): 2 phases, X = U*U', Y = V*V' on the
  // planes U = sym(re + j im), V = sym(re - j im); then
  //   e_R = (X + Y) / 2,  e_I = (X - Y) / (2 j)   (mod p)
  int32_t nphase;    // 3, or 2 for a split modulus
  uint32_t inv2;     // 2^-1 mod p        (split moduli)
  uint32_t inv2j;    // (2 j)^-1 mod p    (split moduli)
};

// Residue-kernel constants for one modulus and one stored representative
// (off = floor(p/2): the symmetric residue t - off; off = 128: t ^ 0x80; off = 0:
// t itself, the unsigned pipeline encoding).
// A value a' is read as 16-bit limbs of v = a' + 2^31 (two limbs), a' + 2^63
// (four) or 2^90 + a' (six); u = sum_i limb_i * (2^(16 i) mod p) + k is congruent to a' + off and
// below 2^27, so one magic reduction gives t = (a' + off) mod p.
struct ResConst {
  uint32_t magic;   // ceil(2^(32+shift) / p), or 2^(32 - log2 p) with shift 0 for p = 2^s
  int32_t shift;
  uint32_t neg_p;   // (uint32)(-p): t = u + q * neg_p
  uint32_t off;     // floor(p/2) (symmetric) or 128
  // dp2a byte tables (each 2^(16 i) mod p < 256 fits a byte):
  //  dw0123 = bytes (c0, c16, c32, c48), dw45 = (c64, c80)
  uint32_t dw0123, dw45;
  uint32_t k31;     // (off - 2^31) mod p
  uint32_t k63;     // (off - 2^63) mod p
  uint32_t kw;      // (off - 2^90) mod p
  uint32_t sum_k;   // (-off) mod p: t_s = (t_re + t_im + sum_k) mod p
  // split moduli (ModConst::nphase == 2): planes U, V instead of re, im, re+im;
  // t_U = (t_re + j t_im + gku) mod p, t_V = (t_re + (p - j) t_im + gkv) mod p
  // with gku = (-j off) mod p, gkv = (-(p - j) off) mod p
  uint32_t split, gj, gjn, gku, gkv;
  // the same planes straight from the value limbs: u_U = sum_i limb_i(re) c_i +
  // sum_i limb_i(im) (j c_i mod p) + kU, congruent to re + j im + off (V: p - j)
  uint32_t uw0123, uw45, vw0123, vw45;  // byte tables of j c_i, (p - j) c_i mod p
  uint32_t ku31, ku63, kuw, kv31, kv63, kvw;  // (off - (1 + j) 2^31|63|90) mod p, V likewise
  uint32_t xor_mask;  // stored byte = t ^ mask: 0x80 per byte (off = 128, signed t - 128) or 0
};

struct DevConsts {
  int32_t n;
  ModConst mc[CRTG_MAX_MODULI];
  ResConst rc[CRTG_MAX_MODULI];  // symmetric representative
  ResConst rx[CRTG_MAX_MODULI];  // pipeline representative: unsigned t (uns) or 128-offset
  int32_t sym;                   // 1: the complex pipeline stores symmetric residues too
  int32_t uns;                   // 1: rx holds unsigned residues t in [0, p) (off = 0; u8 GEMM)
  double coeff_hi[CRTG_MAX_MODULI];
  double coeff_lo[CRTG_MAX_MODULI];
  double p_hi, p_lo;
  float p_fast, p_accu, delta;
  // CRT helpers: coeff_hi[l] = (H2*2^32 + H1*2^16 + H0) * 2^hi_shift with 16-bit
  // limbs (integer-pipe accumulation of the exact S1 sum), Dekker split of p_hi
  // and its reciprocal (division-free quotient with an exact fallback).
  int32_t hi_limb[CRTG_MAX_MODULI][3];
  // limb k of moduli (2i, 2i+1) as two unsigned 16-bit halves (dp2a operand)
  uint32_t limb_pair[CRTG_MAX_MODULI / 2][3];
  double hi_scale;  // 2^hi_shift
  double p_split_hi, p_split_lo, inv_p;
};

__device__ __forceinline__ uint32_t mod_u31(uint32_t u, const ModConst& c) {
  if (c.is_pow2) return u & uint32_t(c.p - 1);
  const uint32_t q = __umulhi(u, c.magic) >> c.shift;
  return u - q * uint32_t(c.p);
}

// residue in [0,p) of a signed 32-bit value with |x| <= 2^30
__device__ __forceinline__ uint32_t mod_i32(int32_t x, const ModConst& c) {
  if (c.is_pow2) return uint32_t(x) & uint32_t(c.p - 1);
  return mod_u31(uint32_t(x + c.bias), c);
}

// symmetric representative of r in [0,p): [-floor(p/2), ceil(p/2)-1]
__device__ __forceinline__ int32_t to_sym(uint32_t r, const ModConst& c) {
  return int32_t(r) - (int32_t(r) >= c.half ? c.p : 0);
}

// np.ldexp(x, e): x * 2^e with a single rounding (CUDA's ldexp is exact /
// correctly rounded, 0 ulp, like glibc scalbn).  When 2^e is representable a
// single multiply gives the identical correctly-rounded result.
__device__ __forceinline__ double ldexp_rn(double x, int e) {
  if (e >= -1022 && e <= 1023) return __dmul_rn(x, __longlong_as_double(int64_t(e + 1023) << 52));
  return ldexp(x, e);
}

// floor(log2|x|) of a positive finite double (frexp exponent - 1), subnormals too
__device__ __forceinline__ int floor_log2(double x) { return ilogb(x); }

// ---------------------------------------------------------------------------
// PTX wrappers (mbarrier, bulk copy, tcgen05)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}

// Warp-collective wait: every lane leaves the spin together.  The plain per-lane
// spin can leave a warp diverged (ptxas moves the retry loop out of line and a
// __syncwarp after it may be elided), and the tcgen05.ld / wait::ld that follow
// are .sync.aligned: executed by part of a warp they return undefined data.
__device__ __forceinline__ void mbar_wait_warp(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!__all_sync(0xffffffffu, done));
}

// 1-D bulk copy global -> shared, completion counted on an mbarrier (TMA engine)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

template <int kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <int kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, s8 x s8 -> s32
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Weight-stationary form (`.ws`): the B operand (shared by consecutive MMAs) is
// kept in collector buffer b0 — FILL reads it from shared memory and keeps it,
// LASTUSE reuses it and releases the buffer (SASS UTCIMMA.WS ... B_KEEP / B_REUSE)
template <int USE>  // 0: fill, 1: lastuse
__device__ __forceinline__ void mma_i8_ws(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  if (USE == 0)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.ws.cta_group::1.kind::i8.collector::b0::fill [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.ws.cta_group::1.kind::i8.collector::b0::lastuse [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp gets row
// (lane base + t), columns [col, col+32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

// 32 lanes x 4 consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}

// 32 lanes x 16 consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B, 8-row groups 1 KiB apart.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

// Shared-memory matrix descriptor: K-major, no swizzle (canonical core matrices
// of 8 rows x 16 bytes stored as 128 contiguous bytes); lbo = byte distance of
// core matrices adjacent in K, sbo = in M / N.
__device__ __forceinline__ uint64_t smem_desc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Instruction descriptor: kind::i8, s8 x s8 -> s32, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

}  // namespace crtg

// ---------------------------------------------------------------------------
// cluster / CTA-pair (cta_group::2) helpers
// ---------------------------------------------------------------------------
namespace crtg {

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// shared::cta address -> shared::cluster address of the same offset in CTA `rank`
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}

// arrive (release, cluster scope) on an mbarrier given by its shared::cluster address
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}

// wait with cluster-scope acquire (barriers that receive remote arrivals)
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}

// 1-D bulk copy global -> the same smem offset in every CTA of `mask`, each
// destination's mbarrier (same offset) receiving the byte count
__device__ __forceinline__ void bulk_g2s_mc(uint32_t dst, const void* src, uint32_t bytes,
                                            uint32_t bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "h"(mask)
      : "memory");
}

// completion of this CTA's prior MMAs -> arrive on the barrier at this smem
// offset in every CTA of `mask` (cta_group::1 MMAs)
__device__ __forceinline__ void mma_commit_mc(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}

template <int kCols>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}

template <int kCols>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}

// D[tmem, both CTAs] (+)= A[smem, both CTAs] * B[smem, N halves in both CTAs]^T
__device__ __forceinline__ void mma_i8_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// completion of the pair's prior MMAs -> arrive on the barrier at this smem
// offset in every CTA of `mask`
__device__ __forceinline__ void mma_commit_pair(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}

}  // namespace crtg
