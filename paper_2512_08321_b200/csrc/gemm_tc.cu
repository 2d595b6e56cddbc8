// gemm_tc.cu — K3: INT8 residue GEMMs on 5th-gen tensor cores (tcgen05, sm_100a).
//
// Replaces the per-modulus loop of emulate_gemm_complex (reference
// emulate.py:224-231) -> complex_gemm_mod (kernel.py:70-120) -> _karatsuba_block
// (kernel.py:45-51) -> gemm_i8_i32 (kernel.py:20-35), and the bound product of
// accurate_scaling (scaling.py:249-258).
//
// One persistent, warp-specialised kernel:
//   warp 0 (lane 0)  producer: 1-D bulk copies (TMA engine) of pre-packed,
//                    pre-swizzled 128x128-byte operand blocks into a 4-stage ring;
//   warp 1 (lane 0)  MMA issuer: tcgen05.mma.kind::i8, M=128 N=256 K=32, s32
//                    accumulators in TMEM (2 x 256 columns, double-buffered);
//   warp 2           TMEM allocator;
//   warps 4..7       epilogue: tcgen05.ld -> registers -> modular epilogue.
// A tile (l, tm, tn) runs one "segment" per operand pair:
//   EPI_KARATSUBA: D = Ar*Br, E = Ai*Bi, F = As*Bs (three sequential K loops into
//     alternating TMEM buffers).  The epilogue keeps D mod p, then (D+E) mod p, as
//     packed bytes in registers, and writes e_R = sym(D-E) and e_I = sym(F-D-E)
//     as int8 — INT32 products never leave the SM.
//   EPI_RAW: writes the int32 accumulators (parity hook for gemm_i8_i32).
//   EPI_BOUND: X = (AR+AI)*(BR+BI) (unsigned bytes, buffer 0) and D = AD*BD
//     (buffer 1).  The reference's cross = AI*BR + AR*BI = (X - D)/2 and
//     cross + diff = AR*BR + AI*BI = (X + D)/2, so its bound
//     max(cross + diff, cross) (scaling.py:251-258) is exactly (X + |D|)/2:
//     two products instead of three.  Row / column maxima by atomicMax.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "gemm_tc.cuh"
#include "gemm_epilogue.cuh"

namespace crtg {

namespace {

constexpr uint32_t kStageA = 16384;  // 128 rows x 128 B
constexpr uint32_t kStageB = 32768;  // 256 rows x 128 B
constexpr uint32_t kStageBytes = kStageA + kStageB;
constexpr int kStages = 4;
constexpr int kTmemCols = 512;
constexpr int kEpiThreads = 256;            // 8 epilogue warps
constexpr int kThreads = 128 + kEpiThreads;  // producer, MMA, TMEM alloc, spare + epilogue
constexpr int kGroupM = 16;  // rasterisation: 16 row tiles share each column sweep
// Karatsuba / split epilogue state in shared memory (gemm_epilogue.cuh
// karatsuba_phase_sm): 32 words per epilogue thread behind the operand ring
#ifndef CRTG_EPI_SMEM
#define CRTG_EPI_SMEM 1
#endif
constexpr uint32_t kStateBytes = CRTG_EPI_SMEM ? kEpiThreads * 32 * 4 : 0;

struct Seg {
  int a_plane, b_plane, buf, accumulate;
};


template <int MODE>
__device__ __forceinline__ Seg seg_of(int s) {
  if (MODE == EPI_BOUND) {
    // X = AS*BS -> buffer 0 (unsigned); D = AD*BD -> buffer 1
    if (s == 0) return {0, 0, 0, 0};
    return {2, 2, 1, 0};
  }
  return {s, s, -1, 0};
}

__device__ __forceinline__ void decode_tile(int t, const GemmArgs& g, int& l, int& tm, int& tn) {
  const int per = g.mt * g.nt;
  l = t / per;
  const int r = t - l * per;
  const int G = g.group_m > 0 ? g.group_m : kGroupM;
  const int grp = r / (G * g.nt);
  const int first = grp * G;
  const int gm = min(G, g.mt - first);
  const int in = r - grp * G * g.nt;
  tm = first + in % gm + g.mt0;
  tn = in / gm + g.nt0;
}

// unit of a persistent CTA in round r: boustrophedon over the rounds (round r
// covers units [r G, (r + 1) G); odd rounds in reverse CTA order), so a CTA
// that got an early unit of a round gets a late one of the next
__device__ __forceinline__ int unit_of(int r) {
  const int G = int(gridDim.x), b = int(blockIdx.x);
  return r * G + ((r & 1) ? G - 1 - b : b);
}

}  // namespace

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_gemm_i8(const __grid_constant__ GemmArgs g) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ __align__(8) uint64_t empty_bar[kStages];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ uint32_t tmem_slot;
  __shared__ int8_t lord[CRTG_MAX_MODULI];  // processing order of the moduli

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // 1024-byte aligned operand ring (SWIZZLE_128B atoms)
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tfull_bar[b]), 1);
      mbar_init(smem_u32(&tempty_bar[b]), kEpiThreads);
    }
    fence_mbar_init();
    // Karatsuba: the three-product moduli first, the two-product (split) ones
    // last, so that with the snake order below the CTAs that run one unit more
    // than others run cheap ones (1024^3 N=14: 448 units on 148 CTAs, longest
    // CTA 12 -> 10 products)
    int o = 0;
    for (int pass = 0; pass < 2; ++pass)
      for (int l = 0; l < g.nl; ++l)
        if (MODE != EPI_KARATSUBA ? pass == 0 : (g.mc[l].nphase == 2) == (pass == 1))
          lord[o++] = int8_t(l);
  }
  if (warp == 2) tmem_alloc<kTmemCols>(smem_u32(&tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_begin();  // barriers and TMEM are set up; operands are read from here on

  const int total = g.nl * g.mt * g.nt;

  if (warp == 0 && lane == 0) {
    // ---------------- producer ----------------
    uint32_t stage = 0, phase = 0;
    for (int r = 0; r * int(gridDim.x) < total; ++r) {
      const int t = unit_of(r);
      if (t >= total) continue;
      int l, tm, tn;
      decode_tile(t, g, l, tm, tn);
      l = lord[l];
      const int nseg = MODE == EPI_BOUND ? 2 : tile_segments<MODE>(g, l);
      for (int s = 0; s < nseg; ++s) {
        const Seg sg = seg_of<MODE>(s);
        const int8_t* a = g.a + (int64_t)(l * g.planes_per_l + sg.a_plane) * g.a_plane;
        const int8_t* b = g.b + (int64_t)(l * g.planes_per_l + sg.b_plane) * g.b_plane;
        for (int kb = 0; kb < g.kb; ++kb) {
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full_bar[stage]);
          const uint32_t sa = smem_base + stage * kStageBytes;
          mbar_expect_tx(fb, kStageBytes);
          bulk_g2s(sa, a + ((int64_t)kb * g.a_rb + tm) * kBlockBytes, kStageA, fb);
          bulk_g2s(sa + kStageA, b + ((int64_t)kb * g.b_rb + 2 * tn) * kBlockBytes, kStageB, fb);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    // unsigned operands (bits 7 / 10 clear): the Karatsuba / split residues in
    // [0, p) (g.uns) and the accurate-mode X = (R+I)(R'+I') bytes of the bound product
    const uint32_t idesc_s = idesc_i8(128, 256);
    const uint32_t idesc_u = idesc_s & ~((1u << 7) | (1u << 10));
    const uint32_t idesc = (MODE == EPI_KARATSUBA || MODE == EPI_REAL) && g.uns ? idesc_u : idesc_s;
    uint32_t stage = 0, phase = 0, gslot = 0;
    for (int r = 0; r * int(gridDim.x) < total; ++r) {
      const int t = unit_of(r);
      if (t >= total) continue;
      int l, tm, tn;
      decode_tile(t, g, l, tm, tn);
      l = lord[l];
      const int nseg = MODE == EPI_BOUND ? 2 : tile_segments<MODE>(g, l);
      if (MODE == EPI_BOUND) {
        const uint32_t par = ((gslot >> 1) & 1) ^ 1;
        mbar_wait(smem_u32(&tempty_bar[0]), par);
        mbar_wait(smem_u32(&tempty_bar[1]), par);
        tc_fence_after();
      }
      for (int s = 0; s < nseg; ++s) {
        const Seg sg = seg_of<MODE>(s);
        uint32_t buf;
        if (MODE == EPI_BOUND) {
          buf = sg.buf;
        } else {
          buf = gslot & 1;
          mbar_wait(smem_u32(&tempty_bar[buf]), ((gslot >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        const uint32_t d = tmem + buf * 256;
        for (int kb = 0; kb < g.kb; ++kb) {
          mbar_wait(smem_u32(&full_bar[stage]), phase);
          tc_fence_after();
          const uint32_t sa = smem_base + stage * kStageBytes;
          const uint64_t ad = smem_desc_sw128(sa);
          const uint64_t bd = smem_desc_sw128(sa + kStageA);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            // advance 32 bytes of K inside the 128-byte swizzle atom
            mma_i8(d, ad + 2 * kk, bd + 2 * kk,
                   (MODE == EPI_BOUND && s == 0) ? idesc_u : idesc,
                   (kb | kk | sg.accumulate) != 0);
          }
          mma_commit(smem_u32(&empty_bar[stage]));  // frees the smem slot when MMAs finish
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (MODE == EPI_BOUND) {
          mma_commit(smem_u32(&tfull_bar[s]));
        } else {
          mma_commit(smem_u32(&tfull_bar[buf]));
          ++gslot;
        }
      }
      if (MODE == EPI_BOUND) gslot += 2;
    }
  } else if (warp >= 4) {
    // ------- epilogue (8 warps: lane quarter warp % 4, column half (warp - 4) / 4) -------
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const uint32_t lane_addr = tmem + (uint32_t(32 * q) << 16) + uint32_t(128 * half);
    uint32_t gslot = 0;
    uint32_t st[32];  // packed per-column state across the three Karatsuba phases
    uint32_t* sst = reinterpret_cast<uint32_t*>(smem_raw + (smem_base - smem_u32(smem_raw)) +
                                                kStages * kStageBytes) +
                    (threadIdx.x - 128);
#pragma unroll
    for (int i = 0; i < 32; ++i) st[i] = 0;
    for (int r = 0; r * int(gridDim.x) < total; ++r) {
      const int t = unit_of(r);
      if (t >= total) continue;
      int l, tm, tn;
      decode_tile(t, g, l, tm, tn);
      l = lord[l];
      const int row = tm * 128 + 32 * q + lane;
      const bool row_ok = row < g.m;
      const int col_base = tn * 256 + 128 * half;
      if (MODE == EPI_BOUND) {
        const uint32_t par = (gslot >> 1) & 1;
        mbar_wait_warp(smem_u32(&tfull_bar[0]), par);
        mbar_wait_warp(smem_u32(&tfull_bar[1]), par);
        tc_fence_after();
        int32_t rmax = 0;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t xs[32], df[32];
          tmem_ld32(lane_addr + c * 32, xs);
          tmem_ld32(lane_addr + 256 + c * 32, df);
          tmem_wait_ld();
          int32_t mine = 0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            // X <= k * 128^2 <= 2^30 and |D| <= k * 64^2: no int32 overflow
            const int32_t bnd = (int32_t(xs[i]) + abs(int32_t(df[i]))) >> 1;
            rmax = max(rmax, bnd);
            const int32_t cm = __reduce_max_sync(0xffffffffu, bnd);
            if (lane == i) mine = cm;
          }
          atomicMax(g.col_max + col_base + c * 32 + lane, mine);
        }
        if (row_ok) atomicMax(g.row_max + row, rmax);
        tc_fence_before();
        mbar_arrive(smem_u32(&tempty_bar[0]));
        mbar_arrive(smem_u32(&tempty_bar[1]));
        gslot += 2;
        continue;
      }
      const ModConst mc = g.mc[l];
      const int nseg = tile_segments<MODE>(g, l);
      for (int s = 0; s < nseg; ++s) {
        const uint32_t buf = gslot & 1;
        mbar_wait_warp(smem_u32(&tfull_bar[buf]), (gslot >> 1) & 1);
        tc_fence_after();
        if (MODE == EPI_KARATSUBA && CRTG_EPI_SMEM)
          karatsuba_epilogue_sm<4>(g, lane_addr + buf * 256, s, l, row, row_ok, col_base, mc, sst,
                                   kEpiThreads);
        else
          epilogue_phase<MODE, 4>(g, lane_addr + buf * 256, s, l, row, row_ok, col_base, mc, st);
        tc_fence_before();
        mbar_arrive(smem_u32(&tempty_bar[buf]));
        ++gslot;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

// ---------------------------------------------------------------------------
// Wide-tile Karatsuba / split kernel: 256 x 256 output tile per CTA.
//
// The 128 x 256 kernel above pulls 48 KiB from L2 per 128 x 256 x 128 MACs.
// Measured on B200 (tools/power_data.py, profiles/r01_gemm_reuse_experiment.json):
// with operands already in shared memory a second MMA costs far less than one
// whose operands crossed the L2 -> SM network, i.e. the power-capped GEMM pays
// for L2 -> SMEM bytes, not for MACs alone.  Two M = 128 MMAs that share one
// 256-column B tile (rows 0-127 -> TMEM columns [0,256), rows 128-255 ->
// [256,512)) cut that traffic to 64 KiB per 256 x 256 x 128 MACs (-33%), with
// no peer-SM traffic (the CTA-pair kernel moves the same third over DSMEM).
// The price: the accumulators fill all 512 TMEM columns, so each segment's
// epilogue (TMEM -> registers -> bytes, ~2% of a segment) is not overlapped.
// ---------------------------------------------------------------------------
namespace {
constexpr uint32_t kWStageA = 32768;  // 256 rows x 128 B (two packed blocks)
constexpr uint32_t kWStageB = 32768;  // 256 rows x 128 B
constexpr uint32_t kWStageBytes = kWStageA + kWStageB;
// CRTG_WS=1 (default): weight-stationary MMAs keep the shared B slice in a
// collector buffer for the second (rows 128-255) MMA instead of re-reading
// shared memory (a third less SMEM -> tensor-core traffic; measured within
// noise of the plain form, clock 100-200 MHz higher, bit-identical)
#ifndef CRTG_WS
#define CRTG_WS 1
#endif
#ifndef CRTG_W_STAGES
#define CRTG_W_STAGES 3
#endif
constexpr int kWStages = CRTG_W_STAGES;
constexpr int kWGroupM = 8;  // 256-row tiles per column sweep
#ifndef CRTG_MOD_INNER
#define CRTG_MOD_INNER 0
#endif
// boustrophedon unit order with the three-product moduli first (as k_gemm_i8)
#ifndef CRTG_W_SNAKE
#define CRTG_W_SNAKE 1
#endif

__device__ __forceinline__ void decode_tile_w(int t, const GemmArgs& g, int& l, int& tm2,
                                              int& tn) {
  const int mt2 = g.mt >> 1;
  const int per = mt2 * g.nt;
#if CRTG_MOD_INNER
  // experiment: modulus index innermost, so the N moduli of
  // one output tile run back to back (the ordering an in-CTA CRT would need)
  l = t % g.nl;
  const int r = t / g.nl;
  (void)per;
#else
  l = t / per;
  const int r = t - l * per;
#endif
  const int G = g.group_m > 0 ? g.group_m : kWGroupM;
  const int grp = r / (G * g.nt);
  const int first = grp * G;
  const int gm = min(G, mt2 - first);
  const int in = r - grp * G * g.nt;
  tm2 = first + in % gm + (g.mt0 >> 1);
  tn = in / gm + g.nt0;
}
}  // namespace

// EW epilogue warps: 8 (lane quarter x row half, 256 columns each) or 16 (also
// x column half, 128 columns each: the non-overlapped drain takes half as long)
template <int MODE, int EW>
__global__ void __launch_bounds__(128 + 32 * EW, 1) k_gemm_w(const __grid_constant__ GemmArgs g) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kWStages];
  __shared__ __align__(8) uint64_t empty_bar[kWStages];
  __shared__ __align__(8) uint64_t tfull_bar, tempty_bar;
  __shared__ uint32_t tmem_slot;
  __shared__ int8_t lord[CRTG_MAX_MODULI];  // processing order of the moduli (CRTG_W_SNAKE)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kWStages; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    mbar_init(smem_u32(&tfull_bar), 1);
    mbar_init(smem_u32(&tempty_bar), 32 * EW);
    fence_mbar_init();
    int o = 0;  // three-product moduli first (see k_gemm_i8)
    for (int pass = 0; pass < 2; ++pass)
      for (int l = 0; l < g.nl; ++l)
        if (!CRTG_W_SNAKE || MODE != EPI_KARATSUBA ? pass == 0
                                                    : (g.mc[l].nphase == 2) == (pass == 1))
          lord[o++] = int8_t(l);
  }
  if (warp == 2) tmem_alloc<kTmemCols>(smem_u32(&tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_begin();
  const int total = g.nl * (g.mt >> 1) * g.nt;

  if (warp == 0 && lane == 0) {
    // ---------------- producer: A rows [256 tm2, +256) and B rows [256 tn, +256) ----------------
    uint32_t stage = 0, phase = 0;
    for (int r = 0; r * int(gridDim.x) < total; ++r) {
      const int t = CRTG_W_SNAKE ? unit_of(r) : r * int(gridDim.x) + int(blockIdx.x);
      if (t >= total) continue;
      int l, tm2, tn;
      decode_tile_w(t, g, l, tm2, tn);
      l = lord[l];
      const int nseg = tile_segments<MODE>(g, l);
      for (int s = 0; s < nseg; ++s) {
        const int8_t* a = g.a + (int64_t)(l * g.planes_per_l + s) * g.a_plane;
        const int8_t* b = g.b + (int64_t)(l * g.planes_per_l + s) * g.b_plane;
        for (int kb = 0; kb < g.kb; ++kb) {
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full_bar[stage]);
          const uint32_t sa = smem_base + stage * kWStageBytes;
          mbar_expect_tx(fb, kWStageBytes);
          bulk_g2s(sa, a + ((int64_t)kb * g.a_rb + 2 * tm2) * kBlockBytes, kWStageA, fb);
          bulk_g2s(sa + kWStageA, b + ((int64_t)kb * g.b_rb + 2 * tn) * kBlockBytes, kWStageB, fb);
          if (++stage == kWStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer: two M=128 MMAs per K step share the B tile ----------------
    // Karatsuba / split on unsigned residue bytes in [0, p): bits 7 / 10 clear
    const uint32_t idesc = (MODE == EPI_KARATSUBA || MODE == EPI_REAL) && g.uns
                               ? (idesc_i8(128, 256) & ~((1u << 7) | (1u << 10)))
                               : idesc_i8(128, 256);
    uint32_t stage = 0, phase = 0, gslot = 0;
    for (int r = 0; r * int(gridDim.x) < total; ++r) {
      const int t = CRTG_W_SNAKE ? unit_of(r) : r * int(gridDim.x) + int(blockIdx.x);
      if (t >= total) continue;
      int l, tm2, tn;
      decode_tile_w(t, g, l, tm2, tn);
      l = lord[l];
      const int nseg = tile_segments<MODE>(g, l);
      for (int s = 0; s < nseg; ++s) {
        mbar_wait(smem_u32(&tempty_bar), (gslot & 1) ^ 1);  // epilogue drained both halves
        tc_fence_after();
        for (int kb = 0; kb < g.kb; ++kb) {
          mbar_wait(smem_u32(&full_bar[stage]), phase);
          tc_fence_after();
          const uint32_t sa = smem_base + stage * kWStageBytes;
          const uint64_t a0 = smem_desc_sw128(sa);
          const uint64_t a1 = smem_desc_sw128(sa + kWStageA / 2);
          const uint64_t bd = smem_desc_sw128(sa + kWStageA);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t acc = (kb | kk) != 0;
            if (CRTG_WS) {
              mma_i8_ws<0>(tmem, a0 + 2 * kk, bd + 2 * kk, idesc, acc);
              mma_i8_ws<1>(tmem + 256, a1 + 2 * kk, bd + 2 * kk, idesc, acc);
            } else {
              mma_i8(tmem, a0 + 2 * kk, bd + 2 * kk, idesc, acc);
              mma_i8(tmem + 256, a1 + 2 * kk, bd + 2 * kk, idesc, acc);
            }
          }
          mma_commit(smem_u32(&empty_bar[stage]));
          if (++stage == kWStages) { stage = 0; phase ^= 1; }
        }
        mma_commit(smem_u32(&tfull_bar));
        ++gslot;
      }
    }
  } else if (warp >= 4) {
    // ------- epilogue: lane quarter warp % 4, row half, (EW = 16) column half -------
    constexpr int NCH = EW == 16 ? 4 : 8;  // 32-column chunks per thread
    const int q = warp & 3;
    const int idx = (warp - 4) >> 2;
    const int half = EW == 16 ? idx >> 1 : idx;
    const int colh = EW == 16 ? idx & 1 : 0;
    const uint32_t lane_addr =
        tmem + (uint32_t(32 * q) << 16) + uint32_t(256 * half) + uint32_t(32 * NCH * colh);
    uint32_t gslot = 0;
    uint32_t st[NCH * 8];
#pragma unroll
    for (int i = 0; i < NCH * 8; ++i) st[i] = 0;
    for (int r = 0; r * int(gridDim.x) < total; ++r) {
      const int t = CRTG_W_SNAKE ? unit_of(r) : r * int(gridDim.x) + int(blockIdx.x);
      if (t >= total) continue;
      int l, tm2, tn;
      decode_tile_w(t, g, l, tm2, tn);
      l = lord[l];
      const int row = tm2 * 256 + 128 * half + 32 * q + lane;
      const bool row_ok = row < g.m;
      const int col_base = tn * 256 + 32 * NCH * colh;
      const ModConst mc = g.mc[l];
      const int nseg = tile_segments<MODE>(g, l);
      for (int s = 0; s < nseg; ++s) {
        mbar_wait_warp(smem_u32(&tfull_bar), gslot & 1);  // warp-converged for tcgen05.ld
        tc_fence_after();
        epilogue_phase<MODE, NCH>(g, lane_addr, s, l, row, row_ok, col_base, mc, st);
        tc_fence_before();
        mbar_arrive(smem_u32(&tempty_bar));
        ++gslot;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

size_t gemm_smem_bytes() { return size_t(kStages) * kStageBytes + kStateBytes + 1024; }

template <int MODE>
int launch_wide_mode(const GemmArgs& g, int grid, size_t smem, cudaStream_t stream) {
  const cudaError_t err = cudaFuncSetAttribute(
      k_gemm_w<MODE, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (err != cudaSuccess) return int(err);
  launch_k(k_gemm_w<MODE, 8>, grid, 128 + 32 * 8, smem, stream, g);
  return launched(1);
}

int launch_gemm_wide(int mode, const GemmArgs& g, int num_sms, cudaStream_t stream) {
  const int total = g.nl * (g.mt >> 1) * g.nt;
  if (total <= 0) return 0;
  const int grid = total < num_sms ? total : num_sms;
  const size_t smem = size_t(kWStages) * kWStageBytes + 1024;
  // 8 epilogue warps (16 halve the non-overlapped drain but hit the 96-register
  // cap and spill: 10% slower)
  return mode == EPI_REAL ? launch_wide_mode<EPI_REAL>(g, grid, smem, stream)
                          : launch_wide_mode<EPI_KARATSUBA>(g, grid, smem, stream);
}

int launch_gemm(int mode, const GemmArgs& g, int num_sms, cudaStream_t stream) {
  const int total = g.nl * g.mt * g.nt;
  if (total <= 0) return 0;
  const int grid = total < num_sms ? total : num_sms;
  const size_t smem = gemm_smem_bytes();
  cudaError_t err;
  switch (mode) {
    case EPI_KARATSUBA:
      err = cudaFuncSetAttribute(k_gemm_i8<EPI_KARATSUBA>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (err != cudaSuccess) return int(err);
      launch_k(k_gemm_i8<EPI_KARATSUBA>, grid, kThreads, smem, stream, g);
      break;
    case EPI_RAW:
      err = cudaFuncSetAttribute(k_gemm_i8<EPI_RAW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem));
      if (err != cudaSuccess) return int(err);
      launch_k(k_gemm_i8<EPI_RAW>, grid, kThreads, smem, stream, g);
      break;
    case EPI_REAL:
      err = cudaFuncSetAttribute(k_gemm_i8<EPI_REAL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem));
      if (err != cudaSuccess) return int(err);
      launch_k(k_gemm_i8<EPI_REAL>, grid, kThreads, smem, stream, g);
      break;
    default:
      err = cudaFuncSetAttribute(k_gemm_i8<EPI_BOUND>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (err != cudaSuccess) return int(err);
      launch_k(k_gemm_i8<EPI_BOUND>, grid, kThreads, smem, stream, g);
      break;
  }
  return launched(1);
}

}  // namespace crtg
