// gemm_pair.cu — K3 on a CTA pair: tcgen05.mma.cta_group::2, 256x256 tiles.
//
// Same job as gemm_tc.cu (reference kernel.py:45-51 / 20-35), laid out for two
// SMs of a TPC working on one 256-row x 256-column tile:
//   * cluster (2,1,1); CTA rank r owns A rows [128r, 128r+128) of the tile and
//     B columns [128r, 128r+128) — so each SM streams 32 KiB per 128-byte K step
//     instead of 48 KiB (B is split across the pair, not replicated), 6 stages;
//   * the leader (rank 0) issues tcgen05.mma.cta_group::2 (M=256, N=256, K=32);
//     each CTA's TMEM holds its 128 rows x 256 columns (2 buffers = 512 cols);
//   * both CTAs load their halves with 2-D tensor TMA (.cta_group::2) whose
//     completion bytes land on the LEADER's full barrier (peer bit cleared), so
//     the leader's MMA sees the whole pair stage with one wait — the packed
//     operand image is addressed as a [bytes/128][128] uint8 tensor with
//     128x128 boxes (the data is already in SWIZZLE_128B order);
//   * MMA completion is multicast to both CTAs' empty / accumulator-full
//     barriers; both CTAs' epilogues arrive on the leader's accumulator-empty
//     barrier before it reuses a TMEM buffer.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "gemm_epilogue.cuh"
#include "gemm_tc.cuh"

namespace crtg {

namespace {

constexpr uint32_t kPStageA = 16384;  // 128 rows x 128 B (this CTA's A half)
constexpr uint32_t kPStageB = 16384;  // 128 B-columns x 128 B (this CTA's N half)
constexpr uint32_t kPStageBytes = kPStageA + kPStageB;
constexpr int kPStages = 6;
constexpr int kPTmemCols = 512;
constexpr int kPGroupM = 8;  // pair-row tiles per rasterisation sweep

// 2-D tensor TMA, pair form: bytes complete on the leader CTA's mbarrier
__device__ __forceinline__ void tma_load_pair(uint32_t dst, const CUtensorMap* map, int32_t x,
                                              int32_t y, uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void decode_pair(int t, const GemmArgs& g, int& l, int& tm2, int& tn) {
  const int mt2 = g.mt >> 1;  // 256-row pair tiles
  const int per = mt2 * g.nt;
  l = t / per;
  const int r = t - l * per;
  const int grp = r / (kPGroupM * g.nt);
  const int first = grp * kPGroupM;
  const int gm = min(kPGroupM, mt2 - first);
  const int in = r - grp * kPGroupM * g.nt;
  tm2 = first + in % gm + (g.mt0 >> 1);
  tn = in / gm + g.nt0;
}

}  // namespace

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    k_gemm_i8_pair(const __grid_constant__ GemmArgs g, const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kPStages];   // leader: both CTAs' bytes landed
  __shared__ __align__(8) uint64_t empty_bar[kPStages];  // pair MMA done with the stage
  __shared__ __align__(8) uint64_t tfull_bar[2];         // accumulator buffer ready
  __shared__ __align__(8) uint64_t tempty_bar[2];        // leader: 8 epilogue warps done
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tfull_bar[b]), 1);
      mbar_init(smem_u32(&tempty_bar[b]), 8);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<kPTmemCols>(smem_u32(&tmem_slot));
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  const int total = g.nl * (g.mt >> 1) * g.nt;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    // ---------------- producer (both CTAs): this CTA's A half and B half ----------------
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    uint32_t stage = 0, phase = 0;
    for (int t = cid; t < total; t += ncl) {
      int l, tm2, tn;
      decode_pair(t, g, l, tm2, tn);
      const int nseg = tile_segments<MODE>(g, l);
      for (int s = 0; s < nseg; ++s) {
        // rows of the [bytes/128][128] view: one 16 KiB block = 128 rows
        const int64_t a_row0 = (int64_t)(l * g.planes_per_l + s) * (g.a_plane >> 7);
        const int64_t b_row0 = (int64_t)(l * g.planes_per_l + s) * (g.b_plane >> 7);
        for (int kb = 0; kb < g.kb; ++kb) {
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full_bar[stage]);
          const uint32_t fb_leader = fb & 0xFEFFFFFFu;  // same barrier in CTA rank 0
          const uint32_t sa = smem_base + stage * kPStageBytes;
          if (leader) mbar_expect_tx(fb, 2 * kPStageBytes);  // both CTAs' bytes
          tma_load_pair(sa, &map_a, 0,
                        int32_t(a_row0 + ((int64_t)kb * g.a_rb + 2 * tm2 + rank) * 128),
                        fb_leader);
          tma_load_pair(sa + kPStageA, &map_b, 0,
                        int32_t(b_row0 + ((int64_t)kb * g.b_rb + 2 * tn + rank) * 128),
                        fb_leader);
          if (++stage == kPStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    if (leader) {
      // ---------------- MMA issuer (leader only) ----------------
      constexpr uint32_t idesc = idesc_i8(256, 256);
      uint32_t stage = 0, phase = 0, gslot = 0;
      for (int t = cid; t < total; t += ncl) {
        int l, tm2, tn;
        decode_pair(t, g, l, tm2, tn);
        const int nseg = tile_segments<MODE>(g, l);
        for (int s = 0; s < nseg; ++s) {
          const uint32_t buf = gslot & 1;
          mbar_wait_cluster(smem_u32(&tempty_bar[buf]), ((gslot >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + buf * 256;
          for (int kb = 0; kb < g.kb; ++kb) {
            mbar_wait(smem_u32(&full_bar[stage]), phase);
            tc_fence_after();
            const uint32_t sa = smem_base + stage * kPStageBytes;
            const uint64_t ad = smem_desc_sw128(sa);
            const uint64_t bd = smem_desc_sw128(sa + kPStageA);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_i8_pair(d, ad + 2 * kk, bd + 2 * kk, idesc, (kb | kk) != 0);
            mma_commit_pair(smem_u32(&empty_bar[stage]), 0x3);
            if (++stage == kPStages) { stage = 0; phase ^= 1; }
          }
          mma_commit_pair(smem_u32(&tfull_bar[buf]), 0x3);
          ++gslot;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs, own 128 rows) ----------------
    const int q = warp & 3;
    const uint32_t lane_addr = tmem + (uint32_t(32 * q) << 16);
    const uint32_t tempty0 = mapa(smem_u32(&tempty_bar[0]), 0);
    uint32_t gslot = 0;
    uint32_t st[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) st[i] = 0;
    for (int t = cid; t < total; t += ncl) {
      int l, tm2, tn;
      decode_pair(t, g, l, tm2, tn);
      const int row = (2 * tm2 + int(rank)) * 128 + 32 * q + lane;
      const bool row_ok = row < g.m;
      const int col_base = tn * 256;
      const ModConst mc = g.mc[l];
      const int nseg = tile_segments<MODE>(g, l);
      for (int s = 0; s < nseg; ++s) {
        const uint32_t buf = gslot & 1;
        mbar_wait(smem_u32(&tfull_bar[buf]), (gslot >> 1) & 1);
        tc_fence_after();
        epilogue_phase<MODE, 8>(g, lane_addr + buf * 256, s, l, row, row_ok, col_base, mc, st);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty0 + buf * 8);
        ++gslot;
      }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<kPTmemCols>(tmem);
  }
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// the packed planes as a [bytes/128][128] uint8 tensor, 128x128 boxes, no swizzle
int make_map(CUtensorMap* map, const void* base, int64_t bytes) {
  auto fn = encode_fn();
  if (!fn) return int(cudaErrorNotSupported);
  const cuuint64_t dims[2] = {128, cuuint64_t(bytes / 128)};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, 128};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : int(cudaErrorInvalidValue);
}
}  // namespace

int launch_gemm_pair(int mode, const GemmArgs& g, int num_sms, cudaStream_t stream) {
  const int pairs = g.nl * (g.mt >> 1) * g.nt;
  if (pairs <= 0) return 0;
  CUtensorMap map_a, map_b;
  const int64_t planes = int64_t(g.nl) * g.planes_per_l;
  if (int e = make_map(&map_a, g.a, planes * g.a_plane)) return e;
  if (int e = make_map(&map_b, g.b, planes * g.b_plane)) return e;
  int grid = 2 * (pairs < num_sms / 2 ? pairs : num_sms / 2);
  const size_t smem = size_t(kPStages) * kPStageBytes + 1024;
  cudaError_t err;
  if (mode == EPI_RAW) {
    err = cudaFuncSetAttribute(k_gemm_i8_pair<EPI_RAW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(smem));
    if (err != cudaSuccess) return int(err);
    k_gemm_i8_pair<EPI_RAW><<<grid, 256, smem, stream>>>(g, map_a, map_b);
  } else {
    err = cudaFuncSetAttribute(k_gemm_i8_pair<EPI_KARATSUBA>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (err != cudaSuccess) return int(err);
    k_gemm_i8_pair<EPI_KARATSUBA><<<grid, 256, smem, stream>>>(g, map_a, map_b);
  }
  return launched(1);
}

}  // namespace crtg
