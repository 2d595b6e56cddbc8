// gemm_tc.cuh — launch interface of the tcgen05 INT8 residue GEMM (gemm_tc.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace crtg {

enum EpiMode { EPI_KARATSUBA = 0, EPI_RAW = 1, EPI_BOUND = 2, EPI_REAL = 3 };

struct GemmArgs {
  const int8_t* a;   // packed A planes: [nl][planes_per_l] x (k_pad x 128*a_rb)
  const int8_t* b;   // packed B^T planes
  int64_t a_plane;   // bytes per A plane
  int64_t b_plane;   // bytes per B plane
  int a_rb, b_rb;    // 128-row blocks per plane
  int mt, nt, kb;    // 128-row tiles, 256-col tiles, 128-byte K blocks
  int mt0;           // first 128-row tile of this launch (row-chunked launches)
  int nt0;           // first 256-column tile of this launch (column strips)
  int nl;            // moduli handled by this launch
  int planes_per_l;  // planes per modulus (3 = re, im, re+im)
  int nphase;        // segments per tile for KARATSUBA (3) / RAW (1..3)
  int m, n;          // valid output extents
  int8_t* e_re;      // KARATSUBA: [nl][m][e_ld]
  int8_t* e_im;
  int64_t e_plane, e_ld;
  int32_t* raw;      // RAW: [nphase][m][raw_ld]
  int64_t raw_plane, raw_ld;
  int32_t* row_max;  // BOUND: [mt*128]
  int32_t* col_max;  // BOUND: [nt*256]
  unsigned long long* overflow;  // REAL: int32 accumulator overflow (kernel.py:33-34)
  int group_m;       // raster: row tiles per column sweep (0 -> 16)
  int uns;           // KARATSUBA: operands are unsigned residues in [0, p) (u8 x u8)
  ModConst mc[CRTG_MAX_MODULI];
};

size_t gemm_smem_bytes();
// returns a cudaError_t value (0 = success)
int launch_gemm(int mode, const GemmArgs& g, int num_sms, cudaStream_t stream);
// wide-tile KARATSUBA (split) / REAL variant (256 x 256 per CTA, gemm_tc.cu); g.mt and
// g.mt0 must be even
int launch_gemm_wide(int mode, const GemmArgs& g, int num_sms, cudaStream_t stream);

}  // namespace crtg
