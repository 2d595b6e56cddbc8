// residue.cu — K2: scale + truncate + symmetric residues, written straight into the
// packed tcgen05 operand image; plus the accurate-mode bound operands (K1a).
//
// Replaces, per element and fused in one HBM pass:
//   quantize           scaling.py:277-293   a' = trunc(ldexp(a, e))
//   residue_decompose  crt.py:199-218       r_l = sym(a' mod p_l) for every modulus
//   Karatsuba sums     kernel.py:101-103    s_l = sym(r_re + r_im mod p_l)
//   _bound_matrices    scaling.py:216-226   ceil(|x| 2^bar) and their difference
// Integer residues are exact for |a'| < 2^90: a' = M * 2^s with a 53-bit integer
// significand M; M mod p is folded on 32-bit lanes through 2^32 mod p and
// 2^16 mod p, then multiplied by 2^s mod p.  The congruence class equals the
// reference's 2^31 split (crt.py:123-133), so the symmetric residue is identical.
#include "common.cuh"
#include "kernels.cuh"

namespace crtg {

namespace {

constexpr int kTileRows = 32;  // operand rows per CTA
constexpr int kThreads = 256;  // 32 rows x 8 sixteen-byte K chunks

template <typename T>
__device__ __forceinline__ void load_c(const T* p, double& re, double& im);
template <>
__device__ __forceinline__ void load_c<double>(const double* p, double& re, double& im) {
  const double2 v = *reinterpret_cast<const double2*>(p);
  re = v.x;
  im = v.y;
}
template <>
__device__ __forceinline__ void load_c<float>(const float* p, double& re, double& im) {
  const float2 v = *reinterpret_cast<const float2*>(p);
  re = double(v.x);
  im = double(v.y);
}

// integer-valued a' -> (sign, 53-bit significand split, power-of-two shift),
// packed in two registers: hi = M>>32 (21 bits) | s << 24 | neg << 31, lo = M.
struct Dec {
  uint32_t hi;
  uint32_t lo;
};

__device__ __forceinline__ Dec decompose(double v) {
  uint32_t tag = v < 0.0 ? 0x80000000u : 0u;
  double a = fabs(v);
  if (a >= 9007199254740992.0) {  // 2^53: a' = M * 2^s
    const int s = ilogb(a) - 52;
    a = ldexp(a, -s);  // exact
    tag |= uint32_t(s) << 24;
  }
  const uint64_t M = uint64_t(a);
  return {uint32_t(M >> 32) | tag, uint32_t(M)};
}

__device__ __forceinline__ uint32_t residue_u(const Dec& d, const ModConst& c,
                                              const uint16_t* pow2mod) {
  // hi*2^32 + lo_h*2^16 + lo_l  ==  hi*c32 + lo_h*c16 + lo_l   (mod p), < 2^30
  const uint32_t u = (d.hi & 0x1FFFFFu) * c.c32 + (d.lo >> 16) * c.c16 + (d.lo & 0xFFFFu);
  uint32_t r = mod_u31(u, c);
  const uint32_t s = (d.hi >> 24) & 0x3Fu;
  if (s) r = mod_u31(r * uint32_t(pow2mod[s]), c);
  if ((d.hi >> 31) && r) r = uint32_t(c.p) - r;
  return r;
}

template <typename T, int OPERAND, int KIND>
__global__ void __launch_bounds__(kThreads) k_pack(const T* __restrict__ X, int64_t ldx, int rows,
                                                  int kdim, int64_t col0,
                                                  const int32_t* __restrict__ exps,
                                                  const __grid_constant__ DevConsts dc,
                                                  int8_t* __restrict__ out, int64_t plane_bytes,
                                                  int64_t rb_count,
                                                  unsigned long long* __restrict__ overflow) {
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
      const T* p = (OPERAND == 0) ? X + 2 * (int64_t(row) * ldx + h)
                                  : X + 2 * (int64_t(h) * ldx + col0 + row);
      load_c<T>(p, re[t], im[t]);
    }
  }

  // swizzled position of this thread's 16-byte chunk inside the 4 KiB stage tile
  const int soff = (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4);
  // the CTA's 32 rows are one contiguous 4 KiB run of the packed plane
  const int64_t goff = (int64_t(kb) * rb_count + (r0 >> 7)) * kBlockBytes + (r0 & 127) * 128;

  if (KIND == PACK_BARS) {
    // bound operands: ceil(|x| 2^bar) in [0, 64] and their difference
    uint32_t w[3][4] = {};
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int vr = int(ceil(ldexp_rn(fabs(re[t]), e)));
      const int vi = int(ceil(ldexp_rn(fabs(im[t]), e)));
      w[0][t >> 2] |= uint32_t(vr & 0xFF) << (8 * (t & 3));
      w[1][t >> 2] |= uint32_t(vi & 0xFF) << (8 * (t & 3));
      w[2][t >> 2] |= uint32_t((vr - vi) & 0xFF) << (8 * (t & 3));
    }
#pragma unroll
    for (int q = 0; q < 3; ++q)
      *reinterpret_cast<uint4*>(&stage[q][soff]) = make_uint4(w[q][0], w[q][1], w[q][2], w[q][3]);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 3; ++q)
      reinterpret_cast<uint4*>(out + q * plane_bytes + goff)[threadIdx.x] =
          reinterpret_cast<const uint4*>(stage[q])[threadIdx.x];
    return;
  }

  // quantize: a' = trunc(x 2^e), |a'| < 2^90 (else DomainError, flagged)
  Dec dr[16], di[16];
  int bad = 0;
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    double qr = trunc(ldexp_rn(re[t], e));
    double qi = trunc(ldexp_rn(im[t], e));
    if (!(fabs(qr) < 0x1p90)) { bad = 1; qr = 0.0; }
    if (!(fabs(qi) < 0x1p90)) { bad = 1; qi = 0.0; }
    dr[t] = decompose(qr);
    di[t] = decompose(qi);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(overflow, 1ull);

  for (int l = 0; l < dc.n; ++l) {
    const ModConst mc = dc.mc[l];
    const uint16_t* p2 = dc.pow2mod[l];
    uint32_t w[3][4] = {};
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const uint32_t ur = residue_u(dr[t], mc, p2);
      const uint32_t ui = residue_u(di[t], mc, p2);
      uint32_t us = ur + ui;
      us -= (us >= uint32_t(mc.p)) ? uint32_t(mc.p) : 0u;
      const int sh = 8 * (t & 3);
      w[0][t >> 2] |= (uint32_t(to_sym(ur, mc)) & 0xFF) << sh;
      w[1][t >> 2] |= (uint32_t(to_sym(ui, mc)) & 0xFF) << sh;
      w[2][t >> 2] |= (uint32_t(to_sym(us, mc)) & 0xFF) << sh;
    }
#pragma unroll
    for (int q = 0; q < 3; ++q)
      *reinterpret_cast<uint4*>(&stage[q][soff]) = make_uint4(w[q][0], w[q][1], w[q][2], w[q][3]);
    __syncthreads();
    int8_t* base = out + int64_t(3 * l) * plane_bytes + goff;
#pragma unroll
    for (int q = 0; q < 3; ++q)
      reinterpret_cast<uint4*>(base + q * plane_bytes)[threadIdx.x] =
          reinterpret_cast<const uint4*>(stage[q])[threadIdx.x];
    __syncthreads();
  }
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

template <typename T, int OP, int KIND>
void launch_one(const void* X, int64_t ldx, int64_t rows, int64_t kdim, int64_t col0,
                const int32_t* exps, const DevConsts& dc, int8_t* out, int64_t plane_bytes,
                int64_t rb_count, unsigned long long* overflow, cudaStream_t s) {
  // cover every padded row of the plane so the GEMM reads zeros there
  dim3 grid(unsigned((kdim + 127) / 128), unsigned(rb_count * 128 / kTileRows));
  k_pack<T, OP, KIND><<<grid, kThreads, 0, s>>>(static_cast<const T*>(X), ldx, int(rows),
                                                int(kdim), col0, exps, dc, out, plane_bytes,
                                                rb_count, overflow);
}

}  // namespace

int launch_pack(bool single, int operand, int kind, const void* X, int64_t ldx, int64_t rows,
                int64_t kdim, int64_t col0, const int32_t* exps, const DevConsts& dc,
                int8_t* out, int64_t plane_bytes, int64_t rb_count,
                unsigned long long* overflow, cudaStream_t s) {
  if (rows <= 0 || kdim <= 0) return 0;
#define CRTG_PACK(T, OP, KIND) \
  launch_one<T, OP, KIND>(X, ldx, rows, kdim, col0, exps, dc, out, plane_bytes, rb_count, overflow, s)
  if (single) {
    if (operand == 0) {
      if (kind == PACK_BARS) CRTG_PACK(float, 0, PACK_BARS); else CRTG_PACK(float, 0, PACK_RESIDUE);
    } else {
      if (kind == PACK_BARS) CRTG_PACK(float, 1, PACK_BARS); else CRTG_PACK(float, 1, PACK_RESIDUE);
    }
  } else {
    if (operand == 0) {
      if (kind == PACK_BARS) CRTG_PACK(double, 0, PACK_BARS); else CRTG_PACK(double, 0, PACK_RESIDUE);
    } else {
      if (kind == PACK_BARS) CRTG_PACK(double, 1, PACK_BARS); else CRTG_PACK(double, 1, PACK_RESIDUE);
    }
  }
#undef CRTG_PACK
  return int(cudaGetLastError());
}

int launch_pack_i8(const int8_t* X, int trans, int64_t rows, int64_t kdim, int8_t* out,
                   int64_t rb_count, cudaStream_t s) {
  const int64_t kpad = round_up(kdim, 128);
  const int64_t rpad = rb_count * 128;
  const int64_t total = rpad * (kpad / 16);
  if (total <= 0) return 0;
  k_pack_i8<<<unsigned((total + 255) / 256), 256, 0, s>>>(X, trans, rows, kdim, kpad, out, rb_count,
                                                          total);
  return int(cudaGetLastError());
}

int launch_unpack_i8(const int8_t* packed, int64_t rows, int64_t kdim, int64_t rb_count,
                     int8_t* out, cudaStream_t s) {
  const int64_t total = rows * kdim;
  if (total <= 0) return 0;
  k_unpack_i8<<<unsigned((total + 255) / 256), 256, 0, s>>>(packed, rows, kdim, rb_count, out);
  return int(cudaGetLastError());
}

}  // namespace crtg
