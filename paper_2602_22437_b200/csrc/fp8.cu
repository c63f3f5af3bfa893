// N2: FP8 E4M3 128x128 block quantization of the parameters
// fused with the AllGather (1 byte per element on the wire instead of 2).
//
// One 256-thread CTA per tile (persistent loop over the rank's tile table):
// the tile's fp32 master weights are loaded once into registers (16-B
// vectors, warp w owns rows w, w+8, ..., lane l owns columns 4l..4l+3), the
// tile absmax A is reduced (warp shuffle + shared memory), and every element
// is converted with inv = fl(448 / A) by the hardware E4M3 conversion
// (cvt.rn.satfinite.e4m3x2.f32: round to nearest even, saturating -- the
// oracle's R18/R19).  Each 4-code word is stored into the local gathered
// code buffer and, for M > 1, into every peer's (NVLink stores), so the
// quantization and the AllGather are one kernel; the per-tile scale
// fl(A / 448) goes to every rank's scale array at the tile's global slot.
// HBM: 4 B read + 1 B written per owned element; NVLink: every rank sends
// (m-1) x its S code bytes and receives (m-1) S, plus 4 B per tile.
#include <cuda_fp8.h>

#include <cstdint>

#include "devmath.cuh"
#include "kernels.cuh"
#include "p2p_dev.cuh"

namespace rsdb {

constexpr int FP8_NT = 256;
constexpr int FP8_WARPS = FP8_NT / 32;
constexpr float E4M3_MAX = 448.0f;

// two fp32 -> two E4M3 codes, little-endian: byte 0 = a, byte 1 = b
__device__ __forceinline__ uint32_t e4m3x2(float a, float b) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ uint32_t e4m3x4(float a, float b, float c, float d) {
  return e4m3x2(a, b) | (e4m3x2(c, d) << 16);
}

__device__ __forceinline__ float block_absmax(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax_nan(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5;
  __syncthreads();  // red[] of the previous tile has been consumed
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float a = red[0];
#pragma unroll
  for (int i = 1; i < FP8_WARPS; ++i) a = fmax_nan(a, red[i]);
  return a;
}

// R19 + R28: inv = min(fl(448 / A), FLT_MAX) (finite for every A > 0)
__device__ __forceinline__ float tile_inv(float A) {
  return A > 0.f ? fminf(__fdiv_rn(E4M3_MAX, A), FLT_MAX_F) : 0.f;
}

template <int M>
__device__ __forceinline__ void put_codes(const P2PPtrs& codes, int rank, int64_t i, uint32_t w) {
#pragma unroll
  for (int r = 0; r < M; ++r) {
    const int rr = (rank + r) % M;  // own first, then the peers in rotated order
    const void* base = nullptr;
#pragma unroll
    for (int j = 0; j < M; ++j)
      if (j == rr) base = codes.p[j];
    *reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(const_cast<void*>(base)) + i) = w;
  }
}
template <int M>
__device__ __forceinline__ void put_code(const P2PPtrs& codes, int64_t i, uint8_t c) {
#pragma unroll
  for (int r = 0; r < M; ++r) static_cast<uint8_t*>(const_cast<void*>(codes.p[r]))[i] = c;
}

template <int M, bool SYNC>
__global__ void __launch_bounds__(FP8_NT) fp8_quant_ag_kernel(const Fp8Tile* __restrict__ tiles,
                                                             int64_t ntiles, const float* __restrict__ master,
                                                             P2PPtrs codes, P2PPtrs scales, int rank,
                                                             P2PSignals sg, uint64_t epoch) {
  __shared__ float red[FP8_WARPS];
  if constexpr (SYNC) p2p_start(sg, rank, M, epoch);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Fp8Tile T = tiles[t];
    float A;
    const bool vec = T.rows <= 128 && T.cols <= 128 && (T.cols & 3) == 0 && (T.pitch & 3) == 0 &&
                     (T.off & 3) == 0;
    if (vec) {
      float4 x[16];
      float a = 0.f;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int row = w + FP8_WARPS * k, col = 4 * lane;
        if (row < T.rows && col < T.cols) {
          x[k] = __ldcs(reinterpret_cast<const float4*>(master + T.off + int64_t(row) * T.pitch + col));
          a = fmax_nan(a, fmax_nan(fmax_nan(fabsf(x[k].x), fabsf(x[k].y)), fmax_nan(fabsf(x[k].z), fabsf(x[k].w))));
        } else {
          x[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      A = block_absmax(a, red);
      const float inv = tile_inv(A);
      const uint32_t fixed = A > 0.f ? 0x7F7F7F7Fu : 0u;  // zero tile: codes 0 (R19); NaN/inf tile: NaN (R28)
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int row = w + FP8_WARPS * k, col = 4 * lane;
        if (row < T.rows && col < T.cols) {
          const uint32_t c = A > 0.f && A <= FLT_MAX_F
                                 ? e4m3x4(__fmul_rn(x[k].x, inv), __fmul_rn(x[k].y, inv),
                                          __fmul_rn(x[k].z, inv), __fmul_rn(x[k].w, inv))
                                 : fixed;
          put_codes<M>(codes, rank, T.off + int64_t(row) * T.pitch + col, c);
        }
      }
    } else {
      // generic tile (odd widths / misaligned rows): element-wise, two passes
      const int n = T.rows * T.cols;
      float a = 0.f;
      for (int e = threadIdx.x; e < n; e += FP8_NT) {
        const int row = e / T.cols, col = e - row * T.cols;
        a = fmax_nan(a, fabsf(master[T.off + int64_t(row) * T.pitch + col]));
      }
      A = block_absmax(a, red);
      const float inv = tile_inv(A);
      const uint8_t fixed = A > 0.f ? 0x7F : 0;
      for (int e = threadIdx.x; e < n; e += FP8_NT) {
        const int row = e / T.cols, col = e - row * T.cols;
        const int64_t o = T.off + int64_t(row) * T.pitch + col;
        put_code<M>(codes, o, A > 0.f && A <= FLT_MAX_F ? uint8_t(e4m3x2(__fmul_rn(master[o], inv), 0.f) & 0xffu)
                                                       : fixed);
      }
    }
    if (threadIdx.x == 0) {
      // scale fl(A / 448); A = 0 -> 0; NaN / +inf kept (R28)
      const float sc = A <= FLT_MAX_F ? __fdiv_rn(A, E4M3_MAX) : A;
#pragma unroll
      for (int r = 0; r < M; ++r) static_cast<float*>(const_cast<void*>(scales.p[r]))[T.slot] = sc;
    }
  }
  if constexpr (SYNC) p2p_done(sg, rank, M, epoch);
}

template <int M, bool SYNC>
static cudaError_t fp8_mbs(const Fp8Tile* tiles, int64_t ntiles, const float* master, const P2PPtrs& codes,
                           const P2PPtrs& scales, int rank, const P2PSignals& sg, uint64_t epoch,
                           cudaStream_t st) {
  static const int grid = [] {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fp8_quant_ag_kernel<M, SYNC>, FP8_NT, 0);
    return num_sms() * (b < 1 ? 1 : b);
  }();
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(ntiles, grid_share(grid, sg)));
  fp8_quant_ag_kernel<M, SYNC><<<blocks, FP8_NT, 0, st>>>(tiles, ntiles, master, codes, scales, rank, sg,
                                                          epoch);
  return cudaGetLastError();
}

cudaError_t launch_fp8_quant_ag(const Fp8Tile* tiles, int64_t ntiles, const float* master, const P2PPtrs& codes,
                                const P2PPtrs& scales, int m, int rank, const P2PSignals* sg, uint64_t epoch,
                                cudaStream_t st) {
  if (m == 1) return fp8_mbs<1, false>(tiles, ntiles, master, codes, scales, rank, P2PSignals{}, 0, st);
  if (!sg) return cudaErrorInvalidValue;
  switch (m) {
#define FP8_CASE(MM) \
  case MM:           \
    return fp8_mbs<MM, true>(tiles, ntiles, master, codes, scales, rank, *sg, epoch, st);
    FP8_CASE(2) FP8_CASE(3) FP8_CASE(4) FP8_CASE(5) FP8_CASE(6) FP8_CASE(7) FP8_CASE(8)
#undef FP8_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace rsdb
