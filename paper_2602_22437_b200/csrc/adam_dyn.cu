// N2: block-wise 8-bit Adam with the dynamic (tree) code map
// of Dettmers et al. (reading R25) instead of the linear absmax code.
//
// The two 256-entry maps (signed for m, unsigned for v) are built on the host
// in double exactly as R25 writes them, rounded once to float and kept in
// __constant__ memory; every CTA copies them to shared memory.  Per block:
// dequantise (map[code] * A), the same fp32 AdamW update as the linear
// kernels (adam_elem), block absmax, then requantise each moment to the
// nearest map value of y = m / A: an 8-step branch-free binary search over
// the shared-memory map and one fp32 distance comparison (ties -> lower
// code), i.e. the oracle's decision in the oracle's precision.  One
// 256-thread CTA per block (8 elements per thread in registers); blocks
// longer than 2048 elements take a two-pass loop.  A variant for the
// paper's setting, not the bench default: the map lookups make it ALU/LSU
// heavier than the linear codec (~16 shared loads per element).
#include <cuda_bf16.h>

#include <cmath>
#include <cstdint>

#include "adam_dev.cuh"
#include "kernels.cuh"

namespace rsdb {

constexpr int DYN_NT = 256;
constexpr int DYN_EPT = ADAM_TILE / DYN_NT;  // 8

__constant__ float c_dyn_map[2][256];  // [0] signed (first moment), [1] unsigned (second)

// R25: values +-D_i * (0.1 + (j + 0.5) * (0.9 / (n - 1))), D_i = 1e-6 .. 1e0,
// n = 2^i + 1 (signed) or 2^(i+1) + 1 (unsigned); plus 0 and 1; ascending
static void build_dyn_map(bool is_signed, float out[256]) {
  static const double D[7] = {1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 1e-1, 1e0};
  float v[256];
  int k = 0;
  v[k++] = 0.0f;
  v[k++] = 1.0f;
  for (int i = 0; i < 7; ++i) {
    const int n = (is_signed ? (1 << i) : (1 << (i + 1))) + 1;
    for (int j = 0; j < n - 1; ++j) {
      const double mu = 0.1 + (j + 0.5) * (0.9 / (n - 1));
      v[k++] = float(D[i] * mu);
      if (is_signed) v[k++] = float(-(D[i] * mu));
    }
  }
  // insertion sort (256 values, host, once)
  for (int a = 1; a < 256; ++a)
    for (int b = a; b > 0 && v[b - 1] > v[b]; --b) std::swap(v[b - 1], v[b]);
  for (int a = 0; a < 256; ++a) out[a] = v[a];
}

void dyn_maps(float m_map[256], float v_map[256]) {
  build_dyn_map(true, m_map);
  build_dyn_map(false, v_map);
}

static cudaError_t ensure_dyn_maps() {
  static bool done = false;
  if (done) return cudaSuccess;
  float h[2][256];
  dyn_maps(h[0], h[1]);
  const cudaError_t e = cudaMemcpyToSymbol(c_dyn_map, h, sizeof h);
  if (e == cudaSuccess) done = true;
  return e;
}

__device__ __forceinline__ uint32_t dyn_code(const float* map, float y) {
  int lo = 0;  // number of map values < y (capped at 255)
#pragma unroll
  for (int st = 128; st >= 1; st >>= 1)
    if (map[lo + st - 1] < y) lo += st;
  const int hi = lo < 1 ? 1 : lo;
  const float d_hi = __fsub_rn(map[hi], y);
  const float d_lo = __fsub_rn(y, map[hi - 1]);
  return uint32_t(d_hi < d_lo ? hi : hi - 1);
}

template <bool PARAM_BF16>
__global__ void __launch_bounds__(DYN_NT) adam8_dyn_kernel(const AdamBlock* __restrict__ tbl, int64_t nblocks,
                                                          AdamPtrs P, AdamScalars s) {
  __shared__ float mapm[256], mapv[256];
  __shared__ float red_m[2][DYN_NT / 32], red_v[2][DYN_NT / 32];
  mapm[threadIdx.x] = c_dyn_map[0][threadIdx.x];
  mapv[threadIdx.x] = c_dyn_map[1][threadIdx.x];
  __syncthreads();
  const uint32_t zero_m = 127, zero_v = 0;  // codes of 0.0 in the two maps
  uint8_t* mq = reinterpret_cast<uint8_t*>(P.mq);
  int it = 0;
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++it) {
    const AdamBlock blk = tbl[b];
    const float Am = P.mabs[blk.slot], Av = P.vabs[blk.slot];
    float* rm = red_m[it & 1];
    float* rv = red_v[it & 1];
    auto elem = [&](int i, float& m, float& v) -> float {  // update element i, returns new p
      const int64_t o = blk_off(blk, i);
      const float mt = __fmul_rn(mapm[mq[blk.state_off + o]], Am);
      const float vt = __fmul_rn(mapv[P.vq[blk.state_off + o]], Av);
      const ElemOut r = adam_elem(P.master[blk.state_off + o], P.grad[blk.grad_off + o], mt, vt, s);
      m = r.m;
      v = r.v;
      return r.p;
    };
    auto store = [&](int i, float p, float m, float v, float am, float av) {
      const int64_t o = blk_off(blk, i);
      P.master[blk.state_off + o] = p;
      mq[blk.state_off + o] = uint8_t(am > 0.f ? dyn_code(mapm, __fdiv_rn(m, am)) : zero_m);
      P.vq[blk.state_off + o] = uint8_t(av > 0.f ? dyn_code(mapv, __fdiv_rn(v, av)) : zero_v);
      if constexpr (PARAM_BF16)
        static_cast<__nv_bfloat16*>(P.param)[blk.param_off + o] = __float2bfloat16_rn(p);
      else
        static_cast<float*>(P.param)[blk.param_off + o] = p;
    };
    float am = 0.f, av = 0.f;
    if (blk.len <= ADAM_TILE) {
      float p[DYN_EPT], m[DYN_EPT], v[DYN_EPT];
#pragma unroll
      for (int e = 0; e < DYN_EPT; ++e) {
        const int i = int(threadIdx.x) + e * DYN_NT;
        if (i < blk.len) {
          p[e] = elem(i, m[e], v[e]);
          am = fmaxf(am, fabsf(m[e]));
          av = fmaxf(av, v[e]);
        }
      }
      block_max2<DYN_NT / 32>(am, av, rm, rv);
#pragma unroll
      for (int e = 0; e < DYN_EPT; ++e) {
        const int i = int(threadIdx.x) + e * DYN_NT;
        if (i < blk.len) store(i, p[e], m[e], v[e], am, av);
      }
    } else {  // two passes: absmax, then recompute + store (inputs are read twice)
      for (int i = threadIdx.x; i < blk.len; i += DYN_NT) {
        float m, v;
        elem(i, m, v);
        am = fmaxf(am, fabsf(m));
        av = fmaxf(av, v);
      }
      block_max2<DYN_NT / 32>(am, av, rm, rv);
      __syncthreads();  // every thread has read the old state before anyone stores
      for (int i = threadIdx.x; i < blk.len; i += DYN_NT) {
        float m, v;
        const float p = elem(i, m, v);
        store(i, p, m, v, am, av);
      }
    }
    if (threadIdx.x == 0) {
      P.mabs[blk.slot] = am;
      P.vabs[blk.slot] = av;
    }
  }
}

cudaError_t launch_adam8_dyn(const AdamBlock* tbl, int64_t nblocks, const AdamPtrs& p, const AdamScalars& s,
                             cudaStream_t st) {
  if (nblocks == 0) return cudaSuccess;
  if (cudaError_t e = ensure_dyn_maps()) return e;
  int per = 0;
  if (p.param_bf16)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, adam8_dyn_kernel<true>, DYN_NT, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, adam8_dyn_kernel<false>, DYN_NT, 0);
  const int64_t cap = int64_t(num_sms()) * (per < 1 ? 1 : per);
  const int grid = int(nblocks < cap ? nblocks : cap);
  if (p.param_bf16)
    adam8_dyn_kernel<true><<<grid, DYN_NT, 0, st>>>(tbl, nblocks, p, s);
  else
    adam8_dyn_kernel<false><<<grid, DYN_NT, 0, st>>>(tbl, nblocks, p, s);
  return cudaGetLastError();
}

}  // namespace rsdb
