// N2: block-wise 8-bit Adam with the dynamic (tree) code map
// of Dettmers et al. (reading R25) instead of the linear absmax code.
//
// The two 256-entry maps (signed for m, unsigned for v) are built on the host
// in double exactly as R25 writes them, rounded once to float and kept in
// __constant__ memory together with bucket tables; every CTA copies them to
// shared memory.  Per block: dequantise (map[code] * A), the same fp32 AdamW
// update as the linear kernels (adam_elem), block absmax, then requantise
// each moment to the nearest map value of y = fl(m / A) -- the oracle's
// decision in the oracle's precision: hi = first code with map[hi] >= y,
// code = hi if fl(map[hi] - y) < fl(y - map[hi-1]) else hi - 1.  hi is found
// without a binary search: a 1792-entry table indexed by the exponent and 6
// mantissa bits of |y| (one bucket spans <= 1.6 % in value, <= 2 map values)
// gives a lower bound, corrected by a short forward scan.  Full contiguous
// 2048-element blocks use 16-B vector loads (4 elements per thread per quad);
// other blocks a masked element path; blocks > 2048 elements two passes.
#include <cuda_bf16.h>

#include <cmath>
#include <cstdint>
#include <cstring>

#include "adam_dev.cuh"
#include "kernels.cuh"

namespace rsdb {

constexpr int DYN_NT = 256;
constexpr int DYN_E0 = 100;                        // |y| < 2^(100-127) share bucket 0
constexpr int DYN_NB = (127 - DYN_E0 + 1) * 64;    // buckets: exponents E0..127 x 6 mantissa bits

struct DynTables {
  float map[2][256];              // [0] signed (first moment), [1] unsigned (second)
  uint8_t lb[3][DYN_NB];          // lower bounds of hi: [0] signed y>0, [1] signed y<0, [2] unsigned
};
__constant__ DynTables c_dyn;

__host__ __device__ inline int dyn_bucket(float a) {  // a = |y| >= 0
  uint32_t bits;
  memcpy(&bits, &a, 4);
  const int k = int(bits >> 17) - (DYN_E0 << 6);
  return k < 0 ? 0 : (k >= DYN_NB ? DYN_NB - 1 : k);
}

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
  for (int a = 1; a < 256; ++a)  // insertion sort (host, once)
    for (int b = a; b > 0 && v[b - 1] > v[b]; --b) std::swap(v[b - 1], v[b]);
  for (int a = 0; a < 256; ++a) out[a] = v[a];
}

void dyn_maps(float m_map[256], float v_map[256]) {
  build_dyn_map(true, m_map);
  build_dyn_map(false, v_map);
}

// lower bound of "first index with map >= y" over every y in bucket b of sign s
static void build_lb(const float* map, bool negative, uint8_t* lb) {
  for (int b = 0; b < DYN_NB; ++b) {
    // bucket b holds |y| in [lo, hi): lo = float with bits (b + E0*64) << 17
    uint32_t lo_bits = uint32_t(b + (DYN_E0 << 6)) << 17, hi_bits = lo_bits + (1u << 17);
    float lo, hi;
    memcpy(&lo, &lo_bits, 4);
    memcpy(&hi, &hi_bits, 4);
    if (b == 0) lo = 0.f;
    const float ymin = negative ? -hi : lo;  // smallest y of the bucket
    int k = 0;
    while (k < 255 && map[k] < ymin) ++k;
    lb[b] = uint8_t(k);
  }
}

static cudaError_t ensure_dyn_tables() {
  static bool done = false;
  if (done) return cudaSuccess;
  static DynTables h;
  dyn_maps(h.map[0], h.map[1]);
  build_lb(h.map[0], false, h.lb[0]);
  build_lb(h.map[0], true, h.lb[1]);
  build_lb(h.map[1], false, h.lb[2]);
  const cudaError_t e = cudaMemcpyToSymbol(c_dyn, &h, sizeof h);
  if (e == cudaSuccess) done = true;
  return e;
}

// nearest map value of y (R25): hi from the bucket bound + forward scan
__device__ __forceinline__ uint32_t dyn_code(const float* map, const uint8_t* lb_pos, const uint8_t* lb_neg,
                                             float y) {
  int hi = (y < 0.f ? lb_neg : lb_pos)[dyn_bucket(fabsf(y))];
  while (hi < 255 && map[hi] < y) ++hi;
  hi = hi < 1 ? 1 : hi;
  const float d_hi = __fsub_rn(map[hi], y);
  const float d_lo = __fsub_rn(y, map[hi - 1]);
  return uint32_t(d_hi < d_lo ? hi : hi - 1);
}

struct DynSmem {
  float map[2][256];
  uint8_t lb[3][DYN_NB];
};

template <bool PARAM_BF16>
__global__ void __launch_bounds__(DYN_NT) adam8_dyn_kernel(const AdamBlock* __restrict__ tbl, int64_t nblocks,
                                                          AdamPtrs P, AdamScalars s) {
  __shared__ DynSmem T;
  __shared__ float red_m[2][DYN_NT / 32], red_v[2][DYN_NT / 32];
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(&c_dyn);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&T);
    for (int i = threadIdx.x; i < int(sizeof(DynSmem) / 4); i += DYN_NT) dst[i] = src[i];
  }
  __syncthreads();
  const float* mapm = T.map[0];
  const float* mapv = T.map[1];
  constexpr uint32_t zero_m = 127, zero_v = 0;  // codes of 0.0 in the two maps
  uint8_t* mq = reinterpret_cast<uint8_t*>(P.mq);
  using G = AdamGeom<DYN_NT>;  // 2 quads per thread
  int it = 0;
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++it) {
    const AdamBlock blk = tbl[b];
    const float Am = P.mabs[blk.slot], Av = P.vabs[blk.slot];
    float* rm = red_m[it & 1];
    float* rv = red_v[it & 1];
    // R27: A = 0, NaN or +inf -> the code of 0 everywhere
    auto qm = [&](float m, float am) {
      return am > 0.f && am <= FLT_MAX_F ? dyn_code(mapm, T.lb[0], T.lb[1], __fdiv_rn(m, am)) : zero_m;
    };
    auto qv = [&](float v, float av) {
      return av > 0.f && av <= FLT_MAX_F ? dyn_code(mapv, T.lb[2], T.lb[2], __fdiv_rn(v, av)) : zero_v;
    };
    float am = 0.f, av = 0.f;
    const bool fast = blk.len == ADAM_TILE && blk.cols == blk.len && (blk.state_off & 3) == 0 &&
                      (blk.grad_off & 3) == 0 && (blk.param_off & 3) == 0;
    if (fast) {
      float p[G::EPT], m[G::EPT], v[G::EPT];
#pragma unroll
      for (int k = 0; k < G::Q; ++k) {
        const int a = G::quad(k);
        const int4 pv = ld_na_v4(P.master + blk.state_off + a);
        const int4 gv = ld_nc_v4(P.grad + blk.grad_off + a);
        const uint32_t cm = ld_na_u32(mq + blk.state_off + a);
        const uint32_t cv = ld_na_u32(P.vq + blk.state_off + a);
        const float pp[4] = {__int_as_float(pv.x), __int_as_float(pv.y), __int_as_float(pv.z),
                             __int_as_float(pv.w)};
        const float gg[4] = {__int_as_float(gv.x), __int_as_float(gv.y), __int_as_float(gv.z),
                             __int_as_float(gv.w)};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float mt = __fmul_rn(mapm[(cm >> (8 * j)) & 0xffu], Am);
          const float vt = __fmul_rn(mapv[(cv >> (8 * j)) & 0xffu], Av);
          const ElemOut r = adam_elem(pp[j], gg[j], mt, vt, s);
          p[4 * k + j] = r.p;
          m[4 * k + j] = r.m;
          v[4 * k + j] = r.v;
          am = fmax_nan(am, fabsf(r.m));
          av = fmax_nan(av, r.v);
        }
      }
      block_max2<G::WARPS>(am, av, rm, rv);
#pragma unroll
      for (int k = 0; k < G::Q; ++k) {
        const int a = G::quad(k);
        const float* pk = &p[4 * k];
        st_f4(P.master + blk.state_off + a, make_float4(pk[0], pk[1], pk[2], pk[3]));
        st_u32(mq + blk.state_off + a, qm(m[4 * k], am) | (qm(m[4 * k + 1], am) << 8) |
                                           (qm(m[4 * k + 2], am) << 16) | (qm(m[4 * k + 3], am) << 24));
        st_u32(P.vq + blk.state_off + a, qv(v[4 * k], av) | (qv(v[4 * k + 1], av) << 8) |
                                             (qv(v[4 * k + 2], av) << 16) | (qv(v[4 * k + 3], av) << 24));
        if constexpr (PARAM_BF16)
          st_u2(static_cast<uint16_t*>(P.param) + blk.param_off + a,
                make_uint2(pack_bf16x2(pk[0], pk[1]), pack_bf16x2(pk[2], pk[3])));
        else
          st_f4(static_cast<float*>(P.param) + blk.param_off + a, make_float4(pk[0], pk[1], pk[2], pk[3]));
      }
    } else {
      auto elem = [&](int i, float& m, float& v) -> float {  // update element i, returns new p
        const int64_t o = blk_off(blk, i);
        const float mt = __fmul_rn(mapm[mq[blk.state_off + o]], Am);
        const float vt = __fmul_rn(mapv[P.vq[blk.state_off + o]], Av);
        const ElemOut r = adam_elem(P.master[blk.state_off + o], P.grad[blk.grad_off + o], mt, vt, s);
        m = r.m;
        v = r.v;
        return r.p;
      };
      auto store = [&](int i, float p, float m, float v) {
        const int64_t o = blk_off(blk, i);
        P.master[blk.state_off + o] = p;
        mq[blk.state_off + o] = uint8_t(qm(m, am));
        P.vq[blk.state_off + o] = uint8_t(qv(v, av));
        if constexpr (PARAM_BF16)
          static_cast<__nv_bfloat16*>(P.param)[blk.param_off + o] = __float2bfloat16_rn(p);
        else
          static_cast<float*>(P.param)[blk.param_off + o] = p;
      };
      constexpr int EPT = ADAM_TILE / DYN_NT;
      if (blk.len <= ADAM_TILE) {
        float p[EPT], m[EPT], v[EPT];
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          const int i = int(threadIdx.x) + e * DYN_NT;
          if (i < blk.len) {
            p[e] = elem(i, m[e], v[e]);
            am = fmax_nan(am, fabsf(m[e]));
            av = fmax_nan(av, v[e]);
          }
        }
        block_max2<G::WARPS>(am, av, rm, rv);
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          const int i = int(threadIdx.x) + e * DYN_NT;
          if (i < blk.len) store(i, p[e], m[e], v[e]);
        }
      } else {  // two passes: absmax, then recompute + store (each thread owns its elements)
        for (int i = threadIdx.x; i < blk.len; i += DYN_NT) {
          float m, v;
          elem(i, m, v);
          am = fmax_nan(am, fabsf(m));
          av = fmax_nan(av, v);
        }
        block_max2<G::WARPS>(am, av, rm, rv);
        for (int i = threadIdx.x; i < blk.len; i += DYN_NT) {
          float m, v;
          const float p = elem(i, m, v);
          store(i, p, m, v);
        }
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
  if (cudaError_t e = ensure_dyn_tables()) return e;
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
