// N2: block-wise 8-bit Adam with the dynamic (tree) code map
// of Dettmers et al. (reading R25) instead of the linear absmax code.
//
// The two 256-entry maps (signed for m, unsigned for v) are built on the host
// in double exactly as R25 writes them, rounded once to float and kept in
// __constant__ memory; every CTA copies them to shared memory REPLICATED PER
// LANE (map[k] at word k * 32 + lane), so the data-dependent lookups of a warp
// never conflict on a bank (the round-1 kernel, with one copy and a bucket
// table, was bound by 3-4-way conflicted lookups at 0.39 of HBM).  Per block:
// dequantise (map[code] * A), the same fp32 AdamW update as the linear
// kernels (adam_elem), block absmax, then requantise each moment to the
// nearest map value of y = fl(m / A) -- the oracle's decision in the oracle's
// precision: hi = first code with map[hi] >= y (clamped to [1, 255]), code =
// hi if fl(map[hi] - y) < fl(y - map[hi-1]) else hi - 1.  hi is found from
// the map's closed form (R25: decade i holds 2^i (signed) / 2^(i+1)
// (unsigned) equally spaced values of [0.1 D_i, D_i]): decade by six fp32
// comparisons, index inside the decade by one multiply-add, then two
// correcting scans on the exact fp32 map values (normally zero steps), so
// the decision is the table's, not the approximation's.  Full contiguous
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

struct DynTables {
  float map[2][256];  // [0] signed (first moment), [1] unsigned (second)
};
__constant__ DynTables c_dyn;

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

static cudaError_t ensure_dyn_tables() {
  static bool done = false;
  if (done) return cudaSuccess;
  static DynTables h;
  dyn_maps(h.map[0], h.map[1]);
  const cudaError_t e = cudaMemcpyToSymbol(c_dyn, &h, sizeof h);
  if (e == cudaSuccess) done = true;
  return e;
}

// lane-replicated map: entry k of this lane's copy
__device__ __forceinline__ float rmap(const float* rep, int k, int lane) { return rep[(k << 5) | lane]; }

// Candidate position of a = |y| <= 1 among the map's positive decade values
// (R25 closed form; decade i holds 2^(i+w) equally spaced values of
// [0.1 D_i, D_i], w = 0 signed / 1 unsigned, whose first index is 128 + 2^i - 1
// (signed) or 2^(i+1) - 1 (unsigned)).  Plain fp32 operations (_rn: no FMA
// contraction) so tests/test_dyn_candidate.py can replay it bit for bit:
// for EVERY fp32 y in [-1, 1] the true hi (first index with map >= y,
// clamped to [1, 255]) lies within one of the clamped candidate.
// per-binade decade table (shared memory, 32 entries -- any lane pattern of
// <= 32 distinct words is bank-conflict free up to the 8-B entry pairing):
// for the binade [2^(E-127), 2^(E-126)) of biased exponent E = DYN_E0 + e,
// x = the decade count of its lower end (#{thresholds 1e-6 .. 1e-1 <= 2^(E-127)})
// and y = the one threshold inside the binade (bits; +inf if none).  Then
// #{thresholds <= a} = x + (a >= y) for every a in the binade -- the same
// comparisons as a six-step cascade on the same float thresholds.
constexpr int DYN_E0 = 100;  // 2^-27 < 1e-6 / 10: everything below is decade 0
struct DynDecade {
  int2 bin[32];     // {decade count at the binade's start, threshold bits}
  float dinv[8];    // 10^(6 - i), i = 0..6
};
__device__ __forceinline__ float dyn_th(int k) {  // thresholds 1e-6 .. 1e-1 (float32)
  return k == 0 ? 1e-6f : k == 1 ? 1e-5f : k == 2 ? 1e-4f : k == 3 ? 1e-3f : k == 4 ? 1e-2f : 1e-1f;
}
__device__ __forceinline__ void dyn_decade_init(DynDecade& D) {
  const int e = int(threadIdx.x);
  if (e < 32) {
    const float lo = __uint_as_float(uint32_t(DYN_E0 + e) << 23), hi = 2.f * lo;
    int cnt = 0;
    float t = __uint_as_float(0x7f800000u);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      if (dyn_th(k) <= lo) ++cnt;
      else if (dyn_th(k) < hi) t = dyn_th(k);
    }
    D.bin[e] = make_int2(cnt, int(__float_as_uint(t)));
  } else if (e < 32 + 7) {
    const int i = e - 32;  // 10^(6 - i)
    D.dinv[i] = i == 0 ? 1e6f : i == 1 ? 1e5f : i == 2 ? 1e4f : i == 3 ? 1e3f : i == 4 ? 1e2f : i == 5 ? 1e1f : 1.f;
  }
}

template <bool SIGNED>
__device__ __forceinline__ int dyn_candidate(const DynDecade& D, float a) {
  constexpr int W = SIGNED ? 0 : 1;
  int e = int(__float_as_uint(a) >> 23) - DYN_E0;  // a >= 0, <= 1: e <= 27
  e = e < 0 ? 0 : e;
  const int2 bt = D.bin[e];
  const int i = bt.x + int(a >= __int_as_float(bt.y));
  const float Dinv = D.dinv[i];
  const int cnt = 1 << (i + W);
  float u = __fsub_rn(__fmul_rn(a, Dinv), 0.1f);
  u = __fmul_rn(__fmul_rn(u, __int2float_rn(cnt)), 1.0f / 0.9f);
  int j = __float2int_rn(__fsub_rn(u, 0.5f));
  j = min(max(j, 0), cnt - 1);
  return (SIGNED ? 127 : 0) + cnt + j;
}

// nearest map value of y (R25, the oracle's fp32 rule; ties -> lower code),
// branch free: hi is one of c-1, c, c+1 (c the clamped candidate), decided by
// two comparisons on the exact map values map[c-2 .. c+1] (4 conflict-free
// lookups in this lane's copy)
template <bool SIGNED>
__device__ __forceinline__ uint32_t dyn_code(const float* rep, const DynDecade& D, int lane, float y) {
  int c;
  if (SIGNED) {
    const int p = dyn_candidate<true>(D, fabsf(y));
    c = y < 0.f ? 255 - p : p;  // -map[p] sits at 254 - p; hi is the index after it
  } else {
    c = dyn_candidate<false>(D, y);
  }
  c = c < 2 ? 2 : (c > 254 ? 254 : c);
  const float* q = rep + ((c - 2) << 5) + lane;
  const float v0 = q[0], v1 = q[32], v2 = q[64], v3 = q[96];
  const bool a1 = v1 >= y, a2 = v2 >= y;
  const int hi = a1 ? c - 1 : (a2 ? c : c + 1);
  const float hv = a1 ? v1 : (a2 ? v2 : v3);
  const float lv = a1 ? v0 : (a2 ? v1 : v2);
  return uint32_t(__fsub_rn(hv, y) < __fsub_rn(y, lv) ? hi : hi - 1);
}

// y = fl32(x / A) through fp64: float(double(x) * RN64(1/A)) -- the relative
// error of the double product (< 2^-51.9) is below the distance of any
// quotient of two floats to a float rounding boundary (>= 2^-49 relative),
// so this is exactly the IEEE fp32 quotient the oracle takes (no slow path,
// no branch); rA = 1.0 / double(A) once per block
__device__ __forceinline__ float div_exact(float x, double rA) {
  return __double2float_rn(__dmul_rn(double(x), rA));
}

struct DynSmem {
  float rep[2][256 * 32];  // lane-replicated maps (64 KB)
};

template <bool PARAM_BF16>
__global__ void __launch_bounds__(DYN_NT, 3) adam8_dyn_kernel(const AdamBlock* __restrict__ tbl, int64_t nblocks,
                                                          AdamPtrs P, AdamScalars s) {
  extern __shared__ __align__(16) float dyn_smem[];
  DynSmem& T = *reinterpret_cast<DynSmem*>(dyn_smem);
  __shared__ float red_m[2][DYN_NT / 32], red_v[2][DYN_NT / 32];
  __shared__ DynDecade dec;
  dyn_decade_init(dec);
  for (int i = threadIdx.x; i < 2 * 256 * 32; i += DYN_NT) {
    const int w = i >> 13, k = (i >> 5) & 255;
    T.rep[w][i & 8191] = c_dyn.map[w][k];
  }
  __syncthreads();
  const int lane = int(threadIdx.x) & 31;
  const float* mapm = T.rep[0];
  const float* mapv = T.rep[1];
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
    // block-uniform: A finite and > 0 (else the code of 0), 1/A in fp64
    double rAm = 0.0, rAv = 0.0;
    bool okm = false, okv = false;
    auto qm = [&](float m, float) { return okm ? dyn_code<true>(mapm, dec, lane, div_exact(m, rAm)) : zero_m; };
    auto qv = [&](float v, float) { return okv ? dyn_code<false>(mapv, dec, lane, div_exact(v, rAv)) : zero_v; };
    auto set_div = [&](float am_, float av_) {
      okm = am_ > 0.f && am_ <= FLT_MAX_F;
      okv = av_ > 0.f && av_ <= FLT_MAX_F;
      rAm = okm ? 1.0 / double(am_) : 0.0;
      rAv = okv ? 1.0 / double(av_) : 0.0;
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
          const float mt = __fmul_rn(rmap(mapm, int((cm >> (8 * j)) & 0xffu), lane), Am);
          const float vt = __fmul_rn(rmap(mapv, int((cv >> (8 * j)) & 0xffu), lane), Av);
          const ElemOut r = adam_elem(pp[j], gg[j], mt, vt, s);
          p[4 * k + j] = r.p;
          m[4 * k + j] = r.m;
          v[4 * k + j] = r.v;
          am = fmax_nan(am, fabsf(r.m));
          av = fmax_nan(av, r.v);
        }
      }
      block_max2<G::WARPS>(am, av, rm, rv);
      set_div(am, av);
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
        const float mt = __fmul_rn(rmap(mapm, mq[blk.state_off + o], lane), Am);
        const float vt = __fmul_rn(rmap(mapv, P.vq[blk.state_off + o], lane), Av);
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
        set_div(am, av);
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
        set_div(am, av);
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
  constexpr int smem = int(sizeof(DynSmem));
  static bool attr = false;
  if (!attr) {
    if (cudaError_t e = cudaFuncSetAttribute(adam8_dyn_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))
      return e;
    if (cudaError_t e = cudaFuncSetAttribute(adam8_dyn_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))
      return e;
    attr = true;
  }
  int per = 0;
  if (p.param_bf16)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, adam8_dyn_kernel<true>, DYN_NT, smem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, adam8_dyn_kernel<false>, DYN_NT, smem);
  const int64_t cap = int64_t(num_sms()) * (per < 1 ? 1 : per);
  const int grid = int(nblocks < cap ? nblocks : cap);
  if (p.param_bf16)
    adam8_dyn_kernel<true><<<grid, DYN_NT, smem, st>>>(tbl, nblocks, p, s);
  else
    adam8_dyn_kernel<false><<<grid, DYN_NT, smem, st>>>(tbl, nblocks, p, s);
  return cudaGetLastError();
}

}  // namespace rsdb
