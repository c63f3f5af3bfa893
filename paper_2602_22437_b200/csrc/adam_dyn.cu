// N2: block-wise 8-bit Adam with the dynamic (tree) code map
// of Dettmers et al. (reading R25) instead of the linear absmax code.
//
// The two 256-entry maps (signed for m, unsigned for v) are built on the host
// in double exactly as R25 writes them and rounded once to float.  Per block:
// dequantise (map[code] * A), the same fp32 AdamW update as the linear
// kernels (adam_elem), block absmax, then requantise each moment to the
// nearest map value of y = fl(m / A) -- the oracle's decision in the oracle's
// precision: hi = first code with map[hi] >= y (clamped to [1, 255]), code =
// hi if fl(map[hi] - y) < fl(y - map[hi-1]) else hi - 1.
//
// That decision is a non-decreasing step function of y with 255 steps, so
// the kernel does not search the map: it looks it up.  The host cuts the
// fp32 values of [-1, 1] into bins by their sign, exponent and top MB
// mantissa bits (MB = 6 signed / 7 unsigned; magnitudes below 2^-27 share the
// first bin) and evaluates the decision rule itself at the bin ends.  Every
// bin holds at most one step: neighbouring map values of decade i lie
// 0.9 D_i / 2^i (signed) or / 2^(i+1) (unsigned) apart, wider than any bin
// (2^e / 2^MB for the binade [2^e, 2^(e+1)) below D_i) -- and
// build_dyn_table checks it, the launch fails otherwise.  So one 32-bit
// entry per bin -- the code at the bin's low end and the low mantissa bits
// where the step sits -- gives the code with one lookup and one integer
// comparison: ~10 instructions per moment instead of the ~40 of the
// closed-form search it replaces (profiles/r2/dyn/).  The
// tables are exported by rsdb_dynamic_code_tables; tests/test_dyn_table.py
// replays the lookup against the oracle's rule, and
// tests/dyn_table_exhaustive.py over every fp32 y in [-1, 1].
// Full contiguous 2048-element blocks use 16-B vector loads (4 elements per
// thread per quad); other blocks a masked element path; blocks > 2048
// elements two passes.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <type_traits>

#include "adam_dev.cuh"
#include "kernels.cuh"

namespace rsdb {

constexpr int DYN_NT = 256;
constexpr int DYN_E0 = 100;  // first binade with its own bins: [2^-27, 2^-26)
constexpr int DYN_MB_M = 6, DYN_MB_V = 7;  // mantissa bits of the bin index
constexpr int DYN_NB_M = 28 << DYN_MB_M;   // bins per sign, binades 2^-27 .. 2^0
constexpr int DYN_NB_V = 28 << DYN_MB_V;
static_assert(DYN_TABLE_M_LEN == 2 * DYN_NB_M && DYN_TABLE_V_LEN == DYN_NB_V, "table sizes");

struct DynTables {
  float map[2][256];              // [0] signed (first moment), [1] unsigned (second)
  uint32_t tm[2 * DYN_NB_M];      // signed: [sign][bin]
  uint32_t tv[DYN_NB_V];          // unsigned
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

// the decision rule (host, fp32 arithmetic)
static int dyn_rule(const float map[256], float y) {
  int hi = int(std::lower_bound(map, map + 256, y) - map);  // first map[hi] >= y
  hi = hi < 1 ? 1 : (hi > 255 ? 255 : hi);
  const float d_hi = map[hi] - y, d_lo = y - map[hi - 1];
  return d_hi < d_lo ? hi : hi - 1;
}
static float fbits(uint32_t b) {
  float f;
  std::memcpy(&f, &b, 4);
  return f;
}

// Entry of bin `idx` (magnitude bits [L, L + 2^SH), SH = 23 - MB; bin 0 also
// takes every magnitude below) on side `neg`: bits 31..24 the code at the
// bin's low end in y (the largest magnitude when negative), bits 23..0 the
// comparison value: with yl = mag & LOW (positive) or LOW - (mag & LOW)
// (negative), code = c0 + (yl >= thr); thr = LOW + 1 when the bin holds no
// step.  Returns false if a bin holds more than one step (or bin 0 one).
static bool build_dyn_table(const float map[256], int MB, bool neg, uint32_t* out, int nb) {
  const int SH = 23 - MB;
  const uint32_t LOW = (1u << SH) - 1, ONE = 0x3F800000u;
  for (int idx = 0; idx < nb; ++idx) {
    const uint32_t L = (uint32_t(DYN_E0 << MB) + uint32_t(idx)) << SH;
    uint32_t lo = idx == 0 ? 0u : L, hi = L + LOW;
    if (lo > ONE) lo = ONE;  // bins above 1.0 are never used: same entry as 1.0
    if (hi > ONE) hi = ONE;
    auto code = [&](uint32_t mag) { return dyn_rule(map, neg ? -fbits(mag) : fbits(mag)); };
    const int c_small = code(lo), c_big = code(hi);  // at the smallest / largest magnitude
    const int c0 = neg ? c_big : c_small, c1 = neg ? c_small : c_big;
    uint32_t thr = LOW + 1;
    if (c1 != c0) {
      if (c1 != c0 + 1 || idx == 0) return false;
      // transition magnitude: positive, the smallest with code c1; negative,
      // the largest with code c1 (code(-mag) falls as mag grows)
      uint32_t a = lo, b = hi;
      if (!neg) {  // code(a) = c0, code(b) = c1: find the first b
        while (b - a > 1) {
          const uint32_t m = a + (b - a) / 2;
          (code(m) == c1 ? b : a) = m;
        }
        thr = b & LOW;
      } else {  // code(a) = c1, code(b) = c0: find the last a
        while (b - a > 1) {
          const uint32_t m = a + (b - a) / 2;
          (code(m) == c1 ? a : b) = m;
        }
        thr = LOW - (a & LOW);
      }
    }
    out[idx] = (uint32_t(c0) << 24) | thr;
  }
  return true;
}

static bool dyn_tables(DynTables& h) {
  dyn_maps(h.map[0], h.map[1]);
  return build_dyn_table(h.map[0], DYN_MB_M, false, h.tm, DYN_NB_M) &&
         build_dyn_table(h.map[0], DYN_MB_M, true, h.tm + DYN_NB_M, DYN_NB_M) &&
         build_dyn_table(h.map[1], DYN_MB_V, false, h.tv, DYN_NB_V);
}

bool dyn_code_tables(uint32_t* m_tab, uint32_t* v_tab) {
  static DynTables h;
  if (!dyn_tables(h)) return false;
  std::memcpy(m_tab, h.tm, sizeof h.tm);
  std::memcpy(v_tab, h.tv, sizeof h.tv);
  return true;
}

static cudaError_t ensure_dyn_tables() {  // once per device: __constant__ lives in each device's module
  static DynTables h;
  static const bool built = dyn_tables(h);
  if (!built) return cudaErrorInvalidValue;  // a bin with two steps: cannot happen for R25's maps
  if (!once_per_device(&c_dyn)) return cudaSuccess;
  return cudaMemcpyToSymbol(c_dyn, &h, sizeof h);
}

// dequantisation map replicated 8 times in shared memory (entry k of copy c
// at word k * 8 + c, lane uses copy lane & 7): a warp's 32 lookups fall into
// at most 4 words per bank
__device__ __forceinline__ float rmap(const float* rep, int k, int lane) { return rep[(k << 3) | (lane & 7)]; }

// the code of y = fl(m / A) in [-1, 1] (signed) / [0, 1] (unsigned): one
// table lookup and one comparison (see the file comment)
template <bool SIGNED>
__device__ __forceinline__ uint32_t dyn_code(const uint32_t* tab, float y) {
  constexpr int MB = SIGNED ? DYN_MB_M : DYN_MB_V;
  constexpr int SH = 23 - MB;
  constexpr uint32_t LOW = (1u << SH) - 1;
  const uint32_t b = __float_as_uint(y);
  const uint32_t mag = b & 0x7fffffffu;
  int idx = int(mag >> SH) - (DYN_E0 << MB);
  idx = idx < 0 ? 0 : idx;
  uint32_t yl = mag & LOW;
  if (SIGNED) {
    const uint32_t sgn = b >> 31;
    idx += int(sgn) * DYN_NB_M;
    yl ^= (0u - sgn) & LOW;
  }
  const uint32_t e = tab[idx];
  return (e >> 24) + (yl >= (e & 0xffffffu) ? 1u : 0u);
}

// y = fl32(x / A) through fp64: float(double(x) * RN64(1/A)) -- the relative
// error of the double product (< 2^-51.9) is below the distance of any
// quotient of two floats to a float rounding boundary (>= 2^-49 relative),
// so this is exactly the IEEE fp32 quotient the oracle takes (no slow path,
// no branch); rA = 1.0 / double(A) once per block
__device__ __forceinline__ float div_exact(float x, double rA) {
  return __double2float_rn(__dmul_rn(double(x), rA));
}

constexpr int DYN_STAGES = 1;
struct DynSmem {
  AdamStage stage[DYN_STAGES];  // TMA ring: the next block's inputs (20 KB)
  float rep[2][256 * 8];        // dequantisation maps, 8 copies (16 KB)
  uint32_t tm[2 * DYN_NB_M];    // code tables (28 KB)
  uint32_t tv[DYN_NB_V];
};

// Persistent CTAs walk the block table; as soon as a block's inputs are in
// registers, thread 0 bulk-copies the CTA's next block (fp32 master + grad,
// both code arrays: 20 KB) into the one stage (as adam8_tma_kernel), so the
// code decision of one block overlaps the loads of the next (without the
// stage: long-scoreboard stalls 3.7 per issued instruction; with two stages
// the 100 KB of shared memory leave 2 CTAs per SM and it is slower:
// profiles/r2/dyn/).  Blocks a bulk copy cannot take (misaligned, partial,
// 2-D, long) load directly.
template <bool PARAM_BF16>
__global__ void __launch_bounds__(DYN_NT, 3) adam8_dyn_kernel(const AdamBlock* __restrict__ tbl, int64_t nblocks,
                                                          AdamPtrs P, AdamScalars s) {
  extern __shared__ __align__(128) uint8_t dyn_smem[];
  DynSmem& T = *reinterpret_cast<DynSmem*>(dyn_smem);
  __shared__ __align__(8) uint64_t full[DYN_STAGES];
  __shared__ float red_m[2][DYN_NT / 32], red_v[2][DYN_NT / 32];
  // the block's table entry and its two stored absmax travel with the stage
  // (entry stored by thread 0, absmax by cp.async completing on the stage's
  // barrier), so no thread starts a block with the dependent global loads
  // tbl[b] -> absmax[slot] (with them: long-scoreboard 2.9 per issue)
  __shared__ AdamBlock ent[DYN_STAGES];
  __shared__ __align__(8) float ent_abs[DYN_STAGES][2];
  auto issue = [&](int64_t b, int st) {  // thread 0: stage st <- block b
    const AdamBlock nb = tbl[b];
    ent[st] = nb;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(&ent_abs[st][0])), "l"(P.mabs + nb.slot)
                 : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(&ent_abs[st][1])), "l"(P.vabs + nb.slot)
                 : "memory");
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[st])) : "memory");
    if (adam_tma_ok(nb)) {
      mbar_arrive_expect_tx(&full[st], ADAM_STAGE_TX);
      bulk_g2s(T.stage[st].p, P.master + nb.state_off, sizeof(float) * ADAM_TILE, &full[st]);
      bulk_g2s(T.stage[st].g, P.grad + nb.grad_off, sizeof(float) * ADAM_TILE, &full[st]);
      bulk_g2s(T.stage[st].mq, P.mq + nb.state_off, ADAM_TILE, &full[st]);
      bulk_g2s(T.stage[st].vq, P.vq + nb.state_off, ADAM_TILE, &full[st]);
    } else {
      mbar_arrive(&full[st]);
    }
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < DYN_STAGES; ++st) mbar_init(&full[st], 2);  // the copies' arrival + thread 0's
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int st = 0; st < DYN_STAGES; ++st) {
      const int64_t b = blockIdx.x + int64_t(st) * gridDim.x;
      if (b < nblocks) issue(b, st);
    }
  }
  for (int i = threadIdx.x; i < 2 * 256 * 8; i += DYN_NT) {
    const int w = i >> 11, k = (i >> 3) & 255;
    T.rep[w][i & 2047] = c_dyn.map[w][k];
  }
  for (int i = threadIdx.x; i < 2 * DYN_NB_M; i += DYN_NT) T.tm[i] = c_dyn.tm[i];
  for (int i = threadIdx.x; i < DYN_NB_V; i += DYN_NT) T.tv[i] = c_dyn.tv[i];
  __syncthreads();
  const int lane = int(threadIdx.x) & 31;
  const float* mapm = T.rep[0];
  const float* mapv = T.rep[1];
  constexpr uint32_t zero_m = 127, zero_v = 0;  // codes of 0.0 in the two maps
  uint8_t* mq = reinterpret_cast<uint8_t*>(P.mq);
  using G = AdamGeom<DYN_NT>;  // 2 quads per thread
  int it = 0;
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++it) {
    const int st = it % DYN_STAGES;
    const uint32_t ph = uint32_t(it / DYN_STAGES) & 1u;
    mbar_wait(&full[st], ph);
    const AdamBlock blk = ent[st];
    const float Am = ent_abs[st][0], Av = ent_abs[st][1];
    float* rm = red_m[it & 1];
    float* rv = red_v[it & 1];
    auto refill = [&]() {  // after the absmax barrier: every thread has read stage st
      if (threadIdx.x == 0) {
        const int64_t nb = b + int64_t(DYN_STAGES) * gridDim.x;
        if (nb < nblocks) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(nb, st);
        }
      }
    };
    // R27: A = 0, NaN or +inf -> the code of 0 everywhere
    // block-uniform: A finite and > 0 (else the code of 0), 1/A in fp64
    double rAm = 0.0, rAv = 0.0;
    bool okm = false, okv = false;
    auto qm = [&](float m) { return okm ? dyn_code<true>(T.tm, div_exact(m, rAm)) : zero_m; };
    auto qv = [&](float v) { return okv ? dyn_code<false>(T.tv, div_exact(v, rAv)) : zero_v; };
    auto set_div = [&](float am_, float av_) {
      okm = am_ > 0.f && am_ <= FLT_MAX_F;
      okv = av_ > 0.f && av_ <= FLT_MAX_F;
      rAm = okm ? 1.0 / double(am_) : 0.0;
      rAv = okv ? 1.0 / double(av_) : 0.0;
    };
    float am = 0.f, av = 0.f;
    const bool staged = adam_tma_ok(blk);
    const bool fast = staged || (blk.len == ADAM_TILE && blk.cols == blk.len && (blk.state_off & 3) == 0 &&
                                 (blk.grad_off & 3) == 0 && (blk.param_off & 3) == 0);
    if (fast) {
      const AdamStage& S = T.stage[st];
      float p[G::EPT], m[G::EPT], v[G::EPT];
      // the source (stage / global) and the codec's "both absmax usable" test
      // are block-uniform: compile each case as its own straight-line code
      auto update = [&](auto staged_t) {
#pragma unroll
        for (int k = 0; k < G::Q; ++k) {
          const int a = G::quad(k);
          int4 pv, gv;
          uint32_t cm, cv;
          if constexpr (decltype(staged_t)::value) {
            pv = *reinterpret_cast<const int4*>(S.p + a);
            gv = *reinterpret_cast<const int4*>(S.g + a);
            cm = *reinterpret_cast<const uint32_t*>(S.mq + a);
            cv = *reinterpret_cast<const uint32_t*>(S.vq + a);
          } else {
            pv = ld_na_v4(P.master + blk.state_off + a);
            gv = ld_nc_v4(P.grad + blk.grad_off + a);
            cm = ld_na_u32(mq + blk.state_off + a);
            cv = ld_na_u32(P.vq + blk.state_off + a);
          }
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
      };
      if (staged)
        update(std::true_type{});
      else
        update(std::false_type{});
      block_max2<G::WARPS>(am, av, rm, rv);
      refill();
      set_div(am, av);
      auto store_all = [&](auto ok_t) {
        auto QM = [&](float x) {
          if constexpr (decltype(ok_t)::value) return dyn_code<true>(T.tm, div_exact(x, rAm));
          else return qm(x);
        };
        auto QV = [&](float x) {
          if constexpr (decltype(ok_t)::value) return dyn_code<false>(T.tv, div_exact(x, rAv));
          else return qv(x);
        };
#pragma unroll
        for (int k = 0; k < G::Q; ++k) {
          const int a = G::quad(k);
          const float* pk = &p[4 * k];
          st_f4(P.master + blk.state_off + a, make_float4(pk[0], pk[1], pk[2], pk[3]));
          st_u32(mq + blk.state_off + a, QM(m[4 * k]) | (QM(m[4 * k + 1]) << 8) | (QM(m[4 * k + 2]) << 16) |
                                             (QM(m[4 * k + 3]) << 24));
          st_u32(P.vq + blk.state_off + a, QV(v[4 * k]) | (QV(v[4 * k + 1]) << 8) | (QV(v[4 * k + 2]) << 16) |
                                               (QV(v[4 * k + 3]) << 24));
          if constexpr (PARAM_BF16)
            st_u2(static_cast<uint16_t*>(P.param) + blk.param_off + a,
                  make_uint2(pack_bf16x2(pk[0], pk[1]), pack_bf16x2(pk[2], pk[3])));
          else
            st_f4(static_cast<float*>(P.param) + blk.param_off + a, make_float4(pk[0], pk[1], pk[2], pk[3]));
        }
      };
      if (okm && okv)
        store_all(std::true_type{});
      else
        store_all(std::false_type{});
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
        mq[blk.state_off + o] = uint8_t(qm(m));
        P.vq[blk.state_off + o] = uint8_t(qv(v));
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
        refill();
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
        refill();
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
  if (once_per_device(reinterpret_cast<const void*>(adam8_dyn_kernel<true>))) {
    if (cudaError_t e = cudaFuncSetAttribute(adam8_dyn_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))
      return e;
    if (cudaError_t e = cudaFuncSetAttribute(adam8_dyn_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))
      return e;
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
