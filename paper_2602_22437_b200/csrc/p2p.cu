// Fused collectives over NVLink peer memory, one process
// per GPU, peers' buffers mapped with CUDA IPC (rsdb_p2p_create) -- or, for
// the single-device multi-rank test mode (rsdb_p2p_create_local), several
// logical ranks on one device sharing it.
//
//  rs_tma_kernel        a6+a7: rank k bulk-loads (TMA) G_r[kS + i] (bf16) from
//        every rank r into shared memory, y = sum_{r=0..m-1} fp32(G_r) * scale
//        in rank order (fp32), padding -> 0, writes its fp32 shard.  Wire
//        bytes per rank (m-1) S 2, vs (m-1) S 4 for the fp32 NCCL
//        ReduceScatter, and no separate m*S cast pass.
//  copy-engine AG       a4: rank k's copy engine pushes its shard into every
//        peer's buffer with cudaMemcpyAsync over the mappings (rotated peer
//        order) between a start and a done barrier kernel.
//  rs_adam_tma_kernel   a6+a7+a8 (+ a4 with PUSH): the ReduceScatter feeds
//        the 8-bit Adam update of the shard; with PUSH every updated bf16
//        parameter is also stored into every peer's gathered buffer -- the
//        whole step in one kernel.
// Round 1 measured the alternatives (8/16-B peer loads and stores, a TMA
// AllGather, a copy-engine ReduceScatter, a warp-specialised fused kernel;
// DESIGN.md §7b, profiles/r1/); only the measured best of each is built.
//
// Start/done barriers between the ranks: p2p_dev.cuh.
#include <cuda_bf16.h>

#include <type_traits>

#include "adam_dev.cuh"
#include "kernels.cuh"
#include "p2p_dev.cuh"

namespace rsdb {



__device__ __forceinline__ int first_pad_after_p(const int64_t* pad, int npad, int64_t x) {
  int lo = 0, hi = npad;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (pad[2 * mid + 1] > x)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}
__device__ __forceinline__ bool in_pad_p(const int64_t* pad, int npad, int j, int64_t i) {
  for (; j < npad && pad[2 * j] <= i; ++j)
    if (i < pad[2 * j + 1]) return true;
  return false;
}

// One term of the rank-order sum acc = ((0 + x_0) + x_1) + ..., x_r = fl(g_r *
// scale): the first term as ONE fma(g, scale, +0) (= 0 + fl(g * scale) exactly,
// signed zeros included), later ones with the product rounded on its own
// (__fmul_rn: no FMA contraction into the add, which matters when
// scale = fl(1/m) is not exact, m = 3, 5, ...).
__device__ __forceinline__ float rank_acc(float acc, float g, float scale, bool first) {
  return first ? __fmaf_rn(g, scale, 0.f) : __fadd_rn(acc, __fmul_rn(g, scale));
}

// Zero the padding positions of 4 consecutive outputs starting at e0.
__device__ __forceinline__ void pad_zero4(const int64_t* pad, int npad, int64_t e0, float& a0,
                                          float& a1, float& a2, float& a3) {
  if (npad <= 0) return;
  const int j = first_pad_after_p(pad, npad, e0);
  if (j < npad && pad[2 * j] < e0 + 4) {
    if (in_pad_p(pad, npad, j, e0 + 0)) a0 = 0.f;
    if (in_pad_p(pad, npad, j, e0 + 1)) a1 = 0.f;
    if (in_pad_p(pad, npad, j, e0 + 2)) a2 = 0.f;
    if (in_pad_p(pad, npad, j, e0 + 3)) a3 = 0.f;
  }
}

// ---------------- TMA (bulk-copy) variants over NVLink ----------------
// The data movement is issued by ONE thread per CTA as 1-D bulk copies
// (cp.async.bulk) straight from the peers' mapped memory into a ring of
// shared-memory stages (mbarrier complete_tx), so NVLink sees large
// transactions and the SMs issue almost no load instructions.
__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
}
__device__ __forceinline__ void tbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

constexpr int RS_TMA_THREADS = 256;
constexpr int RS_TMA_TILE = 2048;  // elements per tile (8 per thread)
constexpr int RS_TMA_STAGES = 3;

template <int M>
__global__ void __launch_bounds__(RS_TMA_THREADS) rs_tma_kernel(P2PPtrs grads, float* __restrict__ out,
                                                               int64_t S, int rank, float scale,
                                                               const int64_t* __restrict__ pad, int npad,
                                                               P2PSignals sg, uint64_t epoch) {
  extern __shared__ __align__(128) uint8_t rs_smem[];
  __shared__ __align__(8) uint64_t bar[RS_TMA_STAGES];
  // stage s, rank r: RS_TMA_TILE bf16 at rs_smem + (s*M + r) * RS_TMA_TILE*2
  uint16_t* stage = reinterpret_cast<uint16_t*>(rs_smem);
  p2p_start(sg, rank, M, epoch);
  const int64_t base = int64_t(rank) * S;
  const int64_t ntiles = (S + RS_TMA_TILE - 1) / RS_TMA_TILE;
  auto issue = [&](int64_t t, int s) {
    const int64_t e0 = t * RS_TMA_TILE;
    const uint32_t len = uint32_t(imin64(RS_TMA_TILE, S - e0)) * 2;  // bytes, multiple of 16
    tbar_expect(&bar[s], len * M);
#pragma unroll
    for (int r = 0; r < M; ++r)
      tma_g2s(stage + (s * M + r) * RS_TMA_TILE,
              static_cast<const uint16_t*>(grads.p[r]) + base + e0, len, &bar[s]);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < RS_TMA_STAGES; ++s) tbar_init(&bar[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < RS_TMA_STAGES; ++s) {
      const int64_t t = blockIdx.x + int64_t(s) * gridDim.x;
      if (t < ntiles) issue(t, s);
    }
  }
  __syncthreads();
  int it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % RS_TMA_STAGES;
    tbar_wait(&bar[s], uint32_t(it / RS_TMA_STAGES) & 1u);
    const int64_t e0 = t * RS_TMA_TILE;
    const int len = int(imin64(RS_TMA_TILE, S - e0));
    // two quads per thread: [4t, 4t+4) and [1024 + 4t, ...)
    float a[2][4];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int k = 0; k < 4; ++k) a[q][k] = 0.f;
#pragma unroll
    for (int r = 0; r < M; ++r) {
      const uint16_t* src = stage + (s * M + r) * RS_TMA_TILE;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int i = 4 * threadIdx.x + q * (RS_TMA_TILE / 2);
        const uint2 w = *reinterpret_cast<const uint2*>(src + i);
        a[q][0] = rank_acc(a[q][0], __uint_as_float(w.x << 16), scale, r == 0);
        a[q][1] = rank_acc(a[q][1], __uint_as_float(w.x & 0xffff0000u), scale, r == 0);
        a[q][2] = rank_acc(a[q][2], __uint_as_float(w.y << 16), scale, r == 0);
        a[q][3] = rank_acc(a[q][3], __uint_as_float(w.y & 0xffff0000u), scale, r == 0);
      }
    }
    __syncthreads();  // every thread has read stage s
    if (threadIdx.x == 0) {
      const int64_t tn = t + int64_t(RS_TMA_STAGES) * gridDim.x;
      if (tn < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(tn, s);
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i = 4 * threadIdx.x + q * (RS_TMA_TILE / 2);
      if (i < len) {  // len is a multiple of 8: whole quads
        pad_zero4(pad, npad, base + e0 + i, a[q][0], a[q][1], a[q][2], a[q][3]);
        *reinterpret_cast<float4*>(out + e0 + i) = make_float4(a[q][0], a[q][1], a[q][2], a[q][3]);
      }
    }
  }
  p2p_done(sg, rank, M, epoch);
}

template <int M>
static cudaError_t rs_tma_m(const P2PPtrs& grads, float* out, int64_t S, int rank, float scale,
                            const int64_t* pad, int npad, const P2PSignals& sg, uint64_t epoch,
                            cudaStream_t st) {
  const size_t smem = size_t(RS_TMA_TILE) * 2 * M * RS_TMA_STAGES;
  if (once_per_device(reinterpret_cast<const void*>(rs_tma_kernel<M>)))
    cudaFuncSetAttribute(rs_tma_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  static const int grid = [&] {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rs_tma_kernel<M>, RS_TMA_THREADS, smem);
    // 2 CTAs per SM (6 tiles of every rank in flight per SM) already saturate
    // the peer reads; the full occupancy (8) only adds contention: 128 MB unit
    // at N = 2, 120 vs 130 us (profiles/r2/latency/rs_grid.txt)
    b = b < 1 ? 1 : (b > 2 ? 2 : b);
    return num_sms() * b;
  }();
  const int64_t tiles = (S + RS_TMA_TILE - 1) / RS_TMA_TILE;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(tiles, grid_share(grid, sg)));
  rs_tma_kernel<M><<<blocks, RS_TMA_THREADS, smem, st>>>(grads, out, S, rank, scale, pad, npad, sg, epoch);
  return cudaGetLastError();
}

// Start (phase 0) or done (phase 1) barrier alone, one CTA: brackets the
// copy-engine AllGathers; rsdb_p2p_barrier.
template <int M>
__global__ void __launch_bounds__(32) p2p_barrier_kernel(P2PSignals sg, int rank, uint64_t epoch, int phase) {
  if (phase == 0)
    p2p_start(sg, rank, M, epoch);
  else
    p2p_done(sg, rank, M, epoch);
}

template <int M>
static cudaError_t ag_ce_m(const P2PPtrs& params, int64_t bytes_S, int rank, const P2PSignals& sg,
                           uint64_t epoch, cudaStream_t st) {
  // PUSH: this rank's copy engine writes its own shard into every peer's
  // buffer (same offsets).  A copy-engine pull from a peer costs ~10 us more
  // to start and streams slower (1 MB: 14.7 vs 5.1 us; 64 MB: 100 vs 94 us,
  // profiles/r2/latency/probe_barrier.txt).  The start barrier orders the
  // writes after every peer's prior work on its buffer; the done barrier
  // (signalled after this stream's copies complete) after every peer's
  // pushes into this rank.  The barriers are kernels: stream memory
  // operations (cuStreamWaitValue64) would save ~9 us of engine hand-offs
  // but block the whole hardware queue while they wait, and streams share
  // hardware queues -- in the ZeRO-3 schedule (AllGather stream + compute
  // stream) that deadlocked two ranks (profiles/r2/latency/README.md).
  p2p_barrier_kernel<M><<<1, 32, 0, st>>>(sg, rank, epoch, 0);
  const char* mine = static_cast<const char*>(params.p[rank]) + int64_t(rank) * bytes_S;
  for (int p = 1; p < M; ++p) {  // rotated peer order: ranks do not all write one GPU at once
    const int r = (rank + p) % M;
    char* dst = static_cast<char*>(const_cast<void*>(params.p[r])) + int64_t(rank) * bytes_S;
    cudaError_t e = cudaMemcpyAsync(dst, mine, size_t(bytes_S), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  p2p_barrier_kernel<M><<<1, 32, 0, st>>>(sg, rank, epoch, 1);
  return cudaGetLastError();
}

// AllGather from persistent shards (K-slot ring mode):
// every rank's copy engine pushes its persistent shard into region `rank` of
// every rank's slot (dsts.p[r]: rank r's slot, mapped; the own one by a local
// copy), rotated peer order, between the start/done barrier kernels (push:
// see ag_ce_m).
template <int M>
static cudaError_t ag_shards_ce_m(const P2PPtrs& dsts, const void* shard, int64_t bytes_S, int rank,
                                  const P2PSignals& sg, uint64_t epoch, cudaStream_t st) {
  p2p_barrier_kernel<M><<<1, 32, 0, st>>>(sg, rank, epoch, 0);
  for (int p = 0; p < M; ++p) {
    const int r = (rank + p) % M;
    char* dst = static_cast<char*>(const_cast<void*>(dsts.p[r])) + int64_t(rank) * bytes_S;
    cudaError_t e = cudaMemcpyAsync(dst, shard, size_t(bytes_S), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  p2p_barrier_kernel<M><<<1, 32, 0, st>>>(sg, rank, epoch, 1);
  return cudaGetLastError();
}

cudaError_t launch_ag_shards(const P2PPtrs& dsts, const void* shard, int64_t bytes_S, int rank, int m,
                             const P2PSignals* sg, uint64_t epoch, cudaStream_t st) {
  if (m == 1)
    return cudaMemcpyAsync(const_cast<void*>(dsts.p[0]), shard, size_t(bytes_S), cudaMemcpyDeviceToDevice, st);
  if (!sg) return cudaErrorInvalidValue;
  switch (m) {
#define AGS_CASE(MM) \
  case MM:           \
    return ag_shards_ce_m<MM>(dsts, shard, bytes_S, rank, *sg, epoch, st);
    AGS_CASE(2) AGS_CASE(3) AGS_CASE(4) AGS_CASE(5) AGS_CASE(6) AGS_CASE(7) AGS_CASE(8)
#undef AGS_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_rs_p2p(const P2PPtrs& grads, float* out, int64_t S, int rank, int m, float scale,
                          const int64_t* pad, int npad, const P2PSignals& sg, uint64_t epoch,
                          cudaStream_t st) {
  switch (m) {
#define RS_CASE(M) \
  case M:          \
    return rs_tma_m<M>(grads, out, S, rank, scale, pad, npad, sg, epoch, st);
    RS_CASE(2) RS_CASE(3) RS_CASE(4) RS_CASE(5) RS_CASE(6) RS_CASE(7) RS_CASE(8)
#undef RS_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_p2p_barrier(const P2PSignals& sg, int rank, int m, uint64_t epoch, cudaStream_t st) {
  switch (m) {
#define BAR_CASE(M)                                                 \
  case M:                                                           \
    p2p_barrier_kernel<M><<<1, 32, 0, st>>>(sg, rank, epoch, 0);    \
    p2p_barrier_kernel<M><<<1, 32, 0, st>>>(sg, rank, epoch, 1);    \
    return cudaGetLastError();
    BAR_CASE(2) BAR_CASE(3) BAR_CASE(4) BAR_CASE(5) BAR_CASE(6) BAR_CASE(7) BAR_CASE(8)
#undef BAR_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_ag_p2p(const P2PPtrs& params, int64_t bytes_S, int rank, int m,
                          const P2PSignals& sg, uint64_t epoch, cudaStream_t st) {
  switch (m) {
#define AG_CASE(M) \
  case M:          \
    return ag_ce_m<M>(params, bytes_S, rank, sg, epoch, st);
    AG_CASE(2) AG_CASE(3) AG_CASE(4) AG_CASE(5) AG_CASE(6) AG_CASE(7) AG_CASE(8)
#undef AG_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

// ---------------- ReduceScatter fused with the 8-bit Adam step ----------------
// a6 + a7 + a8 in ONE kernel over NVLink: for every quantization block of
// this rank's shard, one thread bulk-loads the block's bf16 gradients from all
// M ranks (TMA over the IPC mappings) plus the local fp32 master and the m / v
// codes into a shared-memory stage; the CTA sums the M gradients in rank
// order in fp32 (bit-identical to rs_p2p / the oracle's rank-order sum) and
// runs the 8-bit Adam update on the block.  The fp32 reduced gradient never
// reaches HBM (-8 B per owned element) and the optimizer's HBM traffic
// overlaps the NVLink-bound reduction.  M = 1 (world 1): the cast + Adam.
constexpr int RSA_NT = 128;

template <int M>
struct RsaGeom {
  // ring depth: 3 at world 1, 2 with peers (more CTAs per SM; +0.5-0.7 % at
  // N = 2 / 4, profiles/r1/v14_misc/stages_ab)
  static constexpr int STAGES = M == 1 ? 3 : 2;
  static constexpr int G_BYTES = M * ADAM_TILE * 2;
  static constexpr int ABS_OFF = G_BYTES + ADAM_TILE * 6;  // 16-B chunks holding the block's absmax
  static constexpr int STAGE_BYTES = ABS_OFF + 32;
};

__device__ __forceinline__ bool rsa_fits(const AdamBlock& b) {
  return b.cols == b.len && b.len <= ADAM_TILE && (b.len & 15) == 0 && (b.state_off & 15) == 0 &&
         (b.grad_off & 7) == 0 && (b.param_off & 3) == 0;
}

// AllGather fused into the step: every bf16 parameter the Adam tail writes is
// also stored into every peer's parameter array at the same index (NVLink
// stores, made visible by the system fence of the done barrier).
// Peers are visited in rank-rotated order (rank+1, rank+2, ...) so that the
// ranks do not all store into the same GPU at the same moment.
template <int M>
struct PeerPush {
  uint16_t* peer[M > 1 ? M - 1 : 1];  // peer[j] = rank (rank + 1 + j) mod M
  __device__ void init(const P2PPtrs& params, int rank) {
#pragma unroll
    for (int j = 0; j < M - 1; ++j) {
      const int r = (rank + 1 + j) % M;
      uint16_t* q = nullptr;
#pragma unroll
      for (int k = 0; k < M; ++k)  // compile-time indices into params.p
        if (k == r) q = static_cast<uint16_t*>(const_cast<void*>(params.p[k]));
      peer[j] = q;
    }
  }
  __device__ void quad(int64_t i, uint2 bits) const {
#pragma unroll
    for (int j = 0; j < M - 1; ++j) *reinterpret_cast<uint2*>(peer[j] + i) = bits;
  }
  __device__ void one(int64_t i, __nv_bfloat16 h) const {
#pragma unroll
    for (int j = 0; j < M - 1; ++j) reinterpret_cast<__nv_bfloat16*>(peer[j])[i] = h;
  }
};

// Reduced gradient of one element straight from the peers' bf16 buffers
// (rank-order fp32 sum x scale, as rs_p2p), for the two-pass long blocks.
template <int M>
struct PeerGradSum {
  P2PPtrs grads;
  int64_t base;
  float scale;
  __device__ float operator()(int64_t o) const {
    float acc = 0.f;
#pragma unroll
    for (int q = 0; q < M; ++q)
      acc = rank_acc(acc, __uint_as_float(uint32_t(static_cast<const uint16_t*>(grads.p[q])[base + o]) << 16),
                     scale, q == 0);
    return acc;
  }
};

// Single-role variant: all 128 threads compute; thread 0 also issues the
// refill of the stage it just consumed, from the after-reduce hook.
template <int M, bool PARAM_BF16, bool SYNC, bool PUSH>
__global__ void __launch_bounds__(RSA_NT) rs_adam_tma_kernel(const AdamBlock* __restrict__ tbl,
                                                            int64_t nblocks, P2PPtrs grads,
                                                            P2PPtrs params, float scale, AdamPtrs P,
                                                            AdamScalars s, P2PSignals sg, int rank,
                                                            uint64_t epoch, int nst,
                                                            const AdamBlockC* __restrict__ ctbl,
                                                            const UnitBase* __restrict__ ubase,
                                                            int n_units) {
  using Gm = RsaGeom<M>;
  using G = AdamGeom<RSA_NT>;
  using PushT = std::conditional_t<PUSH, PeerPush<M>, NoPush>;
  PushT push{};
  if constexpr (PUSH) push.init(params, rank);
  extern __shared__ __align__(128) uint8_t rsa_smem[];
  __shared__ __align__(8) uint64_t full[3];
  __shared__ float red_m[2][G::WARPS], red_v[2][G::WARPS];
  __shared__ UnitBase s_ub[RSA_MAX_UNITS];
  if (ctbl)
    for (int i = threadIdx.x; i < n_units; i += RSA_NT) s_ub[i] = ubase[i];
  if constexpr (SYNC) p2p_start(sg, rank, M, epoch);  // (contains a CTA barrier)
  else __syncthreads();
  // block b's descriptor: the compact 16-B entry + its unit's bases, or the full entry
  auto desc = [&](int64_t b) -> AdamBlock {
    if (ctbl) {
      const AdamBlockC c = ctbl[b];
      const UnitBase& u = s_ub[c.unit];
      return AdamBlock{u.state + c.off, u.grad + c.off, u.param + c.off, c.len, c.slot, c.len, c.len};
    }
    return tbl[b];
  };
  auto issue = [&](int64_t b, int st) {
    const AdamBlock nb = desc(b);
    uint8_t* S = rsa_smem + st * Gm::STAGE_BYTES;
    if (rsa_fits(nb)) {
      const uint32_t L = uint32_t(nb.len);
      tbar_expect(&full[st], L * (2 * M + 6));
#pragma unroll
      for (int r = 0; r < M; ++r)
        tma_g2s(S + r * ADAM_TILE * 2, static_cast<const uint16_t*>(grads.p[r]) + nb.grad_off, L * 2,
                &full[st]);
      tma_g2s(S + Gm::G_BYTES, P.master + nb.state_off, L * 4, &full[st]);
      tma_g2s(S + Gm::G_BYTES + ADAM_TILE * 4, P.mq + nb.state_off, L, &full[st]);
      tma_g2s(S + Gm::G_BYTES + ADAM_TILE * 5, P.vq + nb.state_off, L, &full[st]);
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&full[st])) : "memory");
    }
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < nst; ++st) tbar_init(&full[st]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int st = 0; st < nst; ++st) {
      const int64_t b = blockIdx.x + int64_t(st) * gridDim.x;
      if (b < nblocks) issue(b, st);
    }
  }
  __syncthreads();
  int it = 0, st = 0;
  uint32_t phase = 0;
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++it) {
    const AdamBlock blk = desc(b);
    const float sm = P.mabs[blk.slot] / 127.0f;
    const float sv = P.vabs[blk.slot] / 255.0f;
    float* rm = red_m[it & 1];
    float* rv = red_v[it & 1];
    auto refill = [&]() {
      if (threadIdx.x == 0) {
        const int64_t nb = b + int64_t(nst) * gridDim.x;
        if (nb < nblocks) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(nb, st);
        }
      }
    };
    tbar_wait(&full[st], phase);
    BlockRegs<RSA_NT> r;
    if (rsa_fits(blk)) {
      const uint8_t* S = rsa_smem + st * Gm::STAGE_BYTES;
      const uint16_t* Sg = reinterpret_cast<const uint16_t*>(S);
      const float* Sp = reinterpret_cast<const float*>(S + Gm::G_BYTES);
      const uint8_t* Sm = S + Gm::G_BYTES + ADAM_TILE * 4;
      const uint8_t* Sv = S + Gm::G_BYTES + ADAM_TILE * 5;
#pragma unroll
      for (int k = 0; k < G::Q; ++k) {
        const int e0 = G::quad(k);
        float a[4] = {0.f, 0.f, 0.f, 0.f};
        float4 pv = make_float4(0.f, 0.f, 0.f, 0.f);
        uint32_t cm = 0x80808080u, cv = 0u;  // decode to m = v = 0 for masked quads
        if (e0 < blk.len) {
#pragma unroll
          for (int q = 0; q < M; ++q) {  // rank order
            const uint2 w = *reinterpret_cast<const uint2*>(Sg + q * ADAM_TILE + e0);
            a[0] = rank_acc(a[0], __uint_as_float(w.x << 16), scale, q == 0);
            a[1] = rank_acc(a[1], __uint_as_float(w.x & 0xffff0000u), scale, q == 0);
            a[2] = rank_acc(a[2], __uint_as_float(w.y << 16), scale, q == 0);
            a[3] = rank_acc(a[3], __uint_as_float(w.y & 0xffff0000u), scale, q == 0);
          }
          pv = *reinterpret_cast<const float4*>(Sp + e0);
          cm = *reinterpret_cast<const uint32_t*>(Sm + e0);
          cv = *reinterpret_cast<const uint32_t*>(Sv + e0);
        }
        r.g[4 * k + 0] = a[0], r.g[4 * k + 1] = a[1], r.g[4 * k + 2] = a[2], r.g[4 * k + 3] = a[3];
        r.p[4 * k + 0] = pv.x, r.p[4 * k + 1] = pv.y, r.p[4 * k + 2] = pv.z, r.p[4 * k + 3] = pv.w;
        dq4_m(cm, sm, &r.mt[4 * k]);
        dq4_v(cv, sv, &r.vt[4 * k]);
      }
      if (blk.len == ADAM_TILE)
        adam_block_tail<RSA_NT, PARAM_BF16, 1>(r, blk, P, s, rm, rv, refill, push);
      else
        adam_block_tail<RSA_NT, PARAM_BF16, 2>(r, blk, P, s, rm, rv, refill, push);
    } else if (blk.len > ADAM_TILE) {
      // long block (q > 2048, 2-D tiles such as 128x128): two passes, the
      // rank-order sum of the peers' gradients recomputed in each
      adam_block_two_pass<RSA_NT, PARAM_BF16>(blk, sm, sv, P, s, rm, rv, refill,
                                              PeerGradSum<M>{grads, blk.grad_off, scale}, push);
    } else {
      // generic: gradients summed straight from the peers' memory, masked & strided
#pragma unroll
      for (int e = 0; e < G::EPT; ++e) {
        const int i = G::idx(e);
        float acc = 0.f;
        if (i < blk.len) {
          const int64_t o = blk_off(blk, i);
#pragma unroll
          for (int q = 0; q < M; ++q)
            acc = rank_acc(acc, __uint_as_float(uint32_t(static_cast<const uint16_t*>(grads.p[q])[blk.grad_off + o]) << 16), scale, q == 0);
          r.p[e] = P.master[blk.state_off + o];
          r.mt[e] = (byte_f(uint32_t(uint8_t(P.mq[blk.state_off + o])) ^ 0x80u, 0) - 8388736.0f) * sm;
          r.vt[e] = (byte_f(uint32_t(P.vq[blk.state_off + o]), 0) - 8388608.0f) * sv;
        } else {
          r.p[e] = r.mt[e] = r.vt[e] = 0.f;
        }
        r.g[e] = acc;
      }
      adam_block_tail<RSA_NT, PARAM_BF16, 0>(r, blk, P, s, rm, rv, refill, push);
    }
    if (++st == nst) {  // ring position and mbarrier phase of the next block
      st = 0;
      phase ^= 1u;
    }
  }
  if constexpr (SYNC) p2p_done(sg, rank, M, epoch);
}

template <int M, bool SYNC, bool PUSH>
static cudaError_t rs_adam_mbs(const AdamBlock* tbl, int64_t nblocks, const P2PPtrs& grads,
                               const P2PPtrs& params, float scale, const AdamPtrs& P,
                               const AdamScalars& s, const P2PSignals& sg, int rank, uint64_t epoch,
                               cudaStream_t st, const AdamBlockC* ctbl, const UnitBase* ubase, int n_units) {
  constexpr int nst = RsaGeom<M>::STAGES;
  const size_t smem = size_t(RsaGeom<M>::STAGE_BYTES) * nst;
  if (once_per_device(reinterpret_cast<const void*>(rs_adam_tma_kernel<M, true, SYNC, PUSH>)))
    cudaFuncSetAttribute(rs_adam_tma_kernel<M, true, SYNC, PUSH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
  static const int grid = [&] {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rs_adam_tma_kernel<M, true, SYNC, PUSH>, RSA_NT, smem);
    return num_sms() * (b < 1 ? 1 : b);
  }();
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(nblocks, grid_share(grid, sg)));
  rs_adam_tma_kernel<M, true, SYNC, PUSH><<<blocks, RSA_NT, smem, st>>>(
      tbl, nblocks, grads, params, scale, P, s, sg, rank, epoch, nst, ctbl, ubase, n_units);
  return cudaGetLastError();
}

cudaError_t launch_rs_adam_p2p(const AdamBlock* tbl, int64_t nblocks, const P2PPtrs& grads, int m,
                               float scale, const AdamPtrs& P, const AdamScalars& s,
                               const P2PSignals* sg, int rank, uint64_t epoch, cudaStream_t st,
                               const P2PPtrs* push_params, const AdamBlockC* ctbl,
                               const UnitBase* ubase, int n_units) {
  if (!P.param_bf16) return cudaErrorInvalidValue;  // the fused path is for bf16 units
  const P2PPtrs none_p{};
  if (m == 1) {
    P2PSignals none{};
    return rs_adam_mbs<1, false, false>(tbl, nblocks, grads, none_p, scale, P, s, none, rank, epoch, st, ctbl,
                                        ubase, n_units);
  }
  if (!sg) return cudaErrorInvalidValue;
  switch (m) {
#define RSA_CASE(MM)                                                                                     \
  case MM:                                                                                               \
    return push_params ? rs_adam_mbs<MM, true, true>(tbl, nblocks, grads, *push_params, scale, P, s, *sg, \
                                                     rank, epoch, st, ctbl, ubase, n_units)              \
                       : rs_adam_mbs<MM, true, false>(tbl, nblocks, grads, none_p, scale, P, s, *sg,     \
                                                      rank, epoch, st, ctbl, ubase, n_units);
    RSA_CASE(2) RSA_CASE(3) RSA_CASE(4) RSA_CASE(5) RSA_CASE(6) RSA_CASE(7) RSA_CASE(8)
#undef RSA_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace rsdb
