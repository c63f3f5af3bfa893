// Fused collectives over NVLink peer memory, one process
// per GPU, peers' buffers mapped with CUDA IPC (rsdb_p2p_create).
//
//  rs_p2p_kernel / rs_tma_kernel   a6+a7: rank k pulls G_r[kS + i] (bf16) from
//        every rank r, y = sum_{r=0..m-1} fp32(G_r) * scale in rank order
//        (fp32), padding -> 0, writes its fp32 shard.  Wire bytes per rank
//        (m-1) S 2, vs (m-1) S 4 for the fp32 NCCL ReduceScatter, and no
//        separate m*S cast pass.
//  ag_p2p_kernel / ag_tma_kernel / copy-engine AG   a4: rank k pulls every
//        peer's shard into its own buffer (rotated peer order).
//  rs_adam_tma_kernel (default) / rs_adam_ws_kernel   a6+a7+a8 (+ a4 with
//        PUSH): the ReduceScatter feeds the 8-bit Adam update of the shard;
//        with PUSH every updated bf16 parameter is also stored into every
//        peer's gathered buffer -- the whole step in one kernel.
//
// Start/done barriers between the ranks: p2p_dev.cuh.
#include <cuda_bf16.h>

#include <cstdlib>
#include <type_traits>
#include <cstring>

#include "adam_dev.cuh"
#include "kernels.cuh"
#include "p2p_dev.cuh"

namespace rsdb {

constexpr int P2P_THREADS = 512;

// peer loads; FL = 0: ld.global.cv (uncached), 1: ld.global.nc (read-only
// path; the peer does not write its buffer between the barriers), 2: weak ld.global
template <int FL>
__device__ __forceinline__ uint2 ld_peer_v2(const void* p) {
  uint2 r;
  if constexpr (FL == 0)
    asm volatile("ld.global.cv.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  else if constexpr (FL == 1)
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  else
    asm volatile("ld.global.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
template <int FL>
__device__ __forceinline__ int4 ld_peer_v4(const void* p) {
  int4 r;
  if constexpr (FL == 0)
    asm volatile("ld.global.cv.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  else if constexpr (FL == 1)
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  else
    asm volatile("ld.global.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

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

// grads: M pointers to each rank's unit grad_full base (bf16).  out = this
// rank's grad_f32 + rank*S.  pad: padding intervals of the global buffer.
// Templated on the world size M so the peer loop unrolls with static indices
// (no local-memory copy of the pointer table) and all M x U peer loads are in
// flight before the rank-ordered accumulation.  VEC = bf16 elements per load
// (4: 8-byte loads, one coalesced float4 store; 8: 16-byte loads, two float4
// stores), FL = peer-load flavour.
template <int M, int VEC, int FL>
__global__ void __launch_bounds__(P2P_THREADS) rs_p2p_kernel(P2PPtrs grads, float* __restrict__ out,
                                                            int64_t S, int rank, float scale,
                                                            const int64_t* __restrict__ pad, int npad,
                                                            P2PSignals sg, uint64_t epoch) {
  constexpr int U = (M <= 2 ? 8 : (M <= 4 ? 4 : 2)) * 4 / VEC;  // vectors per thread per iteration
  p2p_start(sg, rank, M, epoch);
  const int64_t base = int64_t(rank) * S;
  const int64_t nvec = S / VEC;  // S is a multiple of g_coll = 8 for bf16 units
  const int64_t stride = int64_t(gridDim.x) * P2P_THREADS * U;
  const uint16_t* g[M];
#pragma unroll
  for (int r = 0; r < M; ++r) g[r] = static_cast<const uint16_t*>(grads.p[r]) + base;
  for (int64_t v0 = int64_t(blockIdx.x) * P2P_THREADS * U + threadIdx.x; v0 < nvec; v0 += stride) {
    uint32_t w[M][U][VEC / 2];
#pragma unroll
    for (int r = 0; r < M; ++r)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = v0 + int64_t(u) * P2P_THREADS;
        if constexpr (VEC == 4) {
          const uint2 x = v < nvec ? ld_peer_v2<FL>(g[r] + 4 * v) : make_uint2(0u, 0u);
          w[r][u][0] = x.x;
          w[r][u][1] = x.y;
        } else {
          const int4 x = v < nvec ? ld_peer_v4<FL>(g[r] + 8 * v) : make_int4(0, 0, 0, 0);
          w[r][u][0] = uint32_t(x.x);
          w[r][u][1] = uint32_t(x.y);
          w[r][u][2] = uint32_t(x.z);
          w[r][u][3] = uint32_t(x.w);
        }
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = v0 + int64_t(u) * P2P_THREADS;
      if (v >= nvec) break;
      // rank-order accumulation: acc = ((0 + x_0) + x_1) + ... (fp32), x_r = fl(fp32(G_r) * scale)
      float a[VEC];
#pragma unroll
      for (int k = 0; k < VEC; ++k) a[k] = 0.f;
#pragma unroll
      for (int r = 0; r < M; ++r)
#pragma unroll
        for (int k = 0; k < VEC / 2; ++k) {
          a[2 * k] = rank_acc(a[2 * k], __uint_as_float(w[r][u][k] << 16), scale, r == 0);
          a[2 * k + 1] = rank_acc(a[2 * k + 1], __uint_as_float(w[r][u][k] & 0xffff0000u), scale, r == 0);
        }
#pragma unroll
      for (int k = 0; k < VEC / 4; ++k) {
        const int64_t e0 = base + VEC * v + 4 * k;
        pad_zero4(pad, npad, e0, a[4 * k], a[4 * k + 1], a[4 * k + 2], a[4 * k + 3]);
        *reinterpret_cast<float4*>(out + VEC * v + 4 * k) =
            make_float4(a[4 * k], a[4 * k + 1], a[4 * k + 2], a[4 * k + 3]);
      }
    }
  }
  p2p_done(sg, rank, M, epoch);
}

// params: M pointers to each rank's unit param_full base.  PUSH = false: copy
// every peer's shard [r*S, (r+1)*S) into this rank's buffer (peer loads);
// PUSH = true: write this rank's shard into every peer's buffer (peer stores,
// made visible by the system fence of the done barrier).  bytes_S = S * elem.
template <int M, bool PUSH, int FL>
__global__ void __launch_bounds__(P2P_THREADS) ag_p2p_kernel(P2PPtrs params, int64_t bytes_S, int rank,
                                                            P2PSignals sg, uint64_t epoch) {
  constexpr int U = 4;
  p2p_start(sg, rank, M, epoch);
  char* buf[M];
#pragma unroll
  for (int r = 0; r < M; ++r) buf[r] = static_cast<char*>(const_cast<void*>(params.p[r]));
  char* mine = static_cast<char*>(const_cast<void*>(params.p[0]));
#pragma unroll
  for (int r = 0; r < M; ++r)
    if (r == rank) mine = buf[r];
  const int64_t nvec = bytes_S / 16;  // S * elem is a multiple of 16 (g_coll)
  const int64_t stride = int64_t(gridDim.x) * P2P_THREADS * U;
  for (int64_t v0 = int64_t(blockIdx.x) * P2P_THREADS * U + threadIdx.x; v0 < nvec; v0 += stride) {
    if constexpr (PUSH) {
      int4 w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = v0 + int64_t(u) * P2P_THREADS;
        if (v < nvec) w[u] = ld_peer_v4<1>(mine + int64_t(rank) * bytes_S + 16 * v);
      }
#pragma unroll
      for (int r = 0; r < M; ++r) {
        if (r == rank) continue;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t v = v0 + int64_t(u) * P2P_THREADS;
          if (v < nvec) *reinterpret_cast<int4*>(buf[r] + int64_t(rank) * bytes_S + 16 * v) = w[u];
        }
      }
    } else {
#pragma unroll
      for (int r = 0; r < M; ++r) {
        if (r == rank) continue;
        int4 w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t v = v0 + int64_t(u) * P2P_THREADS;
          if (v < nvec) w[u] = ld_peer_v4<FL>(buf[r] + int64_t(r) * bytes_S + 16 * v);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t v = v0 + int64_t(u) * P2P_THREADS;
          if (v < nvec) *reinterpret_cast<int4*>(mine + int64_t(r) * bytes_S + 16 * v) = w[u];
        }
      }
    }
  }
  p2p_done(sg, rank, M, epoch);
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
__device__ __forceinline__ void tma_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

constexpr int AG_TMA_CHUNK = 16384;  // bytes per stage
constexpr int AG_TMA_STAGES = 4;

template <int M>
__global__ void __launch_bounds__(32) ag_tma_kernel(P2PPtrs params, int64_t bytes_S, int rank,
                                                   P2PSignals sg, uint64_t epoch) {
  extern __shared__ __align__(128) uint8_t ag_smem[];
  __shared__ __align__(8) uint64_t bar[AG_TMA_STAGES];
  p2p_start(sg, rank, M, epoch);
  if (threadIdx.x == 0) {
    char* buf[M];
#pragma unroll
    for (int r = 0; r < M; ++r) buf[r] = static_cast<char*>(const_cast<void*>(params.p[r]));
    char* mine = buf[0];
#pragma unroll
    for (int r = 0; r < M; ++r)
      if (r == rank) mine = buf[r];
    for (int s = 0; s < AG_TMA_STAGES; ++s) tbar_init(&bar[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int64_t per = (bytes_S + AG_TMA_CHUNK - 1) / AG_TMA_CHUNK;  // chunks per peer shard
    const int64_t total = per * (M - 1);
    // chunk j -> (peer r, byte offset inside the global buffer, length)
    // peer slot p = j / per reads from rank (rank + 1 + p) % M: at any moment the
    // ranks read from distinct peers (a permutation), so no GPU's links are
    // shared by several readers while others idle
    auto chunk = [&](int64_t j, int& r, int64_t& off, uint32_t& len) {
      const int p = int(j / per);
      const int64_t c = j - int64_t(p) * per;
      r = (rank + 1 + p) % M;
      off = int64_t(r) * bytes_S + c * AG_TMA_CHUNK;
      len = uint32_t(imin64(AG_TMA_CHUNK, bytes_S - c * AG_TMA_CHUNK));
    };
    auto issue = [&](int64_t j, int s) {
      int r;
      int64_t off;
      uint32_t len;
      chunk(j, r, off, len);
      const char* src = buf[0];
#pragma unroll
      for (int q = 0; q < M; ++q)
        if (q == r) src = buf[q];
      tbar_expect(&bar[s], len);
      tma_g2s(ag_smem + s * AG_TMA_CHUNK, src + off, len, &bar[s]);
    };
    for (int s = 0; s < AG_TMA_STAGES; ++s) {
      const int64_t j = blockIdx.x + int64_t(s) * gridDim.x;
      if (j < total) issue(j, s);
    }
    int it = 0;
    for (int64_t j = blockIdx.x; j < total; j += gridDim.x, ++it) {
      const int s = it % AG_TMA_STAGES;
      tbar_wait(&bar[s], uint32_t(it / AG_TMA_STAGES) & 1u);
      int r;
      int64_t off;
      uint32_t len;
      chunk(j, r, off, len);
      tma_s2g(mine + off, ag_smem + s * AG_TMA_CHUNK, len);
      const int64_t jn = j + int64_t(AG_TMA_STAGES) * gridDim.x;
      if (jn < total) {
        tma_wait_read_all();  // the store above has read stage s
        issue(jn, s);
      }
    }
    tma_wait_all();
  }
  p2p_done(sg, rank, M, epoch);
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
static cudaError_t ag_tma_m(const P2PPtrs& params, int64_t bytes_S, int rank, const P2PSignals& sg,
                            uint64_t epoch, cudaStream_t st) {
  const size_t smem = size_t(AG_TMA_CHUNK) * AG_TMA_STAGES;
  static const int grid = [&] {
    cudaFuncSetAttribute(ag_tma_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, ag_tma_kernel<M>, 32, smem);
    return num_sms() * (b < 1 ? 1 : b);
  }();
  const int64_t chunks = (bytes_S + AG_TMA_CHUNK - 1) / AG_TMA_CHUNK * (M - 1);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(chunks, grid));
  ag_tma_kernel<M><<<blocks, 32, smem, st>>>(params, bytes_S, rank, sg, epoch);
  return cudaGetLastError();
}

template <int M>
static cudaError_t rs_tma_m(const P2PPtrs& grads, float* out, int64_t S, int rank, float scale,
                            const int64_t* pad, int npad, const P2PSignals& sg, uint64_t epoch,
                            cudaStream_t st) {
  const size_t smem = size_t(RS_TMA_TILE) * 2 * M * RS_TMA_STAGES;
  static const int grid = [&] {
    cudaFuncSetAttribute(rs_tma_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rs_tma_kernel<M>, RS_TMA_THREADS, smem);
    return num_sms() * (b < 1 ? 1 : b);
  }();
  const int64_t tiles = (S + RS_TMA_TILE - 1) / RS_TMA_TILE;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(tiles, grid));
  rs_tma_kernel<M><<<blocks, RS_TMA_THREADS, smem, st>>>(grads, out, S, rank, scale, pad, npad, sg, epoch);
  return cudaGetLastError();
}

// Start (phase 0) or done (phase 1) barrier alone, one CTA: brackets the
// copy-engine AllGather variant (cudaMemcpyAsync over the IPC mappings).
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
  p2p_barrier_kernel<M><<<1, 32, 0, st>>>(sg, rank, epoch, 0);
  char* mine = static_cast<char*>(const_cast<void*>(params.p[rank]));
  for (int p = 1; p < M; ++p) {  // rotated peer order: a permutation per step (see ag_tma_kernel)
    const int r = (rank + p) % M;
    const char* src = static_cast<const char*>(params.p[r]) + int64_t(r) * bytes_S;
    cudaError_t e = cudaMemcpyAsync(mine + int64_t(r) * bytes_S, src, size_t(bytes_S),
                                    cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  p2p_barrier_kernel<M><<<1, 32, 0, st>>>(sg, rank, epoch, 1);
  return cudaGetLastError();
}

// AllGather from persistent shards (K-slot ring mode):
// dst[r*bytes_S ...] = shard_r for every rank r, the local shard by a local
// copy and the peers' over NVLink by the copy engines (rotated peer order),
// between the start/done barriers.
template <int M>
static cudaError_t ag_shards_ce_m(const P2PPtrs& shards, char* dst, int64_t bytes_S, int rank,
                                  const P2PSignals& sg, uint64_t epoch, cudaStream_t st) {
  p2p_barrier_kernel<M><<<1, 32, 0, st>>>(sg, rank, epoch, 0);
  for (int p = 0; p < M; ++p) {
    const int r = (rank + p) % M;
    cudaError_t e = cudaMemcpyAsync(dst + int64_t(r) * bytes_S, shards.p[r], size_t(bytes_S),
                                    cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  p2p_barrier_kernel<M><<<1, 32, 0, st>>>(sg, rank, epoch, 1);
  return cudaGetLastError();
}

cudaError_t launch_ag_shards(const P2PPtrs& shards, void* dst, int64_t bytes_S, int rank, int m,
                             const P2PSignals* sg, uint64_t epoch, cudaStream_t st) {
  char* d = static_cast<char*>(dst);
  if (m == 1) return cudaMemcpyAsync(d, shards.p[0], size_t(bytes_S), cudaMemcpyDeviceToDevice, st);
  if (!sg) return cudaErrorInvalidValue;
  switch (m) {
#define AGS_CASE(MM) \
  case MM:           \
    return ag_shards_ce_m<MM>(shards, d, bytes_S, rank, *sg, epoch, st);
    AGS_CASE(2) AGS_CASE(3) AGS_CASE(4) AGS_CASE(5) AGS_CASE(6) AGS_CASE(7) AGS_CASE(8)
#undef AGS_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

// ---- ReduceScatter through the copy engines (RSDB_P2P_RS=ce) ----
// The peers' bf16 slices of this rank's shard are copied over NVLink by the
// copy engines (cudaMemcpyAsync over the IPC mappings, rotated peer order,
// on an auxiliary stream) into a local staging area, chunk by chunk; a local
// kernel reduces each chunk in rank order (fp32, x scale, padding -> 0) as
// soon as its copies have landed, so copies and reduction overlap.
template <int M>
__global__ void __launch_bounds__(256) rs_local_reduce_kernel(const uint16_t* __restrict__ own,
                                                             const uint16_t* __restrict__ stage,
                                                             float* __restrict__ out, int64_t c0,
                                                             int64_t len, int64_t S, int rank, float scale,
                                                             const int64_t* __restrict__ pad, int npad) {
  const uint16_t* src[M];
#pragma unroll
  for (int r = 0; r < M; ++r) {
    const int p = (r - rank + M) % M;  // 0: own slice; p >= 1: staging slot p - 1
    src[r] = p == 0 ? own : stage + int64_t(p - 1) * S;
  }
  const int64_t nv = len / 4;  // chunks are multiples of 8 elements
  for (int64_t v = int64_t(blockIdx.x) * 256 + threadIdx.x; v < nv; v += int64_t(gridDim.x) * 256) {
    const int64_t i = c0 + 4 * v;
    float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int r = 0; r < M; ++r) {  // rank order, as the oracle
      const uint2 w = ld_nc_v2(src[r] + i);
      a[0] = rank_acc(a[0], __uint_as_float(w.x << 16), scale, r == 0);
      a[1] = rank_acc(a[1], __uint_as_float(w.x & 0xffff0000u), scale, r == 0);
      a[2] = rank_acc(a[2], __uint_as_float(w.y << 16), scale, r == 0);
      a[3] = rank_acc(a[3], __uint_as_float(w.y & 0xffff0000u), scale, r == 0);
    }
    pad_zero4(pad, npad, int64_t(rank) * S + i, a[0], a[1], a[2], a[3]);
    *reinterpret_cast<float4*>(out + i) = make_float4(a[0], a[1], a[2], a[3]);
  }
}

template <int M>
static cudaError_t rs_ce_m(const P2PPtrs& grads, float* out, uint16_t* stage, int64_t S, int rank, float scale,
                           const int64_t* pad, int npad, const P2PSignals& sg, uint64_t epoch, cudaStream_t st,
                           cudaStream_t aux, cudaEvent_t* ev, int nchunk) {
  p2p_barrier_kernel<M><<<1, 32, 0, st>>>(sg, rank, epoch, 0);
  cudaError_t e = cudaEventRecord(ev[nchunk], st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(aux, ev[nchunk], 0);
  if (e != cudaSuccess) return e;
  const int64_t chunk = ((S + nchunk - 1) / nchunk + 7) / 8 * 8;
  const uint16_t* own = static_cast<const uint16_t*>(grads.p[rank]) + int64_t(rank) * S;
  for (int c = 0; c < nchunk; ++c) {
    const int64_t c0 = int64_t(c) * chunk;
    if (c0 >= S) break;
    const int64_t len = std::min<int64_t>(chunk, S - c0);
    for (int p = 1; p < M; ++p) {
      const int r = (rank + p) % M;
      e = cudaMemcpyAsync(stage + int64_t(p - 1) * S + c0,
                          static_cast<const uint16_t*>(grads.p[r]) + int64_t(rank) * S + c0, size_t(len) * 2,
                          cudaMemcpyDeviceToDevice, aux);
      if (e != cudaSuccess) return e;
    }
    e = cudaEventRecord(ev[c], aux);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev[c], 0);
    if (e != cudaSuccess) return e;
    const int grid = int(std::min<int64_t>(int64_t(num_sms()) * 8, std::max<int64_t>(1, (len / 4 + 255) / 256)));
    rs_local_reduce_kernel<M><<<grid, 256, 0, st>>>(own, stage, out, c0, len, S, rank, scale, pad, npad);
  }
  p2p_barrier_kernel<M><<<1, 32, 0, st>>>(sg, rank, epoch, 1);
  return cudaGetLastError();
}

cudaError_t launch_rs_ce(const P2PPtrs& grads, float* out, uint16_t* stage, int64_t S, int rank, int m, float scale,
                         const int64_t* pad, int npad, const P2PSignals& sg, uint64_t epoch, cudaStream_t st,
                         cudaStream_t aux, cudaEvent_t* ev, int nchunk) {
  switch (m) {
#define RSCE_CASE(MM) \
  case MM:            \
    return rs_ce_m<MM>(grads, out, stage, S, rank, scale, pad, npad, sg, epoch, st, aux, ev, nchunk);
    RSCE_CASE(2) RSCE_CASE(3) RSCE_CASE(4) RSCE_CASE(5) RSCE_CASE(6) RSCE_CASE(7) RSCE_CASE(8)
#undef RSCE_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

bool rs_use_ce() {
  static const bool v = [] {
    const char* e = getenv("RSDB_P2P_RS");
    return e && !strcmp(e, "ce");
  }();
  return v;
}

template <typename K>
static int p2p_grid(K kernel) {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, P2P_THREADS, 0);
  return num_sms() * (b < 1 ? 1 : b);
}

// Variant switch (experiments; defaults = measured best):
// RSDB_P2P_RS = v4cv | v4nc | v4ld | v8cv | v8nc | v8ld | tma ;
// RSDB_P2P_AG = pullcv | pullnc | push | tma | ce   (defaults: RS tma, AG ce; profiles/r1)
static int p2p_env(const char* name, const char* const* opts, int n, int dflt) {
  const char* e = getenv(name);
  if (!e) return dflt;
  for (int i = 0; i < n; ++i)
    if (!strcmp(e, opts[i])) return i;
  return dflt;
}
static int rs_variant() {
  static const char* o[] = {"v4cv", "v4nc", "v4ld", "v8cv", "v8nc", "v8ld", "tma"};
  static int v = p2p_env("RSDB_P2P_RS", o, 7, 6);  // tma: 604-614 GB/s wire (profiles/r1)
  return v;
}
static int ag_variant() {
  static const char* o[] = {"pullcv", "pullnc", "push", "tma", "ce"};
  static int v = p2p_env("RSDB_P2P_AG", o, 5, 4);  // ce: 701 GB/s at N=2 and 4 (profiles/r1)
  return v;
}

template <int M, int VEC, int FL>
static cudaError_t rs_p2p_mvf(const P2PPtrs& grads, float* out, int64_t S, int rank, float scale,
                              const int64_t* pad, int npad, const P2PSignals& sg, uint64_t epoch,
                              cudaStream_t st) {
  static const int grid = p2p_grid(rs_p2p_kernel<M, VEC, FL>);
  const int64_t per = int64_t(P2P_THREADS) * VEC * ((M <= 2 ? 8 : (M <= 4 ? 4 : 2)) * 4 / VEC);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((S + per - 1) / per, grid));
  rs_p2p_kernel<M, VEC, FL><<<blocks, P2P_THREADS, 0, st>>>(grads, out, S, rank, scale, pad, npad, sg,
                                                             epoch);
  return cudaGetLastError();
}

template <int M>
static cudaError_t rs_p2p_m(const P2PPtrs& grads, float* out, int64_t S, int rank, float scale,
                            const int64_t* pad, int npad, const P2PSignals& sg, uint64_t epoch,
                            cudaStream_t st) {
  switch (rs_variant()) {
    case 1: return rs_p2p_mvf<M, 4, 1>(grads, out, S, rank, scale, pad, npad, sg, epoch, st);
    case 2: return rs_p2p_mvf<M, 4, 2>(grads, out, S, rank, scale, pad, npad, sg, epoch, st);
    case 3: return rs_p2p_mvf<M, 8, 0>(grads, out, S, rank, scale, pad, npad, sg, epoch, st);
    case 4: return rs_p2p_mvf<M, 8, 1>(grads, out, S, rank, scale, pad, npad, sg, epoch, st);
    case 5: return rs_p2p_mvf<M, 8, 2>(grads, out, S, rank, scale, pad, npad, sg, epoch, st);
    case 6: return rs_tma_m<M>(grads, out, S, rank, scale, pad, npad, sg, epoch, st);
    default: return rs_p2p_mvf<M, 4, 0>(grads, out, S, rank, scale, pad, npad, sg, epoch, st);
  }
}

template <int M, bool PUSH, int FL>
static cudaError_t ag_p2p_mvf(const P2PPtrs& params, int64_t bytes_S, int rank, const P2PSignals& sg,
                              uint64_t epoch, cudaStream_t st) {
  static const int grid = p2p_grid(ag_p2p_kernel<M, PUSH, FL>);
  const int64_t per = int64_t(P2P_THREADS) * 4;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((bytes_S / 16 + per - 1) / per, grid));
  ag_p2p_kernel<M, PUSH, FL><<<blocks, P2P_THREADS, 0, st>>>(params, bytes_S, rank, sg, epoch);
  return cudaGetLastError();
}

template <int M>
static cudaError_t ag_p2p_m(const P2PPtrs& params, int64_t bytes_S, int rank, const P2PSignals& sg,
                            uint64_t epoch, cudaStream_t st) {
  switch (ag_variant()) {
    case 1: return ag_p2p_mvf<M, false, 1>(params, bytes_S, rank, sg, epoch, st);
    case 2: return ag_p2p_mvf<M, true, 1>(params, bytes_S, rank, sg, epoch, st);
    case 3: return ag_tma_m<M>(params, bytes_S, rank, sg, epoch, st);
    case 4: return ag_ce_m<M>(params, bytes_S, rank, sg, epoch, st);
    default: return ag_p2p_mvf<M, false, 0>(params, bytes_S, rank, sg, epoch, st);
  }
}

cudaError_t launch_rs_p2p(const P2PPtrs& grads, float* out, int64_t S, int rank, int m, float scale,
                          const int64_t* pad, int npad, const P2PSignals& sg, uint64_t epoch,
                          cudaStream_t st) {
  switch (m) {
#define RS_CASE(M) \
  case M:          \
    return rs_p2p_m<M>(grads, out, S, rank, scale, pad, npad, sg, epoch, st);
    RS_CASE(1) RS_CASE(2) RS_CASE(3) RS_CASE(4) RS_CASE(5) RS_CASE(6) RS_CASE(7) RS_CASE(8)
#undef RS_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_ag_p2p(const P2PPtrs& params, int64_t bytes_S, int rank, int m,
                          const P2PSignals& sg, uint64_t epoch, cudaStream_t st) {
  switch (m) {
#define AG_CASE(M) \
  case M:          \
    return ag_p2p_m<M>(params, bytes_S, rank, sg, epoch, st);
    AG_CASE(1) AG_CASE(2) AG_CASE(3) AG_CASE(4) AG_CASE(5) AG_CASE(6) AG_CASE(7) AG_CASE(8)
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

constexpr int RSA_MAX_STAGES = 4;
template <int M>
struct RsaGeom {
  // default ring depth (RSDB_RSA_STAGES overrides): 3 at world 1, 2 with peers
  // (more CTAs per SM; +0.5-0.7 % at N = 2 / 4, profiles/r1/v14_misc/stages_ab)
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
  __shared__ __align__(8) uint64_t full[RSA_MAX_STAGES];
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
    } else {
      // generic: gradients summed straight from the peers' memory, masked & strided
#pragma unroll
      for (int e = 0; e < G::EPT; ++e) {
        const int i = G::idx(e);
        float acc = 0.f;
        if (i < blk.len && blk.len <= ADAM_TILE) {
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


// Warp-specialised: warps 0..3 compute (128 threads, the shared Adam tail),
// warp 4 is the producer -- it reads the block table, writes each stage's
// descriptor to shared memory and issues the stage's bulk copies (peers'
// gradients, master, codes, absmax chunks), waiting on the stage's "empty"
// mbarrier, which the compute warps arrive on as soon as the block is in
// registers (after the absmax reduction).  So no compute warp ever waits on
// a global load of the table or on issuing copies.
constexpr int RSA_THREADS = RSA_NT + 32;

template <int M, bool PARAM_BF16, bool SYNC, bool PUSH>
__global__ void __launch_bounds__(RSA_THREADS, 4) rs_adam_ws_kernel(const AdamBlock* __restrict__ tbl,
                                                                    int64_t nblocks, P2PPtrs grads,
                                                                    P2PPtrs params, float scale, AdamPtrs P,
                                                                    AdamScalars s, P2PSignals sg, int rank,
                                                                    uint64_t epoch, int nst, int abs_tma) {
  using Gm = RsaGeom<M>;
  using G = AdamGeom<RSA_NT>;
  using PushT = std::conditional_t<PUSH, PeerPush<M>, NoPush>;
  extern __shared__ __align__(128) uint8_t rsa_smem[];
  __shared__ __align__(8) uint64_t full[RSA_MAX_STAGES];
  __shared__ __align__(8) uint64_t empty[RSA_MAX_STAGES];
  __shared__ float red_m[2][G::WARPS], red_v[2][G::WARPS];
  __shared__ AdamBlock sdesc[RSA_MAX_STAGES];
  if (threadIdx.x == 0) {
    for (int st = 0; st < nst; ++st) {
      tbar_init(&full[st]);   // one arrival: the producer's arrive.expect_tx
      tbar_init(&empty[st]);  // one arrival: compute thread 0 after the block is in registers
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (SYNC) p2p_start(sg, rank, M, epoch);  // (contains a CTA-wide barrier)
  else __syncthreads();

  if (threadIdx.x >= RSA_NT) {  // ---------------- producer warp
    if (threadIdx.x == RSA_NT) {
      int it = 0, st = 0;
      AdamBlock nb = blockIdx.x < nblocks ? tbl[blockIdx.x] : AdamBlock{};
      for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++it) {
        const AdamBlock cur = nb;
        if (b + gridDim.x < nblocks) nb = tbl[b + gridDim.x];  // prefetch the next entry
        // reuse of stage st: wait for the compute warps' release of its previous
        // block, i.e. completion number it/nst - 1 of empty[st]
        if (it >= nst) tbar_wait(&empty[st], uint32_t((it / nst - 1) & 1));
        uint8_t* S = rsa_smem + st * Gm::STAGE_BYTES;
        sdesc[st] = cur;
        const bool fits = rsa_fits(cur);
        const uint32_t L = uint32_t(cur.len);
        const uint32_t tx = (fits ? L * (2 * M + 6) : 0u) + (abs_tma ? 32u : 0u);
        if (tx == 0) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&full[st])) : "memory");
        } else {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tbar_expect(&full[st], tx);
          if (fits) {
#pragma unroll
            for (int r = 0; r < M; ++r)
              tma_g2s(S + r * ADAM_TILE * 2, static_cast<const uint16_t*>(grads.p[r]) + cur.grad_off, L * 2,
                      &full[st]);
            tma_g2s(S + Gm::G_BYTES, P.master + cur.state_off, L * 4, &full[st]);
            tma_g2s(S + Gm::G_BYTES + ADAM_TILE * 4, P.mq + cur.state_off, L, &full[st]);
            tma_g2s(S + Gm::G_BYTES + ADAM_TILE * 5, P.vq + cur.state_off, L, &full[st]);
          }
          if (abs_tma) {  // the 16-B chunks holding the block's two absmax values
            tma_g2s(S + Gm::ABS_OFF, P.mabs + (cur.slot & ~3), 16, &full[st]);
            tma_g2s(S + Gm::ABS_OFF + 16, P.vabs + (cur.slot & ~3), 16, &full[st]);
          }
        }
        if (++st == nst) st = 0;
      }
    }
  } else {  // ---------------------------------------- compute warps
    PushT push{};
    if constexpr (PUSH) push.init(params, rank);
    int it = 0, st = 0;
    uint32_t phase = 0;
    for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++it) {
      float* rm = red_m[it & 1];
      float* rv = red_v[it & 1];
      auto release = [&]() {  // the whole stage is in registers: hand it back to the producer
        if (threadIdx.x == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[st])) : "memory");
      };
      tbar_wait(&full[st], phase);
      const AdamBlock blk = sdesc[st];
      float am0, av0;
      if (abs_tma) {
        const float* Sa = reinterpret_cast<const float*>(rsa_smem + st * Gm::STAGE_BYTES + Gm::ABS_OFF);
        am0 = Sa[blk.slot & 3];
        av0 = Sa[4 + (blk.slot & 3)];
      } else {
        am0 = P.mabs[blk.slot];
        av0 = P.vabs[blk.slot];
      }
      const float sm = am0 / 127.0f;
      const float sv = av0 / 255.0f;
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
          adam_block_tail<RSA_NT, PARAM_BF16, 1>(r, blk, P, s, rm, rv, release, push);
        else
          adam_block_tail<RSA_NT, PARAM_BF16, 2>(r, blk, P, s, rm, rv, release, push);
      } else {
        // generic: gradients summed straight from the peers' memory, masked & strided
#pragma unroll
        for (int e = 0; e < G::EPT; ++e) {
          const int i = G::idx(e);
          float acc = 0.f;
          if (i < blk.len && blk.len <= ADAM_TILE) {
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
        adam_block_tail<RSA_NT, PARAM_BF16, 0>(r, blk, P, s, rm, rv, release, push);
      }
      if (++st == nst) {  // ring position and mbarrier phase of the next block
        st = 0;
        phase ^= 1u;
      }
    }
  }
  if constexpr (SYNC) p2p_done(sg, rank, M, epoch);  // (contains a CTA-wide barrier)
}

// RSDB_RSA_KERNEL=ws: the warp-specialised kernel (producer warp); default:
// the single-role kernel (measured faster at N=1)
static bool rsa_warp_specialised() {
  const char* e = std::getenv("RSDB_RSA_KERNEL");
  return e && std::strcmp(e, "ws") == 0;
}

static int rsa_stages(int def) {
  static const int env = [] {
    const char* e = std::getenv("RSDB_RSA_STAGES");
    return e ? std::atoi(e) : 0;
  }();
  return env >= 2 && env <= RSA_MAX_STAGES ? env : def;
}

template <int M, bool SYNC, bool PUSH>
static cudaError_t rs_adam_mbs(const AdamBlock* tbl, int64_t nblocks, const P2PPtrs& grads,
                               const P2PPtrs& params, float scale, const AdamPtrs& P,
                               const AdamScalars& s, const P2PSignals& sg, int rank, uint64_t epoch,
                               cudaStream_t st, int abs_tma, const AdamBlockC* ctbl, const UnitBase* ubase,
                               int n_units) {
  static const int nst = rsa_stages(RsaGeom<M>::STAGES);
  static const bool ws = rsa_warp_specialised();
  const size_t smem = size_t(RsaGeom<M>::STAGE_BYTES) * nst;
  static const int grid = [&] {
    int b = 0;
    if (ws) {
      cudaFuncSetAttribute(rs_adam_ws_kernel<M, true, SYNC, PUSH>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rs_adam_ws_kernel<M, true, SYNC, PUSH>, RSA_THREADS,
                                                    smem);
    } else {
      cudaFuncSetAttribute(rs_adam_tma_kernel<M, true, SYNC, PUSH>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rs_adam_tma_kernel<M, true, SYNC, PUSH>, RSA_NT,
                                                    smem);
    }
    return num_sms() * (b < 1 ? 1 : b);
  }();
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(nblocks, grid));
  if (ws)
    rs_adam_ws_kernel<M, true, SYNC, PUSH><<<blocks, RSA_THREADS, smem, st>>>(
        tbl, nblocks, grads, params, scale, P, s, sg, rank, epoch, nst, abs_tma);
  else
    rs_adam_tma_kernel<M, true, SYNC, PUSH><<<blocks, RSA_NT, smem, st>>>(
        tbl, nblocks, grads, params, scale, P, s, sg, rank, epoch, nst, ctbl, ubase, n_units);
  return cudaGetLastError();
}

cudaError_t launch_rs_adam_p2p(const AdamBlock* tbl, int64_t nblocks, const P2PPtrs& grads, int m,
                               float scale, const AdamPtrs& P, const AdamScalars& s,
                               const P2PSignals* sg, int rank, uint64_t epoch, cudaStream_t st,
                               const P2PPtrs* push_params, int abs_tma, const AdamBlockC* ctbl,
                               const UnitBase* ubase, int n_units) {
  if (rsa_warp_specialised()) ctbl = nullptr;  // the warp-specialised variant reads the full table
  if (!P.param_bf16) return cudaErrorInvalidValue;  // the fused path is for bf16 units
  const P2PPtrs none_p{};
  if (m == 1) {
    P2PSignals none{};
    return rs_adam_mbs<1, false, false>(tbl, nblocks, grads, none_p, scale, P, s, none, rank, epoch, st,
                                        abs_tma, ctbl, ubase, n_units);
  }
  if (!sg) return cudaErrorInvalidValue;
  switch (m) {
#define RSA_CASE(MM)                                                                                  \
  case MM:                                                                                            \
    return push_params ? rs_adam_mbs<MM, true, true>(tbl, nblocks, grads, *push_params, scale, P, s,  \
                                                     *sg, rank, epoch, st, abs_tma, ctbl, ubase,      \
                                                     n_units)                                         \
                       : rs_adam_mbs<MM, true, false>(tbl, nblocks, grads, none_p, scale, P, s, *sg,  \
                                                      rank, epoch, st, abs_tma, ctbl, ubase, n_units);
    RSA_CASE(2) RSA_CASE(3) RSA_CASE(4) RSA_CASE(5) RSA_CASE(6) RSA_CASE(7) RSA_CASE(8)
#undef RSA_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace rsdb
