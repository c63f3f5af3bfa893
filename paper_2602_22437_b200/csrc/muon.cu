// N3: distributed Muon over RaggedShard, Algorithm 2
// (P:436-458), device side.  The host driver (capi.cc, rsdb_muon_step) runs
//
//   momentum   every rank, its shard:  buf <- mu buf + g;  u <- g + mu buf   (R21)
//   gather     ONE kernel over NVLink: each root pulls every owner's piece of
//              u for the matrices it was assigned (SelectRoot, R24) into a
//              contiguous matrix in its workspace (fp32, or bf16 for the
//              tensor-core Newton-Schulz) -- Redistribute(u, RaggedShard(r))
//   NS         on the root: Frobenius normalisation (fp64 sum of squares) and
//              5 quintic iterations as cuBLAS GEMMs (R22)
//   apply      ONE kernel over NVLink: each owner pulls its piece of o from the
//              root and applies w <- w - eta * sqrt(max(1, rows/cols)) * o to
//              its fp32 master shard, writing the bf16 parameter shard for the
//              next AllGather -- Redistribute(o, p) fused with the update (R23)
//
// gather/apply are bracketed by the p2p start/done barriers (p2p_dev.cuh):
// the start barrier orders them after every rank's momentum / NS work, the
// done barrier keeps the sources alive until every rank finished reading.
#include <cuda_bf16.h>

#include <cstdint>

#include "kernels.cuh"
#include "p2p_dev.cuh"

namespace rsdb {

constexpr int MUON_NT = 256;
constexpr int64_t MUON_CHUNK = 8192;  // elements per CTA work item

__global__ void __launch_bounds__(MUON_NT) muon_momentum_kernel(const int64_t* __restrict__ segs,
                                                               int64_t nseg, float* __restrict__ buf,
                                                               const float* __restrict__ grad,
                                                               float* __restrict__ u, float mu) {
  for (int64_t s = 0; s < nseg; ++s) {
    const int64_t off = segs[2 * s], n = segs[2 * s + 1];
    for (int64_t i = int64_t(blockIdx.x) * MUON_NT + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * MUON_NT) {
      const float g = grad[off + i];
      const float b = __fmaf_rn(mu, buf[off + i], g);
      buf[off + i] = b;
      u[off + i] = __fmaf_rn(mu, b, g);
    }
  }
}

__device__ __forceinline__ int64_t seg_of(const MuonSeg* segs, int64_t nseg, int64_t c) {
  int64_t lo = 0, hi = nseg - 1;  // last segment with chunk_begin <= c
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (segs[mid].chunk_begin <= c)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ const void* peer_ptr(const P2PPtrs& p, int r) {
  const void* q = nullptr;
#pragma unroll
  for (int j = 0; j < P2P_MAX_RANKS; ++j)
    if (j == r) q = p.p[j];
  return q;
}

// Redistribute(u, RaggedShard(root)): dst[seg.dst_off + i] = u_peer[seg.src_off + i]
template <bool BF16, bool SYNC>
__global__ void __launch_bounds__(MUON_NT) muon_gather_kernel(const MuonSeg* __restrict__ segs, int64_t nseg,
                                                             int64_t nchunks, P2PPtrs u, void* ws, int m,
                                                             int rank, P2PSignals sg, uint64_t epoch) {
  if constexpr (SYNC) p2p_start(sg, rank, m, epoch);
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const MuonSeg S = segs[seg_of(segs, nseg, c)];
    const int64_t e0 = (c - S.chunk_begin) * MUON_CHUNK;
    const int64_t n = S.n - e0 < MUON_CHUNK ? S.n - e0 : MUON_CHUNK;
    const float* src = static_cast<const float*>(peer_ptr(u, S.peer)) + S.src_off + e0;
    for (int64_t i = threadIdx.x; i < n; i += MUON_NT) {
      const float v = __ldcv(src + i);  // peer memory: bypass L1
      if constexpr (BF16)
        static_cast<__nv_bfloat16*>(ws)[S.dst_off + e0 + i] = __float2bfloat16_rn(v);
      else
        static_cast<float*>(ws)[S.dst_off + e0 + i] = v;
    }
  }
  if constexpr (SYNC) p2p_done(sg, rank, m, epoch);
}

// Redistribute(o, p) fused with w <- w - coef * o and the bf16 shard;
// coef = fl(lr * shape scale) (the segment's coef holds the shape scale)
template <bool BF16, bool SYNC>
__global__ void __launch_bounds__(MUON_NT) muon_apply_kernel(const MuonSeg* __restrict__ segs, int64_t nseg,
                                                            int64_t nchunks, P2PPtrs ws, float* master,
                                                            __nv_bfloat16* param, double lr, int m, int rank,
                                                            P2PSignals sg, uint64_t epoch) {
  if constexpr (SYNC) p2p_start(sg, rank, m, epoch);
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const MuonSeg S = segs[seg_of(segs, nseg, c)];
    const int64_t e0 = (c - S.chunk_begin) * MUON_CHUNK;
    const int64_t n = S.n - e0 < MUON_CHUNK ? S.n - e0 : MUON_CHUNK;
    const void* src = peer_ptr(ws, S.peer);
    const float coef = float(lr * double(S.coef));
    for (int64_t i = threadIdx.x; i < n; i += MUON_NT) {
      float o;
      if constexpr (BF16)
        o = __bfloat162float(
            __ushort_as_bfloat16(__ldcv(static_cast<const unsigned short*>(src) + S.src_off + e0 + i)));
      else
        o = __ldcv(static_cast<const float*>(src) + S.src_off + e0 + i);
      const int64_t d = S.dst_off + e0 + i;
      const float w = __fmaf_rn(-coef, o, master[d]);
      master[d] = w;
      if (param) param[d] = __float2bfloat16_rn(w);
    }
  }
  if constexpr (SYNC) p2p_done(sg, rank, m, epoch);
}

// ||X||_F^2 in fp64 (one atomic per CTA), then X *= 1 / (||X||_F + eps)
template <bool BF16>
__global__ void __launch_bounds__(MUON_NT) muon_sumsq_kernel(const void* __restrict__ x, int64_t n,
                                                            double* out) {
  double acc = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * MUON_NT + threadIdx.x; i < n; i += int64_t(gridDim.x) * MUON_NT) {
    const float v = BF16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(x)[i])
                         : static_cast<const float*>(x)[i];
    acc += double(v) * double(v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[MUON_NT / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < MUON_NT / 32; ++i) s += red[i];
    atomicAdd(out, s);
  }
}

template <bool BF16>
__global__ void __launch_bounds__(MUON_NT) muon_scale_kernel(void* __restrict__ x, int64_t n,
                                                            const double* ss, double eps) {
  const float f = float(1.0 / (sqrt(*ss) + eps));
  for (int64_t i = int64_t(blockIdx.x) * MUON_NT + threadIdx.x; i < n; i += int64_t(gridDim.x) * MUON_NT) {
    if constexpr (BF16) {
      __nv_bfloat16* p = static_cast<__nv_bfloat16*>(x) + i;
      *p = __float2bfloat16_rn(__bfloat162float(*p) * f);
    } else {
      static_cast<float*>(x)[i] *= f;
    }
  }
}

// Normalisation fused with the layout change of the tensor-core
// Newton-Schulz (ns_umma.cu): X (rows x cols, contiguous bf16) -> s*X into
// `same` (rows x cols, ld ld_same) and (s*X)^T into `trans` (cols x rows, ld
// ld_trans), s = 1 / (||X||_F + eps) from muon_sumsq_kernel (the same fp32
// product as muon_scale_kernel).  32 x 32 tiles through shared memory, so
// both writes are coalesced.
__global__ void __launch_bounds__(256) muon_scale_transpose_kernel(const __nv_bfloat16* __restrict__ x, int rows,
                                                                   int cols, const double* ss, double eps,
                                                                   __nv_bfloat16* same, int64_t ld_same,
                                                                   __nv_bfloat16* trans, int64_t ld_trans) {
  __shared__ __nv_bfloat16 tile[32][33];
  const float f = float(1.0 / (sqrt(*ss) + eps));
  const int tx = int(threadIdx.x) & 31, ty = int(threadIdx.x) >> 5;  // 32 x 8
  const int64_t tiles_c = (cols + 31) / 32, tiles = tiles_c * ((rows + 31) / 32);
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int r0 = int(t / tiles_c) * 32, c0 = int(t % tiles_c) * 32;
    for (int i = ty; i < 32; i += 8) {
      const int r = r0 + i, c = c0 + tx;
      if (r < rows && c < cols) {
        const __nv_bfloat16 v = __float2bfloat16_rn(__bfloat162float(x[int64_t(r) * cols + c]) * f);
        same[int64_t(r) * ld_same + c] = v;
        tile[i][tx] = v;
      }
    }
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {
      const int c = c0 + i, r = r0 + tx;
      if (c < cols && r < rows) trans[int64_t(c) * ld_trans + r] = tile[tx][i];
    }
    __syncthreads();
  }
}

// strided -> contiguous copy (the Newton-Schulz result back into the matrix
// slot): one row per CTA iteration, 16-B vectors when rows stay aligned
__global__ void __launch_bounds__(256) muon_copy2d_kernel(const __nv_bfloat16* __restrict__ src, int64_t ld,
                                                          int rows, int cols, __nv_bfloat16* __restrict__ dst) {
  const bool vec = (cols % 8) == 0 && (ld % 8) == 0 && (reinterpret_cast<uintptr_t>(src) % 16) == 0 &&
                   (reinterpret_cast<uintptr_t>(dst) % 16) == 0;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const __nv_bfloat16* s = src + int64_t(r) * ld;
    __nv_bfloat16* d = dst + int64_t(r) * cols;
    if (vec) {
      for (int c = threadIdx.x * 8; c < cols; c += 256 * 8)
        *reinterpret_cast<uint4*>(d + c) = *reinterpret_cast<const uint4*>(s + c);
    } else {
      for (int c = threadIdx.x; c < cols; c += 256) d[c] = s[c];
    }
  }
}

static int grid_for(int64_t items);

cudaError_t launch_muon_scale_transpose(const void* x, int rows, int cols, double* ss, double eps, void* same,
                                        int64_t ld_same, void* trans, int64_t ld_trans, cudaStream_t st) {
  const int64_t n = int64_t(rows) * cols;
  if (n == 0) return cudaSuccess;
  if (cudaError_t e = cudaMemsetAsync(ss, 0, sizeof(double), st)) return e;
  muon_sumsq_kernel<true><<<grid_for((n + MUON_NT - 1) / MUON_NT), MUON_NT, 0, st>>>(x, n, ss);
  const int64_t tiles = ((rows + 31) / 32) * int64_t((cols + 31) / 32);
  muon_scale_transpose_kernel<<<grid_for(tiles), 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(x), rows, cols, ss, eps, static_cast<__nv_bfloat16*>(same), ld_same,
      static_cast<__nv_bfloat16*>(trans), ld_trans);
  return cudaGetLastError();
}

cudaError_t launch_muon_copy2d(const void* src, int64_t ld, int rows, int cols, void* dst, cudaStream_t st) {
  const int64_t n = int64_t(rows) * cols;
  if (n == 0) return cudaSuccess;
  muon_copy2d_kernel<<<grid_for(rows), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(src), ld, rows, cols,
                                                     static_cast<__nv_bfloat16*>(dst));
  return cudaGetLastError();
}

static int grid_for(int64_t items) {
  const int64_t cap = int64_t(num_sms()) * 8;
  return int(items < 1 ? 1 : (items < cap ? items : cap));
}
// barrier kernels: every CTA resident at once (its share of the device when
// several logical ranks share it, rsdb_p2p_create_local)
template <typename K>
static int grid_sync(K kernel, int64_t items, const P2PSignals& sg) {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, MUON_NT, 0);
  const int64_t res = int64_t(num_sms()) * (b < 1 ? 1 : b);
  const int64_t g = grid_for(items);
  return int(grid_share(g < res ? g : res, sg));
}

cudaError_t launch_muon_momentum(const int64_t* segs, int64_t nseg, int64_t max_n, float* buf,
                                 const float* grad, float* u, float mu, cudaStream_t st) {
  if (nseg == 0) return cudaSuccess;
  muon_momentum_kernel<<<grid_for((max_n + MUON_NT - 1) / MUON_NT), MUON_NT, 0, st>>>(segs, nseg, buf, grad,
                                                                                    u, mu);
  return cudaGetLastError();
}

cudaError_t launch_muon_gather(const MuonSeg* segs, int64_t nseg, int64_t nchunks, const P2PPtrs& u,
                               void* ws, int bf16, int m, int rank, const P2PSignals* sg, uint64_t epoch,
                               cudaStream_t st) {
  const P2PSignals none{};
  if (m > 1 && !sg) return cudaErrorInvalidValue;
  const int g = grid_for(nchunks);
  if (bf16) {
    if (m > 1)
      muon_gather_kernel<true, true><<<grid_sync(muon_gather_kernel<true, true>, nchunks, *sg), MUON_NT, 0, st>>>(segs, nseg, nchunks, u, ws, m, rank, *sg, epoch);
    else if (nchunks)
      muon_gather_kernel<true, false><<<g, MUON_NT, 0, st>>>(segs, nseg, nchunks, u, ws, m, rank, none, 0);
  } else {
    if (m > 1)
      muon_gather_kernel<false, true><<<grid_sync(muon_gather_kernel<false, true>, nchunks, *sg), MUON_NT, 0, st>>>(segs, nseg, nchunks, u, ws, m, rank, *sg, epoch);
    else if (nchunks)
      muon_gather_kernel<false, false><<<g, MUON_NT, 0, st>>>(segs, nseg, nchunks, u, ws, m, rank, none, 0);
  }
  return cudaGetLastError();
}

cudaError_t launch_muon_apply(const MuonSeg* segs, int64_t nseg, int64_t nchunks, const P2PPtrs& ws,
                              int bf16, float* master, void* param_bf16, double lr, int m, int rank,
                              const P2PSignals* sg, uint64_t epoch, cudaStream_t st) {
  const P2PSignals none{};
  auto* pb = static_cast<__nv_bfloat16*>(param_bf16);
  if (m > 1 && !sg) return cudaErrorInvalidValue;
  const int g = grid_for(nchunks);
  if (bf16) {
    if (m > 1)
      muon_apply_kernel<true, true><<<grid_sync(muon_apply_kernel<true, true>, nchunks, *sg), MUON_NT, 0, st>>>(segs, nseg, nchunks, ws, master, pb, lr, m, rank, *sg,
                                                           epoch);
    else if (nchunks)
      muon_apply_kernel<true, false><<<g, MUON_NT, 0, st>>>(segs, nseg, nchunks, ws, master, pb, lr, m, rank, none,
                                                            0);
  } else {
    if (m > 1)
      muon_apply_kernel<false, true><<<grid_sync(muon_apply_kernel<false, true>, nchunks, *sg), MUON_NT, 0, st>>>(segs, nseg, nchunks, ws, master, pb, lr, m, rank, *sg,
                                                            epoch);
    else if (nchunks)
      muon_apply_kernel<false, false><<<g, MUON_NT, 0, st>>>(segs, nseg, nchunks, ws, master, pb, lr, m, rank,
                                                             none, 0);
  }
  return cudaGetLastError();
}

cudaError_t launch_muon_normalize(void* x, int64_t n, int bf16, double* ss, double eps, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(ss, 0, sizeof(double), st);
  if (e != cudaSuccess) return e;
  const int g = grid_for((n + MUON_NT - 1) / MUON_NT);
  if (bf16) {
    muon_sumsq_kernel<true><<<g, MUON_NT, 0, st>>>(x, n, ss);
    muon_scale_kernel<true><<<g, MUON_NT, 0, st>>>(x, n, ss, eps);
  } else {
    muon_sumsq_kernel<false><<<g, MUON_NT, 0, st>>>(x, n, ss);
    muon_scale_kernel<false><<<g, MUON_NT, 0, st>>>(x, n, ss, eps);
  }
  return cudaGetLastError();
}

}  // namespace rsdb
