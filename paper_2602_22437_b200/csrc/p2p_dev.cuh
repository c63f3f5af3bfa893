// Device-side signalling between ranks over NVLink peer memory, shared by
// p2p.cu (collectives, fused RS+Adam) and fp8.cu (FP8 quantize + AllGather).
//
// Per-rank signal buffer (uint64 words):
//   [0, 8)   start[r] = epoch written by rank r when it enters the call
//   [8, 16)  done[r]  = epoch written by rank r when all its CTAs finished
//   [16]     CTA completion counter of this rank's running kernel
//   [17]     error flag: bit 0 = a barrier wait exceeded sg.timeout_ns (the
//            kernel then gives up waiting instead of hanging the device;
//            rsdb_p2p_check reports and clears it)
// p2p_start: block 0 publishes `epoch` to every peer (release store),
// every CTA waits until all peers have published -- every rank's prior stream
// work is then complete.  p2p_done: the last CTA (atomic counter) fences,
// publishes to every peer and waits for all peers, so the kernel -- and the
// stream -- moves on only once nobody reads this rank's buffers and every
// store into the peers (push variants) is visible.
#pragma once
#include <cstdint>

#include "kernels.cuh"

namespace rsdb {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// sg.peer is indexed with compile-time indices only (a runtime index into a
// kernel-parameter array would copy the struct to the local-memory stack)
__device__ __forceinline__ uint64_t* sg_peer(const P2PSignals& sg, int i) {
  uint64_t* q = nullptr;
#pragma unroll
  for (int r = 0; r < P2P_MAX_RANKS; ++r)
    if (r == i) q = sg.peer[r];
  return q;
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// spin until *p >= epoch, or set the error flag after sg.timeout_ns
__device__ __forceinline__ void wait_epoch(const P2PSignals& sg, const uint64_t* p, uint64_t epoch) {
  if (ld_acquire_sys(p) >= epoch) return;
  const uint64_t t0 = global_ns();
  while (ld_acquire_sys(p) < epoch) {
    if (global_ns() - t0 > sg.timeout_ns) {
      atomicOr(reinterpret_cast<unsigned long long*>(sg.local + P2P_ERR_WORD), 1ull);
      return;
    }
  }
}

__device__ __forceinline__ void p2p_start(const P2PSignals& sg, int rank, int m, uint64_t epoch) {
  // st.release.sys alone publishes everything before it (cumulative); a
  // separate fence.sc.sys in front of it cost ~1 us per barrier
  // (profiles/r2/latency/probe_barrier.txt)
  if (blockIdx.x == 0 && threadIdx.x < m && int(threadIdx.x) != rank)
    st_release_sys(sg_peer(sg, int(threadIdx.x)) + rank, epoch);
  if (threadIdx.x == 0) {
    for (int r = 0; r < m; ++r) {
      if (r == rank) continue;
      wait_epoch(sg, sg.local + r, epoch);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void p2p_done(const P2PSignals& sg, int rank, int m, uint64_t epoch) {
  __syncthreads();  // this CTA's peer reads are complete (values consumed)
  if (threadIdx.x == 0) {
    __threadfence_system();  // this CTA's (possibly remote, push variant) stores
    unsigned int* ctr = reinterpret_cast<unsigned int*>(sg.local + 16);
    const unsigned int old = atomicAdd(ctr, 1u);
    if (old == gridDim.x - 1) {
      // every CTA's fence + counter increment precede this one's (their
      // release patterns); this read of the counter + the fence below is the
      // matching acquire pattern, so the release stores below carry every
      // CTA's (remote) stores to the peers
      atomicExch(ctr, 0u);
      __threadfence_system();
#pragma unroll
      for (int r = 0; r < P2P_MAX_RANKS; ++r)
        if (r < m && r != rank) st_release_sys(sg.peer[r] + 8 + rank, epoch);
      for (int r = 0; r < m; ++r) {
        if (r == rank) continue;
        wait_epoch(sg, sg.local + 8 + r, epoch);
      }
    }
  }
}

}  // namespace rsdb
