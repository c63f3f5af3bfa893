// Probe: where the ~15 us of a p2p start + done barrier pair goes (two GPUs,
// one process, peer access).  Not part of the library.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_barrier scripts/probe_barrier.cu -lcuda
// Prints one line per measurement: name, microseconds per iteration.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ void st_rel(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_rlx(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acq(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_rlx(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// ping-pong: rank 0 writes i to peer, waits for i back
__global__ void pingpong(uint64_t* mine, uint64_t* peer, int rank, int iters, int relaxed) {
  for (int i = 1; i <= iters; ++i) {
    if (rank == 0) {
      relaxed ? st_rlx(peer, i) : st_rel(peer, i);
      while ((relaxed ? ld_rlx(mine) : ld_acq(mine)) < uint64_t(i)) {
      }
    } else {
      while ((relaxed ? ld_rlx(mine) : ld_acq(mine)) < uint64_t(i)) {
      }
      relaxed ? st_rlx(peer, i) : st_rel(peer, i);
    }
  }
}

// barrier kernel variants (one CTA of 32, both ranks publish then wait)
// 0: current (threadfence_system + st.release.sys; ld.acquire.sys poll)
// 1: st.release.sys only; ld.acquire.sys poll
// 2: st.relaxed.sys after fence.acq_rel.sys; ld.relaxed.sys poll + fence after
// 3: no signalling (empty kernel: launch floor)
__global__ void barrier_k(uint64_t* mine, uint64_t* peer, uint64_t epoch, int variant) {
  if (variant == 3) return;
  if (threadIdx.x == 0) {
    if (variant == 0) {
      __threadfence_system();
      st_rel(peer, epoch);
      while (ld_acq(mine) < epoch) {
      }
    } else if (variant == 1) {
      st_rel(peer, epoch);
      while (ld_acq(mine) < epoch) {
      }
    } else {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      st_rlx(peer, epoch);
      while (ld_rlx(mine) < epoch) {
      }
      asm volatile("fence.acq_rel.sys;" ::: "memory");
    }
  }
  __syncthreads();
}

// device-side epoch (graph-friendly): epoch = ++*ctr
__global__ void barrier_dev(uint64_t* mine, uint64_t* peer, uint64_t* ctr) {
  if (threadIdx.x == 0) {
    const uint64_t e = *ctr + 1;
    *ctr = e;
    __threadfence_system();
    st_rel(peer, e);
    while (ld_acq(mine) < e) {
    }
  }
  __syncthreads();
}

__global__ void spin_until(volatile int* flag) {
  while (*flag == 0) {
  }
}

struct Dev {
  cudaStream_t st;
  uint64_t* sig;  // [0] barrier word, [1] pingpong word, [2] dev counter
  cudaEvent_t a, b;
  char* buf;
};

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  Dev d[2];
  int* hflag;
  CK(cudaHostAlloc(&hflag, 4, cudaHostAllocMapped | cudaHostAllocPortable));
  const size_t BUF = 256ull << 20;
  for (int r = 0; r < 2; ++r) {
    CK(cudaSetDevice(r));
    CK(cudaDeviceEnablePeerAccess(1 - r, 0));
    CK(cudaStreamCreateWithFlags(&d[r].st, cudaStreamNonBlocking));
    CK(cudaMalloc(&d[r].sig, 4096));
    CK(cudaMemset(d[r].sig, 0, 4096));
    CK(cudaMalloc(&d[r].buf, BUF));
    CK(cudaEventCreate(&d[r].a));
    CK(cudaEventCreate(&d[r].b));
  }
  for (int r = 0; r < 2; ++r) { CK(cudaSetDevice(r)); CK(cudaDeviceSynchronize()); }

  uint64_t epoch = 0;
  auto gate = [&](int r) {
    CK(cudaSetDevice(r));
    spin_until<<<1, 1, 0, d[r].st>>>(hflag);
  };
  auto run = [&](const char* name, int iters, auto body) {
    *(volatile int*)hflag = 0;
    for (int r = 0; r < 2; ++r) gate(r);
    for (int r = 0; r < 2; ++r) { CK(cudaSetDevice(r)); CK(cudaEventRecord(d[r].a, d[r].st)); }
    for (int i = 0; i < iters; ++i)
      for (int r = 0; r < 2; ++r) {
        CK(cudaSetDevice(r));
        body(r, i);
      }
    for (int r = 0; r < 2; ++r) { CK(cudaSetDevice(r)); CK(cudaEventRecord(d[r].b, d[r].st)); }
    *(volatile int*)hflag = 1;
    float ms[2];
    for (int r = 0; r < 2; ++r) {
      CK(cudaSetDevice(r));
      CK(cudaEventSynchronize(d[r].b));
      CK(cudaEventElapsedTime(&ms[r], d[r].a, d[r].b));
    }
    printf("%-44s %8.2f us/iter (rank0 %.2f, rank1 %.2f)\n", name, 1e3 * (ms[0] > ms[1] ? ms[0] : ms[1]) / iters,
           1e3 * ms[0] / iters, 1e3 * ms[1] / iters);
    fflush(stdout);
  };

  // ping-pong inside one kernel
  for (int relaxed = 0; relaxed < 2; ++relaxed) {
    for (int r = 0; r < 2; ++r) { CK(cudaSetDevice(r)); CK(cudaMemset(d[r].sig + 1, 0, 8)); }
    for (int r = 0; r < 2; ++r) { CK(cudaSetDevice(r)); CK(cudaDeviceSynchronize()); }
    run(relaxed ? "pingpong round trip (relaxed)" : "pingpong round trip (rel/acq)", 1, [&](int r, int) {
      pingpong<<<1, 1, 0, d[r].st>>>(d[r].sig + 1, d[1 - r].sig + 1, r, 10000, relaxed);
    });
    printf("  (divide by 10000 -> round trip)\n");
  }
  const int K = 400;
  const char* names[4] = {"barrier kernel: fence.sys + st.release", "barrier kernel: st.release only",
                          "barrier kernel: relaxed + acq_rel fences", "empty kernel (launch floor)"};
  for (int v = 0; v < 4; ++v) {
    run(names[v], K, [&](int r, int i) {
      barrier_k<<<1, 32, 0, d[r].st>>>(d[r].sig, d[1 - r].sig, epoch + 1 + i, v);
    });
    epoch += K;
  }
  // 148-CTA barrier kernel (all CTAs wait, as p2p_start)
  run("empty kernel, 148 CTAs x 256", K, [&](int r, int i) { barrier_k<<<148, 256, 0, d[r].st>>>(d[r].sig, d[1 - r].sig, 0, 3); });
  // CUDA graph of K device-epoch barriers
  {
    cudaGraphExec_t ge[2];
    for (int r = 0; r < 2; ++r) {
      CK(cudaSetDevice(r));
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(d[r].st, cudaStreamCaptureModeThreadLocal));
      for (int i = 0; i < K; ++i) barrier_dev<<<1, 32, 0, d[r].st>>>(d[r].sig + 3, d[1 - r].sig + 3, d[r].sig + 2);
      CK(cudaStreamEndCapture(d[r].st, &g));
      CK(cudaGraphInstantiate(&ge[r], g, 0));
    }
    run("graph of barrier kernels (device epoch)", 1, [&](int r, int) { CK(cudaGraphLaunch(ge[r], d[r].st)); });
    printf("  (divide by %d)\n", K);
  }
  // stream memory operations: write peer word, wait own word
  {
    CUresult cr;
    for (int r = 0; r < 2; ++r) { CK(cudaSetDevice(r)); CK(cudaMemset(d[r].sig + 4, 0, 8)); }
    for (int r = 0; r < 2; ++r) { CK(cudaSetDevice(r)); CK(cudaDeviceSynchronize()); }
    bool ok = true;
    run("stream write-value (peer) + wait-value", K, [&](int r, int i) {
      if (!ok) return;
      cr = cuStreamWriteValue64((CUstream)d[r].st, (CUdeviceptr)(d[1 - r].sig + 4), i + 1, 0);
      if (cr != CUDA_SUCCESS) {
        printf("cuStreamWriteValue64 -> %d\n", int(cr));
        ok = false;
        return;
      }
      cr = cuStreamWaitValue64((CUstream)d[r].st, (CUdeviceptr)(d[r].sig + 4), i + 1, CU_STREAM_WAIT_VALUE_GEQ);
      if (cr != CUDA_SUCCESS) {
        printf("cuStreamWaitValue64 -> %d\n", int(cr));
        ok = false;
      }
    });
  }
  // copy engine: peer pull of 1 MB / 64 MB alone, and between barrier kernels
  for (size_t mb : {1, 8, 64}) {
    const size_t bytes = mb << 20;
    char name[96];
    snprintf(name, sizeof name, "CE peer pull %zu MB alone", mb);
    run(name, 50, [&](int r, int) { CK(cudaMemcpyAsync(d[r].buf, d[1 - r].buf + BUF / 2, bytes, cudaMemcpyDeviceToDevice, d[r].st)); });
    snprintf(name, sizeof name, "barrier + CE pull %zu MB + barrier", mb);
    run(name, 50, [&](int r, int i) {
      barrier_k<<<1, 32, 0, d[r].st>>>(d[r].sig, d[1 - r].sig, epoch + 1 + 2 * i, 0);
      CK(cudaMemcpyAsync(d[r].buf, d[1 - r].buf + BUF / 2, bytes, cudaMemcpyDeviceToDevice, d[r].st));
      barrier_k<<<1, 32, 0, d[r].st>>>(d[r].sig, d[1 - r].sig, epoch + 2 + 2 * i, 0);
    });
    epoch += 100;
    snprintf(name, sizeof name, "CE push %zu MB alone", mb);
    run(name, 50, [&](int r, int) { CK(cudaMemcpyAsync(d[1 - r].buf + BUF / 2, d[r].buf, bytes, cudaMemcpyDeviceToDevice, d[r].st)); });
    snprintf(name, sizeof name, "barrier + CE push %zu MB + barrier", mb);
    run(name, 50, [&](int r, int i) {
      barrier_k<<<1, 32, 0, d[r].st>>>(d[r].sig, d[1 - r].sig, epoch + 1 + 2 * i, 1);
      CK(cudaMemcpyAsync(d[1 - r].buf + BUF / 2, d[r].buf, bytes, cudaMemcpyDeviceToDevice, d[r].st));
      barrier_k<<<1, 32, 0, d[r].st>>>(d[r].sig, d[1 - r].sig, epoch + 2 + 2 * i, 1);
    });
    epoch += 100;
    snprintf(name, sizeof name, "memop barrier + CE push %zu MB + memop", mb);
    static uint64_t mep = 1000;
    run(name, 50, [&](int r, int i) {
      const uint64_t e1 = mep + 2 * i + 1, e2 = mep + 2 * i + 2;
      cuStreamWriteValue64((CUstream)d[r].st, (CUdeviceptr)(d[1 - r].sig + 4), e1, 0);
      cuStreamWaitValue64((CUstream)d[r].st, (CUdeviceptr)(d[r].sig + 4), e1, CU_STREAM_WAIT_VALUE_GEQ);
      CK(cudaMemcpyAsync(d[1 - r].buf + BUF / 2, d[r].buf, bytes, cudaMemcpyDeviceToDevice, d[r].st));
      cuStreamWriteValue64((CUstream)d[r].st, (CUdeviceptr)(d[1 - r].sig + 4), e2, 0);
      cuStreamWaitValue64((CUstream)d[r].st, (CUdeviceptr)(d[r].sig + 4), e2, CU_STREAM_WAIT_VALUE_GEQ);
    });
    mep += 200;
  }
  printf("done\n");
  return 0;
}
