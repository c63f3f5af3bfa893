// Probe: NVLink throughput of SM-issued bulk copies between two GPUs (one
// process, peer access): TMA bulk PUSH (shared -> peer global,
// cp.async.bulk.global.shared::cta) against bulk PULL (peer global -> shared)
// and 16-B st.global pushes, for a 64 MB buffer, at several grid sizes.
// Not part of the library.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/pbn scripts/probe_bulk_nvlink.cu
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

__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

constexpr int TILE = 16384;  // bytes per bulk op
constexpr int STAGES = 4;

// push (pull with the pointers swapped): each CTA streams its tiles of src (local) -> smem (bulk load) -> dst (peer, bulk store)
__global__ void __launch_bounds__(32) bulk_push(const char* src, char* dst, int64_t bytes) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t ntiles = bytes / TILE;
  int it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % STAGES;
    char* buf = sm + s * TILE;
    if (it >= STAGES) {  // the bulk store that used this stage must have read it
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(TILE) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(buf)),
                 "l"(src + t * TILE), "r"(TILE), "r"(sa(&bar[s]))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D1;\n\tbra W1;\nD1:\n\t}" ::"r"(
            sa(&bar[s])),
        "r"(uint32_t(it / STAGES) & 1u)
        : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + t * TILE), "r"(sa(buf)),
                 "r"(TILE)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// 16-B st.global pushes, 256 threads
__global__ void __launch_bounds__(256) st_push(const int4* src, int4* dst, int64_t n16) {
  for (int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x; i < n16; i += int64_t(gridDim.x) * 256) dst[i] = src[i];
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) return printf("need 2 GPUs\n"), 0;
  const int64_t B = 64ll << 20;
  char *a[2], *b[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int r = 0; r < 2; ++r) {
    CK(cudaSetDevice(r));
    CK(cudaDeviceEnablePeerAccess(1 - r, 0));
    CK(cudaMalloc(&a[r], B));
    CK(cudaMalloc(&b[r], B));
    CK(cudaMemset(a[r], r + 1, B));
    CK(cudaStreamCreateWithFlags(&st[r], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[r]));
    CK(cudaEventCreate(&e1[r]));
    CK(cudaFuncSetAttribute(bulk_push, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE * STAGES));
  }
  // both GPUs run the same kind of transfer at the same time (both link directions loaded, as in a collective)
  auto run = [&](const char* name, int grid, int kind) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      for (int r = 0; r < 2; ++r) {
        CK(cudaSetDevice(r));
        CK(cudaDeviceSynchronize());
      }
      for (int r = 0; r < 2; ++r) {
        CK(cudaSetDevice(r));
        CK(cudaEventRecord(e0[r], st[r]));
        if (kind == 0) bulk_push<<<grid, 32, TILE * STAGES, st[r]>>>(a[r], b[1 - r], B);       // push to peer
        if (kind == 1) bulk_push<<<grid, 32, TILE * STAGES, st[r]>>>(a[1 - r], b[r], B);       // pull from peer
        if (kind == 2) st_push<<<grid, 256, 0, st[r]>>>((const int4*)a[r], (int4*)b[1 - r], B / 16);
        if (kind == 3) CK(cudaMemcpyAsync(b[1 - r], a[r], B, cudaMemcpyDeviceToDevice, st[r]));  // CE push
        CK(cudaEventRecord(e1[r], st[r]));
      }
      float ms = 0;
      for (int r = 0; r < 2; ++r) {
        CK(cudaSetDevice(r));
        CK(cudaEventSynchronize(e1[r]));
        float t;
        CK(cudaEventElapsedTime(&t, e0[r], e1[r]));
        ms = t > ms ? t : ms;
      }
      best = ms < best ? ms : best;
    }
    printf("%-28s grid %5d  %8.1f us  %7.1f GB/s\n", name, grid, best * 1e3, B / (best * 1e-3) / 1e9);
    fflush(stdout);
  };
  for (int g : {148, 296, 592, 1184}) run("TMA bulk push 16 KB", g, 0);
  for (int g : {148, 296, 592, 1184}) run("TMA bulk pull 16 KB", g, 1);
  for (int g : {148, 296, 592, 1184}) run("st.global.v4 push", g, 2);
  run("copy engine push", 0, 3);
  printf("done\n");
  return 0;
}
