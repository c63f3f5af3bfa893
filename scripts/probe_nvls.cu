// Probe: NVLS (NVSwitch multicast) AllGather / ReduceScatter bandwidth
// against copy-engine pushes, through torch's symmetric memory (multicast
// address).  Not part of the library: evidence for DESIGN.md §11 (why the
// fused step does not use NVLS).  Built as a small shared library and
// driven by scripts/probe_nvls.py under torchrun.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
//        -o /tmp/libprobe_nvls.so scripts/probe_nvls.cu
#include <cuda_runtime.h>

#include <cstdint>

// AllGather: every rank stores its slice (local src) through the multicast
// address mc + off: the switch writes it into every rank's buffer
__global__ void nvls_ag_kernel(const uint4* __restrict__ src, char* mc, int64_t off, int64_t n16) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += int64_t(gridDim.x) * blockDim.x) {
    const uint4 v = src[i];
    char* a = mc + off + i * 16;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
  }
}

// ReduceScatter: every rank loads its slice through the multicast address
// with an in-switch reduction (bf16 pairs, fp32 accumulation) and stores the
// sums locally
__global__ void nvls_rs_kernel(const char* mc, int64_t off, uint4* __restrict__ dst, int64_t n16) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += int64_t(gridDim.x) * blockDim.x) {
    uint4 v;
    const char* a = mc + off + i * 16;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(a)
                 : "memory");
    dst[i] = v;
  }
}

extern "C" int probe_nvls_ag(const void* src, void* mc, int64_t off, int64_t bytes, int grid, void* stream) {
  nvls_ag_kernel<<<grid, 512, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const uint4*>(src),
                                                                        static_cast<char*>(mc), off, bytes / 16);
  return int(cudaGetLastError());
}

extern "C" int probe_nvls_rs(const void* mc, int64_t off, void* dst, int64_t bytes, int grid, void* stream) {
  nvls_rs_kernel<<<grid, 512, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const char*>(mc), off,
                                                                        static_cast<uint4*>(dst), bytes / 16);
  return int(cudaGetLastError());
}

// copy-engine push AllGather for comparison: this rank's slice into every peer's buffer
extern "C" int probe_ce_ag(void* const* peers, int world, int rank, int64_t bytes, void* stream) {
  const char* mine = static_cast<const char*>(peers[rank]) + int64_t(rank) * bytes;
  for (int p = 1; p < world; ++p) {
    const int r = (rank + p) % world;
    cudaError_t e = cudaMemcpyAsync(static_cast<char*>(peers[r]) + int64_t(rank) * bytes, mine, size_t(bytes),
                                    cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return int(e);
  }
  return 0;
}
