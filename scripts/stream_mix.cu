// Microbenchmark: does the number of concurrent HBM streams (separate arrays
// read / written by one kernel) change achievable bandwidth on B200?
// The fused RS+Adam kernel at N=1 reads 4 arrays (bf16 grad, fp32 master,
// m codes, v codes) and writes 4 (master, codes, codes, bf16 param); a copy
// reads 1 and writes 1.  Same bytes, different stream counts:
//   mix1: 1 read array (8 B/elem) -> 1 write array (8 B/elem)
//   mix2: 2 reads (4+4) -> 2 writes (4+4)
//   mix4: the fused kernel's byte mix, 4 reads (2,4,1,1) -> 4 writes (4,1,1,2)
// Each thread moves 4 elements per iteration with vector accesses; grid =
// 148 SMs x 8 CTAs, grid-stride.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void mix1(const uint2* __restrict__ a, uint2* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n / 4; i += int64_t(gridDim.x) * blockDim.x) {
    const int4 v0 = reinterpret_cast<const int4*>(a)[2 * i];
    const int4 v1 = reinterpret_cast<const int4*>(a)[2 * i + 1];
    reinterpret_cast<int4*>(b)[2 * i] = v0;
    reinterpret_cast<int4*>(b)[2 * i + 1] = v1;
  }
}

__global__ void mix2(const float4* __restrict__ a0, const float4* __restrict__ a1, float4* __restrict__ b0,
                     float4* __restrict__ b1, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n / 4; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 x = a0[i], y = a1[i];
    b0[i] = y;
    b1[i] = x;
  }
}

__global__ void mix4(const uint2* __restrict__ g, const float4* __restrict__ p, const uint32_t* __restrict__ m,
                     const uint32_t* __restrict__ v, float4* __restrict__ po, uint32_t* __restrict__ mo,
                     uint32_t* __restrict__ vo, uint2* __restrict__ bo, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n / 4; i += int64_t(gridDim.x) * blockDim.x) {
    const uint2 gg = g[i];
    float4 pp = p[i];
    const uint32_t mm = m[i], vv = v[i];
    pp.x += __uint_as_float(gg.x);
    po[i] = pp;
    mo[i] = mm ^ gg.y;
    vo[i] = vv ^ gg.x;
    bo[i] = make_uint2(mm, vv);
  }
}

int main() {
  const int64_t n = int64_t(1) << 30;  // elements: 8 GB read + 8 GB written per pass
  char* buf;
  const size_t bytes = size_t(n) * 16 + (64 << 20);
  if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(buf, 1, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 8, nt = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto R = [&](int64_t off) { return buf + off; };
  for (int rep = 0; rep < 2; ++rep) {
    for (int kind = 1; kind <= 4; kind *= 2) {
      for (int w = 0; w < 2; ++w) {  // warm-up, then timed
        cudaEventRecord(e0);
        for (int it = 0; it < 5; ++it) {
          if (kind == 1)
            mix1<<<grid, nt>>>(reinterpret_cast<uint2*>(R(0)), reinterpret_cast<uint2*>(R(n * 8)), n);
          else if (kind == 2)
            mix2<<<grid, nt>>>(reinterpret_cast<float4*>(R(0)), reinterpret_cast<float4*>(R(n * 4)),
                               reinterpret_cast<float4*>(R(n * 8)), reinterpret_cast<float4*>(R(n * 12)), n);
          else  // reads: g 2B, p 4B, m 1B, v 1B; writes: p 4B, m 1B, v 1B, b 2B
            mix4<<<grid, nt>>>(reinterpret_cast<uint2*>(R(0)), reinterpret_cast<float4*>(R(n * 2)),
                               reinterpret_cast<uint32_t*>(R(n * 6)), reinterpret_cast<uint32_t*>(R(n * 7)),
                               reinterpret_cast<float4*>(R(n * 8)), reinterpret_cast<uint32_t*>(R(n * 12)),
                               reinterpret_cast<uint32_t*>(R(n * 13)), reinterpret_cast<uint2*>(R(n * 14)), n);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (w) printf("{\"kernel\": \"mix%d\", \"streams_read\": %d, \"streams_written\": %d, \"gbs\": %.1f}\n",
                      kind, kind, kind, 5.0 * 16.0 * double(n) / (ms * 1e-3) / 1e9);
      }
    }
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
