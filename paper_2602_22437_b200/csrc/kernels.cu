// sm_100a kernels of the RaggedShard/DBuffer collective step.
//
//  cast_scale_kernel  a6  fused DBuffer group op: bf16|f32 -> f32 * 1/m,
//                         padding written 0.  HBM-bound: 6 B/elem (bf16 src).
//  adam8_kernel       a8  block-wise 8-bit Adam on the local ragged shard.
//                         HBM-bound: 18 B/elem (+ 16 B of absmax per block).
//  copy_seg_kernel        batched ragged copy (FSDP2 Copy-In/Copy-Out baseline).
//
// No tensor cores: no stage is a dense contraction.  Everything is 16-byte
// vectorised, coalesced, read-once streaming (ld.global.nc.L1::no_allocate),
// on a persistent grid of (resident CTAs per SM) x (148 SMs).
#include <cuda_bf16.h>

#include "kernels.cuh"

namespace rsdb {

// ----------------------------------------------------------------------------
// helpers
// ----------------------------------------------------------------------------
__device__ __forceinline__ int4 ld_nc_v4(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_nc_v2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}
// coherent streaming loads for data the same kernel later overwrites
__device__ __forceinline__ int4 ld_na_v4(const void* p) {
  int4 r;
  asm volatile("ld.global.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_na_v2(const void* p) {
  uint2 r;
  asm volatile("ld.global.L1::no_allocate.v2.u32 {%0, %1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// fp32 -> bf16 round-to-nearest-even, packed pair (lo = a, hi = b)
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// small-integer <-> float without the quarter-rate I2F/F2I pipe:
// 2^23 + x has x in its low mantissa bits for 0 <= x < 2^23.
__device__ __forceinline__ float u8_to_f(uint32_t byte) {
  return __uint_as_float(0x4B000000u | byte) - 8388608.0f;
}
__device__ __forceinline__ float s8_to_f(uint32_t byte) {  // two's complement byte
  return __uint_as_float(0x4B000000u | ((byte ^ 0x80u) & 0xffu)) - 8388736.0f;
}
// round-to-nearest-even of |x| < 2^22 returned as int: (x + 1.5*2^23) keeps
// the rounded integer in the mantissa (the FADD rounds RNE).
__device__ __forceinline__ int rne_int(float x) {
  return __float_as_int(__fadd_rn(x, 12582912.0f)) - 0x4B400000;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename K>
static int resident_blocks(K kernel, int threads, size_t smem) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem) != cudaSuccess || b < 1)
    b = 1;
  return b;
}

// ----------------------------------------------------------------------------
// a6: fused cast + scale + padding zero
// ----------------------------------------------------------------------------
constexpr int CAST_THREADS = 256;
constexpr int CAST_UNROLL = 4;
constexpr int CAST_SMEM_PAD = 256;  // padding intervals cached in shared memory

// first interval j with hi_j > x (pad = lo0, hi0, lo1, hi1, ... ascending)
__device__ __forceinline__ int first_pad_after(const int64_t* pad, int npad, int64_t x) {
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
__device__ __forceinline__ bool in_pad_from(const int64_t* pad, int npad, int j, int64_t i) {
  for (; j < npad && pad[2 * j] <= i; ++j)
    if (i < pad[2 * j + 1]) return true;
  return false;
}

template <bool SRC_BF16>
__global__ void __launch_bounds__(CAST_THREADS) cast_scale_kernel(const void* __restrict__ src,
                                                                  float* __restrict__ dst,
                                                                  int64_t n, float scale,
                                                                  const int64_t* __restrict__ pad_g,
                                                                  int npad) {
  __shared__ int64_t spad[2 * CAST_SMEM_PAD];
  const int64_t* pad = pad_g;
  if (npad > 0 && npad <= CAST_SMEM_PAD) {
    for (int i = threadIdx.x; i < 2 * npad; i += CAST_THREADS) spad[i] = pad_g[i];
    __syncthreads();
    pad = spad;
  }
  constexpr int V = SRC_BF16 ? 8 : 4;  // elements per 16-byte source vector
  const int64_t nvec = n / V;
  const int64_t stride = int64_t(gridDim.x) * CAST_THREADS * CAST_UNROLL;
  for (int64_t base = int64_t(blockIdx.x) * CAST_THREADS * CAST_UNROLL + threadIdx.x; base < nvec;
       base += stride) {
    int4 raw[CAST_UNROLL];
#pragma unroll
    for (int u = 0; u < CAST_UNROLL; ++u) {
      const int64_t c = base + u * CAST_THREADS;
      if (c < nvec) raw[u] = ld_nc_v4(static_cast<const int4*>(src) + c);
    }
#pragma unroll
    for (int u = 0; u < CAST_UNROLL; ++u) {
      const int64_t c = base + u * CAST_THREADS;
      if (c >= nvec) break;
      float f[V];
      if constexpr (SRC_BF16) {
        const uint32_t w[4] = {uint32_t(raw[u].x), uint32_t(raw[u].y), uint32_t(raw[u].z),
                               uint32_t(raw[u].w)};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          f[2 * k] = bf16lo(w[k]) * scale;
          f[2 * k + 1] = bf16hi(w[k]) * scale;
        }
      } else {
        f[0] = __int_as_float(raw[u].x) * scale;
        f[1] = __int_as_float(raw[u].y) * scale;
        f[2] = __int_as_float(raw[u].z) * scale;
        f[3] = __int_as_float(raw[u].w) * scale;
      }
      const int64_t e0 = c * V;
      if (npad > 0) {
        const int j = first_pad_after(pad, npad, e0);
        if (j < npad && pad[2 * j] < e0 + V) {
#pragma unroll
          for (int k = 0; k < V; ++k)
            if (in_pad_from(pad, npad, j, e0 + k)) f[k] = 0.f;
        }
      }
      float4* d = reinterpret_cast<float4*>(dst + e0);
#pragma unroll
      for (int k = 0; k < V / 4; ++k) d[k] = make_float4(f[4 * k], f[4 * k + 1], f[4 * k + 2], f[4 * k + 3]);
    }
  }
  // scalar tail (n % V elements) by block 0
  if (blockIdx.x == 0) {
    for (int64_t i = nvec * V + threadIdx.x; i < n; i += CAST_THREADS) {
      float x = SRC_BF16 ? bf16lo(static_cast<const uint16_t*>(src)[i]) * scale
                         : static_cast<const float*>(src)[i] * scale;
      if (npad > 0 && in_pad_from(pad, npad, first_pad_after(pad, npad, i), i)) x = 0.f;
      dst[i] = x;
    }
  }
}

// misaligned fallback: one element per thread
template <bool SRC_BF16>
__global__ void cast_scale_scalar_kernel(const void* __restrict__ src, float* __restrict__ dst,
                                         int64_t n, float scale, const int64_t* __restrict__ pad,
                                         int npad) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    float x = SRC_BF16 ? bf16lo(static_cast<const uint16_t*>(src)[i]) * scale
                       : static_cast<const float*>(src)[i] * scale;
    if (npad > 0 && in_pad_from(pad, npad, first_pad_after(pad, npad, i), i)) x = 0.f;
    dst[i] = x;
  }
}

cudaError_t launch_cast_scale(const void* src, int src_bf16, float* dst, int64_t n, float scale,
                              const int64_t* pad_dev, int32_t npad, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const bool aligned = (reinterpret_cast<uintptr_t>(src) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(dst) % 16 == 0);
  const int V = src_bf16 ? 8 : 4;
  const int64_t nvec = n / V;
  if (!aligned) {
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 16);
    if (src_bf16)
      cast_scale_scalar_kernel<true><<<blocks, 256, 0, st>>>(src, dst, n, scale, pad_dev, npad);
    else
      cast_scale_scalar_kernel<false><<<blocks, 256, 0, st>>>(src, dst, n, scale, pad_dev, npad);
    return cudaGetLastError();
  }
  static int occ_bf16 = resident_blocks(cast_scale_kernel<true>, CAST_THREADS, 0);
  static int occ_f32 = resident_blocks(cast_scale_kernel<false>, CAST_THREADS, 0);
  const int64_t per_block = int64_t(CAST_THREADS) * CAST_UNROLL;
  const int64_t want = std::max<int64_t>(1, (nvec + per_block - 1) / per_block);
  const int64_t cap = int64_t(num_sms()) * (src_bf16 ? occ_bf16 : occ_f32);
  const int64_t blocks = std::min(want, cap);
  if (src_bf16)
    cast_scale_kernel<true><<<blocks, CAST_THREADS, 0, st>>>(src, dst, n, scale, pad_dev, npad);
  else
    cast_scale_kernel<false><<<blocks, CAST_THREADS, 0, st>>>(src, dst, n, scale, pad_dev, npad);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------
// a8: block-wise 8-bit Adam
// ----------------------------------------------------------------------------
constexpr int ADAM_THREADS = 256;
constexpr int ADAM_EPT = 8;                            // elements per thread
constexpr int ADAM_TILE = ADAM_THREADS * ADAM_EPT;     // 2048: single-pass block size
constexpr int ADAM_WARPS = ADAM_THREADS / 32;

struct ElemOut {
  float p, m, v;
};

// Steps 1-6 of the update for one element (O4); FMA-contracted where noted.
__device__ __forceinline__ ElemOut adam_elem(float p, float g, float mt, float vt,
                                             const AdamScalars& s) {
  ElemOut o;
  o.m = fmaf(s.w1, g - mt, mt);                    // mt + (1-b1)(g - mt)     (lerp)
  o.v = fmaf(s.b2, vt, s.w2 * (g * g));            // b2 vt + (1-b2) g^2
  const float denom = fmaf(sqrt_approx(o.v), s.inv_bc2s, s.eps);  // sqrt(v)/bc2s + eps
  o.p = fmaf(-s.step_size, __fdividef(o.m, denom), p * s.c_wd);   // p*c_wd - ss*m/denom
  return o;
}

__device__ __forceinline__ void block_max2(float& a, float& b, float* sa, float* sb) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sa[w] = a;
    sb[w] = b;
  }
  __syncthreads();
  a = sa[0];
  b = sb[0];
#pragma unroll
  for (int i = 1; i < ADAM_WARPS; ++i) {
    a = fmaxf(a, sa[i]);
    b = fmaxf(b, sb[i]);
  }
}

__device__ __forceinline__ uint32_t qm_code(float m, float inv) {  // -> byte of int8
  int q = rne_int(m * inv);
  q = max(-127, min(127, q));
  return uint32_t(q) & 0xffu;
}
__device__ __forceinline__ uint32_t qv_code(float v, float inv) {
  int q = rne_int(v * inv);
  q = max(0, min(255, q));
  return uint32_t(q);
}

template <bool PARAM_BF16>
__global__ void __launch_bounds__(ADAM_THREADS) adam8_kernel(const AdamBlock* __restrict__ tbl,
                                                             int64_t nblocks, AdamPtrs P,
                                                             AdamScalars s) {
  __shared__ float red_m[ADAM_WARPS], red_v[ADAM_WARPS];
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
    const AdamBlock blk = tbl[b];
    const int64_t slot = blk.slot;
    const float sm = P.mabs[slot] / 127.0f;  // dequantization scales (IEEE div)
    const float sv = P.vabs[slot] / 255.0f;
    float* __restrict__ master = P.master + blk.state_off;
    int8_t* __restrict__ mq = P.mq + blk.state_off;
    uint8_t* __restrict__ vq = P.vq + blk.state_off;
    const float* __restrict__ grad = P.grad + blk.grad_off;
    const int len = blk.len;

    if (len <= ADAM_TILE) {
      // ---------------- single pass: the block lives in registers ----------
      const int i0 = threadIdx.x * ADAM_EPT;
      const bool vec = (i0 + ADAM_EPT <= len) && ((blk.state_off & 7) == 0) &&
                       ((blk.grad_off & 3) == 0) && ((blk.param_off & 7) == 0);
      float p[ADAM_EPT], g[ADAM_EPT], mt[ADAM_EPT], vt[ADAM_EPT];
      if (vec) {
        const int4 p0 = ld_na_v4(master + i0), p1 = ld_na_v4(master + i0 + 4);
        const int4 g0 = ld_nc_v4(grad + i0), g1 = ld_nc_v4(grad + i0 + 4);
        const uint2 cm = ld_na_v2(mq + i0), cv = ld_na_v2(vq + i0);
        p[0] = __int_as_float(p0.x); p[1] = __int_as_float(p0.y);
        p[2] = __int_as_float(p0.z); p[3] = __int_as_float(p0.w);
        p[4] = __int_as_float(p1.x); p[5] = __int_as_float(p1.y);
        p[6] = __int_as_float(p1.z); p[7] = __int_as_float(p1.w);
        g[0] = __int_as_float(g0.x); g[1] = __int_as_float(g0.y);
        g[2] = __int_as_float(g0.z); g[3] = __int_as_float(g0.w);
        g[4] = __int_as_float(g1.x); g[5] = __int_as_float(g1.y);
        g[6] = __int_as_float(g1.z); g[7] = __int_as_float(g1.w);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          mt[k] = s8_to_f((cm.x >> (8 * k)) & 0xffu) * sm;
          mt[k + 4] = s8_to_f((cm.y >> (8 * k)) & 0xffu) * sm;
          vt[k] = u8_to_f((cv.x >> (8 * k)) & 0xffu) * sv;
          vt[k + 4] = u8_to_f((cv.y >> (8 * k)) & 0xffu) * sv;
        }
      } else {
#pragma unroll
        for (int k = 0; k < ADAM_EPT; ++k) {
          const int i = i0 + k;
          if (i < len) {
            p[k] = master[i];
            g[k] = grad[i];
            mt[k] = s8_to_f(uint32_t(uint8_t(mq[i]))) * sm;
            vt[k] = u8_to_f(uint32_t(vq[i])) * sv;
          } else {
            p[k] = g[k] = mt[k] = vt[k] = 0.f;
          }
        }
      }
      float m[ADAM_EPT], v[ADAM_EPT];
      float am = 0.f, av = 0.f;
#pragma unroll
      for (int k = 0; k < ADAM_EPT; ++k) {
        const ElemOut o = adam_elem(p[k], g[k], mt[k], vt[k], s);
        const bool live = (i0 + k) < len;
        p[k] = o.p;
        m[k] = live ? o.m : 0.f;
        v[k] = live ? o.v : 0.f;
        am = fmaxf(am, fabsf(m[k]));
        av = fmaxf(av, v[k]);
      }
      block_max2(am, av, red_m, red_v);
      const float im = am > 0.f ? 127.0f / am : 0.f;
      const float iv = av > 0.f ? 255.0f / av : 0.f;
      if (vec) {
        uint2 cm, cv;
        cm.x = qm_code(m[0], im) | (qm_code(m[1], im) << 8) | (qm_code(m[2], im) << 16) |
               (qm_code(m[3], im) << 24);
        cm.y = qm_code(m[4], im) | (qm_code(m[5], im) << 8) | (qm_code(m[6], im) << 16) |
               (qm_code(m[7], im) << 24);
        cv.x = qv_code(v[0], iv) | (qv_code(v[1], iv) << 8) | (qv_code(v[2], iv) << 16) |
               (qv_code(v[3], iv) << 24);
        cv.y = qv_code(v[4], iv) | (qv_code(v[5], iv) << 8) | (qv_code(v[6], iv) << 16) |
               (qv_code(v[7], iv) << 24);
        reinterpret_cast<float4*>(master + i0)[0] = make_float4(p[0], p[1], p[2], p[3]);
        reinterpret_cast<float4*>(master + i0)[1] = make_float4(p[4], p[5], p[6], p[7]);
        *reinterpret_cast<uint2*>(mq + i0) = cm;
        *reinterpret_cast<uint2*>(vq + i0) = cv;
        if constexpr (PARAM_BF16) {
          uint4 o;
          o.x = pack_bf16x2(p[0], p[1]);
          o.y = pack_bf16x2(p[2], p[3]);
          o.z = pack_bf16x2(p[4], p[5]);
          o.w = pack_bf16x2(p[6], p[7]);
          *reinterpret_cast<uint4*>(static_cast<uint16_t*>(P.param) + blk.param_off + i0) = o;
        } else {
          float* pp = static_cast<float*>(P.param) + blk.param_off + i0;
          reinterpret_cast<float4*>(pp)[0] = make_float4(p[0], p[1], p[2], p[3]);
          reinterpret_cast<float4*>(pp)[1] = make_float4(p[4], p[5], p[6], p[7]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < ADAM_EPT; ++k) {
          const int i = i0 + k;
          if (i < len) {
            master[i] = p[k];
            mq[i] = int8_t(qm_code(m[k], im));
            vq[i] = uint8_t(qv_code(v[k], iv));
            if constexpr (PARAM_BF16) {
              const __nv_bfloat16 h = __float2bfloat16_rn(p[k]);
              static_cast<__nv_bfloat16*>(P.param)[blk.param_off + i] = h;
            } else {
              static_cast<float*>(P.param)[blk.param_off + i] = p[k];
            }
          }
        }
      }
      if (threadIdx.x == 0) {
        P.mabs[slot] = am;
        P.vabs[slot] = av;
      }
    } else {
      // ---------------- two passes for blocks longer than 2048 -------------
      float am = 0.f, av = 0.f;
      for (int i = threadIdx.x; i < len; i += ADAM_THREADS) {
        const ElemOut o = adam_elem(0.f, grad[i], s8_to_f(uint32_t(uint8_t(mq[i]))) * sm,
                                    u8_to_f(uint32_t(vq[i])) * sv, s);
        am = fmaxf(am, fabsf(o.m));
        av = fmaxf(av, o.v);
      }
      block_max2(am, av, red_m, red_v);
      const float im = am > 0.f ? 127.0f / am : 0.f;
      const float iv = av > 0.f ? 255.0f / av : 0.f;
      __syncthreads();  // every thread has read the old codes of ITS elements
                        // only, so no cross-thread hazard; keep reduction smem safe
      for (int i = threadIdx.x; i < len; i += ADAM_THREADS) {
        const ElemOut o = adam_elem(master[i], grad[i], s8_to_f(uint32_t(uint8_t(mq[i]))) * sm,
                                    u8_to_f(uint32_t(vq[i])) * sv, s);
        master[i] = o.p;
        mq[i] = int8_t(qm_code(o.m, im));
        vq[i] = uint8_t(qv_code(o.v, iv));
        if constexpr (PARAM_BF16)
          static_cast<__nv_bfloat16*>(P.param)[blk.param_off + i] = __float2bfloat16_rn(o.p);
        else
          static_cast<float*>(P.param)[blk.param_off + i] = o.p;
      }
      if (threadIdx.x == 0) {
        P.mabs[slot] = am;
        P.vabs[slot] = av;
      }
    }
    __syncthreads();  // red_m/red_v reused by the next block
  }
}

cudaError_t launch_adam8(const AdamBlock* table_dev, int64_t nblocks, const AdamPtrs& p,
                         const AdamScalars& s, int32_t /*max_len*/, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  static int occ_bf = resident_blocks(adam8_kernel<true>, ADAM_THREADS, 0);
  static int occ_f = resident_blocks(adam8_kernel<false>, ADAM_THREADS, 0);
  const int64_t cap = int64_t(num_sms()) * (p.param_bf16 ? occ_bf : occ_f);
  const int64_t blocks = std::min<int64_t>(nblocks, cap);
  if (p.param_bf16)
    adam8_kernel<true><<<blocks, ADAM_THREADS, 0, st>>>(table_dev, nblocks, p, s);
  else
    adam8_kernel<false><<<blocks, ADAM_THREADS, 0, st>>>(table_dev, nblocks, p, s);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------
// batched ragged copy (+cast, +scale)
// ----------------------------------------------------------------------------
constexpr int COPY_THREADS = 256;
constexpr int64_t COPY_CHUNK = 4096;  // elements per chunk

__device__ __forceinline__ float load_as_f(const void* p, int64_t i, bool bf16) {
  return bf16 ? bf16lo(static_cast<const uint16_t*>(p)[i]) : static_cast<const float*>(p)[i];
}
__device__ __forceinline__ void store_from_f(void* p, int64_t i, float x, bool bf16) {
  if (bf16)
    static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(x);
  else
    static_cast<float*>(p)[i] = x;
}

__global__ void __launch_bounds__(COPY_THREADS) copy_seg_kernel(const CopySeg* __restrict__ segs,
                                                                int64_t nseg, int64_t total_chunks,
                                                                int src_bf16, int dst_bf16,
                                                                float scale) {
  for (int64_t c = blockIdx.x; c < total_chunks; c += gridDim.x) {
    // segment owning chunk c: last s with chunk_begin <= c
    int64_t lo = 0, hi = nseg - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (segs[mid].chunk_begin <= c)
        lo = mid;
      else
        hi = mid - 1;
    }
    const CopySeg sg = segs[lo];
    const int64_t e0 = (c - sg.chunk_begin) * COPY_CHUNK;
    const int64_t n = min(COPY_CHUNK, sg.numel - e0);
    const bool same = src_bf16 == dst_bf16 && scale == 1.0f;
    const int eb_s = src_bf16 ? 2 : 4, eb_d = dst_bf16 ? 2 : 4;
    const char* s = static_cast<const char*>(sg.src) + e0 * eb_s;
    char* d = static_cast<char*>(sg.dst) + e0 * eb_d;
    if (same && (reinterpret_cast<uintptr_t>(s) % 16 == 0) &&
        (reinterpret_cast<uintptr_t>(d) % 16 == 0)) {
      const int64_t nbytes = n * eb_s, nv = nbytes / 16;
      for (int64_t i = threadIdx.x; i < nv; i += COPY_THREADS)
        reinterpret_cast<int4*>(d)[i] = ld_nc_v4(reinterpret_cast<const int4*>(s) + i);
      for (int64_t i = nv * 16 + threadIdx.x; i < nbytes; i += COPY_THREADS) d[i] = s[i];
    } else {
      for (int64_t i = threadIdx.x; i < n; i += COPY_THREADS)
        store_from_f(d, i, load_as_f(s, i, src_bf16) * scale, dst_bf16);
    }
  }
}

cudaError_t launch_copy_segments(const CopySeg* segs_dev, int64_t nseg, int64_t total_chunks,
                                 int src_bf16, int dst_bf16, float scale, cudaStream_t st) {
  if (total_chunks <= 0 || nseg <= 0) return cudaSuccess;
  static int occ = resident_blocks(copy_seg_kernel, COPY_THREADS, 0);
  const int64_t blocks = std::min<int64_t>(total_chunks, int64_t(num_sms()) * occ);
  copy_seg_kernel<<<blocks, COPY_THREADS, 0, st>>>(segs_dev, nseg, total_chunks, src_bf16,
                                                   dst_bf16, scale);
  return cudaGetLastError();
}

}  // namespace rsdb
