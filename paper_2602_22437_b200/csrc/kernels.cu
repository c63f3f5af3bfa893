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

#include <cstdlib>
#include <cstring>

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
__device__ __forceinline__ uint32_t ld_na_u32(const void* p) {
  uint32_t r;
  asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
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
// .ftz approximations: v = 0 or denormal gives sqrt = 0 (the denominator is
// then eps = 1e-8 either way); denom >= eps is never denormal.
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
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
constexpr int CAST_UNROLL = 8;
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
  // Each thread moves 4 elements per vector: an 8-byte (bf16) or 16-byte
  // (f32) load and ONE 16-byte store, so every warp instruction covers a
  // contiguous span (no half-sector strided stores).
  constexpr int V = 4;
  const int64_t nvec = n / V;
  const int64_t stride = int64_t(gridDim.x) * CAST_THREADS * CAST_UNROLL;
  for (int64_t base = int64_t(blockIdx.x) * CAST_THREADS * CAST_UNROLL + threadIdx.x; base < nvec;
       base += stride) {
    float f[CAST_UNROLL][V];
#pragma unroll
    for (int u = 0; u < CAST_UNROLL; ++u) {
      const int64_t c = base + u * CAST_THREADS;
      if (c < nvec) {
        if constexpr (SRC_BF16) {
          const uint2 w = ld_nc_v2(static_cast<const uint2*>(src) + c);
          f[u][0] = bf16lo(w.x);
          f[u][1] = bf16hi(w.x);
          f[u][2] = bf16lo(w.y);
          f[u][3] = bf16hi(w.y);
        } else {
          const int4 w = ld_nc_v4(static_cast<const int4*>(src) + c);
          f[u][0] = __int_as_float(w.x);
          f[u][1] = __int_as_float(w.y);
          f[u][2] = __int_as_float(w.z);
          f[u][3] = __int_as_float(w.w);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < CAST_UNROLL; ++u) {
      const int64_t c = base + u * CAST_THREADS;
      if (c >= nvec) break;
      float x[V];
#pragma unroll
      for (int k = 0; k < V; ++k) x[k] = f[u][k] * scale;
      const int64_t e0 = c * V;
      if (npad > 0) {
        const int j = first_pad_after(pad, npad, e0);
        if (j < npad && pad[2 * j] < e0 + V) {
#pragma unroll
          for (int k = 0; k < V; ++k)
            if (in_pad_from(pad, npad, j, e0 + k)) x[k] = 0.f;
        }
      }
      *reinterpret_cast<float4*>(dst + e0) = make_float4(x[0], x[1], x[2], x[3]);
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
  const int64_t nvec = n / 4;
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
//
// One CTA of NT threads per 2048-element quantization block; thread t owns
// Q = 512/NT quads [4t + 4*NT*k, +4), k < Q, so every warp-wide access is one
// contiguous span.  Two kernels share the per-block body:
//   adam8_kernel      loads straight from global memory (16-B vectors);
//   adam8_tma_kernel  persistent CTAs with a ring of shared-memory stages
//                     filled by 1-D bulk TMA (cp.async.bulk, mbarrier
//                     complete_tx): the next blocks stream in while the
//                     current one is reduced, quantized and stored.
// Blocks that are not full (tails) or not 16-B aligned take a masked
// element path; blocks longer than 2048 take a two-pass path.
//
// Instruction diet (the kernel is HBM-bound only if it issues < ~30
// instructions per element): codes are widened with one PRMT per byte into
// the float 2^23 + code (exact; then FADD/FMUL = the oracle's q * fl(A/127)),
// requantised with the magic-add RNE whose float bits carry the code in
// their low byte (3 PRMT per 4 codes), and no clamp is needed because
// |m| <= A  =>  |m * fl(127/A)| < 127.5 (and 0 <= v * fl(255/A) < 255.5).
// ----------------------------------------------------------------------------
constexpr int ADAM_TILE = 2048;  // single-pass block size

struct ElemOut {
  float p, m, v;
};

template <int NT>
struct AdamGeom {
  static constexpr int Q = ADAM_TILE / (4 * NT);  // quads per thread
  static constexpr int EPT = 4 * Q;               // elements per thread
  static constexpr int WARPS = NT / 32;
  // element index (inside the block) of this thread's e-th element
  __device__ static __forceinline__ int idx(int e) { return 4 * int(threadIdx.x) + (e >> 2) * 4 * NT + (e & 3); }
  __device__ static __forceinline__ int quad(int k) { return 4 * int(threadIdx.x) + 4 * NT * k; }
};

// Steps 1-6 of the update for one element (O4); FMA-contracted.
__device__ __forceinline__ ElemOut adam_elem(float p, float g, float mt, float vt,
                                             const AdamScalars& s) {
  ElemOut o;
  o.m = fmaf(s.w1, g - mt, mt);                    // mt + (1-b1)(g - mt)     (lerp)
  o.v = fmaf(s.b2, vt, s.w2 * (g * g));            // b2 vt + (1-b2) g^2
  const float denom = fmaf(sqrt_approx(o.v), s.inv_bc2s, s.eps);  // sqrt(v)/bc2s + eps
  o.p = fmaf(-s.step_size, o.m * rcp_approx(denom), p * s.c_wd);  // p*c_wd - ss*m/denom
  return o;
}

template <int WARPS>
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
  for (int i = 1; i < WARPS; ++i) {
    a = fmaxf(a, sa[i]);
    b = fmaxf(b, sb[i]);
  }
}

// byte k of w as the float 2^23 + byte (exact)
__device__ __forceinline__ float byte_f(uint32_t w, int k) {
  return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540u + k));
}
// 4 dequantized moments from a word of codes: m signed (bias 128), v unsigned
__device__ __forceinline__ void dq4_m(uint32_t w, float sm, float* out) {
  w ^= 0x80808080u;
#pragma unroll
  for (int k = 0; k < 4; ++k) out[k] = (byte_f(w, k) - 8388736.0f) * sm;  // (code) * fl(A/127)
}
__device__ __forceinline__ void dq4_v(uint32_t w, float sv, float* out) {
#pragma unroll
  for (int k = 0; k < 4; ++k) out[k] = (byte_f(w, k) - 8388608.0f) * sv;  // (code) * fl(A/255)
}
// RNE code in the low byte of the float bits of x + 1.5*2^23 (|x| < 2^22)
__device__ __forceinline__ uint32_t rne_bits(float x) {
  return __float_as_uint(__fadd_rn(x, 12582912.0f));
}
__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040u), __byte_perm(c, d, 0x0040u), 0x5410u);
}
// scalar code (masked path), with the same rounding
__device__ __forceinline__ uint8_t code1(float x) { return uint8_t(rne_bits(x) & 0xffu); }

template <int NT>
struct BlockRegs {
  float p[AdamGeom<NT>::EPT], g[AdamGeom<NT>::EPT], mt[AdamGeom<NT>::EPT], vt[AdamGeom<NT>::EPT];
};

// full, 16-B aligned block from 4 element arrays (global or shared)
template <int NT, bool GLOBAL>
__device__ __forceinline__ void load_fast(BlockRegs<NT>& r, const float* master, const float* grad,
                                          const void* mq, const void* vq, float sm, float sv) {
  using G = AdamGeom<NT>;
  int4 pv[G::Q], gv[G::Q];
  uint32_t cm[G::Q], cv[G::Q];
#pragma unroll
  for (int k = 0; k < G::Q; ++k) {
    const int a = G::quad(k);
    if constexpr (GLOBAL) {
      pv[k] = ld_na_v4(master + a);
      gv[k] = ld_nc_v4(grad + a);
      cm[k] = ld_na_u32(static_cast<const uint8_t*>(mq) + a);
      cv[k] = ld_na_u32(static_cast<const uint8_t*>(vq) + a);
    } else {
      pv[k] = *reinterpret_cast<const int4*>(master + a);
      gv[k] = *reinterpret_cast<const int4*>(grad + a);
      cm[k] = *reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(mq) + a);
      cv[k] = *reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(vq) + a);
    }
  }
#pragma unroll
  for (int k = 0; k < G::Q; ++k) {
    r.p[4 * k + 0] = __int_as_float(pv[k].x);
    r.p[4 * k + 1] = __int_as_float(pv[k].y);
    r.p[4 * k + 2] = __int_as_float(pv[k].z);
    r.p[4 * k + 3] = __int_as_float(pv[k].w);
    r.g[4 * k + 0] = __int_as_float(gv[k].x);
    r.g[4 * k + 1] = __int_as_float(gv[k].y);
    r.g[4 * k + 2] = __int_as_float(gv[k].z);
    r.g[4 * k + 3] = __int_as_float(gv[k].w);
    dq4_m(cm[k], sm, &r.mt[4 * k]);
    dq4_v(cv[k], sv, &r.vt[4 * k]);
  }
}

// element i of a block laid out as rows of `cols` elements `pitch` apart
__device__ __forceinline__ int64_t blk_off(const AdamBlock& b, int i) {
  const int row = i / b.cols;
  return int64_t(row) * b.pitch + (i - row * b.cols);
}

// masked, strided element loads (tails, misaligned blocks, odd tiles)
template <int NT>
__device__ __forceinline__ void load_generic(BlockRegs<NT>& r, const AdamBlock& blk,
                                             const AdamPtrs& P, float sm, float sv) {
  using G = AdamGeom<NT>;
  const float* master = P.master + blk.state_off;
  const float* grad = P.grad + blk.grad_off;
  const int8_t* mq = P.mq + blk.state_off;
  const uint8_t* vq = P.vq + blk.state_off;
#pragma unroll
  for (int e = 0; e < G::EPT; ++e) {
    const int i = G::idx(e);
    if (i < blk.len) {
      const int64_t o = blk_off(blk, i);
      r.p[e] = master[o];
      r.g[e] = grad[o];
      r.mt[e] = (byte_f(uint32_t(uint8_t(mq[o])) ^ 0x80u, 0) - 8388736.0f) * sm;
      r.vt[e] = (byte_f(uint32_t(vq[o]), 0) - 8388608.0f) * sv;
    } else {
      r.p[e] = r.g[e] = r.mt[e] = r.vt[e] = 0.f;
    }
  }
}

// 2-D tile with cols % 4 == 0 (quads never cross a row) and 16-B aligned rows:
// every quad is one 16-B vector at its own row address (N2, 32x32 tiles)
template <int NT>
__device__ __forceinline__ void load_tile(BlockRegs<NT>& r, const AdamBlock& blk, const AdamPtrs& P,
                                          float sm, float sv) {
  using G = AdamGeom<NT>;
  int4 pv[G::Q], gv[G::Q];
  uint32_t cm[G::Q], cv[G::Q];
#pragma unroll
  for (int k = 0; k < G::Q; ++k) {
    const int e0 = G::quad(k);
    if (e0 < blk.len) {
      const int64_t a = blk_off(blk, e0);
      pv[k] = ld_na_v4(P.master + blk.state_off + a);
      gv[k] = ld_nc_v4(P.grad + blk.grad_off + a);
      cm[k] = ld_na_u32(P.mq + blk.state_off + a);
      cv[k] = ld_na_u32(P.vq + blk.state_off + a);
    } else {
      pv[k] = gv[k] = make_int4(0, 0, 0, 0);
      cm[k] = 0x80808080u;  // decodes to m = 0
      cv[k] = 0u;
    }
  }
#pragma unroll
  for (int k = 0; k < G::Q; ++k) {
    r.p[4 * k + 0] = __int_as_float(pv[k].x);
    r.p[4 * k + 1] = __int_as_float(pv[k].y);
    r.p[4 * k + 2] = __int_as_float(pv[k].z);
    r.p[4 * k + 3] = __int_as_float(pv[k].w);
    r.g[4 * k + 0] = __int_as_float(gv[k].x);
    r.g[4 * k + 1] = __int_as_float(gv[k].y);
    r.g[4 * k + 2] = __int_as_float(gv[k].z);
    r.g[4 * k + 3] = __int_as_float(gv[k].w);
    dq4_m(cm[k], sm, &r.mt[4 * k]);
    dq4_v(cv[k], sv, &r.vt[4 * k]);
  }
}

// Update + block absmax + (hook) + requantize + stores, for a block held in
// registers.  `after_reduce` runs once every thread of the CTA has its inputs
// in registers (right after the absmax reduction's barrier).
// MODE 0: masked strided elements; 1: full contiguous 2048 block; 2: 2-D tile quads
template <int NT, bool PARAM_BF16, int MODE, typename Hook>
__device__ __forceinline__ void adam_block_tail(BlockRegs<NT>& r, const AdamBlock& blk,
                                                const AdamPtrs& P, const AdamScalars& s,
                                                float* red_m, float* red_v, Hook after_reduce) {
  using G = AdamGeom<NT>;
  const int len = blk.len;
  float m[G::EPT], v[G::EPT];
  float am = 0.f, av = 0.f;
#pragma unroll
  for (int e = 0; e < G::EPT; ++e) {
    const ElemOut o = adam_elem(r.p[e], r.g[e], r.mt[e], r.vt[e], s);
    const bool live = MODE == 1 || G::idx(e) < len;
    r.p[e] = o.p;
    m[e] = live ? o.m : 0.f;
    v[e] = live ? o.v : 0.f;
    am = fmaxf(am, fabsf(m[e]));
    av = fmaxf(av, v[e]);
  }
  block_max2<G::WARPS>(am, av, red_m, red_v);
  after_reduce();
  const float im = am > 0.f ? 127.0f / am : 0.f;
  const float iv = av > 0.f ? 255.0f / av : 0.f;
  float* __restrict__ master = P.master + blk.state_off;
  uint8_t* __restrict__ mq = reinterpret_cast<uint8_t*>(P.mq) + blk.state_off;
  uint8_t* __restrict__ vq = P.vq + blk.state_off;
  if constexpr (MODE != 0) {
#pragma unroll
    for (int k = 0; k < G::Q; ++k) {
      int64_t a = G::quad(k);
      if constexpr (MODE == 2) {
        if (a >= len) continue;
        a = blk_off(blk, int(a));
      }
      const float* pk = &r.p[4 * k];
      const float* mk = &m[4 * k];
      const float* vk = &v[4 * k];
      *reinterpret_cast<float4*>(master + a) = make_float4(pk[0], pk[1], pk[2], pk[3]);
      *reinterpret_cast<uint32_t*>(mq + a) = pack4(rne_bits(mk[0] * im), rne_bits(mk[1] * im),
                                                   rne_bits(mk[2] * im), rne_bits(mk[3] * im));
      *reinterpret_cast<uint32_t*>(vq + a) = pack4(rne_bits(vk[0] * iv), rne_bits(vk[1] * iv),
                                                   rne_bits(vk[2] * iv), rne_bits(vk[3] * iv));
      if constexpr (PARAM_BF16) {
        uint16_t* pp = static_cast<uint16_t*>(P.param) + blk.param_off;
        *reinterpret_cast<uint2*>(pp + a) =
            make_uint2(pack_bf16x2(pk[0], pk[1]), pack_bf16x2(pk[2], pk[3]));
      } else {
        float* pp = static_cast<float*>(P.param) + blk.param_off;
        *reinterpret_cast<float4*>(pp + a) = make_float4(pk[0], pk[1], pk[2], pk[3]);
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < G::EPT; ++e) {
      const int i = G::idx(e);
      if (i < len) {
        const int64_t o = blk_off(blk, i);
        master[o] = r.p[e];
        mq[o] = code1(m[e] * im);
        vq[o] = code1(v[e] * iv);
        if constexpr (PARAM_BF16)
          static_cast<__nv_bfloat16*>(P.param)[blk.param_off + o] = __float2bfloat16_rn(r.p[e]);
        else
          static_cast<float*>(P.param)[blk.param_off + o] = r.p[e];
      }
    }
  }
  if (threadIdx.x == 0) {
    P.mabs[blk.slot] = am;
    P.vabs[blk.slot] = av;
  }
}

// blocks longer than 2048: pass 1 computes the absmax, pass 2 recomputes and stores
template <int NT, bool PARAM_BF16, typename Hook>
__device__ __forceinline__ void adam_block_two_pass(const AdamBlock& blk, float sm, float sv,
                                                    const AdamPtrs& P, const AdamScalars& s,
                                                    float* red_m, float* red_v, Hook after_reduce) {
  float* __restrict__ master = P.master + blk.state_off;
  uint8_t* __restrict__ mq = reinterpret_cast<uint8_t*>(P.mq) + blk.state_off;
  uint8_t* __restrict__ vq = P.vq + blk.state_off;
  const float* __restrict__ grad = P.grad + blk.grad_off;
  auto mt_of = [&](int64_t o) { return (byte_f(uint32_t(mq[o]) ^ 0x80u, 0) - 8388736.0f) * sm; };
  auto vt_of = [&](int64_t o) { return (byte_f(uint32_t(vq[o]), 0) - 8388608.0f) * sv; };
  float am = 0.f, av = 0.f;
  for (int i = threadIdx.x; i < blk.len; i += NT) {
    const int64_t o = blk_off(blk, i);
    const ElemOut e = adam_elem(0.f, grad[o], mt_of(o), vt_of(o), s);
    am = fmaxf(am, fabsf(e.m));
    av = fmaxf(av, e.v);
  }
  block_max2<AdamGeom<NT>::WARPS>(am, av, red_m, red_v);
  after_reduce();
  const float im = am > 0.f ? 127.0f / am : 0.f;
  const float iv = av > 0.f ? 255.0f / av : 0.f;
  // each thread rewrites exactly the elements it read in pass 1: no hazard
  for (int i = threadIdx.x; i < blk.len; i += NT) {
    const int64_t q = blk_off(blk, i);
    const ElemOut o = adam_elem(master[q], grad[q], mt_of(q), vt_of(q), s);
    master[q] = o.p;
    mq[q] = code1(o.m * im);
    vq[q] = code1(o.v * iv);
    if constexpr (PARAM_BF16)
      static_cast<__nv_bfloat16*>(P.param)[blk.param_off + q] = __float2bfloat16_rn(o.p);
    else
      static_cast<float*>(P.param)[blk.param_off + q] = o.p;
  }
  if (threadIdx.x == 0) {
    P.mabs[blk.slot] = am;
    P.vabs[blk.slot] = av;
  }
}

__device__ __forceinline__ bool adam_fast(const AdamBlock& b) {
  return b.len == ADAM_TILE && b.cols == b.len && ((b.state_off | b.grad_off | b.param_off) & 3) == 0;
}
__device__ __forceinline__ bool adam_tile_fast(const AdamBlock& b) {
  return b.cols != b.len && ((b.cols | b.pitch) & 3) == 0 &&
         ((b.state_off | b.grad_off | b.param_off) & 3) == 0;
}

struct NoHook {
  __device__ void operator()() const {}
};

template <int NT, bool PARAM_BF16>
__device__ __forceinline__ void adam_block_global(const AdamBlock& blk, const AdamPtrs& P,
                                                  const AdamScalars& s, float sm, float sv,
                                                  float* rm, float* rv) {
  if (blk.len <= ADAM_TILE) {
    BlockRegs<NT> r;
    if (adam_fast(blk)) {
      load_fast<NT, true>(r, P.master + blk.state_off, P.grad + blk.grad_off, P.mq + blk.state_off,
                          P.vq + blk.state_off, sm, sv);
      adam_block_tail<NT, PARAM_BF16, 1>(r, blk, P, s, rm, rv, NoHook{});
    } else if (adam_tile_fast(blk)) {
      load_tile<NT>(r, blk, P, sm, sv);
      adam_block_tail<NT, PARAM_BF16, 2>(r, blk, P, s, rm, rv, NoHook{});
    } else {
      load_generic<NT>(r, blk, P, sm, sv);
      adam_block_tail<NT, PARAM_BF16, 0>(r, blk, P, s, rm, rv, NoHook{});
    }
  } else {
    adam_block_two_pass<NT, PARAM_BF16>(blk, sm, sv, P, s, rm, rv, NoHook{});
  }
}

template <int NT, bool PARAM_BF16>
__global__ void __launch_bounds__(NT) adam8_kernel(const AdamBlock* __restrict__ tbl,
                                                   int64_t nblocks, AdamPtrs P, AdamScalars s) {
  __shared__ float red_m[2][AdamGeom<NT>::WARPS], red_v[2][AdamGeom<NT>::WARPS];
  int it = 0;
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++it) {
    const AdamBlock blk = tbl[b];
    const float sm = P.mabs[blk.slot] / 127.0f;  // dequantization scales (IEEE div)
    const float sv = P.vabs[blk.slot] / 255.0f;
    // red_m/red_v are double-buffered: a thread can be at most one block
    // ahead (every block has a barrier), so no trailing __syncthreads.
    adam_block_global<NT, PARAM_BF16>(blk, P, s, sm, sv, red_m[it & 1], red_v[it & 1]);
  }
}

// ---------------- TMA-pipelined variant ----------------
struct __align__(128) AdamStage {
  float p[ADAM_TILE];
  float g[ADAM_TILE];
  uint8_t mq[ADAM_TILE];
  uint8_t vq[ADAM_TILE];
};
constexpr uint32_t ADAM_STAGE_TX = sizeof(float) * ADAM_TILE * 2 + ADAM_TILE * 2;  // 20480

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// bulk copies need 16-B aligned global addresses: codes at state_off % 16
__device__ __forceinline__ bool adam_tma_ok(const AdamBlock& b) {
  return b.len == ADAM_TILE && b.cols == b.len && (b.state_off & 15) == 0 &&
         ((b.grad_off | b.param_off) & 3) == 0;
}

template <int NT, bool PARAM_BF16, int STAGES>
__global__ void __launch_bounds__(NT) adam8_tma_kernel(const AdamBlock* __restrict__ tbl,
                                                       int64_t nblocks, AdamPtrs P, AdamScalars s) {
  extern __shared__ __align__(128) uint8_t adam_smem[];
  AdamStage* stage = reinterpret_cast<AdamStage*>(adam_smem);
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ float red_m[2][AdamGeom<NT>::WARPS], red_v[2][AdamGeom<NT>::WARPS];

  // thread 0 fills stage `st` with block b (or just arrives if b is not TMA-able)
  auto issue = [&](int64_t b, int st) {
    const AdamBlock nb = tbl[b];
    if (adam_tma_ok(nb)) {
      mbar_arrive_expect_tx(&full[st], ADAM_STAGE_TX);
      bulk_g2s(stage[st].p, P.master + nb.state_off, sizeof(float) * ADAM_TILE, &full[st]);
      bulk_g2s(stage[st].g, P.grad + nb.grad_off, sizeof(float) * ADAM_TILE, &full[st]);
      bulk_g2s(stage[st].mq, P.mq + nb.state_off, ADAM_TILE, &full[st]);
      bulk_g2s(stage[st].vq, P.vq + nb.state_off, ADAM_TILE, &full[st]);
    } else {
      mbar_arrive(&full[st]);
    }
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < STAGES; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int st = 0; st < STAGES; ++st) {
      const int64_t b = blockIdx.x + int64_t(st) * gridDim.x;
      if (b < nblocks) issue(b, st);
    }
  }
  __syncthreads();
  int it = 0;
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++it) {
    const int st = it % STAGES;
    const uint32_t ph = uint32_t(it / STAGES) & 1u;
    const AdamBlock blk = tbl[b];
    const float sm = P.mabs[blk.slot] / 127.0f;
    const float sv = P.vabs[blk.slot] / 255.0f;
    float* rm = red_m[it & 1];
    float* rv = red_v[it & 1];
    // refill this stage with block b + STAGES*grid once every thread has
    // consumed it (called right after the absmax barrier)
    auto refill = [&]() {
      if (threadIdx.x == 0) {
        const int64_t nb = b + int64_t(STAGES) * gridDim.x;
        if (nb < nblocks) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads -> async writes
          issue(nb, st);
        }
      }
    };
    mbar_wait(&full[st], ph);
    if (adam_tma_ok(blk)) {
      const AdamStage& S = stage[st];
      BlockRegs<NT> r;
      load_fast<NT, false>(r, S.p, S.g, S.mq, S.vq, sm, sv);
      adam_block_tail<NT, PARAM_BF16, 1>(r, blk, P, s, rm, rv, refill);
    } else if (blk.len <= ADAM_TILE) {
      BlockRegs<NT> r;
      if (adam_fast(blk)) {
        load_fast<NT, true>(r, P.master + blk.state_off, P.grad + blk.grad_off,
                            P.mq + blk.state_off, P.vq + blk.state_off, sm, sv);
        adam_block_tail<NT, PARAM_BF16, 1>(r, blk, P, s, rm, rv, refill);
      } else if (adam_tile_fast(blk)) {
        load_tile<NT>(r, blk, P, sm, sv);
        adam_block_tail<NT, PARAM_BF16, 2>(r, blk, P, s, rm, rv, refill);
      } else {
        load_generic<NT>(r, blk, P, sm, sv);
        adam_block_tail<NT, PARAM_BF16, 0>(r, blk, P, s, rm, rv, refill);
      }
    } else {
      adam_block_two_pass<NT, PARAM_BF16>(blk, sm, sv, P, s, rm, rv, refill);
    }
  }
}

// Variant switch (experiments; the default is the measured best):
// RSDB_ADAM_KERNEL = direct128 | direct256 | tma2 | tma3 | tma4  (TMA: 128 threads)
static int adam_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RSDB_ADAM_KERNEL");
    v = 3;  // measured best on B200: TMA ring of 3 stages, 128 threads (profiles/r1)
    if (e && !strcmp(e, "direct128")) v = 128;
    if (e && !strcmp(e, "direct256")) v = 256;
    if (e && !strcmp(e, "tma2")) v = 2;
    if (e && !strcmp(e, "tma3")) v = 3;
    if (e && !strcmp(e, "tma4")) v = 4;
  }
  return v;
}

template <int NT, bool BF, int ST>
static cudaError_t launch_adam8_tma(const AdamBlock* tbl, int64_t nblocks, const AdamPtrs& p,
                                    const AdamScalars& s, cudaStream_t st) {
  const size_t smem = sizeof(AdamStage) * ST;
  static int occ = [&] {
    cudaFuncSetAttribute(adam8_tma_kernel<NT, BF, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
    return resident_blocks(adam8_tma_kernel<NT, BF, ST>, NT, smem);
  }();
  const int64_t blocks = std::min<int64_t>(nblocks, int64_t(num_sms()) * occ);
  adam8_tma_kernel<NT, BF, ST><<<blocks, NT, smem, st>>>(tbl, nblocks, p, s);
  return cudaGetLastError();
}

template <int NT, bool BF>
static cudaError_t launch_adam8_direct(const AdamBlock* tbl, int64_t nblocks, const AdamPtrs& p,
                                       const AdamScalars& s, cudaStream_t st) {
  static int occ = resident_blocks(adam8_kernel<NT, BF>, NT, 0);
  const int64_t blocks = std::min<int64_t>(nblocks, int64_t(num_sms()) * occ);
  adam8_kernel<NT, BF><<<blocks, NT, 0, st>>>(tbl, nblocks, p, s);
  return cudaGetLastError();
}

cudaError_t launch_adam8(const AdamBlock* table_dev, int64_t nblocks, const AdamPtrs& p,
                         const AdamScalars& s, int32_t /*max_len*/, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  const bool bf = p.param_bf16;
  switch (adam_variant()) {
    case 2:
      return bf ? launch_adam8_tma<128, true, 2>(table_dev, nblocks, p, s, st)
                : launch_adam8_tma<128, false, 2>(table_dev, nblocks, p, s, st);
    case 3:
      return bf ? launch_adam8_tma<128, true, 3>(table_dev, nblocks, p, s, st)
                : launch_adam8_tma<128, false, 3>(table_dev, nblocks, p, s, st);
    case 4:
      return bf ? launch_adam8_tma<128, true, 4>(table_dev, nblocks, p, s, st)
                : launch_adam8_tma<128, false, 4>(table_dev, nblocks, p, s, st);
    case 256:
      return bf ? launch_adam8_direct<256, true>(table_dev, nblocks, p, s, st)
                : launch_adam8_direct<256, false>(table_dev, nblocks, p, s, st);
    default:
      return bf ? launch_adam8_direct<128, true>(table_dev, nblocks, p, s, st)
                : launch_adam8_direct<128, false>(table_dev, nblocks, p, s, st);
  }
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
    } else if ((reinterpret_cast<uintptr_t>(s) % (4 * eb_s) == 0) &&
               (reinterpret_cast<uintptr_t>(d) % (4 * eb_d) == 0)) {
      // cast / scale, 4 elements per thread per vector (8- or 16-byte accesses)
      const int64_t nv = n / 4;
      for (int64_t i = threadIdx.x; i < nv; i += COPY_THREADS) {
        float f[4];
        if (src_bf16) {
          const uint2 w = reinterpret_cast<const uint2*>(s)[i];
          f[0] = bf16lo(w.x), f[1] = bf16hi(w.x), f[2] = bf16lo(w.y), f[3] = bf16hi(w.y);
        } else {
          const float4 w = reinterpret_cast<const float4*>(s)[i];
          f[0] = w.x, f[1] = w.y, f[2] = w.z, f[3] = w.w;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) f[k] *= scale;
        if (dst_bf16)
          reinterpret_cast<uint2*>(d)[i] = make_uint2(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]));
        else
          reinterpret_cast<float4*>(d)[i] = make_float4(f[0], f[1], f[2], f[3]);
      }
      for (int64_t i = nv * 4 + threadIdx.x; i < n; i += COPY_THREADS)
        store_from_f(d, i, load_as_f(s, i, src_bf16) * scale, dst_bf16);
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
