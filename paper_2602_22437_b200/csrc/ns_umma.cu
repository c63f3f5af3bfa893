// N3: the Newton-Schulz GEMMs of distributed Muon (PAPER.md
// Algorithm 2 l.10; reading R22: Muon's quintic, bf16 operands,
// fp32 accumulation) as a hand-written sm_100a tensor-core kernel:
//
//   TMA (cp.async.bulk.tensor.2d, 128-B swizzle) -> shared memory, 4-stage
//   ring -> tcgen05.mma.cta_group::1.kind::f16 (128 x 256 x 16, issued by one
//   thread) accumulating in TMEM (two 256-column accumulators, so the
//   epilogue of tile i overlaps the MMAs of tile i+1) -> tcgen05.ld -> fused
//   epilogue in registers -> bf16 global stores.
//
// One warp-specialised persistent kernel, 192 threads per CTA, one CTA per
// SM: warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer, warps 2-5
// = epilogue (warp w reads TMEM lanes 32 (w % 4) .. + 31).  Both operands are
// K-major (row-major with the contraction dimension contiguous):
//
//   C[M x N] = alpha * sum_k A[m, k] * B[n, k]  (+ beta * D[m, n])
//
// The three GEMMs of one quintic iteration on W (k x L, k <= L) map onto it
// without any transposed operand because A = W W^T and B = bA + cA^2 are
// symmetric and the epilogue of the third GEMM writes W' in both layouts:
//   G1  A  = W W^T                 A-op W   (k x L), B-op W   (k x L)
//   G2  B  = c A A + b A           A-op A   (k x k), B-op A   (k x k), D = A
//   G3  W' = B W + a W, and W'^T   A-op B   (k x k), B-op W^T (L x k), D = W
// (the quintic's two linear combinations live in the G2 / G3 epilogues; the
// Frobenius normalisation is fused with the first transposition, muon.cu).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>

#include "adam_dev.cuh"
#include "kernels.cuh"

namespace rsdb {

constexpr int UG_BM = 128, UG_BN = 256, UG_BK = 64, UG_STAGES = 4;
constexpr int UG_THREADS = 192;
constexpr uint32_t UG_A_BYTES = UG_BM * UG_BK * 2;  // 16 KB
constexpr uint32_t UG_B_BYTES = UG_BN * UG_BK * 2;  // 32 KB
constexpr uint32_t UG_STAGE_BYTES = UG_A_BYTES + UG_B_BYTES;
constexpr int UG_TMEM_COLS = 512;                   // 2 accumulators x 256 fp32 columns
constexpr size_t UG_SMEM = size_t(UG_STAGES) * UG_STAGE_BYTES + 1024 /* align */ + 256 /* barriers */;

struct UmmaEpi {
  float alpha, beta;
  const __nv_bfloat16* D;  // beta * D[m, n] (row-major, ld = ldd) when beta != 0
  __nv_bfloat16* C;        // row-major M x N, ld = ldc
  __nv_bfloat16* CT;       // optional: C^T row-major N x M, ld = ldct
  int64_t ldd, ldc, ldct;
};

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// 32 lanes x 32 bits, 32 consecutive columns: thread t gets row (lane base + t)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// shared-memory matrix descriptor (tcgen05 "version 1"): K-major operand tile
// of rows x 64 bf16 written by TMA with the 128-B swizzle -- 8-row core groups
// of 1024 B (stride byte offset), layout type SWIZZLE_128B (2), 1024-B aligned
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// instruction descriptor, kind::f16: D f32, A/B bf16, both K-major, M = 128, N = 256
constexpr uint32_t UG_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(UG_BN >> 3) << 17) |
                              (uint32_t(UG_BM >> 4) << 24);

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// tile t -> (m0, n0).  Full: m-tiles fastest.  SYM (C symmetric, M == N):
// only tiles that reach the upper triangle (n0 + BN - 1 >= m0), column by
// column -- the rest of C is written by mirroring (epilogue)
template <bool SYM>
__device__ __forceinline__ void tile_coords(int t, int mt, int& m0, int& n0) {
  if constexpr (!SYM) {
    m0 = (t % mt) * UG_BM;
    n0 = (t / mt) * UG_BN;
  } else {
    int j = 0;
    for (;; ++j) {
      const int rows = min(mt, (j + 1) * (UG_BN / UG_BM));  // m-tiles of column j touching col >= row
      if (t < rows) break;
      t -= rows;
    }
    m0 = t * UG_BM;
    n0 = j * UG_BN;
  }
}
__host__ __device__ inline int sym_tiles(int mt, int nt) {
  int n = 0;
  for (int j = 0; j < nt; ++j) n += (mt < (j + 1) * (UG_BN / UG_BM)) ? mt : (j + 1) * (UG_BN / UG_BM);
  return n;
}

// mbarrier wait that traps after ~4 s instead of hanging the device if a
// phase never completes (a protocol bug surfaces as a launch error)
__device__ __forceinline__ void mbar_wait_guard(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  uint64_t t0 = 0;
  for (uint32_t it = 0;; ++it) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (done) return;
    if ((it & 1023) == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (it == 0)
        t0 = t;
      else if (t - t0 > 4000000000ull)
        __trap();
    }
  }
}

template <bool HAS_D, bool HAS_T, bool SYM>
__global__ void __launch_bounds__(UG_THREADS, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b, int M,
                     int N, int K, UmmaEpi ep) {
  extern __shared__ uint8_t ug_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ug_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + UG_STAGES * UG_STAGE_BYTES);
  uint64_t* empty = full + UG_STAGES;
  uint64_t* tfull = empty + UG_STAGES;  // [2]
  uint64_t* tempty = tfull + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = int(threadIdx.x) >> 5, lane = int(threadIdx.x) & 31;
  const int mt = (M + UG_BM - 1) / UG_BM, nt = (N + UG_BN - 1) / UG_BN;
  const int tiles = SYM ? sym_tiles(mt, nt) : mt * nt, kblocks = (K + UG_BK - 1) / UG_BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < UG_STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull + s, 1);
      mbar_init(tempty + s, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(UG_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int m0, n0;
        tile_coords<SYM>(t, mt, m0, n0);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait_guard(empty + s, ph ^ 1);
          uint8_t* sa = smem + s * UG_STAGE_BYTES;
          mbar_arrive_expect_tx(full + s, UG_STAGE_BYTES);
          tma_load_2d(sa, &tma_a, full + s, kb * UG_BK, m0);
          tma_load_2d(sa + UG_A_BYTES, &tma_b, full + s, kb * UG_BK, n0);
          if (++s == UG_STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer (one thread)
      int s = 0, as = 0;
      uint32_t ph = 0, aph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        mbar_wait_guard(tempty + as, aph ^ 1);  // the epilogue drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(as * UG_BN);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait_guard(full + s, ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * UG_STAGE_BYTES);
          const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + UG_A_BYTES);
#pragma unroll
          for (int k = 0; k < UG_BK / 16; ++k)  // +32 B along K inside the 128-B swizzle atom
            tc_mma(d, da + uint64_t(2 * k), db + uint64_t(2 * k), UG_IDESC, (kb | k) != 0);
          tc_commit(empty + s);  // frees the stage when these MMAs have read it
          if (++s == UG_STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit(tfull + as);  // accumulator complete
        if (++as == 2) {
          as = 0;
          aph ^= 1;
        }
      }
    }
  } else {  // ---------------- epilogue: warps 2..5
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int as = 0;
    uint32_t aph = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      int m0, n0;
      tile_coords<SYM>(t, mt, m0, n0);
      mbar_wait_guard(tfull + as, aph);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      const uint32_t tbase = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(as * UG_BN);
#pragma unroll 1
      for (int c = 0; c < UG_BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + uint32_t(c), r);
        const int col0 = n0 + c;
        if (col0 >= N) break;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = ep.alpha * __uint_as_float(r[j]);
        const bool full_cols = col0 + 32 <= N;
        if (row < M) {
          if constexpr (HAS_D) {
            const __nv_bfloat16* dp = ep.D + int64_t(row) * ep.ldd + col0;
            if (full_cols) {
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                const uint4 w = *reinterpret_cast<const uint4*>(dp + j);
                const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  v[j + 2 * h] = fmaf(ep.beta, __uint_as_float(ww[h] << 16), v[j + 2 * h]);
                  v[j + 2 * h + 1] = fmaf(ep.beta, __uint_as_float(ww[h] & 0xffff0000u), v[j + 2 * h + 1]);
                }
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (col0 + j < N) v[j] = fmaf(ep.beta, __bfloat162float(dp[j]), v[j]);
            }
          }
          __nv_bfloat16* cp = ep.C + int64_t(row) * ep.ldc + col0;
          if (SYM && col0 < row + 1) {  // the part left of the diagonal comes from the mirror writes
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j >= row && col0 + j < N) cp[j] = __float2bfloat16_rn(v[j]);
          } else if (full_cols) {
#pragma unroll
            for (int j = 0; j < 32; j += 8)
              *reinterpret_cast<uint4*>(cp + j) = make_uint4(pack2(v[j], v[j + 1]), pack2(v[j + 2], v[j + 3]),
                                                             pack2(v[j + 4], v[j + 5]), pack2(v[j + 6], v[j + 7]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j < N) cp[j] = __float2bfloat16_rn(v[j]);
          }
        }
        if constexpr (HAS_T || SYM) {  // C^T[col][row]: the 32 lanes write 32 consecutive rows (64 B)
          if (row < M) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j < N && (!SYM || col0 + j > row))
                ep.CT[int64_t(col0 + j) * ep.ldct + row] = __float2bfloat16_rn(v[j]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + as);  // one arrival per epilogue warp
      if (++as == 2) {
        as = 0;
        aph ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(UG_TMEM_COLS));
  }
}

// ------------------------------------------------------------------ host
typedef CUresult (*EncodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static cudaError_t encode_kmajor(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld,
                                 int box_rows) {
  static EncodeTiled_t fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    const cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    if (e != cudaSuccess) return e;
    if (!f || q != cudaDriverEntryPointSuccess) return cudaErrorNotSupported;
    fn = reinterpret_cast<EncodeTiled_t>(f);
  }
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(ld) * 2};
  const cuuint32_t box[2] = {cuuint32_t(UG_BK), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_umma_gemm(int M, int N, int K, const void* A, int64_t lda, const void* B, int64_t ldb,
                             float alpha, float beta, const void* D, int64_t ldd, void* C, int64_t ldc, void* CT,
                             int64_t ldct, cudaStream_t st, bool sym) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (sym && (M != N || CT)) return cudaErrorInvalidValue;
  if (K <= 0 || (lda * 2) % 16 || (ldb * 2) % 16 || (reinterpret_cast<uintptr_t>(A) % 16) ||
      (reinterpret_cast<uintptr_t>(B) % 16))
    return cudaErrorInvalidValue;
  if (beta != 0.f && (!D || (ldd % 8) || reinterpret_cast<uintptr_t>(D) % 16)) return cudaErrorInvalidValue;
  if ((ldc % 8) || reinterpret_cast<uintptr_t>(C) % 16) return cudaErrorInvalidValue;
  CUtensorMap ma, mb;
  if (cudaError_t e = encode_kmajor(&ma, A, M, K, lda, UG_BM)) return e;
  if (cudaError_t e = encode_kmajor(&mb, B, N, K, ldb, UG_BN)) return e;
  UmmaEpi ep{alpha, beta, static_cast<const __nv_bfloat16*>(D), static_cast<__nv_bfloat16*>(C),
             static_cast<__nv_bfloat16*>(CT), ldd, ldc, ldct};
  static const char attr_key = 0;
  if (once_per_device(&attr_key)) {
    for (auto k : {umma_gemm_kernel<false, false, false>, umma_gemm_kernel<true, false, false>,
                   umma_gemm_kernel<false, true, false>, umma_gemm_kernel<true, true, false>,
                   umma_gemm_kernel<false, false, true>, umma_gemm_kernel<true, false, true>})
      if (cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(UG_SMEM)))
        return e;
  }
  const int mt = (M + UG_BM - 1) / UG_BM, nt = (N + UG_BN - 1) / UG_BN;
  const int tiles = sym ? sym_tiles(mt, nt) : mt * nt;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  const bool hd = beta != 0.f, ht = CT != nullptr;
  if (sym) {
    ep.CT = ep.C;
    ep.ldct = ep.ldc;
    if (hd)
      umma_gemm_kernel<true, false, true><<<grid, UG_THREADS, UG_SMEM, st>>>(ma, mb, M, N, K, ep);
    else
      umma_gemm_kernel<false, false, true><<<grid, UG_THREADS, UG_SMEM, st>>>(ma, mb, M, N, K, ep);
  } else if (hd && ht)
    umma_gemm_kernel<true, true, false><<<grid, UG_THREADS, UG_SMEM, st>>>(ma, mb, M, N, K, ep);
  else if (hd)
    umma_gemm_kernel<true, false, false><<<grid, UG_THREADS, UG_SMEM, st>>>(ma, mb, M, N, K, ep);
  else if (ht)
    umma_gemm_kernel<false, true, false><<<grid, UG_THREADS, UG_SMEM, st>>>(ma, mb, M, N, K, ep);
  else
    umma_gemm_kernel<false, false, false><<<grid, UG_THREADS, UG_SMEM, st>>>(ma, mb, M, N, K, ep);
  return cudaGetLastError();
}

}  // namespace rsdb
