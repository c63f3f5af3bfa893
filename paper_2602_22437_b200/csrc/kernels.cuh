// Device kernels of the collective step (launchers; definitions in kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace rsdb {

// One 8-bit Adam quantization block: element offsets into the state
// arrays (master / m codes / v codes share indexing), the fp32 gradient array
// and the parameter array, plus the block's slot in the absmax arrays.  A
// block is `len` elements laid out as rows of `cols` elements, `pitch`
// elements apart (contiguous block: cols == pitch == len; 2-D tile, N2:
// cols = tile width, pitch = row length of the tensor).
struct AdamBlock {
  int64_t state_off;
  int64_t grad_off;
  int64_t param_off;
  int32_t len;
  int32_t slot;
  int32_t cols;
  int32_t pitch;
};
// 40 B: every thread of a CTA loads its block's entry on the critical path of
// the block; a 56-B entry (separate m / v code offsets) cost 3.5 % at N = 1
static_assert(sizeof(AdamBlock) == 40, "AdamBlock is 40 bytes");

struct AdamScalars {
  float w1, b2, w2, eps, c_wd, step_size, inv_bc2s;
};

struct AdamPtrs {
  float* master;
  int8_t* mq;
  uint8_t* vq;
  float* mabs;
  float* vabs;
  const float* grad;
  void* param;        // bf16 or f32
  int32_t param_bf16; // 1: bf16, 0: f32
};

// a6: dst[i] = fp32(src[i]) * scale, i in [0, n); positions inside the sorted
// padding intervals pad[2j] <= i < pad[2j+1] are written 0.  src may equal dst
// when src is f32.
cudaError_t launch_cast_scale(const void* src, int src_bf16, float* dst, int64_t n, float scale,
                              const int64_t* pad_dev, int32_t npad, cudaStream_t st);

// a8 over `nblocks` table entries; tiles != 0: the table holds 2-D tiles
// (N2), updated two per stage (adam8_pair_kernel).
cudaError_t launch_adam8(const AdamBlock* table_dev, int64_t nblocks, const AdamPtrs& p,
                         const AdamScalars& s, int32_t tiles, cudaStream_t st);

struct CopySeg {
  const void* src;
  void* dst;
  int64_t numel;
  int64_t chunk_begin;  // prefix sum of chunks (for the block -> segment map)
};
cudaError_t launch_copy_segments(const CopySeg* segs_dev, int64_t nseg, int64_t total_chunks,
                                 int src_bf16, int dst_bf16, float scale, cudaStream_t st);

int num_sms();
// true the first time `key` is seen on the current device (per-device setup)
bool once_per_device(const void* key);

// ---- fused collectives over NVLink peer memory (p2p.cu) ----
constexpr int P2P_MAX_RANKS = 8;
struct P2PPtrs {
  const void* p[P2P_MAX_RANKS];  // per-rank device pointers (own rank: local)
};
struct P2PSignals {
  uint64_t* local;                  // this rank's signal buffer
  uint64_t* peer[P2P_MAX_RANKS];    // every rank's signal buffer, mapped here
  uint64_t timeout_ns;              // barrier spin limit (then the error flag, no hang)
  int32_t grid_div;                 // host: ranks sharing this device (local mode), >= 1
  int32_t max_ctas;                 // host: CTA budget of this channel's kernels (0 = the whole device)
};
// persistent grid of a barrier kernel: every rank's kernel must be resident at
// once, so ranks sharing one device (rsdb_p2p_create_local) split its SMs
inline int64_t grid_share(int64_t grid, const P2PSignals& sg) {
  const int64_t d = sg.grid_div > 1 ? sg.grid_div : 1;
  int64_t g = grid / d > 0 ? grid / d : 1;
  if (sg.max_ctas > 0 && g > sg.max_ctas) g = sg.max_ctas;  // leave SMs to overlapping compute
  return g;
}
constexpr int P2P_ERR_WORD = 17;  // signal-buffer word: barrier timeout flag
cudaError_t launch_rs_p2p(const P2PPtrs& grads, float* out, int64_t S, int rank, int m, float scale,
                          const int64_t* pad, int npad, const P2PSignals& sg, uint64_t epoch,
                          cudaStream_t st);
// device-side barrier of all ranks on `st` (start + done phases)
cudaError_t launch_p2p_barrier(const P2PSignals& sg, int rank, int m, uint64_t epoch, cudaStream_t st);
cudaError_t launch_ag_p2p(const P2PPtrs& params, int64_t bytes_S, int rank, int m,
                          const P2PSignals& sg, uint64_t epoch, cudaStream_t st);
// K-slot ring: push this rank's persistent shard (bytes_S) into region `rank`
// of every rank's slot dsts.p[r] (mapped; dsts.p[rank] local)
cudaError_t launch_ag_shards(const P2PPtrs& dsts, const void* shard, int64_t bytes_S, int rank, int m,
                             const P2PSignals* sg, uint64_t epoch, cudaStream_t st);
// a6 + a7 + a8 fused: ReduceScatter of the bf16 gradients over NVLink and the
// 8-bit Adam update of the local shard in one kernel (sg may be null iff m == 1);
// push_params non-null: also a4 -- every updated bf16 parameter is stored into
// every peer's parameter array (AllGather fused into the step).
// Compact block table for the fused DBuffer step (flat blocks): 16 B per
// block -- the block's unit, its offset inside the unit's shard, length and
// absmax slot -- plus per-unit bases (kept in shared memory), so each CTA
// loads 16 B per block instead of the 40-B AdamBlock on the critical path.
struct AdamBlockC {
  uint32_t unit;
  uint32_t off;
  int32_t len;
  int32_t slot;
};
static_assert(sizeof(AdamBlockC) == 16, "AdamBlockC is 16 bytes");
struct UnitBase {
  int64_t state, grad, param;  // element offsets of the unit's shard in MASTER, GRAD_FULL, PARAM_FULL
};
constexpr int RSA_MAX_UNITS = 64;
cudaError_t launch_rs_adam_p2p(const AdamBlock* tbl, int64_t nblocks, const P2PPtrs& grads, int m,
                               float scale, const AdamPtrs& P, const AdamScalars& s,
                               const P2PSignals* sg, int rank, uint64_t epoch, cudaStream_t st,
                               const P2PPtrs* push_params = nullptr,
                               const AdamBlockC* ctbl = nullptr, const UnitBase* ubase = nullptr,
                               int n_units = 0);

// ---- N2: FP8 E4M3 block quantization fused with the AllGather (fp8.cu) ----
struct Fp8Tile {
  int64_t off;                     // first element, offset inside the rank's shard
  int32_t rows, cols, pitch, slot; // tile shape, row pitch (elements), global scale slot
};
static_assert(sizeof(Fp8Tile) == 24, "Fp8Tile is 24 bytes");
// codes.p[r] / scales.p[r]: rank r's gathered code buffer (already offset by
// this rank's rank*S) / scale array; r == rank is local.  sg may be null iff m == 1.
cudaError_t launch_fp8_quant_ag(const Fp8Tile* tiles, int64_t ntiles, const float* master,
                                const P2PPtrs& codes, const P2PPtrs& scales, int m, int rank,
                                const P2PSignals* sg, uint64_t epoch, cudaStream_t st);

// ---- N2: 8-bit Adam with the dynamic (tree) code map (adam_dyn.cu) ----
// m_q / v_q hold uint8 indices into the signed / unsigned maps of R25.
cudaError_t launch_adam8_dyn(const AdamBlock* tbl, int64_t nblocks, const AdamPtrs& p, const AdamScalars& s,
                             cudaStream_t st);
void dyn_maps(float m_map[256], float v_map[256]);  // host: the two maps (R25)
// host: the kernel's code tables (layout: rsdb_dynamic_code_tables); false if
// a bin would hold two steps of the decision rule
constexpr int DYN_TABLE_M_LEN = 2 * (28 << 6), DYN_TABLE_V_LEN = 28 << 7;
bool dyn_code_tables(uint32_t* m_tab, uint32_t* v_tab);

// ---- N3: distributed Muon (muon.cu) ----
struct MuonSeg {
  int64_t src_off;      // element offset in the source (peer's u shard / root's workspace)
  int64_t dst_off;      // element offset in the destination (root workspace / local master)
  int64_t n;            // elements
  int64_t chunk_begin;  // prefix sum of 8192-element chunks
  int32_t peer;         // rank owning the source
  float coef;           // apply: the shape scale sqrt(max(1, rows/cols)) (x lr in the kernel)
};
static_assert(sizeof(MuonSeg) == 40, "MuonSeg is 40 bytes");
cudaError_t launch_muon_momentum(const int64_t* segs, int64_t nseg, int64_t max_n, float* buf,
                                 const float* grad, float* u, float mu, cudaStream_t st);
cudaError_t launch_muon_gather(const MuonSeg* segs, int64_t nseg, int64_t nchunks, const P2PPtrs& u,
                               void* ws, int bf16, int m, int rank, const P2PSignals* sg, uint64_t epoch,
                               cudaStream_t st);
cudaError_t launch_muon_apply(const MuonSeg* segs, int64_t nseg, int64_t nchunks, const P2PPtrs& ws,
                              int bf16, float* master, void* param_bf16, double lr, int m, int rank,
                              const P2PSignals* sg, uint64_t epoch, cudaStream_t st);
cudaError_t launch_muon_normalize(void* x, int64_t n, int bf16, double* ss, double eps, cudaStream_t st);
// N3 tensor-core Newton-Schulz (ns_umma.cu, muon.cu)
cudaError_t launch_muon_scale_transpose(const void* x, int rows, int cols, double* ss, double eps, void* same,
                                        int64_t ld_same, void* trans, int64_t ld_trans, cudaStream_t st);
cudaError_t launch_muon_copy2d(const void* src, int64_t ld, int rows, int cols, void* dst, cudaStream_t st);
// C[M x N] = alpha * A[M x K] . B[N x K]^T (+ beta * D), bf16 in / out, fp32
// accumulation in TMEM; CT (optional) receives C^T.  sym: the caller
// guarantees C is symmetric (M == N, e.g. W W^T): only the tiles reaching the
// upper triangle are computed and the rest of C is their mirror image.  All K-major (row-major,
// contraction dim contiguous); ld* in elements, multiples of 8; 16-B aligned.
cudaError_t launch_umma_gemm(int M, int N, int K, const void* A, int64_t lda, const void* B, int64_t ldb,
                             float alpha, float beta, const void* D, int64_t ldd, void* C, int64_t ldc, void* CT,
                             int64_t ldct, cudaStream_t st, bool sym = false);

}  // namespace rsdb
