// Internal declarations shared by the C-ABI translation units (capi.cc: core
// -- layouts, comms, units, p2p collectives, DBuffer; capi_ext.cc: the
// SURVEY §8(f) / §7 extensions -- FP8 AllGather, distributed Muon, K-slot ring).
#pragma once
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <climits>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/rsdb.h"
#include "kernels.cuh"
#include "planner.hpp"

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
// thread-local last-error string (rsdb_last_error); fail() sets it and returns st
rsdb_status fail(rsdb_status st, const char* fmt, ...);
void clear_error();
#define OK_CLEAR() (clear_error(), RSDB_OK)
#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) return fail(RSDB_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)
#define NCCL_TRY(expr)                                                                        \
  do {                                                                                        \
    ncclResult_t r_ = (expr);                                                                 \
    if (r_ != ncclSuccess) return fail(RSDB_ENCCL, "%s: %s", #expr, ncclGetErrorString(r_)); \
  } while (0)

struct rsdb_layout {
  rsdb::Layout L;
};

struct rsdb_comm {
  ncclComm_t nc = nullptr;  // null for a local comm (rsdb_comm_create_local)
  int32_t world = 1, rank = 0, device = 0;
  bool local = false;       // one of `world` logical ranks sharing this device
};

// device allocation owned by the library (metadata tables only)
struct DevTable {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevTable() {
    if (p) cudaFree(p);
  }
  rsdb_status alloc(size_t nbytes) {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = nbytes;
    if (nbytes) CUDA_TRY(cudaMalloc(&p, nbytes));
    return RSDB_OK;
  }
  rsdb_status upload(const void* host, size_t nbytes) {
    if (p) {
      cudaFree(p);
      p = nullptr;
    }
    bytes = nbytes;
    if (!nbytes) return RSDB_OK;
    CUDA_TRY(cudaMalloc(&p, nbytes));
    CUDA_TRY(cudaMemcpy(p, host, nbytes, cudaMemcpyHostToDevice));
    return RSDB_OK;
  }
};

struct rsdb_unit {
  rsdb::Layout L;
  rsdb_comm* comm = nullptr;
  int32_t rank = 0;
  rsdb_unit_bufs bufs{};
  int64_t qblock = 0;
  int64_t nblocks = 0;
  int32_t has_tiles = 0;  // 2-D quantization tiles in the block table (N2)
  int64_t npad = 0;
  DevTable pad;     // int64 lo, hi pairs
  DevTable blocks;  // rsdb::AdamBlock, unit-relative (state = shard, grad/param = +rank*S)
  bool has_bound_state = false;  // unit of a DBuffer: optimizer state in its arenas
  rsdb_adam_state bound_state{};
  void* shard = nullptr;  // K-slot ring mode: persistent bf16/f32 parameter shard (S elements)
};

// where the optimizer writes the unit's parameter shard: param_full + rank*S,
// or the persistent shard (ring mode; the table's param offsets carry +rank*S)
inline void* param_target(const rsdb_unit* u) {
  if (!u->shard) return u->bufs.param_full;
  return static_cast<char*>(u->shard) - int64_t(u->rank) * u->L.S * u->L.elem_bytes;
}

// rsdb_dbuffer_step_host: two library-owned copy streams (H2D, D2H) and, per
// unit, the events ordering the pipeline across units and across steps
struct HostPipe {
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_start = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_k, ev_out;  // per unit
  std::vector<char> k_rec, out_rec;              // recorded at least once
  // per unit: block-range chunks [first block, count, shard lo, shard hi) so
  // a chunk's copy-out overlaps the next chunk's kernel, and one event each
  struct Chunk {
    int64_t first, count, lo, hi;
  };
  std::vector<std::vector<Chunk>> chunks;
  std::vector<std::vector<cudaEvent_t>> ev_chunk, ev_chunk_in;
  ~HostPipe() {
    for (auto& v : ev_chunk_in)
      for (cudaEvent_t e : v)
        if (e) cudaEventDestroy(e);
    for (auto& v : ev_chunk)
      for (cudaEvent_t e : v)
        if (e) cudaEventDestroy(e);
    for (auto* v : {&ev_in, &ev_k, &ev_out})
      for (cudaEvent_t e : *v)
        if (e) cudaEventDestroy(e);
    if (ev_start) cudaEventDestroy(ev_start);
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
  }
};

struct rsdb_dbuffer {
  std::unique_ptr<HostPipe> host;  // created by the first rsdb_dbuffer_step_host
  std::vector<std::unique_ptr<rsdb_unit>> units;
  void* base[RSDB_NKINDS]{};
  int64_t nblocks = 0;
  DevTable blocks;        // arena-relative table over all units (grad in GRAD_F32 elements)
  DevTable blocks_fused;  // the same with grad in GRAD_FULL (bf16) elements, for the fused RS+Adam
  DevTable blocks_compact;  // rsdb::AdamBlockC over the fused table (flat blocks only), or empty
  DevTable unit_bases;      // rsdb::UnitBase per unit for the compact table
  int32_t n_units = 0;
  int32_t has_tiles = 0;    // 2-D quantization tiles in the table (N2)
  int32_t m = 1, rank = 0;
  int32_t param_bf16 = 1;
  std::vector<int64_t> grad_bytes;  // per unit, for grouped zero
};

struct rsdb_p2p {
  rsdb_comm* comm = nullptr;
  int32_t n = 0;
  std::vector<char*> local;          // [n]
  std::vector<int64_t> size;         // [n]
  std::vector<std::vector<char*>> peer;  // [n][world], own rank = local
  std::vector<void*> opened;         // IPC mappings to close
  uint64_t epoch = 0;
  uint64_t timeout_ns = 60ull * 1000000000ull;  // barrier spin limit (rsdb_p2p_set_timeout)
  int32_t grid_div = 1;  // logical ranks sharing the device (local mode: world)
  int32_t channel = 0;   // signal words [32c, 32c+32) of every rank's signal buffer (rsdb_p2p_channel)
  int32_t max_ctas = 0;  // CTA budget of the kernels issued through this object (rsdb_p2p_set_max_ctas)
};
constexpr int P2P_CHANNEL_WORDS = 32;  // 256 B per channel, 16 channels in RSDB_P2P_SIGNAL_BYTES

struct rsdb_copy_plan {
  DevTable segs;
  int64_t nseg = 0, total_chunks = 0;
  int32_t src_bf16 = 1, dst_bf16 = 1;
  float scale = 1.f;
};

inline cudaStream_t S_(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline bool aligned16(const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; }

rsdb_status require_device();  // ECUDA (no CPU fallback) when there is no GPU

// shared by the capi*.cc translation units
std::vector<rsdb::QSpec> make_specs(const rsdb::Layout& L, int64_t qblock, const rsdb_qspec* specs);
rsdb_status tiles_of(const rsdb::Layout& L, int32_t rank, const std::vector<rsdb::QSpec>& specs,
                     std::vector<rsdb::QTile>* out);
rsdb_status p2p_find(const rsdb_p2p* p, const void* ptr, int64_t bytes, int32_t* idx, int64_t* off);
rsdb_status p2p_common(rsdb_unit* u, rsdb_p2p* p, rsdb::P2PSignals* sg);
void p2p_signals(const rsdb_p2p* p, int m, rsdb::P2PSignals* sg);  // fill from p's signal buffers
