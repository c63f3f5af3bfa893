// extern "C" boundary of the RaggedShard/DBuffer collective step (include/rsdb.h):
// errors, layouts, comms, units, the NCCL and NVLink-peer collectives, the
// fused RS + Adam kernels and the DBuffer.  Extensions: capi_ext.cc.
#include "capi_internal.hpp"

#include <cstdarg>

static thread_local std::string g_err;

rsdb_status fail(rsdb_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}
void clear_error() { g_err.clear(); }

rsdb_status require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n < 1)
    return fail(RSDB_ECUDA, "no CUDA device available (%s); there is no CPU fallback",
                e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
  return RSDB_OK;
}


extern "C" {

const char* rsdb_last_error(void) { return g_err.c_str(); }
int32_t rsdb_abi_version(void) { return 1; }

// ---------------------------------------------------------------------------
// a1 / a2 / a3
// ---------------------------------------------------------------------------
rsdb_status rsdb_block_elems(int32_t ndim, const int64_t* shape, int32_t kind, int64_t param,
                             int64_t* g_out) {
  std::string err;
  if (!rsdb::block_elems(ndim, shape, kind, param, g_out, &err)) return fail(RSDB_EINVAL, "%s", err.c_str());
  return OK_CLEAR();
}

rsdb_status rsdb_plan(int32_t n, const int64_t* numel, const int64_t* block, int32_t world,
                      int32_t elem_bytes, int32_t gcoll_bytes, rsdb_layout** out) {
  if (!out || n < 0 || (n > 0 && (!numel || !block))) return fail(RSDB_EINVAL, "rsdb_plan: bad pointer or n");
  std::vector<int64_t> e(numel, numel + n), g(block, block + n);
  auto lay = std::make_unique<rsdb_layout>();
  std::string err;
  if (!rsdb::plan(e, g, world, elem_bytes, gcoll_bytes, &lay->L, &err))
    return fail(err.find("internal") != std::string::npos ? RSDB_EINTERNAL : RSDB_EINVAL, "%s",
                err.c_str());
  *out = lay.release();
  return OK_CLEAR();
}

rsdb_status rsdb_plan_ordered(int32_t n, const int64_t* numel, const int64_t* block, int32_t world,
                              int32_t elem_bytes, int32_t gcoll_bytes, int32_t ordering,
                              const int64_t* shape_keys, rsdb_layout** out) {
  if (!out || n < 0 || (n > 0 && (!numel || !block))) return fail(RSDB_EINVAL, "rsdb_plan_ordered: bad pointer or n");
  if (ordering == 2 && n > 0 && !shape_keys) return fail(RSDB_EINVAL, "shape ordering needs keys");
  std::vector<int64_t> e(numel, numel + n), g(block, block + n), k;
  if (shape_keys) k.assign(shape_keys, shape_keys + n);
  auto lay = std::make_unique<rsdb_layout>();
  std::string err;
  if (!rsdb::plan_ordered(e, g, world, elem_bytes, gcoll_bytes, ordering, shape_keys ? &k : nullptr,
                          &lay->L, &err))
    return fail(err.find("internal") != std::string::npos ? RSDB_EINTERNAL : RSDB_EINVAL, "%s",
                err.c_str());
  *out = lay.release();
  return OK_CLEAR();
}

rsdb_status rsdb_layout_from_starts(int32_t n, const int64_t* numel, const int64_t* block,
                                    int32_t world, int32_t elem_bytes, int32_t gcoll_bytes,
                                    int64_t S, const int64_t* starts, int32_t require_gcoll,
                                    rsdb_layout** out) {
  if (!out || n < 0 || (n > 0 && (!numel || !block || !starts)) || world < 1 || S < 0 ||
      !(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4) || gcoll_bytes < 1)
    return fail(RSDB_EINVAL, "rsdb_layout_from_starts: bad argument");
  auto lay = std::make_unique<rsdb_layout>();
  rsdb::Layout& L = lay->L;
  L.m = world;
  L.elem_bytes = elem_bytes;
  L.g_coll = std::max<int64_t>(1, gcoll_bytes / elem_bytes);
  L.S = S;
  L.e.assign(numel, numel + n);
  L.g.assign(block, block + n);
  L.l.assign(starts, starts + n);
  for (int i = 0; i < n; ++i)
    if (L.e[i] < 1 || L.g[i] < 1) return fail(RSDB_EINVAL, "numel/block must be >= 1");
  if (n > 0 && S < 1) return fail(RSDB_EINVAL, "S must be >= 1");
  const int64_t v = rsdb::count_violations(L, require_gcoll != 0);
  if (v) return fail(RSDB_EINVAL, "layout violates %lld constraint(s) of P:226-229", (long long)v);
  *out = lay.release();
  return OK_CLEAR();
}

int64_t rsdb_layout_shard_numel(const rsdb_layout* l) { return l ? l->L.S : -1; }
int64_t rsdb_layout_padding(const rsdb_layout* l) {
  return l ? int64_t(l->L.m) * l->L.S - l->L.E() : -1;
}
int64_t rsdb_layout_total_numel(const rsdb_layout* l) { return l ? l->L.E() : -1; }
int32_t rsdb_layout_world(const rsdb_layout* l) { return l ? l->L.m : -1; }
int32_t rsdb_layout_ntensors(const rsdb_layout* l) { return l ? int32_t(l->L.e.size()) : -1; }
int32_t rsdb_layout_elem_bytes(const rsdb_layout* l) { return l ? l->L.elem_bytes : -1; }

rsdb_status rsdb_layout_starts(const rsdb_layout* l, int64_t* out) {
  if (!l || (!out && !l->L.l.empty())) return fail(RSDB_EINVAL, "null argument");
  std::copy(l->L.l.begin(), l->L.l.end(), out);
  return OK_CLEAR();
}

rsdb_status rsdb_layout_validate(const rsdb_layout* l, int64_t* nv) {
  if (!l || !nv) return fail(RSDB_EINVAL, "null argument");
  *nv = rsdb::count_violations(l->L, true);
  return OK_CLEAR();
}

rsdb_status rsdb_layout_padding_intervals(const rsdb_layout* l, int64_t* n, int64_t* lo, int64_t* hi) {
  if (!l || !n) return fail(RSDB_EINVAL, "null argument");
  auto iv = rsdb::padding_intervals(l->L);
  if (lo && hi) {
    if (*n < int64_t(iv.size())) return fail(RSDB_EINVAL, "array too small");
    for (size_t i = 0; i < iv.size(); ++i) lo[i] = iv[i].first, hi[i] = iv[i].second;
  }
  *n = int64_t(iv.size());
  return OK_CLEAR();
}

rsdb_status rsdb_layout_rank_segments(const rsdb_layout* l, int32_t rank, int64_t* n,
                                      int32_t* tensor, int64_t* local_off, int64_t* len,
                                      int64_t* tensor_off) {
  if (!l || !n) return fail(RSDB_EINVAL, "null argument");
  if (rank < 0 || rank >= l->L.m) return fail(RSDB_EINVAL, "rank %d out of [0,%d)", rank, l->L.m);
  auto segs = rsdb::rank_segments(l->L, rank);
  if (tensor && local_off && len && tensor_off) {
    if (*n < int64_t(segs.size())) return fail(RSDB_EINVAL, "array too small");
    for (size_t i = 0; i < segs.size(); ++i) {
      tensor[i] = segs[i].tensor;
      local_off[i] = segs[i].local_off;
      len[i] = segs[i].len;
      tensor_off[i] = segs[i].tensor_off;
    }
  }
  *n = int64_t(segs.size());
  return OK_CLEAR();
}

rsdb_status rsdb_layout_rank_blocks(const rsdb_layout* l, int32_t rank, int64_t qblock, int64_t* n,
                                    int64_t* off, int32_t* len) {
  if (!l || !n) return fail(RSDB_EINVAL, "null argument");
  if (rank < 0 || rank >= l->L.m) return fail(RSDB_EINVAL, "rank %d out of [0,%d)", rank, l->L.m);
  std::vector<rsdb::QBlock> b;
  std::string err;
  if (!rsdb::rank_blocks(l->L, rank, qblock, &b, &err))
    return fail(qblock < 1 ? RSDB_EINVAL : RSDB_EMISMATCH, "%s", err.c_str());
  if (off && len) {
    if (*n < int64_t(b.size())) return fail(RSDB_EINVAL, "array too small");
    for (size_t i = 0; i < b.size(); ++i) off[i] = b[i].off, len[i] = b[i].len;
  }
  *n = int64_t(b.size());
  return OK_CLEAR();
}

rsdb_status rsdb_layout_to_json(const rsdb_layout* l, char* buf, int64_t cap, int64_t* needed) {
  if (!l || !needed) return fail(RSDB_EINVAL, "null argument");
  const std::string s = rsdb::to_json(l->L);
  *needed = int64_t(s.size()) + 1;
  if (buf && cap >= *needed) std::memcpy(buf, s.c_str(), s.size() + 1);
  return OK_CLEAR();
}

void rsdb_layout_free(rsdb_layout* l) { delete l; }

// ---------------------------------------------------------------------------
// communicator
// ---------------------------------------------------------------------------
static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");

rsdb_status rsdb_unique_id(uint8_t out[128]) {
  if (!out) return fail(RSDB_EINVAL, "null argument");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(out, &id, 128);
  return OK_CLEAR();
}

rsdb_status rsdb_comm_init(const uint8_t id[128], int32_t world, int32_t rank, int32_t device,
                           rsdb_comm** out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world || device < 0)
    return fail(RSDB_EINVAL, "rsdb_comm_init: bad argument");
  if (rsdb_status st = require_device()) return st;
  CUDA_TRY(cudaSetDevice(device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  auto c = std::make_unique<rsdb_comm>();
  c->world = world;
  c->rank = rank;
  c->device = device;
  NCCL_TRY(ncclCommInitRank(&c->nc, world, uid, rank));
  *out = c.release();
  return OK_CLEAR();
}

int32_t rsdb_comm_rank(const rsdb_comm* c) { return c ? c->rank : -1; }
int32_t rsdb_comm_world(const rsdb_comm* c) { return c ? c->world : -1; }
void rsdb_comm_free(rsdb_comm* c) {
  if (!c) return;
  if (c->nc) ncclCommDestroy(c->nc);
  delete c;
}

rsdb_status rsdb_comm_create_local(int32_t world, int32_t rank, rsdb_comm** out) {
  if (!out || world < 1 || world > rsdb::P2P_MAX_RANKS || rank < 0 || rank >= world)
    return fail(RSDB_EINVAL, "rsdb_comm_create_local: need 1 <= world <= %d and 0 <= rank < world",
                rsdb::P2P_MAX_RANKS);
  if (rsdb_status st = require_device()) return st;
  auto c = std::make_unique<rsdb_comm>();
  c->world = world;
  c->rank = rank;
  CUDA_TRY(cudaGetDevice(&c->device));
  c->local = true;
  *out = c.release();
  return OK_CLEAR();
}

// ---------------------------------------------------------------------------
// unit
// ---------------------------------------------------------------------------
// per-tensor quantization specs: explicit (rsdb_qspec*, N2 tiles) or flat qblock
extern "C++" std::vector<rsdb::QSpec> make_specs(const rsdb::Layout& L, int64_t qblock,
                                           const rsdb_qspec* specs) {
  std::vector<rsdb::QSpec> v(L.e.size());
  for (size_t t = 0; t < v.size(); ++t) {
    if (specs)
      v[t] = {specs[t].row_len, specs[t].tile_rows, specs[t].tile_cols};
    else
      v[t] = {0, 0, int32_t(std::min<int64_t>(qblock, INT32_MAX))};
  }
  return v;
}

extern "C++" rsdb_status tiles_of(const rsdb::Layout& L, int32_t rank, const std::vector<rsdb::QSpec>& specs,
                            std::vector<rsdb::QTile>* out) {
  std::string err;
  if (!rsdb::rank_tiles(L, rank, specs, out, &err))
    return fail(err.find("straddles") != std::string::npos ? RSDB_EMISMATCH : RSDB_EINVAL, "%s",
                err.c_str());
  for (auto& t : *out)
    if (int64_t(t.rows) * t.cols > (int64_t{1} << 30) || t.pitch > INT32_MAX)
      return fail(RSDB_EINVAL, "quantization block too large");
  return RSDB_OK;
}

static rsdb_status build_unit(const rsdb::Layout& L, rsdb_comm* comm, int32_t rank,
                              const rsdb_unit_bufs& bufs, const std::vector<rsdb::QSpec>& specs,
                              rsdb_unit* u, std::vector<rsdb::QTile>* blocks_out) {
  if (!(L.elem_bytes == 2 || L.elem_bytes == 4))
    return fail(RSDB_EMISMATCH, "units support bf16 (2 B) or f32 (4 B) elements, got %d B", L.elem_bytes);
  if (rank < 0 || rank >= L.m) return fail(RSDB_EINVAL, "rank %d out of [0,%d)", rank, L.m);
  if (comm && (comm->world != L.m || comm->rank != rank))
    return fail(RSDB_EMISMATCH, "comm (world %d, rank %d) does not match layout world %d / rank %d",
                comm->world, comm->rank, L.m, rank);
  if (!bufs.param_full || !bufs.grad_full || !bufs.grad_f32)
    return fail(RSDB_EINVAL, "unit buffers must be non-null");
  if (!aligned16(bufs.param_full) || !aligned16(bufs.grad_full) || !aligned16(bufs.grad_f32))
    return fail(RSDB_EMISMATCH, "unit buffers must be 16-byte aligned (P:199, P:369)");
  if (L.elem_bytes == 2 && bufs.grad_full == bufs.grad_f32)
    return fail(RSDB_EMISMATCH, "bf16 unit: grad_full must not alias grad_f32");
  std::vector<rsdb::QTile> qb;
  const bool no_blocks = std::all_of(specs.begin(), specs.end(), [](const rsdb::QSpec& q) {
    return q.row_len == 0 && q.tile_rows == 0 && q.tile_cols == 0;
  });  // qblock = 0: collectives-only unit
  if (!no_blocks)
    if (rsdb_status st = tiles_of(L, rank, specs, &qb)) return st;
  u->L = L;
  u->comm = comm;
  u->rank = rank;
  u->bufs = bufs;
  u->nblocks = int64_t(qb.size());
  u->has_tiles = std::any_of(qb.begin(), qb.end(), [](const rsdb::QTile& t) { return t.rows > 1; });
  auto iv = rsdb::padding_intervals(L);
  std::vector<int64_t> pad;
  for (auto& [a, b] : iv) pad.push_back(a), pad.push_back(b);
  u->npad = int64_t(iv.size());
  if (rsdb_status st = require_device()) return st;
  if (rsdb_status st = u->pad.upload(pad.data(), pad.size() * sizeof(int64_t))) return st;
  std::vector<rsdb::AdamBlock> tbl(qb.size());
  const int64_t base = int64_t(rank) * L.S;
  for (size_t i = 0; i < qb.size(); ++i)
    tbl[i] = {qb[i].off, base + qb[i].off, base + qb[i].off, qb[i].rows * qb[i].cols, int32_t(i),
              qb[i].cols, int32_t(qb[i].pitch)};
  if (rsdb_status st = u->blocks.upload(tbl.data(), tbl.size() * sizeof(rsdb::AdamBlock))) return st;
  if (blocks_out) *blocks_out = std::move(qb);
  return RSDB_OK;
}

rsdb_status rsdb_unit_create(const rsdb_layout* l, rsdb_comm* comm, int32_t rank,
                             const rsdb_unit_bufs* bufs, int64_t qblock, rsdb_unit** out) {
  if (!l || !bufs || !out) return fail(RSDB_EINVAL, "null argument");
  if (qblock < 0) return fail(RSDB_EINVAL, "qblock must be >= 0 (0: no optimizer blocks)");
  auto u = std::make_unique<rsdb_unit>();
  if (rsdb_status st = build_unit(l->L, comm, rank, *bufs, make_specs(l->L, qblock, nullptr), u.get(),
                                  nullptr))
    return st;
  *out = u.release();
  return OK_CLEAR();
}

rsdb_status rsdb_unit_create_q(const rsdb_layout* l, rsdb_comm* comm, int32_t rank,
                               const rsdb_unit_bufs* bufs, const rsdb_qspec* specs, rsdb_unit** out) {
  if (!l || !bufs || !out || (!specs && !l->L.e.empty())) return fail(RSDB_EINVAL, "null argument");
  auto u = std::make_unique<rsdb_unit>();
  if (rsdb_status st = build_unit(l->L, comm, rank, *bufs, make_specs(l->L, 0, specs), u.get(), nullptr))
    return st;
  *out = u.release();
  return OK_CLEAR();
}

rsdb_status rsdb_layout_rank_tiles(const rsdb_layout* l, int32_t rank, const rsdb_qspec* specs,
                                   int64_t* n, int64_t* off, int32_t* rows, int32_t* cols,
                                   int64_t* pitch) {
  if (!l || !n || (!specs && !l->L.e.empty())) return fail(RSDB_EINVAL, "null argument");
  if (rank < 0 || rank >= l->L.m) return fail(RSDB_EINVAL, "rank %d out of [0,%d)", rank, l->L.m);
  std::vector<rsdb::QTile> t;
  if (rsdb_status st = tiles_of(l->L, rank, make_specs(l->L, 0, specs), &t)) return st;
  if (off && rows && cols && pitch) {
    if (*n < int64_t(t.size())) return fail(RSDB_EINVAL, "array too small");
    for (size_t i = 0; i < t.size(); ++i)
      off[i] = t[i].off, rows[i] = t[i].rows, cols[i] = t[i].cols, pitch[i] = t[i].pitch;
  }
  *n = int64_t(t.size());
  return OK_CLEAR();
}

int64_t rsdb_unit_num_blocks(const rsdb_unit* u) { return u ? u->nblocks : -1; }
void rsdb_unit_free(rsdb_unit* u) { delete u; }

rsdb_status rsdb_all_gather(rsdb_unit* u, void* stream) {
  if (!u) return fail(RSDB_EINVAL, "null unit");
  if (!u->comm) return fail(RSDB_EINVAL, "unit has no communicator");
  if (!u->comm->nc) return fail(RSDB_EINVAL, "a local comm has no NCCL communicator (use the p2p calls)");
  if (u->L.S == 0) return OK_CLEAR();
  const ncclDataType_t dt = u->L.elem_bytes == 2 ? ncclBfloat16 : ncclFloat32;
  char* full = static_cast<char*>(u->bufs.param_full);
  const void* send = full + int64_t(u->rank) * u->L.S * u->L.elem_bytes;  // in place
  NCCL_TRY(ncclAllGather(send, full, size_t(u->L.S), dt, u->comm->nc, S_(stream)));
  return OK_CLEAR();
}

static rsdb_status cast_scale(rsdb_unit* u, void* stream) {
  const int64_t n = int64_t(u->L.m) * u->L.S;
  const float scale = float(1.0 / double(u->L.m));
  CUDA_TRY(rsdb::launch_cast_scale(u->bufs.grad_full, u->L.elem_bytes == 2,
                                   static_cast<float*>(u->bufs.grad_f32), n, scale,
                                   static_cast<const int64_t*>(u->pad.p), int32_t(u->npad),
                                   S_(stream)));
  return RSDB_OK;
}

rsdb_status rsdb_unit_cast_scale(rsdb_unit* u, void* stream) {
  if (!u) return fail(RSDB_EINVAL, "null unit");
  if (rsdb_status st = cast_scale(u, stream)) return st;
  return OK_CLEAR();
}

static rsdb_status rs_f32(rsdb_unit* u, void* stream) {
  float* g = static_cast<float*>(u->bufs.grad_f32);
  NCCL_TRY(ncclReduceScatter(g, g + int64_t(u->rank) * u->L.S, size_t(u->L.S), ncclFloat32,
                             ncclSum, u->comm->nc, S_(stream)));
  return RSDB_OK;
}

rsdb_status rsdb_reduce_scatter(rsdb_unit* u, void* stream) {
  if (!u) return fail(RSDB_EINVAL, "null unit");
  if (!u->comm) return fail(RSDB_EINVAL, "unit has no communicator");
  if (!u->comm->nc) return fail(RSDB_EINVAL, "a local comm has no NCCL communicator (use the p2p calls)");
  if (u->L.S == 0) return OK_CLEAR();
  if (rsdb_status st = cast_scale(u, stream)) return st;
  if (rsdb_status st = rs_f32(u, stream)) return st;
  return OK_CLEAR();
}

rsdb_status rsdb_unit_reduce_scatter_f32(rsdb_unit* u, void* stream) {
  if (!u) return fail(RSDB_EINVAL, "null unit");
  if (!u->comm) return fail(RSDB_EINVAL, "unit has no communicator");
  if (!u->comm->nc) return fail(RSDB_EINVAL, "a local comm has no NCCL communicator (use the p2p calls)");
  if (u->L.S == 0) return OK_CLEAR();
  if (rsdb_status st = rs_f32(u, stream)) return st;
  return OK_CLEAR();
}

static rsdb_status adam_scalars(const rsdb_adam_cfg* c, int64_t step, rsdb::AdamScalars* s) {
  if (!c) return fail(RSDB_EINVAL, "null cfg");
  if (step < 1) return fail(RSDB_EINVAL, "step must be >= 1");
  if (!(c->beta1 >= 0 && c->beta1 < 1 && c->beta2 >= 0 && c->beta2 < 1 && c->eps >= 0 && c->lr >= 0))
    return fail(RSDB_EINVAL, "invalid Adam hyper-parameters");
  const double lr = c->lr, b1 = c->beta1, b2 = c->beta2;
  s->w1 = float(1.0 - b1);
  s->b2 = float(b2);
  s->w2 = float(1.0 - b2);
  s->eps = float(c->eps);
  s->c_wd = float(1.0 - lr * double(c->weight_decay));
  s->step_size = float(lr / (1.0 - std::pow(b1, double(step))));
  s->inv_bc2s = float(1.0 / std::sqrt(1.0 - std::pow(b2, double(step))));
  return RSDB_OK;
}

rsdb_status rsdb_step_8bit_adam(rsdb_unit* u, const rsdb_adam_state* st, const rsdb_adam_cfg* cfg,
                                int64_t step, void* stream) {
  if (!u || !st) return fail(RSDB_EINVAL, "null argument");
  rsdb::AdamScalars s;
  if (rsdb_status e = adam_scalars(cfg, step, &s)) return e;
  if (u->nblocks == 0) return OK_CLEAR();
  if (!st->master_f32 || !st->m_q || !st->v_q || !st->m_absmax || !st->v_absmax)
    return fail(RSDB_EINVAL, "null state pointer");
  rsdb::AdamPtrs p{static_cast<float*>(st->master_f32), static_cast<int8_t*>(st->m_q),
                   static_cast<uint8_t*>(st->v_q),       static_cast<float*>(st->m_absmax),
                   static_cast<float*>(st->v_absmax),    static_cast<const float*>(u->bufs.grad_f32),
                   param_target(u),                      u->L.elem_bytes == 2};
  CUDA_TRY(rsdb::launch_adam8(static_cast<const rsdb::AdamBlock*>(u->blocks.p), u->nblocks, p, s,
                              u->has_tiles, S_(stream)));
  return OK_CLEAR();
}

rsdb_status rsdb_step_8bit_adam_dynamic(rsdb_unit* u, const rsdb_adam_state* st, const rsdb_adam_cfg* cfg,
                                        int64_t step, void* stream) {
  if (!u || !st) return fail(RSDB_EINVAL, "null argument");
  rsdb::AdamScalars s;
  if (rsdb_status e = adam_scalars(cfg, step, &s)) return e;
  if (u->nblocks == 0) return OK_CLEAR();
  if (!st->master_f32 || !st->m_q || !st->v_q || !st->m_absmax || !st->v_absmax)
    return fail(RSDB_EINVAL, "null state pointer");
  rsdb::AdamPtrs p{static_cast<float*>(st->master_f32), static_cast<int8_t*>(st->m_q),
                   static_cast<uint8_t*>(st->v_q),       static_cast<float*>(st->m_absmax),
                   static_cast<float*>(st->v_absmax),    static_cast<const float*>(u->bufs.grad_f32),
                   param_target(u),                      u->L.elem_bytes == 2};
  CUDA_TRY(rsdb::launch_adam8_dyn(static_cast<const rsdb::AdamBlock*>(u->blocks.p), u->nblocks, p, s,
                                  S_(stream)));
  return OK_CLEAR();
}

rsdb_status rsdb_dynamic_code_maps(float* m_map, float* v_map) {
  if (!m_map || !v_map) return fail(RSDB_EINVAL, "null argument");
  rsdb::dyn_maps(m_map, v_map);
  return OK_CLEAR();
}

rsdb_status rsdb_dynamic_code_tables(uint32_t* m_table, uint32_t* v_table) {
  static_assert(rsdb::DYN_TABLE_M_LEN == RSDB_DYN_TABLE_M_LEN && rsdb::DYN_TABLE_V_LEN == RSDB_DYN_TABLE_V_LEN,
                "table lengths");
  if (!m_table || !v_table) return fail(RSDB_EINVAL, "null argument");
  if (!rsdb::dyn_code_tables(m_table, v_table)) return fail(RSDB_EINVAL, "a table bin holds two steps");
  return OK_CLEAR();
}

// ---------------------------------------------------------------------------
// fused collectives over NVLink peer memory (N1)
// ---------------------------------------------------------------------------
typedef int (*cuMemGetAddressRange_t)(unsigned long long* base, size_t* size, unsigned long long ptr);

static rsdb_status alloc_base(const void* p, char** base, int64_t* size) {
  static cuMemGetAddressRange_t fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) return fail(RSDB_ECUDA, "cuMemGetAddressRange unavailable");
    fn = reinterpret_cast<cuMemGetAddressRange_t>(f);
  }
  unsigned long long b = 0;
  size_t s = 0;
  if (fn(&b, &s, reinterpret_cast<unsigned long long>(p)) != 0)
    return fail(RSDB_EINVAL, "pointer %p is not a device allocation", p);
  *base = reinterpret_cast<char*>(b);
  *size = int64_t(s);
  return RSDB_OK;
}

rsdb_status rsdb_ipc_handle(const void* dev_ptr, uint8_t out[RSDB_IPC_BYTES]) {
  if (!dev_ptr || !out) return fail(RSDB_EINVAL, "null argument");
  if (rsdb_status st = require_device()) return st;
  char* base = nullptr;
  int64_t sz = 0;
  if (rsdb_status st = alloc_base(dev_ptr, &base, &sz)) return st;
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, base));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle is 64 bytes");
  const int64_t off = static_cast<const char*>(dev_ptr) - base;
  std::memcpy(out, &h, 64);
  std::memcpy(out + 64, &off, 8);
  return OK_CLEAR();
}

rsdb_status rsdb_p2p_create(rsdb_comm* comm, int32_t n_bufs, void* const* local_bufs,
                            const int64_t* sizes, const uint8_t* all_handles, rsdb_p2p** out) {
  if (!comm || n_bufs < 1 || !local_bufs || !sizes || !all_handles || !out)
    return fail(RSDB_EINVAL, "rsdb_p2p_create: null argument or n_bufs < 1");
  if (comm->world > rsdb::P2P_MAX_RANKS)
    return fail(RSDB_EINVAL, "p2p collectives support world <= %d", rsdb::P2P_MAX_RANKS);
  if (sizes[0] < RSDB_P2P_SIGNAL_BYTES) return fail(RSDB_EINVAL, "signal buffer too small");
  auto p = std::make_unique<rsdb_p2p>();
  p->comm = comm;
  p->n = n_bufs;
  p->peer.assign(size_t(n_bufs), std::vector<char*>(size_t(comm->world), nullptr));
  for (int32_t i = 0; i < n_bufs; ++i) {
    if (!local_bufs[i] || sizes[i] < 0) return fail(RSDB_EINVAL, "buffer %d invalid", i);
    p->local.push_back(static_cast<char*>(local_bufs[i]));
    p->size.push_back(sizes[i]);
  }
  CUDA_TRY(cudaSetDevice(comm->device));
  auto cleanup = [&]() {
    for (void* q : p->opened) cudaIpcCloseMemHandle(q);
    p->opened.clear();
  };
  for (int32_t r = 0; r < comm->world; ++r) {
    // buffers of one rank may share an allocation (same handle): open it once
    std::vector<std::pair<std::string, void*>> seen;
    for (int32_t i = 0; i < n_bufs; ++i) {
      if (r == comm->rank) {
        p->peer[size_t(i)][size_t(r)] = p->local[size_t(i)];
        continue;
      }
      const uint8_t* h = all_handles + (int64_t(r) * n_bufs + i) * RSDB_IPC_BYTES;
      cudaIpcMemHandle_t mh;
      int64_t off;
      std::memcpy(&mh, h, 64);
      std::memcpy(&off, h + 64, 8);
      const std::string key(reinterpret_cast<const char*>(h), 64);
      void* base = nullptr;
      for (auto& kv : seen)
        if (kv.first == key) base = kv.second;
      if (!base) {
        cudaError_t e = cudaIpcOpenMemHandle(&base, mh, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
          cleanup();
          return fail(RSDB_ECUDA, "cudaIpcOpenMemHandle(rank %d, buffer %d): %s", r, i,
                      cudaGetErrorString(e));
        }
        p->opened.push_back(base);
        seen.emplace_back(key, base);
      }
      p->peer[size_t(i)][size_t(r)] = static_cast<char*>(base) + off;
    }
  }
  *out = p.release();
  return OK_CLEAR();
}

void rsdb_p2p_free(rsdb_p2p* p) {
  if (!p) return;
  for (void* q : p->opened) cudaIpcCloseMemHandle(q);
  delete p;
}

rsdb_status rsdb_p2p_channel(const rsdb_p2p* p, int32_t channel, rsdb_p2p** out) {
  if (!p || !out) return fail(RSDB_EINVAL, "null argument");
  if (channel < 1 || channel >= RSDB_P2P_SIGNAL_BYTES / (P2P_CHANNEL_WORDS * 8))
    return fail(RSDB_EINVAL, "channel must be in [1, %d)", RSDB_P2P_SIGNAL_BYTES / (P2P_CHANNEL_WORDS * 8));
  if (p->channel != 0) return fail(RSDB_EINVAL, "create channels from the base p2p object");
  auto c = std::make_unique<rsdb_p2p>();
  c->comm = p->comm;
  c->n = p->n;
  c->local = p->local;
  c->size = p->size;
  c->peer = p->peer;  // borrowed mappings (c->opened stays empty: p owns them)
  c->timeout_ns = p->timeout_ns;
  c->grid_div = p->grid_div;
  c->channel = channel;
  *out = c.release();
  return OK_CLEAR();
}

rsdb_status rsdb_p2p_create_local(rsdb_comm* comm, int32_t n_bufs, void* const* all_bufs,
                                  const int64_t* sizes, rsdb_p2p** out) {
  if (!comm || n_bufs < 1 || !all_bufs || !sizes || !out)
    return fail(RSDB_EINVAL, "rsdb_p2p_create_local: null argument or n_bufs < 1");
  if (!comm->local) return fail(RSDB_EMISMATCH, "rsdb_p2p_create_local needs a local comm");
  if (sizes[0] < RSDB_P2P_SIGNAL_BYTES) return fail(RSDB_EINVAL, "signal buffer too small");
  auto p = std::make_unique<rsdb_p2p>();
  p->comm = comm;
  p->n = n_bufs;
  p->peer.assign(size_t(n_bufs), std::vector<char*>(size_t(comm->world), nullptr));
  for (int32_t i = 0; i < n_bufs; ++i) {
    if (sizes[i] < 0) return fail(RSDB_EINVAL, "buffer %d size invalid", i);
    for (int32_t r = 0; r < comm->world; ++r) {
      char* b = static_cast<char*>(all_bufs[int64_t(r) * n_bufs + i]);
      if (!b) return fail(RSDB_EINVAL, "buffer %d of rank %d is null", i, r);
      p->peer[size_t(i)][size_t(r)] = b;
    }
    p->local.push_back(p->peer[size_t(i)][size_t(comm->rank)]);
    p->size.push_back(sizes[i]);
  }
  // logical ranks may live on several devices of this process (one process
  // driving N GPUs, e.g. to profile one rank's kernel while its peers run):
  // the grid is shared only among the ranks on this rank's device, and the
  // other devices' memory is made accessible (peer access over NVLink)
  int32_t same = 0;
  for (int32_t r = 0; r < comm->world; ++r) {
    cudaPointerAttributes at{};
    CUDA_TRY(cudaPointerGetAttributes(&at, all_bufs[int64_t(r) * n_bufs]));
    if (at.device == comm->device) {
      ++same;
    } else {
      int ok = 0;
      CUDA_TRY(cudaDeviceCanAccessPeer(&ok, comm->device, at.device));
      if (!ok) return fail(RSDB_ECUDA, "device %d cannot access device %d (no P2P path)", comm->device, at.device);
      int cur = 0;
      CUDA_TRY(cudaGetDevice(&cur));
      CUDA_TRY(cudaSetDevice(comm->device));
      const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();  // clear
      cudaSetDevice(cur);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(RSDB_ECUDA, "cudaDeviceEnablePeerAccess(%d -> %d): %s", comm->device, at.device,
                    cudaGetErrorString(e));
    }
  }
  p->grid_div = same < 1 ? 1 : same;
  *out = p.release();
  return OK_CLEAR();
}

rsdb_status rsdb_p2p_set_max_ctas(rsdb_p2p* p, int32_t max_ctas) {
  if (!p || max_ctas < 0) return fail(RSDB_EINVAL, "null p2p or max_ctas < 0");
  p->max_ctas = max_ctas;
  return OK_CLEAR();
}

rsdb_status rsdb_p2p_set_timeout(rsdb_p2p* p, double seconds) {
  if (!p || !(seconds > 0)) return fail(RSDB_EINVAL, "rsdb_p2p_set_timeout: null p2p or seconds <= 0");
  p->timeout_ns = seconds >= 1.8e10 ? UINT64_MAX : uint64_t(seconds * 1e9);
  return OK_CLEAR();
}

rsdb_status rsdb_p2p_check(rsdb_p2p* p, int64_t* flags) {
  if (!p || !flags) return fail(RSDB_EINVAL, "null argument");
  uint64_t* w = reinterpret_cast<uint64_t*>(p->local[0]) + int64_t(p->channel) * P2P_CHANNEL_WORDS +
                rsdb::P2P_ERR_WORD;
  uint64_t v = 0;
  CUDA_TRY(cudaMemcpy(&v, w, sizeof v, cudaMemcpyDeviceToHost));  // synchronises the device
  *flags = int64_t(v);
  if (v) {
    const uint64_t zero = 0;
    CUDA_TRY(cudaMemcpy(w, &zero, sizeof zero, cudaMemcpyHostToDevice));
    return fail(RSDB_ECUDA, "a p2p barrier timed out (flags 0x%llx): a peer never reached the call; "
                "results of the timed-out calls are invalid", (unsigned long long)v);
  }
  return OK_CLEAR();
}

// locate `ptr` (with `bytes` behind it) inside a registered buffer i (>= 1)
extern "C++" rsdb_status p2p_find(const rsdb_p2p* p, const void* ptr, int64_t bytes, int32_t* idx,
                            int64_t* off) {
  const char* c = static_cast<const char*>(ptr);
  for (int32_t i = 1; i < p->n; ++i) {
    const char* b = p->local[size_t(i)];
    if (c >= b && c + bytes <= b + p->size[size_t(i)]) {
      *idx = i;
      *off = c - b;
      return RSDB_OK;
    }
  }
  return fail(RSDB_EMISMATCH, "unit buffer is not inside a registered p2p buffer");
}

extern "C++" void p2p_signals(const rsdb_p2p* p, int m, rsdb::P2PSignals* sg) {
  const int64_t w = int64_t(p->channel) * P2P_CHANNEL_WORDS;
  sg->local = reinterpret_cast<uint64_t*>(p->local[0]) + w;
  for (int r = 0; r < rsdb::P2P_MAX_RANKS; ++r)
    sg->peer[r] = r < m ? reinterpret_cast<uint64_t*>(p->peer[0][size_t(r)]) + w : nullptr;
  sg->timeout_ns = p->timeout_ns;
  sg->grid_div = p->grid_div;
  sg->max_ctas = p->max_ctas;
}

extern "C++" rsdb_status p2p_common(rsdb_unit* u, rsdb_p2p* p, rsdb::P2PSignals* sg) {
  if (!u || !p) return fail(RSDB_EINVAL, "null argument");
  if (!u->comm || u->comm != p->comm) return fail(RSDB_EMISMATCH, "unit and p2p use different comms");
  const int m = u->L.m;
  if ((u->L.S * u->L.elem_bytes) % 16 != 0)
    return fail(RSDB_EMISMATCH, "p2p collectives need 16-byte aligned shards (S*elem %% 16 == 0; "
                                "planner layouts always are, P:199)");
  p2p_signals(p, m, sg);
  return RSDB_OK;
}

rsdb_status rsdb_reduce_scatter_p2p(rsdb_unit* u, rsdb_p2p* p, void* stream) {
  rsdb::P2PSignals sg;
  if (!u) return fail(RSDB_EINVAL, "null unit");
  if (u->L.m > 1 || p)
    if (rsdb_status st = p2p_common(u, p, &sg)) return st;
  if (u->L.elem_bytes != 2) return fail(RSDB_EMISMATCH, "p2p ReduceScatter needs a bf16 unit");
  if (u->L.S == 0) return OK_CLEAR();
  const int m = u->L.m;
  if (m == 1) {  // no peers: the reduction is the group op alone (a6)
    if (rsdb_status st = cast_scale(u, stream)) return st;
    return OK_CLEAR();
  }
  int32_t bi = 0;
  int64_t off = 0;
  if (rsdb_status st = p2p_find(p, u->bufs.grad_full, int64_t(m) * u->L.S * 2, &bi, &off)) return st;
  rsdb::P2PPtrs g{};
  for (int r = 0; r < m; ++r) g.p[r] = p->peer[size_t(bi)][size_t(r)] + off;
  const float scale = float(1.0 / double(m));
  ++p->epoch;
  float* out = static_cast<float*>(u->bufs.grad_f32) + int64_t(u->rank) * u->L.S;
  CUDA_TRY(rsdb::launch_rs_p2p(g, out, u->L.S, u->rank, m, scale, static_cast<const int64_t*>(u->pad.p),
                               int32_t(u->npad), sg, p->epoch, S_(stream)));
  return OK_CLEAR();
}

rsdb_status rsdb_p2p_barrier(rsdb_p2p* p, void* stream) {
  if (!p) return fail(RSDB_EINVAL, "null p2p");
  const int m = p->comm->world;
  if (m == 1) return OK_CLEAR();
  rsdb::P2PSignals sg;
  p2p_signals(p, m, &sg);
  ++p->epoch;
  CUDA_TRY(rsdb::launch_p2p_barrier(sg, p->comm->rank, m, p->epoch, S_(stream)));
  return OK_CLEAR();
}

rsdb_status rsdb_all_gather_p2p(rsdb_unit* u, rsdb_p2p* p, void* stream) {
  rsdb::P2PSignals sg;
  if (!u) return fail(RSDB_EINVAL, "null unit");
  if (u->L.m > 1 || p)
    if (rsdb_status st = p2p_common(u, p, &sg)) return st;
  if (u->L.S == 0 || u->L.m == 1) return OK_CLEAR();  // world 1: AllGather is the identity
  const int m = u->L.m;
  const int64_t bytes_S = u->L.S * u->L.elem_bytes;
  int32_t bi = 0;
  int64_t off = 0;
  if (rsdb_status st = p2p_find(p, u->bufs.param_full, int64_t(m) * bytes_S, &bi, &off)) return st;
  rsdb::P2PPtrs q{};
  for (int r = 0; r < m; ++r) q.p[r] = p->peer[size_t(bi)][size_t(r)] + off;
  ++p->epoch;
  CUDA_TRY(rsdb::launch_ag_p2p(q, bytes_S, u->rank, m, sg, p->epoch, S_(stream)));
  return OK_CLEAR();
}

static rsdb_status rs_adam_unit(rsdb_unit* u, rsdb_p2p* p, const rsdb_adam_state* st,
                                const rsdb_adam_cfg* cfg, int64_t step, void* stream, bool gather,
                                int64_t first_block = 0, int64_t block_count = -1) {
  if (!u) return fail(RSDB_EINVAL, "null unit");
  if (u->L.elem_bytes != 2) return fail(RSDB_EMISMATCH, "fused ReduceScatter + Adam needs a bf16 unit");
  rsdb::AdamScalars s;
  if (rsdb_status e = adam_scalars(cfg, step, &s)) return e;
  if (!st) {
    if (!u->has_bound_state) return fail(RSDB_EINVAL, "null state and the unit is not part of a DBuffer");
    st = &u->bound_state;
  }
  if (!st->master_f32 || !st->m_q || !st->v_q || (u->nblocks > 0 && (!st->m_absmax || !st->v_absmax)))
    return fail(RSDB_EINVAL, "null state pointer");
  const int m = u->L.m;
  if (gather && u->shard)
    return fail(RSDB_EINVAL, "ring mode (persistent shard): gather with rsdb_all_gather_shards_p2p instead");
  if (u->L.S == 0 || (u->nblocks == 0 && m == 1)) return OK_CLEAR();  // world > 1: barriers count every rank
  rsdb::P2PPtrs g{}, q{};
  rsdb::P2PSignals sg{};
  const bool push = gather && m > 1;
  if (m > 1) {
    if (!p) return fail(RSDB_EINVAL, "world > 1 needs a p2p object");
    if (rsdb_status e = p2p_common(u, p, &sg)) return e;
    int32_t bi = 0;
    int64_t off = 0;
    if (rsdb_status e = p2p_find(p, u->bufs.grad_full, int64_t(m) * u->L.S * 2, &bi, &off)) return e;
    for (int r = 0; r < m; ++r) g.p[r] = p->peer[size_t(bi)][size_t(r)] + off;
    if (push) {
      if (rsdb_status e = p2p_find(p, u->bufs.param_full, int64_t(m) * u->L.S * 2, &bi, &off)) return e;
      for (int r = 0; r < m; ++r) q.p[r] = p->peer[size_t(bi)][size_t(r)] + off;
    }
    ++p->epoch;
  } else {
    g.p[0] = u->bufs.grad_full;
  }
  rsdb::AdamPtrs ap{static_cast<float*>(st->master_f32), static_cast<int8_t*>(st->m_q),
                    static_cast<uint8_t*>(st->v_q),       static_cast<float*>(st->m_absmax),
                    static_cast<float*>(st->v_absmax),    nullptr,
                    param_target(u),                      1};
  const float scale = float(1.0 / double(m));
  const int64_t nb = block_count < 0 ? u->nblocks : block_count;  // a block range (rsdb_dbuffer_step_host)
  if (nb == 0 && m == 1) return OK_CLEAR();
  CUDA_TRY(rsdb::launch_rs_adam_p2p(static_cast<const rsdb::AdamBlock*>(u->blocks.p) + first_block, nb, g, m,
                                    scale, ap, s, m > 1 ? &sg : nullptr, u->rank,
                                    m > 1 ? p->epoch : 0, S_(stream), push ? &q : nullptr));
  return OK_CLEAR();
}

rsdb_status rsdb_reduce_scatter_adam_p2p(rsdb_unit* u, rsdb_p2p* p, const rsdb_adam_state* st,
                                         const rsdb_adam_cfg* cfg, int64_t step, void* stream) {
  return rs_adam_unit(u, p, st, cfg, step, stream, false);
}

rsdb_status rsdb_reduce_scatter_adam_gather_p2p(rsdb_unit* u, rsdb_p2p* p, const rsdb_adam_state* st,
                                                const rsdb_adam_cfg* cfg, int64_t step, void* stream) {
  return rs_adam_unit(u, p, st, cfg, step, stream, true);
}

// ---------------------------------------------------------------------------
// DBuffer batched arenas
// ---------------------------------------------------------------------------
static int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

static rsdb_status kind_sizes(const rsdb::Layout& L, int32_t rank, const std::vector<rsdb::QSpec>& specs,
                              int64_t sz[RSDB_NKINDS]) {
  std::vector<rsdb::QTile> qb;
  if (rsdb_status st = tiles_of(L, rank, specs, &qb)) return st;
  const int64_t full = int64_t(L.m) * L.S;
  sz[RSDB_KIND_PARAM_FULL] = full * L.elem_bytes;
  sz[RSDB_KIND_GRAD_FULL] = L.elem_bytes == 4 ? 0 : full * L.elem_bytes;
  sz[RSDB_KIND_GRAD_F32] = full * 4;
  sz[RSDB_KIND_MASTER] = L.S * 4;
  sz[RSDB_KIND_MQ] = L.S;
  sz[RSDB_KIND_VQ] = L.S;
  sz[RSDB_KIND_MABS] = int64_t(qb.size()) * 4;
  sz[RSDB_KIND_VABS] = int64_t(qb.size()) * 4;
  return RSDB_OK;
}

// per-unit spec vectors: explicit (specs[u] = rsdb_qspec[n_u]) or flat qblock
static rsdb_status unit_specs(const rsdb_layout* const* units, int32_t n_units, int64_t qblock,
                              const rsdb_qspec* const* specs,
                              std::vector<std::vector<rsdb::QSpec>>* out) {
  out->clear();
  for (int32_t u = 0; u < n_units; ++u) {
    if (!units[u]) return fail(RSDB_EINVAL, "null layout %d", u);
    if (specs && !specs[u] && !units[u]->L.e.empty()) return fail(RSDB_EINVAL, "null specs for unit %d", u);
    out->push_back(make_specs(units[u]->L, qblock, specs ? specs[u] : nullptr));
  }
  return RSDB_OK;
}

// MASTER, MQ and VQ share ELEMENT offsets (one "state" index space): the
// common element offset is aligned so that every kind's byte offset is a
// multiple of align_bytes.  Likewise MABS/VABS share a block index space.
static rsdb_status arena_layout(const rsdb_layout* const* units, int32_t n_units, int32_t rank,
                                const std::vector<std::vector<rsdb::QSpec>>& specs, int64_t align,
                                int64_t* bytes, int64_t* offs, std::vector<int64_t>* state_elem_off,
                                std::vector<int64_t>* blk_idx_off) {
  if (!units || n_units < 0 || !bytes || align < 16 || (align & (align - 1)))
    return fail(RSDB_EINVAL, "rsdb_arena_sizes: bad argument (align must be a power of two >= 16)");
  int64_t acc[RSDB_NKINDS] = {0};
  int64_t state_e = 0, blk_e = 0;
  for (int32_t u = 0; u < n_units; ++u) {
    if (!units[u]) return fail(RSDB_EINVAL, "null layout %d", u);
    const rsdb::Layout& L = units[u]->L;
    if (rank < 0 || rank >= L.m) return fail(RSDB_EINVAL, "rank out of range for unit %d", u);
    if (L.m != units[0]->L.m)
      return fail(RSDB_EMISMATCH, "unit %d is planned for world %d, unit 0 for %d (one DBuffer = one FSDP group)",
                  u, L.m, units[0]->L.m);
    int64_t sz[RSDB_NKINDS] = {0};
    if (rsdb_status st = kind_sizes(L, rank, specs[size_t(u)], sz)) return st;
    for (int k : {RSDB_KIND_PARAM_FULL, RSDB_KIND_GRAD_FULL, RSDB_KIND_GRAD_F32}) {
      acc[k] = round_up(acc[k], align);
      if (offs) offs[int64_t(u) * RSDB_NKINDS + k] = acc[k];
      acc[k] += sz[k];
    }
    state_e = round_up(state_e, align);  // align elements => align bytes for 1- and 4-byte kinds
    blk_e = round_up(blk_e, align);
    if (state_elem_off) state_elem_off->push_back(state_e);
    if (blk_idx_off) blk_idx_off->push_back(blk_e);
    if (offs) {
      offs[int64_t(u) * RSDB_NKINDS + RSDB_KIND_MASTER] = state_e * 4;
      offs[int64_t(u) * RSDB_NKINDS + RSDB_KIND_MQ] = state_e;
      offs[int64_t(u) * RSDB_NKINDS + RSDB_KIND_VQ] = state_e;
      offs[int64_t(u) * RSDB_NKINDS + RSDB_KIND_MABS] = blk_e * 4;
      offs[int64_t(u) * RSDB_NKINDS + RSDB_KIND_VABS] = blk_e * 4;
    }
    state_e += L.S;
    blk_e += sz[RSDB_KIND_MABS] / 4;
  }
  for (int k : {RSDB_KIND_PARAM_FULL, RSDB_KIND_GRAD_FULL, RSDB_KIND_GRAD_F32}) bytes[k] = round_up(acc[k], align);
  state_e = round_up(state_e, align);
  blk_e = round_up(blk_e, align);
  bytes[RSDB_KIND_MASTER] = state_e * 4;
  bytes[RSDB_KIND_MQ] = state_e;
  bytes[RSDB_KIND_VQ] = state_e;
  bytes[RSDB_KIND_MABS] = blk_e * 4;
  bytes[RSDB_KIND_VABS] = blk_e * 4;
  return RSDB_OK;
}

static rsdb_status arena_sizes_impl(const rsdb_layout* const* units, int32_t n_units, int32_t rank,
                                    int64_t qblock, const rsdb_qspec* const* specs, int64_t align_bytes,
                                    int64_t* bytes_per_kind, int64_t* unit_offsets) {
  if (!units || n_units < 0) return fail(RSDB_EINVAL, "null argument");
  std::vector<std::vector<rsdb::QSpec>> sp;
  if (rsdb_status st = unit_specs(units, n_units, qblock, specs, &sp)) return st;
  if (rsdb_status st = arena_layout(units, n_units, rank, sp, align_bytes, bytes_per_kind,
                                    unit_offsets, nullptr, nullptr))
    return st;
  return OK_CLEAR();
}

rsdb_status rsdb_arena_sizes(const rsdb_layout* const* units, int32_t n_units, int32_t rank,
                             int64_t qblock, int64_t align_bytes, int64_t* bytes_per_kind,
                             int64_t* unit_offsets) {
  return arena_sizes_impl(units, n_units, rank, qblock, nullptr, align_bytes, bytes_per_kind,
                          unit_offsets);
}

rsdb_status rsdb_arena_sizes_q(const rsdb_layout* const* units, int32_t n_units, int32_t rank,
                               const rsdb_qspec* const* specs, int64_t align_bytes,
                               int64_t* bytes_per_kind, int64_t* unit_offsets) {
  if (!specs) return fail(RSDB_EINVAL, "null specs");
  return arena_sizes_impl(units, n_units, rank, 0, specs, align_bytes, bytes_per_kind, unit_offsets);
}

static rsdb_status dbuffer_create_impl(const rsdb_layout* const* units, int32_t n_units,
                                       rsdb_comm* comm, int32_t rank, int64_t qblock,
                                       const rsdb_qspec* const* specs, int64_t align_bytes,
                                       void* const* arena_base, rsdb_dbuffer** out) {
  if (!units || !arena_base || !out || n_units < 0) return fail(RSDB_EINVAL, "null argument");
  std::vector<std::vector<rsdb::QSpec>> sp;
  if (rsdb_status st = unit_specs(units, n_units, qblock, specs, &sp)) return st;
  int64_t bytes[RSDB_NKINDS];
  std::vector<int64_t> offs(size_t(n_units) * RSDB_NKINDS), st_off, bk_off;
  if (rsdb_status st = arena_layout(units, n_units, rank, sp, align_bytes, bytes, offs.data(), &st_off,
                                    &bk_off))
    return st;
  auto db = std::make_unique<rsdb_dbuffer>();
  for (int k = 0; k < RSDB_NKINDS; ++k) {
    db->base[k] = arena_base[k];
    if (bytes[k] > 0 && !arena_base[k]) return fail(RSDB_EINVAL, "arena %d is null", k);
    if (bytes[k] > 0 && reinterpret_cast<uintptr_t>(arena_base[k]) % align_bytes)
      return fail(RSDB_EMISMATCH, "arena %d not aligned to %lld bytes", k, (long long)align_bytes);
  }
  int32_t pbf = -1;
  std::vector<rsdb::AdamBlock> tbl, tbl_fused;
  std::vector<rsdb::AdamBlockC> tbl_c;
  std::vector<rsdb::UnitBase> ubases;
  bool compact_ok = n_units <= rsdb::RSA_MAX_UNITS;
  for (int32_t u = 0; u < n_units; ++u) {
    const rsdb::Layout& L = units[u]->L;
    const int32_t bf = L.elem_bytes == 2;
    if (pbf >= 0 && bf != pbf)
      return fail(RSDB_EMISMATCH, "one dbuffer holds one parameter dtype (unit %d differs)", u);
    pbf = bf;
    auto at = [&](int k) { return static_cast<char*>(arena_base[k]) + offs[size_t(u) * RSDB_NKINDS + k]; };
    rsdb_unit_bufs b;
    b.param_full = at(RSDB_KIND_PARAM_FULL);
    b.grad_f32 = at(RSDB_KIND_GRAD_F32);
    b.grad_full = bf ? at(RSDB_KIND_GRAD_FULL) : b.grad_f32;
    auto unit = std::make_unique<rsdb_unit>();
    std::vector<rsdb::QTile> qb;
    if (rsdb_status st = build_unit(L, comm, rank, b, sp[size_t(u)], unit.get(), &qb)) return st;
    unit->has_bound_state = true;
    unit->bound_state = {at(RSDB_KIND_MASTER), at(RSDB_KIND_MQ), at(RSDB_KIND_VQ), at(RSDB_KIND_MABS),
                         at(RSDB_KIND_VABS)};
    // arena-relative combined table: state in MASTER/MQ/VQ elements, grad in
    // GRAD_F32 elements, param in PARAM_FULL elements.
    const int64_t gbase = offs[size_t(u) * RSDB_NKINDS + RSDB_KIND_GRAD_F32] / 4 + int64_t(rank) * L.S;
    const int64_t pbase = offs[size_t(u) * RSDB_NKINDS + RSDB_KIND_PARAM_FULL] / L.elem_bytes +
                          int64_t(rank) * L.S;
    if (bk_off[u] + int64_t(qb.size()) > INT32_MAX) return fail(RSDB_EINVAL, "too many blocks");
    const int64_t gbase16 = bf ? offs[size_t(u) * RSDB_NKINDS + RSDB_KIND_GRAD_FULL] / 2 +
                                     int64_t(rank) * L.S
                               : 0;
    ubases.push_back({st_off[u], gbase16, pbase});
    for (size_t i = 0; i < qb.size(); ++i) {
      tbl.push_back({st_off[u] + qb[i].off, gbase + qb[i].off, pbase + qb[i].off,
                     qb[i].rows * qb[i].cols, int32_t(bk_off[u] + int64_t(i)), qb[i].cols,
                     int32_t(qb[i].pitch)});
      tbl_fused.push_back(tbl.back());
      tbl_fused.back().grad_off = gbase16 + qb[i].off;
      const int64_t len = int64_t(qb[i].rows) * qb[i].cols;
      compact_ok = compact_ok && qb[i].rows == 1 && qb[i].off <= INT32_MAX;
      if (compact_ok)
        tbl_c.push_back({uint32_t(u), uint32_t(qb[i].off), int32_t(len), int32_t(bk_off[u] + int64_t(i))});
    }
    db->m = L.m;
    db->rank = rank;
    db->has_tiles |= unit->has_tiles;
    db->grad_bytes.push_back(int64_t(L.m) * L.S * L.elem_bytes);
    db->units.push_back(std::move(unit));
  }
  db->param_bf16 = pbf < 0 ? 1 : pbf;
  db->nblocks = int64_t(tbl.size());
  if (rsdb_status st = db->blocks.upload(tbl.data(), tbl.size() * sizeof(rsdb::AdamBlock))) return st;
  if (db->param_bf16) {
    if (rsdb_status st = db->blocks_fused.upload(tbl_fused.data(),
                                                 tbl_fused.size() * sizeof(rsdb::AdamBlock)))
      return st;
    if (compact_ok && !tbl_c.empty()) {
      if (rsdb_status st = db->blocks_compact.upload(tbl_c.data(), tbl_c.size() * sizeof(rsdb::AdamBlockC)))
        return st;
      if (rsdb_status st = db->unit_bases.upload(ubases.data(), ubases.size() * sizeof(rsdb::UnitBase)))
        return st;
      db->n_units = n_units;
    }
  }
  *out = db.release();
  return OK_CLEAR();
}

static rsdb_status rs_adam_dbuffer(rsdb_dbuffer* d, rsdb_p2p* p, const rsdb_adam_cfg* cfg, int64_t step,
                                   void* stream, bool gather) {
  if (!d) return fail(RSDB_EINVAL, "null dbuffer");
  // the compact 16-B block table (+4 % at N = 1 over the 40-B one)
  const bool use_compact = d->blocks_compact.p != nullptr;
  if (!d->param_bf16) return fail(RSDB_EMISMATCH, "fused ReduceScatter + Adam needs bf16 units");
  rsdb::AdamScalars s;
  if (rsdb_status e = adam_scalars(cfg, step, &s)) return e;
  const int m = d->m;
  // a rank may own no block (e.g. whole-matrix granularity at large m) but at
  // world > 1 it still launches: the kernel's barriers count every rank
  if (d->nblocks == 0 && m == 1) return OK_CLEAR();
  rsdb::P2PPtrs g{}, q{};
  rsdb::P2PSignals sg{};
  const bool push = gather && m > 1;
  if (m > 1) {
    if (!p) return fail(RSDB_EINVAL, "world > 1 needs a p2p object");
    if (!d->units.empty())
      if (rsdb_status e = p2p_common(d->units[0].get(), p, &sg)) return e;
    int32_t bi = 0;
    int64_t off = 0;
    if (rsdb_status e = p2p_find(p, d->base[RSDB_KIND_GRAD_FULL], 1, &bi, &off)) return e;
    if (off != 0) return fail(RSDB_EMISMATCH, "p2p must map the GRAD_FULL arena from its base");
    for (int r = 0; r < m; ++r) g.p[r] = p->peer[size_t(bi)][size_t(r)];
    if (push) {
      if (rsdb_status e = p2p_find(p, d->base[RSDB_KIND_PARAM_FULL], 1, &bi, &off)) return e;
      if (off != 0) return fail(RSDB_EMISMATCH, "p2p must map the PARAM_FULL arena from its base");
      for (int r = 0; r < m; ++r) q.p[r] = p->peer[size_t(bi)][size_t(r)];
    }
    ++p->epoch;
  } else {
    g.p[0] = d->base[RSDB_KIND_GRAD_FULL];
  }
  rsdb::AdamPtrs ap{static_cast<float*>(d->base[RSDB_KIND_MASTER]),
                    static_cast<int8_t*>(d->base[RSDB_KIND_MQ]),
                    static_cast<uint8_t*>(d->base[RSDB_KIND_VQ]),
                    static_cast<float*>(d->base[RSDB_KIND_MABS]),
                    static_cast<float*>(d->base[RSDB_KIND_VABS]),
                    nullptr,
                    d->base[RSDB_KIND_PARAM_FULL],
                    1};
  CUDA_TRY(rsdb::launch_rs_adam_p2p(static_cast<const rsdb::AdamBlock*>(d->blocks_fused.p), d->nblocks, g,
                                    m, float(1.0 / double(m)), ap, s, m > 1 ? &sg : nullptr, d->rank,
                                    m > 1 ? p->epoch : 0, S_(stream), push ? &q : nullptr,
                                    use_compact ? static_cast<const rsdb::AdamBlockC*>(d->blocks_compact.p) : nullptr,
                                    use_compact ? static_cast<const rsdb::UnitBase*>(d->unit_bases.p) : nullptr,
                                    use_compact ? d->n_units : 0));
  return OK_CLEAR();
}

rsdb_status rsdb_dbuffer_reduce_scatter_adam(rsdb_dbuffer* d, rsdb_p2p* p, const rsdb_adam_cfg* cfg,
                                             int64_t step, void* stream) {
  return rs_adam_dbuffer(d, p, cfg, step, stream, false);
}

rsdb_status rsdb_dbuffer_reduce_scatter_adam_gather(rsdb_dbuffer* d, rsdb_p2p* p, const rsdb_adam_cfg* cfg,
                                                    int64_t step, void* stream) {
  return rs_adam_dbuffer(d, p, cfg, step, stream, true);
}

rsdb_status rsdb_dbuffer_create(const rsdb_layout* const* units, int32_t n_units, rsdb_comm* comm,
                                int32_t rank, int64_t qblock, int64_t align_bytes,
                                void* const* arena_base, rsdb_dbuffer** out) {
  return dbuffer_create_impl(units, n_units, comm, rank, qblock, nullptr, align_bytes, arena_base, out);
}

rsdb_status rsdb_dbuffer_create_q(const rsdb_layout* const* units, int32_t n_units, rsdb_comm* comm,
                                  int32_t rank, const rsdb_qspec* const* specs, int64_t align_bytes,
                                  void* const* arena_base, rsdb_dbuffer** out) {
  if (!specs) return fail(RSDB_EINVAL, "null specs");
  return dbuffer_create_impl(units, n_units, comm, rank, 0, specs, align_bytes, arena_base, out);
}

rsdb_unit* rsdb_dbuffer_unit(rsdb_dbuffer* d, int32_t i) {
  if (!d || i < 0 || i >= int32_t(d->units.size())) return nullptr;
  return d->units[size_t(i)].get();
}
int64_t rsdb_dbuffer_num_blocks(const rsdb_dbuffer* d) { return d ? d->nblocks : -1; }

rsdb_status rsdb_dbuffer_step_8bit_adam(rsdb_dbuffer* d, const rsdb_adam_cfg* cfg, int64_t step,
                                        void* stream) {
  if (!d) return fail(RSDB_EINVAL, "null dbuffer");
  rsdb::AdamScalars s;
  if (rsdb_status e = adam_scalars(cfg, step, &s)) return e;
  if (d->nblocks == 0) return OK_CLEAR();
  rsdb::AdamPtrs p{static_cast<float*>(d->base[RSDB_KIND_MASTER]),
                   static_cast<int8_t*>(d->base[RSDB_KIND_MQ]),
                   static_cast<uint8_t*>(d->base[RSDB_KIND_VQ]),
                   static_cast<float*>(d->base[RSDB_KIND_MABS]),
                   static_cast<float*>(d->base[RSDB_KIND_VABS]),
                   static_cast<const float*>(d->base[RSDB_KIND_GRAD_F32]),
                   d->base[RSDB_KIND_PARAM_FULL],
                   d->param_bf16};
  CUDA_TRY(rsdb::launch_adam8(static_cast<const rsdb::AdamBlock*>(d->blocks.p), d->nblocks, p, s, d->has_tiles,
                              S_(stream)));
  return OK_CLEAR();
}

rsdb_status rsdb_dbuffer_step_8bit_adam_dynamic(rsdb_dbuffer* d, const rsdb_adam_cfg* cfg, int64_t step,
                                                void* stream) {
  if (!d) return fail(RSDB_EINVAL, "null dbuffer");
  rsdb::AdamScalars s;
  if (rsdb_status e = adam_scalars(cfg, step, &s)) return e;
  if (d->nblocks == 0) return OK_CLEAR();
  rsdb::AdamPtrs p{static_cast<float*>(d->base[RSDB_KIND_MASTER]),
                   static_cast<int8_t*>(d->base[RSDB_KIND_MQ]),
                   static_cast<uint8_t*>(d->base[RSDB_KIND_VQ]),
                   static_cast<float*>(d->base[RSDB_KIND_MABS]),
                   static_cast<float*>(d->base[RSDB_KIND_VABS]),
                   static_cast<const float*>(d->base[RSDB_KIND_GRAD_F32]),
                   d->base[RSDB_KIND_PARAM_FULL],
                   d->param_bf16};
  CUDA_TRY(rsdb::launch_adam8_dyn(static_cast<const rsdb::AdamBlock*>(d->blocks.p), d->nblocks, p, s,
                                  S_(stream)));
  return OK_CLEAR();
}

rsdb_status rsdb_dbuffer_step_host(rsdb_dbuffer* d, rsdb_p2p* p, const rsdb_adam_cfg* cfg, int64_t step,
                                   const void* const* host_grads, void* const* host_shards, void* stream) {
  if (!d || !host_grads || !host_shards) return fail(RSDB_EINVAL, "null argument");
  if (!d->param_bf16) return fail(RSDB_EMISMATCH, "the host step needs bf16 units");
  const size_t n = d->units.size();
  for (size_t u = 0; u < n; ++u)
    if (!host_grads[u] || !host_shards[u]) return fail(RSDB_EINVAL, "null host buffer for unit %zu", u);
  if (!d->host) {
    auto h = std::make_unique<HostPipe>();
    CUDA_TRY(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming));
    for (auto* v : {&h->ev_in, &h->ev_k, &h->ev_out}) {
      v->assign(n, nullptr);
      for (auto& e : *v) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    h->k_rec.assign(n, 0);
    h->out_rec.assign(n, 0);
    // chunks of <= 16 M shard elements (32 MB of bf16 copy-out) at block
    // boundaries, from the unit's block table (read back once).  The chunk
    // COUNT comes from S, the same on every rank, because at world > 1 every
    // chunk launch is a collective (its barriers count all ranks).  A unit
    // with 2-D tiles (whose rows interleave across neighbouring tiles) is
    // updated by its first launch; its other launches are empty (barriers only)
    constexpr int64_t CHUNK = int64_t(16) << 20;
    h->chunks.resize(n);
    h->ev_chunk.resize(n);
    h->ev_chunk_in.resize(n);
    for (size_t i = 0; i < n; ++i) {
      rsdb_unit* u = d->units[i].get();
      const int64_t S = u->L.S;
      const int64_t nc = std::max<int64_t>(1, (S + CHUNK - 1) / CHUNK);
      std::vector<rsdb::AdamBlock> tb(size_t(u->nblocks));
      if (u->nblocks)
        CUDA_TRY(cudaMemcpy(tb.data(), u->blocks.p, tb.size() * sizeof(rsdb::AdamBlock), cudaMemcpyDeviceToHost));
      const bool flat = std::all_of(tb.begin(), tb.end(), [](const rsdb::AdamBlock& x) { return x.cols == x.len; });
      // chunk c takes the blocks starting in [c S / nc, (c+1) S / nc)
      int64_t b = 0;
      for (int64_t c = 0; c < nc; ++c) {
        const int64_t lim = (c + 1) * S / nc;
        const int64_t first = b;
        while (b < u->nblocks && (c == nc - 1 || !flat || tb[size_t(b)].state_off < lim)) ++b;
        h->chunks[i].push_back({first, b - first, 0, 0});
      }
      auto& ch = h->chunks[i];
      for (size_t c = 0; c < ch.size(); ++c) {  // shard cover: [start of this chunk's first block, next's)
        ch[c].lo = c == 0 ? 0 : (ch[c].count ? tb[size_t(ch[c].first)].state_off : ch[c - 1].hi);
        ch[c].hi = S;
        if (c) ch[c - 1].hi = ch[c].lo;
      }
      if (!flat)  // one copy-out of the whole shard, after the (single) real launch
        for (size_t c = 0; c < ch.size(); ++c) ch[c].lo = ch[c].hi = c == 0 ? 0 : S;
      if (!flat) ch[0].hi = S;
      h->ev_chunk[i].assign(ch.size(), nullptr);
      for (auto& e : h->ev_chunk[i]) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->ev_chunk_in[i].assign(ch.size(), nullptr);
      for (auto& e : h->ev_chunk_in[i]) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    d->host = std::move(h);
  }
  HostPipe& h = *d->host;
  cudaStream_t st = S_(stream);
  // the copies start after everything already on the caller's stream
  CUDA_TRY(cudaEventRecord(h.ev_start, st));
  CUDA_TRY(cudaStreamWaitEvent(h.s_in, h.ev_start, 0));
  CUDA_TRY(cudaStreamWaitEvent(h.s_out, h.ev_start, 0));
  for (size_t i = n; i-- > 0;) {  // FSDP backward order, the same on every rank
    rsdb_unit* u = d->units[i].get();
    const size_t gbytes = size_t(int64_t(u->L.m) * u->L.S * 2);
    const size_t sbytes = size_t(u->L.S * 2);
    // gradients: overwrite only after this unit's previous kernel (whose done
    // barrier also means no peer still reads them)
    if (h.k_rec[i]) CUDA_TRY(cudaStreamWaitEvent(h.s_in, h.ev_k[i], 0));
    // world 1: the gradients chunk by chunk too (chunk c's kernel needs exactly
    // its shard range); world > 1: the whole buffer (every owner's ranges)
    const bool chunk_in = u->L.m == 1 && h.chunks[i].size() > 1;
    if (!chunk_in) {
      if (gbytes)
        CUDA_TRY(cudaMemcpyAsync(u->bufs.grad_full, host_grads[i], gbytes, cudaMemcpyHostToDevice, h.s_in));
      CUDA_TRY(cudaEventRecord(h.ev_in[i], h.s_in));
      CUDA_TRY(cudaStreamWaitEvent(st, h.ev_in[i], 0));
    } else {
      for (size_t c = 0; c < h.chunks[i].size(); ++c) {
        const HostPipe::Chunk& ck = h.chunks[i][c];
        if (ck.hi > ck.lo)
          CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(u->bufs.grad_full) + ck.lo * 2,
                                   static_cast<const char*>(host_grads[i]) + ck.lo * 2, size_t(ck.hi - ck.lo) * 2,
                                   cudaMemcpyHostToDevice, h.s_in));
        CUDA_TRY(cudaEventRecord(h.ev_chunk_in[i][c], h.s_in));
      }
      CUDA_TRY(cudaEventRecord(h.ev_in[i], h.s_in));
    }
    // the shard: rewrite only after its previous copy-out
    if (h.out_rec[i]) CUDA_TRY(cudaStreamWaitEvent(st, h.ev_out[i], 0));
    // the unit in block-range chunks: chunk c's copy-out overlaps chunk c+1's kernel
    const char* shard = static_cast<const char*>(u->bufs.param_full) + int64_t(u->rank) * u->L.S * 2;
    for (size_t c = 0; c < h.chunks[i].size(); ++c) {
      const HostPipe::Chunk& ck = h.chunks[i][c];
      if (chunk_in) CUDA_TRY(cudaStreamWaitEvent(st, h.ev_chunk_in[i][c], 0));
      if (rsdb_status e = rs_adam_unit(u, p, nullptr, cfg, step, stream, u->L.m > 1, ck.first, ck.count))
        return e;
      CUDA_TRY(cudaEventRecord(h.ev_chunk[i][c], st));
      CUDA_TRY(cudaStreamWaitEvent(h.s_out, h.ev_chunk[i][c], 0));
      if (ck.hi > ck.lo)
        CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(host_shards[i]) + ck.lo * 2, shard + ck.lo * 2,
                                 size_t(ck.hi - ck.lo) * 2, cudaMemcpyDeviceToHost, h.s_out));
    }
    (void)sbytes;
    CUDA_TRY(cudaEventRecord(h.ev_k[i], st));
    h.k_rec[i] = 1;
    CUDA_TRY(cudaEventRecord(h.ev_out[i], h.s_out));
    h.out_rec[i] = 1;
  }
  // stream order: the call is complete when the caller's stream reaches here
  if (n) {
    CUDA_TRY(cudaStreamWaitEvent(st, h.ev_in[0], 0));
    CUDA_TRY(cudaStreamWaitEvent(st, h.ev_out[0], 0));
  }
  return OK_CLEAR();
}

rsdb_status rsdb_dbuffer_zero_grads(rsdb_dbuffer* d, void* stream) {
  if (!d) return fail(RSDB_EINVAL, "null dbuffer");
  for (auto& u : d->units)
    CUDA_TRY(cudaMemsetAsync(u->bufs.grad_full, 0,
                             size_t(int64_t(u->L.m) * u->L.S * u->L.elem_bytes), S_(stream)));
  return OK_CLEAR();
}

void rsdb_dbuffer_free(rsdb_dbuffer* d) { delete d; }

// ---------------------------------------------------------------------------
// batched ragged copy
// ---------------------------------------------------------------------------
rsdb_status rsdb_copy_plan_create(const rsdb_segment* segs, int64_t n, int32_t src_dtype,
                                  int32_t dst_dtype, float scale, rsdb_copy_plan** out) {
  if (!out || n < 0 || (n > 0 && !segs)) return fail(RSDB_EINVAL, "null argument");
  if ((src_dtype != RSDB_BF16 && src_dtype != RSDB_F32) || (dst_dtype != RSDB_BF16 && dst_dtype != RSDB_F32))
    return fail(RSDB_EINVAL, "dtype must be RSDB_BF16 or RSDB_F32");
  auto cp = std::make_unique<rsdb_copy_plan>();
  std::vector<rsdb::CopySeg> v;
  int64_t chunks = 0;
  constexpr int64_t CH = 4096;  // must match COPY_CHUNK in kernels.cu
  for (int64_t i = 0; i < n; ++i) {
    if (segs[i].numel < 0 || (segs[i].numel > 0 && (!segs[i].src || !segs[i].dst)))
      return fail(RSDB_EINVAL, "segment %lld invalid", (long long)i);
    if (segs[i].numel == 0) continue;
    v.push_back({segs[i].src, segs[i].dst, segs[i].numel, chunks});
    chunks += (segs[i].numel + CH - 1) / CH;
  }
  cp->nseg = int64_t(v.size());
  cp->total_chunks = chunks;
  cp->src_bf16 = src_dtype == RSDB_BF16;
  cp->dst_bf16 = dst_dtype == RSDB_BF16;
  cp->scale = scale;
  if (!v.empty()) {
    if (rsdb_status st = require_device()) return st;
    if (rsdb_status st = cp->segs.upload(v.data(), v.size() * sizeof(rsdb::CopySeg))) return st;
  }
  *out = cp.release();
  return OK_CLEAR();
}

rsdb_status rsdb_copy_run(const rsdb_copy_plan* cp, void* stream) {
  if (!cp) return fail(RSDB_EINVAL, "null plan");
  CUDA_TRY(rsdb::launch_copy_segments(static_cast<const rsdb::CopySeg*>(cp->segs.p), cp->nseg,
                                      cp->total_chunks, cp->src_bf16, cp->dst_bf16, cp->scale,
                                      S_(stream)));
  return OK_CLEAR();
}

void rsdb_copy_plan_free(rsdb_copy_plan* cp) { delete cp; }

}  // extern "C"
