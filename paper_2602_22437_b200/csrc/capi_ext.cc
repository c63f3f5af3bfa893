// extern "C" extensions of the C ABI (include/rsdb.h): SURVEY §8(f) N2 FP8
// block quantization fused with the AllGather, N3 distributed Muon, and the
// §7 K-slot unsharded ring.
#include "capi_internal.hpp"

extern "C" {

// ---------------------------------------------------------------------------
// N2: FP8 block quantization fused with the AllGather
// ---------------------------------------------------------------------------
struct rsdb_fp8_unit {
  rsdb::Layout L;
  rsdb_comm* comm = nullptr;
  int32_t rank = 0;
  const float* master = nullptr;
  uint8_t* codes = nullptr;
  float* scales = nullptr;
  int64_t ntiles_rank = 0, ntiles_total = 0, first_slot = 0;
  DevTable tiles;  // rsdb::Fp8Tile[ntiles_rank]
};

rsdb_status rsdb_fp8_unit_create(const rsdb_layout* l, const rsdb_qspec* specs, rsdb_comm* comm,
                                 int32_t rank, const float* master_shard, uint8_t* codes_full,
                                 float* scales_full, rsdb_fp8_unit** out) {
  if (!l || !specs || !out) return fail(RSDB_EINVAL, "null argument");
  *out = nullptr;
  const rsdb::Layout& L = l->L;
  if (L.elem_bytes != 1) return fail(RSDB_EMISMATCH, "FP8 units are planned with elem_bytes 1");
  if (rank < 0 || rank >= L.m) return fail(RSDB_EINVAL, "rank %d out of [0,%d)", rank, L.m);
  if (comm && (comm->world != L.m || comm->rank != rank))
    return fail(RSDB_EMISMATCH, "comm does not match the layout's world / rank");
  for (size_t t = 0; t < L.e.size(); ++t)
    if (specs[t].row_len <= 0 || specs[t].tile_rows <= 0 || specs[t].tile_cols <= 0)
      return fail(RSDB_EINVAL, "tensor %zu: FP8 units need a tile spec (row_len, rows, cols)", t);
  const auto sp = make_specs(L, 0, specs);
  auto u = std::make_unique<rsdb_fp8_unit>();
  u->L = L;
  u->comm = comm;
  u->rank = rank;
  std::vector<rsdb::Fp8Tile> mine;
  for (int32_t r = 0; r < L.m; ++r) {
    std::vector<rsdb::QTile> t;
    if (rsdb_status st = tiles_of(L, r, sp, &t)) return st;
    if (r == rank) {
      u->first_slot = u->ntiles_total;
      for (size_t i = 0; i < t.size(); ++i)
        mine.push_back({t[i].off, t[i].rows, t[i].cols, int32_t(t[i].pitch),
                        int32_t(u->ntiles_total + int64_t(i))});
    }
    u->ntiles_total += int64_t(t.size());
  }
  if (u->ntiles_total > INT32_MAX) return fail(RSDB_EINVAL, "too many tiles");
  u->ntiles_rank = int64_t(mine.size());
  if (u->ntiles_rank > 0 && (!master_shard || !codes_full || !scales_full))
    return fail(RSDB_EINVAL, "null buffer");
  if (master_shard && !aligned16(master_shard)) return fail(RSDB_EINVAL, "master_shard must be 16-B aligned");
  u->master = master_shard;
  u->codes = codes_full;
  u->scales = scales_full;
  if (!mine.empty()) {
    if (rsdb_status st = require_device()) return st;
    if (rsdb_status st = u->tiles.upload(mine.data(), mine.size() * sizeof(rsdb::Fp8Tile))) return st;
  }
  *out = u.release();
  return OK_CLEAR();
}

int64_t rsdb_fp8_unit_num_tiles(const rsdb_fp8_unit* u) { return u ? u->ntiles_total : -1; }
int64_t rsdb_fp8_unit_first_slot(const rsdb_fp8_unit* u) { return u ? u->first_slot : -1; }

rsdb_status rsdb_fp8_quantize_all_gather(rsdb_fp8_unit* u, rsdb_p2p* p, void* stream) {
  if (!u) return fail(RSDB_EINVAL, "null unit");
  const int m = u->L.m;
  const int64_t S = u->L.S;
  rsdb::P2PPtrs codes{}, scales{};
  rsdb::P2PSignals sg{};
  if (m > 1) {
    if (!p) return fail(RSDB_EINVAL, "world > 1 needs a p2p object");
    if (!u->comm || u->comm != p->comm) return fail(RSDB_EMISMATCH, "unit and p2p use different comms");
    int32_t bi = 0;
    int64_t off = 0;
    if (rsdb_status e = p2p_find(p, u->codes, int64_t(m) * S, &bi, &off)) return e;
    for (int r = 0; r < m; ++r) codes.p[r] = p->peer[size_t(bi)][size_t(r)] + off + int64_t(u->rank) * S;
    if (rsdb_status e = p2p_find(p, u->scales, u->ntiles_total * 4, &bi, &off)) return e;
    for (int r = 0; r < m; ++r) scales.p[r] = p->peer[size_t(bi)][size_t(r)] + off;
    p2p_signals(p, m, &sg);
    ++p->epoch;
  } else {
    codes.p[0] = u->codes;
    scales.p[0] = u->scales;
  }
  if (u->ntiles_rank == 0 && m == 1) return OK_CLEAR();
  // every rank launches (the barriers count all ranks), even with no tiles
  CUDA_TRY(rsdb::launch_fp8_quant_ag(static_cast<const rsdb::Fp8Tile*>(u->tiles.p), u->ntiles_rank,
                                     u->master, codes, scales, m, u->rank, m > 1 ? &sg : nullptr,
                                     m > 1 ? p->epoch : 0, S_(stream)));
  return OK_CLEAR();
}

void rsdb_fp8_unit_free(rsdb_fp8_unit* u) { delete u; }

// ---------------------------------------------------------------------------
// N3: distributed Muon (Algorithm 2)
// ---------------------------------------------------------------------------
constexpr size_t MUON_CUBLAS_WS = size_t(32) << 20;  // cuBLAS's recommended size on Hopper / Blackwell

struct rsdb_muon {
  rsdb::Layout L;
  rsdb_comm* comm = nullptr;
  int32_t rank = 0, bf16 = 0;
  int64_t esz = 4;
  std::vector<int64_t> rows, cols;
  std::vector<int32_t> roots;
  std::vector<int64_t> xoff;  // element offset of matrix t in its root's workspace
  std::vector<int32_t> mine;  // matrices this rank is the root of
  int64_t ws_bytes = 0, x2_off = 0, a_off = 0, b_off = 0, ss_off = 0;  // bytes, this rank
  // bf16 (tensor-core) mode: W, W^T and their next-iteration copies, padded
  // leading dimensions (multiples of 8 elements, ns_umma.cu)
  int64_t w_off = 0, wt_off = 0, w2_off = 0, w2t_off = 0;
  DevTable mom, gat, app;
  DevTable cublas_ws;  // cuBLAS workspace (MUON_CUBLAS_WS bytes)
  int64_t n_mom = 0, max_mom = 0, n_gat = 0, c_gat = 0, n_app = 0, c_app = 0;
  std::vector<rsdb::MuonSeg> app_host;
  rsdb_muon_bufs b{};
  bool bound = false;
  cublasHandle_t h = nullptr;
  ~rsdb_muon() {
    if (h) cublasDestroy(h);
  }
};

static int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// R24 SelectRoot: decreasing NS cost (stable), least loaded, then most owned, then lowest rank
static std::vector<int32_t> muon_roots(const rsdb::Layout& L, const std::vector<int64_t>& rows,
                                       const std::vector<int64_t>& cols) {
  const size_t n = rows.size();
  std::vector<int32_t> roots(n, -1);
  std::vector<size_t> order;
  for (size_t t = 0; t < n; ++t)
    if (rows[t] > 0) order.push_back(t);
  auto cost = [&](size_t t) { return rows[t] * cols[t] * std::min(rows[t], cols[t]); };
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return cost(a) > cost(b); });
  std::vector<int64_t> load(size_t(L.m), 0);
  for (size_t t : order) {
    int32_t best = 0;
    int64_t best_own = -1;
    for (int32_t k = 0; k < L.m; ++k) {
      const int64_t lo = int64_t(k) * L.S, hi = lo + L.S;
      const int64_t own = std::max<int64_t>(0, std::min(L.l[t] + L.e[t], hi) - std::max(L.l[t], lo));
      if (best_own < 0 || load[size_t(k)] < load[size_t(best)] ||
          (load[size_t(k)] == load[size_t(best)] && own > best_own)) {
        best = k;
        best_own = own;
      }
    }
    roots[t] = best;
    load[size_t(best)] += cost(t);
  }
  return roots;
}

rsdb_status rsdb_muon_create(const rsdb_layout* l, const int64_t* rows, const int64_t* cols,
                             rsdb_comm* comm, int32_t rank, int32_t precision, rsdb_muon** out) {
  if (!l || !rows || !cols || !out) return fail(RSDB_EINVAL, "null argument");
  *out = nullptr;
  const rsdb::Layout& L = l->L;
  if (rank < 0 || rank >= L.m) return fail(RSDB_EINVAL, "rank %d out of [0,%d)", rank, L.m);
  if (L.m > rsdb::P2P_MAX_RANKS) return fail(RSDB_EINVAL, "world > %d", rsdb::P2P_MAX_RANKS);
  if (L.m > 1 && !comm) return fail(RSDB_EINVAL, "world > 1 needs a comm");
  if (comm && (comm->world != L.m || comm->rank != rank))
    return fail(RSDB_EMISMATCH, "comm does not match the layout's world / rank");
  if (precision != RSDB_F32 && precision != RSDB_BF16) return fail(RSDB_EINVAL, "precision must be F32 or BF16");
  auto u = std::make_unique<rsdb_muon>();
  u->L = L;
  u->comm = comm;
  u->rank = rank;
  u->bf16 = precision == RSDB_BF16;
  u->esz = u->bf16 ? 2 : 4;
  const size_t n = L.e.size();
  for (size_t t = 0; t < n; ++t) {
    const bool mat = rows[t] > 0 || cols[t] > 0;
    if (mat && (rows[t] <= 0 || cols[t] <= 0 || rows[t] * cols[t] != L.e[t]))
      return fail(RSDB_EINVAL, "tensor %zu: rows*cols != numel", t);
    if (mat && (rows[t] > INT32_MAX || cols[t] > INT32_MAX))
      return fail(RSDB_EINVAL, "tensor %zu: dimension exceeds int32", t);
    u->rows.push_back(mat ? rows[t] : 0);
    u->cols.push_back(mat ? cols[t] : 0);
  }
  u->roots = muon_roots(L, u->rows, u->cols);
  // every rank's workspace layout (owners need the roots' offsets)
  u->xoff.assign(n, 0);
  std::vector<int64_t> used(size_t(L.m), 0);
  const int64_t A = 256;
  for (size_t t = 0; t < n; ++t) {
    if (u->roots[t] < 0) continue;
    int64_t& o = used[size_t(u->roots[t])];
    u->xoff[t] = o / u->esz;
    o += align_up(u->rows[t] * u->cols[t] * u->esz, A);
    if (u->roots[t] == rank) u->mine.push_back(int32_t(t));
  }
  int64_t maxrc = 0, maxk = 0;
  for (int32_t t : u->mine) {
    maxrc = std::max(maxrc, u->rows[size_t(t)] * u->cols[size_t(t)]);
    const int64_t k = std::min(u->rows[size_t(t)], u->cols[size_t(t)]);
    maxk = std::max(maxk, k * k);
  }
  int64_t off = used[size_t(rank)];
  if (u->bf16) {  // padded W / W^T pairs (2 iterations) + padded A, B
    int64_t maxw = 0, maxkk = 0;
    for (int32_t t : u->mine) {
      const int64_t k = std::min(u->rows[size_t(t)], u->cols[size_t(t)]);
      const int64_t L = std::max(u->rows[size_t(t)], u->cols[size_t(t)]);
      maxw = std::max({maxw, k * align_up(L, 8), L * align_up(k, 8)});
      maxkk = std::max(maxkk, k * align_up(k, 8));
    }
    for (int64_t* o : {&u->w_off, &u->wt_off, &u->w2_off, &u->w2t_off}) {
      *o = off;
      off += align_up(maxw * 2, A);
    }
    u->a_off = off;
    off += align_up(maxkk * 2, A);
    u->b_off = off;
    off += align_up(maxkk * 2, A);
  } else {
    u->x2_off = off;
    off += align_up(maxrc * u->esz, A);
    u->a_off = off;
    off += align_up(maxk * u->esz, A);
    u->b_off = off;
    off += align_up(maxk * u->esz, A);
  }
  u->ss_off = off;
  off += align_up(int64_t(u->mine.size()) * 8, A);
  u->ws_bytes = std::max<int64_t>(off, A);
  // segment tables
  const int64_t CH = 8192;
  std::vector<int64_t> mom;
  std::vector<rsdb::MuonSeg> gat;
  const int64_t lo = int64_t(rank) * L.S, hi = lo + L.S;
  for (size_t t = 0; t < n; ++t) {
    if (u->roots[t] < 0) continue;
    const int64_t a = std::max(L.l[t], lo), b = std::min(L.l[t] + L.e[t], hi);
    if (a < b) {  // my piece: momentum + apply
      mom.push_back(a - lo);
      mom.push_back(b - a);
      u->max_mom = std::max(u->max_mom, b - a);
      const double scale = std::sqrt(std::max(1.0, double(u->rows[t]) / double(u->cols[t])));
      u->app_host.push_back({u->xoff[t] + (a - L.l[t]), a - lo, b - a, 0, u->roots[t], float(scale)});
    }
    if (u->roots[t] == rank)
      for (int32_t k = 0; k < L.m; ++k) {  // every owner's piece -> my workspace
        const int64_t pa = std::max(L.l[t], int64_t(k) * L.S), pb = std::min(L.l[t] + L.e[t], int64_t(k + 1) * L.S);
        if (pa < pb) gat.push_back({pa - int64_t(k) * L.S, u->xoff[t] + (pa - L.l[t]), pb - pa, 0, k, 0.f});
      }
  }
  for (auto& sg : gat) {
    sg.chunk_begin = u->c_gat;
    u->c_gat += (sg.n + CH - 1) / CH;
  }
  for (auto& sg : u->app_host) {
    sg.chunk_begin = u->c_app;
    u->c_app += (sg.n + CH - 1) / CH;
  }
  u->n_mom = int64_t(mom.size() / 2);
  u->n_gat = int64_t(gat.size());
  u->n_app = int64_t(u->app_host.size());
  if (rsdb_status st = require_device()) return st;
  if (rsdb_status st = u->mom.upload(mom.data(), mom.size() * sizeof(int64_t))) return st;
  if (rsdb_status st = u->gat.upload(gat.data(), gat.size() * sizeof(rsdb::MuonSeg))) return st;
  if (rsdb_status st = u->app.upload(u->app_host.data(), u->app_host.size() * sizeof(rsdb::MuonSeg)))
    return st;
  if (cublasCreate(&u->h) != CUBLAS_STATUS_SUCCESS) return fail(RSDB_ECUDA, "cublasCreate failed");
  // cuBLAS workspace owned here and set after every cublasSetStream, so a step
  // never allocates (no implicit synchronisation while peers' kernels wait in
  // a barrier; graph-capturable)
  if (rsdb_status st = u->cublas_ws.alloc(MUON_CUBLAS_WS)) return st;
  *out = u.release();
  return OK_CLEAR();
}

rsdb_status rsdb_muon_select_roots(const rsdb_layout* l, const int64_t* rows, const int64_t* cols,
                                   int32_t* roots) {
  if (!l || !rows || !cols || !roots) return fail(RSDB_EINVAL, "null argument");
  const rsdb::Layout& L = l->L;
  std::vector<int64_t> r, c;
  for (size_t t = 0; t < L.e.size(); ++t) {
    const bool mat = rows[t] > 0 || cols[t] > 0;
    if (mat && (rows[t] <= 0 || cols[t] <= 0 || rows[t] * cols[t] != L.e[t]))
      return fail(RSDB_EINVAL, "tensor %zu: rows*cols != numel", t);
    r.push_back(mat ? rows[t] : 0);
    c.push_back(mat ? cols[t] : 0);
  }
  const auto v = muon_roots(L, r, c);
  std::copy(v.begin(), v.end(), roots);
  return OK_CLEAR();
}

int32_t rsdb_muon_root(const rsdb_muon* u, int32_t t) {
  return (u && t >= 0 && size_t(t) < u->roots.size()) ? u->roots[size_t(t)] : -1;
}
int64_t rsdb_muon_workspace_bytes(const rsdb_muon* u) { return u ? u->ws_bytes : -1; }

rsdb_status rsdb_muon_bind(rsdb_muon* u, const rsdb_muon_bufs* b) {
  if (!u || !b) return fail(RSDB_EINVAL, "null argument");
  if (u->L.S > 0 && (!b->master || !b->momentum || !b->grad || !b->u))
    return fail(RSDB_EINVAL, "null shard buffer");
  if (!b->workspace) return fail(RSDB_EINVAL, "null workspace");
  if (reinterpret_cast<uintptr_t>(b->workspace) % 256) return fail(RSDB_EINVAL, "workspace must be 256-B aligned");
  u->b = *b;
  u->bound = true;
  return OK_CLEAR();
}

#define CUBLAS_TRY(expr)                                                              \
  do {                                                                                \
    cublasStatus_t s_ = (expr);                                                       \
    if (s_ != CUBLAS_STATUS_SUCCESS) return fail(RSDB_ECUDA, "%s: cuBLAS status %d", #expr, int(s_)); \
  } while (0)

static cublasStatus_t muon_gemm(cublasHandle_t h, bool bf16, cublasOperation_t ta, cublasOperation_t tb, int m,
                                int n, int k, float alpha, const void* A, int lda, const void* B, int ldb,
                                float beta, void* C, int ldc) {
  if (bf16)
    return cublasGemmEx(h, ta, tb, m, n, k, &alpha, A, CUDA_R_16BF, lda, B, CUDA_R_16BF, ldb, &beta, C,
                        CUDA_R_16BF, ldc, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  return cublasSgemm(h, ta, tb, m, n, k, &alpha, static_cast<const float*>(A), lda, static_cast<const float*>(B),
                     ldb, &beta, static_cast<float*>(C), ldc);
}

// R22 in bf16 on the tensor cores (ns_umma.cu): W = the matrix as k x L
// (k = min(rows, cols)), kept in both layouts; per iteration three
// tcgen05 GEMMs with the quintic's combinations in their epilogues
static rsdb_status muon_newton_schulz_umma(rsdb_muon* u, int32_t t, int idx, const rsdb_muon_cfg* cfg,
                                           cudaStream_t st) {
  char* ws = static_cast<char*>(u->b.workspace);
  char* X = ws + u->xoff[size_t(t)] * 2;
  double* ss = reinterpret_cast<double*>(ws + u->ss_off) + idx;
  const int64_t R = u->rows[size_t(t)], C = u->cols[size_t(t)];
  if (cfg->ns_steps == 0) {  // normalisation only
    CUDA_TRY(rsdb::launch_muon_normalize(X, R * C, 1, ss, cfg->eps, st));
    return RSDB_OK;
  }
  const bool tall = R > C;
  const int k = int(tall ? C : R), L = int(tall ? R : C);
  const int64_t Lp = align_up(L, 8), kp = align_up(k, 8);
  char* P = ws + u->w_off;    // W   (k x L, ld Lp)
  char* PT = ws + u->wt_off;  // W^T (L x k, ld kp)
  char* Q = ws + u->w2_off;
  char* QT = ws + u->w2t_off;
  char* Am = ws + u->a_off;   // k x k, ld kp
  char* Bm = ws + u->b_off;
  // X (R x C) -> s X, (s X)^T: wide: W = sX, W^T = (sX)^T; tall: W^T = sX, W = (sX)^T
  if (!tall)
    CUDA_TRY(rsdb::launch_muon_scale_transpose(X, int(R), int(C), ss, cfg->eps, P, Lp, PT, kp, st));
  else
    CUDA_TRY(rsdb::launch_muon_scale_transpose(X, int(R), int(C), ss, cfg->eps, PT, kp, P, Lp, st));
  const float a = 3.4445f, b = -4.7750f, c = 2.0315f;
  for (int it = 0; it < cfg->ns_steps; ++it) {
    // A = W W^T (symmetric: the upper-triangle tiles + their mirror)
    CUDA_TRY(rsdb::launch_umma_gemm(k, k, L, P, Lp, P, Lp, 1.f, 0.f, nullptr, 0, Am, kp, nullptr, 0, st, true));
    // B = c A A + b A   (A symmetric: A A = A A^T; B symmetric too)
    CUDA_TRY(rsdb::launch_umma_gemm(k, k, k, Am, kp, Am, kp, c, b, Am, kp, Bm, kp, nullptr, 0, st, true));
    // W' = B W + a W, and W'^T   (B-op rows of W^T)
    CUDA_TRY(rsdb::launch_umma_gemm(k, L, k, Bm, kp, PT, kp, 1.f, a, P, Lp, Q, Lp, QT, kp, st));
    std::swap(P, Q);
    std::swap(PT, QT);
  }
  // the result back into the matrix slot (rows x cols, contiguous)
  if (!tall)
    CUDA_TRY(rsdb::launch_muon_copy2d(P, Lp, int(R), int(C), X, st));
  else
    CUDA_TRY(rsdb::launch_muon_copy2d(PT, kp, int(R), int(C), X, st));
  return RSDB_OK;
}

// R22 on the root's matrix t (row-major rows x cols at X), result left in X;
// fp32 parity mode on cuBLAS SGEMM, bf16 on the hand-written tcgen05 GEMM
static rsdb_status muon_newton_schulz(rsdb_muon* u, int32_t t, int idx, const rsdb_muon_cfg* cfg, cudaStream_t st) {
  const bool bf = u->bf16 != 0;
  if (bf) return muon_newton_schulz_umma(u, t, idx, cfg, st);
  char* ws = static_cast<char*>(u->b.workspace);
  char* X = ws + u->xoff[size_t(t)] * u->esz;
  char* X2 = ws + u->x2_off;
  char* Am = ws + u->a_off;
  char* Bm = ws + u->b_off;
  double* ss = reinterpret_cast<double*>(ws + u->ss_off) + idx;
  const int64_t R = u->rows[size_t(t)], C = u->cols[size_t(t)];
  const int64_t nel = R * C;
  CUDA_TRY(rsdb::launch_muon_normalize(X, nel, bf, ss, cfg->eps, st));
  const bool tall = R > C;
  const int k = int(tall ? C : R), L = int(tall ? R : C);
  const float a = 3.4445f, b = -4.7750f, c = 2.0315f;
  char* P = X;
  char* Q = X2;
  const size_t kk = size_t(k) * size_t(k) * size_t(u->esz), xb = size_t(nel) * size_t(u->esz);
  for (int it = 0; it < cfg->ns_steps; ++it) {
    if (!tall) {  // storage = W^T column-major (L x k), W = X (k x L)
      CUBLAS_TRY(muon_gemm(u->h, bf, CUBLAS_OP_T, CUBLAS_OP_N, k, k, L, 1.f, P, L, P, L, 0.f, Am, k));
    } else {      // storage = W column-major (k x L), W = X^T
      CUBLAS_TRY(muon_gemm(u->h, bf, CUBLAS_OP_N, CUBLAS_OP_T, k, k, L, 1.f, P, k, P, k, 0.f, Am, k));
    }
    CUDA_TRY(cudaMemcpyAsync(Bm, Am, kk, cudaMemcpyDeviceToDevice, st));
    CUBLAS_TRY(muon_gemm(u->h, bf, CUBLAS_OP_N, CUBLAS_OP_N, k, k, k, c, Am, k, Am, k, b, Bm, k));
    CUDA_TRY(cudaMemcpyAsync(Q, P, xb, cudaMemcpyDeviceToDevice, st));
    if (!tall)  // W'^T = a W^T + W^T B^T
      CUBLAS_TRY(muon_gemm(u->h, bf, CUBLAS_OP_N, CUBLAS_OP_T, L, k, k, 1.f, P, L, Bm, k, a, Q, L));
    else        // W' = a W + B W
      CUBLAS_TRY(muon_gemm(u->h, bf, CUBLAS_OP_N, CUBLAS_OP_N, k, L, k, 1.f, Bm, k, P, k, a, Q, k));
    std::swap(P, Q);
  }
  if (P != X) CUDA_TRY(cudaMemcpyAsync(X, P, xb, cudaMemcpyDeviceToDevice, st));
  return RSDB_OK;
}

rsdb_status rsdb_muon_step(rsdb_muon* u, rsdb_p2p* p, const rsdb_muon_cfg* cfg, void* stream) {
  if (!u || !cfg) return fail(RSDB_EINVAL, "null argument");
  if (!u->bound) return fail(RSDB_EINVAL, "rsdb_muon_bind first");
  if (!(cfg->lr >= 0 && cfg->momentum >= 0 && cfg->momentum < 1 && cfg->eps >= 0 && cfg->ns_steps >= 0 &&
        cfg->ns_steps <= 100))
    return fail(RSDB_EINVAL, "invalid Muon hyper-parameters");
  const int m = u->L.m;
  cudaStream_t st = S_(stream);
  rsdb::P2PPtrs up{}, wp{};
  rsdb::P2PSignals sg{};
  if (m > 1) {
    if (!p) return fail(RSDB_EINVAL, "world > 1 needs a p2p object");
    if (p->comm != u->comm) return fail(RSDB_EMISMATCH, "muon and p2p use different comms");
    int32_t bi = 0;
    int64_t off = 0;
    if (rsdb_status e = p2p_find(p, u->b.u, u->L.S * 4, &bi, &off)) return e;
    for (int r = 0; r < m; ++r) up.p[r] = p->peer[size_t(bi)][size_t(r)] + off;
    if (rsdb_status e = p2p_find(p, u->b.workspace, 1, &bi, &off)) return e;
    for (int r = 0; r < m; ++r) wp.p[r] = p->peer[size_t(bi)][size_t(r)] + off;
    p2p_signals(p, m, &sg);
  } else {
    up.p[0] = u->b.u;
    wp.p[0] = u->b.workspace;
  }
  // 1. MomentumUpdate on the shard (R21)
  CUDA_TRY(rsdb::launch_muon_momentum(static_cast<const int64_t*>(u->mom.p), u->n_mom, u->max_mom,
                                      u->b.momentum, u->b.grad, u->b.u, float(cfg->momentum), st));
  // 2. Redistribute(u, RaggedShard(root)): one kernel, every rank launches (barriers)
  if (m > 1) ++p->epoch;
  CUDA_TRY(rsdb::launch_muon_gather(static_cast<const rsdb::MuonSeg*>(u->gat.p), u->n_gat, u->c_gat, up,
                                    u->b.workspace, u->bf16, m, u->rank, m > 1 ? &sg : nullptr,
                                    m > 1 ? p->epoch : 0, st));
  // 3. Newton-Schulz on the root's matrices (R22)
  CUBLAS_TRY(cublasSetStream(u->h, st));
  CUBLAS_TRY(cublasSetWorkspace(u->h, u->cublas_ws.p, u->cublas_ws.bytes));
  for (size_t i = 0; i < u->mine.size(); ++i)
    if (rsdb_status e = muon_newton_schulz(u, u->mine[i], int(i), cfg, st)) return e;
  // 4. Redistribute(o, p) + w -= eta * scale * o (R23): one kernel
  if (m > 1) ++p->epoch;
  CUDA_TRY(rsdb::launch_muon_apply(static_cast<const rsdb::MuonSeg*>(u->app.p), u->n_app, u->c_app, wp,
                                   u->bf16, u->b.master, u->b.param_bf16, cfg->lr, m, u->rank, m > 1 ? &sg : nullptr,
                                   m > 1 ? p->epoch : 0, st));
  return OK_CLEAR();
}

void rsdb_muon_free(rsdb_muon* u) { delete u; }

rsdb_status rsdb_ns_gemm_bf16(int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, const void* B,
                              int64_t ldb, float alpha, float beta, const void* D, int64_t ldd, void* C,
                              int64_t ldc, void* CT, int64_t ldct, void* stream) {
  if (M < 0 || N < 0 || K < 1 || !A || !B || !C || (beta != 0.f && !D))
    return fail(RSDB_EINVAL, "rsdb_ns_gemm_bf16: bad dimensions or null pointer");
  if (lda < K || ldb < K || ldc < N || (beta != 0.f && ldd < N) || (CT && ldct < M) ||
      ((lda | ldb | ldc | (beta != 0.f ? ldd : 0) | (CT ? ldct : 0)) & 7) ||
      !aligned16(A) || !aligned16(B) || !aligned16(C) || (beta != 0.f && !aligned16(D)))
    return fail(RSDB_EINVAL, "rsdb_ns_gemm_bf16: leading dimensions must be >= the row length and multiples "
                             "of 8, pointers 16-B aligned");
  if (rsdb_status st = require_device()) return st;
  CUDA_TRY(rsdb::launch_umma_gemm(M, N, K, A, lda, B, ldb, alpha, beta, D, ldd, C, ldc, CT, ldct, S_(stream)));
  return OK_CLEAR();
}

rsdb_status rsdb_ns_gemm_bf16_sym(int32_t M, int32_t K, const void* A, int64_t lda, const void* B, int64_t ldb,
                                  float alpha, float beta, const void* D, int64_t ldd, void* C, int64_t ldc,
                                  void* stream) {
  if (M < 0 || K < 1 || !A || !B || !C || (beta != 0.f && !D))
    return fail(RSDB_EINVAL, "rsdb_ns_gemm_bf16_sym: bad dimensions or null pointer");
  if (lda < K || ldb < K || ldc < M || (beta != 0.f && ldd < M) ||
      ((lda | ldb | ldc | (beta != 0.f ? ldd : 0)) & 7) || !aligned16(A) || !aligned16(B) || !aligned16(C) ||
      (beta != 0.f && !aligned16(D)))
    return fail(RSDB_EINVAL, "rsdb_ns_gemm_bf16_sym: leading dimensions must be >= the row length and "
                             "multiples of 8, pointers 16-B aligned");
  if (rsdb_status st = require_device()) return st;
  CUDA_TRY(rsdb::launch_umma_gemm(M, M, K, A, lda, B, ldb, alpha, beta, D, ldd, C, ldc, nullptr, 0, S_(stream),
                                  true));
  return OK_CLEAR();
}

// ---------------------------------------------------------------------------
// K-slot unsharded ring
// ---------------------------------------------------------------------------
rsdb_status rsdb_unit_set_shard(rsdb_unit* u, void* shard) {
  if (!u) return fail(RSDB_EINVAL, "null unit");
  if (u->has_bound_state) return fail(RSDB_EMISMATCH, "DBuffer units keep their shard in PARAM_FULL");
  if (shard && !aligned16(shard)) return fail(RSDB_EINVAL, "shard must be 16-byte aligned");
  u->shard = shard;
  return OK_CLEAR();
}

rsdb_status rsdb_unit_rebind(rsdb_unit* u, const rsdb_unit_bufs* b) {
  if (!u || !b) return fail(RSDB_EINVAL, "null argument");
  if (u->has_bound_state) return fail(RSDB_EMISMATCH, "DBuffer units cannot be rebound");
  if (!b->param_full || !b->grad_full || !b->grad_f32) return fail(RSDB_EINVAL, "unit buffers must be non-null");
  if (!aligned16(b->param_full) || !aligned16(b->grad_full) || !aligned16(b->grad_f32))
    return fail(RSDB_EMISMATCH, "unit buffers must be 16-byte aligned (P:199, P:369)");
  if (u->L.elem_bytes == 2 && b->grad_full == b->grad_f32)
    return fail(RSDB_EMISMATCH, "bf16 unit: grad_full must not alias grad_f32");
  u->bufs = *b;
  return OK_CLEAR();
}

rsdb_status rsdb_all_gather_shards_p2p(rsdb_unit* u, rsdb_p2p* p, void* stream) {
  if (!u) return fail(RSDB_EINVAL, "null unit");
  if (!u->shard) return fail(RSDB_EINVAL, "no persistent shard (rsdb_unit_set_shard)");
  const int m = u->L.m;
  const int64_t bytes_S = u->L.S * u->L.elem_bytes;
  if (u->L.S == 0) return OK_CLEAR();
  rsdb::P2PPtrs dst{};
  rsdb::P2PSignals sg{};
  if (m > 1) {
    if (rsdb_status e = p2p_common(u, p, &sg)) return e;
    int32_t bi = 0;
    int64_t off = 0;
    if (rsdb_status e = p2p_find(p, u->bufs.param_full, int64_t(m) * bytes_S, &bi, &off)) return e;
    for (int r = 0; r < m; ++r) dst.p[r] = p->peer[size_t(bi)][size_t(r)] + off;
    ++p->epoch;
  } else {
    dst.p[0] = u->bufs.param_full;
  }
  CUDA_TRY(rsdb::launch_ag_shards(dst, u->shard, bytes_S, u->rank, m, m > 1 ? &sg : nullptr,
                                  m > 1 ? p->epoch : 0, S_(stream)));
  return OK_CLEAR();
}

struct rsdb_ring {
  int32_t k = 0, next = 0;
  std::vector<cudaEvent_t> ev;
  std::vector<bool> held;  // released at least once (has an event to wait on)
  ~rsdb_ring() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
  }
};

rsdb_status rsdb_ring_create(int32_t k, rsdb_ring** out) {
  if (!out || k < 1) return fail(RSDB_EINVAL, "k_slots must be >= 1");
  *out = nullptr;
  if (rsdb_status st = require_device()) return st;
  auto r = std::make_unique<rsdb_ring>();
  r->k = k;
  r->ev.assign(size_t(k), nullptr);
  r->held.assign(size_t(k), false);
  for (auto& e : r->ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  *out = r.release();
  return OK_CLEAR();
}

rsdb_status rsdb_ring_acquire(rsdb_ring* r, void* stream, int32_t* slot) {
  if (!r || !slot) return fail(RSDB_EINVAL, "null argument");
  const int32_t s = r->next;
  r->next = (r->next + 1) % r->k;
  if (r->held[size_t(s)]) CUDA_TRY(cudaStreamWaitEvent(S_(stream), r->ev[size_t(s)], 0));
  *slot = s;
  return OK_CLEAR();
}

rsdb_status rsdb_ring_release(rsdb_ring* r, int32_t slot, void* stream) {
  if (!r || slot < 0 || slot >= r->k) return fail(RSDB_EINVAL, "bad slot");
  CUDA_TRY(cudaEventRecord(r->ev[size_t(slot)], S_(stream)));
  r->held[size_t(slot)] = true;
  return OK_CLEAR();
}

void rsdb_ring_free(rsdb_ring* r) { delete r; }

}  // extern "C"
