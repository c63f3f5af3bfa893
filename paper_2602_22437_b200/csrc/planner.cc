// Host layout planner: Algorithm 1 of PAPER §5 in C++.
//
// Readings:
//  R1  CheckValidShard's dp(t, i; S) is realised by leftmost
//      placement, which keeps every prefix end minimal: feasible <=> end <= mS.
//  R2  LCM prefixes: empty prefix (g_coll) U SortAscending(G) chain (l.21) U
//      element-count-descending chain (P:287 text).
//  R4  Binary search with a pinned probe sequence (feasibility is not
//      monotone on every input, contrary to P:287).
//  R5  Non-dividing blocks allowed (tail block).
//  R6  g_coll = 16 B / element bytes.
// Complexity: O(|T|) per CheckValidShard, O(|T| log E) per candidate.
#include "planner.hpp"

#include <algorithm>
#include <cstdio>
#include <numeric>

namespace rsdb {

int64_t Layout::E() const { return std::accumulate(e.begin(), e.end(), int64_t{0}); }

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

bool block_elems(int32_t ndim, const int64_t* shape, int32_t kind, int64_t param, int64_t* g,
                 std::string* err) {
  if (ndim < 1 || !shape || !g) {
    *err = "block_elems: ndim < 1 or null pointer";
    return false;
  }
  int64_t e = 1;
  for (int i = 0; i < ndim; ++i) {
    if (shape[i] < 1) {
      *err = "block_elems: shape entries must be >= 1";
      return false;
    }
    e *= shape[i];
  }
  switch (kind) {
    case 0:  // FLAT: q contiguous elements
      if (param < 1) break;
      *g = std::min(param, e);
      return true;
    case 1:  // ROWS: r rows of the last dimension
      if (param < 1) break;
      *g = std::min(param * shape[ndim - 1], e);
      return true;
    case 2:  // WHOLE
      *g = e;
      return true;
    case 3:  // ELEM
      *g = 1;
      return true;
    default:
      *err = "block_elems: unknown granularity kind";
      return false;
  }
  *err = "block_elems: param must be >= 1";
  return false;
}

// Leftmost start >= p of a tensor (e elements, block g) under shard size S
// satisfying the Non-Sharded Block constraint P:228; -1 if none.
// Cases of P:287: (1) inside the shard holding p; (2) crossing the next
// boundary B at a block edge without reaching B+S; (3) containing whole
// shards, which needs g | S.  Otherwise start in the next shard at
// B + (S mod g), the leftmost start whose crossing of B+S is aligned.
static int64_t place(int64_t p, int64_t e, int64_t g, int64_t S) {
  const int64_t B = (p / S + 1) * S;
  if (p + e <= B) return p;
  const int64_t l1 = p + (B - p) % g;
  if (l1 + e <= B + S || S % g == 0) return l1;
  const int64_t l2 = B + S % g;
  if (l2 + e <= B + 2 * S) return l2;
  return -1;
}

bool feasible(const std::vector<int64_t>& e, const std::vector<int64_t>& g, int32_t m, int64_t S,
              std::vector<int64_t>* starts) {
  if (starts) starts->clear();
  int64_t p = 0;
  for (size_t t = 0; t < e.size(); ++t) {
    const int64_t l = place(p, e[t], g[t], S);
    if (l < 0) return false;
    if (starts) starts->push_back(l);
    p = l + e[t];
  }
  return p <= static_cast<int64_t>(m) * S;
}

// min{k*gg : feasible(k*gg)} with the pinned probe sequence (R4).
static int64_t search(const std::vector<int64_t>& e, const std::vector<int64_t>& g, int32_t m,
                      int64_t E, int64_t gg) {
  int64_t lo = cdiv(cdiv(E, m), gg);
  int64_t hi = std::max(lo, cdiv(E, gg));
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;  // == floor((lo+hi)/2) for lo,hi >= 0
    if (feasible(e, g, m, mid * gg, nullptr))
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo * gg;
}

// lcm(a, b), or -1 if it exceeds `cap` (no overflow).
static int64_t lcm_capped(int64_t a, int64_t b, int64_t cap) {
  const int64_t q = a / std::gcd(a, b);
  if (q > cap / b) return -1;
  const int64_t r = q * b;
  return r > cap ? -1 : r;
}

bool plan(const std::vector<int64_t>& e, const std::vector<int64_t>& g, int32_t m,
          int32_t elem_bytes, int32_t gcoll_bytes, Layout* out, std::string* err) {
  if (e.size() != g.size()) {
    *err = "plan: numel/block length mismatch";
    return false;
  }
  if (m < 1 || gcoll_bytes < 1 || !(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4)) {
    *err = "plan: world >= 1, gcoll_bytes >= 1 and elem_bytes in {1,2,4} required";
    return false;
  }
  for (size_t t = 0; t < e.size(); ++t) {
    if (e[t] < 1 || g[t] < 1) {
      *err = "plan: numel and block must be >= 1 (tensor " + std::to_string(t) + ")";
      return false;
    }
  }
  Layout L;
  L.m = m;
  L.elem_bytes = elem_bytes;
  L.g_coll = std::max<int64_t>(1, gcoll_bytes / elem_bytes);
  L.e = e;
  L.g = g;
  if (e.empty()) {
    *out = L;
    return true;
  }
  const int64_t E = L.E();
  // candidate LCM prefixes (R2)
  std::vector<int64_t> cand{L.g_coll};
  {
    std::vector<int64_t> gs = g;
    std::sort(gs.begin(), gs.end());
    gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
    int64_t cur = L.g_coll;
    for (int64_t gp : gs) {
      cur = lcm_capped(cur, gp, E);
      if (cur < 0) break;
      cand.push_back(cur);
    }
    std::vector<size_t> idx(e.size());
    std::iota(idx.begin(), idx.end(), size_t{0});
    std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return e[a] > e[b]; });
    cur = L.g_coll;
    for (size_t i : idx) {
      cur = lcm_capped(cur, g[i], E);
      if (cur < 0) break;
      cand.push_back(cur);
    }
    std::sort(cand.begin(), cand.end());
    cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
  }
  int64_t best = -1;
  for (int64_t gg : cand) {
    const int64_t s = search(e, g, m, E, gg);
    if (best < 0 || s < best) best = s;
  }
  L.S = best;
  if (!feasible(e, g, m, best, &L.l)) {
    *err = "plan: internal error, S* infeasible";
    return false;
  }
  *out = L;
  return true;
}

bool plan_ordered(const std::vector<int64_t>& e, const std::vector<int64_t>& g, int32_t m,
                  int32_t elem_bytes, int32_t gcoll_bytes, int32_t ordering,
                  const std::vector<int64_t>* keys, Layout* out, std::string* err) {
  if (ordering == 3) {  // best of the orders
    Layout best;
    bool have = false;
    for (int32_t o = 0; o < 3; ++o) {
      if (o == 2 && !keys) continue;
      Layout L;
      if (!plan_ordered(e, g, m, elem_bytes, gcoll_bytes, o, keys, &L, err)) return false;
      if (!have || L.S < best.S) best = L, have = true;
    }
    *out = best;
    return true;
  }
  std::vector<size_t> perm(e.size());
  std::iota(perm.begin(), perm.end(), size_t{0});
  if (ordering == 1) {
    std::stable_sort(perm.begin(), perm.end(), [&](size_t a, size_t b) { return g[a] > g[b]; });
  } else if (ordering == 2) {
    if (!keys || keys->size() != e.size()) {
      *err = "plan: shape ordering needs one key per tensor";
      return false;
    }
    std::stable_sort(perm.begin(), perm.end(),
                     [&](size_t a, size_t b) { return (*keys)[a] > (*keys)[b]; });
  } else if (ordering != 0) {
    *err = "plan: unknown ordering";
    return false;
  }
  std::vector<int64_t> pe(e.size()), pg(g.size());
  for (size_t k = 0; k < perm.size(); ++k) pe[k] = e[perm[k]], pg[k] = g[perm[k]];
  Layout L;
  if (!plan(pe, pg, m, elem_bytes, gcoll_bytes, &L, err)) return false;
  Layout R = L;
  R.e = e;
  R.g = g;
  for (size_t k = 0; k < perm.size(); ++k) R.l[perm[k]] = L.l[k];
  *out = R;
  return true;
}

int64_t count_violations(const Layout& L, bool require_gcoll) {
  int64_t v = 0;
  const int64_t cap = static_cast<int64_t>(L.m) * L.S;
  if (!L.e.empty() && require_gcoll && L.S % L.g_coll != 0) ++v;
  std::vector<std::pair<int64_t, int64_t>> iv;
  for (size_t t = 0; t < L.e.size(); ++t) {
    const int64_t l = L.l[t], r = l + L.e[t];
    if (l < 0 || r > cap) ++v;
    if (L.S > 0) {
      // boundaries k*S strictly inside (l, r)
      for (int64_t k = l / L.S + 1; k * L.S < r && k <= L.m; ++k)
        if ((k * L.S - l) % L.g[t] != 0) ++v;
    }
    iv.emplace_back(l, r);
  }
  std::sort(iv.begin(), iv.end());
  for (size_t i = 1; i < iv.size(); ++i)
    if (iv[i].first < iv[i - 1].second) ++v;
  return v;
}

std::vector<std::pair<int64_t, int64_t>> padding_intervals(const Layout& L) {
  std::vector<std::pair<int64_t, int64_t>> iv, out;
  for (size_t t = 0; t < L.e.size(); ++t) iv.emplace_back(L.l[t], L.l[t] + L.e[t]);
  std::sort(iv.begin(), iv.end());
  int64_t p = 0;
  for (auto& [a, b] : iv) {
    if (a > p) out.emplace_back(p, a);
    p = std::max(p, b);
  }
  const int64_t end = static_cast<int64_t>(L.m) * L.S;
  if (p < end) out.emplace_back(p, end);
  return out;
}

std::vector<Segment> rank_segments(const Layout& L, int32_t rank) {
  std::vector<Segment> out;
  const int64_t lo = rank * L.S, hi = lo + L.S;
  for (size_t t = 0; t < L.e.size(); ++t) {
    const int64_t a = std::max(L.l[t], lo), b = std::min(L.l[t] + L.e[t], hi);
    if (a < b) out.push_back({static_cast<int32_t>(t), a - lo, b - a, a - L.l[t]});
  }
  return out;
}

bool rank_blocks(const Layout& L, int32_t rank, int64_t q, std::vector<QBlock>* out,
                 std::string* err) {
  out->clear();
  if (q < 1 || q > (int64_t{1} << 30)) {
    *err = "rank_blocks: qblock must be in [1, 2^30]";
    return false;
  }
  const int64_t lo = rank * L.S, hi = lo + L.S;
  for (size_t t = 0; t < L.e.size(); ++t) {
    const int64_t l = L.l[t], e = L.e[t];
    if (l + e <= lo || l >= hi) continue;
    // first block whose end is > lo
    int64_t j0 = l >= lo ? 0 : (lo - l) / q;
    for (int64_t j = j0; j * q < e; ++j) {
      const int64_t a = l + j * q, b = l + std::min((j + 1) * q, e);
      if (b <= lo) continue;
      if (a >= hi) break;
      if (a < lo || b > hi) {
        *err = "rank_blocks: quantization block " + std::to_string(j) + " of tensor " +
               std::to_string(t) + " straddles a shard boundary";
        return false;
      }
      out->push_back({a - lo, static_cast<int32_t>(b - a)});
    }
  }
  return true;
}

bool rank_tiles(const Layout& L, int32_t rank, const std::vector<QSpec>& specs,
                std::vector<QTile>* out, std::string* err) {
  out->clear();
  if (specs.size() != L.e.size()) {
    *err = "rank_tiles: one spec per tensor required";
    return false;
  }
  const int64_t lo = rank * L.S, hi = lo + L.S;
  for (size_t t = 0; t < L.e.size(); ++t) {
    const int64_t l = L.l[t], e = L.e[t];
    if (l + e <= lo || l >= hi) continue;
    const QSpec& q = specs[t];
    if (q.tile_rows == 0) {  // contiguous blocks
      const int64_t n = q.tile_cols;
      if (n < 1 || n > (int64_t{1} << 30)) {
        *err = "rank_tiles: flat block size must be in [1, 2^30]";
        return false;
      }
      for (int64_t j = l >= lo ? 0 : (lo - l) / n; j * n < e; ++j) {
        const int64_t a = l + j * n, b = l + std::min((j + 1) * n, e);
        if (b <= lo) continue;
        if (a >= hi) break;
        if (a < lo || b > hi) {
          *err = "rank_tiles: block " + std::to_string(j) + " of tensor " + std::to_string(t) +
                 " straddles a shard boundary";
          return false;
        }
        out->push_back({a - lo, 1, int32_t(b - a), b - a});
      }
      continue;
    }
    const int64_t C = q.row_len, tr = q.tile_rows, tc = q.tile_cols;
    if (C < 1 || tr < 1 || tc < 1 || e % C != 0 || tr * std::min<int64_t>(tc, C) > (int64_t{1} << 30)) {
      *err = "rank_tiles: invalid tile spec for tensor " + std::to_string(t);
      return false;
    }
    const int64_t Rw = e / C;
    for (int64_t i = 0; i * tr < Rw; ++i) {
      const int64_t rows = std::min(tr, Rw - i * tr);
      const int64_t row_first = l + i * tr * C;
      if (row_first + (rows - 1) * C + C <= lo) continue;  // whole tile-row below the shard
      if (row_first >= hi) break;
      for (int64_t j = 0; j * tc < C; ++j) {
        const int64_t cols = std::min(tc, C - j * tc);
        const int64_t first = row_first + j * tc, last = first + (rows - 1) * C + cols - 1;
        if (last < lo || first >= hi) continue;
        if (first < lo || last >= hi) {
          *err = "rank_tiles: tile (" + std::to_string(i) + "," + std::to_string(j) + ") of tensor " +
                 std::to_string(t) + " straddles a shard boundary";
          return false;
        }
        out->push_back({first - lo, int32_t(rows), int32_t(cols), C});
      }
    }
  }
  return true;
}

std::string to_json(const Layout& L) {
  auto arr = [](const std::vector<int64_t>& v) {
    std::string s = "[";
    for (size_t i = 0; i < v.size(); ++i) {
      if (i) s += ", ";
      s += std::to_string(v[i]);
    }
    return s + "]";
  };
  const int64_t E = L.E();
  return "{\"m\": " + std::to_string(L.m) + ", \"g_coll\": " + std::to_string(L.g_coll) +
         ", \"S\": " + std::to_string(L.S) + ", \"E\": " + std::to_string(E) +
         ", \"padding\": " + std::to_string(static_cast<int64_t>(L.m) * L.S - E) +
         ", \"numel\": " + arr(L.e) + ", \"block\": " + arr(L.g) + ", \"starts\": " + arr(L.l) +
         "}";
}

}  // namespace rsdb
