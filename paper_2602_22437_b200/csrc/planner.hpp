// Host layout planner for grouped RaggedShard tensors (PAPER §5).
// Problem P:212-232; Algorithm 1; case analysis P:287.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace rsdb {

struct Layout {
  int32_t m = 1;            // devices
  int32_t elem_bytes = 2;   // one dtype per unit
  int64_t g_coll = 8;       // collective unit (elements)
  int64_t S = 0;            // per-device shard size (elements)
  std::vector<int64_t> e;   // e_t
  std::vector<int64_t> g;   // g_t
  std::vector<int64_t> l;   // l_t
  int64_t E() const;
};

struct Segment {
  int32_t tensor;
  int64_t local_off, len, tensor_off;
};
struct QBlock {
  int64_t off;
  int32_t len;
};

// a1
bool block_elems(int32_t ndim, const int64_t* shape, int32_t kind, int64_t param, int64_t* g,
                 std::string* err);
// a2: returns false (with err) only on invalid input.
bool plan(const std::vector<int64_t>& e, const std::vector<int64_t>& g, int32_t m,
          int32_t elem_bytes, int32_t gcoll_bytes, Layout* out, std::string* err);
// Tensor orders of P:279: 0 default, 1 by sharding block size (desc, stable),
// 2 by caller shape key (desc, stable), 3 best of the three (smallest S,
// ties to the earlier order).  Starts are reported in input order.
bool plan_ordered(const std::vector<int64_t>& e, const std::vector<int64_t>& g, int32_t m,
                  int32_t elem_bytes, int32_t gcoll_bytes, int32_t ordering,
                  const std::vector<int64_t>* keys, Layout* out, std::string* err);
// CheckValidShard at one S (leftmost placement); starts filled when feasible.
bool feasible(const std::vector<int64_t>& e, const std::vector<int64_t>& g, int32_t m, int64_t S,
              std::vector<int64_t>* starts);
int64_t count_violations(const Layout& L, bool require_gcoll);
std::vector<std::pair<int64_t, int64_t>> padding_intervals(const Layout& L);
// a3
std::vector<Segment> rank_segments(const Layout& L, int32_t rank);
bool rank_blocks(const Layout& L, int32_t rank, int64_t q, std::vector<QBlock>* out,
                 std::string* err);

// Quantization block spec per tensor: tile_rows == 0 ->
// contiguous blocks of tile_cols elements; else tile_rows x tile_cols tiles of
// the [e / row_len, row_len] view (edge tiles smaller).
struct QSpec {
  int64_t row_len;
  int32_t tile_rows;
  int32_t tile_cols;
};
struct QTile {
  int64_t off;    // first element, offset inside the shard
  int32_t rows, cols;
  int64_t pitch;  // elements between rows
};
bool rank_tiles(const Layout& L, int32_t rank, const std::vector<QSpec>& specs,
                std::vector<QTile>* out, std::string* err);
std::string to_json(const Layout& L);

}  // namespace rsdb
