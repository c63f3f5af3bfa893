/* A plain-C client of include/rsdb.h (no Python, no torch): plans BJ config 1
 * (toy: 6 x (W[256,128], b[256]) fp32, 2048-element blocks, m = 2;
 * expected values in tests/golden/toy_config_plan.json), walks the per-rank
 * block tables, and checks the documented error behaviour.  Prints one line
 * "S <S> padding <pad> starts <l_0> ... blocks <n_0> <n_1> json <bytes>" and
 * exits 0, or prints the failure and exits 1.  Built and run by
 * tests/test_capi_host.py::test_plain_c_client. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "rsdb.h"

#define CHECK(expr)                                                                 \
  do {                                                                              \
    rsdb_status st_ = (expr);                                                       \
    if (st_ != RSDB_OK) {                                                           \
      printf("FAIL %s -> %d: %s\n", #expr, (int)st_, rsdb_last_error());          \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

int main(void) {
  enum { N = 12 };
  int64_t numel[N], block[N];
  for (int i = 0; i < 6; ++i) {
    const int64_t w_shape[2] = {256, 128}, b_shape[1] = {256};
    numel[2 * i] = 256 * 128;
    numel[2 * i + 1] = 256;
    CHECK(rsdb_block_elems(2, w_shape, RSDB_GRAN_FLAT, 2048, &block[2 * i]));
    CHECK(rsdb_block_elems(1, b_shape, RSDB_GRAN_FLAT, 2048, &block[2 * i + 1]));
  }
  rsdb_layout* lay = NULL;
  CHECK(rsdb_plan(N, numel, block, 2, 4, 16, &lay));
  int64_t viol = -1;
  CHECK(rsdb_layout_validate(lay, &viol));
  if (viol != 0) {
    printf("FAIL %lld violations\n", (long long)viol);
    return 1;
  }
  int64_t starts[N];
  CHECK(rsdb_layout_starts(lay, starts));
  printf("S %lld padding %lld starts", (long long)rsdb_layout_shard_numel(lay),
         (long long)rsdb_layout_padding(lay));
  for (int i = 0; i < N; ++i) printf(" %lld", (long long)starts[i]);
  printf(" blocks");
  for (int r = 0; r < 2; ++r) {
    int64_t n = 0;
    CHECK(rsdb_layout_rank_blocks(lay, r, 2048, &n, NULL, NULL));
    int64_t* off = malloc(sizeof(int64_t) * (size_t)n);
    int32_t* len = malloc(sizeof(int32_t) * (size_t)n);
    CHECK(rsdb_layout_rank_blocks(lay, r, 2048, &n, off, len));
    int64_t covered = 0;
    for (int64_t j = 0; j < n; ++j) {
      if (off[j] < covered || len[j] < 1 || len[j] > 2048) {
        printf("\nFAIL rank %d block %lld (%lld, %d)\n", r, (long long)j, (long long)off[j], len[j]);
        return 1;
      }
      covered = off[j] + len[j];
    }
    if (covered > rsdb_layout_shard_numel(lay)) {
      printf("\nFAIL rank %d blocks end past S\n", r);
      return 1;
    }
    printf(" %lld", (long long)n);
    free(off);
    free(len);
  }
  int64_t need = 0;
  CHECK(rsdb_layout_to_json(lay, NULL, 0, &need));
  char* js = malloc((size_t)need);
  CHECK(rsdb_layout_to_json(lay, js, need, &need));
  if (strlen(js) + 1 != (size_t)need || strstr(js, "\"S\"") == NULL) {
    printf("\nFAIL json\n");
    return 1;
  }
  printf(" json %lld\n", (long long)need);
  free(js);
  rsdb_layout_free(lay);

  /* documented errors: EINVAL for block < 1 and world < 1, with a message */
  const int64_t bad_block[1] = {0}, one[1] = {4};
  if (rsdb_plan(1, one, bad_block, 2, 4, 16, &lay) != RSDB_EINVAL || !rsdb_last_error()[0]) {
    printf("FAIL block 0 accepted\n");
    return 1;
  }
  if (rsdb_plan(1, one, one, 0, 4, 16, &lay) != RSDB_EINVAL) {
    printf("FAIL world 0 accepted\n");
    return 1;
  }
  /* n = 0 plans S = 0 */
  CHECK(rsdb_plan(0, NULL, NULL, 4, 2, 16, &lay));
  if (rsdb_layout_shard_numel(lay) != 0) {
    printf("FAIL empty plan\n");
    return 1;
  }
  rsdb_layout_free(lay);
  return 0;
}
