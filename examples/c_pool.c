/* The recycling unified allocator from plain C (include/ut.h ut_pool_*).
 *
 *   c_pool system    bookkeeping on the malloc backend (no GPU needed)
 *   c_pool managed   two unified tables of the same size, one after the other, over one
 *                    recycled block; each gathers 1000 rows, checked against a memcpy loop
 *   c_pool pinned    the same on cudaHostAlloc blocks
 * Prints "C-POOL OK" on success. */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ut.h"

#define CHECK(c)                                                                  \
  do {                                                                            \
    if (!(c)) {                                                                   \
      char m[512];                                                                \
      ut_last_error(m, sizeof m);                                                 \
      fprintf(stderr, "%s:%d: %s failed (%s)\n", __FILE__, __LINE__, #c, m);      \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

static int bookkeeping(ut_pool* p) {
  void *a, *b, *z;
  uint64_t cap;
  ut_pool_stats st;
  CHECK(ut_pool_alloc(p, 1000, &a, &cap) == UT_OK && cap == 1024);
  CHECK(ut_pool_alloc(p, 0, &z, &cap) == UT_OK && z == NULL && cap == 0);
  CHECK(ut_pool_free(p, a) == UT_OK);
  CHECK(ut_pool_free(p, a) == UT_EINVAL);                 /* double free */
  CHECK(ut_pool_alloc(p, 900, &b, &cap) == UT_OK && b == a);
  CHECK(ut_pool_get_stats(p, &st) == UT_OK);
  CHECK(st.backend_calls == 1 && st.recycled_hits == 1 && st.bytes_live == 1024);
  CHECK(ut_pool_destroy(p) == UT_EINVAL);                 /* a live block */
  CHECK(ut_pool_free(p, b) == UT_OK);
  return 0;
}

static int tables(ut_pool* p) {
  const uint64_t rows = 5000, rb = 400, n = 1000;
  void* host[2];
  int64_t* idx_h = malloc(n * sizeof *idx_h);
  uint8_t* out_h = malloc(n * rb);
  int64_t* idx_d;
  uint8_t* out_d;
  CHECK(idx_h && out_h);
  CHECK(cudaMalloc((void**)&idx_d, n * sizeof *idx_d) == cudaSuccess);
  CHECK(cudaMalloc((void**)&out_d, n * rb) == cudaSuccess);
  for (int k = 0; k < 2; ++k) {
    ut_table* t = ut_pool_table(p, NULL, rows, rb, &host[k]);   /* same 512-B bucket */
    CHECK(t);
    uint8_t* tab = host[k];
    for (uint64_t i = 0; i < rows * rb; ++i) tab[i] = (uint8_t)(i * 2654435761u >> 13) + k;
    for (uint64_t i = 0; i < n; ++i) idx_h[i] = (int64_t)((i * 7919 + 13 * k) % rows);
    CHECK(cudaMemcpy(idx_d, idx_h, n * sizeof *idx_d, cudaMemcpyHostToDevice) == cudaSuccess);
    CHECK(ut_gather(t, idx_d, n, out_d, NULL) == UT_OK);
    CHECK(cudaMemcpy(out_h, out_d, n * rb, cudaMemcpyDeviceToHost) == cudaSuccess);
    for (uint64_t i = 0; i < n; ++i) CHECK(!memcmp(out_h + i * rb, tab + idx_h[i] * rb, rb));
    CHECK(ut_release(t) == UT_OK);                          /* the block goes back to p */
  }
  ut_pool_stats st;
  CHECK(ut_pool_get_stats(p, &st) == UT_OK);
  CHECK(host[0] == host[1] && st.backend_calls == 1 && st.recycled_hits == 1);
  cudaFree(idx_d);
  cudaFree(out_d);
  free(idx_h);
  free(out_h);
  return 0;
}

int main(int argc, char** argv) {
  const char* kind = argc > 1 ? argv[1] : "system";
  int k = !strcmp(kind, "managed") ? UT_ALLOC_MANAGED : !strcmp(kind, "pinned") ? UT_ALLOC_PINNED
                                                                                  : UT_ALLOC_SYSTEM;
  ut_pool* p = ut_pool_create(k, 0);
  CHECK(p);
  if (k == UT_ALLOC_SYSTEM) {
    if (bookkeeping(p)) return 1;
  } else if (tables(p)) {
    return 1;
  }
  CHECK(ut_pool_release_cached(p) == UT_OK);
  CHECK(ut_pool_destroy(p) == UT_OK);
  printf("C-POOL OK (%s)\n", kind);
  return 0;
}
