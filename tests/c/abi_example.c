/* A plain C caller of libmask (include/mask.h): no Python, no torch.  Builds a two-level index
 * over host-memory data, queries it, reads the level getters back and exercises an argument
 * error.  Prints C_ABI_OK (GPU present) or C_ABI_NO_GPU_OK (no usable GPU: every call that
 * needs the device must fail with MASK_ERR_CUDA, never fall back to the CPU).
 *
 *   gcc -std=c11 -I include tests/c/abi_example.c -L paper_2208_02734_b200 -lmask \
 *       -Wl,-rpath,$PWD/paper_2208_02734_b200 -o /tmp/abi_example && /tmp/abi_example
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mask.h"

#define N 5000
#define D 16
#define NQ 64
#define KNN 5

static uint64_t rng = 88172645463325252ull;
static float unif(void) { /* xorshift64 in [0, 1) */
  rng ^= rng << 13;
  rng ^= rng >> 7;
  rng ^= rng << 17;
  return (float)((rng >> 11) * (1.0 / 9007199254740992.0));
}

static int fail(const char* what, int32_t rc) {
  fprintf(stderr, "FAIL %s: rc=%d (%s)\n", what, rc, mask_last_error());
  return 1;
}

int main(void) {
  if (mask_abi_version() != MASK_ABI_VERSION) return fail("abi version", -1);
  static float X[N * D];
  for (int i = 0; i < N; ++i) { /* 20 clusters */
    const int c = i % 20;
    for (int j = 0; j < D; ++j) X[i * D + j] = (float)(c * 3 + j % 3) + unif();
  }
  int64_t k[2] = {64, 8};
  int64_t init1[64], init2[8];
  for (int i = 0; i < 64; ++i) init1[i] = (int64_t)i * 77; /* distinct rows */
  for (int i = 0; i < 8; ++i) init2[i] = (int64_t)i * 7;
  const int64_t* inits[2] = {init1, init2};
  mask_matrix m;
  memset(&m, 0, sizeof(m));
  m.format = MASK_DENSE_F32;
  m.memory = MASK_MEM_HOST;
  m.dim = D;
  m.rows = N;
  m.n_global = N;
  m.values = X;
  mask_build_params p;
  memset(&p, 0, sizeof(p));
  p.num_levels = 2;
  p.max_iters = 5;
  p.k = k;
  p.init_idx = inits;
  p.empty_policy = MASK_EMPTY_KEEP;
  mask_index* idx = NULL;
  const int32_t rc = mask_build(&m, &p, NULL, NULL, &idx);
  if (!mask_device_ok()) {
    if (rc != MASK_ERR_CUDA || idx != NULL) return fail("build without a GPU must be MASK_ERR_CUDA", rc);
    printf("C_ABI_NO_GPU_OK\n");
    return 0;
  }
  if (rc != MASK_OK) return fail("mask_build", rc);
  if (mask_num_levels(idx) != 2) return fail("mask_num_levels", mask_num_levels(idx));
  int64_t n_items, kk;
  int32_t dim, passes, updates;
  int32_t r = mask_level_info(idx, 1, &n_items, &kk, &dim, &passes, &updates);
  if (r != MASK_OK || n_items != N || kk != 64 || dim != D || passes < 1) return fail("mask_level_info", r);
  static int32_t labels[N];
  if ((r = mask_get_labels(idx, 1, labels)) != MASK_OK) return fail("mask_get_labels", r);
  for (int i = 0; i < N; ++i)
    if (labels[i] < 0 || labels[i] >= 64) return fail("label range", labels[i]);
  /* queries: the first NQ data rows, host memory in and out */
  mask_matrix q = m;
  q.rows = NQ;
  q.n_global = NQ;
  int64_t ids[NQ * KNN];
  float d2[NQ * KNN];
  if ((r = mask_query(idx, &q, KNN, 2, ids, d2, NULL)) != MASK_OK) return fail("mask_query", r);
  for (int i = 0; i < NQ; ++i) {
    for (int j = 0; j < KNN; ++j) {
      const int64_t id = ids[i * KNN + j];
      if (id < -1 || id >= N) return fail("query id range", (int32_t)id);
      if (id >= 0) { /* the reported d^2 is the distance to that row */
        double s = 0.0;
        for (int c = 0; c < D; ++c) {
          const double t = (double)X[i * D + c] - (double)X[id * D + c];
          s += t * t;
        }
        if (fabs(s - d2[i * KNN + j]) > 1e-4 * (s + 1e-3)) return fail("query d2", i);
      }
      if (j > 0 && d2[i * KNN + j] < d2[i * KNN + j - 1]) return fail("query order", i);
    }
  }
  /* argument errors are reported, never truncated */
  if (mask_query(idx, &q, 0, 1, ids, d2, NULL) != MASK_ERR_ARG || mask_last_error()[0] == '\0')
    return fail("k_nn = 0 must be MASK_ERR_ARG", 0);
  mask_free(idx);
  mask_free(NULL);
  printf("C_ABI_OK\n");
  return 0;
}
