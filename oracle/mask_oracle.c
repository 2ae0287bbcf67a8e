/*
 * mask_oracle.c -- plain, slow, obviously-correct FP64 CPU oracle for the MASK hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2208_02734_b200/csrc) and
 * neither side includes or links the other.
 *
 * Citations: "P:n" = line n of the paper text (PAPER.md, arXiv 2208.02734, MASK);
 * "D#" = the numbered readings in DESIGN.md (the paper is silent on them).
 *
 * What is computed (and in which order) follows the paper's algorithms literally:
 *   - distance: Euclidean, squared (P:897 `euclideanDistance`, "Euclidean
 *     distance"; ranking by d^2 is ranking by d, D9), evaluated directly as
 *     sum_i (y_i - c_i)^2 in FP64;
 *   - k-means: Lloyd iterations (P:654-655 `kmeans(nCentroids, points)`,
 *     `kmeans.labels`; Lloyd cited P:176/P:293): assignment to the nearest
 *     prototype (`searchPosMin`; ties -> lowest ordinal, D4) then every
 *     prototype becomes the mean of its members (P:536 centroids minimise the sum
 *     of squared distances); an empty cluster keeps its prototype (D5), or -- the
 *     SPEC option S:128 -- is re-seeded at the farthest row of the pass (D5b);
 *   - levels: the prototypes of level l are the points clustered at level l+1
 *     (Algorithm 1), one global k-means per level (D1);
 *   - query: descend from the top level choosing the nearest child(ren) of the
 *     previously selected prototype(s) (Algorithm 2; beam b,
 *     b = 1 is Algorithm 2, D7), then rank the reached data partition and return
 *     the k lowest (`searchKNN` P:912), ties by (d^2, id) (D4), padded
 *     with (-1, +inf) when the partition holds fewer than k points (D8);
 *   - exact k-NN: "the k closest elements to q" by brute force.
 *
 * Sparse rows (CSR) use the identity ||y - c||^2 = ||c||^2 + sum_{j in nz(y)} (y_j^2
 * - 2 y_j c_j) (D12), with ||c||^2 summed directly; it is pinned against the
 * densified direct form by tests/test_oracle.py.
 *
 * No blocking, fusion or reordering: each distance is a plain loop, each mean a
 * plain ascending-i sum followed by one division.  OpenMP only splits independent
 * rows/queries across threads (each result is computed by one thread in the same
 * order as the sequential code).
 */
#include <math.h>
#include <stdint.h>

enum { ORC_EMPTY_KEEP = 0, ORC_EMPTY_FARTHEST = 1 };
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* threads of the later parallel loops (timing the single-core rate of the CPU baseline) */
void orc_set_num_threads(int t) {
#ifdef _OPENMP
  if (t >= 1) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

/* ------------------------------------------------------------------ distances */

/* Squared Euclidean distance, direct form (D9). */
double orc_dist2(int d, const double* y, const double* c) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) {
    double t = y[i] - c[i];
    s += t * t;
  }
  return s;
}

/* Squared Euclidean distance between a CSR row and a dense vector (D12):
 * ||c||^2 + sum_{j in nz(y)} (y_j^2 - 2 y_j c_j).  cn2 = ||c||^2. */
double orc_dist2_csr_dense(int64_t nnz, const int32_t* col, const double* val,
                           const double* c, double cn2) {
  double s = cn2;
  for (int64_t p = 0; p < nnz; ++p) {
    double y = val[p];
    s += y * y - 2.0 * y * c[col[p]];
  }
  return s;
}

/* Squared Euclidean distance between two CSR rows (sorted column lists):
 * sum over the union of their supports of (a_j - b_j)^2. */
double orc_dist2_csr_csr(int64_t na, const int32_t* ca, const double* va,
                         int64_t nb, const int32_t* cb, const double* vb) {
  double s = 0.0;
  int64_t i = 0, j = 0;
  while (i < na || j < nb) {
    double t;
    if (j >= nb || (i < na && ca[i] < cb[j])) {
      t = va[i++];
    } else if (i >= na || cb[j] < ca[i]) {
      t = vb[j++];
    } else {
      t = va[i++] - vb[j++];
    }
    s += t * t;
  }
  return s;
}

static double sqnorm(int d, const double* c) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += c[i] * c[i];
  return s;
}

/* ------------------------------------------------------------------ assignment */

/* a_i = argmin_j dist(Y_i, P_j), ties -> lowest j (D4).
 * best[i] = the minimum distance, second[i] = the second smallest over j != a_i
 * (+inf when k == 1); either output pointer may be NULL. */
void orc_assign(int64_t n, int d, const double* Y, int64_t k, const double* P,
                int32_t* labels, double* best, double* second) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double* y = Y + i * (int64_t)d;
    double b1 = INFINITY, b2 = INFINITY;
    int64_t a = -1;
    for (int64_t j = 0; j < k; ++j) {
      double t = orc_dist2(d, y, P + j * (int64_t)d);
      if (t < b1) {
        b2 = b1;
        b1 = t;
        a = j;
      } else if (t < b2) {
        b2 = t;
      }
    }
    labels[i] = (int32_t)a;
    if (best) best[i] = b1;
    if (second) second[i] = b2;
  }
}

/* CSR rows against dense prototypes (D12). */
void orc_assign_csr(int64_t n, int d, const int64_t* row_ptr, const int32_t* col,
                    const double* val, int64_t k, const double* P, int32_t* labels,
                    double* best, double* second) {
  double* cn2 = (double*)malloc(sizeof(double) * (size_t)(k > 0 ? k : 1));
  for (int64_t j = 0; j < k; ++j) cn2[j] = sqnorm(d, P + j * (int64_t)d);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < n; ++i) {
    int64_t p0 = row_ptr[i], nz = row_ptr[i + 1] - row_ptr[i];
    double b1 = INFINITY, b2 = INFINITY;
    int64_t a = -1;
    for (int64_t j = 0; j < k; ++j) {
      double t = orc_dist2_csr_dense(nz, col + p0, val + p0, P + j * (int64_t)d, cn2[j]);
      if (t < b1) {
        b2 = b1;
        b1 = t;
        a = j;
      } else if (t < b2) {
        b2 = t;
      }
    }
    labels[i] = (int32_t)a;
    if (best) best[i] = b1;
    if (second) second[i] = b2;
  }
  free(cn2);
}

/* ------------------------------------------------------------------ update */

/* S_j = sum_{a_i = j} Y_i (ascending i), n_j = |{i : a_i = j}|. */
void orc_cluster_sums(int64_t n, int d, const double* Y, const int32_t* labels, int64_t k,
                      double* S, int64_t* counts) {
  memset(S, 0, sizeof(double) * (size_t)(k * d));
  memset(counts, 0, sizeof(int64_t) * (size_t)k);
  for (int64_t i = 0; i < n; ++i) {
    int64_t j = labels[i];
    counts[j] += 1;
    for (int c = 0; c < d; ++c) S[j * d + c] += Y[i * (int64_t)d + c];
  }
}

void orc_cluster_sums_csr(int64_t n, int d, const int64_t* row_ptr, const int32_t* col,
                          const double* val, const int32_t* labels, int64_t k, double* S,
                          int64_t* counts) {
  memset(S, 0, sizeof(double) * (size_t)(k * d));
  memset(counts, 0, sizeof(int64_t) * (size_t)k);
  for (int64_t i = 0; i < n; ++i) {
    int64_t j = labels[i];
    counts[j] += 1;
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) S[j * d + col[p]] += val[p];
  }
}

/* P_new_j = S_j / n_j if n_j > 0, else P_old_j (D5).  Returns max_j ||P_new_j - P_old_j||. */
double orc_means_from_sums(int64_t k, int d, const double* S, const int64_t* counts,
                           const double* P_old, double* P_new) {
  double maxdisp = 0.0;
  for (int64_t j = 0; j < k; ++j) {
    for (int c = 0; c < d; ++c) {
      P_new[j * d + c] = counts[j] > 0 ? S[j * d + c] / (double)counts[j] : P_old[j * d + c];
    }
    double disp = sqrt(orc_dist2(d, P_new + j * d, P_old + j * d));
    if (disp > maxdisp) maxdisp = disp;
  }
  return maxdisp;
}

/* ------------------------------------------------------------------ Lloyd */

/* Empty-cluster repair, SPEC S:128 ("an emptied centroid is re-seeded at the point with the
 * largest distance to its current centroid"; reading D5b): the m prototypes that
 * this update leaves without members, taken in ascending j, are set to the m rows with the
 * largest dist(Y_i, P_t[a_i]) of the pass (best[i]), ordered by (distance descending, i
 * ascending), one row each; every other prototype keeps its member mean.  Returns the
 * largest displacement of a re-seeded prototype (for the tolerance stop, D3). */
typedef struct {
  double d2;
  int64_t i;
} far_t;

static int far_cmp(const void* pa, const void* pb) {
  const far_t* a = (const far_t*)pa;
  const far_t* b = (const far_t*)pb;
  if (a->d2 > b->d2) return -1; /* larger distance first */
  if (a->d2 < b->d2) return 1;
  return (a->i > b->i) - (a->i < b->i); /* then lower row index */
}

static double reseed_farthest(int64_t n, int d, const double* Y, const int64_t* row_ptr,
                              const int32_t* col, const double* val, int64_t k,
                              const int64_t* counts, const double* best, const double* P_old,
                              double* P_new) {
  int64_t m = 0;
  for (int64_t j = 0; j < k; ++j) m += counts[j] == 0;
  if (m == 0 || n == 0) return 0.0;
  far_t* order = (far_t*)malloc(sizeof(far_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    order[i].d2 = best[i];
    order[i].i = i;
  }
  qsort(order, (size_t)n, sizeof(far_t), far_cmp);
  double maxdisp = 0.0;
  int64_t r = 0;
  for (int64_t j = 0; j < k && r < n; ++j) {
    if (counts[j] != 0) continue;
    const int64_t row = order[r++].i;
    double* c = P_new + j * d;
    if (Y) {
      memcpy(c, Y + row * (int64_t)d, sizeof(double) * (size_t)d);
    } else {
      memset(c, 0, sizeof(double) * (size_t)d);
      for (int64_t p = row_ptr[row]; p < row_ptr[row + 1]; ++p) c[col[p]] = val[p];
    }
    double disp = sqrt(orc_dist2(d, c, P_old + j * d));
    if (disp > maxdisp) maxdisp = disp;
  }
  free(order);
  return maxdisp;
}

/* One level of the index: Lloyd k-means from the seeded init rows (D2), following the
 * pseudo-code of DESIGN.md "Oracle" step by step:
 *
 *   P <- Y[init_idx]
 *   for t = 0 .. T-1:
 *       a <- assign(Y, P);  J_t <- sum_i dist(Y_i, P_{a_i})
 *       if t > 0 and a == prev: break          (update would be a no-op)
 *       P <- means(Y, a), empty keeps P_j      (D5)
 *       prev <- a
 *       if tol > 0 and max_j ||dP_j|| <= tol: break   (D3)
 *   labels <- assign(Y, P)                       (final pass, D3)
 *
 * Y is either dense (Y != NULL) or CSR (row_ptr/col/val).  J_trace/changed_trace receive
 * one entry per assignment pass including the final one (capacity T+1).  Returns the number
 * of assignment passes recorded; *updates_run = number of prototype updates performed. */
static int lloyd_impl(int64_t n, int d, const double* Y, const int64_t* row_ptr,
                      const int32_t* col, const double* val, int64_t k,
                      const int64_t* init_idx, int T, double tol, double* P_out,
                      int32_t* labels_out, double* J_trace, int64_t* changed_trace,
                      int* updates_run, double* P_pass, int32_t* lab_pass, int empty_policy) {
  double* P = P_out;
  double* P_new = (double*)malloc(sizeof(double) * (size_t)(k * d));
  double* S = (double*)malloc(sizeof(double) * (size_t)(k * d));
  int64_t* counts = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  int32_t* a = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int32_t* prev = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  double* best = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  int passes = 0, updates = 0;

  /* P <- Y[init_idx] (densify CSR rows) */
  for (int64_t j = 0; j < k; ++j) {
    int64_t r = init_idx[j];
    if (Y) {
      memcpy(P + j * d, Y + r * (int64_t)d, sizeof(double) * (size_t)d);
    } else {
      memset(P + j * d, 0, sizeof(double) * (size_t)d);
      for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) P[j * d + col[p]] = val[p];
    }
  }

  for (int t = 0; t < T; ++t) {
    if (Y) orc_assign(n, d, Y, k, P, a, best, NULL);
    else orc_assign_csr(n, d, row_ptr, col, val, k, P, a, best, NULL);
    /* optional per-pass record (output only): the prototypes this pass used, its labels */
    if (P_pass) memcpy(P_pass + (size_t)passes * (size_t)(k * d), P, sizeof(double) * (size_t)(k * d));
    if (lab_pass) memcpy(lab_pass + (size_t)passes * (size_t)n, a, sizeof(int32_t) * (size_t)n);
    double J = 0.0;
    int64_t changed = 0;
    for (int64_t i = 0; i < n; ++i) {
      J += best[i];
      if (t == 0 || a[i] != prev[i]) ++changed;
    }
    if (J_trace) J_trace[passes] = J;
    if (changed_trace) changed_trace[passes] = changed;
    ++passes;
    if (t > 0 && changed == 0) break;
    if (Y) orc_cluster_sums(n, d, Y, a, k, S, counts);
    else orc_cluster_sums_csr(n, d, row_ptr, col, val, a, k, S, counts);
    double maxdisp = orc_means_from_sums(k, d, S, counts, P, P_new);
    if (empty_policy == ORC_EMPTY_FARTHEST) {
      double rd = reseed_farthest(n, d, Y, row_ptr, col, val, k, counts, best, P, P_new);
      if (rd > maxdisp) maxdisp = rd;
    }
    memcpy(P, P_new, sizeof(double) * (size_t)(k * d));
    ++updates;
    memcpy(prev, a, sizeof(int32_t) * (size_t)n);
    if (tol > 0.0 && maxdisp <= tol) break;
  }

  /* final assignment with the final prototypes */
  if (Y) orc_assign(n, d, Y, k, P, labels_out, best, NULL);
  else orc_assign_csr(n, d, row_ptr, col, val, k, P, labels_out, best, NULL);
  if (P_pass) memcpy(P_pass + (size_t)passes * (size_t)(k * d), P, sizeof(double) * (size_t)(k * d));
  if (lab_pass) memcpy(lab_pass + (size_t)passes * (size_t)n, labels_out, sizeof(int32_t) * (size_t)n);
  {
    double J = 0.0;
    int64_t changed = 0;
    for (int64_t i = 0; i < n; ++i) {
      J += best[i];
      if (updates == 0 || labels_out[i] != prev[i]) ++changed;
    }
    if (J_trace) J_trace[passes] = J;
    if (changed_trace) changed_trace[passes] = changed;
    ++passes;
  }
  if (updates_run) *updates_run = updates;
  free(P_new);
  free(S);
  free(counts);
  free(a);
  free(prev);
  free(best);
  return passes;
}

int orc_lloyd(int64_t n, int d, const double* Y, int64_t k, const int64_t* init_idx, int T,
              double tol, double* P_out, int32_t* labels_out, double* J_trace,
              int64_t* changed_trace, int* updates_run) {
  return lloyd_impl(n, d, Y, NULL, NULL, NULL, k, init_idx, T, tol, P_out, labels_out, J_trace,
                    changed_trace, updates_run, NULL, NULL, ORC_EMPTY_KEEP);
}

/* orc_lloyd / orc_lloyd_csr with a per-pass record: P_pass ((T+1) x k x d) receives the
 * prototypes each assignment pass used, lab_pass ((T+1) x n) the labels it produced (pass
 * index = position in J_trace; the final assignment is the last one).  Either may be NULL. */
int orc_lloyd_trace(int64_t n, int d, const double* Y, const int64_t* row_ptr, const int32_t* col,
                    const double* val, int64_t k, const int64_t* init_idx, int T, double tol,
                    double* P_out, int32_t* labels_out, double* J_trace, int64_t* changed_trace,
                    int* updates_run, double* P_pass, int32_t* lab_pass) {
  return lloyd_impl(n, d, Y, row_ptr, col, val, k, init_idx, T, tol, P_out, labels_out, J_trace,
                    changed_trace, updates_run, P_pass, lab_pass, ORC_EMPTY_KEEP);
}

/* orc_lloyd_trace with an empty-cluster policy (ORC_EMPTY_KEEP = 0: D5; ORC_EMPTY_FARTHEST = 1:
 * D5b).  Y dense or (row_ptr, col, val) CSR; P_pass / lab_pass may be NULL. */
int orc_lloyd_ex(int64_t n, int d, const double* Y, const int64_t* row_ptr, const int32_t* col,
                 const double* val, int64_t k, const int64_t* init_idx, int T, double tol,
                 double* P_out, int32_t* labels_out, double* J_trace, int64_t* changed_trace,
                 int* updates_run, double* P_pass, int32_t* lab_pass, int empty_policy) {
  return lloyd_impl(n, d, Y, row_ptr, col, val, k, init_idx, T, tol, P_out, labels_out, J_trace,
                    changed_trace, updates_run, P_pass, lab_pass, empty_policy);
}

int orc_lloyd_csr(int64_t n, int d, const int64_t* row_ptr, const int32_t* col,
                  const double* val, int64_t k, const int64_t* init_idx, int T, double tol,
                  double* P_out, int32_t* labels_out, double* J_trace, int64_t* changed_trace,
                  int* updates_run) {
  return lloyd_impl(n, d, NULL, row_ptr, col, val, k, init_idx, T, tol, P_out, labels_out,
                    J_trace, changed_trace, updates_run, NULL, NULL, ORC_EMPTY_KEEP);
}

/* ------------------------------------------------------------------ query */

typedef struct {
  double d2;
  int64_t id;
} cand_t;

static int cand_cmp(const void* pa, const void* pb) {
  const cand_t* a = (const cand_t*)pa;
  const cand_t* b = (const cand_t*)pb;
  if (a->d2 < b->d2) return -1;
  if (a->d2 > b->d2) return 1;
  return (a->id > b->id) - (a->id < b->id);
}

/* relative gap between two ordered distances (0 when both are 0) */
static double rel_gap(double lo, double hi) {
  if (hi <= 0.0) return 0.0;
  return (hi - lo) / hi;
}

/* Multilevel descent (Algorithm 2) with explicit child lists (D7).
 *
 * Levels are 1..L (level 1 = prototypes over the data).  For level l (0-based array slot
 * l-1): P[l-1] is k_l x d, offsets[l-1] has k_l+1 entries and members[l-1] lists the items
 * of level l-1 (data rows for l = 1) assigned to each prototype of level l.
 *
 *   S <- top-b of { j < k_L : children_L(j) != {} } by (dist(q, P_L[j]), j)
 *   for l = L-1 .. 1:  C <- union of children_{l+1}(p), p in S
 *                      S <- top-b of { j in C : children_l(j) != {} } by (dist, j)
 *   leaf <- union of children_1(p), p in S
 *   result <- first knn of leaf sorted by (dist(q, X_i), i); pad (-1, +inf)   (D8)
 *
 * Data X is dense (X != NULL, n x d) or CSR (xrp/xcol/xval); queries likewise (Q or
 * qrp/qcol/qval).  min_gap[q] (optional) = the smallest relative gap between the last
 * kept and the first dropped candidate over every selection this query made (the
 * tie-window exemption of the parity tests). */
void orc_query(int L, const int64_t* k_per_level, const double* const* P,
               const int64_t* const* offsets, const int64_t* const* members, int d,
               const double* X, const int64_t* xrp, const int32_t* xcol, const double* xval,
               int64_t nq, const double* Q, const int64_t* qrp, const int32_t* qcol,
               const double* qval, int knn, int beam, int64_t* ids_out, double* d2_out,
               double* min_gap) {
  /* ||c||^2 per level for the sparse-query formula */
  double** cn2 = (double**)calloc((size_t)L, sizeof(double*));
  if (Q == NULL) {
    for (int l = 0; l < L; ++l) {
      cn2[l] = (double*)malloc(sizeof(double) * (size_t)k_per_level[l]);
      for (int64_t j = 0; j < k_per_level[l]; ++j) cn2[l][j] = sqnorm(d, P[l] + j * d);
    }
  }
  int64_t maxk = 0;
  for (int l = 0; l < L; ++l) maxk = k_per_level[l] > maxk ? k_per_level[l] : maxk;

#pragma omp parallel
  {
    int64_t cap = maxk + 16;
    cand_t* cand = (cand_t*)malloc(sizeof(cand_t) * (size_t)cap);
    int64_t* sel = (int64_t*)malloc(sizeof(int64_t) * (size_t)(beam > 0 ? beam : 1));
#pragma omp for schedule(dynamic, 16)
    for (int64_t qi = 0; qi < nq; ++qi) {
      const double* q = Q ? Q + qi * (int64_t)d : NULL;
      int64_t q0 = Q ? 0 : qrp[qi], qn = Q ? 0 : qrp[qi + 1] - qrp[qi];
      double gap = INFINITY;
      int64_t nsel = 0;
      /* top level: every prototype with children */
      {
        int l = L - 1;
        int64_t nc = 0;
        for (int64_t j = 0; j < k_per_level[l]; ++j) {
          if (offsets[l][j + 1] == offsets[l][j]) continue; /* childless: skipped */
          double t = q ? orc_dist2(d, q, P[l] + j * d)
                       : orc_dist2_csr_dense(qn, qcol + q0, qval + q0, P[l] + j * d, cn2[l][j]);
          cand[nc].d2 = t;
          cand[nc].id = j;
          ++nc;
        }
        qsort(cand, (size_t)nc, sizeof(cand_t), cand_cmp);
        nsel = nc < beam ? nc : beam;
        if (nc > nsel) {
          double g = rel_gap(cand[nsel - 1].d2, cand[nsel].d2);
          if (g < gap) gap = g;
        }
        for (int64_t s = 0; s < nsel; ++s) sel[s] = cand[s].id;
      }
      /* levels L-1 .. 1 */
      for (int l = L - 2; l >= 0; --l) {
        int64_t nc = 0;
        for (int64_t s = 0; s < nsel; ++s) {
          int64_t p = sel[s];
          for (int64_t m = offsets[l + 1][p]; m < offsets[l + 1][p + 1]; ++m) {
            int64_t j = members[l + 1][m];
            if (offsets[l][j + 1] == offsets[l][j]) continue;
            double t = q ? orc_dist2(d, q, P[l] + j * d)
                         : orc_dist2_csr_dense(qn, qcol + q0, qval + q0, P[l] + j * d, cn2[l][j]);
            if (nc >= cap) {
              cap *= 2;
              cand = (cand_t*)realloc(cand, sizeof(cand_t) * (size_t)cap);
            }
            cand[nc].d2 = t;
            cand[nc].id = j;
            ++nc;
          }
        }
        qsort(cand, (size_t)nc, sizeof(cand_t), cand_cmp);
        nsel = nc < beam ? nc : beam;
        if (nc > nsel && nsel > 0) {
          double g = rel_gap(cand[nsel - 1].d2, cand[nsel].d2);
          if (g < gap) gap = g;
        }
        for (int64_t s = 0; s < nsel; ++s) sel[s] = cand[s].id;
      }
      /* data layer: rank the reached partition(s) */
      int64_t nc = 0;
      for (int64_t s = 0; s < nsel; ++s) {
        int64_t p = sel[s];
        for (int64_t m = offsets[0][p]; m < offsets[0][p + 1]; ++m) {
          int64_t i = members[0][m];
          double t;
          if (X && q) t = orc_dist2(d, q, X + i * (int64_t)d);
          else if (!X && !q)
            t = orc_dist2_csr_csr(qn, qcol + q0, qval + q0, xrp[i + 1] - xrp[i], xcol + xrp[i],
                                  xval + xrp[i]);
          else if (X && !q) {
            /* sparse query vs dense row: sum over all coordinates */
            double s2 = 0.0;
            int64_t pq = 0;
            for (int c = 0; c < d; ++c) {
              double qv = 0.0;
              if (pq < qn && qcol[q0 + pq] == c) qv = qval[q0 + pq++];
              double tt = qv - X[i * (int64_t)d + c];
              s2 += tt * tt;
            }
            t = s2;
          } else {
            /* dense query vs sparse row */
            double s2 = 0.0;
            int64_t px = xrp[i], pe = xrp[i + 1];
            for (int c = 0; c < d; ++c) {
              double xv = 0.0;
              if (px < pe && xcol[px] == c) xv = xval[px++];
              double tt = q[c] - xv;
              s2 += tt * tt;
            }
            t = s2;
          }
          if (nc >= cap) {
            cap *= 2;
            cand = (cand_t*)realloc(cand, sizeof(cand_t) * (size_t)cap);
          }
          cand[nc].d2 = t;
          cand[nc].id = i;
          ++nc;
        }
      }
      qsort(cand, (size_t)nc, sizeof(cand_t), cand_cmp);
      if (nc > knn && knn > 0) {
        double g = rel_gap(cand[knn - 1].d2, cand[knn].d2);
        if (g < gap) gap = g;
      }
      for (int r = 0; r < knn; ++r) {
        ids_out[qi * knn + r] = r < nc ? cand[r].id : -1;
        d2_out[qi * knn + r] = r < nc ? cand[r].d2 : INFINITY;
      }
      if (min_gap) min_gap[qi] = gap;
    }
    free(cand);
    free(sel);
  }
  for (int l = 0; l < L; ++l) free(cn2[l]);
  free(cn2);
}

/* Exact k-NN by brute force: first knn of all points by (dist, id).
 * kth_gap[q] (optional) = relative gap between the knn-th and (knn+1)-th distances. */
void orc_knn_exact(int64_t n, int d, const double* X, const int64_t* xrp, const int32_t* xcol,
                   const double* xval, int64_t nq, const double* Q, const int64_t* qrp,
                   const int32_t* qcol, const double* qval, int knn, int64_t* ids_out,
                   double* d2_out, double* kth_gap) {
#pragma omp parallel
  {
    cand_t* cand = (cand_t*)malloc(sizeof(cand_t) * (size_t)(n > 0 ? n : 1));
#pragma omp for schedule(dynamic, 4)
    for (int64_t qi = 0; qi < nq; ++qi) {
      for (int64_t i = 0; i < n; ++i) {
        double t;
        if (X && Q) {
          t = orc_dist2(d, Q + qi * (int64_t)d, X + i * (int64_t)d);
        } else if (!X && !Q) {
          t = orc_dist2_csr_csr(qrp[qi + 1] - qrp[qi], qcol + qrp[qi], qval + qrp[qi],
                                xrp[i + 1] - xrp[i], xcol + xrp[i], xval + xrp[i]);
        } else {
          t = NAN; /* mixed formats are not used by the harness */
        }
        cand[i].d2 = t;
        cand[i].id = i;
      }
      qsort(cand, (size_t)n, sizeof(cand_t), cand_cmp);
      for (int r = 0; r < knn; ++r) {
        ids_out[qi * knn + r] = r < n ? cand[r].id : -1;
        d2_out[qi * knn + r] = r < n ? cand[r].d2 : INFINITY;
      }
      if (kth_gap) kth_gap[qi] = (n > knn && knn > 0) ? rel_gap(cand[knn - 1].d2, cand[knn].d2) : INFINITY;
    }
    free(cand);
  }
}
