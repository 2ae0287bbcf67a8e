/*
 * mask.h -- C-ABI of libmask.so, the B200 (sm_100a) hot path of MASK
 * ("Multilevel Approximate Similarity search with k-means", arXiv 2208.02734).
 *
 * Citations: "P:n" = line n of the paper text; "D#" = a reading of the paper
 * recorded in DESIGN.md (the paper is silent/ambiguous there).
 *
 * Problem statement implemented:
 *   - a dataset X of n feature vectors in R^dim under the Euclidean distance;
 *   - a multilevel index: level 1 clusters X into k[0] prototypes with Lloyd k-means
 *     (P:654-655), level l+1 clusters the k[l-1] prototypes of level l into k[l]
 *     (P:634-637), one global k-means per level (D1), seeded random-point initialisation
 *     (D2), T Lloyd iterations or a tolerance, then a final assignment (D3);
 *   - batched approximate k-NN: descend from the top level through the children of the
 *     selected prototype(s) and rank the reached data partition (Algorithm 2).
 *
 * Conventions shared by every entry point:
 *   - every function returns a mask_status (0 = OK, < 0 = error) unless noted; on error
 *     mask_last_error() returns a thread-local human-readable message;
 *   - "device" pointers are CUDA global-memory pointers on the caller's current device;
 *     "host" pointers are ordinary (preferably pinned) host memory.  mask_matrix.memory
 *     says which one its arrays are;
 *   - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).  All
 *     work is enqueued on it and every call returns only after the stream has completed the
 *     call's work, so device faults surface as MASK_ERR_CUDA from the same call;
 *   - all input pointers are borrowed for the duration of the call only, except with
 *     MASK_BORROW_DATA (see mask_build);
 *   - the library never falls back to the CPU: every arithmetic step runs in its CUDA
 *     kernels; a missing GPU is MASK_ERR_CUDA.
 */
#ifndef MASK_H_
#define MASK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MASK_ABI_VERSION 1

typedef enum {
  MASK_OK = 0,
  MASK_ERR_ARG = -1,         /* invalid argument / shape / inconsistent CSR               */
  MASK_ERR_NONFINITE = -2,   /* NaN/Inf input (only checked with MASK_VALIDATE_FINITE)    */
  MASK_ERR_OOM = -3,         /* device allocation failed                                  */
  MASK_ERR_CUDA = -4,        /* CUDA runtime/launch/device fault, or no usable GPU        */
  MASK_ERR_NCCL = -5,        /* NCCL failure (multi-GPU)                                  */
  MASK_ERR_UNSUPPORTED = -6  /* valid request this build does not implement               */
} mask_status;

/* mask_matrix.format */
enum { MASK_DENSE_F32 = 0, MASK_CSR_F32 = 1 };
/* mask_matrix.memory */
enum { MASK_MEM_DEVICE = 0, MASK_MEM_HOST = 1 };
/* mask_build_params.empty_policy.  KEEP (D5, default): a prototype without members keeps its
 * position.  FARTHEST (D5b, "an emptied centroid is re-seeded at the point with the
 * largest distance to its current centroid"): after each update the m prototypes left empty,
 * in ascending index, move to the m rows with the largest distance to their prototype in that
 * pass (distance descending, then lower row index); the other prototypes keep their member
 * means.  FARTHEST runs the per-pass loop (no fused small levels), synchronises once per pass
 * to read the empty count, and is single-GPU (MASK_ERR_UNSUPPORTED with a multi-rank comm). */
enum { MASK_EMPTY_KEEP = 0, MASK_EMPTY_FARTHEST = 1 };
/* mask_build_params.flags */
enum {
  MASK_VALIDATE_FINITE = 1 << 0, /* scan inputs for NaN/Inf -> MASK_ERR_NONFINITE          */
  MASK_BORROW_DATA = 1 << 1,     /* index keeps a pointer to device `data` instead of a copy */
  MASK_FORCE_SIMT = 1 << 2,      /* dense assignment on the FP32 SIMT kernel only (testing) */
  MASK_NO_FIXUP = 1 << 3,        /* disable the near-tie re-check of the tensor path (testing)*/
  /* 1 << 4: unused (formerly a per-pass statistics read-back; the loop now reads back once per level) */
  MASK_TIME_KERNELS = 1 << 5,    /* record CUDA-event device times of the step kernels        */
  MASK_NO_SORT = 1 << 6,         /* small d: keep the data order in K1 (no per-pass label sort) */
  MASK_NO_FUSED = 1 << 7,        /* small levels: per-pass kernels instead of the fused loop    */
  MASK_TIME_ASSIGN = 1 << 8,     /* like MASK_TIME_KERNELS for the assignment class only (one
                                    event pair per pass: the cheapest live kernel timing)      */
  MASK_NO_PARTITION_COPY = 1 << 9, /* dense: skip the partition-ordered copy of the rows that
                                    mask_query's leaf scans read (saves n*dim floats)          */
  MASK_TC_TF32 = 1 << 12,        /* dense d = 64 / 128: 3xTF32 even where 3xFP16 is enabled   */
  MASK_CSR_TC = 1 << 11,         /* CSR: K3T (hot columns on tcgen05 3xTF32 + SIMT tail in the
                                    epilogue) instead of the chunk-major SIMT K3; measured slower
                                    at C4 (DESIGN.md §6 K3T), kept for A/B and testing         */
  MASK_TRACE_PASSES = 1 << 10    /* keep, per level, the prototypes every assignment pass used
                                    and the labels it produced, on the device, read back with
                                    mask_get_pass (parity tests of the production path: unlike
                                    iter_cb it changes no kernel choice and adds no host sync;
                                    costs (T+1) x (n_items + k*dim) words per level)          */
};

/* kernel classes of mask_get_timing */
enum { MASK_T_ASSIGN = 0, MASK_T_FIXUP = 1, MASK_T_UPDATE = 2, MASK_T_FINALIZE = 3, MASK_T_NCLASS = 4 };

/*
 * A matrix of `rows` points in R^dim.
 *   MASK_DENSE_F32: `values` = rows*dim fp32, row-major, row stride dim.
 *   MASK_CSR_F32:   row_ptr = rows+1 int64 (row_ptr[0] = 0, non-decreasing, row_ptr[rows]
 *                   = nnz), col_idx = nnz int32 strictly increasing within a row and < dim,
 *                   values = nnz fp32.
 * Multi-GPU (mask_build with a communicator): the matrix is this rank's shard, global rows
 * [row_offset, row_offset + rows) of an n_global-row dataset.  Single GPU: row_offset = 0,
 * n_global = rows.
 */
typedef struct {
  int32_t format;          /* MASK_DENSE_F32 | MASK_CSR_F32                          */
  int32_t memory;          /* MASK_MEM_DEVICE | MASK_MEM_HOST                        */
  int32_t dim;             /* >= 1                                                   */
  int32_t _pad;
  int64_t rows;            /* >= 0 local rows                                        */
  int64_t n_global;        /* total rows over all ranks (== rows on one GPU)         */
  int64_t row_offset;      /* first global row of this shard                         */
  const float* values;     /* dense values or CSR values                             */
  const int64_t* row_ptr;  /* CSR only                                               */
  const int32_t* col_idx;  /* CSR only                                               */
  int64_t nnz;             /* CSR only                                               */
} mask_matrix;

/*
 * Test-only step-parity hook, called after every assignment pass of every level (pass =
 * 0..passes-1, the last one being the final assignment) with HOST copies of the prototypes
 * P_t (k x dim fp32) that pass used and of the labels it produced (this rank's items).
 */
typedef void (*mask_iter_cb)(int32_t level, int32_t pass, const float* P_host, int64_t k,
                             int32_t dim, const int32_t* labels_host, int64_t n_items,
                             void* user);

typedef struct {
  int32_t num_levels;             /* L >= 1                                                */
  int32_t max_iters;              /* T >= 0 Lloyd (assign, update) pairs (D3)              */
  const int64_t* k;               /* host, k[0..L-1] bottom first; 1 <= k[l] <= n_l where
                                     n_0 = n_global, n_l = k[l-1]                          */
  double tol;                     /* >= 0; > 0 also stops when max_j |c_j'-c_j| <= tol     */
  uint64_t seed;                  /* init sampling seed, used for every level whose
                                     init_idx (or init_idx[l]) is NULL (mask_seeded_init)  */
  const int64_t* const* init_idx; /* host, optional; init_idx[l] = k[l] distinct indices
                                     into the level-l input (global row ids for level 1)
                                     (D2); NULL -> drawn from `seed`                       */
  int32_t empty_policy;           /* MASK_EMPTY_KEEP (default) or MASK_EMPTY_FARTHEST        */
  int32_t flags;                  /* MASK_* flags above                                    */
  mask_iter_cb iter_cb;           /* NULL in production                                    */
  void* iter_cb_user;
} mask_build_params;

typedef struct mask_comm mask_comm;   /* wraps an NCCL communicator; NULL = single GPU */
typedef struct mask_index mask_index; /* opaque; owns every device buffer it allocated */

/* ---------------------------------------------------------------- library */
int32_t mask_abi_version(void);
/* thread-local message of the last failure on this thread ("" if none); never NULL */
const char* mask_last_error(void);
/* 1 if a CUDA device usable by this build (sm_100) is present, else 0 */
int32_t mask_device_ok(void);

/* ---------------------------------------------------------------- multi-GPU
 * One process per GPU.  Rank 0 calls mask_comm_unique_id, the caller broadcasts the 128
 * bytes over its own process group, then every rank calls mask_comm_init (collective).
 * The communicator is used by mask_build (ONE allreduce per Lloyd iteration of the packed
 * [sums | counts | J | changed], BASELINE.json north_star) and must outlive the builds that
 * use it. */
int32_t mask_comm_unique_id(uint8_t id_out[128]);
int32_t mask_comm_init(const uint8_t id[128], int32_t world, int32_t rank, mask_comm** out);

/* Host transport (testing): a communicator whose collectives are carried out by the caller's
 * `fn` on host buffers, so every world > 1 branch of mask_build can run with several processes
 * sharing one GPU (the library drains its stream, stages the buffer through host memory,
 * calls fn, copies the result back).  fn(kind, buf, send, count, dtype, arg, user) is called
 * in the same order on every rank and returns 0 on success:
 *   MASK_COLL_ALLREDUCE: buf (count elements) <- elementwise sum (arg = MASK_COLL_SUM) or max
 *                        (MASK_COLL_MAX) over the ranks, in place;
 *   MASK_COLL_BROADCAST: buf (count elements) <- rank `arg`'s buf;
 *   MASK_COLL_ALLGATHER: buf (world * count elements) <- every rank's send (count elements),
 *                        rank-major.
 * dtype: MASK_COLL_F32 / F64 / I32 / I64 / U64.  A non-zero return fails the call with
 * MASK_ERR_NCCL and marks the communicator unusable.  Performance runs use mask_comm_init. */
enum { MASK_COLL_ALLREDUCE = 0, MASK_COLL_BROADCAST = 1, MASK_COLL_ALLGATHER = 2 };
enum { MASK_COLL_F32 = 0, MASK_COLL_F64 = 1, MASK_COLL_I32 = 2, MASK_COLL_I64 = 3, MASK_COLL_U64 = 4 };
enum { MASK_COLL_SUM = 0, MASK_COLL_MAX = 1 };
typedef int32_t (*mask_host_collective_fn)(int32_t kind, void* buf, const void* send, int64_t count,
                                           int32_t dtype, int32_t arg, void* user);
int32_t mask_comm_init_host(int32_t world, int32_t rank, mask_host_collective_fn fn, void* user,
                            mask_comm** out);
void mask_comm_free(mask_comm* comm); /* NULL-safe */

/* ---------------------------------------------------------------- build
 * Build the multilevel index (Algorithm 1 levels, read as one global Lloyd
 * k-means per level, D1).  Collective over `comm` when comm != NULL (every rank calls it
 * with identical params and its own shard).  On success *out owns: per level the
 * prototypes (k_l x dim fp32), labels of the level's items, child lists, the per-pass trace
 * (J_t, changed_t); and a copy of the data for leaf scans (all n_global rows on every rank
 * after the build), unless MASK_BORROW_DATA is set with device data on one GPU, in which
 * case the caller keeps `data` alive and unchanged until mask_free.
 * Errors: MASK_ERR_ARG (L < 1, k[l] out of range, bad init indices, bad CSR, dim < 1, or --
 * with a communicator -- ranks disagreeing on the parameters / init indices, checked with one
 * allreduce of a hash), MASK_ERR_NONFINITE, MASK_ERR_OOM, MASK_ERR_CUDA, MASK_ERR_NCCL.  *out
 * is NULL on error. */
int32_t mask_build(const mask_matrix* data, const mask_build_params* params, mask_comm* comm,
                   void* stream, mask_index** out);

/* ---------------------------------------------------------------- grouped build
 * The paper's own construction (Algorithm 1): the data
 * layer's n rows are split, in `perm` order, into g_1 = floor(n / length_group) groups of
 * balanced sizes (the last n mod g_1 groups hold one more row, G1); every group is
 * clustered independently into n_centroids prototypes (Lloyd from the group's first
 * n_centroids items, max_iters iterations, no-change stop, empty clusters keep; G3, D3-D5);
 * the g_i * n_centroids prototypes (group-major) are the next layer's items, re-chunked
 * contiguously (G2); layers continue while floor(n_i / length_group) >= 1 (the
 * floor recurrence).  The index has the same shape as mask_build's (levels = centroid layers,
 * labels = global prototype ids, explicit child lists), so mask_query / the getters apply
 * (D7: descent over explicit children).  Dense data only, single GPU.
 *   perm: optional host array of `rows` distinct indices (the seeded random split; NULL =
 *         data order); borrowed for the call.
 * Errors: MASK_ERR_ARG (n_centroids < 1 or >= length_group, rows < length_group, a group
 * smaller than n_centroids, perm not a permutation), MASK_ERR_UNSUPPORTED (CSR data, depth >
 * 16 layers, a group's working set > 200 KB of shared memory), MASK_ERR_CUDA. */
typedef struct {
  int32_t length_group; /* points per group (paper's lengthGroup) */
  int32_t n_centroids;  /* prototypes per group (paper's nCentroids) */
  int32_t max_iters;    /* Lloyd iterations per group (T >= 0) */
  int32_t flags;        /* MASK_BORROW_DATA */
  const int64_t* perm;  /* data-layer order (host, rows entries) or NULL */
} mask_grouped_params;

/* Depth (number of centroid layers) of the grouped construction for n points; writes the
 * prototypes per layer to layer_k[0..min(depth, cap)) when non-NULL.  <0 on bad arguments. */
int32_t mask_grouped_depth(int64_t n, int32_t length_group, int32_t n_centroids, int64_t* layer_k, int32_t cap);
int32_t mask_build_grouped(const mask_matrix* data, const mask_grouped_params* params, void* stream,
                           mask_index** out);

/* §5.1 relocation step ("reassigned to that partition ... the multilevel index is
 * built again"; reading G8) for a grouped index `idx` built over the data-layer order
 * `order_in`, after a beam-1 1-NN point search of every point (`got[i]` = the row mask_query
 * returned for point i, -1 = none).  A found point (got[i] == i) keeps its data-layer group
 * (positions of order_in split into floor(n / length_group) balanced groups, the last n mod g
 * one larger, G1), and so does a point whose search reached no partition; a missed point
 * targets the group of the partition its search reached (level-1 prototype of got[i] //
 * n_centroids).  order_out = the points sorted by (target group, keys[i]); keys: distinct
 * values in [0, 2^32) (the iteration's seeded order keys).  reached_out (optional) = the group
 * each point's search reached (-1 = none); *misses_out = the number of points not found.
 * Device arrays of n_items(level 1) entries (int64); returns after the stream completes.
 * Errors: MASK_ERR_ARG (NULL arguments, n_centroids not dividing the level-1 prototype count). */
int32_t mask_relocate(const mask_index* idx, const int64_t* got, const int64_t* order_in, const int64_t* keys,
                      int32_t n_centroids, int64_t* order_out, int64_t* reached_out, int64_t* misses_out,
                      void* stream);

/* ---------------------------------------------------------------- query
 * Batched approximate k-NN (Algorithm 2) of `queries` (same dim/format family
 * as the index: dense queries against a dense index, CSR queries against a CSR index).
 * beam b >= 1 prototypes are kept per level (b = 1 is Algorithm 2; D7); childless
 * prototypes are skipped.  Results: ids_out[q*k_nn + r] (global row id, int64) and
 * d2_out[...] (squared Euclidean distance, fp32) sorted by (d2, id) (D4); a partition
 * smaller than k_nn is padded with (-1, +inf) (D8).  Output buffers live in the same
 * memory kind as `queries` (device or host).  Non-collective; concurrent calls on one
 * index are allowed.  beam <= 32 keeps the per-level selection in registers (warp bitonic top-b);
 * 32 < beam <= 256 (dense queries) keeps it in shared memory (merge-path top-b, same order and
 * result).  Errors: MASK_ERR_ARG (k_nn < 1 or > 32, beam < 1 or > 256, dim or
 * format mismatch), MASK_ERR_CUDA. */
int32_t mask_query(const mask_index* idx, const mask_matrix* queries, int32_t k_nn,
                   int32_t beam, int64_t* ids_out, float* d2_out, void* stream);

/* ---------------------------------------------------------------- range search
 * Range query (Algorithm 3): for each query q_i every data row
 * x with ||q_i - x|| <= radius[i] among the partitions reached by a multi-path descent:
 *   MASK_RANGE_PAPER: at each level keep the candidates c with ||q - c|| <= r (Algorithm 3's
 *                     selectCandidates; may miss rows, like the paper);
 *   MASK_RANGE_COVER: keep c with ||q - c|| <= r + cover(c), cover(c) >= the distance from c to
 *                     every row below it (triangle inequality): the result equals the
 *                     brute-force range scan (lossless).  Cover radii are computed on first use.
 * Results are grouped by query and sorted by (d^2, id): row ids ids_out[offsets_out[i] ..
 * offsets_out[i+1]) and squared distances d2_out[...].  queries / radius / outputs live in the
 * same memory kind (device or host).  *total_out always receives the number of results; when it
 * exceeds max_results the call fails with MASK_ERR_ARG (never silent truncation) and the caller
 * retries with a larger buffer.  Dense index only (MASK_ERR_UNSUPPORTED for CSR).  Non-collective. */
enum { MASK_RANGE_PAPER = 0, MASK_RANGE_COVER = 1 };
int32_t mask_range_query(const mask_index* idx, const mask_matrix* queries, const float* radius, int32_t mode,
                         int64_t max_results, int64_t* offsets_out, int64_t* ids_out, float* d2_out,
                         int64_t* total_out, void* stream);

/* ---------------------------------------------------------------- insertion
 * Dynamic insertion: each new point descends like a beam-1
 * query (top level: nearest prototype with children; then the nearest of its children, ...)
 * and joins the data partition of the level-1 prototype it reaches; prototypes are unchanged.
 * New rows get ids n, n+1, ... (n = rows indexed so far); partition_out (optional, rows
 * entries, same memory kind as `points`) receives the level-1 prototype of each.  A
 * subsequent query with an inserted vector descends identically and finds it.  Mutates the
 * index (single writer: no concurrent queries during the call); the index keeps its own copy
 * of the grown data (a MASK_BORROW_DATA buffer is copied).  Dense single-GPU indexes only
 * (MASK_ERR_UNSUPPORTED otherwise); MASK_ERR_ARG on a dim mismatch. */
int32_t mask_insert(mask_index* idx, const mask_matrix* points, int64_t* partition_out, void* stream);

/* ---------------------------------------------------------------- partition split
 * Partition split and local rebuild ("if one partition grows beyond a certain
 * threshold, it can be split in smaller data groups and reconstruct just the local part of the
 * index covering that specific region, without affecting the rest of the structure"; SURVEY
 * §8(f) NEXT-4; reading S1).  For every level-1 prototype j, in ascending order,
 * whose partition holds n_j > threshold rows: its rows in ascending id order are clustered by
 * the library's Lloyd loop (max_iters iterations + the final assignment, empty groups keep,
 * lowest index on ties) into s = ceil(n_j / threshold) groups from the init rows
 * mask_seeded_init(seed + j, 1, n_j, s); group 0 keeps id j, groups 1..s-1 take the next new
 * level-1 ids (k_1, k_1 + 1, ... in order of j, then group); each new prototype's level-2
 * parent is j's; every other prototype, label and upper level is unchanged (so the descent
 * reaches the new partitions through j's parent).  Partitions created by the call are not
 * split again in it.  Mutates the index (single writer); level 1 then has k_1 + (new ids)
 * prototypes (mask_level_info); a MASK_TRACE_PASSES trace of level 1 is dropped.  Dense
 * single-GPU indexes only (MASK_ERR_UNSUPPORTED otherwise); MASK_ERR_ARG on threshold < 1 or
 * max_iters < 0.  *n_split_out (optional) = the number of partitions split. */
typedef struct {
  int64_t threshold; /* split partitions with more rows than this (>= 1)                    */
  int32_t max_iters; /* Lloyd iterations of each local k-means (>= 0)                      */
  int32_t flags;     /* MASK_FORCE_SIMT / MASK_NO_FUSED for the local Lloyd loop (else 0)   */
  uint64_t seed;     /* local init seed (partition j draws from seed + j)                   */
} mask_split_params;
int32_t mask_split(mask_index* idx, const mask_split_params* params, int64_t* n_split_out, void* stream);

/* ---------------------------------------------------------------- distributed mode
 * The paper's §3.4 "Indexing distributed datasets": every
 * node (one GPU, one process) builds its own index over its own rows with comm = NULL (zero
 * collectives: mask_collective_count() does not move); "just the top level centroids from
 * each node need to be recorded" by the coordinator; a query is answered either
 * by all nodes or only by the "nodes that have centroids whose distance to the target query
 * object is lower than a given threshold epsilon"; the answers are merged.
 *
 * mask_top_prototypes: the index's top-level prototypes that have children (reading C2), in
 * id order, into host_out (count x dim fp32, caller-allocated with room for k_L rows; may be
 * NULL to query the count); *count_out = their number.
 *
 * mask_route: routed_out[q * n_nodes + n] = 1 iff some registry row c with node_of[c] = n has
 * ||q - c||^2 < epsilon^2 (strict, reading C1; FP32), else 0; epsilon = +inf routes every
 * query to every node; epsilon = 0 to none.  registry: device n_registry x dim fp32
 * (row-major), node_of: device int32 in [0, n_nodes), queries: device (dense or CSR, dim =
 * the registry's), routed_out: device uint8 nq x n_nodes.  MASK_ERR_ARG on n_nodes < 1,
 * epsilon < 0 or NULL pointers; MASK_ERR_UNSUPPORTED for host queries.
 *
 * mask_query_routed: mask_query (device queries and outputs only) answering query q only if
 * routed[q * routed_stride] != 0 -- the rest get (-1, +inf) padding -- and reporting global
 * ids id_base + local row id.  A node passes routed_out + its node number and stride n_nodes.
 *
 * mask_merge: the coordinator's merge: ids / d2 hold n_nodes blocks of nq x k_nn answers
 * (node-major; each row sorted by (d^2, id), padded with (-1, +inf)); writes the k_nn best per
 * query by (d^2, node, id) (reading C3) to ids_out / d2_out (nq x k_nn), padded with (-1, +inf).
 * All device buffers.  MASK_ERR_ARG on n_nodes outside [1, 64] or k_nn outside [1, 32].
 *
 * mask_collective_count: the number of NCCL calls the library has issued in this process (the
 * zero-communication counter of the independent per-node build). */
int32_t mask_top_prototypes(const mask_index* idx, float* host_out, int64_t* count_out);
int32_t mask_route(const float* registry, const int32_t* node_of, int64_t n_registry, int32_t n_nodes,
                   const mask_matrix* queries, double epsilon, uint8_t* routed_out, void* stream);
int32_t mask_query_routed(const mask_index* idx, const mask_matrix* queries, const uint8_t* routed,
                          int64_t routed_stride, int64_t id_base, int32_t k_nn, int32_t beam, int64_t* ids_out,
                          float* d2_out, void* stream);
int32_t mask_merge(const int64_t* ids, const float* d2, int32_t n_nodes, int64_t nq, int32_t k_nn, int64_t* ids_out,
                   float* d2_out, void* stream);
int64_t mask_collective_count(void);

/* ---------------------------------------------------------------- seeded initialisation
 * The init indices mask_build draws when init_idx is NULL (D2: k distinct indices, uniform
 * without replacement): Floyd's algorithm -- for j = n-k .. n-1: t = u(j+1); take t unless
 * already taken, else j -- with u(m) = next() mod m and next() the SplitMix64 sequence
 * state += 0x9E3779B97F4A7C15; z = state; z = (z ^ z>>30) * 0xBF58476D1CE4E5B9;
 * z = (z ^ z>>27) * 0x94D049BB133111EB; return z ^ z>>31, started from state = seed + level *
 * 0x9E3779B97F4A7C15 (level 1 = the data level).  out[0..k) = the indices in the order they
 * are taken (prototype j starts at item out[j]).  Host only; MASK_ERR_ARG unless 1 <= k <= n,
 * level >= 1, out != NULL. */
int32_t mask_seeded_init(uint64_t seed, int32_t level, int64_t n, int64_t k, int64_t* out);

/* Test hook (failure-path tests): the nth next device allocation of the library (0 = the next
 * one) fails as if the device were out of memory, so the call making it returns MASK_ERR_OOM
 * and releases what it had allocated; -1 disarms it.  Not for production use. */
void mask_debug_fail_alloc(int64_t nth);

void mask_free(mask_index* idx); /* NULL-safe */

/* ---------------------------------------------------------------- step entry points
 * The two Lloyd steps of one level as separate calls (the §8(a) rows a3-a7, a9), used by
 * the kernel parity tests and the per-kernel timing of bench.py.  Single GPU.
 *
 * mask_assign: a_i = argmin_j ||x_i - c_j||^2 (lowest j on ties, D4) for every
 * row of `data` against prototypes P (device, k x dim fp32, row-major).  Writes device
 * labels_out[rows] (int32) and, if non-NULL, device d2_out[rows] (fp32 squared distance
 * to the chosen prototype).  Dense rows use the tcgen05 3xTF32 (d = 64 / 128: 3xFP16) kernel with a near-tie
 * FP32 re-check when dim allows, else the FP32 SIMT kernel; CSR rows the sparse kernel.
 * *n_flagged (optional, host) receives the number of rows the near-tie re-check recomputed.
 */
int32_t mask_assign(const mask_matrix* data, const float* P, int64_t k, int32_t flags,
                    int32_t* labels_out, float* d2_out, int64_t* n_flagged, void* stream);

/* mask_update: P_out_j = mean of the rows with labels == j, or P_in_j if none (D5).
 * P_in/P_out device k x dim fp32 (may alias); counts_out device int32[k] (optional).
 * *max_disp (optional, host) = max_j ||P_out_j - P_in_j||. */
int32_t mask_update(const mask_matrix* data, const int32_t* labels, int64_t k,
                    const float* P_in, float* P_out, int32_t* counts_out, double* max_disp,
                    void* stream);

/* ---------------------------------------------------------------- introspection
 * Levels are numbered 1..L (level 1 = prototypes over the data). Host outputs. */
int32_t mask_num_levels(const mask_index* idx);
int32_t mask_level_info(const mask_index* idx, int32_t level, int64_t* n_items, int64_t* k,
                        int32_t* dim, int32_t* passes, int32_t* updates);
int32_t mask_get_prototypes(const mask_index* idx, int32_t level, float* host_out /* k*dim */);
int32_t mask_get_labels(const mask_index* idx, int32_t level,
                        int32_t* host_out /* n_items of the level (level 1: n_global) */);
/* children of prototype j: members[offsets[j] .. offsets[j+1]) in ascending item id */
int32_t mask_get_children(const mask_index* idx, int32_t level, int64_t* host_offsets /* k+1 */,
                          int64_t* host_members /* n_items */);
/* per assignment pass: J_t = sum_i ||y_i - c_{a_i}||^2 (GPU estimate), changed_t = rows whose
 * label changed vs the previous pass (all rows at pass 0), empties_t = prototypes left
 * without members by the update that followed (0 for the final pass).  Returns the number
 * of passes written (<= cap) or < 0 on error. */
int32_t mask_get_trace(const mask_index* idx, int32_t level, double* J, int64_t* changed,
                       int64_t* empties, int32_t cap);
/* per assignment pass, like mask_get_trace: dmax_t = max_j ||c_j' - c_j|| of the update that
 * followed it (the tolerance-stop quantity, D3; 0 when no update followed).  Returns the number
 * of passes written or < 0 on error. */
int32_t mask_get_displacement(const mask_index* idx, int32_t level, double* dmax, int32_t cap);

/* per assignment pass of a build made with MASK_TRACE_PASSES (pass = 0 .. passes-1 as in
 * mask_level_info, the last one being the final assignment): P_host (k x dim fp32, may be NULL)
 * receives the prototypes the pass used and labels_host (may be NULL) the labels it produced
 * for this rank's items of the level (labels_host needs room for n_items of mask_level_info).
 * Returns the number of labels written (this rank's items: the shard's rows at level 1 of a
 * multi-GPU build) or < 0: MASK_ERR_ARG on a bad level / pass, MASK_ERR_UNSUPPORTED when the
 * build did not keep the trace. */
int32_t mask_get_pass(const mask_index* idx, int32_t level, int32_t pass, float* P_host, int32_t* labels_host);

/* ---------------------------------------------------------------- diagnostics
 * Cumulative number of CUDA kernel launches issued by this library in this process. */
int64_t mask_kernel_launches(void);
/* Device time of the step kernels of one level, measured with CUDA events recorded on the
 * build stream around each launch (only when the build ran with MASK_TIME_KERNELS):
 * out[2*c] = total milliseconds, out[2*c+1] = number of launches, for kernel class
 * c = MASK_T_ASSIGN .. MASK_T_FINALIZE; cap = number of doubles out can hold (>= 2*c+2 for
 * class c to be written); out[2*MASK_T_NCLASS] (cap > 8) = the assignment kernel the level
 * used (0 = K2 FP32 SIMT, 1 = K1 tcgen05 3xTF32, 2 = K3 CSR, 3 = K11 fused small level,
 * 4 = K12 grouped, 5 = K3T CSR on tcgen05, 6 = K1 tcgen05 3xFP16).  Returns the number of
 * doubles written or < 0 on error. */
int32_t mask_get_timing(const mask_index* idx, int32_t level, double* out, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* MASK_H_ */
