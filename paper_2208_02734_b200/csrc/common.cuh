// common.cuh -- host/device helpers shared by the libmask kernels (not by the oracle).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/mask.h"

namespace mask {

// Host-side error carried up to the C boundary, which converts it to a mask_status.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define MASK_CUDA(x)                                                                        \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      ::mask::fail(e_ == cudaErrorMemoryAllocation ? MASK_ERR_OOM : MASK_ERR_CUDA,          \
                   std::string(#x) + ": " + cudaGetErrorString(e_) + " (" + __FILE__ + ":" + \
                       std::to_string(__LINE__) + ")");                                     \
  } while (0)

// every kernel launch is followed by exactly one MASK_LAUNCH_CHECK (it also counts launches)
void count_launch();
#define MASK_LAUNCH_CHECK()           \
  do {                                \
    ::mask::count_launch();           \
    MASK_CUDA(cudaGetLastError());    \
  } while (0)

#define MASK_REQUIRE(cond, code, msg)               \
  do {                                                \
    if (!(cond)) ::mask::fail((code), std::string(msg)); \
  } while (0)

// Process-wide caching device allocator (mask_api.cu): blocks are rounded up to a size class
// and recycled instead of cudaFree'd, so builds and queries do not synchronise the device on
// allocation.  pool_trim() returns the cached blocks to the driver.
void* pool_alloc(size_t bytes);
void pool_free(void* p, size_t bytes);
void pool_trim();

// Owning device buffer (pool-backed).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) p = static_cast<T*>(pool_alloc(count * sizeof(T)));
  }
  void release() {
    if (p) pool_free(p, n * sizeof(T));
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
};

inline unsigned grid_for(int64_t work, int block, int64_t cap = 148LL * 64) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

inline int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// ------------------------------------------------------------------ kernel entry points
// (defined in the .cu files; all enqueue on `st` and never synchronise)

// K2: FP32 SIMT assignment, direct (x - c)^2 sums; labels + squared distance of the winner.
// K2b: blocked SIMT assignment for large d (dimension streamed through shared memory);
// keys_ws = n u64 scratch
void launch_assign_blocked(const float* X, int64_t n, int d, const float* P, int64_t k, unsigned long long* keys_ws,
                           int32_t* labels, float* best, cudaStream_t st, const int* active = nullptr);
void launch_assign_simt(const float* X, int64_t n, int d, const float* P, int64_t k,
                        int32_t* labels, float* best, cudaStream_t st, const int* active = nullptr);

// K1: tcgen05 3xTF32 assignment (dense, d % 8 == 0, d <= 256).  Writes labels, best (d^2
// estimate incl. ||x||^2), and appends rows whose top-2 gap is within the error bound to
// flag_rows / flag_count (device).  Returns false if the shape is unsupported.
bool tc_supported(int64_t n, int d, int64_t k);
// columns of the K1 B operand arrays Pb/Ps: d, or d+2 rounded up to 4 when ||x||^2 and ||c||^2
// are folded into the contraction (small d)
int tc_operand_cols(int d);
void launch_assign_tc(const float* X, int64_t n, int d, const float* P, const float* Pb,
                      const float* Ps, const float* cn2, int64_t k, const float* xn2,
                      int32_t* labels, float* best, int32_t* flag_rows, int32_t* flag_count,
                      cudaStream_t st, const int* active = nullptr, const int32_t* perm = nullptr,
                      const int32_t* prev_lab = nullptr, int32_t* lab2 = nullptr, int2* flag_pair = nullptr,
                      const void* Hb = nullptr, const void* Hs = nullptr, float h16_scale = 1.f,
                      float h16_err_abs = 0.f);
// K1 3xFP16 operands: per-level power-of-two scale of the data (one host read of max |x|) and the
// per-pass FP16 split of s (-2c) [k x d] (big, small)
bool tc_h16_enabled();  // 3xFP16 for d = 64 / 128 (default; environment MASK_TC_H16=0 disables)
float h16_level_scale(const float* X, int64_t cnt, float* maxabs_out, cudaStream_t st);
void launch_prep_h16(const float* P, const double* P64, int64_t k, int d, float s, void* Hb, void* Hs, cudaStream_t st,
                     const int* active = nullptr);
// Counting sort of rows by label: perm = rows of label 0, then 1, ...; cnt_ws = k int32.
// perm_old (optional): a previous sort, visited in its order (equal labels adjacent -> warp-
// aggregated atomics); perm must not alias it.  copy_to (optional): copy_to[row] = labels[row].
// cnt_zeroed: cnt_ws is already zero (the Lloyd loop's finalize zeroes it for the next sort).
void launch_label_sort(const int32_t* labels, int64_t n, int64_t k, const int32_t* perm_old, int32_t* perm,
                       int32_t* cnt_ws, int32_t* copy_to, cudaStream_t st, const int* active = nullptr,
                       bool cnt_zeroed = false);
// K11: the whole Lloyd loop of a small dense level in one cooperative launch (same stats /
// control words as run_level's multi-kernel loop; bar_ws = 2 unsigned; S = k*d zeroed doubles).
bool small_level_supported(int64_t n, int d, int64_t k);
void launch_small_level(const float* Y, int64_t n, int d, int64_t k, float* P, int32_t* lab, int32_t* prev,
                        float* best, double* S, int32_t* counts, double* J, unsigned long long* changed,
                        uint32_t* fin, int* ctrl, unsigned* bar_ws, int T, double tol, cudaStream_t st,
                        float* P_trace = nullptr, int32_t* lab_trace = nullptr);
// K12: one layer of the grouped construction (Algorithm 1): g groups of the n_items rows of Y
// (through perm when given), nc prototypes each, T Lloyd iterations per group; P_out = g*nc x d
// (group-major), labels[row] = global prototype id.
size_t group_lloyd_smem(int64_t n_items, int64_t g, int nc, int d);
void launch_group_lloyd(const float* Y, int d, const int64_t* perm, int64_t n_items, int64_t g, int nc, int T,
                        float* P_out, int32_t* labels, cudaStream_t st);
// K4: exact FP32 direct re-check of the flagged rows against all k prototypes, sized on the
// device from the flagged count (no host round trip); keys_ws = cap u64.
// flag_pair (optional): per flagged row (j1, j2): j2 >= 0 -> the only two candidates, decided
// exactly (FP64 direct distances, lower index on ties); j2 < 0 -> full re-check, through the
// compacted list rescan_rows / rescan_count (n int32 / 1 int32 workspace)
void launch_fixup_device(const float* X, int d, const float* P, int64_t k, const int32_t* flag_rows,
                         const int32_t* flag_count, int64_t cap, unsigned long long* keys_ws, int32_t* labels,
                         float* best, cudaStream_t st, const int* active = nullptr, const int2* flag_pair = nullptr,
                         int32_t* rescan_rows = nullptr, int32_t* rescan_count = nullptr,
                         const double* P64 = nullptr, double* P64T = nullptr /* k*d workspace */);
// FP64-prototype levels (D15): FP64 sums, FP64 finalize (P64 and its fp32 rounding P)
void launch_update_dense64(const float* X, int64_t n, int d, const int32_t* labels, double* S, int32_t* counts,
                           cudaStream_t st, const int* active, const int32_t* perm);
void launch_f32_to_f64(const float* a, int64_t n, double* b, cudaStream_t st);
// FP64 sums over label-sorted rows without atomics (warp per cluster; end = the sort's end offsets)
// D5b: re-seed the prototypes this update left empty at the pass's farthest rows
// (dense X or CSR rp/col/val); single rank; synchronises the stream (rare-path option).
void reseed_farthest(const float* X, const int64_t* rp, const int32_t* col, const float* val, int d, int64_t n,
                     int64_t k, const float* best, const int32_t* counts, float* P, double* P64, uint32_t* stat,
                     const int* active, cudaStream_t st);
bool update_seg64_supported(int d);
void launch_update_seg64(const float* X, int d, const int32_t* perm, const int32_t* labels, const int32_t* end,
                         int64_t n, double* S, int32_t* counts, cudaStream_t st, const int* active);
// prototype operands for K1: Pb = tf32_rn(-2c), Ps = tf32_rn(-2c - Pb), cn2 = ||c||^2; with
// kc > d the augmented columns [d] = split(||c||^2), [d+1] = (1, 0), rest 0 (row stride kc)
// flag_count (optional): reset to 0 (the list K1 appends near-tie rows to)
void launch_prep_protos(const float* P, int64_t k, int d, int kc, float* Pb, float* Ps, float* cn2,
                        cudaStream_t st, int64_t k_rows, int fold, const int* active = nullptr,
                        int32_t* flag_count = nullptr, const double* P64 = nullptr);
// rows of the K1 B operand arrays (k padded to whole 256-prototype tiles)
int64_t tc_operand_rows(int64_t k);
void launch_row_norms(const float* X, int64_t n, int d, float* xn2, cudaStream_t st);

// K3: CSR rows x dense prototypes (sparse assignment).
void launch_assign_csr(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t n,
                       int d, const float* PT /* d x k transposed */, const float* cn2, int64_t k,
                       int32_t* labels, float* best, cudaStream_t st, const int* active = nullptr);
void launch_transpose(const float* P, int64_t k, int d, float* PT, cudaStream_t st, const int* active = nullptr);
// K3 chunk-major: colslot[c] = hot slot of column c (< 128) or -1; hotcols[h] = column of slot
// h (or -1); state = n float2 (running argmin across chunks).
bool csr_chunked_supported(int d, int64_t k);
int csr_chunked_hot();  // number of hot columns (slots) the kernel stages
void launch_assign_csr_chunked(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t n, int d,
                               const float* PT, const float* cn2, int64_t k, const int16_t* colslot,
                               const int32_t* hotcols, float2* state, int32_t* labels, float* best, cudaStream_t st,
                               const int* active = nullptr);
// K3T (assign_csr_tc.cu): CSR hot columns on tcgen05 (3xTF32) + SIMT tail in the epilogue.
int64_t csr_tc_rows(int64_t k);  // prototype rows padded to whole tiles
int csr_tc_hot();                // hot columns H
// per level: Xh [n x H] dense hot block, tail {col, -2v} at each row's CSR offset, ntail [n], xn2 [n]
void launch_csr_tc_level(const int64_t* rp, const int32_t* col, const float* val, int64_t n, const int16_t* colslot,
                         float* Xh, int2* tail, int32_t* ntail, float* xn2, cudaStream_t st);
// per pass: Hb/Hs [csr_tc_rows(k) x H] split -2 c_hot, cn2 [csr_tc_rows(k)] (+inf pad), PT [d x csr_tc_rows(k)]
void launch_csr_tc_prep(const float* P, int64_t k, int d, const int32_t* hotcols, float* Hb, float* Hs, float* cn2,
                        float* PT, cudaStream_t st, const int* active = nullptr);
void launch_assign_csr_tc(const float* Xh, const int64_t* rp, const int2* tail, const int32_t* ntail, const float* xn2,
                          int64_t n, const float* Hb, const float* Hs, const float* PT, const float* cn2, int64_t k,
                          int32_t* labels, float* best, cudaStream_t st, const int* active = nullptr);
void launch_i64_to_i32(const int64_t* a, int64_t n, int32_t* b, cudaStream_t st);
// per-column non-zero counts (d int32, zeroed here)
void launch_col_hist(const int32_t* col, int64_t nnz, int d, int32_t* cnt, cudaStream_t st);

// K5/K6: cluster sums and counts (S, counts must be zeroed by the caller).
// perm (optional): rows sorted by these labels (launch_label_sort) -> run-accumulating kernel
void launch_update_dense(const float* X, int64_t n, int d, const int32_t* labels, int64_t k,
                         float* S, int32_t* counts, cudaStream_t st, const int* active = nullptr,
                         const int32_t* perm = nullptr);
// K6 over rows sorted by label (perm, end = per-label end offsets from launch_label_sort)
bool csr_sorted_update_supported(int d);
void launch_update_csr_sorted(const int64_t* row_ptr, const int32_t* col, const float* val, int d,
                              const int32_t* perm, const int32_t* labels, const int32_t* end, int64_t n, int64_t k,
                              float* S, int32_t* counts, cudaStream_t st, const int* active);
void launch_update_csr(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t n,
                       int d, const int32_t* labels, float* S, int32_t* counts, cudaStream_t st,
                       const int* active = nullptr);
// Device-side Lloyd loop control fused into the last block of a per-pass kernel:
// ctrl = {active, passes run, stats ticket, finalize ticket}; t = pass, T = iteration cap.
struct LoopCtl {
  int* ctrl = nullptr;
  int t = 0, T = 0;
  double tol = 0.0;
  int32_t* zero_cnt = nullptr;  // finalize: also zero these k counters (label sort)
};
// K7: P_j <- S_j / n_j (keep if n_j == 0); zeroes S and counts; stats[0] = max disp^2 (as
// float bits, atomicMax), stats[1] = empties.  `stat` must be zeroed by the caller.  With
// lc.ctrl: the tolerance stop / pass count of the loop (k_after_update's logic) in the last block.
void launch_finalize(float* P, float* S, int32_t* counts, int64_t k, int d, uint32_t* stat,
                     int keep_counts, cudaStream_t st, const int* active = nullptr, LoopCtl lc = LoopCtl());
void launch_finalize64(double* P64, float* P, double* S, int32_t* counts, int64_t k, int d, uint32_t* stat,
                       cudaStream_t st, const int* active, LoopCtl lc);
// pass statistics: J = sum best (double), changed = #(cur != prev).  With lc.ctrl: the
// no-change stop test (k_after_stats's logic, single GPU) in the last block.
void launch_pass_stats(const int32_t* cur, const int32_t* prev, const float* best, int64_t n,
                       double* J, unsigned long long* changed, cudaStream_t st, const int* active = nullptr,
                       LoopCtl lc = LoopCtl());
// K10: P[j] = Y[idx[j]] (dense) / densified CSR row
void launch_gather_rows(const float* Y, int d, const int64_t* idx, int64_t k, int64_t row_offset,
                        int64_t n_local, float* P, cudaStream_t st);
void launch_gather_csr_rows(const int64_t* row_ptr, const int32_t* col, const float* val, int d,
                            const int64_t* idx, int64_t k, int64_t row_offset, int64_t n_local,
                            float* P, cudaStream_t st);
// K8: child lists by counting sort: offsets (k+1, int64), members (n, int32; order within a
// segment unspecified)
void launch_children(const int32_t* labels, int64_t n, int64_t k, int64_t* offsets,
                     int32_t* members, int32_t* cursor_ws, cudaStream_t st);
// CSR structure check on the device: *err = OR of 1 (row_ptr), 2 (column range), 4 (column order)
void launch_check_csr(const int64_t* rp, const int32_t* col, int64_t rows, int64_t nnz, int dim, int* err,
                      cudaStream_t st);
// device top-H column selection for K3's hot set from a column histogram: hotcols[0..H) and
// colslot[d] (slot or -1); columns by non-zero count (more first), lower index on equal counts,
// zero-count columns never hot
void launch_select_hot(const int32_t* cnt, int d, int H, int32_t* hotcols, int16_t* colslot, cudaStream_t st);
// finite check: flag set to 1 if any non-finite value
void launch_check_finite(const float* v, int64_t count, int32_t* flag, cudaStream_t st);
void launch_fill(float* p, int64_t count, float v, cudaStream_t st);

// K9: batched query descent.
struct QLevel {
  const float* P;
  const int64_t* offsets;
  const int32_t* members;
  int64_t k;
  // this level's prototypes in the parent level's child-list order (Pc[m] = P[parent.members[m]]),
  // or nullptr: the descent then reads every parent's children as contiguous rows
  const float* Pc = nullptr;
};
constexpr int kMaxLevels = 16;
struct QIndex {
  QLevel lv[kMaxLevels];
  int L;
  int dim;
  const float* X;           // dense data rows (n x dim) or nullptr
  const int64_t* xrp;       // CSR data
  const int32_t* xcol;
  const float* xval;
  // §3.4 distributed mode (K14): when `routed` is set, query q is answered only if
  // routed[q * rstride] != 0 (else padded); result ids are id_base + local row id
  const uint8_t* routed = nullptr;
  int64_t rstride = 0;
  int64_t id_base = 0;
  // dense data rows in level-1 partition order (Xp[pos] = X[members_1[pos]]), or nullptr: leaf
  // scans then read contiguous rows at addresses known before the member ids arrive
  const float* Xp = nullptr;
  // leaf-grouped queries: when set, the descent writes each query's selected level-1
  // prototypes (beam entries, -1 padded) here and skips the leaf scan
  int32_t* sel_out = nullptr;
  // with sel_out: the level (index into lv) whose selection is handed over (0: level 1)
  int sel_stop = 0;
};
// Leaf-grouped batched k-NN (dense, partition-ordered rows): descent -> (query, leaf) pairs
// grouped by leaf -> every leaf's rows staged in shared memory once for all its queries ->
// per-query merge of the per-leaf top-k lists.  Same result order (d^2, id) as the per-query
// kernel.  Returns false (nothing launched) when the batch does not qualify.
bool launch_query_grouped(const QIndex& qi, const float* Q, int64_t nq, int knn, int beam, int64_t* ids, float* d2,
                          cudaStream_t st);
// Xp[pos * d ...] = X[members[pos] * d ...] for pos < n (the partition-ordered copy of the rows)
void launch_gather_partition(const float* X, int d, const int32_t* members, int64_t n, float* Xp, cudaStream_t st);
// stable LSD radix sort (sort.cu) of (key, value) pairs on key bits [begin_bit, end_bit), in
// place; synchronises the stream
void radix_sort_pairs(uint64_t* keys, int64_t* vals, int64_t n, int begin_bit, int end_bit, cudaStream_t st);
// §5.1 relocation step (relocate.cu, reading G8): next data-layer order of a grouped index
void launch_relocate(const int64_t* got, const int64_t* order_in, const int64_t* keys, const int32_t* lab1, int64_t n,
                     int64_t n_groups, int n_centroids, int64_t* order_out, int64_t* reached_out,
                     unsigned long long* misses, cudaStream_t st);
// K13 range search: cover radii (cover[l] = k_l float bits) and the multi-path descent; returns
// the number of results, writing them (sorted by query, d^2, id) and per-query counts only when
// ids_out != nullptr and the count fits cap_out.
void launch_cover_radii(const float* X, int d, const QIndex& qi, const int32_t* const* labels,
                        const int64_t* n_items, unsigned* const* cover, cudaStream_t st);
int64_t range_search(const QIndex& qi, const unsigned* const* cover, const float* Q, int64_t nq, const float* radius,
                     int mode, int64_t* ids_out, float* d2_out, int64_t* qcount, int64_t cap_out, cudaStream_t st);
// leaf_only: ids[q] = the level-1 prototype reached by the beam-1 descent (no data layer)
void launch_query_dense(const QIndex& qi, const float* Q, int64_t nq, int knn, int beam,
                        int64_t* ids, float* d2, cudaStream_t st, bool leaf_only = false);
void launch_query_csr(const QIndex& qi, const float* cn2_levels_flat, const int64_t* cn2_off,
                      const int64_t* qrp, const int32_t* qcol, const float* qval, int64_t nq,
                      int knn, int beam, int64_t* ids, float* d2, cudaStream_t st);
void launch_level_norms(const float* P, int64_t k, int d, float* cn2, cudaStream_t st, const int* active = nullptr);
// K14 distributed mode (§3.4): routing of queries to nodes by the registered top-level
// prototypes, and the (d^2, node, id) merge of the nodes' answers
void launch_route_dense(const float* reg, const int32_t* node_of, int64_t R, int W, const float* Q, int64_t nq, int d,
                        float eps2, bool all, uint8_t* routed, cudaStream_t st);
void launch_route_csr(const float* reg, float* reg_n2 /* R floats of workspace */, const int32_t* node_of, int64_t R, int W, int d,
                      const int64_t* qrp, const int32_t* qcol, const float* qval, int64_t nq, float eps2, bool all,
                      uint8_t* routed, cudaStream_t st);
void launch_merge(const int64_t* ids, const float* d2, int W, int64_t nq, int k, int64_t* ids_out, float* d2_out,
                  cudaStream_t st);

}  // namespace mask
