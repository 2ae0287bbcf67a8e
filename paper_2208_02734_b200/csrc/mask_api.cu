// mask_api.cu -- the C-ABI of libmask.so (include/mask.h) and the host orchestrator:
// argument validation, the level loop (Algorithm 1, read as one global
// k-means per level, D1), the Lloyd loop of each level (D2/D3/D5), the NCCL
// combine step for row-sharded multi-GPU builds (BASELINE.json north_star: "each
// iteration's partial sums and counts are combined with a single NCCL allreduce"), child
// lists, the query entry point (Algorithm 2) and introspection.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_set>
#include <vector>

#include "common.cuh"

#include <atomic>
#include <map>
#include <mutex>

using namespace mask;

namespace {
std::atomic<int64_t> g_launches{0};
std::atomic<int64_t> g_nccl_calls{0};  // every NCCL call the library issues (mask_collective_count)
}

void mask::count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ------------------------------------------------------------------ caching device allocator
// Blocks are recycled instead of cudaFree'd.  A block released while an API call's stream may
// still be using it (a DevBuf leaving scope right after the launches that read it) carries an
// event recorded on that stream at release: the same stream may take it again at once (stream
// order), any other stream or thread only after the event has completed.  Blocks released
// outside an API call (mask_free: nothing is in flight by the synchronous call contract) carry
// no event.
namespace {
std::mutex g_pool_mu;
struct FreeBlock {
  void* p;
  cudaStream_t st;  // stream whose pending work may still use the block (when ev != nullptr)
  cudaEvent_t ev;   // recorded on st at release, or nullptr
};
std::multimap<size_t, FreeBlock> g_pool;  // size class -> free block
std::vector<cudaEvent_t> g_event_cache;   // completed events for reuse (under g_pool_mu)
thread_local bool g_have_stream = false;  // inside an API call that named its stream
thread_local cudaStream_t g_cur_stream = nullptr;
size_t size_class(size_t bytes) {
  if (bytes <= (1u << 20)) {  // small: next power of two >= 512 B
    size_t c = 512;
    while (c < bytes) c <<= 1;
    return c;
  }
  return (bytes + (1u << 20) - 1) & ~size_t((1u << 20) - 1);  // large: whole MiB
}
}  // namespace

namespace {
std::atomic<int64_t> g_fail_alloc{-1};  // test hook: the n-th next device allocation fails
}

void* mask::pool_alloc(size_t bytes) {
  if (g_fail_alloc.load(std::memory_order_relaxed) >= 0 && g_fail_alloc.fetch_sub(1) == 0)
    ::mask::fail(MASK_ERR_OOM, "injected device allocation failure (mask_debug_fail_alloc)");
  const size_t c = size_class(bytes);
  {
    std::lock_guard<std::mutex> g(g_pool_mu);
    auto range = g_pool.equal_range(c);
    for (auto it = range.first; it != range.second; ++it) {
      FreeBlock& b = it->second;
      bool ready = b.ev == nullptr || (g_have_stream && b.st == g_cur_stream);
      if (!ready) {
        const cudaError_t q = cudaEventQuery(b.ev);
        if (q == cudaErrorNotReady) continue;
        cudaGetLastError();  // (an error here resurfaces at the caller's next CUDA call)
        ready = true;
      }
      void* p = b.p;
      if (b.ev) g_event_cache.push_back(b.ev);  // re-recorded before any later wait on it
      g_pool.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, c);
  if (e == cudaErrorMemoryAllocation) {  // give the idle cache back and retry once
    cudaGetLastError();
    pool_trim();
    e = cudaMalloc(&p, c);
  }
  MASK_CUDA(e);
  return p;
}

void mask::pool_free(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> g(g_pool_mu);
  FreeBlock b{p, g_cur_stream, nullptr};
  if (g_have_stream) {
    cudaEvent_t ev = nullptr;
    if (!g_event_cache.empty()) {
      ev = g_event_cache.back();
      g_event_cache.pop_back();
    } else if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      ev = nullptr;
    }
    if (ev && cudaEventRecord(ev, g_cur_stream) == cudaSuccess) {
      b.ev = ev;
    } else {  // no event: wait for the stream instead of handing out a block in use
      cudaGetLastError();
      if (ev) g_event_cache.push_back(ev);
      cudaStreamSynchronize(g_cur_stream);
      cudaGetLastError();
    }
  }
  g_pool.emplace(size_class(bytes), b);
}

void mask::pool_trim() {
  std::lock_guard<std::mutex> g(g_pool_mu);
  for (auto it = g_pool.begin(); it != g_pool.end();) {
    FreeBlock& b = it->second;
    if (b.ev && cudaEventQuery(b.ev) == cudaErrorNotReady) {  // still in use by a stream
      ++it;
      continue;
    }
    cudaGetLastError();
    if (b.ev) g_event_cache.push_back(b.ev);
    cudaFree(b.p);
    it = g_pool.erase(it);
  }
}

namespace {

thread_local std::string g_err;

// the stream the pool orders this thread's releases on (set by as_stream inside a call)
struct StreamCtx {  // saved / restored so a nested entry point leaves the caller's context intact
  bool have = g_have_stream;
  cudaStream_t st = g_cur_stream;
  StreamCtx() { g_have_stream = false; }
  ~StreamCtx() {
    g_have_stream = have;
    g_cur_stream = st;
  }
};

template <class F>
int32_t guarded(F&& f) {
  StreamCtx sc;
  try {
    g_err.clear();
    f();
    return MASK_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return MASK_ERR_OOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MASK_ERR_CUDA;
  }
}

// NVTX ranges around the API calls and levels (free when no profiler is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

#define MASK_NCCL(x)                                                                     \
  do {                                                                                   \
    g_nccl_calls.fetch_add(1, std::memory_order_relaxed);                               \
    ncclResult_t r_ = (x);                                                               \
    if (r_ != ncclSuccess)                                                               \
      ::mask::fail(MASK_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_));      \
  } while (0)

// Pinned host scratch for per-pass statistics (one 64-byte block per thread, kept for the
// life of the thread so builds do not pay a pinned allocation).
struct HostStats {
  double* J = nullptr;
  unsigned long long* changed = nullptr;
  uint32_t* fin = nullptr;
  int32_t* flags = nullptr;
  HostStats() {
    thread_local void* base = nullptr;
    if (!base) MASK_CUDA(cudaMallocHost(&base, 64));
    J = reinterpret_cast<double*>(base);
    changed = reinterpret_cast<unsigned long long*>(static_cast<char*>(base) + 8);
    fin = reinterpret_cast<uint32_t*>(static_cast<char*>(base) + 16);
    flags = reinterpret_cast<int32_t*>(static_cast<char*>(base) + 24);
  }
};

}  // namespace

struct mask_comm {
  ncclComm_t comm = nullptr;           // NCCL transport (one GPU per rank)
  mask_host_collective_fn host = nullptr;  // host transport (mask_comm_init_host), or nullptr
  void* host_user = nullptr;
  bool host_failed = false;
  int world = 1;
  int rank = 0;
  bool usable() const { return host ? !host_failed : comm != nullptr; }
};

namespace {

// ---- collectives over either transport.  NCCL: enqueued on the build stream (the path every
// GPU count runs).  Host transport (mask_comm_init_host, the multi-rank tests on one GPU): the
// stream is drained, the buffer staged through host memory, the caller's function exchanges
// it, and the result is copied back -- the same call sequence, so every world > 1 branch of
// mask_build runs.
enum CollType { kF32 = MASK_COLL_F32, kF64 = MASK_COLL_F64, kI32 = MASK_COLL_I32, kI64 = MASK_COLL_I64,
                kU64 = MASK_COLL_U64 };
size_t coll_size(CollType t) { return (t == kF32 || t == kI32) ? 4 : 8; }
ncclDataType_t coll_nccl(CollType t) {
  switch (t) {
    case kF32: return ncclFloat;
    case kF64: return ncclDouble;
    case kI32: return ncclInt32;
    case kI64: return ncclInt64;
    default: return ncclUint64;
  }
}

void host_call(mask_comm* c, int kind, void* buf, const void* send, size_t count, CollType t, int arg) {
  g_nccl_calls.fetch_add(1, std::memory_order_relaxed);
  const int32_t r = c->host(kind, buf, send, (int64_t)count, (int32_t)t, arg, c->host_user);
  if (r != 0) {
    c->host_failed = true;
    ::mask::fail(MASK_ERR_NCCL, "host collective failed (code " + std::to_string(r) + ")");
  }
}

void coll_allreduce(mask_comm* c, void* dev, size_t count, CollType t, bool max_op, cudaStream_t st) {
  if (!c->host) {
    MASK_NCCL(ncclAllReduce(dev, dev, count, coll_nccl(t), max_op ? ncclMax : ncclSum, c->comm, st));
    return;
  }
  std::vector<char> h(count * coll_size(t));
  MASK_CUDA(cudaMemcpyAsync(h.data(), dev, h.size(), cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaStreamSynchronize(st));
  host_call(c, MASK_COLL_ALLREDUCE, h.data(), nullptr, count, t, max_op ? MASK_COLL_MAX : MASK_COLL_SUM);
  MASK_CUDA(cudaMemcpyAsync(dev, h.data(), h.size(), cudaMemcpyHostToDevice, st));
  MASK_CUDA(cudaStreamSynchronize(st));
}

// recv <- root's send (send is read on the root only; may alias recv)
void coll_broadcast(mask_comm* c, const void* send, void* recv, size_t count, CollType t, int root, cudaStream_t st) {
  if (!c->host) {
    MASK_NCCL(ncclBroadcast(send, recv, count, coll_nccl(t), root, c->comm, st));
    return;
  }
  std::vector<char> h(count * coll_size(t));
  if (c->rank == root && count) {
    MASK_CUDA(cudaMemcpyAsync(h.data(), send, h.size(), cudaMemcpyDeviceToHost, st));
    MASK_CUDA(cudaStreamSynchronize(st));
  }
  host_call(c, MASK_COLL_BROADCAST, h.data(), nullptr, count, t, root);
  if (count) {
    MASK_CUDA(cudaMemcpyAsync(recv, h.data(), h.size(), cudaMemcpyHostToDevice, st));
    MASK_CUDA(cudaStreamSynchronize(st));
  }
}

// recv[r * count ...] <- rank r's send (count elements each)
void coll_allgather(mask_comm* c, const void* send, void* recv, size_t count, CollType t, cudaStream_t st) {
  if (!c->host) {
    MASK_NCCL(ncclAllGather(send, recv, count, coll_nccl(t), c->comm, st));
    return;
  }
  std::vector<char> hs(count * coll_size(t)), hr(count * coll_size(t) * c->world);
  MASK_CUDA(cudaMemcpyAsync(hs.data(), send, hs.size(), cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaStreamSynchronize(st));
  host_call(c, MASK_COLL_ALLGATHER, hr.data(), hs.data(), count, t, 0);
  MASK_CUDA(cudaMemcpyAsync(recv, hr.data(), hr.size(), cudaMemcpyHostToDevice, st));
  MASK_CUDA(cudaStreamSynchronize(st));
}

// ncclGroupStart/End around a batch of collectives (no-op for the host transport, whose
// calls complete one by one in the same order on every rank)
struct CollGroup {
  mask_comm* c;
  explicit CollGroup(mask_comm* cm) : c(cm) {
    if (!c->host) MASK_NCCL(ncclGroupStart());
  }
  void end() {
    if (c && !c->host) MASK_NCCL(ncclGroupEnd());
    c = nullptr;
  }
  ~CollGroup() {
    if (c && !c->host) ncclGroupEnd();  // unwinding: close the group, error already raised
  }
};

}  // namespace

namespace {

struct Level {
  int64_t n_items = 0;  // items clustered at this level (level 1: n_global)
  int64_t k = 0;
  int dim = 0;
  DevBuf<float> P;            // k x dim
  DevBuf<int32_t> labels;     // n_items
  DevBuf<int64_t> offsets;    // k + 1
  DevBuf<int32_t> members;    // n_items
  std::vector<double> J;
  std::vector<int64_t> changed, empties;
  std::vector<double> dmax;  // per pass: max_j ||c_j' - c_j|| of the update that followed
  int updates = 0;
  double t_ms[MASK_T_NCLASS] = {0, 0, 0, 0};
  int64_t t_count[MASK_T_NCLASS] = {0, 0, 0, 0};
  int assign_kernel = -1;  // 0 = K2 SIMT, 1 = K1 tcgen05 3xTF32, 2 = K3 CSR, 3 = K11 fused small level,
                           // 4 = K12 grouped, 5 = K3T CSR hot block on tcgen05, 6 = K1 3xFP16
  // MASK_TRACE_PASSES: slot t < T = loop pass t, slot T = the final pass (T + 1 slots)
  DevBuf<float> P_trace;        // (T+1) x k x dim
  DevBuf<int32_t> lab_trace;    // (T+1) x n_items (this rank's items)
  int trace_T = -1;             // T of the traced build (-1: no trace)
  int trace_loop_passes = 0;    // loop passes run (the final pass follows them)
  int64_t trace_n = 0;          // items per label slot
};

// A level's input rows as seen by this rank.
struct Input {
  int format = MASK_DENSE_F32;
  int dim = 0;
  int64_t n_local = 0, n_global = 0, row_offset = 0;
  const float* X = nullptr;
  const int64_t* rp = nullptr;
  const int32_t* col = nullptr;
  const float* val = nullptr;
  int64_t nnz = 0;
};

}  // namespace

struct mask_index {
  int dim = 0;
  int format = MASK_DENSE_F32;
  int64_t n_global = 0;
  // data rows for leaf scans (global row ids)
  const float* X = nullptr;
  const int64_t* rp = nullptr;
  const int32_t* col = nullptr;
  const float* val = nullptr;
  DevBuf<float> own_X, own_val;
  DevBuf<float> Xpart;  // dense rows in level-1 partition order (leaf scans of mask_query)
  // Pchild[l]: level-(l+1) prototypes in level-(l+2) child-list order (the descent's contiguous
  // child scans; dense indexes, l < L - 1; empty entries: none kept)
  std::vector<DevBuf<float>> Pchild;
  DevBuf<int64_t> own_rp;
  DevBuf<int32_t> own_col;
  std::vector<Level> levels;
  // sparse-query support: ||c||^2 per level, flattened
  DevBuf<float> cn2_flat;
  DevBuf<int64_t> cn2_off;
  // range search (K13): cover radii per level, computed on the first MASK_RANGE_COVER query
  // (and again after an insertion)
  mutable std::mutex cover_mu;
  mutable bool cover_valid = false;
  mutable std::vector<DevBuf<unsigned>> cover;
};

namespace {

// The call's stream; also the stream the caching pool orders this thread's releases on.
cudaStream_t as_stream(void* s) {
  g_cur_stream = reinterpret_cast<cudaStream_t>(s);
  g_have_stream = true;
  return g_cur_stream;
}

void check_matrix(const mask_matrix* m, const char* what) {
  MASK_REQUIRE(m != nullptr, MASK_ERR_ARG, std::string(what) + ": NULL matrix");
  MASK_REQUIRE(m->format == MASK_DENSE_F32 || m->format == MASK_CSR_F32, MASK_ERR_ARG,
               std::string(what) + ": unknown format");
  MASK_REQUIRE(m->memory == MASK_MEM_DEVICE || m->memory == MASK_MEM_HOST, MASK_ERR_ARG,
               std::string(what) + ": unknown memory kind");
  MASK_REQUIRE(m->dim >= 1, MASK_ERR_ARG, std::string(what) + ": dim must be >= 1");
  MASK_REQUIRE(m->rows >= 0, MASK_ERR_ARG, std::string(what) + ": rows must be >= 0");
  MASK_REQUIRE(m->rows < (int64_t(1) << 31), MASK_ERR_UNSUPPORTED,
               std::string(what) + ": rows must be < 2^31");
  if (m->rows > 0) MASK_REQUIRE(m->values != nullptr, MASK_ERR_ARG, std::string(what) + ": NULL values");
  if (m->format == MASK_CSR_F32) {
    MASK_REQUIRE(m->row_ptr != nullptr && (m->nnz == 0 || m->col_idx != nullptr), MASK_ERR_ARG,
                 std::string(what) + ": NULL CSR arrays");
    MASK_REQUIRE(m->nnz >= 0, MASK_ERR_ARG, std::string(what) + ": nnz < 0");
  }
}

// CSR structure check (sorted, unique, in range) of device arrays: one kernel, one 4-byte read.
void check_csr_device(const int64_t* rp, const int32_t* col, int64_t rows, int64_t nnz, int dim, cudaStream_t st) {
  DevBuf<int> err(1);
  launch_check_csr(rp, col, rows, nnz, dim, err.p, st);
  int h = 0;
  MASK_CUDA(cudaMemcpyAsync(&h, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaStreamSynchronize(st));
  MASK_REQUIRE(!(h & 1), MASK_ERR_ARG, "CSR: row_ptr[0] must be 0, non-decreasing, row_ptr[rows] == nnz");
  MASK_REQUIRE(!(h & 2), MASK_ERR_ARG, "CSR: column index out of range");
  MASK_REQUIRE(!(h & 4), MASK_ERR_ARG, "CSR: columns not strictly increasing in a row");
}

// Host-side CSR structure check of host arrays (argument validation before any device work;
// device arrays are checked on the device by check_csr_device).
void check_host_csr(const mask_matrix* m) {
  const int64_t* rp = m->row_ptr;
  const int32_t* col = m->col_idx;
  MASK_REQUIRE(rp[0] == 0 && rp[m->rows] == m->nnz, MASK_ERR_ARG, "CSR: row_ptr[0] must be 0 and row_ptr[rows] == nnz");
  for (int64_t r = 0; r < m->rows; ++r) {
    MASK_REQUIRE(rp[r + 1] >= rp[r], MASK_ERR_ARG, "CSR: row_ptr not non-decreasing");
    for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
      MASK_REQUIRE(col[p] >= 0 && col[p] < m->dim, MASK_ERR_ARG, "CSR: column index out of range");
      if (p > rp[r]) MASK_REQUIRE(col[p] > col[p - 1], MASK_ERR_ARG, "CSR: columns not strictly increasing in a row");
    }
  }
}

// Scratch of one level's Lloyd loop.
struct LloydWS {
  DevBuf<int32_t> lab_prev, lab_cur;
  DevBuf<int32_t> lab2;  // K1 second-best prototype of each row (pruning bound of the next pass)
  DevBuf<int32_t> perm, sort_cnt;  // rows sorted by the last pass's labels (update + next K1)
  DevBuf<int32_t> perm_old;        // the sort before (visit order of the next sort)
  bool have_prev = false;          // lab_prev holds a complete labeling (pass >= 1)
  bool have_perm = false;          // perm is sorted by lab_prev's labels
  DevBuf<float> best;
  DevBuf<float> S;
  DevBuf<int32_t> counts;
  DevBuf<float> Pb, Ps, cn2, xn2, PT;
  DevBuf<int32_t> flag_rows, flag_count;
  DevBuf<int2> flag_pair;                     // K1 -> K4: the two candidates of a flagged row
  DevBuf<double> P64;  // FP64 prototypes of a dense per-pass level (D15); nullptr otherwise
  DevBuf<double> S64;  // their FP64 sums (+ the packed counts / J / changed tail for N1)
  DevBuf<double> P64T; // K4 re-scan: dimension-major copy of P64
  DevBuf<int32_t> rescan_rows, rescan_count;  // K4: flagged rows that need the full re-check
  DevBuf<unsigned long long> fix_keys;
  DevBuf<int16_t> colslot;  // K3 chunk-major: hot slot of each column (-1 = read from L2)
  DevBuf<int32_t> hotcols;  // the hot columns (most non-zeros)
  DevBuf<float2> csr_state; // running argmin across prototype chunks
  // K3T (CSR, hot columns on tcgen05): per level the dense hot block, the tail non-zeros and
  // their counts; per pass the split hot prototype slice, ||c||^2 (+inf padded), padded PT
  DevBuf<float> k3_Xh, k3_Hb, k3_Hs, k3_cn2, k3_PT;
  DevBuf<int2> k3_tail;
  DevBuf<int32_t> k3_ntail;
  // K1 3xFP16 (d = 64 / 128): per-level scale of the data, per-pass FP16 split of s (-2c)
  DevBuf<uint16_t> h16_b, h16_s;
  float h16_scale = 1.f, h16_err_abs = 0.f;
  bool xn2_ready = false;
  int kernel_id = -1;
};

// CUDA-event pairs recorded around every launch of a kernel class during a level, read once
// at the end of the level (no synchronisation inside the loop).  Only the first `executed`
// pairs of a class count (passes skipped on the device after convergence are excluded).
struct EventLog {
  std::vector<cudaEvent_t> ev[MASK_T_NCLASS];
  unsigned classes;  // bit c: class c is timed (MASK_TIME_ASSIGN: the assignment class only)
  explicit EventLog(unsigned cls) : classes(cls) {}
  ~EventLog() {
    for (auto& v : ev)
      for (auto e : v) cudaEventDestroy(e);
  }
  void mark(int c, cudaStream_t st) {
    if (!(classes & (1u << c))) return;
    cudaEvent_t e;
    MASK_CUDA(cudaEventCreate(&e));
    MASK_CUDA(cudaEventRecord(e, st));
    ev[c].push_back(e);
  }
  // sum of the first `pairs` (start, stop) intervals of class c
  double total_ms(int c, size_t pairs) const {
    double ms = 0.0;
    for (size_t i = 0; i + 1 < ev[c].size() && i / 2 < pairs; i += 2) {
      float t = 0.f;
      MASK_CUDA(cudaEventElapsedTime(&t, ev[c][i], ev[c][i + 1]));
      ms += t;
    }
    return ms;
  }
  size_t pairs(int c) const { return ev[c].size() / 2; }
};

// One assignment pass: labels_out[i] = argmin_j ||x_i - c_j||^2, best[i] = its d^2.
// `active` (device, may be NULL): the pass is a no-op on the device once the level converged.
void assign_pass(const Input& in, const float* P, int64_t k, int flags, int32_t* labels_out, float* best,
                 LloydWS& ws, cudaStream_t st, const int* active, EventLog* ev) {
  const int64_t n = in.n_local;
  const int d = in.dim;
  if (n == 0) return;
  if (in.format == MASK_CSR_F32 && (flags & MASK_CSR_TC) && !(flags & MASK_FORCE_SIMT)) {
    // K3T (opt-in): hot columns on tcgen05 (3xTF32), tail non-zeros in the epilogue (DESIGN.md §6 K3T)
    const int H = csr_tc_hot();
    const int64_t kr = csr_tc_rows(k);
    if (!ws.k3_Xh.p) {  // per level: hot set, dense hot block, tail lists, ||x||^2
      DevBuf<int32_t> cnt(d);
      launch_col_hist(in.col, in.nnz, d, cnt.p, st);
      ws.colslot.alloc(d);
      ws.hotcols.alloc(H);
      launch_select_hot(cnt.p, d, H, ws.hotcols.p, ws.colslot.p, st);
      ws.k3_Xh.alloc((size_t)n * H);
      ws.k3_tail.alloc((size_t)std::max<int64_t>(in.nnz, 1));
      ws.k3_ntail.alloc(n);
      ws.xn2.alloc(n);
      launch_csr_tc_level(in.rp, in.col, in.val, n, ws.colslot.p, ws.k3_Xh.p, ws.k3_tail.p, ws.k3_ntail.p, ws.xn2.p,
                          st);
      ws.k3_Hb.alloc((size_t)kr * H);
      ws.k3_Hs.alloc((size_t)kr * H);
      ws.k3_cn2.alloc(kr);
      ws.k3_PT.alloc((size_t)kr * d);
    }
    launch_csr_tc_prep(P, k, d, ws.hotcols.p, ws.k3_Hb.p, ws.k3_Hs.p, ws.k3_cn2.p, ws.k3_PT.p, st, active);
    ws.kernel_id = 5;
    if (ev) ev->mark(MASK_T_ASSIGN, st);
    launch_assign_csr_tc(ws.k3_Xh.p, in.rp, ws.k3_tail.p, ws.k3_ntail.p, ws.xn2.p, n, ws.k3_Hb.p, ws.k3_Hs.p,
                         ws.k3_PT.p, ws.k3_cn2.p, k, labels_out, best, st, active);
    if (ev) ev->mark(MASK_T_ASSIGN, st);
    return;
  }
  if (in.format == MASK_CSR_F32) {
    if (!ws.PT.p) ws.PT.alloc((size_t)k * d);
    if (!ws.cn2.p) ws.cn2.alloc(k);
    launch_transpose(P, k, d, ws.PT.p, st, active);
    launch_level_norms(P, k, d, ws.cn2.p, st, active);
    ws.kernel_id = 2;
    const bool chunked = csr_chunked_supported(d, k) && !(flags & MASK_FORCE_SIMT);
    if (chunked && !ws.colslot.p) {
      // hot set = the csr_chunked_hot() columns with the most non-zeros (selected on the device)
      DevBuf<int32_t> cnt(d);
      launch_col_hist(in.col, in.nnz, d, cnt.p, st);
      const int H = csr_chunked_hot();
      ws.colslot.alloc(d);
      ws.hotcols.alloc(H);
      ws.csr_state.alloc(std::max<int64_t>(n, 1));
      launch_select_hot(cnt.p, d, H, ws.hotcols.p, ws.colslot.p, st);
    }
    if (ev) ev->mark(MASK_T_ASSIGN, st);
    if (chunked)
      launch_assign_csr_chunked(in.rp, in.col, in.val, n, d, ws.PT.p, ws.cn2.p, k, ws.colslot.p, ws.hotcols.p,
                                ws.csr_state.p, labels_out, best, st, active);
    else
      launch_assign_csr(in.rp, in.col, in.val, n, d, ws.PT.p, ws.cn2.p, k, labels_out, best, st, active);
    if (ev) ev->mark(MASK_T_ASSIGN, st);
    return;
  }
  const bool use_tc = !(flags & MASK_FORCE_SIMT) && tc_supported(n, d, k) && ((uintptr_t)in.X % 16 == 0);
  if (!use_tc) {
    ws.kernel_id = 0;
    if (d > 64 && (int64_t)ws.fix_keys.n < n) ws.fix_keys.alloc((size_t)n);
    if (ev) ev->mark(MASK_T_ASSIGN, st);
    if (d <= 64) launch_assign_simt(in.X, n, d, P, k, labels_out, best, st, active);
    else launch_assign_blocked(in.X, n, d, P, k, ws.fix_keys.p, labels_out, best, st, active);  // large d
    if (ev) ev->mark(MASK_T_ASSIGN, st);
    return;
  }
  // ||c||^2 is padded with +inf to a whole number of 256-prototype tiles (K1 reads it unmasked)
  const int64_t k_pad = (k + 255) / 256 * 256;
  const int kc = tc_operand_cols(d);
  if (!ws.Pb.p) {
    ws.Pb.alloc((size_t)tc_operand_rows(k) * kc);
    ws.Ps.alloc((size_t)tc_operand_rows(k) * kc);
    ws.cn2.alloc(tc_operand_rows(k));  // +inf beyond k: the epilogue reads whole tiles
    ws.flag_rows.alloc(n);
    ws.flag_pair.alloc(n);
    ws.rescan_rows.alloc(n);
    ws.rescan_count.alloc(1);
    ws.flag_count.alloc(1);
    ws.fix_keys.alloc((size_t)n);
    launch_fill(ws.cn2.p + k, tc_operand_rows(k) - k, INFINITY, st);
    ws.lab2.alloc(n);
    MASK_CUDA(cudaMemsetAsync(ws.lab2.p, 0xff, sizeof(int32_t) * n, st));
  }
  const bool h16 = tc_h16_enabled() && (d == 64 || d == 128) && !(flags & MASK_TC_TF32);
  if (!ws.xn2_ready) {
    ws.xn2.alloc(n);
    launch_row_norms(in.X, n, d, ws.xn2.p, st);
    ws.xn2_ready = true;
    if (h16) {  // one host read per level: max |x| -> the FP16 scale and the subnormal error term
      float maxabs = 0.f;
      ws.h16_scale = h16_level_scale(in.X, n * (int64_t)d, &maxabs, st);
      // a score's absolute error from FP16 subnormal parts <= 2^-25 / s per operand element:
      // sum_i (|dx_i| |2c_i| + |x_i| |d(2c)_i|) <= 3 d maxabs 2^-25 / s; doubled for a gap
      ws.h16_err_abs = (float)(6.0 * d * (double)maxabs * std::ldexp(1.0, -25) / ws.h16_scale);
      ws.h16_b.alloc((size_t)tc_operand_rows(k) * d);
      ws.h16_s.alloc((size_t)tc_operand_rows(k) * d);
      MASK_CUDA(cudaMemsetAsync(ws.h16_b.p, 0, sizeof(uint16_t) * tc_operand_rows(k) * d, st));
      MASK_CUDA(cudaMemsetAsync(ws.h16_s.p, 0, sizeof(uint16_t) * tc_operand_rows(k) * d, st));
    }
  }
  launch_prep_protos(P, k, d, kc, ws.Pb.p, ws.Ps.p, ws.cn2.p, st, tc_operand_rows(k), d <= 24 ? 1 : 0, active,
                     ws.flag_count.p, ws.P64.p);
  const bool h16_on = h16 && ws.h16_b.p;
  if (h16_on) launch_prep_h16(P, ws.P64.p, k, d, ws.h16_scale, ws.h16_b.p, ws.h16_s.p, st, active);
  ws.kernel_id = h16_on ? 6 : 1;
  if (ev) ev->mark(MASK_T_ASSIGN, st);
  // small d (persistent K1): visit rows grouped by their previous label (perm, sorted after
  // the previous pass), so the rows of a warp share their nearest prototypes and the
  // bound-pruned epilogue skips most chunks warp-wide
  const int32_t* perm = (ws.have_perm && !(flags & MASK_NO_SORT)) ? ws.perm.p : nullptr;
  launch_assign_tc(in.X, n, d, P, ws.Pb.p, ws.Ps.p, ws.cn2.p, k, ws.xn2.p, labels_out, best, ws.flag_rows.p,
                   ws.flag_count.p, st, active, perm, ws.have_prev ? ws.lab_prev.p : nullptr, ws.lab2.p,
                   ws.flag_pair.p, h16_on ? ws.h16_b.p : nullptr, h16_on ? ws.h16_s.p : nullptr, ws.h16_scale,
                   ws.h16_err_abs);
  if (ev) ev->mark(MASK_T_ASSIGN, st);
  // near-tie re-check (K4), sized on the device from the flagged count (no host round trip)
  if (!(flags & MASK_NO_FIXUP)) {
    if (ev) ev->mark(MASK_T_FIXUP, st);
    launch_fixup_device(in.X, d, P, k, ws.flag_rows.p, ws.flag_count.p, n, ws.fix_keys.p, labels_out, best, st,
                        active, ws.flag_pair.p, ws.rescan_rows.p, ws.rescan_count.p, ws.P64.p, ws.P64T.p);
    if (ev) ev->mark(MASK_T_FIXUP, st);
  }
}

// ---- N1 packing: one fp32 allreduce per pass carries the sums, the counts and the pass stats.
// An integer v is sent as (v >> 12, v & 4095): each half's sum over the ranks stays below 2^24
// (n < 2^36 rows, < 4096 ranks), so the fp32 sums are exact.  J (double) as hi + lo floats.
__global__ void k_pack_pass(const int32_t* __restrict__ counts, int64_t k, const double* __restrict__ J,
                            const unsigned long long* __restrict__ ch, float* __restrict__ tail,
                            const int* __restrict__ active) {
  if (active && !*active) return;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = counts[j];
    tail[j] = (float)(c >> 12);
    tail[k + j] = (float)(c & 4095);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const double v = *J;
    const float hi = (float)v;
    tail[2 * k] = hi;
    tail[2 * k + 1] = (float)(v - (double)hi);
    const unsigned long long c = *ch;
    tail[2 * k + 2] = (float)(c >> 12);
    tail[2 * k + 3] = (float)(c & 4095ull);
  }
}
// inverse of k_pack_pass on the combined buffer; with ctrl: the no-change stop test of pass t
__global__ void k_unpack_pass(const float* __restrict__ tail, int64_t k, int32_t* __restrict__ counts,
                              double* __restrict__ J, unsigned long long* __restrict__ ch, int* ctrl, int t,
                              const int* __restrict__ active) {
  if (active && !*active) return;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x)
    counts[j] = (int32_t)tail[j] * 4096 + (int32_t)tail[k + j];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *J = (double)tail[2 * k] + (double)tail[2 * k + 1];
    const unsigned long long c = (unsigned long long)tail[2 * k + 2] * 4096ull + (unsigned long long)tail[2 * k + 3];
    *ch = c;
    if (ctrl && t > 0 && c == 0) {  // no label changed anywhere: stop before the update (D3)
      ctrl[0] = 0;
      ctrl[1] = t + 1;
    }
  }
}
void launch_pack_pass(const int32_t* counts, int64_t k, const double* J, const unsigned long long* ch, float* tail,
                      cudaStream_t st, const int* active) {
  k_pack_pass<<<grid_for(std::max<int64_t>(k, 1), 256), 256, 0, st>>>(counts, k, J, ch, tail, active);
  MASK_LAUNCH_CHECK();
}
void launch_unpack_pass(const float* tail, int64_t k, int32_t* counts, double* J, unsigned long long* ch, int* ctrl,
                        int t, cudaStream_t st, const int* active) {
  k_unpack_pass<<<grid_for(std::max<int64_t>(k, 1), 256), 256, 0, st>>>(tail, k, counts, J, ch, ctrl, t, active);
  MASK_LAUNCH_CHECK();
}
// FP64 levels: the pass's N1 buffer is FP64 throughout, [S (k x d) | counts (k) | J | changed]
// (integers exact below 2^53)
__global__ void k_pack_pass64(const int32_t* __restrict__ counts, int64_t k, const double* __restrict__ J,
                              const unsigned long long* __restrict__ ch, double* __restrict__ tail,
                              const int* __restrict__ active) {
  if (active && !*active) return;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x)
    tail[j] = (double)counts[j];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    tail[k] = *J;
    tail[k + 1] = (double)*ch;
  }
}
__global__ void k_unpack_pass64(const double* __restrict__ tail, int64_t k, int32_t* __restrict__ counts,
                                double* __restrict__ J, unsigned long long* __restrict__ ch, int* ctrl, int t,
                                const int* __restrict__ active) {
  if (active && !*active) return;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x)
    counts[j] = (int32_t)tail[j];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *J = tail[k];
    const unsigned long long c = (unsigned long long)tail[k + 1];
    *ch = c;
    if (ctrl && t > 0 && c == 0) {
      ctrl[0] = 0;
      ctrl[1] = t + 1;
    }
  }
}
__global__ void k_copy_labels(int32_t* __restrict__ dst, const int32_t* __restrict__ src, int64_t n,
                              const int* __restrict__ active) {
  if (active && !*active) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// Lloyd k-means for one level (SURVEY §8(c) pseudo-code; mirrors the oracle's order):
//   P <- init rows; for t < T: a <- assign(P); trace; stop if no label changed (t > 0);
//   P <- means (empty keeps, D5); stop if tol > 0 and max displacement <= tol;
//   final assignment -> labels.
// The whole loop is enqueued at once: the stop tests run on the device (k_unpack_pass with a
// communicator, the last blocks of k_pass_stats / k_finalize) and later passes become no-ops, so the host synchronises once per level
// (unless the test-only iteration callback needs host copies after every pass).
// After a host synchronisation of a communicator build: a failed or hung peer surfaces as an
// asynchronous NCCL error; abort the communicator (every later collective returns at once) and
// fail the call with MASK_ERR_NCCL instead of waiting forever.
void check_comm(mask_comm* comm) {
  if (!comm || comm->host) return;
  ncclResult_t ar = ncclSuccess;
  const ncclResult_t r = ncclCommGetAsyncError(comm->comm, &ar);
  if (r != ncclSuccess || ar != ncclSuccess) {
    ncclCommAbort(comm->comm);
    comm->comm = nullptr;
    ::mask::fail(MASK_ERR_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(r != ncclSuccess ? r : ar));
  }
}

void run_level(const Input& in, int64_t k, const int64_t* init_idx_host, const mask_build_params* p,
               mask_comm* comm, int level_no, cudaStream_t st, Level& L, HostStats& hs) {
  char nv[32];
  std::snprintf(nv, sizeof(nv), "mask level %d", level_no);
  NvtxRange range(nv);
  const int d = in.dim;
  const int64_t n = in.n_local;
  const int T = p->max_iters;
  L.k = k;
  L.dim = d;
  L.P.alloc((size_t)k * d);
  LloydWS ws;
  ws.lab_prev.alloc(std::max<int64_t>(n, 1));
  ws.lab_cur.alloc(std::max<int64_t>(n, 1));
  ws.best.alloc(std::max<int64_t>(n, 1));
  // dense levels run by the per-pass kernels keep FP64 prototypes and sums (D15): the K4
  // decisions and the update then follow the oracle's FP64 arithmetic; fp32 P is their rounding
  const bool farthest = p->empty_policy == MASK_EMPTY_FARTHEST;
  const bool fused_level = in.format == MASK_DENSE_F32 && !comm && !p->iter_cb && !(p->flags & MASK_FORCE_SIMT) &&
                           !(p->flags & MASK_NO_FUSED) && !farthest && small_level_supported(n, d, k);
  const bool p64 = in.format == MASK_DENSE_F32 && !fused_level;
  if (p64) {
    ws.P64.alloc((size_t)k * d);
    ws.P64T.alloc((size_t)k * d);
    ws.S64.alloc((size_t)k * d + (size_t)k + 2);
  } else {
    ws.S.alloc((size_t)k * d + (comm ? 2 * (size_t)k + 8 : 0));  // + the packed tail (N1)
  }
  ws.counts.alloc(k);
  // per-pass statistics (slot T+1 = final pass) and loop control
  DevBuf<double> Jd(T + 2);
  DevBuf<unsigned long long> chd(T + 2);
  DevBuf<uint32_t> fin(2 * (T + 2));
  DevBuf<int> ctrl(4);
  MASK_CUDA(cudaMemsetAsync(Jd.p, 0, sizeof(double) * (T + 2), st));
  MASK_CUDA(cudaMemsetAsync(chd.p, 0, sizeof(unsigned long long) * (T + 2), st));
  MASK_CUDA(cudaMemsetAsync(fin.p, 0, sizeof(uint32_t) * 2 * (T + 2), st));
  const int ctrl_init[4] = {1, 0, 0, 0};
  MASK_CUDA(cudaMemcpyAsync(ctrl.p, ctrl_init, sizeof(ctrl_init), cudaMemcpyHostToDevice, st));
  if (p64) MASK_CUDA(cudaMemsetAsync(ws.S64.p, 0, sizeof(double) * k * d, st));
  else MASK_CUDA(cudaMemsetAsync(ws.S.p, 0, sizeof(float) * k * d, st));
  MASK_CUDA(cudaMemsetAsync(ws.counts.p, 0, sizeof(int32_t) * k, st));
  MASK_CUDA(cudaMemsetAsync(ws.lab_prev.p, 0xff, sizeof(int32_t) * std::max<int64_t>(n, 1), st));
  const int* active = ctrl.p;
  const bool tracing = (p->flags & MASK_TRACE_PASSES) != 0;
  if (tracing) {
    L.P_trace.alloc((size_t)(T + 1) * k * d);
    L.lab_trace.alloc((size_t)(T + 1) * std::max<int64_t>(n, 1));
    L.trace_T = T;
    L.trace_n = n;
  }
  auto trace_P = [&](int slot) {
    if (tracing)
      MASK_CUDA(cudaMemcpyAsync(L.P_trace.p + (size_t)slot * k * d, L.P.p, sizeof(float) * k * d,
                                cudaMemcpyDeviceToDevice, st));
  };
  auto trace_labels = [&](int slot) {
    if (tracing && n)
      MASK_CUDA(cudaMemcpyAsync(L.lab_trace.p + (size_t)slot * n, ws.lab_cur.p, sizeof(int32_t) * n,
                                cudaMemcpyDeviceToDevice, st));
  };

  // ---- seeded init (D2): gather the owned init rows, combine across ranks
  DevBuf<int64_t> idx(k);
  MASK_CUDA(cudaMemcpyAsync(idx.p, init_idx_host, sizeof(int64_t) * k, cudaMemcpyHostToDevice, st));
  if (in.format == MASK_CSR_F32) {
    MASK_CUDA(cudaMemsetAsync(L.P.p, 0, sizeof(float) * k * d, st));
    launch_gather_csr_rows(in.rp, in.col, in.val, d, idx.p, k, in.row_offset, n, L.P.p, st);
  } else {
    launch_gather_rows(in.X, d, idx.p, k, in.row_offset, n, L.P.p, st);
  }
  if (comm) coll_allreduce(comm, L.P.p, (size_t)k * d, kF32, false, st);
  if (p64) launch_f32_to_f64(L.P.p, (int64_t)k * d, ws.P64.p, st);

  // every event pair costs a few microseconds of device time per pass (~5 % of a C2 build for
  // all four classes), so MASK_TIME_ASSIGN times the assignment kernel alone
  const unsigned ev_classes = (p->flags & MASK_TIME_KERNELS) ? (1u << MASK_T_NCLASS) - 1u
                              : (p->flags & MASK_TIME_ASSIGN) ? (1u << MASK_T_ASSIGN) : 0u;
  std::unique_ptr<EventLog> ev(ev_classes ? new EventLog(ev_classes) : nullptr);

  // test-only step-parity hook: host copies of the P_t a pass used and the labels it produced
  auto emit_cb = [&](int pass, const float* P_used, const int32_t* labels_dev) {
    std::vector<float> Ph((size_t)k * d);
    std::vector<int32_t> lh(n);
    MASK_CUDA(cudaMemcpyAsync(Ph.data(), P_used, sizeof(float) * Ph.size(), cudaMemcpyDeviceToHost, st));
    if (n) MASK_CUDA(cudaMemcpyAsync(lh.data(), labels_dev, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    MASK_CUDA(cudaStreamSynchronize(st));
    p->iter_cb(level_no, pass, Ph.data(), k, d, lh.data(), n, p->iter_cb_user);
  };
  DevBuf<float> P_snap;  // P used by the pass (only kept for the callback)
  if (p->iter_cb) P_snap.alloc((size_t)k * d);

  // pass statistics into slot `slot` (this rank's rows; with a communicator they are combined
  // in the pass's single allreduce below, or -- final pass -- in one small allreduce)
  auto pass_stats = [&](int slot, const int* act, LoopCtl lc) {
    launch_pass_stats(ws.lab_cur.p, ws.lab_prev.p, ws.best.p, n, Jd.p + slot, chd.p + slot, st, act, lc);
  };
  // multi-GPU combine (N1): ONE allreduce per Lloyd iteration of the packed fp32 buffer
  // [S (k x d) | counts split hi/lo (2k) | J hi/lo | changed hi/lo] (BASELINE north_star
  // "combined with a single NCCL allreduce"); the integer parts are split into 12-bit low
  // halves and the rest so every fp32 partial sum stays exact
  const size_t pack_tail = (size_t)k * d;
  auto combine = [&](int slot, int t, bool with_sums, const int* act) {
    if (p64) {  // FP64 buffer: [S | counts | J | changed], or the stats alone after the sums
      double* tail = ws.S64.p + (with_sums ? pack_tail : 0);
      const int64_t kk = with_sums ? k : 0;
      k_pack_pass64<<<grid_for(std::max<int64_t>(kk, 1), 256), 256, 0, st>>>(ws.counts.p, kk, Jd.p + slot,
                                                                           chd.p + slot, tail, act);
      MASK_LAUNCH_CHECK();
      coll_allreduce(comm, ws.S64.p, with_sums ? pack_tail + (size_t)k + 2 : 2, kF64, false, st);
      k_unpack_pass64<<<grid_for(std::max<int64_t>(kk, 1), 256), 256, 0, st>>>(tail, kk, ws.counts.p, Jd.p + slot,
                                                                             chd.p + slot, with_sums ? ctrl.p : nullptr,
                                                                             t, act);
      MASK_LAUNCH_CHECK();
      return;
    }
    // with sums: the whole buffer; stats only (final pass, S no longer needed): its first 4 floats
    float* tail = ws.S.p + (with_sums ? pack_tail : 0);
    const int64_t kk = with_sums ? k : 0;
    launch_pack_pass(ws.counts.p, kk, Jd.p + slot, chd.p + slot, tail, st, act);
    const size_t count = with_sums ? pack_tail + 2 * (size_t)k + 4 : 4;
    coll_allreduce(comm, ws.S.p, count, kF32, false, st);
    launch_unpack_pass(tail, kk, ws.counts.p, Jd.p + slot, chd.p + slot, with_sums ? ctrl.p : nullptr, t, st, act);
  };

  // small dense level without a communicator or step hook: the whole loop in one launch (K11)
  const bool fused = fused_level;
  if (fused) {
    DevBuf<unsigned> bar(2);
    DevBuf<double> S64((size_t)k * d);
    MASK_CUDA(cudaMemsetAsync(S64.p, 0, sizeof(double) * k * d, st));
    if (ev) ev->mark(MASK_T_ASSIGN, st);
    launch_small_level(in.X, n, d, k, L.P.p, ws.lab_cur.p, ws.lab_prev.p, ws.best.p, S64.p, ws.counts.p, Jd.p,
                       chd.p, fin.p, ctrl.p, bar.p, T, p->tol, st, tracing ? L.P_trace.p : nullptr,
                       tracing ? L.lab_trace.p : nullptr);
    if (ev) ev->mark(MASK_T_ASSIGN, st);
    ws.kernel_id = 3;
  }
  for (int t = 0; t < T && !fused; ++t) {
    if (p->iter_cb) MASK_CUDA(cudaMemcpyAsync(P_snap.p, L.P.p, sizeof(float) * k * d, cudaMemcpyDeviceToDevice, st));
    trace_P(t);  // (passes skipped on the device after convergence fill slots never read back)
    assign_pass(in, L.P.p, k, p->flags, ws.lab_cur.p, ws.best.p, ws, st, active, ev.get());
    trace_labels(t);
    LoopCtl lc;
    lc.t = t;
    lc.T = T;
    lc.tol = p->tol;
    if (!comm) lc.ctrl = ctrl.p;  // single GPU: stop test fused into the stats kernel
    pass_stats(t, active, lc);
    if (p->iter_cb) {  // host view of the control state (test-only path)
      int h[4];
      MASK_CUDA(cudaMemcpyAsync(h, ctrl.p, sizeof(h), cudaMemcpyDeviceToHost, st));
      MASK_CUDA(cudaStreamSynchronize(st));
      if (h[0] || h[1] == t + 1) emit_cb(t, P_snap.p, ws.lab_cur.p);
      if (!h[0]) break;
    }
    // ---- rows sorted by this pass's labels: run-accumulated update now, warp-coherent K1 rows
    // in the next pass (its previous labels are these)
    const bool sorted = !(p->flags & MASK_NO_SORT) && n >= 4096 &&
                        (in.format == MASK_DENSE_F32 || csr_sorted_update_supported(d));
    // (the sort also performs the lab_prev <- lab_cur copy; a skipped pass leaves the buffers
    // swapped on the host, which only changes a row order: every consumer accepts any order)
    if (sorted) {
      if (!ws.perm.p) {
        ws.perm.alloc(n);
        ws.perm_old.alloc(n);
        ws.sort_cnt.alloc(k);
        MASK_CUDA(cudaMemsetAsync(ws.sort_cnt.p, 0, sizeof(int32_t) * k, st));
      }
      std::swap(ws.perm, ws.perm_old);
      launch_label_sort(ws.lab_cur.p, n, k, ws.have_perm ? ws.perm_old.p : nullptr, ws.perm.p, ws.sort_cnt.p,
                        ws.lab_prev.p, st, active, /*cnt_zeroed=*/true);
      ws.have_perm = true;
    }
    // ---- update: S_j, n_j (K5/K6) -> allreduce (N1) -> P_j = S_j / n_j (K7)
    if (ev) ev->mark(MASK_T_UPDATE, st);
    if (in.format == MASK_CSR_F32 && sorted)
      launch_update_csr_sorted(in.rp, in.col, in.val, d, ws.perm.p, ws.lab_cur.p, ws.sort_cnt.p, n, k, ws.S.p,
                               ws.counts.p, st, active);
    else if (in.format == MASK_CSR_F32)
      launch_update_csr(in.rp, in.col, in.val, n, d, ws.lab_cur.p, ws.S.p, ws.counts.p, st, active);
    else if (p64 && sorted && update_seg64_supported(d) && ((uintptr_t)in.X % 16) == 0)
      launch_update_seg64(in.X, d, ws.perm.p, ws.lab_cur.p, ws.sort_cnt.p, n, ws.S64.p, ws.counts.p, st, active);
    else if (p64)
      launch_update_dense64(in.X, n, d, ws.lab_cur.p, ws.S64.p, ws.counts.p, st, active, sorted ? ws.perm.p : nullptr);
    else
      launch_update_dense(in.X, n, d, ws.lab_cur.p, k, ws.S.p, ws.counts.p, st, active,
                          sorted ? ws.perm.p : nullptr);
    if (ev) ev->mark(MASK_T_UPDATE, st);
    // the combined statistics decide the no-change stop identically on every rank (the update
    // of a pass that changed no label is then not applied: K7 is skipped, as in the oracle)
    if (comm) combine(t, t, true, active);
    if (farthest)  // D5b: between the update (counts) and K7 (which keeps the re-seeded rows)
      reseed_farthest(in.format == MASK_DENSE_F32 ? in.X : nullptr, in.rp, in.col, in.val, d, n, k, ws.best.p,
                      ws.counts.p, L.P.p, p64 ? ws.P64.p : nullptr, fin.p + 2 * t, active, st);
    if (ev) ev->mark(MASK_T_FINALIZE, st);
    LoopCtl lf = lc;
    lf.ctrl = ctrl.p;  // tolerance stop / pass count (fin is identical on every rank)
    lf.zero_cnt = sorted ? ws.sort_cnt.p : nullptr;
    if (p64) launch_finalize64(ws.P64.p, L.P.p, ws.S64.p, ws.counts.p, k, d, fin.p + 2 * t, st, active, lf);
    else launch_finalize(L.P.p, ws.S.p, ws.counts.p, k, d, fin.p + 2 * t, 0, st, active, lf);
    if (ev) ev->mark(MASK_T_FINALIZE, st);
    if (!sorted) {
      k_copy_labels<<<grid_for(n, 256), 256, 0, st>>>(ws.lab_prev.p, ws.lab_cur.p, n, active);
      MASK_LAUNCH_CHECK();
    }
    ws.have_prev = true;
    if (p->iter_cb) {
      int h[4];
      MASK_CUDA(cudaMemcpyAsync(h, ctrl.p, sizeof(h), cudaMemcpyDeviceToHost, st));
      MASK_CUDA(cudaStreamSynchronize(st));
      if (!h[0]) break;
    }
  }
  // ---- final assignment with the final prototypes (D3): always runs, stats into slot T+1
  if (!fused) {
    if (p->iter_cb) MASK_CUDA(cudaMemcpyAsync(P_snap.p, L.P.p, sizeof(float) * k * d, cudaMemcpyDeviceToDevice, st));
    trace_P(T);
    assign_pass(in, L.P.p, k, p->flags, ws.lab_cur.p, ws.best.p, ws, st, nullptr, ev.get());
    trace_labels(T);
    pass_stats(T + 1, nullptr, LoopCtl());
    if (comm) combine(T + 1, T + 1, false, nullptr);
  }

  // ---- one read-back per level: control state and the per-pass trace
  int h_ctrl[4];
  std::vector<double> hJ(T + 2);
  std::vector<unsigned long long> hch(T + 2);
  std::vector<uint32_t> hfin(2 * (T + 2));
  MASK_CUDA(cudaMemcpyAsync(h_ctrl, ctrl.p, sizeof(h_ctrl), cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaMemcpyAsync(hJ.data(), Jd.p, sizeof(double) * (T + 2), cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaMemcpyAsync(hch.data(), chd.p, sizeof(unsigned long long) * (T + 2), cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaMemcpyAsync(hfin.data(), fin.p, sizeof(uint32_t) * 2 * (T + 2), cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaStreamSynchronize(st));
  check_comm(comm);
  const int loop_passes = T > 0 ? h_ctrl[1] : 0;  // assignment passes run inside the loop
  int updates = 0;
  for (int t = 0; t < loop_passes; ++t) {
    L.J.push_back(hJ[t]);
    L.changed.push_back((int64_t)hch[t]);
    const bool updated = !(t > 0 && hch[t] == 0);  // a no-change pass stops before its update
    L.empties.push_back(updated ? (int64_t)hfin[2 * t + 1] : 0);
    float d2max;
    std::memcpy(&d2max, &hfin[2 * t], sizeof(d2max));
    L.dmax.push_back(updated ? std::sqrt((double)d2max) : 0.0);
    updates += updated ? 1 : 0;
  }
  L.J.push_back(hJ[T + 1]);
  L.changed.push_back((int64_t)hch[T + 1]);
  L.empties.push_back(0);
  L.dmax.push_back(0.0);
  L.updates = updates;
  L.trace_loop_passes = loop_passes;
  if (p->iter_cb) emit_cb(loop_passes, P_snap.p, ws.lab_cur.p);
  L.labels = std::move(ws.lab_cur);
  L.n_items = n;
  L.assign_kernel = ws.kernel_id;
  if (ev) {
    // loop launches of a class: one per executed pass (+ the final pass for assign/fixup)
    const size_t run_assign = (size_t)loop_passes + 1, run_upd = (size_t)updates;
    const size_t runs[MASK_T_NCLASS] = {run_assign, run_assign, run_upd, run_upd};
    for (int c = 0; c < MASK_T_NCLASS; ++c) {
      const size_t np = ev->pairs(c);
      if (!np) continue;
      // the final pass's pair is the last one recorded; loop pairs are the first ones
      size_t loop_pairs = (c <= MASK_T_FIXUP) ? std::min(np - 1, runs[c] - 1) : std::min(np, runs[c]);
      double ms = ev->total_ms(c, loop_pairs);
      int64_t cnt = (int64_t)loop_pairs;
      if (c <= MASK_T_FIXUP) {  // add the final pass
        float t = 0.f;
        MASK_CUDA(cudaEventElapsedTime(&t, ev->ev[c][2 * (np - 1)], ev->ev[c][2 * (np - 1) + 1]));
        ms += t;
        cnt += 1;
      }
      L.t_ms[c] += ms;
      L.t_count[c] += cnt;
    }
  }
}

// Gather per-rank row blocks into one n_global buffer on every rank (a broadcast per root).
template <class T>
void allgather_rows(mask_comm* comm, const T* local, int64_t local_count, T* global,
                    const std::vector<int64_t>& counts, cudaStream_t st, CollType ty) {
  (void)local_count;
  int64_t off = 0;
  CollGroup g(comm);
  for (int r = 0; r < comm->world; ++r) {
    if (counts[r] > 0)
      coll_broadcast(comm, r == comm->rank ? (const void*)local : (const void*)(global + off), global + off,
                     (size_t)counts[r], ty, r, st);
    off += counts[r];
  }
  g.end();
}

std::vector<int64_t> allgather_scalar(mask_comm* comm, int64_t v, cudaStream_t st) {
  DevBuf<int64_t> buf(comm->world);
  DevBuf<int64_t> mine(1);
  MASK_CUDA(cudaMemcpyAsync(mine.p, &v, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  coll_allgather(comm, mine.p, buf.p, 1, kI64, st);
  std::vector<int64_t> out(comm->world);
  MASK_CUDA(cudaMemcpyAsync(out.data(), buf.p, sizeof(int64_t) * comm->world, cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaStreamSynchronize(st));
  return out;
}

__global__ void k_add_offset(int64_t* v, int64_t n, int64_t off) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] += off;
}

// The partition-ordered copy of the dense rows (K9's contiguous leaf scans) is an optimisation:
// when the device cannot hold it the index keeps none and queries scan through the member ids.
void gather_partition_best_effort(mask_index* idx, cudaStream_t st) {
  const int64_t N = idx->n_global;
  const int d = idx->dim;
  try {
    idx->Xpart.alloc((size_t)N * d);
  } catch (const Error& e) {
    if (e.code != MASK_ERR_OOM) throw;
    cudaGetLastError();
    idx->Xpart.release();
    return;
  }
  launch_gather_partition(idx->X, d, idx->levels[0].members.p, N, idx->Xpart.p, st);
}

// The child-ordered prototype copies (Pchild) are an optimisation like Xpart: sum_l k_l x d
// floats, skipped per level when the device cannot hold them.  Rebuilt whenever child lists change.
void gather_child_protos(mask_index* idx, cudaStream_t st) {
  idx->Pchild.clear();
  if (idx->format != MASK_DENSE_F32) return;
  const int L = (int)idx->levels.size();
  idx->Pchild.resize(std::max(L - 1, 0));
  for (int l = 0; l + 1 < L; ++l) {
    const int64_t k = idx->levels[l].k;
    if (idx->levels[l + 1].n_items != k || k == 0) continue;
    try {
      idx->Pchild[l].alloc((size_t)k * idx->dim);
    } catch (const Error& e) {
      if (e.code != MASK_ERR_OOM) throw;
      cudaGetLastError();
      idx->Pchild[l].release();
      continue;
    }
    launch_gather_partition(idx->levels[l].P.p, idx->dim, idx->levels[l + 1].members.p, k, idx->Pchild[l].p, st);
  }
}
const float* pchild_ptr(const mask_index* idx, int l) {
  return l < (int)idx->Pchild.size() ? idx->Pchild[l].p : nullptr;
}

void build_impl(const mask_matrix* data, const mask_build_params* p, mask_comm* comm,
                cudaStream_t st, mask_index** out) {
  MASK_REQUIRE(out != nullptr, MASK_ERR_ARG, "out is NULL");
  *out = nullptr;
  check_matrix(data, "data");
  MASK_REQUIRE(p != nullptr, MASK_ERR_ARG, "params is NULL");
  MASK_REQUIRE(p->num_levels >= 1 && p->num_levels <= kMaxLevels, MASK_ERR_ARG,
               "num_levels must be in [1, 16]");
  MASK_REQUIRE(p->max_iters >= 0, MASK_ERR_ARG, "max_iters must be >= 0");
  MASK_REQUIRE(p->tol >= 0.0, MASK_ERR_ARG, "tol must be >= 0");
  MASK_REQUIRE(p->k != nullptr, MASK_ERR_ARG, "k is NULL");
  MASK_REQUIRE(p->empty_policy == MASK_EMPTY_KEEP || p->empty_policy == MASK_EMPTY_FARTHEST, MASK_ERR_ARG,
               "empty_policy must be MASK_EMPTY_KEEP or MASK_EMPTY_FARTHEST");
  MASK_REQUIRE(p->empty_policy == MASK_EMPTY_KEEP || !comm || comm->world == 1, MASK_ERR_UNSUPPORTED,
               "MASK_EMPTY_FARTHEST is single-GPU (the farthest rows would need a cross-rank selection)");
  const int world = comm ? comm->world : 1;
  const int rank = comm ? comm->rank : 0;
  if (!comm) {
    MASK_REQUIRE(data->n_global == data->rows && data->row_offset == 0, MASK_ERR_ARG,
                 "single GPU: n_global must equal rows and row_offset must be 0");
  } else {
    MASK_REQUIRE(data->row_offset >= 0 && data->row_offset + data->rows <= data->n_global, MASK_ERR_ARG,
                 "shard outside [0, n_global)");
  }
  const int64_t N = data->n_global;
  MASK_REQUIRE(N >= 1, MASK_ERR_ARG, "empty dataset");
  int64_t n_prev = N;
  // init indices per level: the caller's, or drawn from `seed` (mask_seeded_init) when
  // init_idx (or init_idx[l]) is NULL -- identical on every rank
  std::vector<std::vector<int64_t>> drawn((size_t)p->num_levels);
  std::vector<const int64_t*> inits((size_t)p->num_levels);
  for (int l = 0; l < p->num_levels; ++l) {
    const int64_t k = p->k[l];
    MASK_REQUIRE(k >= 1 && k <= n_prev, MASK_ERR_ARG,
                 "k[" + std::to_string(l) + "] must be in [1, n_items of the level]");
    if (p->init_idx && p->init_idx[l]) {
      inits[l] = p->init_idx[l];
      std::unordered_set<int64_t> seen;
      seen.reserve((size_t)k * 2);
      for (int64_t j = 0; j < k; ++j) {
        const int64_t v = inits[l][j];
        MASK_REQUIRE(v >= 0 && v < n_prev, MASK_ERR_ARG, "init index out of range");
        MASK_REQUIRE(seen.insert(v).second, MASK_ERR_ARG, "init indices must be distinct");
      }
    } else {
      drawn[l].resize((size_t)k);
      mask_seeded_init(p->seed, l + 1, n_prev, k, drawn[l].data());
      inits[l] = drawn[l].data();
    }
    n_prev = k;
  }
  if (data->format == MASK_CSR_F32 && data->memory == MASK_MEM_HOST) check_host_csr(data);
  int ndev = 0;
  MASK_CUDA(cudaGetDeviceCount(&ndev));
  MASK_REQUIRE(ndev > 0, MASK_ERR_CUDA, "no CUDA device");
  if (comm && world > 1) {
    // every rank must build the same index: a hash of the parameters and init indices, its
    // max and min over the ranks must agree (MASK_ERR_ARG on every rank otherwise)
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
    mix((uint64_t)p->num_levels);
    mix((uint64_t)p->max_iters);
    uint64_t tb;
    std::memcpy(&tb, &p->tol, sizeof(tb));
    mix(tb);
    mix((uint64_t)p->flags);
    mix((uint64_t)data->dim);
    mix((uint64_t)data->format);
    mix((uint64_t)data->n_global);
    for (int l = 0; l < p->num_levels; ++l) {
      mix((uint64_t)p->k[l]);
      for (int64_t j = 0; j < p->k[l]; ++j) mix((uint64_t)inits[l][j]);
    }
    const int64_t hv[2] = {(int64_t)(h >> 1), -(int64_t)(h >> 1)};  // max of both = (max h, -min h)
    DevBuf<int64_t> hd(2);
    MASK_CUDA(cudaMemcpyAsync(hd.p, hv, sizeof(hv), cudaMemcpyHostToDevice, st));
    coll_allreduce(comm, hd.p, 2, kI64, true, st);
    int64_t hr[2];
    MASK_CUDA(cudaMemcpyAsync(hr, hd.p, sizeof(hr), cudaMemcpyDeviceToHost, st));
    MASK_CUDA(cudaStreamSynchronize(st));
    MASK_REQUIRE(hr[0] == -hr[1], MASK_ERR_ARG, "ranks disagree on the build parameters or init indices");
  }

  auto idx = std::make_unique<mask_index>();
  idx->dim = data->dim;
  idx->format = data->format;
  idx->n_global = N;
  const int d = data->dim;

  // ---- bring this rank's shard to the device
  Input in;
  in.format = data->format;
  in.dim = d;
  in.n_local = data->rows;
  in.n_global = N;
  in.row_offset = data->row_offset;
  in.nnz = data->nnz;
  DevBuf<float> loc_X, loc_val;
  DevBuf<int64_t> loc_rp;
  DevBuf<int32_t> loc_col;
  const bool borrow = (p->flags & MASK_BORROW_DATA) && data->memory == MASK_MEM_DEVICE && !comm;
  // world > 1 gathers every rank's rows into the index's own copy at the end of level 1, so the
  // shard is read in place; a single GPU (with or without a one-rank communicator) keeps the
  // data it was given, so it copies unless the caller lends it (MASK_BORROW_DATA)
  const bool in_place = borrow || (comm && world > 1);
  if (data->format == MASK_DENSE_F32) {
    const size_t cnt = (size_t)data->rows * d;
    if (data->memory == MASK_MEM_DEVICE && in_place) {
      in.X = data->values;
    } else {
      loc_X.alloc(std::max<size_t>(cnt, 1));
      MASK_CUDA(cudaMemcpyAsync(loc_X.p, data->values, sizeof(float) * cnt,
                                data->memory == MASK_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
      in.X = loc_X.p;
    }
  } else {
    if (data->memory == MASK_MEM_DEVICE && in_place) {
      in.rp = data->row_ptr;
      in.col = data->col_idx;
      in.val = data->values;
    } else {
      const auto kind = data->memory == MASK_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
      loc_rp.alloc(data->rows + 1);
      loc_col.alloc(std::max<int64_t>(data->nnz, 1));
      loc_val.alloc(std::max<int64_t>(data->nnz, 1));
      MASK_CUDA(cudaMemcpyAsync(loc_rp.p, data->row_ptr, sizeof(int64_t) * (data->rows + 1), kind, st));
      if (data->nnz) {
        MASK_CUDA(cudaMemcpyAsync(loc_col.p, data->col_idx, sizeof(int32_t) * data->nnz, kind, st));
        MASK_CUDA(cudaMemcpyAsync(loc_val.p, data->values, sizeof(float) * data->nnz, kind, st));
      }
      in.rp = loc_rp.p;
      in.col = loc_col.p;
      in.val = loc_val.p;
    }
  }
  if (data->format == MASK_CSR_F32 && data->memory == MASK_MEM_DEVICE) {
    if (comm && world > 1) {  // every rank fails together (no rank left waiting in a collective)
      DevBuf<int> err(1);
      launch_check_csr(in.rp, in.col, data->rows, data->nnz, d, err.p, st);
      coll_allreduce(comm, err.p, 1, kI32, true, st);
      int h = 0;
      MASK_CUDA(cudaMemcpyAsync(&h, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      MASK_CUDA(cudaStreamSynchronize(st));
      MASK_REQUIRE(h == 0, MASK_ERR_ARG, "CSR structure invalid on some rank (row_ptr / column range / order)");
    } else {
      check_csr_device(in.rp, in.col, data->rows, data->nnz, d, st);
    }
  }
  if (p->flags & MASK_VALIDATE_FINITE) {
    DevBuf<int32_t> flag(1);
    MASK_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int32_t), st));
    if (data->format == MASK_DENSE_F32) launch_check_finite(in.X, (int64_t)data->rows * d, flag.p, st);
    else launch_check_finite(in.val, data->nnz, flag.p, st);
    int32_t h = 0;
    MASK_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    MASK_CUDA(cudaStreamSynchronize(st));
    if (comm) {
      // every rank must agree on the outcome
      DevBuf<int32_t> f2(1);
      MASK_CUDA(cudaMemcpyAsync(f2.p, &h, sizeof(int32_t), cudaMemcpyHostToDevice, st));
      coll_allreduce(comm, f2.p, 1, kI32, true, st);
      MASK_CUDA(cudaMemcpyAsync(&h, f2.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      MASK_CUDA(cudaStreamSynchronize(st));
    }
    MASK_REQUIRE(h == 0, MASK_ERR_NONFINITE, "data contains NaN or Inf");
  }

  HostStats hs;
  idx->levels.resize(p->num_levels);
  // ---- level 1: the (sharded) data
  run_level(in, p->k[0], inits[0], p, comm, 1, st, idx->levels[0], hs);

  // ---- end of level 1: every rank gets all labels (and all data rows for leaf scans)
  if (comm && world > 1) {
    const auto counts = allgather_scalar(comm, data->rows, st);
    Level& L1 = idx->levels[0];
    DevBuf<int32_t> glab(N);
    allgather_rows<int32_t>(comm, L1.labels.p, data->rows, glab.p, counts, st, kI32);
    L1.labels = std::move(glab);
    L1.n_items = N;
    if (data->format == MASK_DENSE_F32) {
      idx->own_X.alloc((size_t)N * d);
      std::vector<int64_t> ecounts(world);
      for (int r = 0; r < world; ++r) ecounts[r] = counts[r] * d;
      allgather_rows<float>(comm, in.X, data->rows * d, idx->own_X.p, ecounts, st, kF32);
      idx->X = idx->own_X.p;
    } else {
      const auto nnzs = allgather_scalar(comm, data->nnz, st);
      int64_t total = 0;
      std::vector<int64_t> nnz_off(world + 1, 0);
      for (int r = 0; r < world; ++r) nnz_off[r + 1] = nnz_off[r] + nnzs[r];
      total = nnz_off[world];
      idx->own_col.alloc(std::max<int64_t>(total, 1));
      idx->own_val.alloc(std::max<int64_t>(total, 1));
      idx->own_rp.alloc(N + 1);
      allgather_rows<int32_t>(comm, in.col, data->nnz, idx->own_col.p, nnzs, st, kI32);
      allgather_rows<float>(comm, in.val, data->nnz, idx->own_val.p, nnzs, st, kF32);
      // row_ptr: each rank contributes rows entries rebased by its nnz offset
      DevBuf<int64_t> rp_loc(std::max<int64_t>(data->rows, 1));
      if (data->rows) {
        MASK_CUDA(cudaMemcpyAsync(rp_loc.p, in.rp, sizeof(int64_t) * data->rows, cudaMemcpyDeviceToDevice, st));
        k_add_offset<<<grid_for(data->rows, 256), 256, 0, st>>>(rp_loc.p, data->rows, nnz_off[rank]);
        MASK_LAUNCH_CHECK();
      }
      allgather_rows<int64_t>(comm, rp_loc.p, data->rows, idx->own_rp.p, counts, st, kI64);
      MASK_CUDA(cudaMemcpyAsync(idx->own_rp.p + N, &total, sizeof(int64_t), cudaMemcpyHostToDevice, st));
      idx->rp = idx->own_rp.p;
      idx->col = idx->own_col.p;
      idx->val = idx->own_val.p;
    }
    MASK_CUDA(cudaStreamSynchronize(st));
  } else {
    // single GPU: keep the working copy (or the borrowed pointer)
    if (data->format == MASK_DENSE_F32) {
      if (loc_X.p) idx->own_X = std::move(loc_X);
      idx->X = idx->own_X.p ? idx->own_X.p : in.X;
    } else {
      if (loc_rp.p) {
        idx->own_rp = std::move(loc_rp);
        idx->own_col = std::move(loc_col);
        idx->own_val = std::move(loc_val);
      }
      idx->rp = idx->own_rp.p ? idx->own_rp.p : in.rp;
      idx->col = idx->own_col.p ? idx->own_col.p : in.col;
      idx->val = idx->own_val.p ? idx->own_val.p : in.val;
    }
  }

  // ---- levels 2..L: replicated on every rank (P6); rank 0's result is broadcast so the
  //      replicas stay bitwise identical whatever the atomics' summation order
  for (int l = 1; l < p->num_levels; ++l) {
    Level& prev = idx->levels[l - 1];
    Input up;
    up.format = MASK_DENSE_F32;
    up.dim = d;
    up.n_local = up.n_global = prev.k;
    up.row_offset = 0;
    up.X = prev.P.p;
    run_level(up, p->k[l], inits[l], p, nullptr, l + 1, st, idx->levels[l], hs);
    if (comm && world > 1) {
      Level& L = idx->levels[l];
      CollGroup g(comm);
      coll_broadcast(comm, L.P.p, L.P.p, (size_t)L.k * d, kF32, 0, st);
      coll_broadcast(comm, L.labels.p, L.labels.p, (size_t)L.n_items, kI32, 0, st);
      g.end();
    }
  }
  // ---- child lists (K8) for every level
  for (auto& L : idx->levels) {
    L.offsets.alloc(L.k + 1);
    L.members.alloc(std::max<int64_t>(L.n_items, 1));
    DevBuf<int32_t> cursor(L.k);
    launch_children(L.labels.p, L.n_items, L.k, L.offsets.p, L.members.p, cursor.p, st);
  }
  // ---- dense rows in level-1 partition order for the leaf scans (one gather, n x d floats)
  if (idx->format == MASK_DENSE_F32 && !(p->flags & MASK_NO_PARTITION_COPY))
    gather_partition_best_effort(idx.get(), st);
  gather_child_protos(idx.get(), st);
  if (idx->format == MASK_CSR_F32) {
    // ||c||^2 per level for sparse queries
    int64_t tot = 0;
    std::vector<int64_t> off(p->num_levels);
    for (int l = 0; l < p->num_levels; ++l) {
      off[l] = tot;
      tot += idx->levels[l].k;
    }
    idx->cn2_flat.alloc(tot);
    idx->cn2_off.alloc(p->num_levels);
    for (int l = 0; l < p->num_levels; ++l)
      launch_level_norms(idx->levels[l].P.p, idx->levels[l].k, d, idx->cn2_flat.p + off[l], st);
    MASK_CUDA(cudaMemcpyAsync(idx->cn2_off.p, off.data(), sizeof(int64_t) * off.size(), cudaMemcpyHostToDevice, st));
  }
  MASK_CUDA(cudaStreamSynchronize(st));
  *out = idx.release();
}

// Grouped construction (Algorithm 1; G1-G5): layer sizes by the floor
// recurrence g_i = floor(n_{i-1} / lengthGroup), n_i = g_i * nCentroids, while g_i >= 1.
int grouped_layers(int64_t n, int64_t lg, int64_t nc, std::vector<std::pair<int64_t, int64_t>>* out) {
  int depth = 0;
  int64_t g = n / lg;
  while (g >= 1) {
    if (out) out->push_back({n, g});
    ++depth;
    n = g * nc;
    g = n / lg;
  }
  return depth;
}

void build_grouped_impl(const mask_matrix* data, const mask_grouped_params* p, cudaStream_t st, mask_index** out) {
  MASK_REQUIRE(out != nullptr, MASK_ERR_ARG, "out is NULL");
  *out = nullptr;
  check_matrix(data, "data");
  MASK_REQUIRE(p != nullptr, MASK_ERR_ARG, "params is NULL");
  MASK_REQUIRE(data->format == MASK_DENSE_F32, MASK_ERR_UNSUPPORTED, "grouped build takes dense data");
  MASK_REQUIRE(data->n_global == data->rows && data->row_offset == 0, MASK_ERR_ARG,
               "grouped build is single-GPU: n_global must equal rows");
  MASK_REQUIRE(p->length_group >= 2 && p->n_centroids >= 1 && p->n_centroids < p->length_group, MASK_ERR_ARG,
               "need 1 <= n_centroids < length_group (the layer sizes do not shrink otherwise)");
  MASK_REQUIRE(p->max_iters >= 0, MASK_ERR_ARG, "max_iters must be >= 0");
  const int64_t N = data->rows;
  std::vector<std::pair<int64_t, int64_t>> layers;
  grouped_layers(N, p->length_group, p->n_centroids, &layers);
  MASK_REQUIRE(!layers.empty(), MASK_ERR_ARG, "fewer points than length_group: no centroid layer");
  MASK_REQUIRE((int)layers.size() <= kMaxLevels, MASK_ERR_UNSUPPORTED, "grouped depth exceeds 16 layers");
  for (const auto& lg : layers)
    MASK_REQUIRE(lg.first / lg.second >= p->n_centroids, MASK_ERR_ARG,
                 "a group holds fewer items than n_centroids");
  const int d = data->dim;
  auto idx = std::make_unique<mask_index>();
  idx->dim = d;
  idx->format = MASK_DENSE_F32;
  idx->n_global = N;
  const size_t cnt = (size_t)N * d;
  const bool borrow = (p->flags & MASK_BORROW_DATA) && data->memory == MASK_MEM_DEVICE;
  if (borrow) {
    idx->X = data->values;
  } else {
    idx->own_X.alloc(std::max<size_t>(cnt, 1));
    MASK_CUDA(cudaMemcpyAsync(idx->own_X.p, data->values, sizeof(float) * cnt,
                              data->memory == MASK_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
    idx->X = idx->own_X.p;
  }
  DevBuf<int64_t> perm;
  if (p->perm) {
    std::vector<char> seen(N, 0);
    for (int64_t i = 0; i < N; ++i) {
      const int64_t v = p->perm[i];
      MASK_REQUIRE(v >= 0 && v < N && !seen[v], MASK_ERR_ARG, "perm must be a permutation of [0, rows)");
      seen[v] = 1;
    }
    perm.alloc(N);
    MASK_CUDA(cudaMemcpyAsync(perm.p, p->perm, sizeof(int64_t) * N, cudaMemcpyHostToDevice, st));
  }
  idx->levels.resize(layers.size());
  const float* Y = idx->X;
  for (size_t l = 0; l < layers.size(); ++l) {
    Level& L = idx->levels[l];
    const int64_t n_items = layers[l].first, g = layers[l].second;
    L.n_items = n_items;
    L.k = g * p->n_centroids;
    L.dim = d;
    L.P.alloc((size_t)L.k * d);
    L.labels.alloc(n_items);
    L.assign_kernel = 4;
    launch_group_lloyd(Y, d, l == 0 ? perm.p : nullptr, n_items, g, p->n_centroids, p->max_iters, L.P.p,
                       L.labels.p, st);
    L.offsets.alloc(L.k + 1);
    L.members.alloc(std::max<int64_t>(n_items, 1));
    DevBuf<int32_t> cursor(L.k);
    launch_children(L.labels.p, n_items, L.k, L.offsets.p, L.members.p, cursor.p, st);
    MASK_CUDA(cudaStreamSynchronize(st));  // cursor / perm scratch go out of scope
    Y = L.P.p;
  }
  gather_child_protos(idx.get(), st);
  MASK_CUDA(cudaStreamSynchronize(st));
  *out = idx.release();
}

const Level& level_of(const mask_index* idx, int level) {
  MASK_REQUIRE(idx != nullptr, MASK_ERR_ARG, "index is NULL");
  MASK_REQUIRE(level >= 1 && level <= (int)idx->levels.size(), MASK_ERR_ARG, "level out of range");
  return idx->levels[level - 1];
}

}  // namespace

// ============================================================================== C ABI
extern "C" {

int32_t mask_abi_version(void) { return MASK_ABI_VERSION; }

const char* mask_last_error(void) { return g_err.c_str(); }

int32_t mask_device_ok(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return 0;
  }
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  return major == 10 ? 1 : 0;
}

int32_t mask_comm_unique_id(uint8_t id_out[128]) {
  return guarded([&] {
    MASK_REQUIRE(id_out != nullptr, MASK_ERR_ARG, "id_out is NULL");
    ncclUniqueId id;
    MASK_NCCL(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(id_out, &id, 128);
  });
}

int32_t mask_comm_init(const uint8_t id[128], int32_t world, int32_t rank, mask_comm** out) {
  return guarded([&] {
    MASK_REQUIRE(id != nullptr && out != nullptr, MASK_ERR_ARG, "NULL argument");
    MASK_REQUIRE(world >= 1 && rank >= 0 && rank < world, MASK_ERR_ARG, "bad world/rank");
    *out = nullptr;
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    auto c = std::make_unique<mask_comm>();
    c->world = world;
    c->rank = rank;
    MASK_NCCL(ncclCommInitRank(&c->comm, world, uid, rank));
    *out = c.release();
  });
}

int32_t mask_comm_init_host(int32_t world, int32_t rank, mask_host_collective_fn fn, void* user, mask_comm** out) {
  return guarded([&] {
    MASK_REQUIRE(fn != nullptr && out != nullptr, MASK_ERR_ARG, "NULL argument");
    MASK_REQUIRE(world >= 1 && rank >= 0 && rank < world, MASK_ERR_ARG, "bad world/rank");
    auto c = std::make_unique<mask_comm>();
    c->world = world;
    c->rank = rank;
    c->host = fn;
    c->host_user = user;
    *out = c.release();
  });
}

void mask_comm_free(mask_comm* comm) {
  if (!comm) return;
  if (comm->comm) ncclCommDestroy(comm->comm);
  delete comm;
}

int32_t mask_build(const mask_matrix* data, const mask_build_params* params, mask_comm* comm,
                   void* stream, mask_index** out) {
  NvtxRange range("mask_build");
  return guarded([&] {
    MASK_REQUIRE(!comm || comm->usable(), MASK_ERR_NCCL, "communicator was aborted after an earlier NCCL error");
    build_impl(data, params, comm, as_stream(stream), out);
  });
}

int32_t mask_grouped_depth(int64_t n, int32_t length_group, int32_t n_centroids, int64_t* layer_k, int32_t cap) {
  if (n < 0 || n_centroids < 1 || n_centroids >= length_group) return MASK_ERR_ARG;
  std::vector<std::pair<int64_t, int64_t>> layers;
  const int depth = grouped_layers(n, length_group, n_centroids, &layers);
  for (int i = 0; i < depth && i < cap && layer_k; ++i) layer_k[i] = layers[i].second * n_centroids;
  return depth;
}

int32_t mask_build_grouped(const mask_matrix* data, const mask_grouped_params* params, void* stream,
                           mask_index** out) {
  return guarded([&] { build_grouped_impl(data, params, as_stream(stream), out); });
}

int32_t mask_relocate(const mask_index* idx, const int64_t* got, const int64_t* order_in, const int64_t* keys,
                      int32_t n_centroids, int64_t* order_out, int64_t* reached_out, int64_t* misses_out,
                      void* stream) {
  return guarded([&] {
    MASK_REQUIRE(idx && got && order_in && keys && order_out && misses_out, MASK_ERR_ARG, "NULL argument");
    MASK_REQUIRE(!idx->levels.empty() && n_centroids >= 1 && idx->levels[0].k % n_centroids == 0, MASK_ERR_ARG,
                 "n_centroids must divide the level-1 prototype count");
    cudaStream_t st = as_stream(stream);
    const int64_t n = idx->levels[0].n_items;
    const int64_t groups = idx->levels[0].k / n_centroids;
    DevBuf<unsigned long long> miss(1);
    launch_relocate(got, order_in, keys, idx->levels[0].labels.p, n, groups, n_centroids, order_out, reached_out,
                    miss.p, st);
    unsigned long long h = 0;
    MASK_CUDA(cudaMemcpy(&h, miss.p, sizeof(h), cudaMemcpyDeviceToHost));
    *misses_out = (int64_t)h;
  });
}

namespace {
QIndex make_qindex(const mask_index* idx) {
  QIndex qi{};
  qi.L = (int)idx->levels.size();
  qi.dim = idx->dim;
  qi.X = idx->X;
  qi.xrp = idx->rp;
  qi.xcol = idx->col;
  qi.xval = idx->val;
  for (int l = 0; l < qi.L; ++l) {
    qi.lv[l].P = idx->levels[l].P.p;
    qi.lv[l].offsets = idx->levels[l].offsets.p;
    qi.lv[l].members = idx->levels[l].members.p;
    qi.lv[l].k = idx->levels[l].k;
    qi.lv[l].Pc = pchild_ptr(idx, l);
  }
  return qi;
}
}  // namespace

int32_t mask_range_query(const mask_index* idx, const mask_matrix* queries, const float* radius, int32_t mode,
                         int64_t max_results, int64_t* offsets_out, int64_t* ids_out, float* d2_out,
                         int64_t* total_out, void* stream) {
  return guarded([&] {
    MASK_REQUIRE(idx != nullptr, MASK_ERR_ARG, "index is NULL");
    check_matrix(queries, "queries");
    MASK_REQUIRE(idx->format == MASK_DENSE_F32 && queries->format == MASK_DENSE_F32, MASK_ERR_UNSUPPORTED,
                 "range search takes a dense index and dense queries");
    MASK_REQUIRE(queries->dim == idx->dim, MASK_ERR_ARG, "query dim differs from the index dim");
    MASK_REQUIRE(mode == MASK_RANGE_PAPER || mode == MASK_RANGE_COVER, MASK_ERR_ARG, "unknown range mode");
    MASK_REQUIRE(radius != nullptr && total_out != nullptr, MASK_ERR_ARG, "NULL radius / total_out");
    MASK_REQUIRE(max_results >= 0, MASK_ERR_ARG, "max_results must be >= 0");
    cudaStream_t st = as_stream(stream);
    const int64_t nq = queries->rows;
    const int d = idx->dim;
    const bool host = queries->memory == MASK_MEM_HOST;
    DevBuf<float> qv, rv;
    const float* Q = queries->values;
    const float* R = radius;
    if (host) {
      qv.alloc(std::max<int64_t>(nq * d, 1));
      rv.alloc(std::max<int64_t>(nq, 1));
      if (nq) {
        MASK_CUDA(cudaMemcpyAsync(qv.p, Q, sizeof(float) * nq * d, cudaMemcpyHostToDevice, st));
        MASK_CUDA(cudaMemcpyAsync(rv.p, R, sizeof(float) * nq, cudaMemcpyHostToDevice, st));
      }
      Q = qv.p;
      R = rv.p;
    }
    const QIndex qi = make_qindex(idx);
    std::vector<unsigned*> cov;
    if (mode == MASK_RANGE_COVER) {
      std::lock_guard<std::mutex> lock(idx->cover_mu);
      if (!idx->cover_valid) {
        idx->cover.resize(qi.L);
        std::vector<const int32_t*> labs(qi.L);
        std::vector<int64_t> ns(qi.L);
        std::vector<unsigned*> cp(qi.L);
        for (int l = 0; l < qi.L; ++l) {
          idx->cover[l].alloc(idx->levels[l].k);
          labs[l] = idx->levels[l].labels.p;
          ns[l] = idx->levels[l].n_items;
          cp[l] = idx->cover[l].p;
        }
        launch_cover_radii(idx->X, d, qi, labs.data(), ns.data(), cp.data(), st);
        MASK_CUDA(cudaStreamSynchronize(st));
        idx->cover_valid = true;
      }
      for (auto& c : idx->cover) cov.push_back(c.p);
    }
    DevBuf<int64_t> qcount(std::max<int64_t>(nq, 1)), ids_d;
    DevBuf<float> d2_d;
    int64_t total = 0;
    if (nq) {
      int64_t* ids = ids_out;
      float* d2 = d2_out;
      // the descent runs once; the results are written only when they fit
      total = range_search(qi, cov.empty() ? nullptr : cov.data(), Q, nq, R, mode, nullptr, nullptr, nullptr, 0, st);
      *total_out = total;
      MASK_REQUIRE(total <= max_results, MASK_ERR_ARG,
                   "max_results too small: the range query has " + std::to_string(total) + " results");
      MASK_REQUIRE(offsets_out != nullptr && (total == 0 || (ids_out != nullptr && d2_out != nullptr)), MASK_ERR_ARG,
                   "NULL outputs");
      if (host) {
        ids_d.alloc(std::max<int64_t>(total, 1));
        d2_d.alloc(std::max<int64_t>(total, 1));
        ids = ids_d.p;
        d2 = d2_d.p;
      }
      range_search(qi, cov.empty() ? nullptr : cov.data(), Q, nq, R, mode, ids, d2, qcount.p, total, st);
      std::vector<int64_t> hc(nq);
      MASK_CUDA(cudaMemcpyAsync(hc.data(), qcount.p, sizeof(int64_t) * nq, cudaMemcpyDeviceToHost, st));
      if (host && total) {
        MASK_CUDA(cudaMemcpyAsync(ids_out, ids, sizeof(int64_t) * total, cudaMemcpyDeviceToHost, st));
        MASK_CUDA(cudaMemcpyAsync(d2_out, d2, sizeof(float) * total, cudaMemcpyDeviceToHost, st));
      }
      MASK_CUDA(cudaStreamSynchronize(st));
      std::vector<int64_t> off(nq + 1, 0);
      for (int64_t q = 0; q < nq; ++q) off[q + 1] = off[q] + hc[q];
      if (host) std::copy(off.begin(), off.end(), offsets_out);
      else MASK_CUDA(cudaMemcpy(offsets_out, off.data(), sizeof(int64_t) * (nq + 1), cudaMemcpyHostToDevice));
    } else {
      *total_out = 0;
      if (offsets_out) {
        const int64_t z = 0;
        if (host) offsets_out[0] = 0;
        else MASK_CUDA(cudaMemcpy(offsets_out, &z, sizeof(int64_t), cudaMemcpyHostToDevice));
      }
    }
  });
}

int32_t mask_insert(mask_index* idx, const mask_matrix* points, int64_t* partition_out, void* stream) {
  return guarded([&] {
    MASK_REQUIRE(idx != nullptr, MASK_ERR_ARG, "index is NULL");
    check_matrix(points, "points");
    MASK_REQUIRE(idx->format == MASK_DENSE_F32 && points->format == MASK_DENSE_F32, MASK_ERR_UNSUPPORTED,
                 "insertion takes a dense index and dense points");
    MASK_REQUIRE(points->dim == idx->dim, MASK_ERR_ARG, "point dim differs from the index dim");
    const int64_t m = points->rows;
    if (m == 0) return;
    cudaStream_t st = as_stream(stream);
    const int d = idx->dim;
    const int64_t n = idx->n_global;
    Level& L1 = idx->levels[0];
    // new rows appended to the index's own copy of the data (a borrowed buffer is copied first)
    DevBuf<float> X2((size_t)(n + m) * d);
    MASK_CUDA(cudaMemcpyAsync(X2.p, idx->X, sizeof(float) * n * d, cudaMemcpyDeviceToDevice, st));
    MASK_CUDA(cudaMemcpyAsync(X2.p + n * d, points->values, sizeof(float) * m * d,
                              points->memory == MASK_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                              st));
    // the level-1 prototype each new point's descent reaches
    const QIndex qi = make_qindex(idx);
    DevBuf<int64_t> leaf(m);
    launch_query_dense(qi, X2.p + n * d, m, 1, 1, leaf.p, nullptr, st, true);
    DevBuf<int32_t> lab2(n + m);
    MASK_CUDA(cudaMemcpyAsync(lab2.p, L1.labels.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
    launch_i64_to_i32(leaf.p, m, lab2.p + n, st);
    DevBuf<int64_t> off(L1.k + 1);
    DevBuf<int32_t> mem(n + m), cursor(L1.k);
    launch_children(lab2.p, n + m, L1.k, off.p, mem.p, cursor.p, st);
    if (partition_out) {
      if (points->memory == MASK_MEM_HOST)
        MASK_CUDA(cudaMemcpyAsync(partition_out, leaf.p, sizeof(int64_t) * m, cudaMemcpyDeviceToHost, st));
      else
        MASK_CUDA(cudaMemcpyAsync(partition_out, leaf.p, sizeof(int64_t) * m, cudaMemcpyDeviceToDevice, st));
    }
    MASK_CUDA(cudaStreamSynchronize(st));
    idx->own_X = std::move(X2);
    idx->X = idx->own_X.p;
    idx->n_global = n + m;
    L1.labels = std::move(lab2);
    L1.offsets = std::move(off);
    L1.members = std::move(mem);
    L1.n_items = n + m;
    if (idx->Xpart.p) {  // the partitions changed: re-gather the partition-ordered rows
      idx->Xpart.release();  // (the old copy goes first: peak = data + one copy)
      gather_partition_best_effort(idx, st);
    }
    gather_child_protos(idx, st);
    MASK_CUDA(cudaStreamSynchronize(st));
    std::lock_guard<std::mutex> lock(idx->cover_mu);
    idx->cover_valid = false;
  });
}

namespace {
__global__ void k_relabel_split(const int64_t* __restrict__ rows, const int32_t* __restrict__ loc, int64_t m,
                                int32_t j, int32_t base, int32_t* __restrict__ labels) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = loc[r];
    labels[rows[r]] = g == 0 ? j : base + g - 1;
  }
}

// Partition split + local rebuild (mask.h mask_split, reading S1).
void split_impl(mask_index* idx, const mask_split_params* p, int64_t* n_split_out, cudaStream_t st) {
  MASK_REQUIRE(idx != nullptr && p != nullptr, MASK_ERR_ARG, "NULL argument");
  MASK_REQUIRE(idx->format == MASK_DENSE_F32, MASK_ERR_UNSUPPORTED, "partition split takes a dense index");
  MASK_REQUIRE(p->threshold >= 1 && p->max_iters >= 0, MASK_ERR_ARG, "threshold must be >= 1 and max_iters >= 0");
  Level& L1 = idx->levels[0];
  const int64_t n = L1.n_items, k1 = L1.k;
  const int d = idx->dim;
  std::vector<int32_t> lab(n);
  if (n) MASK_CUDA(cudaMemcpyAsync(lab.data(), L1.labels.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> cnt(k1, 0);
  for (int64_t i = 0; i < n; ++i) ++cnt[lab[i]];
  std::vector<int64_t> todo;
  int64_t extra = 0;
  for (int64_t j = 0; j < k1; ++j)
    if (cnt[j] > p->threshold) {
      todo.push_back(j);
      extra += (cnt[j] + p->threshold - 1) / p->threshold - 1;
    }
  if (n_split_out) *n_split_out = (int64_t)todo.size();
  if (todo.empty()) return;
  MASK_REQUIRE(k1 + extra < (int64_t(1) << 31), MASK_ERR_UNSUPPORTED, "too many prototypes after the split");
  // rows of each split partition in ascending id order
  std::vector<std::vector<int64_t>> rows(todo.size());
  {
    std::vector<int64_t> slot(k1, -1);
    for (size_t t = 0; t < todo.size(); ++t) {
      slot[todo[t]] = (int64_t)t;
      rows[t].reserve((size_t)cnt[todo[t]]);
    }
    for (int64_t i = 0; i < n; ++i)
      if (slot[lab[i]] >= 0) rows[slot[lab[i]]].push_back(i);
  }
  const int64_t k1n = k1 + extra;
  DevBuf<float> P1((size_t)k1n * d);
  MASK_CUDA(cudaMemcpyAsync(P1.p, L1.P.p, sizeof(float) * k1 * d, cudaMemcpyDeviceToDevice, st));
  std::vector<int32_t> parents;  // level-2 labels of the new ids
  std::vector<int32_t> lab2;
  const bool upper = idx->levels.size() >= 2;
  if (upper) {
    lab2.resize(k1);
    MASK_CUDA(cudaMemcpyAsync(lab2.data(), idx->levels[1].labels.p, sizeof(int32_t) * k1, cudaMemcpyDeviceToHost, st));
    MASK_CUDA(cudaStreamSynchronize(st));
  }
  mask_build_params bp{};
  bp.num_levels = 1;
  bp.max_iters = p->max_iters;
  bp.tol = 0.0;
  bp.flags = p->flags & (MASK_FORCE_SIMT | MASK_NO_FUSED | MASK_NO_SORT | MASK_NO_FIXUP);
  HostStats hs;
  int64_t nxt = k1;
  for (size_t t = 0; t < todo.size(); ++t) {
    const int64_t j = todo[t];
    const int64_t nj = (int64_t)rows[t].size();
    const int64_t sgrp = (nj + p->threshold - 1) / p->threshold;
    DevBuf<int64_t> rdev(nj);
    MASK_CUDA(cudaMemcpyAsync(rdev.p, rows[t].data(), sizeof(int64_t) * nj, cudaMemcpyHostToDevice, st));
    DevBuf<float> Y((size_t)nj * d);
    launch_gather_rows(idx->X, d, rdev.p, nj, 0, n, Y.p, st);
    std::vector<int64_t> init((size_t)sgrp);
    MASK_REQUIRE(mask_seeded_init(p->seed + (uint64_t)j, 1, nj, sgrp, init.data()) == MASK_OK, MASK_ERR_ARG,
                 "seeded init failed");
    Input in;
    in.format = MASK_DENSE_F32;
    in.dim = d;
    in.n_local = in.n_global = nj;
    in.X = Y.p;
    Level Lj;
    run_level(in, sgrp, init.data(), &bp, nullptr, 1, st, Lj, hs);
    // group 0 -> prototype j, groups 1.. -> new ids nxt, nxt + 1, ...
    MASK_CUDA(cudaMemcpyAsync(P1.p + j * d, Lj.P.p, sizeof(float) * d, cudaMemcpyDeviceToDevice, st));
    if (sgrp > 1)
      MASK_CUDA(cudaMemcpyAsync(P1.p + nxt * d, Lj.P.p + d, sizeof(float) * (sgrp - 1) * d, cudaMemcpyDeviceToDevice,
                                st));
    k_relabel_split<<<grid_for(nj, 256), 256, 0, st>>>(rdev.p, Lj.labels.p, nj, (int32_t)j, (int32_t)nxt, L1.labels.p);
    MASK_LAUNCH_CHECK();
    if (upper)
      for (int64_t g = 1; g < sgrp; ++g) parents.push_back(lab2[j]);
    nxt += sgrp - 1;
    MASK_CUDA(cudaStreamSynchronize(st));  // Y / rdev / Lj leave scope
  }
  L1.P = std::move(P1);
  L1.k = k1n;
  L1.offsets.alloc(k1n + 1);
  {
    DevBuf<int32_t> cursor(k1n);
    launch_children(L1.labels.p, n, k1n, L1.offsets.p, L1.members.p, cursor.p, st);
  }
  L1.P_trace.release();
  L1.lab_trace.release();
  L1.trace_T = -1;
  if (upper) {
    Level& L2 = idx->levels[1];
    DevBuf<int32_t> l2((size_t)k1n);
    MASK_CUDA(cudaMemcpyAsync(l2.p, L2.labels.p, sizeof(int32_t) * k1, cudaMemcpyDeviceToDevice, st));
    MASK_CUDA(cudaMemcpyAsync(l2.p + k1, parents.data(), sizeof(int32_t) * parents.size(), cudaMemcpyHostToDevice, st));
    L2.labels = std::move(l2);
    L2.n_items = k1n;
    L2.members.alloc((size_t)k1n);
    DevBuf<int32_t> cursor(L2.k);
    launch_children(L2.labels.p, k1n, L2.k, L2.offsets.p, L2.members.p, cursor.p, st);
    L2.P_trace.release();
    L2.lab_trace.release();
    L2.trace_T = -1;
  }
  if (idx->Xpart.p) {
    idx->Xpart.release();
    gather_partition_best_effort(idx, st);
  }
  gather_child_protos(idx, st);
  MASK_CUDA(cudaStreamSynchronize(st));
  std::lock_guard<std::mutex> lock(idx->cover_mu);
  idx->cover_valid = false;
}

int32_t query_impl(const mask_index* idx, const mask_matrix* queries, int32_t k_nn, int32_t beam,
                   int64_t* ids_out, float* d2_out, void* stream, const uint8_t* routed, int64_t rstride,
                   int64_t id_base) {
  return guarded([&] {
    MASK_REQUIRE(idx != nullptr, MASK_ERR_ARG, "index is NULL");
    check_matrix(queries, "queries");
    MASK_REQUIRE(k_nn >= 1 && k_nn <= 32, MASK_ERR_ARG, "k_nn must be in [1, 32]");
    MASK_REQUIRE(beam >= 1 && beam <= 256, MASK_ERR_ARG, "beam must be in [1, 256]");
    MASK_REQUIRE(beam <= 32 || (queries->format == MASK_DENSE_F32 && !routed), MASK_ERR_UNSUPPORTED,
                 "beam > 32 is supported for dense queries (mask_query)");
    MASK_REQUIRE(queries->dim == idx->dim, MASK_ERR_ARG, "query dim differs from the index dim");
    MASK_REQUIRE(queries->format == idx->format, MASK_ERR_UNSUPPORTED,
                 "query format must match the index format");
    MASK_REQUIRE(ids_out != nullptr && d2_out != nullptr, MASK_ERR_ARG, "NULL outputs");
    cudaStream_t st = as_stream(stream);
    const int64_t nq = queries->rows;
    if (nq == 0) return;
    QIndex qi{};
    qi.L = (int)idx->levels.size();
    qi.dim = idx->dim;
    qi.X = idx->X;
    qi.xrp = idx->rp;
    qi.xcol = idx->col;
    qi.xval = idx->val;
    for (int l = 0; l < qi.L; ++l) {
      qi.lv[l].P = idx->levels[l].P.p;
      qi.lv[l].offsets = idx->levels[l].offsets.p;
      qi.lv[l].members = idx->levels[l].members.p;
      qi.lv[l].k = idx->levels[l].k;
      qi.lv[l].Pc = pchild_ptr(idx, l);
    }
    const bool host = queries->memory == MASK_MEM_HOST;
    DevBuf<float> qv;
    DevBuf<int64_t> qrp;
    DevBuf<int32_t> qcol;
    DevBuf<int64_t> ids_d;
    DevBuf<float> d2_d;
    const float* Qv = queries->values;
    const int64_t* Qrp = queries->row_ptr;
    const int32_t* Qcol = queries->col_idx;
    int64_t* ids = ids_out;
    float* d2 = d2_out;
    if (queries->format == MASK_CSR_F32 && host) check_host_csr(queries);
    if (host) {
      if (queries->format == MASK_DENSE_F32) {
        qv.alloc((size_t)nq * queries->dim);
        MASK_CUDA(cudaMemcpyAsync(qv.p, Qv, sizeof(float) * nq * queries->dim, cudaMemcpyHostToDevice, st));
      } else {
        qv.alloc(std::max<int64_t>(queries->nnz, 1));
        qrp.alloc(nq + 1);
        qcol.alloc(std::max<int64_t>(queries->nnz, 1));
        MASK_CUDA(cudaMemcpyAsync(qrp.p, Qrp, sizeof(int64_t) * (nq + 1), cudaMemcpyHostToDevice, st));
        if (queries->nnz) {
          MASK_CUDA(cudaMemcpyAsync(qv.p, Qv, sizeof(float) * queries->nnz, cudaMemcpyHostToDevice, st));
          MASK_CUDA(cudaMemcpyAsync(qcol.p, Qcol, sizeof(int32_t) * queries->nnz, cudaMemcpyHostToDevice, st));
        }
        Qrp = qrp.p;
        Qcol = qcol.p;
      }
      Qv = qv.p;
      ids_d.alloc((size_t)nq * k_nn);
      d2_d.alloc((size_t)nq * k_nn);
      ids = ids_d.p;
      d2 = d2_d.p;
    } else if (queries->format == MASK_CSR_F32) {
      check_csr_device(Qrp, Qcol, nq, queries->nnz, queries->dim, st);
    }
    qi.routed = routed;
    qi.rstride = rstride;
    qi.id_base = id_base;
    qi.Xp = idx->Xpart.p;
    if (idx->format == MASK_DENSE_F32) {
      if (!launch_query_grouped(qi, Qv, nq, k_nn, beam, ids, d2, st))
        launch_query_dense(qi, Qv, nq, k_nn, beam, ids, d2, st);
    }
    else
      launch_query_csr(qi, idx->cn2_flat.p, idx->cn2_off.p, Qrp, Qcol, Qv, nq, k_nn, beam, ids, d2, st);
    if (host) {
      MASK_CUDA(cudaMemcpyAsync(ids_out, ids, sizeof(int64_t) * nq * k_nn, cudaMemcpyDeviceToHost, st));
      MASK_CUDA(cudaMemcpyAsync(d2_out, d2, sizeof(float) * nq * k_nn, cudaMemcpyDeviceToHost, st));
    }
    MASK_CUDA(cudaStreamSynchronize(st));
  });
}
}  // namespace

int32_t mask_split(mask_index* idx, const mask_split_params* params, int64_t* n_split_out, void* stream) {
  NvtxRange range("mask_split");
  return guarded([&] { split_impl(idx, params, n_split_out, as_stream(stream)); });
}

int32_t mask_query(const mask_index* idx, const mask_matrix* queries, int32_t k_nn, int32_t beam,
                   int64_t* ids_out, float* d2_out, void* stream) {
  NvtxRange range("mask_query");
  return query_impl(idx, queries, k_nn, beam, ids_out, d2_out, stream, nullptr, 0, 0);
}

// ---------------------------------------------------------------- §3.4 distributed mode (K14)
int32_t mask_query_routed(const mask_index* idx, const mask_matrix* queries, const uint8_t* routed,
                          int64_t routed_stride, int64_t id_base, int32_t k_nn, int32_t beam, int64_t* ids_out,
                          float* d2_out, void* stream) {
  if (queries && queries->memory != MASK_MEM_DEVICE)
    return guarded([&] { MASK_REQUIRE(false, MASK_ERR_UNSUPPORTED, "mask_query_routed takes device queries"); });
  if (!routed || routed_stride < 1)
    return guarded([&] { MASK_REQUIRE(false, MASK_ERR_ARG, "routed must be non-NULL with stride >= 1"); });
  return query_impl(idx, queries, k_nn, beam, ids_out, d2_out, stream, routed, routed_stride, id_base);
}

int32_t mask_top_prototypes(const mask_index* idx, float* host_out, int64_t* count_out) {
  return guarded([&] {
    MASK_REQUIRE(idx != nullptr && count_out != nullptr, MASK_ERR_ARG, "NULL argument");
    const auto& top = idx->levels.back();
    const int64_t k = top.k, d = idx->dim;
    std::vector<int64_t> off(k + 1);
    std::vector<float> P((size_t)k * d);
    MASK_CUDA(cudaMemcpy(off.data(), top.offsets.p, sizeof(int64_t) * (k + 1), cudaMemcpyDeviceToHost));
    MASK_CUDA(cudaMemcpy(P.data(), top.P.p, sizeof(float) * k * d, cudaMemcpyDeviceToHost));
    int64_t c = 0;
    for (int64_t j = 0; j < k; ++j) {
      if (off[j + 1] == off[j]) continue;  // childless: represents no data (reading C2)
      if (host_out) std::memcpy(host_out + c * d, P.data() + j * d, sizeof(float) * d);
      ++c;
    }
    *count_out = c;
  });
}

int32_t mask_route(const float* registry, const int32_t* node_of, int64_t n_registry, int32_t n_nodes,
                   const mask_matrix* queries, double epsilon, uint8_t* routed_out, void* stream) {
  return guarded([&] {
    check_matrix(queries, "queries");
    MASK_REQUIRE(queries->memory == MASK_MEM_DEVICE, MASK_ERR_UNSUPPORTED, "mask_route takes device queries");
    MASK_REQUIRE(n_nodes >= 1 && n_registry >= 0, MASK_ERR_ARG, "n_nodes must be >= 1, n_registry >= 0");
    MASK_REQUIRE(n_registry == 0 || (registry != nullptr && node_of != nullptr), MASK_ERR_ARG, "NULL registry");
    MASK_REQUIRE(epsilon >= 0.0, MASK_ERR_ARG, "epsilon must be >= 0");
    cudaStream_t st = as_stream(stream);
    const int64_t nq = queries->rows;
    if (nq == 0) return;
    MASK_REQUIRE(routed_out != nullptr, MASK_ERR_ARG, "NULL output");
    const bool all = std::isinf(epsilon);
    const float eps2 = all ? INFINITY : (float)(epsilon * epsilon);
    if (queries->format == MASK_DENSE_F32) {
      launch_route_dense(registry, node_of, n_registry, n_nodes, queries->values, nq, queries->dim, eps2, all,
                         routed_out, st);
    } else {
      check_csr_device(queries->row_ptr, queries->col_idx, nq, queries->nnz, queries->dim, st);
      DevBuf<float> n2;
      n2.alloc(std::max<int64_t>(n_registry, 1));
      launch_route_csr(registry, n2.p, node_of, n_registry, n_nodes, queries->dim, queries->row_ptr,
                       queries->col_idx, queries->values, nq, eps2, all, routed_out, st);
      MASK_CUDA(cudaStreamSynchronize(st));
    }
    MASK_CUDA(cudaStreamSynchronize(st));
  });
}

int32_t mask_merge(const int64_t* ids, const float* d2, int32_t n_nodes, int64_t nq, int32_t k_nn, int64_t* ids_out,
                   float* d2_out, void* stream) {
  return guarded([&] {
    MASK_REQUIRE(k_nn >= 1 && k_nn <= 32 && nq >= 0, MASK_ERR_ARG, "k_nn must be in [1, 32], nq >= 0");
    MASK_REQUIRE(nq == 0 || (ids && d2 && ids_out && d2_out), MASK_ERR_ARG, "NULL argument");
    cudaStream_t st = as_stream(stream);
    launch_merge(ids, d2, n_nodes, nq, k_nn, ids_out, d2_out, st);
    MASK_CUDA(cudaStreamSynchronize(st));
  });
}

int64_t mask_collective_count(void) { return g_nccl_calls.load(); }

void mask_debug_fail_alloc(int64_t nth) { g_fail_alloc.store(nth); }

// Seeded init (D2; mask.h): Floyd's sampling of k distinct indices in [0, n), driven by a
// SplitMix64 stream keyed by (seed, level); the order is the insertion order.
int32_t mask_seeded_init(uint64_t seed, int32_t level, int64_t n, int64_t k, int64_t* out) {
  if (n < 1 || k < 1 || k > n || out == nullptr || level < 1) return MASK_ERR_ARG;
  uint64_t state = seed + (uint64_t)level * 0x9E3779B97F4A7C15ull;
  auto next = [&]() {
    state += 0x9E3779B97F4A7C15ull;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  std::unordered_set<int64_t> chosen;
  chosen.reserve((size_t)k * 2);
  int64_t c = 0;
  for (int64_t j = n - k; j < n; ++j) {
    const int64_t t = (int64_t)(next() % (uint64_t)(j + 1));
    const int64_t v = chosen.count(t) ? j : t;
    chosen.insert(v);
    out[c++] = v;
  }
  return MASK_OK;
}

void mask_free(mask_index* idx) { delete idx; }

int32_t mask_assign(const mask_matrix* data, const float* P, int64_t k, int32_t flags,
                    int32_t* labels_out, float* d2_out, int64_t* n_flagged, void* stream) {
  return guarded([&] {
    check_matrix(data, "data");
    MASK_REQUIRE(data->memory == MASK_MEM_DEVICE, MASK_ERR_UNSUPPORTED, "mask_assign takes device data");
    MASK_REQUIRE(P != nullptr && labels_out != nullptr, MASK_ERR_ARG, "NULL argument");
    MASK_REQUIRE(k >= 1, MASK_ERR_ARG, "k must be >= 1");
    cudaStream_t st = as_stream(stream);
    if (data->format == MASK_CSR_F32) check_csr_device(data->row_ptr, data->col_idx, data->rows, data->nnz, data->dim, st);
    Input in;
    in.format = data->format;
    in.dim = data->dim;
    in.n_local = in.n_global = data->rows;
    in.X = data->values;
    in.rp = data->row_ptr;
    in.col = data->col_idx;
    in.val = data->values;
    in.nnz = data->nnz;
    LloydWS ws;
    DevBuf<float> best_tmp;
    float* best = d2_out;
    if (!best) {
      best_tmp.alloc(std::max<int64_t>(data->rows, 1));
      best = best_tmp.p;
    }
    HostStats hs;
    *hs.flags = 0;
    assign_pass(in, P, k, flags, labels_out, best, ws, st, nullptr, nullptr);
    if (ws.flag_count.p)
      MASK_CUDA(cudaMemcpyAsync(hs.flags, ws.flag_count.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    MASK_CUDA(cudaStreamSynchronize(st));
    if (n_flagged) *n_flagged = *hs.flags;
  });
}

int32_t mask_update(const mask_matrix* data, const int32_t* labels, int64_t k, const float* P_in,
                    float* P_out, int32_t* counts_out, double* max_disp, void* stream) {
  return guarded([&] {
    check_matrix(data, "data");
    MASK_REQUIRE(data->memory == MASK_MEM_DEVICE, MASK_ERR_UNSUPPORTED, "mask_update takes device data");
    MASK_REQUIRE(labels != nullptr && P_in != nullptr && P_out != nullptr, MASK_ERR_ARG, "NULL argument");
    MASK_REQUIRE(k >= 1, MASK_ERR_ARG, "k must be >= 1");
    cudaStream_t st = as_stream(stream);
    const int d = data->dim;
    DevBuf<float> S((size_t)k * d);
    DevBuf<int32_t> counts(k);
    DevBuf<uint32_t> fin(2);
    MASK_CUDA(cudaMemsetAsync(S.p, 0, sizeof(float) * k * d, st));
    MASK_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(int32_t) * k, st));
    MASK_CUDA(cudaMemsetAsync(fin.p, 0, sizeof(uint32_t) * 2, st));
    if (P_out != P_in)
      MASK_CUDA(cudaMemcpyAsync(P_out, P_in, sizeof(float) * k * d, cudaMemcpyDeviceToDevice, st));
    if (data->format == MASK_CSR_F32)
      launch_update_csr(data->row_ptr, data->col_idx, data->values, data->rows, d, labels, S.p, counts.p, st);
    else
      launch_update_dense(data->values, data->rows, d, labels, k, S.p, counts.p, st);
    launch_finalize(P_out, S.p, counts.p, k, d, fin.p, 1, st);
    if (counts_out)
      MASK_CUDA(cudaMemcpyAsync(counts_out, counts.p, sizeof(int32_t) * k, cudaMemcpyDeviceToDevice, st));
    uint32_t h[2] = {0, 0};
    MASK_CUDA(cudaMemcpyAsync(h, fin.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    MASK_CUDA(cudaStreamSynchronize(st));
    if (max_disp) {
      float f;
      std::memcpy(&f, &h[0], sizeof(float));
      *max_disp = std::sqrt((double)f);
    }
  });
}

int64_t mask_kernel_launches(void) { return g_launches.load(); }

int32_t mask_get_timing(const mask_index* idx, int32_t level, double* out, int32_t cap) {
  int32_t written = 0;
  const int32_t rc = guarded([&] {
    const Level& L = level_of(idx, level);
    MASK_REQUIRE(out != nullptr || cap == 0, MASK_ERR_ARG, "NULL output");
    for (int c = 0; c < MASK_T_NCLASS && 2 * c + 1 < cap; ++c) {
      out[2 * c] = L.t_ms[c];
      out[2 * c + 1] = (double)L.t_count[c];
      written = 2 * c + 2;
    }
    if (cap > 2 * MASK_T_NCLASS) {
      out[2 * MASK_T_NCLASS] = (double)L.assign_kernel;
      written = 2 * MASK_T_NCLASS + 1;
    }
  });
  return rc == MASK_OK ? written : rc;
}

int32_t mask_num_levels(const mask_index* idx) { return idx ? (int32_t)idx->levels.size() : 0; }

int32_t mask_level_info(const mask_index* idx, int32_t level, int64_t* n_items, int64_t* k,
                        int32_t* dim, int32_t* passes, int32_t* updates) {
  return guarded([&] {
    const Level& L = level_of(idx, level);
    if (n_items) *n_items = L.n_items;
    if (k) *k = L.k;
    if (dim) *dim = L.dim;
    if (passes) *passes = (int32_t)L.J.size();
    if (updates) *updates = L.updates;
  });
}

int32_t mask_get_prototypes(const mask_index* idx, int32_t level, float* host_out) {
  return guarded([&] {
    const Level& L = level_of(idx, level);
    MASK_REQUIRE(host_out != nullptr, MASK_ERR_ARG, "NULL output");
    MASK_CUDA(cudaMemcpy(host_out, L.P.p, sizeof(float) * L.k * L.dim, cudaMemcpyDeviceToHost));
  });
}

int32_t mask_get_labels(const mask_index* idx, int32_t level, int32_t* host_out) {
  return guarded([&] {
    const Level& L = level_of(idx, level);
    MASK_REQUIRE(host_out != nullptr, MASK_ERR_ARG, "NULL output");
    if (L.n_items)
      MASK_CUDA(cudaMemcpy(host_out, L.labels.p, sizeof(int32_t) * L.n_items, cudaMemcpyDeviceToHost));
  });
}

int32_t mask_get_children(const mask_index* idx, int32_t level, int64_t* host_offsets,
                          int64_t* host_members) {
  return guarded([&] {
    const Level& L = level_of(idx, level);
    MASK_REQUIRE(host_offsets != nullptr && host_members != nullptr, MASK_ERR_ARG, "NULL output");
    MASK_CUDA(cudaMemcpy(host_offsets, L.offsets.p, sizeof(int64_t) * (L.k + 1), cudaMemcpyDeviceToHost));
    std::vector<int32_t> m(L.n_items);
    if (L.n_items)
      MASK_CUDA(cudaMemcpy(m.data(), L.members.p, sizeof(int32_t) * L.n_items, cudaMemcpyDeviceToHost));
    for (int64_t j = 0; j < L.k; ++j) std::sort(m.begin() + host_offsets[j], m.begin() + host_offsets[j + 1]);
    for (int64_t i = 0; i < L.n_items; ++i) host_members[i] = m[i];
  });
}

int32_t mask_get_trace(const mask_index* idx, int32_t level, double* J, int64_t* changed,
                       int64_t* empties, int32_t cap) {
  int32_t written = 0;
  const int32_t rc = guarded([&] {
    const Level& L = level_of(idx, level);
    MASK_REQUIRE(cap >= 0, MASK_ERR_ARG, "cap < 0");
    const int32_t np = (int32_t)std::min<size_t>(L.J.size(), (size_t)cap);
    for (int32_t t = 0; t < np; ++t) {
      if (J) J[t] = L.J[t];
      if (changed) changed[t] = L.changed[t];
      if (empties) empties[t] = t < (int32_t)L.empties.size() ? L.empties[t] : 0;
    }
    written = np;
  });
  return rc == MASK_OK ? written : rc;
}

int32_t mask_get_pass(const mask_index* idx, int32_t level, int32_t pass, float* P_host, int32_t* labels_host) {
  int32_t written = 0;
  const int32_t rc = guarded([&] {
    const Level& L = level_of(idx, level);
    MASK_REQUIRE(L.trace_T >= 0 && L.P_trace.p, MASK_ERR_UNSUPPORTED, "the build did not keep a pass trace (MASK_TRACE_PASSES)");
    MASK_REQUIRE(pass >= 0 && pass <= L.trace_loop_passes, MASK_ERR_ARG, "pass out of range");
    const int slot = pass < L.trace_loop_passes ? pass : L.trace_T;
    if (P_host)
      MASK_CUDA(cudaMemcpy(P_host, L.P_trace.p + (size_t)slot * L.k * L.dim, sizeof(float) * L.k * L.dim,
                           cudaMemcpyDeviceToHost));
    const int64_t n = L.trace_n;
    if (labels_host && n)
      MASK_CUDA(cudaMemcpy(labels_host, L.lab_trace.p + (size_t)slot * n, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    written = (int32_t)n;
  });
  return rc == MASK_OK ? written : rc;
}

int32_t mask_get_displacement(const mask_index* idx, int32_t level, double* dmax, int32_t cap) {
  int32_t written = 0;
  const int32_t rc = guarded([&] {
    const Level& L = level_of(idx, level);
    MASK_REQUIRE(cap >= 0 && dmax != nullptr, MASK_ERR_ARG, "cap < 0 or NULL output");
    const int32_t np = (int32_t)std::min<size_t>(L.dmax.size(), (size_t)cap);
    for (int32_t t = 0; t < np; ++t) dmax[t] = L.dmax[t];
    written = np;
  });
  return rc == MASK_OK ? written : rc;
}

}  // extern "C"
