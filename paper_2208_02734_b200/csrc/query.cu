// query.cu -- K9: batched approximate k-NN by multilevel descent (§3.3,
// Algorithm 2; point/k-NN query prose P:846-884).
//
// One warp per query.  At the top level every prototype with children is a candidate; at
// each lower level the candidates are the children of the b prototypes kept at the level
// above (explicit child lists, D7; childless prototypes skipped); at the data layer the
// candidates are the rows of the reached partition(s).  Every selection is a warp-level
// bitonic top-K (K = beam for the levels, K = k_nn at the leaf) over chunks of 32
// candidates with (d^2, id) ordering (D4): sort the chunk with a 32-lane bitonic network,
// merge it into the running sorted top-32 (min against the reversed chunk, then a bitonic
// merge), skipping chunks whose best candidate cannot enter the current top-K (ballot).
// Distances are FP32 direct sums of squares.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace mask {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int32_t PAD_ID = 0x7fffffff;

__device__ __forceinline__ bool key_lt(float da, int32_t ia, float db, int32_t ib) {
  return da < db || (da == db && ia < ib);
}

// Ascending bitonic sort of one (d, id) key per lane across the warp.
__device__ __forceinline__ void warp_sort32(float& d, int32_t& id, int lane) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const float od = __shfl_xor_sync(FULL, d, stride);
      const int32_t oi = __shfl_xor_sync(FULL, id, stride);
      const bool up = (lane & size) == 0 || size == 32;
      const bool lower = (lane & stride) == 0;
      const bool keep_min = (lower == up);
      const bool other_less = key_lt(od, oi, d, id);
      const bool take = keep_min ? other_less : key_lt(d, id, od, oi);
      if (take) {
        d = od;
        id = oi;
      }
    }
  }
}

// Bitonic merge of a bitonic warp sequence into ascending order.
__device__ __forceinline__ void warp_merge32(float& d, int32_t& id, int lane) {
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) {
    const float od = __shfl_xor_sync(FULL, d, stride);
    const int32_t oi = __shfl_xor_sync(FULL, id, stride);
    const bool lower = (lane & stride) == 0;
    const bool take = lower ? key_lt(od, oi, d, id) : key_lt(d, id, od, oi);
    if (take) {
      d = od;
      id = oi;
    }
  }
}

// Running top-K (K <= 32) held as a sorted warp vector: lane r holds the r-th best.
struct WarpTopK {
  float d;
  int32_t id;
  int K;
  __device__ void reset(int k) {
    K = k;
    d = INFINITY;
    id = PAD_ID;
  }
  // offer one candidate per lane (pass +inf / PAD_ID for none)
  __device__ void offer(float cd, int32_t cid, int lane) {
    const float kd = __shfl_sync(FULL, d, K - 1);
    const int32_t ki = __shfl_sync(FULL, id, K - 1);
    unsigned m = __ballot_sync(FULL, key_lt(cd, cid, kd, ki));
    if (!m) return;
    if (__popc(m) <= 8) {
      // few entrants (the common case once the list has warmed up): insert them one at a time
      // (up to 8: ~20 instructions each against ~250 for the sort + merge below)
      // (shift the entries above each one's rank up by a lane; lane 31 drops out).  Keeps the
      // same invariant as the sort + merge below: lanes < K hold the best K keys offered.
      do {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const float xd = __shfl_sync(FULL, cd, src);
        const int32_t xi = __shfl_sync(FULL, cid, src);
        const float pd = __shfl_up_sync(FULL, d, 1);
        const int32_t pi = __shfl_up_sync(FULL, id, 1);
        if (key_lt(xd, xi, d, id)) {
          const bool shift = lane > 0 && key_lt(xd, xi, pd, pi);
          d = shift ? pd : xd;
          id = shift ? pi : xi;
        }
      } while (m);
      return;
    }
    warp_sort32(cd, cid, lane);
    if (__shfl_sync(FULL, id, 0) == PAD_ID && __shfl_sync(FULL, d, 0) == INFINITY) {  // empty: the sorted chunk
      d = cd;
      id = cid;
      return;
    }
    const float rd = __shfl_sync(FULL, cd, 31 - lane);
    const int32_t ri = __shfl_sync(FULL, cid, 31 - lane);
    if (key_lt(rd, ri, d, id)) {
      d = rd;
      id = ri;
    }
    warp_merge32(d, id, lane);
  }
};

__device__ __forceinline__ float dist_dense(const float* __restrict__ q, const float* __restrict__ x,
                                            int d) {
  float s = 0.f;
  if ((d & 3) == 0 && ((uintptr_t)x & 15) == 0) {
    // the row's 16-byte loads are issued QB at a time before their arithmetic: the descent is
    // bound by the latency of these gathers (one candidate row per lane)
    constexpr int QB = 8;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const float4* q4 = reinterpret_cast<const float4*>(q);
    const int d4 = d >> 2;
    if (d4 <= 4) {  // short rows: the plain loop (its loads are already all in flight)
      for (int i = 0; i < d4; ++i) {
        const float4 a = __ldg(x4 + i);
        const float4 b = q4[i];
        float t = b.x - a.x;
        s = fmaf(t, t, s);
        t = b.y - a.y;
        s = fmaf(t, t, s);
        t = b.z - a.z;
        s = fmaf(t, t, s);
        t = b.w - a.w;
        s = fmaf(t, t, s);
      }
      return s;
    }
    for (int i0 = 0; i0 < d4; i0 += QB) {
      float4 a[QB];
#pragma unroll
      for (int u = 0; u < QB; ++u) a[u] = i0 + u < d4 ? __ldg(x4 + i0 + u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < QB; ++u) {
        if (i0 + u >= d4) break;
        const float4 b = q4[i0 + u];
        float t = b.x - a[u].x;
        s = fmaf(t, t, s);
        t = b.y - a[u].y;
        s = fmaf(t, t, s);
        t = b.z - a[u].z;
        s = fmaf(t, t, s);
        t = b.w - a[u].w;
        s = fmaf(t, t, s);
      }
    }
  } else {
    for (int i = 0; i < d; ++i) {
      const float t = q[i] - __ldg(x + i);
      s = fmaf(t, t, s);
    }
  }
  return s;
}

__device__ __forceinline__ bool has_children(const QLevel& L, int64_t j) {
  return L.offsets[j + 1] > L.offsets[j];
}

constexpr int kWarpsPerBlock = 4;

}  // namespace

// Distances of the warp's 32 candidates (lane L owns candidate id cid, PAD_ID = none), LPC lanes
// per candidate: at step s the lane group g = L / LPC evaluates candidate s * (32 / LPC) + g with
// one 16-byte load per lane per 4 * LPC dimensions, reduces over its LPC lanes, and the owner
// lane picks its value up.  Fewer L1 wavefronts per byte than one row per lane but more
// instructions: used for wide beams (many candidates per query), LPC = 1 otherwise.
template <int LPC>
__device__ __forceinline__ float coop_dist(const float* __restrict__ q, const float* __restrict__ base, int d,
                                           int32_t cid, int lane) {
  if constexpr (LPC == 1) {
    return cid == PAD_ID ? INFINITY : dist_dense(q, base + (int64_t)cid * d, d);
  } else {
    constexpr int G = 32 / LPC;
    const int g = lane / LPC, e = lane % LPC;
    const int d4 = d >> 2;
    float mine = INFINITY;
#pragma unroll
    for (int s = 0; s < LPC; ++s) {
      const int32_t id = __shfl_sync(FULL, cid, s * G + g);
      float acc = 0.f;
      if (id != PAD_ID) {
        const float4* x4 = reinterpret_cast<const float4*>(base + (int64_t)id * d);
        const float4* q4 = reinterpret_cast<const float4*>(q);
        for (int c = e; c < d4; c += LPC) {
          const float4 xv = __ldg(x4 + c);
          const float4 qv = q4[c];
          float t = qv.x - xv.x;
          acc = fmaf(t, t, acc);
          t = qv.y - xv.y;
          acc = fmaf(t, t, acc);
          t = qv.z - xv.z;
          acc = fmaf(t, t, acc);
          t = qv.w - xv.w;
          acc = fmaf(t, t, acc);
        }
      }
#pragma unroll
      for (int o = LPC / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
      const float v = __shfl_sync(FULL, acc, (lane % G) * LPC);
      if (lane / G == s) mine = v;
    }
    return cid == PAD_ID ? INFINITY : mine;
  }
}

// Distances of 32 CONTIGUOUS rows (row-major, d = 4G floats, 16-byte aligned) to q, with
// coalesced loads: lane l loads float4 number l + 32 i (i < G) of the block -- column group
// c = l % G of row i (32/G) + l / G -- so every load instruction reads 512 contiguous bytes (4
// L1 wavefronts, against 32 for one row per lane); the G partial sums of a row, spread over G
// lanes, are then combined by a transposed butterfly (G - 1 shuffles per lane), after which lane
// l holds the distance of row (l % G)(32/G) + l / G.  Rows >= nvalid give +inf.
template <int G>
__device__ __forceinline__ float block_dist32(const float4* __restrict__ base4, int nvalid, float4 qc, int lane,
                                              int& row_out) {
  constexpr int RPI = 32 / G;  // rows per load instruction
  float v[G];
#pragma unroll
  for (int i = 0; i < G; ++i) {
    const int r = i * RPI + lane / G;
    float acc = 0.f;
    if (r < nvalid) {
      const float4 xv = __ldg(base4 + lane + 32 * i);
      float t = qc.x - xv.x;
      acc = fmaf(t, t, acc);
      t = qc.y - xv.y;
      acc = fmaf(t, t, acc);
      t = qc.z - xv.z;
      acc = fmaf(t, t, acc);
      t = qc.w - xv.w;
      acc = fmaf(t, t, acc);
    }
    v[i] = acc;
  }
  // step with lane mask m keeps the lower half of the values on lanes with (l & m) == 0 and the
  // upper half on the others, adding the partner's copy: after the last step lane l holds index
  // i = l % G summed over its G lanes
#pragma unroll
  for (int m = G / 2, n = G; m >= 1; m >>= 1, n >>= 1) {
    const bool upper = (lane & m) != 0;
#pragma unroll
    for (int j = 0; j < n / 2; ++j) {
      const float send = upper ? v[j] : v[j + n / 2];
      const float keep = upper ? v[j + n / 2] : v[j];
      v[j] = keep + __shfl_xor_sync(FULL, send, m);
    }
  }
  const int r = (lane % G) * RPI + lane / G;
  row_out = r;
  return r < nvalid ? v[0] : INFINITY;
}

// Leaf scan of rows [m0, m1) of the partition-ordered copy Xp into the running top-k.
template <int G>
__device__ __forceinline__ void leaf_scan_coalesced(const QIndex& qi, const float* q, int64_t m0, int64_t m1,
                                                    const int32_t* __restrict__ members, WarpTopK& top, int lane) {
  const float4 qc = reinterpret_cast<const float4*>(q)[lane % G];
  for (int64_t m = m0; m < m1; m += 32) {
    const int nvalid = (int)min64(32, m1 - m);
    int r;
    const float cd = block_dist32<G>(reinterpret_cast<const float4*>(qi.Xp + m * (int64_t)(4 * G)), nvalid, qc, lane, r);
    const int32_t cid = r < nvalid ? members[m + r] : PAD_ID;
    top.offer(cd, cid, lane);
  }
}

// block_dist32 for a runtime G (d = 4G, G a power of two <= 32; others: G = 0, not called).
// q: 16-byte aligned.
__device__ __forceinline__ float block_dist_any(int G, const float* __restrict__ base, int nvalid, const float* q,
                                                int lane, int& r) {
  const float4* b4 = reinterpret_cast<const float4*>(base);
  const float4 qc = reinterpret_cast<const float4*>(q)[lane % G];
  switch (G) {
    case 1: return block_dist32<1>(b4, nvalid, qc, lane, r);
    case 2: return block_dist32<2>(b4, nvalid, qc, lane, r);
    case 4: return block_dist32<4>(b4, nvalid, qc, lane, r);
    case 8: return block_dist32<8>(b4, nvalid, qc, lane, r);
    case 16: return block_dist32<16>(b4, nvalid, qc, lane, r);
    default: return block_dist32<32>(b4, nvalid, qc, lane, r);
  }
}
__host__ __device__ __forceinline__ int coalesced_g(int d) {
  const int g = d >> 2;
  return ((d & 3) == 0 && g >= 1 && g <= 32 && (g & (g - 1)) == 0) ? g : 0;
}
// Descent step over 32 consecutive candidates: the top level's prototypes j0.. (contiguous in
// L.P) or the children m.. of a parent (contiguous in L.Pc).  Lane l gets one candidate (its
// distance and id, PAD_ID / +inf for none or a prototype without children).
__device__ __forceinline__ void top_block(const QLevel& L, int G, const float* q, int d, int64_t j0, int lane,
                                          float& cd, int32_t& cid) {
  const int nv = (int)min64(32, L.k - j0);
  int r;
  const float v = block_dist_any(G, L.P + j0 * d, nv, q, lane, r);
  cid = (r < nv && has_children(L, j0 + r)) ? (int32_t)(j0 + r) : PAD_ID;
  cd = cid == PAD_ID ? INFINITY : v;
}
__device__ __forceinline__ void child_block(const QLevel& L, const QLevel& up, int G, const float* q, int d, int64_t m,
                                            int64_t m1, int lane, float& cd, int32_t& cid) {
  const int nv = (int)min64(32, m1 - m);
  int r;
  const float v = block_dist_any(G, L.Pc + m * d, nv, q, lane, r);
  cid = PAD_ID;
  if (r < nv) {
    const int32_t j = up.members[m + r];
    if (has_children(L, j)) cid = j;
  }
  cd = cid == PAD_ID ? INFINITY : v;
}

// Dense queries against a dense index.  Shared memory: one q vector (d floats) per warp.
template <int LPC>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_query_dense(QIndex qi, const float* __restrict__ Q, int64_t nq, int knn, int beam,
                  int64_t* __restrict__ ids_out, float* __restrict__ d2_out, int leaf_only) {
  extern __shared__ __align__(16) float sq[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int d = qi.dim;
  const int dpad = (d + 3) & ~3;
  float* q = sq + w * dpad;
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t qid = (int64_t)blockIdx.x * kWarpsPerBlock + w; qid < nq; qid += nwarps) {
    if (qi.routed && !qi.routed[qid * qi.rstride]) {  // §3.4: not routed to this node
      if (lane < knn) {
        ids_out[qid * knn + lane] = -1;
        if (d2_out) d2_out[qid * knn + lane] = INFINITY;
      }
      continue;
    }
    __syncwarp();
    for (int i = lane; i < d; i += 32) q[i] = Q[qid * d + i];
    __syncwarp();
    WarpTopK top;
    // ---- top level: all prototypes with children
    {
      const QLevel& L = qi.lv[qi.L - 1];
      top.reset(beam);
      const int G = coalesced_g(d);
      for (int64_t j0 = 0; j0 < L.k; j0 += 32) {
        if (G) {
          float cd;
          int32_t cid;
          top_block(L, G, q, d, j0, lane, cd, cid);
          top.offer(cd, cid, lane);
          continue;
        }
        const int64_t j = j0 + lane;
        const int32_t cid = (j < L.k && has_children(L, j)) ? (int32_t)j : PAD_ID;
        top.offer(coop_dist<LPC>(q, L.P, d, cid, lane), cid, lane);
      }
    }
    // ---- levels L-1 .. 1: children of the kept prototypes
    for (int l = qi.L - 2; l >= (qi.sel_out ? qi.sel_stop : 0); --l) {
      const QLevel& up = qi.lv[l + 1];
      const QLevel& L = qi.lv[l];
      const float sel_d = top.d;
      const int32_t sel_id = top.id;
      const int nsel = beam;
      top.reset(beam);
      for (int s = 0; s < nsel; ++s) {
        const int32_t p = __shfl_sync(FULL, sel_id, s);
        const float pd = __shfl_sync(FULL, sel_d, s);
        if (p == PAD_ID || pd == INFINITY && p == PAD_ID) continue;
        const int64_t m0 = up.offsets[p], m1 = up.offsets[p + 1];
        const int G = L.Pc ? coalesced_g(d) : 0;
        for (int64_t m = m0; m < m1; m += 32) {
          if (G) {
            float cd;
            int32_t cid;
            child_block(L, up, G, q, d, m, m1, lane, cd, cid);
            top.offer(cd, cid, lane);
            continue;
          }
          const int64_t mm = m + lane;
          int32_t cid = PAD_ID;
          if (mm < m1) {
            const int32_t j = up.members[mm];
            if (has_children(L, j)) cid = j;
          }
          top.offer(coop_dist<LPC>(q, L.P, d, cid, lane), cid, lane);
        }
      }
    }
    if (leaf_only) {  // insertion: the level-1 prototype the descent reaches
      if (lane == 0) ids_out[qid] = top.id == PAD_ID ? -1 : (int64_t)top.id;
      continue;
    }
    if (qi.sel_out) {  // leaf-grouped queries: hand the level-1 selection over
      if (lane < beam) qi.sel_out[qid * beam + lane] = top.id == PAD_ID ? -1 : top.id;
      continue;
    }
    // ---- data layer: rows of the reached partition(s)
    {
      const QLevel& L1 = qi.lv[0];
      const float sel_d = top.d;
      const int32_t sel_id = top.id;
      (void)sel_d;
      top.reset(knn);
      // partition-ordered rows with d = 4G (G a power of two <= 32): 32 contiguous rows per
      // coalesced block (block_dist32); otherwise one row (or LPC lanes) per candidate
      const int G = (qi.Xp && (d & 3) == 0) ? d >> 2 : 0;
      for (int s = 0; s < beam; ++s) {
        const int32_t p = __shfl_sync(FULL, sel_id, s);
        if (p == PAD_ID) continue;
        const int64_t m0 = L1.offsets[p], m1 = L1.offsets[p + 1];
        switch (G) {
          case 1: leaf_scan_coalesced<1>(qi, q, m0, m1, L1.members, top, lane); continue;
          case 2: leaf_scan_coalesced<2>(qi, q, m0, m1, L1.members, top, lane); continue;
          case 4: leaf_scan_coalesced<4>(qi, q, m0, m1, L1.members, top, lane); continue;
          case 8: leaf_scan_coalesced<8>(qi, q, m0, m1, L1.members, top, lane); continue;
          case 16: leaf_scan_coalesced<16>(qi, q, m0, m1, L1.members, top, lane); continue;
          case 32: leaf_scan_coalesced<32>(qi, q, m0, m1, L1.members, top, lane); continue;
          default: break;
        }
        for (int64_t m = m0; m < m1; m += 32) {
          const int64_t mm = m + lane;
          const int32_t cid = mm < m1 ? (int32_t)L1.members[mm] : PAD_ID;
          // partition-ordered rows: the row address is the position itself (no wait on the id)
          const float cd = qi.Xp ? coop_dist<LPC>(q, qi.Xp, d, mm < m1 ? (int32_t)mm : PAD_ID, lane)
                                 : coop_dist<LPC>(q, qi.X, d, cid, lane);
          top.offer(cd, cid, lane);
        }
      }
    }
    if (lane < knn) {
      const bool pad = top.id == PAD_ID;
      ids_out[qid * knn + lane] = pad ? -1 : qi.id_base + (int64_t)top.id;
      d2_out[qid * knn + lane] = pad ? INFINITY : top.d;
    }
  }
}

// ---------------------------------------------------------------------------------------
// Wide beams (32 < b <= kMaxWideBeam): the per-level selection keeps its sorted top-b list in
// shared memory.  A chunk of 32 candidates is filtered against the current b-th key (ballot),
// sorted with the warp bitonic network, staged in shared memory and merged into the list by
// merge path (every lane finds the split of its output positions by binary search), keeping the
// first b: the same (d^2, id) order and the same result as a sort of all candidates (D4).
constexpr int kMaxWideBeam = 256;
constexpr int kWideWarps = 2;

struct SmemTopK {
  float* d;        // [K] sorted ascending by (d, id); first n valid
  int32_t* id;
  float* td;       // [K] merge output
  int32_t* tid;
  float* cd;       // [32] the staged chunk
  int32_t* cid;
  int K, n;
  __device__ void reset(int k) {
    K = k;
    n = 0;
  }
  __device__ void offer(float v, int32_t j, int lane) {
    const float thd = n == K ? d[K - 1] : INFINITY;
    const int32_t thi = n == K ? id[K - 1] : PAD_ID;
    const bool acc = j != PAD_ID && key_lt(v, j, thd, thi);
    unsigned m32 = __ballot_sync(FULL, acc);
    if (!m32) return;
    const int m = __popc(m32);
    if (m <= 4 && n == K) {
      // few entrants into a full list (the common case once it has warmed up): insert each at
      // its rank (count of smaller list keys), shifting the tail by one through the merge
      // buffer; the last key drops out.  Same list as the sort + merge below.
      do {
        const int src = __ffs(m32) - 1;
        m32 &= m32 - 1;
        const float xd = __shfl_sync(FULL, v, src);
        const int32_t xi = __shfl_sync(FULL, j, src);
        int below = 0;
        for (int o = lane; o < n; o += 32) below += key_lt(d[o], id[o], xd, xi) ? 1 : 0;
        const int pos = __reduce_add_sync(FULL, below);
        if (pos >= K) continue;  // (an earlier insert raised the bar past it)
        for (int o = pos + lane; o < K - 1; o += 32) {
          td[o] = d[o];
          tid[o] = id[o];
        }
        __syncwarp();
        for (int o = pos + 1 + lane; o < K; o += 32) {
          d[o] = td[o - 1];
          id[o] = tid[o - 1];
        }
        if (lane == 0) {
          d[pos] = xd;
          id[pos] = xi;
        }
        __syncwarp();
      } while (m32);
      return;
    }
    float cv = acc ? v : INFINITY;
    int32_t cj = acc ? j : PAD_ID;
    warp_sort32(cv, cj, lane);  // the m accepted keys first, ascending
    cd[lane] = cv;
    cid[lane] = cj;
    __syncwarp();
    const int out = min(K, n + m);
    for (int o = lane; o < out; o += 32) {
      int lo = max(0, o - m), hi = min(o, n);
      while (lo < hi) {  // i = number of list keys among the first o outputs
        const int mid = (lo + hi) >> 1;
        if (key_lt(d[mid], id[mid], cd[o - 1 - mid], cid[o - 1 - mid])) lo = mid + 1;
        else hi = mid;
      }
      const int i = lo, jj = o - lo;
      const bool from_list = jj >= m || (i < n && key_lt(d[i], id[i], cd[jj], cid[jj]));
      td[o] = from_list ? d[i] : cd[jj];
      tid[o] = from_list ? id[i] : cid[jj];
    }
    __syncwarp();
    for (int o = lane; o < out; o += 32) {
      d[o] = td[o];
      id[o] = tid[o];
    }
    n = out;
    __syncwarp();
  }
};

__global__ void __launch_bounds__(kWideWarps * 32)
    k_query_dense_wide(QIndex qi, const float* __restrict__ Q, int64_t nq, int knn, int beam,
                       int64_t* __restrict__ ids_out, float* __restrict__ d2_out) {
  extern __shared__ __align__(16) float wsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int d = qi.dim;
  const int dpad = (d + 3) & ~3;
  // per warp: q (dpad floats), two lists + merge buffer of kMaxWideBeam (d, id), chunk of 32
  const int per_warp = dpad + 6 * kMaxWideBeam + 64;
  float* base = wsm + (size_t)w * per_warp;
  float* q = base;
  SmemTopK cur, nxt;
  cur.d = base + dpad;
  cur.id = reinterpret_cast<int32_t*>(cur.d + kMaxWideBeam);
  nxt.d = reinterpret_cast<float*>(cur.id + kMaxWideBeam);
  nxt.id = reinterpret_cast<int32_t*>(nxt.d + kMaxWideBeam);
  cur.td = nxt.td = reinterpret_cast<float*>(nxt.id + kMaxWideBeam);
  cur.tid = nxt.tid = reinterpret_cast<int32_t*>(cur.td + kMaxWideBeam);
  cur.cd = nxt.cd = reinterpret_cast<float*>(cur.tid + kMaxWideBeam);
  cur.cid = nxt.cid = reinterpret_cast<int32_t*>(cur.cd + 32);
  const int64_t nwarps = (int64_t)gridDim.x * kWideWarps;
  for (int64_t qid = (int64_t)blockIdx.x * kWideWarps + w; qid < nq; qid += nwarps) {
    __syncwarp();
    for (int i = lane; i < d; i += 32) q[i] = Q[qid * d + i];
    __syncwarp();
    {  // top level: every prototype with children
      const QLevel& L = qi.lv[qi.L - 1];
      cur.reset(beam);
      const int G = coalesced_g(d);
      for (int64_t j0 = 0; j0 < L.k; j0 += 32) {
        if (G) {
          float cd;
          int32_t cid;
          top_block(L, G, q, d, j0, lane, cd, cid);
          cur.offer(cd, cid, lane);
          continue;
        }
        const int64_t j = j0 + lane;
        const int32_t cid = (j < L.k && has_children(L, j)) ? (int32_t)j : PAD_ID;
        cur.offer(coop_dist<1>(q, L.P, d, cid, lane), cid, lane);
      }
    }
    for (int l = qi.L - 2; l >= (qi.sel_out ? qi.sel_stop : 0); --l) {  // children of the kept prototypes
      const QLevel& up = qi.lv[l + 1];
      const QLevel& L = qi.lv[l];
      nxt.reset(beam);
      for (int s = 0; s < cur.n; ++s) {
        const int32_t p = cur.id[s];
        const int64_t m0 = up.offsets[p], m1 = up.offsets[p + 1];
        const int G = L.Pc ? coalesced_g(d) : 0;
        for (int64_t m = m0; m < m1; m += 32) {
          if (G) {
            float cd;
            int32_t cid;
            child_block(L, up, G, q, d, m, m1, lane, cd, cid);
            nxt.offer(cd, cid, lane);
            continue;
          }
          const int64_t mm = m + lane;
          int32_t cid = PAD_ID;
          if (mm < m1) {
            const int32_t j = up.members[mm];
            if (has_children(L, j)) cid = j;
          }
          nxt.offer(coop_dist<1>(q, L.P, d, cid, lane), cid, lane);
        }
      }
      // the next level's selection becomes the current one (swap the list storage)
      float* td_ = cur.d;
      int32_t* ti_ = cur.id;
      cur.d = nxt.d;
      cur.id = nxt.id;
      cur.n = nxt.n;
      nxt.d = td_;
      nxt.id = ti_;
      __syncwarp();
    }
    if (qi.sel_out) {  // leaf-grouped queries: hand the level-1 selection over
      for (int s2 = lane; s2 < beam; s2 += 32) qi.sel_out[qid * beam + s2] = s2 < cur.n ? cur.id[s2] : -1;
      continue;
    }
    // data layer: rows of the reached partitions
    const QLevel& L1 = qi.lv[0];
    WarpTopK top;
    top.reset(knn);
    const int G = (qi.Xp && (d & 3) == 0) ? d >> 2 : 0;
    for (int s = 0; s < cur.n; ++s) {
      const int32_t p = cur.id[s];
      const int64_t m0 = L1.offsets[p], m1 = L1.offsets[p + 1];
      switch (G) {
        case 1: leaf_scan_coalesced<1>(qi, q, m0, m1, L1.members, top, lane); continue;
        case 2: leaf_scan_coalesced<2>(qi, q, m0, m1, L1.members, top, lane); continue;
        case 4: leaf_scan_coalesced<4>(qi, q, m0, m1, L1.members, top, lane); continue;
        case 8: leaf_scan_coalesced<8>(qi, q, m0, m1, L1.members, top, lane); continue;
        case 16: leaf_scan_coalesced<16>(qi, q, m0, m1, L1.members, top, lane); continue;
        case 32: leaf_scan_coalesced<32>(qi, q, m0, m1, L1.members, top, lane); continue;
        default: break;
      }
      for (int64_t m = m0; m < m1; m += 32) {
        const int64_t mm = m + lane;
        const int32_t cid = mm < m1 ? (int32_t)L1.members[mm] : PAD_ID;
        const float cd = qi.Xp ? coop_dist<1>(q, qi.Xp, d, mm < m1 ? (int32_t)mm : PAD_ID, lane)
                               : coop_dist<1>(q, qi.X, d, cid, lane);
        top.offer(cd, cid, lane);
      }
    }
    if (lane < knn) {
      const bool pad = top.id == PAD_ID;
      ids_out[qid * knn + lane] = pad ? -1 : qi.id_base + (int64_t)top.id;
      d2_out[qid * knn + lane] = pad ? INFINITY : top.d;
    }
  }
}

// ---------------------------------------------------------------------------------------
// Leaf-grouped scan (large batches).  The per-query kernel reads every reached partition once
// per query: at C3 with beam 128 that is ~5 MB of rows per query, from HBM (the partitions a
// query reaches are scattered over the 2.56 GB copy).  The grouped form sorts the (query,
// leaf) pairs by leaf, so all queries of a leaf are served while its rows are on chip:
//   pairs: e = q * beam + s for every selected leaf, grouped by leaf (counting sort);
//   k_leaf_scan: a warp per work item of kLeafPG consecutive pairs (dynamic queue, items in
//     leaf order so concurrently running items share leaves in L2); per leaf segment of the
//     item: the segment's query vectors and running top-k lists in shared memory, then for
//     each 32-row chunk of the leaf every lane holds one row in registers and the warp streams
//     the segment's queries past it (q broadcast from shared memory);
//   k_merge_partials: warp per query, the beam partial lists -> the final top-k.
constexpr int kLeafPG = 16;
constexpr int kChildPG = 32;  // pairs per work item of the grouped level-1 step
constexpr int kLeafWarps = 4;

// slots: 0 = every slot of a query's selection, 1 = slot 0 only, 2 = slots 1 .. beam-1
__device__ __forceinline__ bool slot_in(int64_t e, int beam, int slots) {
  return slots == 0 || ((e % beam == 0) == (slots == 1));
}
__global__ void k_pair_hist(const int32_t* __restrict__ sel, int64_t m, int32_t* __restrict__ cnt, int beam = 1,
                            int slots = 0) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t l = sel[e];
    if (l >= 0 && slot_in(e, beam, slots)) atomicAdd(cnt + l, 1);
  }
}
// single-block exclusive scan of k counts -> off[0..k] (int64); cnt becomes the scatter cursor
__global__ void __launch_bounds__(1024) k_pair_scan(int32_t* __restrict__ cnt, int64_t k, int64_t* __restrict__ off) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t per = (k + blockDim.x - 1) / blockDim.x;
  const int64_t a = t * per, b = min64(k, a + per);
  int64_t s = 0;
  for (int64_t j = a; j < b; ++j) s += cnt[j];
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {
    const int64_t v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = part[t] - s;
  for (int64_t j = a; j < b; ++j) {
    off[j] = run;
    const int32_t c = cnt[j];
    cnt[j] = (int32_t)run;  // (counts per leaf < 2^31)
    run += c;
  }
  if (t == blockDim.x - 1) off[k] = part[t];
}
__global__ void k_pair_scatter(const int32_t* __restrict__ sel, int64_t m, int32_t* __restrict__ cursor,
                               int64_t* __restrict__ pairs, int beam = 1, int slots = 0) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t l = sel[e];
    if (l >= 0 && slot_in(e, beam, slots)) pairs[atomicAdd(cursor + l, 1)] = e;
  }
}

// Stage the query vectors of pairs[s0 .. s0 + np) (np <= 32) into qs[j * D4M + c] (zero beyond
// d4) with every load of the warp in flight together: lane j holds pair j's row offset, and
// the warp sweeps the np x D4M grid of float4s four loads per lane at a time (a per-pair loop
// would wait one L2 round trip per pair).
template <int D4M>
__device__ __forceinline__ void stage_queries(const float* __restrict__ Q, int d4, int beam,
                                              const int64_t* __restrict__ pairs, int64_t s0, int np, float4* qs,
                                              int lane) {
  const int64_t my = lane < np ? (pairs[s0 + lane] / beam) * (int64_t)d4 : 0;
  const float4* Q4 = reinterpret_cast<const float4*>(Q);
  const int total = np * D4M;
  for (int base = 0; base < total; base += 128) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int f = base + u * 32 + lane;
      const int j = f / D4M, c = f % D4M;
      const int64_t off = __shfl_sync(FULL, my, j & 31);
      v[u] = (f < total && c < d4) ? __ldg(Q4 + off + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int f = base + u * 32 + lane;
      if (f < total) qs[f] = v[u];
    }
  }
}

template <int D4M>  // float4 registers per row: d / 4 <= D4M
__global__ void __launch_bounds__(kLeafWarps * 32)
    k_leaf_scan(QIndex qi, const float* __restrict__ Q, const int32_t* __restrict__ sel,
                const int64_t* __restrict__ pairs, const int64_t* __restrict__ loff, int64_t k1, int beam, int knn,
                int* __restrict__ queue, int32_t* __restrict__ part_id, float* __restrict__ part_d, int use_tau) {
  extern __shared__ __align__(16) float4 lsm4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int d = qi.dim, d4 = d >> 2;
  float4* qs = lsm4 + (size_t)w * (kLeafPG * D4M + kLeafPG * 16);  // [kLeafPG][D4M]
  float* ld = reinterpret_cast<float*>(qs + kLeafPG * D4M);          // [kLeafPG][32]
  int32_t* li = reinterpret_cast<int32_t*>(ld + kLeafPG * 32);       // [kLeafPG][32]
  const QLevel& L1 = qi.lv[0];
  const float4* Xp4 = reinterpret_cast<const float4*>(qi.Xp);
  const int64_t npairs = loff[k1];
  const int64_t nitems = (npairs + kLeafPG - 1) / kLeafPG;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(queue, 1);
    item = __shfl_sync(FULL, item, 0);
    if (item >= nitems) break;
    const int64_t i1 = min64(npairs, (int64_t)(item + 1) * kLeafPG);
    for (int64_t s0 = (int64_t)item * kLeafPG; s0 < i1;) {
      const int32_t p = sel[pairs[s0]];
      const int64_t s1 = min64(i1, loff[p + 1]);
      const int np = (int)(s1 - s0);
      __syncwarp();
      stage_queries<D4M>(Q, d4, beam, pairs, s0, np, qs, lane);
      // use_tau: the query's slot-0 list (its nearest partition, scanned in the first phase)
      // already holds k rows at or below its k-th distance tau, so this pair's list starts as k
      // sentinels (tau, PAD): only rows with d^2 <= tau enter it (exact: the merge takes the
      // best k of all lists, and slot 0 supplies k keys <= (tau, its k-th id))
      float tau_l = INFINITY;
      if (use_tau && lane < np) {
        const int64_t e = pairs[s0 + lane];
        tau_l = part_d[(e - e % beam) * knn + knn - 1];
      }
      for (int j = 0; j < np; ++j) {
        ld[j * 32 + lane] = __shfl_sync(FULL, tau_l, j);
        li[j * 32 + lane] = PAD_ID;
      }
      __syncwarp();
      const int64_t m0 = L1.offsets[p], m1 = L1.offsets[p + 1];
      for (int64_t c = m0; c < m1; c += 32) {
        const int64_t r = c + lane;
        const bool valid = r < m1;
        float4 x[D4M];
#pragma unroll
        for (int f = 0; f < D4M; ++f) x[f] = (valid && f < d4) ? __ldg(Xp4 + r * d4 + f) : make_float4(0.f, 0.f, 0.f, 0.f);
        const int32_t cid = valid ? L1.members[r] : PAD_ID;
        for (int j = 0; j < np; ++j) {
          WarpTopK top;
          top.K = knn;
          top.d = ld[j * 32 + lane];
          top.id = li[j * 32 + lane];
          const float4* qj = qs + j * D4M;
          float a0 = 0.f, a1 = 0.f;
#pragma unroll
          for (int f = 0; f < D4M; ++f) {
            const float4 qv = qj[f];
            float t = qv.x - x[f].x;
            a0 = fmaf(t, t, a0);
            t = qv.y - x[f].y;
            a1 = fmaf(t, t, a1);
            t = qv.z - x[f].z;
            a0 = fmaf(t, t, a0);
            t = qv.w - x[f].w;
            a1 = fmaf(t, t, a1);
          }
          top.offer(valid ? a0 + a1 : INFINITY, cid, lane);
          ld[j * 32 + lane] = top.d;
          li[j * 32 + lane] = top.id;
        }
      }
      __syncwarp();
      for (int j = 0; j < np; ++j) {
        const int64_t e = pairs[s0 + j];
        if (lane < knn) {
          part_d[e * knn + lane] = ld[j * 32 + lane];
          part_id[e * knn + lane] = li[j * 32 + lane];
        }
      }
      s0 = s1;
    }
  }
}

__global__ void k_merge_partials(const int32_t* __restrict__ sel, const int32_t* __restrict__ part_id,
                                 const float* __restrict__ part_d, int64_t nq, int beam, int knn, int64_t id_base,
                                 int64_t* __restrict__ ids_out, float* __restrict__ d2_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t qid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); qid < nq; qid += warps) {
    WarpTopK top;
    top.reset(knn);
    // each partial list holds knn entries (padded); offer them 32 at a time
    const int64_t tot = (int64_t)beam * knn;
    for (int64_t c = 0; c < tot; c += 32) {
      const int64_t e = c + lane;
      float cd = INFINITY;
      int32_t cid = PAD_ID;
      if (e < tot && sel[qid * beam + e / knn] >= 0) {
        cd = part_d[qid * tot + e];
        cid = part_id[qid * tot + e];
      }
      top.offer(cd, cid, lane);
    }
    if (lane < knn) {
      const bool pad = top.id == PAD_ID;
      ids_out[qid * knn + lane] = pad ? -1 : id_base + (int64_t)top.id;
      d2_out[qid * knn + lane] = pad ? INFINITY : top.d;
    }
  }
}

// ---------------------------------------------------------------------------------------
// Grouped descent step into level 1 (wide beams).  The per-query descent stops one level above
// (sel_stop = 1) and hands over each query's selected level-2 prototypes; the (query, parent)
// pairs are grouped by parent, a warp per work item holds 32 of the parent's children (rows of
// the child-ordered copy Pc) in registers and streams the item's queries past them, writing
// every child's distance to the pair's slice of a candidate buffer (offsets = exclusive scan of
// the children counts, so a query's candidates are contiguous); a warp per query then selects
// its top-beam from them (same (d^2, id) order as the per-query kernel).
constexpr int kScanB = 1024;

// counts[e] = children of the pair's parent (0 for a padded slot); block-local exclusive scan
__global__ void __launch_bounds__(kScanB) k_cand_scan1(const int32_t* __restrict__ sel, const int64_t* __restrict__ up_off,
                                                       int64_t m, int64_t* __restrict__ coff, int64_t* __restrict__ bsum) {
  __shared__ int64_t wsum[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t e = (int64_t)blockIdx.x * kScanB + t;
  int64_t c = 0;
  if (e < m) {
    const int32_t p = sel[e];
    c = p >= 0 ? up_off[p + 1] - up_off[p] : 0;
  }
  int64_t x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t v = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(FULL, v, o);
      if (lane >= o) v += y;
    }
    wsum[lane] = v;
  }
  __syncthreads();
  const int64_t excl = x - c + (w ? wsum[w - 1] : 0);
  if (e < m) coff[e] = excl;
  if (t == kScanB - 1) bsum[blockIdx.x] = wsum[31];
}
// single block: exclusive scan of the block sums in place, total at bsum[nb]
__global__ void __launch_bounds__(1024) k_cand_scan2(int64_t* __restrict__ bsum, int64_t nb) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t per = (nb + blockDim.x - 1) / blockDim.x;
  const int64_t a = t * per, b = min64(nb, a + per);
  int64_t s = 0;
  for (int64_t j = a; j < b; ++j) s += bsum[j];
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {
    const int64_t v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = part[t] - s;
  for (int64_t j = a; j < b; ++j) {
    const int64_t c = bsum[j];
    bsum[j] = run;
    run += c;
  }
  if (t == blockDim.x - 1) bsum[nb] = part[t];
}
__global__ void k_cand_scan3(int64_t* __restrict__ coff, int64_t m, const int64_t* __restrict__ bsum) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= m; e += (int64_t)gridDim.x * blockDim.x)
    coff[e] = e < m ? coff[e] + bsum[e / kScanB] : bsum[(m + kScanB - 1) / kScanB];
}

template <int D4M>
__global__ void __launch_bounds__(kLeafWarps * 32)
    k_child_dist(QIndex qi, int lvl, const float* __restrict__ Q, const int32_t* __restrict__ sel,
                 const int64_t* __restrict__ pairs, const int64_t* __restrict__ poff, int64_t kp, int beam,
                 const int64_t* __restrict__ coff, int64_t base, int* __restrict__ queue,
                 float* __restrict__ cand_d, int32_t* __restrict__ cand_id) {
  extern __shared__ __align__(16) float4 csm4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int d = qi.dim, d4 = d >> 2;
  float4* qs = csm4 + (size_t)w * (kChildPG * D4M + kChildPG / 2);  // [kChildPG][D4M] queries
  int64_t* co = reinterpret_cast<int64_t*>(qs + kChildPG * D4M);      // [kChildPG] candidate offsets
  const QLevel& L = qi.lv[lvl];
  const QLevel& up = qi.lv[lvl + 1];
  const float4* Pc4 = reinterpret_cast<const float4*>(L.Pc);
  const int64_t npairs = poff[kp];
  const int64_t nitems = (npairs + kChildPG - 1) / kChildPG;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(queue, 1);
    item = __shfl_sync(FULL, item, 0);
    if (item >= nitems) break;
    const int64_t i1 = min64(npairs, (int64_t)(item + 1) * kChildPG);
    for (int64_t s0 = (int64_t)item * kChildPG; s0 < i1;) {
      const int32_t p = sel[pairs[s0]];
      const int64_t s1 = min64(i1, poff[p + 1]);
      const int np = (int)(s1 - s0);
      __syncwarp();
      stage_queries<D4M>(Q, d4, beam, pairs, s0, np, qs, lane);
      for (int j = lane; j < np; j += 32) co[j] = coff[pairs[s0 + j]] - base;
      __syncwarp();
      const int64_t m0 = up.offsets[p], m1 = up.offsets[p + 1];
      for (int64_t c = m0; c < m1; c += 32) {
        const int64_t r = c + lane;
        int32_t cid = PAD_ID;
        if (r < m1) {
          const int32_t j = up.members[r];
          if (has_children(L, j)) cid = j;
        }
        float4 x[D4M];
#pragma unroll
        for (int f = 0; f < D4M; ++f)
          x[f] = (r < m1 && f < d4) ? __ldg(Pc4 + r * d4 + f) : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j = 0; j < np; ++j) {
          const float4* qj = qs + j * D4M;
          float a0 = 0.f, a1 = 0.f;
#pragma unroll
          for (int f = 0; f < D4M; ++f) {
            const float4 qv = qj[f];
            float t = qv.x - x[f].x;
            a0 = fmaf(t, t, a0);
            t = qv.y - x[f].y;
            a1 = fmaf(t, t, a1);
            t = qv.z - x[f].z;
            a0 = fmaf(t, t, a0);
            t = qv.w - x[f].w;
            a1 = fmaf(t, t, a1);
          }
          if (r < m1) {
            const int64_t o = co[j] + (r - m0);
            cand_d[o] = cid == PAD_ID ? INFINITY : a0 + a1;
            cand_id[o] = cid;
          }
        }
      }
      s0 = s1;
    }
  }
}

// warp per query: top-beam of its candidates [coff[q beam], coff[(q + 1) beam]) -> sel_out
__global__ void __launch_bounds__(kWideWarps * 32)
    k_select_cands(const int64_t* __restrict__ coff, int64_t cbase, const float* __restrict__ cand_d,
                   const int32_t* __restrict__ cand_id, int64_t nq, int beam, int32_t* __restrict__ sel_out) {
  extern __shared__ __align__(16) float ssm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * kWideWarps;
  float* base = ssm + (size_t)w * (4 * kMaxWideBeam + 64);
  SmemTopK cur;
  cur.d = base;
  cur.id = reinterpret_cast<int32_t*>(cur.d + kMaxWideBeam);
  cur.td = reinterpret_cast<float*>(cur.id + kMaxWideBeam);
  cur.tid = reinterpret_cast<int32_t*>(cur.td + kMaxWideBeam);
  cur.cd = reinterpret_cast<float*>(cur.tid + kMaxWideBeam);
  cur.cid = reinterpret_cast<int32_t*>(cur.cd + 32);
  for (int64_t q = (int64_t)blockIdx.x * kWideWarps + w; q < nq; q += nwarps) {
    const int64_t a = coff[q * beam] - cbase, b = coff[(q + 1) * beam] - cbase;
    // the loads of the next kPF chunks are in flight while a chunk is offered (the selection is
    // otherwise bound by one load latency per 32 candidates)
    constexpr int kPF = 4;
    float pv[kPF];
    int32_t pj[kPF];
#pragma unroll
    for (int i = 0; i < kPF; ++i) {
      const int64_t o = a + 32 * i + lane;
      pv[i] = o < b ? cand_d[o] : INFINITY;
      pj[i] = o < b ? cand_id[o] : PAD_ID;
    }
    auto sweep = [&](auto&& offer) {
      for (int64_t c = a; c < b; c += 32 * kPF) {
#pragma unroll
        for (int i = 0; i < kPF; ++i) {
          const float v = pv[i];
          const int32_t j = pj[i];
          const int64_t o = c + 32 * (i + kPF) + lane;
          pv[i] = o < b ? cand_d[o] : INFINITY;
          pj[i] = o < b ? cand_id[o] : PAD_ID;
          if (c + 32 * i < b) offer(v, j);  // (uniform across the warp)
        }
      }
    };
    if (beam <= 32) {
      WarpTopK top;
      top.reset(beam);
      sweep([&](float v, int32_t j) { top.offer(v, j, lane); });
      if (lane < beam) sel_out[q * beam + lane] = top.id == PAD_ID ? -1 : top.id;
    } else {
      __syncwarp();
      cur.reset(beam);
      sweep([&](float v, int32_t j) { cur.offer(v, j, lane); });
      for (int s2 = lane; s2 < beam; s2 += 32) sel_out[q * beam + s2] = s2 < cur.n ? cur.id[s2] : -1;
    }
  }
}

// The grouped step into level 1: fills sel (nq x beam level-1 prototype ids, -1 padded).
// Returns false (nothing launched) when the index has no level above 1 or no child-ordered copy.
__global__ void k_gather_coff(const int64_t* __restrict__ coff, int64_t nq, int beam, int64_t qb, int64_t nbnd,
                              int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nbnd; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = coff[min64(i * qb, nq) * beam];
}

// Candidates held at once by the grouped step (8 B each): queries are taken in chunks whose
// candidates fit (parents are skewed: C5 after Lloyd averages ~700 children per selected parent
// against 64 per parent overall, 23e9 candidates for 1e6 queries at beam 32).
constexpr int64_t kCandBudget = int64_t(1) << 29;  // 4 GiB of (d^2, id)
constexpr int64_t kCandQB = 1024;                  // chunk boundary granularity (queries)

// The grouped step into level 1: fills sel (nq x beam level-1 prototype ids, -1 padded).
// Returns false when the index has no level above 1 or no child-ordered copy, or the candidate
// buffer cannot be had (the caller then runs the per-query descent).
// One grouped descent step: from each query's selection sel2 at level lvl+1 (index into lv) to
// its top-b among their children at level lvl, written to sel.
static bool grouped_level_step(const QIndex& qi, const float* Q, int64_t nq, int beam, int lvl,
                               const int32_t* sel2_in, int32_t* sel, cudaStream_t st) {
  const int d = qi.dim, d4 = d >> 2;
  const int d4m = d4 <= 4 ? 4 : d4 <= 8 ? 8 : d4 <= 16 ? 16 : 32;
  const int64_t m = nq * (int64_t)beam;
  const int64_t k2 = qi.lv[lvl + 1].k;
  DevBuf<int32_t> cnt(k2), queue(1);
  DevBuf<int64_t> poff(k2 + 1), pairs(m), coff(m + 1);
  const int64_t nb = (m + kScanB - 1) / kScanB;
  DevBuf<int64_t> bsum(nb + 1);
  // candidate offsets (exclusive scan of the selected parents' children counts, query-major)
  k_cand_scan1<<<(unsigned)nb, kScanB, 0, st>>>(sel2_in, qi.lv[lvl + 1].offsets, m, coff.p, bsum.p);
  MASK_LAUNCH_CHECK();
  k_cand_scan2<<<1, 1024, 0, st>>>(bsum.p, nb);
  MASK_LAUNCH_CHECK();
  k_cand_scan3<<<grid_for(m + 1, 256), 256, 0, st>>>(coff.p, m, bsum.p);
  MASK_LAUNCH_CHECK();
  // chunk boundaries every kCandQB queries
  const int64_t nbnd = (nq + kCandQB - 1) / kCandQB + 1;
  DevBuf<int64_t> bnd_d(nbnd);
  k_gather_coff<<<grid_for(nbnd, 256), 256, 0, st>>>(coff.p, nq, beam, kCandQB, nbnd, bnd_d.p);
  MASK_LAUNCH_CHECK();
  std::vector<int64_t> bnd(nbnd);
  MASK_CUDA(cudaMemcpyAsync(bnd.data(), bnd_d.p, sizeof(int64_t) * nbnd, cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaStreamSynchronize(st));
  std::vector<std::pair<int64_t, int64_t>> chunks;  // [boundary index a, b)
  const char* benv = getenv("MASK_QUERY_CAND_BUDGET");  // (tests: force many chunks)
  const int64_t budget = benv ? std::max<int64_t>(1, atoll(benv)) : kCandBudget;
  int64_t most = 1;
  for (int64_t i = 0; i + 1 < nbnd;) {
    int64_t j = i + 1;
    while (j + 1 < nbnd && bnd[j + 1] - bnd[i] <= budget) ++j;
    chunks.emplace_back(i, j);
    most = std::max<int64_t>(most, bnd[j] - bnd[i]);
    i = j;
  }
  // the candidate buffer is best-effort: on OOM the per-query descent runs
  DevBuf<float> cd;
  DevBuf<int32_t> cid;
  try {
    cd.alloc(most);
    cid.alloc(most);
  } catch (const Error& e) {
    if (e.code != MASK_ERR_OOM) throw;
    cudaGetLastError();
    if (getenv("MASK_DEBUG_QUERY")) fprintf(stderr, "grouped level step: %lld candidates: %s\n", (long long)most, e.what());
    return false;
  }
  const size_t smem = (size_t)kLeafWarps * (kChildPG * d4m + kChildPG / 2) * sizeof(float4);
  const unsigned g = (unsigned)num_sms() * 8;
  const size_t ssmem = (size_t)kWideWarps * (4 * kMaxWideBeam + 64) * sizeof(float);
  for (const auto& c : chunks) {
    const int64_t qa = c.first * kCandQB, qb = std::min<int64_t>(c.second * kCandQB, nq);
    const int64_t nqc = qb - qa, mc = nqc * beam, base = bnd[c.first];
    const int32_t* sel2c = sel2_in + qa * beam;
    const int64_t* coffc = coff.p + qa * beam;
    const float* Qc = Q + qa * d;
    // the chunk's (query, parent) pairs grouped by parent
    MASK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * k2, st));
    k_pair_hist<<<grid_for(mc, 256), 256, 0, st>>>(sel2c, mc, cnt.p);
    MASK_LAUNCH_CHECK();
    k_pair_scan<<<1, 1024, 0, st>>>(cnt.p, k2, poff.p);
    MASK_LAUNCH_CHECK();
    k_pair_scatter<<<grid_for(mc, 256), 256, 0, st>>>(sel2c, mc, cnt.p, pairs.p);
    MASK_LAUNCH_CHECK();
    MASK_CUDA(cudaMemsetAsync(queue.p, 0, sizeof(int), st));
    switch (d4m) {
#define MASK_CD(D)                                                                                              \
  case D:                                                                                                       \
    MASK_CUDA(cudaFuncSetAttribute(k_child_dist<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));   \
    k_child_dist<D><<<g, kLeafWarps * 32, smem, st>>>(qi, lvl, Qc, sel2c, pairs.p, poff.p, k2, beam, coffc, base, \
                                                      queue.p, cd.p, cid.p);                                    \
    break;
      MASK_CD(4)
      MASK_CD(8)
      MASK_CD(16)
      MASK_CD(32)
#undef MASK_CD
    }
    MASK_LAUNCH_CHECK();
    const unsigned sg = (unsigned)std::min<int64_t>((nqc + kWideWarps - 1) / kWideWarps, (int64_t)num_sms() * 32);
    k_select_cands<<<sg, kWideWarps * 32, ssmem, st>>>(coffc, base, cd.p, cid.p, nqc, beam, sel + qa * beam);
    MASK_LAUNCH_CHECK();
  }
  MASK_CUDA(cudaStreamSynchronize(st));  // (the scratch above is released at return)
  return true;
}

// The grouped descent into level 1: the per-query kernel selects at level `start` (index into
// lv; 1 = level 2), then grouped steps take every lower level down to level 1's selection in
// sel.  False when an index level lacks its child-ordered copy or a step's candidate buffer
// cannot be had (the caller then runs the per-query descent).
static bool grouped_level1_selection(const QIndex& qi, const float* Q, int64_t nq, int beam, int32_t* sel,
                                     cudaStream_t st) {
  if (qi.L < 2) return false;
  // grouped steps from the top level down for beams >= 32, from level 2 otherwise
  // (MASK_GROUPED_FROM_TOP=0/1 overrides; C3 beam 128 53.4 -> 51.5 ms, beam 8 6.11 -> 6.19 ms)
  const char* tenv = getenv("MASK_GROUPED_FROM_TOP");
  const bool from_top = tenv ? atoi(tenv) != 0 : beam >= 32;
  const int start = from_top ? qi.L - 1 : 1;
  for (int l = 0; l < start; ++l)
    if (!qi.lv[l].Pc) return false;
  const int64_t m = nq * (int64_t)beam;
  DevBuf<int32_t> cur(m), nxt(start > 1 ? m : 0);
  QIndex q2 = qi;
  q2.sel_out = cur.p;
  q2.sel_stop = start;
  launch_query_dense(q2, Q, nq, 1, beam, nullptr, nullptr, st, false);  // per-query descent to `start`
  for (int lvl = start - 1; lvl >= 0; --lvl) {
    int32_t* out = lvl == 0 ? sel : nxt.p;
    if (!grouped_level_step(qi, Q, nq, beam, lvl, cur.p, out, st)) return false;
    if (lvl > 0) std::swap(cur, nxt);
  }
  return true;
}

bool launch_query_grouped(const QIndex& qi, const float* Q, int64_t nq, int knn, int beam, int64_t* ids, float* d2,
                          cudaStream_t st) {
  // MASK_QUERY_GROUPED=0 / 1: never / always (A/B and tests; read per call)
  const char* env = getenv("MASK_QUERY_GROUPED");
  const int mode = env ? atoi(env) : -1;
  const int64_t m = nq * (int64_t)beam;
  const int d = qi.dim;
  if (mode == 0 || !qi.Xp || qi.routed || qi.L < 1 || (d & 3) || d > 128) return false;
  // the per-query kernel keeps: batches under 32,768 queries (C2's 1e4 at beam 16: 0.60 ms
  // per-query against 0.68 ms grouped -- the grouped pipeline's dozen launches dominate a
  // sub-millisecond batch), fewer than 65,536 (query, partition) pairs, and batches averaging
  // under two queries per partition (C3 at beam 1: 1.5, 1.50 vs 1.54 ms; C5 at beam 1: 3.8,
  // 71 vs 44 ms)
  if (m == 0 || (mode != 1 && (m < 65536 || m < 2 * qi.lv[0].k || nq < 32768))) return false;
  const size_t part_bytes = (size_t)m * knn * 8;
  if (part_bytes > ((size_t)8 << 30)) return false;
  const int d4 = d >> 2;
  const int d4m = d4 <= 4 ? 4 : d4 <= 8 ? 8 : d4 <= 16 ? 16 : 32;
  const size_t smem = (size_t)kLeafWarps * (kLeafPG * d4m + kLeafPG * 16) * sizeof(float4);
  const int64_t k1 = qi.lv[0].k;
  DevBuf<int32_t> sel(m), cnt(k1), pid((size_t)m * knn), queue(1);
  DevBuf<int64_t> off(k1 + 1), pairs(m);
  DevBuf<float> pd((size_t)m * knn);
  // MASK_GROUPED_LEVEL=0/1 overrides the grouped step into level 1 (default: beams >= 2)
  const char* glenv = getenv("MASK_GROUPED_LEVEL");
  const bool glevel = glenv ? atoi(glenv) != 0 : beam >= 2;
  if (!(glevel && grouped_level1_selection(qi, Q, nq, beam, sel.p, st))) {
    QIndex q2 = qi;
    q2.sel_out = sel.p;
    launch_query_dense(q2, Q, nq, knn, beam, ids, d2, st, false);  // descent only
  }
  // two phases for beams >= 8 (MASK_LEAF_TAU=0/1 overrides; C3 beam 128 69 -> 58 ms, beam 2
  // 2.31 -> 2.61 ms): each query's nearest partition (slot 0) first, then the other slots with
  // that list's k-th distance as the entry bar
  const char* tauenv = getenv("MASK_LEAF_TAU");
  const bool two_phase = beam >= 2 && (tauenv ? atoi(tauenv) != 0 : beam >= 8);
  const unsigned lgrid = (unsigned)num_sms() * 8;
  for (int phase = two_phase ? 1 : 0; phase <= (two_phase ? 2 : 0); ++phase) {
    MASK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * k1, st));
    k_pair_hist<<<grid_for(m, 256), 256, 0, st>>>(sel.p, m, cnt.p, beam, phase);
    MASK_LAUNCH_CHECK();
    k_pair_scan<<<1, 1024, 0, st>>>(cnt.p, k1, off.p);
    MASK_LAUNCH_CHECK();
    k_pair_scatter<<<grid_for(m, 256), 256, 0, st>>>(sel.p, m, cnt.p, pairs.p, beam, phase);
    MASK_LAUNCH_CHECK();
    MASK_CUDA(cudaMemsetAsync(queue.p, 0, sizeof(int), st));
    const int use_tau = phase == 2 ? 1 : 0;
    switch (d4m) {
#define MASK_LEAF(D)                                                                                        \
  case D:                                                                                                   \
    MASK_CUDA(cudaFuncSetAttribute(k_leaf_scan<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k_leaf_scan<D><<<lgrid, kLeafWarps * 32, smem, st>>>(qi, Q, sel.p, pairs.p, off.p, k1, beam, knn, queue.p, \
                                                         pid.p, pd.p, use_tau);                             \
    break;
      MASK_LEAF(4)
      MASK_LEAF(8)
      MASK_LEAF(16)
      MASK_LEAF(32)
#undef MASK_LEAF
    }
    MASK_LAUNCH_CHECK();
  }
  k_merge_partials<<<grid_for(nq * 32, 256), 256, 0, st>>>(sel.p, pid.p, pd.p, nq, beam, knn, qi.id_base, ids, d2);
  MASK_LAUNCH_CHECK();
  return true;
}

__global__ void k_gather_partition(const float* __restrict__ X, int d, const int32_t* __restrict__ members, int64_t n,
                                   float* __restrict__ Xp) {
  const int64_t total = n * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = e / d;
    Xp[e] = __ldg(X + (int64_t)members[pos] * d + (e - pos * d));
  }
}

void launch_gather_partition(const float* X, int d, const int32_t* members, int64_t n, float* Xp, cudaStream_t st) {
  if (n <= 0) return;
  k_gather_partition<<<grid_for(n * d, 256, (int64_t)num_sms() * 32), 256, 0, st>>>(X, d, members, n, Xp);
  MASK_LAUNCH_CHECK();
}

void launch_query_dense(const QIndex& qi, const float* Q, int64_t nq, int knn, int beam,
                        int64_t* ids, float* d2, cudaStream_t st, bool leaf_only) {
  if (nq <= 0) return;
  const int dpad = (qi.dim + 3) & ~3;
  const size_t smem = (size_t)kWarpsPerBlock * dpad * sizeof(float);
  MASK_REQUIRE(smem <= 200 * 1024, MASK_ERR_UNSUPPORTED, "query: dim too large for dense queries");
  // wide beams (>= 8 prototypes kept per level) visit many candidates per query: 8 lanes per
  // candidate row there (C3: beam 16 57 -> 47 ms, beam 32 110 -> 77 ms), one lane per row otherwise
  const bool coop = (qi.dim & 3) == 0 && qi.dim >= 32 && beam >= 8 && ((uintptr_t)qi.X & 15) == 0;
  const int64_t blocks = (nq + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const unsigned grid = (unsigned)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  const int lo = leaf_only ? 1 : 0;
  if (beam > 32) {  // wide beams: shared-memory selection lists
    MASK_REQUIRE(!leaf_only && !qi.routed && beam <= kMaxWideBeam, MASK_ERR_UNSUPPORTED,
                 "query: beam > 32 is supported for plain dense queries up to 256");
    const size_t wsmem = (size_t)kWideWarps * (dpad + 6 * kMaxWideBeam + 64) * sizeof(float);
    MASK_REQUIRE(wsmem <= 200 * 1024, MASK_ERR_UNSUPPORTED, "query: dim too large for wide beams");
    if (wsmem > 48 * 1024)
      MASK_CUDA(cudaFuncSetAttribute(k_query_dense_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem));
    const int64_t wblocks = (nq + kWideWarps - 1) / kWideWarps;
    const unsigned wgrid = (unsigned)(wblocks < (int64_t)num_sms() * 32 ? wblocks : (int64_t)num_sms() * 32);
    k_query_dense_wide<<<wgrid, kWideWarps * 32, wsmem, st>>>(qi, Q, nq, knn, beam, ids, d2);
    MASK_LAUNCH_CHECK();
    return;
  }
  if (coop) {
    if (smem > 48 * 1024)
      MASK_CUDA(cudaFuncSetAttribute(k_query_dense<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_query_dense<8><<<grid, kWarpsPerBlock * 32, smem, st>>>(qi, Q, nq, knn, beam, ids, d2, lo);
  } else {
    if (smem > 48 * 1024)
      MASK_CUDA(cudaFuncSetAttribute(k_query_dense<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_query_dense<1><<<grid, kWarpsPerBlock * 32, smem, st>>>(qi, Q, nq, knn, beam, ids, d2, lo);
  }
  MASK_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------------
// CSR queries against a CSR-data index (prototypes dense).  q's non-zeros are staged in
// shared memory.  Prototype distance: ||c||^2 + sum_{p in nz(q)} (q_p^2 - 2 q_p c[col_p])
// (D12); data-row distance: direct sum over the union of the two sorted supports.
constexpr int kMaxQueryNnz = 1024;

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_query_csr(QIndex qi, const float* __restrict__ cn2_flat, const int64_t* __restrict__ cn2_off,
                const int64_t* __restrict__ qrp, const int32_t* __restrict__ qcol,
                const float* __restrict__ qval, int64_t nq, int knn, int beam,
                int64_t* __restrict__ ids_out, float* __restrict__ d2_out) {
  __shared__ int32_t s_col[kWarpsPerBlock][kMaxQueryNnz];
  __shared__ float s_val[kWarpsPerBlock][kMaxQueryNnz];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int d = qi.dim;
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t qid = (int64_t)blockIdx.x * kWarpsPerBlock + w; qid < nq; qid += nwarps) {
    if (qi.routed && !qi.routed[qid * qi.rstride]) {  // §3.4: not routed to this node
      if (lane < knn) {
        ids_out[qid * knn + lane] = -1;
        d2_out[qid * knn + lane] = INFINITY;
      }
      continue;
    }
    const int64_t p0 = qrp[qid];
    const int64_t qn = qrp[qid + 1] - p0;
    // the query's non-zeros: staged in shared memory up to kMaxQueryNnz, else read in place
    // from global memory (any length; never truncated)
    const bool staged = qn <= kMaxQueryNnz;
    const int32_t* qc = staged ? s_col[w] : qcol + p0;
    const float* qv = staged ? s_val[w] : qval + p0;
    __syncwarp();
    if (staged)
      for (int i = lane; i < qn; i += 32) {
        s_col[w][i] = qcol[p0 + i];
        s_val[w][i] = qval[p0 + i];
      }
    __syncwarp();
    float qq = 0.f;
    for (int64_t i = 0; i < qn; ++i) qq = fmaf(qv[i], qv[i], qq);
    auto proto_dist = [&](int l, int64_t j) {
      const float* c = qi.lv[l].P + j * d;
      float s = 0.f;
      for (int64_t i = 0; i < qn; ++i) s = fmaf(qv[i], __ldg(c + qc[i]), s);
      return cn2_flat[cn2_off[l] + j] + qq - 2.f * s;
    };
    WarpTopK top;
    {
      const int l = qi.L - 1;
      const QLevel& L = qi.lv[l];
      top.reset(beam);
      for (int64_t j0 = 0; j0 < L.k; j0 += 32) {
        const int64_t j = j0 + lane;
        float cd = INFINITY;
        int32_t cid = PAD_ID;
        if (j < L.k && has_children(L, j)) {
          cd = proto_dist(l, j);
          cid = (int32_t)j;
        }
        top.offer(cd, cid, lane);
      }
    }
    for (int l = qi.L - 2; l >= 0; --l) {
      const QLevel& up = qi.lv[l + 1];
      const QLevel& L = qi.lv[l];
      const int32_t sel_id = top.id;
      top.reset(beam);
      for (int s = 0; s < beam; ++s) {
        const int32_t p = __shfl_sync(FULL, sel_id, s);
        if (p == PAD_ID) continue;
        const int64_t m0 = up.offsets[p], m1 = up.offsets[p + 1];
        for (int64_t m = m0; m < m1; m += 32) {
          const int64_t mm = m + lane;
          float cd = INFINITY;
          int32_t cid = PAD_ID;
          if (mm < m1) {
            const int32_t j = up.members[mm];
            if (has_children(L, j)) {
              cd = proto_dist(l, j);
              cid = j;
            }
          }
          top.offer(cd, cid, lane);
        }
      }
    }
    {
      const QLevel& L1 = qi.lv[0];
      const int32_t sel_id = top.id;
      top.reset(knn);
      for (int s = 0; s < beam; ++s) {
        const int32_t p = __shfl_sync(FULL, sel_id, s);
        if (p == PAD_ID) continue;
        const int64_t m0 = L1.offsets[p], m1 = L1.offsets[p + 1];
        for (int64_t m = m0; m < m1; m += 32) {
          const int64_t mm = m + lane;
          float cd = INFINITY;
          int32_t cid = PAD_ID;
          if (mm < m1) {
            const int32_t i = L1.members[mm];
            int64_t a = qi.xrp[i];
            const int64_t ae = qi.xrp[i + 1];
            int64_t b = 0;
            float s = 0.f;
            while (a < ae || b < qn) {
              float t;
              const int32_t ca = a < ae ? __ldg(qi.xcol + a) : 0x7fffffff;
              const int32_t cb = b < qn ? qc[b] : 0x7fffffff;
              if (ca < cb) {
                t = __ldg(qi.xval + a);
                ++a;
              } else if (cb < ca) {
                t = qv[b];
                ++b;
              } else {
                t = __ldg(qi.xval + a) - qv[b];
                ++a;
                ++b;
              }
              s = fmaf(t, t, s);
            }
            cd = s;
            cid = i;
          }
          top.offer(cd, cid, lane);
        }
      }
    }
    if (lane < knn) {
      const bool pad = top.id == PAD_ID;
      ids_out[qid * knn + lane] = pad ? -1 : qi.id_base + (int64_t)top.id;
      d2_out[qid * knn + lane] = pad ? INFINITY : top.d;
    }
  }
}

void launch_query_csr(const QIndex& qi, const float* cn2_flat, const int64_t* cn2_off,
                      const int64_t* qrp, const int32_t* qcol, const float* qval, int64_t nq,
                      int knn, int beam, int64_t* ids, float* d2, cudaStream_t st) {
  if (nq <= 0) return;
  const int64_t blocks = (nq + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const unsigned grid = (unsigned)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  k_query_csr<<<grid, kWarpsPerBlock * 32, 0, st>>>(qi, cn2_flat, cn2_off, qrp, qcol, qval, nq, knn,
                                                     beam, ids, d2);
  MASK_LAUNCH_CHECK();
}

}  // namespace mask
