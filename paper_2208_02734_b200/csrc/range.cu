// range.cu -- K13: range search over the multilevel index (Algorithm 3, P:917-960;
// SURVEY §8(f) NEXT-2) and the prototypes' cover radii.
//
// Multi-path descent: at the top level every prototype with children is tested; at each lower
// level the candidates are the children of the prototypes kept above; at the data layer the
// rows of the kept level-1 prototypes with ||q - x|| <= r are returned, sorted by (d^2, id).
//   mode PAPER (Algorithm 3's `selectCandidates(sortVecCentroids, radius)`): keep c iff
//        ||q - c|| <= r;
//   mode COVER: keep c iff ||q - c|| <= r + cover(c), where cover(c) bounds the distance from c
//        to every data row below it (level 1: max over members; level l: max over children i of
//        ||c_i - c|| + cover(c_i), the triangle inequality), so no row within r is lost: the
//        result equals the brute-force range scan (lossless, SPEC range_query).
// The descent is level-synchronous over all queries: (query, prototype) frontier entries are
// appended with atomics (one warp per entry, lanes over its children), the host reads the
// frontier size once per level (grows the buffer when needed).  FP32 direct distances; the
// cover test carries a 1e-6 relative slack for the rounding of the radii themselves.
#include <cuda_runtime.h>


#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace mask {

namespace {

__device__ __forceinline__ float dist2_dense(const float* a, const float* b, int d) {
  float acc = 0.f;
  for (int c = 0; c < d; ++c) {
    const float t = a[c] - b[c];
    acc = fmaf(t, t, acc);
  }
  return acc;
}

// cover radius, level 1: cover[j] = max_{labels[i] = j} ||x_i - c_j|| (float bits, atomicMax)
__global__ void k_cover_rows(const float* __restrict__ X, int d, const float* __restrict__ P,
                             const int32_t* __restrict__ labels, int64_t n, unsigned* __restrict__ cover) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = labels[i];
    const float r = sqrtf(dist2_dense(X + i * d, P + (int64_t)j * d, d));
    atomicMax(cover + j, __float_as_uint(r));
  }
}

// cover radius, level l >= 2: cover[j] = max over children i of ||c_i - c_j|| + cover_prev[i]
__global__ void k_cover_up(const float* __restrict__ Pprev, const unsigned* __restrict__ cover_prev, int d,
                           const float* __restrict__ P, const int32_t* __restrict__ labels, int64_t n,
                           unsigned* __restrict__ cover) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = labels[i];
    const float r = sqrtf(dist2_dense(Pprev + i * d, P + (int64_t)j * d, d)) + __uint_as_float(cover_prev[i]);
    atomicMax(cover + j, __float_as_uint(r));
  }
}

__device__ __forceinline__ bool keep(float d2, float r, float cover, int mode) {
  const float lim = mode == MASK_RANGE_COVER ? (r + cover) * (1.f + 1e-6f) : r;
  return d2 <= lim * lim;
}

// top level: (q, j) for every query and every prototype with children
__global__ void k_range_top(const float* __restrict__ Q, int64_t nq, int d, const float* __restrict__ P,
                            const int64_t* __restrict__ offsets, const unsigned* __restrict__ cover, int64_t k,
                            const float* __restrict__ radius, int mode, int2* __restrict__ out,
                            unsigned long long* __restrict__ count, int64_t cap) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nq * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / k, j = e - q * k;
    if (offsets[j + 1] == offsets[j]) continue;  // childless: leads to no row
    const float d2 = dist2_dense(Q + q * d, P + j * d, d);
    if (keep(d2, radius[q], cover ? __uint_as_float(cover[j]) : 0.f, mode)) {
      const unsigned long long slot = atomicAdd(count, 1ull);
      if ((int64_t)slot < cap) out[slot] = make_int2((int)q, (int)j);
    }
  }
}

// one level down: warp per frontier entry (q, j), lanes over j's children i (prototypes of the
// level below, or data rows when leaf != 0: then results (q, row, d^2) are appended)
__global__ void k_range_expand(const int2* __restrict__ in, int64_t n_in, const float* __restrict__ Q, int d,
                               const int64_t* __restrict__ offsets, const int32_t* __restrict__ members,
                               const float* __restrict__ Pc, const unsigned* __restrict__ cover_c,
                               const int64_t* __restrict__ offsets_c, const float* __restrict__ radius, int mode,
                               int leaf, int2* __restrict__ out, float* __restrict__ out_d2,
                               unsigned long long* __restrict__ count, int64_t cap) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < n_in; w += warps) {
    const int2 f = in[w];
    const float r = radius[f.x];
    const float* q = Q + (int64_t)f.x * d;
    for (int64_t p = offsets[f.y] + lane; p < offsets[f.y + 1]; p += 32) {
      const int32_t i = members[p];
      const float d2 = dist2_dense(q, Pc + (int64_t)i * d, d);
      bool ok;
      if (leaf) ok = d2 <= r * r;
      else ok = offsets_c[i + 1] > offsets_c[i] && keep(d2, r, cover_c ? __uint_as_float(cover_c[i]) : 0.f, mode);
      if (ok) {
        const unsigned long long slot = atomicAdd(count, 1ull);
        if ((int64_t)slot < cap) {
          out[slot] = make_int2(f.x, i);
          if (leaf) out_d2[slot] = d2;
        }
      }
    }
  }
}

__global__ void k_gather_u64(const unsigned long long* __restrict__ in, const int64_t* __restrict__ ix, int64_t n,
                             unsigned long long* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = in[ix[e]];
}

__global__ void k_range_keys(const int2* __restrict__ res, const float* __restrict__ d2, int64_t n,
                             unsigned long long* __restrict__ key_qd, unsigned long long* __restrict__ key_id,
                             int64_t* __restrict__ idx) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    key_qd[e] = ((unsigned long long)(uint32_t)res[e].x << 32) | __float_as_uint(d2[e]);
    key_id[e] = (unsigned long long)(uint32_t)res[e].y;
    idx[e] = e;
  }
}

__global__ void k_range_write(const int64_t* __restrict__ order, const int2* __restrict__ res,
                              const float* __restrict__ d2, int64_t n, int64_t* __restrict__ ids_out,
                              float* __restrict__ d2_out, int64_t* __restrict__ qcount) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = order[e];
    ids_out[e] = res[s].y;
    d2_out[e] = d2[s];
    atomicAdd(reinterpret_cast<unsigned long long*>(qcount + res[s].x), 1ull);
  }
}

}  // namespace

void launch_cover_radii(const float* X, int d, const QIndex& qi, const int32_t* const* labels,
                        const int64_t* n_items, unsigned* const* cover, cudaStream_t st) {
  for (int l = 0; l < qi.L; ++l) {
    MASK_CUDA(cudaMemsetAsync(cover[l], 0, sizeof(unsigned) * qi.lv[l].k, st));
    const unsigned grid = grid_for(n_items[l], 256);
    if (l == 0)
      k_cover_rows<<<grid, 256, 0, st>>>(X, d, qi.lv[0].P, labels[0], n_items[0], cover[0]);
    else
      k_cover_up<<<grid, 256, 0, st>>>(qi.lv[l - 1].P, cover[l - 1], d, qi.lv[l].P, labels[l], n_items[l], cover[l]);
    MASK_LAUNCH_CHECK();
  }
}

// Runs the descent; returns the number of results.  If ids_out is non-null (capacity cap_out),
// writes the sorted results and per-query counts (qcount, nq entries, device).
int64_t range_search(const QIndex& qi, const unsigned* const* cover, const float* Q, int64_t nq, const float* radius,
                     int mode, int64_t* ids_out, float* d2_out, int64_t* qcount, int64_t cap_out, cudaStream_t st) {
  const int d = qi.dim;
  const int L = qi.L;
  DevBuf<unsigned long long> cnt(1);
  int64_t cap = std::max<int64_t>(1 << 16, nq * 64);
  DevBuf<int2> cur, nxt;
  DevBuf<float> res_d2;
  auto read_count = [&]() {
    unsigned long long h = 0;
    MASK_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    MASK_CUDA(cudaStreamSynchronize(st));
    return (int64_t)h;
  };
  const QLevel& top = qi.lv[L - 1];
  int64_t n_cur = 0;
  for (;;) {  // top level (re-run with a larger buffer if it overflowed)
    cur.alloc(cap);
    MASK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
    k_range_top<<<grid_for(nq * top.k, 256), 256, 0, st>>>(Q, nq, d, top.P, top.offsets,
                                                          cover ? cover[L - 1] : nullptr, top.k, radius, mode, cur.p,
                                                          cnt.p, cap);
    MASK_LAUNCH_CHECK();
    n_cur = read_count();
    if (n_cur <= cap) break;
    cap = n_cur;
  }
  for (int l = L - 1; l >= 0; --l) {  // expand level l+1's kept prototypes into level l (l = 0: rows)
    const QLevel& lv = qi.lv[l];
    const bool leaf = l == 0;
    const float* Pc = leaf ? qi.X : qi.lv[l - 1].P;
    const int64_t* offc = leaf ? nullptr : qi.lv[l - 1].offsets;
    const unsigned* covc = (leaf || !cover) ? nullptr : cover[l - 1];
    int64_t capn = std::max<int64_t>(cap, n_cur * 4);
    int64_t n_next = 0;
    for (;;) {
      nxt.alloc(std::max<int64_t>(capn, 1));
      if (leaf) res_d2.alloc(std::max<int64_t>(capn, 1));
      MASK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
      if (n_cur > 0) {
        k_range_expand<<<grid_for(n_cur * 32, 256), 256, 0, st>>>(cur.p, n_cur, Q, d, lv.offsets, lv.members, Pc, covc,
                                                                  offc, radius, mode, leaf ? 1 : 0, nxt.p,
                                                                  leaf ? res_d2.p : nullptr, cnt.p, capn);
        MASK_LAUNCH_CHECK();
      }
      n_next = read_count();
      if (n_next <= capn) break;
      capn = n_next;
    }
    std::swap(cur, nxt);
    n_cur = n_next;
    cap = capn;
  }
  // cur holds (q, row) results with res_d2; sort by (q, d^2, row) when the caller has room
  const int64_t n = n_cur;
  if (ids_out == nullptr || n > cap_out) return n;
  MASK_CUDA(cudaMemsetAsync(qcount, 0, sizeof(int64_t) * nq, st));
  if (n == 0) return 0;
  DevBuf<unsigned long long> kqd(n), kid(n), kqd_g(n);
  DevBuf<int64_t> ix(n);
  k_range_keys<<<grid_for(n, 256), 256, 0, st>>>(cur.p, res_d2.p, n, kqd.p, kid.p, ix.p);
  MASK_LAUNCH_CHECK();
  // LSD on the two keys (sort.cu, stable): by row id, then by (query, d^2 bits) carrying the
  // permutation -- equal (query, d^2) keep ascending row ids
  radix_sort_pairs(reinterpret_cast<uint64_t*>(kid.p), ix.p, n, 0, 32, st);
  k_gather_u64<<<grid_for(n, 256), 256, 0, st>>>(kqd.p, ix.p, n, kqd_g.p);
  MASK_LAUNCH_CHECK();
  radix_sort_pairs(reinterpret_cast<uint64_t*>(kqd_g.p), ix.p, n, 0, 64, st);
  k_range_write<<<grid_for(n, 256), 256, 0, st>>>(ix.p, cur.p, res_d2.p, n, ids_out, d2_out, qcount);
  MASK_LAUNCH_CHECK();
  return n;
}

}  // namespace mask
