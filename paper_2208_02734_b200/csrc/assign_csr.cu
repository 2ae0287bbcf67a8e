// assign_csr.cu -- K3: sparse (CSR) rows against dense prototypes (the high-dimensional,
// high-sparsity workload of PAPER.md §4.3; BASELINE.json configs[3]).
//
//   s_ij = ||c_j||^2 - 2 sum_{p in nz(i)} v_p c_j[col_p]          (D12; ||x_i||^2 is a row
//   constant, added back to the winner: d^2 = s + ||x_i||^2)
//
// One warp per row; the row's non-zeros are staged in registers/shared memory and the
// prototypes are read through the transposed copy PT (d x k, row = feature), so for a fixed
// non-zero the 32 lanes read 32 consecutive prototypes (coalesced 128-byte gathers).  Each
// lane accumulates R = 8 prototypes at a time (a 256-prototype chunk per warp iteration),
// keeping a running (s, j) argmin; lowest j wins ties (D4).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "common.cuh"

namespace mask {

namespace {
constexpr int kRowsPerBlock = 8;  // warps per block
constexpr int kR = 8;             // prototypes per lane per chunk
constexpr int kMaxNnzSmem = 256;  // staged non-zeros per row (longer rows stream from global)
}  // namespace

__global__ void __launch_bounds__(kRowsPerBlock * 32)
    k_assign_csr(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                 const float* __restrict__ val, int64_t n, const float* __restrict__ PT,
                 const float* __restrict__ cn2, int64_t k, int32_t* __restrict__ labels,
                 float* __restrict__ best_out, const int* __restrict__ active) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  __shared__ int32_t s_col[kRowsPerBlock][kMaxNnzSmem];
  __shared__ float s_val[kRowsPerBlock][kMaxNnzSmem];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * kRowsPerBlock;
  for (int64_t r = (int64_t)blockIdx.x * kRowsPerBlock + w; r < n; r += nwarps) {
    const int64_t p0 = rp[r];
    const int nz = (int)(rp[r + 1] - p0);
    const int nzs = nz < kMaxNnzSmem ? nz : kMaxNnzSmem;
    __syncwarp();
    float xx = 0.f;
    for (int i = lane; i < nzs; i += 32) {
      s_col[w][i] = col[p0 + i];
      s_val[w][i] = val[p0 + i];
    }
    for (int i = lane; i < nz; i += 32) {
      const float v = val[p0 + i];
      xx = fmaf(v, v, xx);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xx += __shfl_xor_sync(0xffffffffu, xx, o);
    __syncwarp();
    float b = INFINITY;
    int64_t a = INT64_MAX;
    for (int64_t j0 = 0; j0 < k; j0 += 32 * kR) {
      float acc[kR];
#pragma unroll
      for (int t = 0; t < kR; ++t) acc[t] = 0.f;
      for (int p = 0; p < nz; ++p) {
        const int32_t c = p < kMaxNnzSmem ? s_col[w][p] : col[p0 + p];
        const float v = p < kMaxNnzSmem ? s_val[w][p] : val[p0 + p];
        const float* row = PT + (int64_t)c * k + j0 + lane;
#pragma unroll
        for (int t = 0; t < kR; ++t) {
          const int64_t j = j0 + lane + 32 * t;
          if (j < k) acc[t] = fmaf(v, __ldg(row + 32 * t), acc[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < kR; ++t) {
        const int64_t j = j0 + lane + 32 * t;
        if (j < k) {
          const float s = fmaf(-2.f, acc[t], __ldg(cn2 + j));
          if (s < b) {  // j increases with t for a fixed lane: strict < keeps the lowest j
            b = s;
            a = j;
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, b, o);
      const int64_t oa = __shfl_xor_sync(0xffffffffu, a, o);
      if (ob < b || (ob == b && oa < a)) {
        b = ob;
        a = oa;
      }
    }
    if (lane == 0) {
      labels[r] = (int32_t)a;
      if (best_out) best_out[r] = fmaxf(b + xx, 0.f);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// K3 (chunk-major): the same scores with the loops swapped so the prototype working set is
// shared.  Persistent CTAs (one per SM) each own a contiguous range of rows and sweep the
// prototypes in 256-wide chunks; all CTAs work on the same chunk at about the same time, so the
// chunk's slice of PT (d x 256 floats: 10 MB at C4) stays L2-resident instead of every row
// streaming all of PT from HBM.  The HOT most frequent columns (Zipf-distributed features,
// SURVEY §8(d) G4) have their chunk rows staged in shared memory once per CTA and chunk, so
// most non-zeros read shared memory; the rest read L2 (two 16-byte loads per lane and
// non-zero).  A row's running argmin across chunks lives
// in `state` (global, L2); the last chunk writes the label and d^2 = s + ||x||^2.
// (Lane l covers prototypes j0 + 128 i + 4 l + (0..3): conflict-free 16-byte loads.)
constexpr int kPL = 8;          // prototypes per lane (8 FMAs per non-zero per warp visit)
constexpr int kChunk = 32 * kPL;  // prototypes per chunk
constexpr int kHot = 128;       // columns staged per chunk (kHot x kChunk floats = 128 KB)
constexpr int kG = 4;           // non-zeros in flight per warp step (kG x kPL floats of loads)
constexpr int kCsrWarps = 24;   // warps per CTA (85 registers each; measured best of 16/24/32 warps,
                                // 8/16 prototypes per lane, 64/128 hot columns)

// one staged non-zero: element offset of its P^T row (tail: col * k; hot: slot * kChunk), value
struct __align__(16) NzEntry {
  int64_t off;
  float v;
  float pad;
};

// Lane l covers the chunk's prototypes 128 i + 4 l + (0..3), i < kPL / 4: each float4 load of
// the warp reads 512 contiguous bytes (4 wavefronts; a 32-byte lane stride would need 8)
__device__ __forceinline__ int pl_off(int u, int lane) { return (u >> 2) * 128 + 4 * lane + (u & 3); }

// r[i] = the 4 floats at p + 128 i (p = chunk base + 4 lane, 16-byte aligned)
template <bool SMEM>
__device__ __forceinline__ void load_pl(const float* p, float4 (&r)[kPL / 4]) {
#pragma unroll
  for (int i = 0; i < kPL / 4; ++i)
    r[i] = SMEM ? *reinterpret_cast<const float4*>(p + 128 * i) : __ldg(reinterpret_cast<const float4*>(p + 128 * i));
}
__device__ __forceinline__ void fma_pl(float v, const float4 (&r)[kPL / 4], float (&acc)[kPL]) {
#pragma unroll
  for (int i = 0; i < kPL / 4; ++i) {
    acc[4 * i + 0] = fmaf(v, r[i].x, acc[4 * i + 0]);
    acc[4 * i + 1] = fmaf(v, r[i].y, acc[4 * i + 1]);
    acc[4 * i + 2] = fmaf(v, r[i].z, acc[4 * i + 2]);
    acc[4 * i + 3] = fmaf(v, r[i].w, acc[4 * i + 3]);
  }
}

__global__ void __launch_bounds__(kCsrWarps * 32, 1)
    k_assign_csr_chunked(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                         const float* __restrict__ val, int64_t n, int d, const float* __restrict__ PT,
                         const float* __restrict__ cn2, int64_t k, const int16_t* __restrict__ colslot,
                         const int32_t* __restrict__ hotcols, float2* __restrict__ state,
                         int32_t* __restrict__ labels, float* __restrict__ best_out, const int* __restrict__ active) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  extern __shared__ __align__(16) uint8_t smem_raw[];
  float* hotPT = reinterpret_cast<float*>(smem_raw);                                       // [kHot][kChunk]
  NzEntry* lists = reinterpret_cast<NzEntry*>(smem_raw + kHot * kChunk * sizeof(float));  // [warps][2][32]
  int16_t* slot = reinterpret_cast<int16_t*>(lists + kCsrWarps * 64);                      // [d]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  NzEntry* lt_list = lists + w * 64;
  NzEntry* hot_list = lt_list + 32;
  for (int c = threadIdx.x; c < d; c += blockDim.x) slot[c] = colslot[c];
  const int64_t r0 = n * blockIdx.x / gridDim.x, r1 = n * (blockIdx.x + 1) / gridDim.x;
  const int nch = (int)((k + kChunk - 1) / kChunk);
  const bool kvec = (k & 3) == 0;  // 16-byte aligned PT rows
  for (int ch = 0; ch < nch; ++ch) {
    const int64_t j0 = (int64_t)ch * kChunk;
    __syncthreads();  // previous chunk's readers are done with hotPT
    for (int e = threadIdx.x; e < kHot * (kChunk / 4); e += blockDim.x) {
      const int h = e / (kChunk / 4), q = e - h * (kChunk / 4);
      const int64_t j = j0 + 4 * q;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (hotcols[h] >= 0) {
        const float* src = PT + (int64_t)hotcols[h] * k + j;
        if (j + 3 < k && kvec) v = *reinterpret_cast<const float4*>(src);
        else {
          if (j < k) v.x = src[0];
          if (j + 1 < k) v.y = src[1];
          if (j + 2 < k) v.z = src[2];
          if (j + 3 < k) v.w = src[3];
        }
      }
      reinterpret_cast<float4*>(hotPT)[e] = v;
    }
    __syncthreads();
    // this lane's kPL prototypes of the chunk: ||c||^2 (+inf beyond k: never chosen)
    float cc[kPL];
#pragma unroll
    for (int u = 0; u < kPL; ++u) {
      const int64_t j = j0 + pl_off(u, lane);
      cc[u] = j < k ? __ldg(cn2 + j) : INFINITY;
    }
    const bool vec_ok = j0 + pl_off(kPL - 1, lane) < k && kvec;
    for (int64_t r = r0 + w; r < r1; r += kCsrWarps) {
      const int64_t p0 = rp[r], p1 = rp[r + 1];
      float acc[kPL];
#pragma unroll
      for (int u = 0; u < kPL; ++u) acc[u] = 0.f;
      for (int64_t pb = p0; pb < p1; pb += 32) {
        const int m = p1 - pb < 32 ? (int)(p1 - pb) : 32;
        // each lane resolves one non-zero's hot slot; the warp compacts the block into a tail
        // (L2) list and a hot (shared-memory) list of {element offset, value}, padded to a
        // multiple of kG with zero entries, then walks each list kG entries at a time: one
        // broadcast 16-byte LDS per entry, both loads issued before the FMAs
        int32_t msl = -1;
        int64_t moff = 0;
        float mv = 0.f;
        if (lane < m) {
          const int32_t mc = __ldg(col + pb + lane);
          mv = __ldg(val + pb + lane);
          msl = slot[mc];
          moff = msl >= 0 ? (int64_t)msl * kChunk : (int64_t)mc * k;
        }
        const unsigned lt = (1u << lane) - 1u;
        const unsigned tb = __ballot_sync(0xffffffffu, lane < m && msl < 0);
        const unsigned hb = __ballot_sync(0xffffffffu, lane < m && msl >= 0);
        const int nt = __popc(tb), nh = __popc(hb);
        __syncwarp();  // the previous block's readers are done with the lists
        if (lane < m) {
          NzEntry* dst = msl < 0 ? lt_list + __popc(tb & lt) : hot_list + __popc(hb & lt);
          *dst = NzEntry{moff, mv, 0.f};
        }
        const int ntp = (nt + kG - 1) / kG * kG, nhp = (nh + kG - 1) / kG * kG;
        if (lane >= nt && lane < ntp) lt_list[lane] = NzEntry{0, 0.f, 0.f};
        if (lane >= nh && lane < nhp) hot_list[lane] = NzEntry{0, 0.f, 0.f};
        __syncwarp();
        for (int i = 0; i < ntp; i += kG) {
          float vq[kG];
          float4 rb[kG][kPL / 4];
#pragma unroll
          for (int g = 0; g < kG; ++g) {
            const NzEntry e = lt_list[i + g];
            vq[g] = e.v;
            const float* src = PT + e.off + j0;
            if (vec_ok) {
              load_pl<false>(src + 4 * lane, rb[g]);
            } else {
              float tt[kPL];
#pragma unroll
              for (int u = 0; u < kPL; ++u) tt[u] = j0 + pl_off(u, lane) < k ? __ldg(src + pl_off(u, lane)) : 0.f;
#pragma unroll
              for (int u = 0; u < kPL / 4; ++u) rb[g][u] = make_float4(tt[4 * u], tt[4 * u + 1], tt[4 * u + 2], tt[4 * u + 3]);
            }
          }
#pragma unroll
          for (int g = 0; g < kG; ++g) fma_pl(vq[g], rb[g], acc);
        }
        for (int i = 0; i < nhp; i += kG) {
          float vq[kG];
          float4 rb[kG][kPL / 4];
#pragma unroll
          for (int g = 0; g < kG; ++g) {
            const NzEntry e = hot_list[i + g];
            vq[g] = e.v;
            load_pl<true>(hotPT + e.off + 4 * lane, rb[g]);
          }
#pragma unroll
          for (int g = 0; g < kG; ++g) fma_pl(vq[g], rb[g], acc);
        }
      }
      // lane argmin over its kPL (j increasing: strict < keeps the lowest j), then the warp's
      float bv = INFINITY;
      int32_t bj = 0x7fffffff;
#pragma unroll
      for (int u = 0; u < kPL; ++u) {
        const float sv = fmaf(-2.f, acc[u], cc[u]);
        if (sv < bv) {
          bv = sv;
          bj = (int32_t)(j0 + pl_off(u, lane));
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int32_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ov < bv || (ov == bv && oj < bj)) {
          bv = ov;
          bj = oj;
        }
      }
      if (ch > 0) {  // earlier chunks hold lower j: they win ties
        const float2 st = state[r];
        if (!(bv < st.x)) {
          bv = st.x;
          bj = __float_as_int(st.y);
        }
      }
      if (ch + 1 < nch) {
        if (lane == 0) state[r] = make_float2(bv, __int_as_float(bj));
      } else {
        float xx = 0.f;
        for (int64_t p = p0 + lane; p < p1; p += 32) {
          const float v = __ldg(val + p);
          xx = fmaf(v, v, xx);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) xx += __shfl_xor_sync(0xffffffffu, xx, o);
        if (lane == 0) {
          labels[r] = bj;
          if (best_out) best_out[r] = fmaxf(bv + xx, 0.f);
        }
      }
    }
  }
}

size_t csr_chunked_smem(int d) {
  return (size_t)kHot * kChunk * sizeof(float) + (size_t)kCsrWarps * 64 * sizeof(NzEntry) + (size_t)d * sizeof(int16_t);
}

int csr_chunked_hot() { return kHot; }

bool csr_chunked_supported(int d, int64_t k) {
  (void)k;
  return d <= 32767 && csr_chunked_smem(d) <= 227 * 1024;
}

void launch_assign_csr_chunked(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t n, int d,
                               const float* PT, const float* cn2, int64_t k, const int16_t* colslot,
                               const int32_t* hotcols, float2* state, int32_t* labels, float* best, cudaStream_t st,
                               const int* active) {
  if (n <= 0) return;
  const size_t smem = csr_chunked_smem(d);
  static bool attr = false;
  if (!attr) {
    MASK_CUDA(cudaFuncSetAttribute(k_assign_csr_chunked, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  const int64_t grid = std::min<int64_t>(num_sms(), (n + kCsrWarps - 1) / kCsrWarps);
  k_assign_csr_chunked<<<(unsigned)grid, kCsrWarps * 32, smem, st>>>(row_ptr, col, val, n, d, PT, cn2, k, colslot,
                                                                    hotcols, state, labels, best, active);
  MASK_LAUNCH_CHECK();
}

// Column statistics for the hot set: cnt[c] = non-zeros in column c (shared-memory histogram
// per block when d fits, else global atomics).
__global__ void k_col_hist(const int32_t* __restrict__ col, int64_t nnz, int d, int32_t* __restrict__ cnt) {
  extern __shared__ int32_t h[];
  const bool sm = d <= 12288;
  if (sm)
    for (int c = threadIdx.x; c < d; c += blockDim.x) h[c] = 0;
  __syncthreads();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = col[p];
    if (sm) atomicAdd(h + c, 1);
    else atomicAdd(cnt + c, 1);
  }
  __syncthreads();
  if (sm)
    for (int c = threadIdx.x; c < d; c += blockDim.x)
      if (h[c]) atomicAdd(cnt + c, h[c]);
}

void launch_col_hist(const int32_t* col, int64_t nnz, int d, int32_t* cnt, cudaStream_t st) {
  MASK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * d, st));
  if (nnz <= 0) return;
  const size_t smem = d <= 12288 ? (size_t)d * sizeof(int32_t) : 0;
  k_col_hist<<<grid_for(nnz, 256, (int64_t)num_sms() * 4), 256, smem, st>>>(col, nnz, d, cnt);
  MASK_LAUNCH_CHECK();
}

void launch_assign_csr(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t n,
                       int d, const float* PT, const float* cn2, int64_t k, int32_t* labels,
                       float* best, cudaStream_t st, const int* active) {
  (void)d;
  if (n <= 0) return;
  const int64_t blocks = (n + kRowsPerBlock - 1) / kRowsPerBlock;
  const unsigned grid = (unsigned)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  k_assign_csr<<<grid, kRowsPerBlock * 32, 0, st>>>(row_ptr, col, val, n, PT, cn2, k, labels, best, active);
  MASK_LAUNCH_CHECK();
}

// K3 hot set on the device (no host round trip): the H columns with the most non-zeros (lower
// index on equal counts; never a zero-count column).  One block: a binary search for the count
// threshold c* = min{c : #(cnt > c) < H}, then every column above c* and the lowest-index
// columns at c* until H, slots in ascending column order within each group.
__global__ void __launch_bounds__(1024) k_select_hot(const int32_t* __restrict__ cnt, int d, int H,
                                                     int32_t* __restrict__ hotcols, int16_t* __restrict__ colslot) {
  __shared__ int s_red[32];
  __shared__ int s_scan[32];
  __shared__ int s_base;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  auto block_sum = [&](int v) {
    v = __reduce_add_sync(0xffffffffu, v);
    __syncthreads();
    if (lane == 0) s_red[w] = v;
    __syncthreads();
    int t = lane < nw ? s_red[lane] : 0;
    return __reduce_add_sync(0xffffffffu, t);
  };
  auto block_max = [&](int v) {
    v = __reduce_max_sync(0xffffffffu, v);
    __syncthreads();
    if (lane == 0) s_red[w] = v;
    __syncthreads();
    int t = lane < nw ? s_red[lane] : 0;
    return __reduce_max_sync(0xffffffffu, t);
  };
  for (int c = tid; c < d; c += blockDim.x) colslot[c] = -1;
  for (int h = tid; h < H; h += blockDim.x) hotcols[h] = -1;
  int m = 0;
  for (int c = tid; c < d; c += blockDim.x) m = max(m, cnt[c]);
  const int M = block_max(m);
  auto greater = [&](int thr) {
    int g = 0;
    for (int c = tid; c < d; c += blockDim.x) g += cnt[c] > thr ? 1 : 0;
    return block_sum(g);
  };
  int lo = 0, hi = M;
  while (lo < hi) {  // (uniform across the block)
    const int mid = lo + (hi - lo) / 2;
    if (greater(mid) < H) hi = mid;
    else lo = mid + 1;
  }
  const int cstar = lo;
  // ordered compaction: pass 0 = columns above c*, pass 1 = columns at c* (c* > 0) up to H
  if (tid == 0) s_base = 0;
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1 && cstar == 0) break;
    for (int c0 = 0; c0 < d; c0 += blockDim.x) {
      const int c = c0 + tid;
      const bool f = c < d && (pass == 0 ? cnt[c] > cstar : cnt[c] == cstar);
      const unsigned b = __ballot_sync(0xffffffffu, f);
      if (lane == 0) s_scan[w] = __popc(b);
      __syncthreads();
      int before = 0, total = 0;
      for (int i = 0; i < nw; ++i) {
        const int v = s_scan[i];
        before += i < w ? v : 0;
        total += v;
      }
      const int pos = s_base + before + __popc(b & ((1u << lane) - 1));
      if (f && pos < H) {
        hotcols[pos] = c;
        colslot[c] = (int16_t)pos;
      }
      __syncthreads();
      if (tid == 0) s_base += total;
      __syncthreads();
    }
  }
}

void launch_select_hot(const int32_t* cnt, int d, int H, int32_t* hotcols, int16_t* colslot, cudaStream_t st) {
  k_select_hot<<<1, 1024, 0, st>>>(cnt, d, H, hotcols, colslot);
  MASK_LAUNCH_CHECK();
}

}  // namespace mask
