// sort.cu -- stable LSD radix sort of (uint64 key, int64 value) pairs, 8-bit digits.
// Used by the range search's result ordering (K13) and the relocation step (relocate.cu).
//
// Per digit pass: (1) a block per 4096-element tile counts its digits (hist[digit][tile]);
// (2) an exclusive scan of hist in (digit, tile) order gives every tile's first output slot
// per digit; (3) each tile re-reads its elements in order, 256 at a time, and ranks them
// stably: within a warp by __match_any_sync (rank = earlier lanes with the same digit), across
// the block's warps by a per-digit prefix over warps, across rounds by a running per-digit
// base.  Keys and values ping-pong between the caller's buffers and scratch.
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#include "common.cuh"

namespace mask {

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;

__global__ void __launch_bounds__(kSortThreads) k_radix_hist(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                                             int64_t ntiles, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int i = threadIdx.x; i < kSortTile; i += kSortThreads) {
    const int64_t e = base + i;
    if (e < n) atomicAdd(&h[(keys[e] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan of m uint32 counts into uint64 offsets: block-local scan + block sums
__global__ void __launch_bounds__(1024) k_scan_u32_1(const uint32_t* __restrict__ in, int64_t m,
                                                     uint64_t* __restrict__ out, uint64_t* __restrict__ bsum) {
  __shared__ uint64_t ws[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t e = (int64_t)blockIdx.x * 1024 + t;
  const uint64_t c = e < m ? in[e] : 0;
  uint64_t x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    uint64_t v = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    ws[lane] = v;
  }
  __syncthreads();
  if (e < m) out[e] = x - c + (w ? ws[w - 1] : 0);
  if (t == 1023) bsum[blockIdx.x] = ws[31];
}
__global__ void __launch_bounds__(1024) k_scan_u32_2(uint64_t* __restrict__ bsum, int64_t nb) {
  __shared__ uint64_t part[1024];
  const int t = threadIdx.x;
  const int64_t per = (nb + 1023) / 1024;
  const int64_t a = t * per, b = a + per < nb ? a + per : nb;
  uint64_t s = 0;
  for (int64_t j = a; j < b; ++j) s += bsum[j];
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const uint64_t v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  uint64_t run = part[t] - s;
  for (int64_t j = a; j < b; ++j) {
    const uint64_t c = bsum[j];
    bsum[j] = run;
    run += c;
  }
}
__global__ void k_scan_u32_3(uint64_t* __restrict__ out, int64_t m, const uint64_t* __restrict__ bsum) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
    out[e] += bsum[e / 1024];
}

__global__ void __launch_bounds__(kSortThreads) k_radix_scatter(const uint64_t* __restrict__ kin,
                                                                const int64_t* __restrict__ vin, int64_t n, int shift,
                                                                int64_t ntiles, const uint64_t* __restrict__ off,
                                                                uint64_t* __restrict__ kout, int64_t* __restrict__ vout) {
  constexpr int W = kSortThreads / 32;
  __shared__ uint32_t wcnt[W][256];
  __shared__ uint64_t base[256];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  base[t] = off[(int64_t)t * ntiles + blockIdx.x];  // (kSortThreads == 256 digits)
  const int64_t tile0 = (int64_t)blockIdx.x * kSortTile;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < kSortItems; ++r) {
    for (int i = t; i < W * 256; i += kSortThreads) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const int64_t e = tile0 + (int64_t)r * kSortThreads + t;
    const bool valid = e < n;
    uint64_t k = 0;
    int64_t v = 0;
    uint32_t dg = 256;  // (invalid: its own group, never counted)
    if (valid) {
      k = kin[e];
      v = vin[e];
      dg = (uint32_t)((k >> shift) & 255u);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, dg);
    const int rank = __popc(peers & lt);
    if (valid && rank == 0) wcnt[w][dg] = __popc(peers);
    __syncthreads();
    // per digit (thread t = digit t): exclusive prefix over the warps, then the round's total
    {
      uint32_t run = 0;
#pragma unroll
      for (int ww = 0; ww < W; ++ww) {
        const uint32_t c = wcnt[ww][t];
        wcnt[ww][t] = run;
        run += c;
      }
      __syncthreads();
      if (valid) {
        const uint64_t pos = base[dg] + wcnt[w][dg] + rank;
        kout[pos] = k;
        vout[pos] = v;
      }
      __syncthreads();
      base[t] += run;
    }
    __syncthreads();
  }
}

}  // namespace

void radix_sort_pairs(uint64_t* keys, int64_t* vals, int64_t n, int begin_bit, int end_bit, cudaStream_t st) {
  if (n <= 1) return;
  const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
  const int64_t m = 256 * ntiles;
  const int64_t nb = (m + 1023) / 1024;
  DevBuf<uint64_t> k2(n), off(m), bsum(nb + 1);
  DevBuf<int64_t> v2(n);
  DevBuf<uint32_t> hist(m);
  uint64_t* ka = keys;
  uint64_t* kb = k2.p;
  int64_t* va = vals;
  int64_t* vb = v2.p;
  int passes = 0;
  for (int shift = begin_bit; shift < end_bit; shift += 8, ++passes) {
    k_radix_hist<<<(unsigned)ntiles, kSortThreads, 0, st>>>(ka, n, shift, ntiles, hist.p);
    MASK_LAUNCH_CHECK();
    k_scan_u32_1<<<(unsigned)nb, 1024, 0, st>>>(hist.p, m, off.p, bsum.p);
    MASK_LAUNCH_CHECK();
    k_scan_u32_2<<<1, 1024, 0, st>>>(bsum.p, nb);
    MASK_LAUNCH_CHECK();
    k_scan_u32_3<<<grid_for(m, 256), 256, 0, st>>>(off.p, m, bsum.p);
    MASK_LAUNCH_CHECK();
    k_radix_scatter<<<(unsigned)ntiles, kSortThreads, 0, st>>>(ka, va, n, shift, ntiles, off.p, kb, vb);
    MASK_LAUNCH_CHECK();
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  if (passes & 1) {  // the result is in the scratch buffers: copy back
    MASK_CUDA(cudaMemcpyAsync(keys, ka, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, st));
    MASK_CUDA(cudaMemcpyAsync(vals, va, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st));
  }
  MASK_CUDA(cudaStreamSynchronize(st));  // (scratch goes out of scope)
}

}  // namespace mask
