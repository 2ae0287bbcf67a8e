// kernels_lloyd.cu -- SIMT kernels of one Lloyd level:
//   K2  FP32 SIMT assignment (small d / upper levels / fallback)
//   K4  near-tie FP32 re-check of rows flagged by the tensor-core assignment (K1)
//   K5  dense cluster sums + counts,  K6 CSR cluster sums + counts
//   K7  finalize: c_j <- S_j / n_j, keep empty (D5), displacement, empties
//   K8  child lists by counting sort
//   K10 seeded-init gather
// plus per-pass statistics, row norms and the 3xTF32 prototype operand split.
//
// Paper: assignment = `euclideanDistance` + `searchPosMin`, update =
// k-means prototype = mean of members, levels P:631-638.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include <map>
#include <mutex>

#include <cfloat>
#include <algorithm>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace mask {

// ====================================================================== K2 SIMT assignment
// One thread per row; prototypes staged through shared memory in chunks and read by
// broadcast.  Direct squared distance sum_i (x_i - c_i)^2 with FP32 FMA accumulation;
// strict "<" over ascending j keeps the lowest ordinal on ties (D4).
template <int DT>
__global__ void __launch_bounds__(256) k_assign_simt(const float* __restrict__ X, int64_t n,
                                                     int d, const float* __restrict__ P,
                                                     int64_t k, int kc_max,
                                                     int32_t* __restrict__ labels,
                                                     float* __restrict__ best_out,
                                                     const int* __restrict__ active) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  extern __shared__ float sP[];
  const int D = DT > 0 ? DT : d;
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = row < n;
  float x[DT > 0 ? DT : 1];
  if (DT > 0) {
#pragma unroll
    for (int i = 0; i < (DT > 0 ? DT : 1); ++i) x[i] = valid ? X[row * D + i] : 0.f;
  }
  float b1 = INFINITY;
  int64_t a = 0;
  for (int64_t j0 = 0; j0 < k; j0 += kc_max) {
    const int kc = (int)min64(kc_max, k - j0);
    __syncthreads();
    for (int t = threadIdx.x; t < kc * D; t += blockDim.x) sP[t] = P[j0 * D + t];
    __syncthreads();
    if (valid) {
      for (int jj = 0; jj < kc; ++jj) {
        const float* c = sP + jj * D;
        float s = 0.f;
        if (DT > 0) {
#pragma unroll
          for (int i = 0; i < (DT > 0 ? DT : 1); ++i) {
            float t = x[i] - c[i];
            s = fmaf(t, t, s);
          }
        } else {
          const float* xr = X + row * D;
          for (int i = 0; i < D; ++i) {
            float t = __ldg(xr + i) - c[i];
            s = fmaf(t, t, s);
          }
        }
        if (s < b1) {
          b1 = s;
          a = j0 + jj;
        }
      }
    }
  }
  if (valid) {
    labels[row] = (int32_t)a;
    if (best_out) best_out[row] = b1;
  }
}

void launch_assign_simt(const float* X, int64_t n, int d, const float* P, int64_t k,
                        int32_t* labels, float* best, cudaStream_t st, const int* active) {
  if (n <= 0) return;
  const int block = 256;
  int kc = (int)min64(k, 40 * 1024 / (4 * (int64_t)d));
  if (kc < 1) kc = 1;
  size_t smem = (size_t)kc * d * sizeof(float);
  if (smem > 48 * 1024) {
    MASK_REQUIRE(smem <= 200 * 1024, MASK_ERR_UNSUPPORTED, "SIMT assignment: dim too large");
  }
  unsigned grid = (unsigned)((n + block - 1) / block);
#define MASK_SIMT_CASE(DV)                                                                \
  case DV: {                                                                              \
    if (smem > 48 * 1024)                                                                 \
      MASK_CUDA(cudaFuncSetAttribute(k_assign_simt<DV>,                                   \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k_assign_simt<DV><<<grid, block, smem, st>>>(X, n, d, P, k, kc, labels, best, active);        \
    break;                                                                                \
  }
  switch (d) {
    MASK_SIMT_CASE(1)
    MASK_SIMT_CASE(2)
    MASK_SIMT_CASE(3)
    MASK_SIMT_CASE(4)
    MASK_SIMT_CASE(8)
    MASK_SIMT_CASE(16)
    MASK_SIMT_CASE(32)
    MASK_SIMT_CASE(64)
    default: {
      if (smem > 48 * 1024)
        MASK_CUDA(cudaFuncSetAttribute(k_assign_simt<0>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_assign_simt<0><<<grid, block, smem, st>>>(X, n, d, P, k, kc, labels, best, active);
    }
  }
#undef MASK_SIMT_CASE
  MASK_LAUNCH_CHECK();
}

// ====================================================================== K4 near-tie re-check
namespace {
constexpr int FX_R = 32, FX_P = 128;
}

// Blocked SIMT argmin (K4 re-check and the large-d assignment): rows = rows[0..count) (or the
// identity when rows == nullptr), count = min(*count_dev, cap) (or cap when count_dev ==
// nullptr), read on the device so no host round trip is needed.  Block b walks work items (32-row
// block, prototype split) b, b + gridDim.x, ...; each item sweeps its 128-prototype tiles with
// the dimension streamed through shared memory in chunks of FX_DK (thread = 4 rows x 4
// prototypes, direct FP32 sums of squares); per row the best (d^2, j) is merged with a 64-bit
// atomicMin on (d^2 bits << 32 | j).
constexpr int FX_DK = 64;

__global__ void __launch_bounds__(256) k_blocked_argmin(const float* __restrict__ X, int d,
                                                        const float* __restrict__ P, int64_t k,
                                                        const int32_t* __restrict__ rows,
                                                        const int32_t* __restrict__ count_dev, int64_t cap,
                                                        int nsm, unsigned long long* __restrict__ keys,
                                                        const int* __restrict__ active) {
  using Acc = float;  // (FP32 keys: the shared key code below)
  constexpr bool EXACT = false;
  constexpr int jbits = 0;
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  __shared__ float xs[FX_R * (FX_DK + 1)];
  __shared__ float cs[FX_P * (FX_DK + 1)];
  const int64_t nf = count_dev ? min64(*count_dev, cap) : cap;
  if (nf <= 0) return;
  constexpr int dp = FX_DK + 1;
  const int t = threadIdx.x;
  const int rg = t & 7, pg = t >> 3;
  const int64_t row_blocks = (nf + FX_R - 1) / FX_R;
  const int64_t ntile = (k + FX_P - 1) / FX_P;
  int64_t splits = (4LL * nsm + row_blocks - 1) / row_blocks;
  splits = splits < 1 ? 1 : (splits > ntile ? ntile : splits);
  const int64_t tps = (ntile + splits - 1) / splits;
  splits = (ntile + tps - 1) / tps;
  for (int64_t w = blockIdx.x; w < row_blocks * splits; w += gridDim.x) {
    const int64_t f0 = (w / splits) * FX_R;
    const int64_t t0 = (w % splits) * tps;
    const int64_t t1 = min64(ntile, t0 + tps);
    Acc bv[4];
    int64_t bj[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      bv[a] = (Acc)INFINITY;
      bj[a] = INT64_MAX;
    }
    for (int64_t tile = t0; tile < t1; ++tile) {
      const int64_t j0 = tile * FX_P;
      float acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
      for (int k0 = 0; k0 < d; k0 += FX_DK) {
        const int dk = d - k0 < FX_DK ? d - k0 : FX_DK;
        __syncthreads();
        for (int e = t; e < FX_R * dk; e += 256) {
          const int r = e / dk, c = e - r * dk;
          const int64_t f = f0 + r;
          const int64_t row = f < nf ? (rows ? (int64_t)rows[f] : f) : -1;
          xs[r * dp + c] = row >= 0 ? X[row * d + k0 + c] : 0.f;
        }
        for (int e = t; e < FX_P * dk; e += 256) {
          const int p = e / dk, c = e - p * dk;
          cs[p * dp + c] = (j0 + p < k) ? P[(j0 + p) * d + k0 + c] : 0.f;
        }
        __syncthreads();
        for (int i = 0; i < dk; ++i) {
          float xv[4], cv[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) xv[a] = xs[(rg * 4 + a) * dp + i];
#pragma unroll
          for (int b = 0; b < 4; ++b) cv[b] = cs[(pg * 4 + b) * dp + i];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const float df = xv[a] - cv[b];
              acc[a][b] = fmaf(df, df, acc[a][b]);
            }
        }
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int64_t j = j0 + pg * 4 + b;
        if (j < k) {
#pragma unroll
          for (int a = 0; a < 4; ++a)
            if (acc[a][b] < bv[a]) {  // j increases with (tile, b) for this thread: keeps lowest j
              bv[a] = acc[a][b];
              bj[a] = j;
            }
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int64_t f = f0 + rg * 4 + a;
      if (f < nf && bj[a] != INT64_MAX) {
        unsigned long long key;
        if constexpr (EXACT) {
          const unsigned long long m = (1ull << jbits) - 1ull;
          key = ((unsigned long long)__double_as_longlong((double)bv[a]) & ~m) | (unsigned long long)bj[a];
        } else {
          key = ((unsigned long long)__float_as_uint(fmaxf((float)bv[a], 0.f)) << 32) | (unsigned long long)(uint32_t)bj[a];
        }
        atomicMin(keys + f, key);
      }
    }
  }
}

__global__ void k_keys_init(const int32_t* __restrict__ count_dev, int64_t cap, unsigned long long* keys,
                            const int* __restrict__ active) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  const int64_t nf = count_dev ? min64(*count_dev, cap) : cap;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x)
    keys[f] = ~0ull;
}

// key formats: jbits == 0: (fp32 bits of d^2) << 32 | j;  jbits > 0 (exact re-check): the FP64
// d^2 bits with the low jbits replaced by j (order = d^2 to 2^-(52-jbits) relative, then j)
__global__ void k_keys_write(const int32_t* __restrict__ rows, const int32_t* __restrict__ count_dev, int64_t cap,
                             const unsigned long long* __restrict__ keys, int32_t* __restrict__ labels,
                             float* __restrict__ best, const int* __restrict__ active, int jbits) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  const int64_t nf = count_dev ? min64(*count_dev, cap) : cap;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = keys[f];
    const int64_t row = rows ? (int64_t)rows[f] : f;
    if (jbits == 0) {
      labels[row] = (int32_t)(key & 0xffffffffu);
      if (best) best[row] = __uint_as_float((uint32_t)(key >> 32));
    } else {
      const unsigned long long m = (1ull << jbits) - 1ull;
      labels[row] = (int32_t)(key & m);
      if (best) best[row] = (float)__longlong_as_double((long long)(key & ~m));
    }
  }
}

// Register-blocked exact argmin for d <= 256 (the K4 re-check at C3/C5 scale): a work item is
// 32 rows x a prototype range; the 32 rows stay in shared memory for the whole range, each
// 128-prototype tile is staged once, and a thread computes 4 rows x 4 prototypes with 16-byte
// shared-memory loads along the dimension (4 dims per load): direct FP32 (x - c)^2 sums in
// dimension order, the same arithmetic as the FP32 direct form of the oracle comparison.
constexpr int RB_R = 32, RB_P = 128;

// EXACT (the K4 full re-check): FP64 sums of separately rounded squares of the FP64 differences
// in dimension order (the oracle's arithmetic), key = FP64 d^2 with its low jbits replaced by j.
template <bool EXACT>
__global__ void __launch_bounds__(256) k_rb_argmin(const float* __restrict__ X, int d, int d4p,
                                                   const float* __restrict__ P, int64_t k,
                                                   const int32_t* __restrict__ rows,
                                                   const int32_t* __restrict__ count_dev, int64_t cap, int nsm,
                                                   unsigned long long* __restrict__ keys,
                                                   const int* __restrict__ active, int jbits) {
  using Acc = typename std::conditional<EXACT, double, float>::type;
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  extern __shared__ float4 rsm[];
  const int64_t nf = count_dev ? min64(*count_dev, cap) : cap;
  if (nf <= 0) return;
  // row stride d4p float4 (d/4 rounded up, +1 when even: conflict-free 16-byte column reads)
  float4* xs = rsm;                  // [RB_R][d4p]
  float4* cs = rsm + RB_R * d4p;     // [RB_P][d4p]
  const int t = threadIdx.x;
  const int rg = t & 7, pg = t >> 3;  // rows a*8+rg, prototypes b*32+pg (a, b < 4): interleaved so
                                      // the 16-byte smem reads of a warp hit distinct banks
  const int d4 = (d + 3) / 4;
  const bool vec = (d & 3) == 0 && ((uintptr_t)X & 15) == 0 && ((uintptr_t)P & 15) == 0;
  const int64_t row_blocks = (nf + RB_R - 1) / RB_R;
  const int64_t ntile = (k + RB_P - 1) / RB_P;
  // enough (row block, prototype range) items to fill every resident CTA (nsm = the grid)
  int64_t splits = ((int64_t)nsm + row_blocks - 1) / row_blocks;
  splits = splits < 1 ? 1 : (splits > ntile ? ntile : splits);
  const int64_t tps = (ntile + splits - 1) / splits;
  splits = (ntile + tps - 1) / tps;
  for (int64_t w = blockIdx.x; w < row_blocks * splits; w += gridDim.x) {
    const int64_t f0 = (w / splits) * RB_R;
    const int64_t t0 = (w % splits) * tps;
    const int64_t t1 = min64(ntile, t0 + tps);
    __syncthreads();
    for (int e = t; e < RB_R * d4; e += 256) {
      const int r = e / d4, c4 = e - r * d4;
      const int64_t f = f0 + r;
      const int64_t row = f < nf ? (rows ? (int64_t)rows[f] : f) : -1;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row >= 0) {
        const float* src = X + row * d + 4 * c4;
        if (vec) {
          v = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          v.x = src[0];
          if (4 * c4 + 1 < d) v.y = src[1];
          if (4 * c4 + 2 < d) v.z = src[2];
          if (4 * c4 + 3 < d) v.w = src[3];
        }
      }
      xs[r * d4p + c4] = v;
    }
    Acc bv[4];
    int64_t bj[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      bv[a] = (Acc)INFINITY;
      bj[a] = INT64_MAX;
    }
    for (int64_t tile = t0; tile < t1; ++tile) {
      const int64_t j0 = tile * RB_P;
      __syncthreads();
      for (int e = t; e < RB_P * d4; e += 256) {
        const int pr = e / d4, c4 = e - pr * d4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j0 + pr < k) {
          const float* src = P + (j0 + pr) * d + 4 * c4;
          if (vec) {
            v = __ldg(reinterpret_cast<const float4*>(src));
          } else {
            v.x = src[0];
            if (4 * c4 + 1 < d) v.y = src[1];
            if (4 * c4 + 2 < d) v.z = src[2];
            if (4 * c4 + 3 < d) v.w = src[3];
          }
        }
        cs[pr * d4p + c4] = v;
      }
      __syncthreads();
      Acc acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = (Acc)0;
      for (int c4 = 0; c4 < d4; ++c4) {
        float4 xv[4], cv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) xv[a] = xs[(a * 8 + rg) * d4p + c4];
#pragma unroll
        for (int b = 0; b < 4; ++b) cv[b] = cs[(b * 32 + pg) * d4p + c4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {  // dimensions in increasing order (zero padding adds 0)
            if constexpr (EXACT) {
              double df = (double)xv[a].x - (double)cv[b].x;
              acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(df, df));
              df = (double)xv[a].y - (double)cv[b].y;
              acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(df, df));
              df = (double)xv[a].z - (double)cv[b].z;
              acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(df, df));
              df = (double)xv[a].w - (double)cv[b].w;
              acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(df, df));
            } else {
              float df = xv[a].x - cv[b].x;
              acc[a][b] = fmaf(df, df, acc[a][b]);
              df = xv[a].y - cv[b].y;
              acc[a][b] = fmaf(df, df, acc[a][b]);
              df = xv[a].z - cv[b].z;
              acc[a][b] = fmaf(df, df, acc[a][b]);
              df = xv[a].w - cv[b].w;
              acc[a][b] = fmaf(df, df, acc[a][b]);
            }
          }
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int64_t j = j0 + b * 32 + pg;
        if (j < k) {
#pragma unroll
          for (int a = 0; a < 4; ++a)
            if (acc[a][b] < bv[a]) {  // j increases with (tile, b) for this thread: keeps lowest j
              bv[a] = acc[a][b];
              bj[a] = j;
            }
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int64_t f = f0 + a * 8 + rg;
      if (f < nf && bj[a] != INT64_MAX) {
        unsigned long long key;
        if constexpr (EXACT) {
          const unsigned long long m = (1ull << jbits) - 1ull;
          key = ((unsigned long long)__double_as_longlong((double)bv[a]) & ~m) | (unsigned long long)bj[a];
        } else {
          key = ((unsigned long long)__float_as_uint(fmaxf((float)bv[a], 0.f)) << 32) | (unsigned long long)(uint32_t)bj[a];
        }
        atomicMin(keys + f, key);
      }
    }
  }
}

// The exact re-check against FP64 prototypes, register-blocked like k_rb_argmin: 32 flagged rows
// (FP64 in shared memory) x 128-prototype FP64 tiles, 4 rows x 4 prototypes per thread, the
// oracle's arithmetic (FP64 difference, separately rounded square and sum, dimension order),
// double2 shared-memory reads (row stride d2p double2, odd: conflict-free), merged across the
// prototype splits with the exact 64-bit key (FP64 d^2 with the low jbits = j).
__global__ void __launch_bounds__(256) k_rb_argmin64(const float* __restrict__ X, int d, int d2p,
                                                     const double* __restrict__ P, int64_t k,
                                                     const int32_t* __restrict__ rows,
                                                     const int32_t* __restrict__ count_dev, int64_t cap, int nsm,
                                                     unsigned long long* __restrict__ keys,
                                                     const int* __restrict__ active, int jbits) {
  if (active && !*active) return;
  extern __shared__ double2 rsm64[];
  const int64_t nf = count_dev ? min64(*count_dev, cap) : cap;
  if (nf <= 0) return;
  double2* xs = rsm64;               // [RB_R][d2p]
  double2* cs = rsm64 + RB_R * d2p;  // [RB_P][d2p]
  const int t = threadIdx.x;
  const int rg = t & 7, pg = t >> 3;
  const int d2 = (d + 1) / 2;
  const int64_t row_blocks = (nf + RB_R - 1) / RB_R;
  const int64_t ntile = (k + RB_P - 1) / RB_P;
  int64_t splits = ((int64_t)nsm + row_blocks - 1) / row_blocks;
  splits = splits < 1 ? 1 : (splits > ntile ? ntile : splits);
  const int64_t tps = (ntile + splits - 1) / splits;
  splits = (ntile + tps - 1) / tps;
  const unsigned long long jm = (1ull << jbits) - 1ull;
  for (int64_t w = blockIdx.x; w < row_blocks * splits; w += gridDim.x) {
    const int64_t f0 = (w / splits) * RB_R;
    const int64_t t0 = (w % splits) * tps;
    const int64_t t1 = min64(ntile, t0 + tps);
    __syncthreads();
    for (int e = t; e < RB_R * d2; e += 256) {
      const int r = e / d2, c2 = e - r * d2;
      const int64_t f = f0 + r;
      const int64_t row = f < nf ? (rows ? (int64_t)rows[f] : f) : -1;
      double2 v = make_double2(0.0, 0.0);
      if (row >= 0) {
        const float* src = X + row * d + 2 * c2;
        v.x = (double)src[0];
        if (2 * c2 + 1 < d) v.y = (double)src[1];
      }
      xs[r * d2p + c2] = v;
    }
    double bv[4];
    int64_t bj[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      bv[a] = INFINITY;
      bj[a] = INT64_MAX;
    }
    for (int64_t tile = t0; tile < t1; ++tile) {
      const int64_t j0 = tile * RB_P;
      __syncthreads();
      for (int e = t; e < RB_P * d2; e += 256) {
        const int pr = e / d2, c2 = e - pr * d2;
        double2 v = make_double2(0.0, 0.0);
        if (j0 + pr < k) {
          const double* src = P + (j0 + pr) * d + 2 * c2;
          v.x = src[0];
          if (2 * c2 + 1 < d) v.y = src[1];
        }
        cs[pr * d2p + c2] = v;
      }
      __syncthreads();
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
      for (int c2 = 0; c2 < d2; ++c2) {
        double2 xv[4], cv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) xv[a] = xs[(a * 8 + rg) * d2p + c2];
#pragma unroll
        for (int b = 0; b < 4; ++b) cv[b] = cs[(b * 32 + pg) * d2p + c2];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {  // dimensions in increasing order (zero padding adds 0)
            double df = xv[a].x - cv[b].x;
            acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(df, df));
            df = xv[a].y - cv[b].y;
            acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(df, df));
          }
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int64_t j = j0 + b * 32 + pg;
        if (j < k) {
#pragma unroll
          for (int a = 0; a < 4; ++a)
            if (acc[a][b] < bv[a]) {
              bv[a] = acc[a][b];
              bj[a] = j;
            }
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int64_t f = f0 + a * 8 + rg;
      if (f < nf && bj[a] != INT64_MAX)
        atomicMin(keys + f, ((unsigned long long)__double_as_longlong(bv[a]) & ~jm) | (unsigned long long)bj[a]);
    }
  }
}

static void launch_blocked(const float* X, int d, const float* P, int64_t k, const int32_t* rows,
                           const int32_t* count_dev, int64_t cap, unsigned long long* keys_ws, int32_t* labels,
                           float* best, cudaStream_t st, const int* active, bool exact = false) {
  k_keys_init<<<num_sms() * 2, 256, 0, st>>>(count_dev, cap, keys_ws, active);
  MASK_LAUNCH_CHECK();
  const int d4 = (d + 3) / 4;
  const int d4p = d4 | 1;  // odd float4 stride
  const size_t rb_smem = (size_t)(RB_R + RB_P) * d4p * sizeof(float4);
  int jbits = 0;  // exact keys: bits of j (the rest of the 64-bit key orders the FP64 d^2)
  if (exact)
    while ((int64_t(1) << jbits) < k) ++jbits;
  if (exact && jbits == 0) jbits = 1;
  const auto kern = exact ? k_rb_argmin<true> : k_rb_argmin<false>;
  if (d <= 256 && rb_smem <= 200 * 1024) {
    static int attr_for[2] = {-1, -1};
    if (rb_smem > 48 * 1024 && attr_for[exact] < (int)rb_smem) {
      MASK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr_for[exact] = 200 * 1024;
    }
    // one wave of resident CTAs (the flagged count is only known on the device: small counts
    // split the prototypes finely so every CTA gets one short item)
    static std::map<std::pair<size_t, bool>, int> occ_cache;
    int occ = 0;
    {
      static std::mutex mu;
      std::lock_guard<std::mutex> lock(mu);
      auto it = occ_cache.find({rb_smem, exact});
      if (it == occ_cache.end()) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, rb_smem) != cudaSuccess) occ = 2;
        (void)cudaGetLastError();
        it = occ_cache.emplace(std::make_pair(rb_smem, exact), std::max(1, std::min(occ, 8))).first;
      }
      occ = it->second;
    }
    const int grid = num_sms() * occ;
    kern<<<grid, 256, rb_smem, st>>>(X, d, d4p, P, k, rows, count_dev, cap, grid, keys_ws, active, jbits);
  } else {
    jbits = 0;  // (the plain blocked kernel keeps FP32 keys)
    k_blocked_argmin<<<num_sms() * 4, 256, 0, st>>>(X, d, P, k, rows, count_dev, cap, num_sms(), keys_ws, active);
  }
  MASK_LAUNCH_CHECK();
  k_keys_write<<<num_sms() * 2, 256, 0, st>>>(rows, count_dev, cap, keys_ws, labels, best, active, jbits);
  MASK_LAUNCH_CHECK();
}

// Two-candidate re-check: the exact decision between the only two prototypes a flagged row can
// take (K4): FP64 direct sums of squares in dimension order (separately rounded
// products and sums, as the oracle's FP64 loop), smaller distance, then lower index (D4).
// Rows without a pair are appended to the full re-check list.
template <class T>
__global__ void k_fix_pairs(const float* __restrict__ X, int d, const T* __restrict__ P,
                            const int32_t* __restrict__ flag_rows, const int2* __restrict__ flag_pair,
                            const int32_t* __restrict__ flag_count, int64_t cap, int32_t* __restrict__ labels,
                            float* __restrict__ best, int32_t* __restrict__ rescan_rows,
                            int32_t* __restrict__ rescan_count, const int* __restrict__ active) {
  if (active && !*active) return;
  const int64_t nf = min64(*flag_count, cap);
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
    const int32_t row = flag_rows[f];
    const int2 jp = flag_pair[f];
    if (jp.y < 0) {
      rescan_rows[atomicAdd(rescan_count, 1)] = row;
      continue;
    }
    const float* x = X + (int64_t)row * d;
    const T* c1 = P + (int64_t)jp.x * d;
    const T* c2 = P + (int64_t)jp.y * d;
    double s1 = 0.0, s2 = 0.0;
    for (int i = 0; i < d; ++i) {
      const double xi = (double)x[i];
      const double t1 = xi - (double)c1[i], t2 = xi - (double)c2[i];
      s1 = __dadd_rn(s1, __dmul_rn(t1, t1));
      s2 = __dadd_rn(s2, __dmul_rn(t2, t2));
    }
    const bool first = s1 < s2 || (s1 == s2 && jp.x < jp.y);
    labels[row] = first ? jp.x : jp.y;
    best[row] = (float)(first ? s1 : s2);
  }
}

// P64T[i * k + j] = P64[j * d + i] (dimension-major copy for the re-scan's coalesced reads)
__global__ void k_transpose64(const double* __restrict__ P, int64_t k, int d, double* __restrict__ PT,
                              const int* __restrict__ active) {
  if (active && !*active) return;
  const int64_t total = k * (int64_t)d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / k, j = e - i * k;
    PT[e] = P[j * d + i];
  }
}

// Exact full re-check of one flagged row per block against the FP64 prototypes: the oracle's
// distance arithmetic (sequential in the dimension) for every prototype, thread per prototype
// reading the dimension-major copy (coalesced), (d^2, j) minimum over the block.
__global__ void __launch_bounds__(256) k_rescan64(const float* __restrict__ X, int d, const double* __restrict__ PT,
                                                  int64_t k, const int32_t* __restrict__ rows,
                                                  const int32_t* __restrict__ count, int32_t* __restrict__ labels,
                                                  float* __restrict__ best, const int* __restrict__ active) {
  if (active && !*active) return;
  __shared__ double sd[8];
  __shared__ int64_t sj[8];
  extern __shared__ double sx[];  // the row, FP64
  const int64_t nf = *count;
  for (int64_t f = blockIdx.x; f < nf; f += gridDim.x) {
    const int32_t row = rows[f];
    for (int i = threadIdx.x; i < d; i += blockDim.x) sx[i] = (double)X[(int64_t)row * d + i];
    __syncthreads();
    double bd = INFINITY;
    int64_t bj = INT64_MAX;
    for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {  // j increasing per thread: keeps lowest
      double s = 0.0;
      for (int i = 0; i < d; ++i) {
        const double t = sx[i] - PT[(int64_t)i * k + j];
        s = __dadd_rn(s, __dmul_rn(t, t));
      }
      if (s < bd) {
        bd = s;
        bj = j;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, o);
      const int64_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (od < bd || (od == bd && oj < bj)) {
        bd = od;
        bj = oj;
      }
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
      sd[w] = bd;
      sj[w] = bj;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int u = 1; u < (int)(blockDim.x >> 5); ++u)
        if (sd[u] < bd || (sd[u] == bd && sj[u] < bj)) {
          bd = sd[u];
          bj = sj[u];
        }
      labels[row] = (int32_t)bj;
      best[row] = (float)bd;
    }
    __syncthreads();
  }
}

void launch_fixup_device(const float* X, int d, const float* P, int64_t k, const int32_t* flag_rows,
                         const int32_t* flag_count, int64_t cap, unsigned long long* keys_ws, int32_t* labels,
                         float* best, cudaStream_t st, const int* active, const int2* flag_pair,
                         int32_t* rescan_rows, int32_t* rescan_count, const double* P64, double* P64T) {
  if (!flag_pair) {
    launch_blocked(X, d, P, k, flag_rows, flag_count, cap, keys_ws, labels, best, st, active);
    return;
  }
  MASK_CUDA(cudaMemsetAsync(rescan_count, 0, sizeof(int32_t), st));
  if (P64)
    k_fix_pairs<double><<<num_sms() * 4, 256, 0, st>>>(X, d, P64, flag_rows, flag_pair, flag_count, cap, labels, best,
                                                       rescan_rows, rescan_count, active);
  else
    k_fix_pairs<float><<<num_sms() * 4, 256, 0, st>>>(X, d, P, flag_rows, flag_pair, flag_count, cap, labels, best,
                                                      rescan_rows, rescan_count, active);
  MASK_LAUNCH_CHECK();
  static const bool dbg = getenv("MASK_DEBUG_FIXUP") != nullptr;
  if (dbg) {  // development: flagged / re-scanned counts and the first pairs
    int32_t hc[2] = {0, 0};
    cudaMemcpyAsync(hc, flag_count, 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(hc + 1, rescan_count, 4, cudaMemcpyDeviceToHost, st);
    int2 hp[8];
    int32_t hr[8];
    cudaMemcpyAsync(hp, flag_pair, sizeof(hp), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(hr, flag_rows, sizeof(hr), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "[fixup] flagged %d rescan %d |", hc[0], hc[1]);
    for (int i = 0; i < 8 && i < hc[0]; ++i) fprintf(stderr, " %d:(%d,%d)", hr[i], hp[i].x, hp[i].y);
    fprintf(stderr, "\n");
  }
  if (P64) {  // the level's FP64 prototypes: the re-scan reads them (oracle arithmetic)
    const int d2 = (d + 1) / 2;
    const int d2p = d2 | 1;
    const size_t smem = (size_t)(RB_R + RB_P) * d2p * sizeof(double2);
    if (smem <= 200 * 1024) {  // register-blocked: 32 rows share every staged prototype tile
      int jbits = 1;
      while ((int64_t(1) << jbits) < k) ++jbits;
      static int attr = 0;
      if (smem > 48 * 1024 && !attr) {
        MASK_CUDA(cudaFuncSetAttribute(k_rb_argmin64, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = 1;
      }
      int occ = 1;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rb_argmin64, 256, smem) != cudaSuccess) occ = 1;
      (void)cudaGetLastError();
      const int grid = num_sms() * std::max(1, std::min(occ, 8));
      k_keys_init<<<num_sms() * 2, 256, 0, st>>>(rescan_count, cap, keys_ws, active);
      MASK_LAUNCH_CHECK();
      k_rb_argmin64<<<grid, 256, smem, st>>>(X, d, d2p, P64, k, rescan_rows, rescan_count, cap, grid, keys_ws, active,
                                             jbits);
      MASK_LAUNCH_CHECK();
      k_keys_write<<<num_sms() * 2, 256, 0, st>>>(rescan_rows, rescan_count, cap, keys_ws, labels, best, active,
                                                  jbits);
      MASK_LAUNCH_CHECK();
      return;
    }
    MASK_REQUIRE(P64T != nullptr, MASK_ERR_CUDA, "fix-up: no FP64 transpose workspace");
    k_transpose64<<<grid_for(k * d, 256), 256, 0, st>>>(P64, k, d, P64T, active);
    MASK_LAUNCH_CHECK();
    k_rescan64<<<num_sms() * 4, 256, (size_t)d * sizeof(double), st>>>(X, d, P64T, k, rescan_rows, rescan_count,
                                                                        labels, best, active);
    MASK_LAUNCH_CHECK();
    return;
  }
  launch_blocked(X, d, P, k, rescan_rows, rescan_count, cap, keys_ws, labels, best, st, active, /*exact=*/true);
}

void launch_assign_blocked(const float* X, int64_t n, int d, const float* P, int64_t k, unsigned long long* keys_ws,
                           int32_t* labels, float* best, cudaStream_t st, const int* active) {
  if (n <= 0) return;
  launch_blocked(X, d, P, k, nullptr, nullptr, n, keys_ws, labels, best, st, active);
}

// ====================================================================== operand prep
__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// One warp per prototype: Pb = tf32(-2c), Ps = tf32(-2c - Pb) (3xTF32 split of the B operand,
// the factor -2 is exact), cn2 = ||c||^2 accumulated in FP64 then rounded.
template <class T>
__global__ void k_prep_protos(const T* __restrict__ P, int64_t k, int64_t k_rows, int d, int kc, int fold,
                              float* __restrict__ Pb, float* __restrict__ Ps, float* __restrict__ cn2,
                              const int* __restrict__ active, int32_t* __restrict__ flag_count) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  if (flag_count && blockIdx.x == 0 && threadIdx.x == 0) *flag_count = 0;  // K1's near-tie list
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < k; j += warps) {
    double s = 0.0;
    for (int i = lane; i < d; i += 32) {
      const T c = P[j * d + i];
      s += (double)c * (double)c;
      // -2c split into two TF32 parts (from the FP64 prototype when the level keeps one: the
      // split then represents the FP64 value, not its fp32 rounding)
      const double m2 = -2.0 * (double)c;
      const float b = tf32_rn((float)m2);
      const float r = tf32_rn((float)(m2 - (double)b));
      if (Pb) Pb[j * kc + i] = b;
      if (Ps) Ps[j * kc + i] = r;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0 && cn2) cn2[j] = (float)s;
    if (Pb && kc > d) {
      // columns beyond d: zeros, except with `fold` the K step F = d rounded up to 8 of the big part:
      // [F] = ||c||^2 big, [F+1] = ||c||^2 small (A side: 1, 1), [F+2] = [F+3] = 1 (A side:
      // ||x||^2 big, small)
      const float hb = tf32_rn((float)s);
      const float hs = tf32_rn((float)(s - (double)hb));
      const int F = (d + 7) / 8 * 8;
      for (int i = d + lane; i < kc; i += 32) {
        float v = 0.f;
        if (fold && i >= F) v = i == F ? hb : (i == F + 1 ? hs : (i <= F + 3 ? 1.0f : 0.f));
        Pb[j * kc + i] = v;
        Ps[j * kc + i] = 0.f;
      }
    }
  }
  // pad rows [k, k_rows): never the nearest (folded: a huge ||c||^2; else ||c||^2 = +inf in cn2)
  if (Pb) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (k_rows - k) * kc;
         e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t j = k + e / kc;
      const int i = (int)(e % kc);
      Pb[j * kc + i] = (fold && i == (d + 7) / 8 * 8) ? 1e30f : 0.f;
      Ps[j * kc + i] = 0.f;
    }
  }
}

void launch_prep_protos(const float* P, int64_t k, int d, int kc, float* Pb, float* Ps, float* cn2,
                        cudaStream_t st, int64_t k_rows, int fold, const int* active, int32_t* flag_count,
                        const double* P64) {
  if (k_rows < k) k_rows = k;
  if (P64)
    k_prep_protos<double><<<grid_for(k * 32, 256), 256, 0, st>>>(P64, k, k_rows, d, kc, fold, Pb, Ps, cn2, active,
                                                                  flag_count);
  else
    k_prep_protos<float><<<grid_for(k * 32, 256), 256, 0, st>>>(P, k, k_rows, d, kc, fold, Pb, Ps, cn2, active,
                                                                 flag_count);
  MASK_LAUNCH_CHECK();
}

void launch_level_norms(const float* P, int64_t k, int d, float* cn2, cudaStream_t st, const int* active) {
  launch_prep_protos(P, k, d, d, nullptr, nullptr, cn2, st, k, 0, active, nullptr);
}

__global__ void k_row_norms(const float* __restrict__ X, int64_t n, int d, float* __restrict__ xn2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  const float* x = X + i * d;
  for (int c = 0; c < d; ++c) {
    double v = x[c];
    s += v * v;
  }
  xn2[i] = (float)s;
}

void launch_row_norms(const float* X, int64_t n, int d, float* xn2, cudaStream_t st) {
  if (n <= 0) return;
  k_row_norms<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(X, n, d, xn2);
  MASK_LAUNCH_CHECK();
}

// ====================================================================== K5 dense update
// Element-parallel: thread e covers X[e] (coalesced reads), scatters into S[label*d + col]
// with L2 float atomics (red.global.add); the col == 0 thread counts the row.
// Rows with d % 4 == 0 use one 16-byte vector red per 4 columns.
__global__ void k_update_dense_v4(const float4* __restrict__ X4, int64_t n, int d4,
                                  const int32_t* __restrict__ labels, float* __restrict__ S,
                                  int32_t* __restrict__ counts, const int* __restrict__ active) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  const int64_t total = n * (int64_t)d4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t row = e / d4;
    const int c4 = (int)(e - row * d4);
    const int32_t j = __ldg(labels + row);
    float4 v = __ldg(X4 + e);
    float* dst = S + ((int64_t)j * d4 + c4) * 4;
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
    if (c4 == 0) atomicAdd(counts + j, 1);
  }
}

__global__ void k_update_dense(const float* __restrict__ X, int64_t n, int d,
                               const int32_t* __restrict__ labels, float* __restrict__ S,
                               int32_t* __restrict__ counts, const int* __restrict__ active) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  const int64_t total = n * (int64_t)d;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t row = e / d;
    const int c = (int)(e - row * d);
    const int32_t j = __ldg(labels + row);
    atomicAdd(S + (int64_t)j * d + c, __ldg(X + e));
    if (c == 0) atomicAdd(counts + j, 1);
  }
}

// Rows visited in label-sorted order (perm from launch_label_sort of these labels, or of the
// previous pass's: runs are then long but not perfect).  Each warp walks CH consecutive
// positions; a row is covered by L = pow2 >= d/4 lanes (one float4 each), R = 32/L rows per
// step.  Every lane group accumulates its run of equal labels in registers and flushes it with
// one red.global.add.v4 per float4 when the label changes: a run of m rows costs d/4 vector
// reds instead of m*d/4 (atomics were the limit of the element-parallel kernel).
// Acc = double (the FP64 sums of a level that keeps FP64 prototypes): the run is accumulated
// in FP64 and flushed with four scalar FP64 reds.
// NB batches of U rows per lane group and warp: FP64 sums flush with four scalar atomics, so
// their warps cover 4x longer stretches of the sorted order (fewer run flushes per cluster).
template <int L, class Acc = float>
__global__ void __launch_bounds__(256) k_update_runs(const float4* __restrict__ X4, const int32_t* __restrict__ perm,
                                                      int64_t n, int d4, const int32_t* __restrict__ labels,
                                                      Acc* __restrict__ S, int32_t* __restrict__ counts,
                                                      const int* __restrict__ active) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  constexpr int NB = sizeof(Acc) == 8 ? 16 : 4;
  constexpr int R = 32 / L, U = 4, CH = R * U * NB;  // NB batches of U independent rows per lane group
  const int lane = threadIdx.x & 31, slot = lane / L, c4 = lane % L;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t p0 = w * CH;
  if (p0 >= n) return;
  const int64_t p1 = p0 + CH < n ? p0 + CH : n;
  struct A4 {
    Acc x, y, z, w;
  } acc{0, 0, 0, 0};
  int32_t cur = -1, cnt = 0;
  auto flush = [&]() {
    if (c4 < d4) {
      Acc* dst = S + ((int64_t)cur * d4 + c4) * 4;
      if constexpr (sizeof(Acc) == 4) {
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"((float)acc.x), "f"((float)acc.y),
                     "f"((float)acc.z), "f"((float)acc.w)
                     : "memory");
      } else {
        atomicAdd(dst + 0, acc.x);
        atomicAdd(dst + 1, acc.y);
        atomicAdd(dst + 2, acc.z);
        atomicAdd(dst + 3, acc.w);
      }
    }
    if (c4 == 0) atomicAdd(counts + cur, cnt);
  };
  for (int64_t pb = p0 + slot; pb < p1; pb += R * U) {
    // U independent rows in flight per lane group (perm -> label, row -> x) before reducing
    int64_t row[U];
    int32_t lab[U];
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = pb + (int64_t)u * R;
      row[u] = p < p1 ? (perm ? (int64_t)__ldg(perm + p) : p) : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      lab[u] = row[u] >= 0 ? __ldg(labels + row[u]) : -1;
      v[u] = (row[u] >= 0 && c4 < d4) ? __ldg(X4 + row[u] * d4 + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (lab[u] < 0) continue;
      if (lab[u] != cur) {
        if (cur >= 0) flush();
        cur = lab[u];
        acc = A4{0, 0, 0, 0};
        cnt = 0;
      }
      acc.x += (Acc)v[u].x;
      acc.y += (Acc)v[u].y;
      acc.z += (Acc)v[u].z;
      acc.w += (Acc)v[u].w;
      ++cnt;
    }
  }
  if (cur >= 0) flush();
}

// FP64 sums (a level that keeps FP64 prototypes): run kernel over the label-sorted rows, or one
// FP64 atomic per element without a sort
__global__ void k_update_dense64(const float* __restrict__ X, int64_t n, int d, const int32_t* __restrict__ labels,
                                 double* __restrict__ S, int32_t* __restrict__ counts, const int* __restrict__ active) {
  if (active && !*active) return;
  const int64_t total = n * (int64_t)d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / d;
    const int c = (int)(e - i * d);
    const int32_t j = labels[i];
    atomicAdd(S + (int64_t)j * d + c, (double)X[e]);
    if (c == 0) atomicAdd(counts + j, 1);
  }
}

void launch_update_dense64(const float* X, int64_t n, int d, const int32_t* labels, double* S, int32_t* counts,
                           cudaStream_t st, const int* active, const int32_t* perm) {
  if (n <= 0) return;
  if (perm && d % 4 == 0 && d <= 128 && ((uintptr_t)X % 16) == 0) {
    const int d4 = d / 4;
    const int L = d4 <= 1 ? 1 : d4 <= 2 ? 2 : d4 <= 4 ? 4 : d4 <= 8 ? 8 : d4 <= 16 ? 16 : 32;
    const int64_t ch = (32 / L) * 64;  // positions per warp (k_update_runs CH with NB = 16)
    const int64_t warps = (n + ch - 1) / ch;
    const unsigned grid = (unsigned)((warps + 7) / 8);
    const float4* X4 = reinterpret_cast<const float4*>(X);
    if (d4 <= 1) k_update_runs<1, double><<<grid, 256, 0, st>>>(X4, perm, n, d4, labels, S, counts, active);
    else if (d4 <= 2) k_update_runs<2, double><<<grid, 256, 0, st>>>(X4, perm, n, d4, labels, S, counts, active);
    else if (d4 <= 4) k_update_runs<4, double><<<grid, 256, 0, st>>>(X4, perm, n, d4, labels, S, counts, active);
    else if (d4 <= 8) k_update_runs<8, double><<<grid, 256, 0, st>>>(X4, perm, n, d4, labels, S, counts, active);
    else if (d4 <= 16) k_update_runs<16, double><<<grid, 256, 0, st>>>(X4, perm, n, d4, labels, S, counts, active);
    else k_update_runs<32, double><<<grid, 256, 0, st>>>(X4, perm, n, d4, labels, S, counts, active);
  } else {
    k_update_dense64<<<grid_for(n * d, 256, (int64_t)num_sms() * 16), 256, 0, st>>>(X, n, d, labels, S, counts,
                                                                                   active);
  }
  MASK_LAUNCH_CHECK();
}

// FP64 sums over the label-sorted rows (perm; end[j] = the sort's end offset of label j), cut
// into fixed chunks of kSeg64 positions, one warp per chunk: for every cluster piece in its
// chunk the warp accumulates the rows in FP64 registers (L lanes per row, one float4 each, R =
// 32/L rows per step, U rows in flight per lane group), combines its R row groups with
// shuffles, and flushes -- a cluster wholly inside the chunk with plain stores of S_j and n_j,
// a piece of a cluster cut by a chunk boundary with FP64 atomics (S and counts arrive zeroed).
// Chunks keep a huge cluster spread over many warps; most clusters need no atomics.
constexpr int kSeg64 = 128;  // (measured: 64 / 128 / 256 / 512 rows: C3 0.53 / 0.54 / 0.58 / 0.64 ms, C2 23 / 21 / 31 / 49 us per pass)
template <int L>
__global__ void __launch_bounds__(256) k_update_seg64(const float4* __restrict__ X4, const int32_t* __restrict__ perm,
                                                       const int32_t* __restrict__ labels,
                                                       const int32_t* __restrict__ end, int64_t n, int d4,
                                                       double* __restrict__ S, int32_t* __restrict__ counts,
                                                       const int* __restrict__ active) {
  if (active && !*active) return;
  constexpr int R = 32 / L, U = 4;
  const int lane = threadIdx.x & 31, slot = lane / L, c4 = lane % L;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t nchunks = (n + kSeg64 - 1) / kSeg64;
  for (int64_t ch = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); ch < nchunks; ch += warps) {
    const int32_t q0 = (int32_t)(ch * kSeg64), q1 = (int32_t)min64(n, (ch + 1) * kSeg64);
    int32_t j = __ldg(labels + __ldg(perm + q0));
    for (int32_t a = q0; a < q1;) {
      const int32_t cs = j ? __ldg(end + j - 1) : 0, ce = __ldg(end + j);
      const int32_t b = ce < q1 ? ce : q1;  // this piece: positions [a, b)
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      for (int32_t p = a + slot; p < b; p += R * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int32_t q = p + u * R;
          v[u] = (q < b && c4 < d4) ? __ldg(X4 + (int64_t)__ldg(perm + q) * d4 + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          a0 += (double)v[u].x;
          a1 += (double)v[u].y;
          a2 += (double)v[u].z;
          a3 += (double)v[u].w;
        }
      }
#pragma unroll
      for (int o = L; o < 32; o <<= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
        a3 += __shfl_xor_sync(0xffffffffu, a3, o);
      }
      const bool whole = a == cs && b == ce;
      if (slot == 0 && c4 < d4) {
        double* dst = S + ((int64_t)j * d4 + c4) * 4;
        if (whole) {
          dst[0] = a0;
          dst[1] = a1;
          dst[2] = a2;
          dst[3] = a3;
        } else {
          atomicAdd(dst + 0, a0);
          atomicAdd(dst + 1, a1);
          atomicAdd(dst + 2, a2);
          atomicAdd(dst + 3, a3);
        }
      }
      if (lane == 0) {
        if (whole) counts[j] = b - a;
        else atomicAdd(counts + j, b - a);
      }
      a = b;
      if (a < q1) j = __ldg(labels + __ldg(perm + a));  // (empty clusters have no positions)
    }
  }
}

bool update_seg64_supported(int d) { return d % 4 == 0 && d <= 128; }

void launch_update_seg64(const float* X, int d, const int32_t* perm, const int32_t* labels, const int32_t* end,
                         int64_t n, double* S, int32_t* counts, cudaStream_t st, const int* active) {
  if (n <= 0) return;
  const int d4 = d / 4;
  const int L = d4 <= 1 ? 1 : d4 <= 2 ? 2 : d4 <= 4 ? 4 : d4 <= 8 ? 8 : d4 <= 16 ? 16 : 32;
  const int64_t nchunks = (n + kSeg64 - 1) / kSeg64;
  const unsigned grid = grid_for(nchunks * 32, 256, (int64_t)num_sms() * 16);
  const float4* X4 = reinterpret_cast<const float4*>(X);
  if (L == 1) k_update_seg64<1><<<grid, 256, 0, st>>>(X4, perm, labels, end, n, d4, S, counts, active);
  else if (L == 2) k_update_seg64<2><<<grid, 256, 0, st>>>(X4, perm, labels, end, n, d4, S, counts, active);
  else if (L == 4) k_update_seg64<4><<<grid, 256, 0, st>>>(X4, perm, labels, end, n, d4, S, counts, active);
  else if (L == 8) k_update_seg64<8><<<grid, 256, 0, st>>>(X4, perm, labels, end, n, d4, S, counts, active);
  else if (L == 16) k_update_seg64<16><<<grid, 256, 0, st>>>(X4, perm, labels, end, n, d4, S, counts, active);
  else k_update_seg64<32><<<grid, 256, 0, st>>>(X4, perm, labels, end, n, d4, S, counts, active);
  MASK_LAUNCH_CHECK();
}

// K7 for FP64 sums: P64_j = S_j / n_j in FP64 (the oracle's "sum, then one division"), P_j its
// fp32 rounding; empty clusters keep both (D5); displacement in FP64; S and counts zeroed.
__global__ void k_finalize64(double* __restrict__ P64, float* __restrict__ P, double* __restrict__ S,
                             int32_t* __restrict__ counts, int64_t k, int d, uint32_t* __restrict__ stat,
                             const int* __restrict__ active, LoopCtl lc);

void launch_update_dense(const float* X, int64_t n, int d, const int32_t* labels, int64_t k,
                         float* S, int32_t* counts, cudaStream_t st, const int* active, const int32_t* perm) {
  (void)k;
  if (n <= 0) return;
  if (perm && d % 4 == 0 && d <= 128 && ((uintptr_t)X % 16) == 0) {
    const int d4 = d / 4;
    const int L = d4 <= 1 ? 1 : d4 <= 2 ? 2 : d4 <= 4 ? 4 : d4 <= 8 ? 8 : d4 <= 16 ? 16 : 32;
    const int64_t ch = (32 / L) * 16;  // positions per warp (k_update_runs CH)
    const int64_t warps = (n + ch - 1) / ch;
    const unsigned grid = (unsigned)((warps + 7) / 8);
    const float4* X4 = reinterpret_cast<const float4*>(X);
    if (d4 <= 1) k_update_runs<1><<<grid, 256, 0, st>>>(X4, perm, n, d4, labels, S, counts, active);
    else if (d4 <= 2) k_update_runs<2><<<grid, 256, 0, st>>>(X4, perm, n, d4, labels, S, counts, active);
    else if (d4 <= 4) k_update_runs<4><<<grid, 256, 0, st>>>(X4, perm, n, d4, labels, S, counts, active);
    else if (d4 <= 8) k_update_runs<8><<<grid, 256, 0, st>>>(X4, perm, n, d4, labels, S, counts, active);
    else if (d4 <= 16) k_update_runs<16><<<grid, 256, 0, st>>>(X4, perm, n, d4, labels, S, counts, active);
    else k_update_runs<32><<<grid, 256, 0, st>>>(X4, perm, n, d4, labels, S, counts, active);
  } else if (d % 4 == 0 && ((uintptr_t)X % 16) == 0) {
    const int d4 = d / 4;
    k_update_dense_v4<<<grid_for(n * d4, 256, (int64_t)num_sms() * 16), 256, 0, st>>>(
        reinterpret_cast<const float4*>(X), n, d4, labels, S, counts, active);
  } else {
    k_update_dense<<<grid_for(n * d, 256, (int64_t)num_sms() * 16), 256, 0, st>>>(X, n, d, labels,
                                                                                 S, counts, active);
  }
  MASK_LAUNCH_CHECK();
}

// ====================================================================== K6 CSR update
// Warp per row: lanes over the row's non-zeros scatter into S[label*d + col].
__global__ void k_update_csr(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const float* __restrict__ val, int64_t n, int d,
                             const int32_t* __restrict__ labels, float* __restrict__ S,
                             int32_t* __restrict__ counts, const int* __restrict__ active) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const int32_t j = labels[r];
    float* Sj = S + (int64_t)j * d;
    for (int64_t p = rp[r] + lane; p < rp[r + 1]; p += 32) atomicAdd(Sj + col[p], val[p]);
    if (lane == 0) atomicAdd(counts + j, 1);
  }
}

void launch_update_csr(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t n,
                       int d, const int32_t* labels, float* S, int32_t* counts, cudaStream_t st,
                       const int* active) {
  if (n <= 0) return;
  k_update_csr<<<grid_for(n * 32, 256, (int64_t)num_sms() * 16), 256, 0, st>>>(row_ptr, col, val,
                                                                              n, d, labels, S,
                                                                              counts, active);
  MASK_LAUNCH_CHECK();
}

// K6 over label-sorted rows.  The sorted row order (perm) is cut into segments of kSegRows
// positions; a CTA takes a segment and, for every cluster j present in it (rows perm[start ..
// stop) with label j), accumulates those rows into a dense d-float shared-memory row with
// shared atomics, then flushes it: a cluster wholly inside the segment is written to S_j with
// plain coalesced stores (n_j = its row count), a cluster cut by a segment boundary adds its
// non-zero entries with global atomics.  No k x d atomics sweep, S is written about once per
// pass, and a huge cluster is spread over many CTAs.  S and the counts arrive zeroed
// (previous finalize / level start).  end[j] = the label sort's scatter cursor = end offset of
// label j in perm.
constexpr int kSegRows = 256;

__global__ void __launch_bounds__(256) k_update_csr_sorted(const int64_t* __restrict__ rp,
                                                           const int32_t* __restrict__ col,
                                                           const float* __restrict__ val, int d,
                                                           const int32_t* __restrict__ perm,
                                                           const int32_t* __restrict__ labels,
                                                           const int32_t* __restrict__ end, int64_t n, int64_t k,
                                                           float* __restrict__ S, int32_t* __restrict__ counts,
                                                           const int* __restrict__ active) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  extern __shared__ __align__(16) float acc[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool vec = (d & 3) == 0;
  const int64_t nseg = (n + kSegRows - 1) / kSegRows;
  // acc is zeroed once here; every write-out below leaves it zeroed for the next piece
  for (int c = threadIdx.x; c < d; c += blockDim.x) acc[c] = 0.f;
  __syncthreads();
  for (int64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
    const int32_t q0 = (int32_t)(sg * kSegRows), q1 = (int32_t)min64(n, (sg + 1) * kSegRows);
    const int32_t j0 = labels[perm[q0]], j1 = labels[perm[q1 - 1]];
    for (int32_t j = j0; j <= j1; ++j) {
      const int32_t cs = j ? end[j - 1] : 0, ce = end[j];
      const int32_t a = cs > q0 ? cs : q0, b = ce < q1 ? ce : q1;
      if (b <= a) continue;  // empty cluster (uniform across the CTA)
      // a warp takes 4 rows at a time and issues all their loads (2 non-zeros per lane and
      // row) before the shared atomics: perm -> row_ptr -> (col, val) is a latency chain
      constexpr int RW = 4;
      for (int32_t qa = a + w * RW; qa < b; qa += nw * RW) {
        int64_t r0 = 0, r1 = 0;
        if (lane < RW && qa + lane < b) {
          const int64_t r = perm[qa + lane];
          r0 = rp[r];
          r1 = rp[r + 1];
        }
        int32_t cq[RW][2];
        float vq[RW][2];
#pragma unroll
        for (int u = 0; u < RW; ++u) {
          const int64_t s0 = __shfl_sync(0xffffffffu, r0, u), s1 = __shfl_sync(0xffffffffu, r1, u);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t pp = s0 + h * 32 + lane;
            cq[u][h] = pp < s1 ? __ldg(col + pp) : -1;
            vq[u][h] = pp < s1 ? __ldg(val + pp) : 0.f;
          }
        }
#pragma unroll
        for (int u = 0; u < RW; ++u) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (cq[u][h] >= 0) atomicAdd(acc + cq[u][h], vq[u][h]);
          const int64_t s0 = __shfl_sync(0xffffffffu, r0, u), s1 = __shfl_sync(0xffffffffu, r1, u);
          for (int64_t pp = s0 + 64 + lane; pp < s1; pp += 32) atomicAdd(acc + __ldg(col + pp), __ldg(val + pp));
        }
      }
      __syncthreads();
      float* Sj = S + (int64_t)j * d;
      // S is zero on entry (zeroed at the level start and by K7 after every pass), so only the
      // non-zero parts of the piece are written; the read also re-zeroes acc for the next piece
      if (a == cs && b == ce) {  // the whole cluster: plain stores of the non-zero float4s
        if (vec) {
          for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
            const float4 v = reinterpret_cast<const float4*>(acc)[c];
            reinterpret_cast<float4*>(acc)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f) reinterpret_cast<float4*>(Sj)[c] = v;
          }
        } else {
          for (int c = threadIdx.x; c < d; c += blockDim.x) {
            const float v = acc[c];
            acc[c] = 0.f;
            if (v != 0.f) Sj[c] = v;
          }
        }
        if (threadIdx.x == 0) counts[j] = b - a;
      } else {  // a piece of a cluster that other segments share
        for (int c = threadIdx.x; c < d; c += blockDim.x) {
          const float v = acc[c];
          acc[c] = 0.f;
          if (v != 0.f) atomicAdd(Sj + c, v);
        }
        if (threadIdx.x == 0) atomicAdd(counts + j, b - a);
      }
      __syncthreads();  // acc (zeroed) is reused by the next cluster
    }
  }
}

bool csr_sorted_update_supported(int d) { return (size_t)d * sizeof(float) <= 200 * 1024; }

void launch_update_csr_sorted(const int64_t* row_ptr, const int32_t* col, const float* val, int d,
                              const int32_t* perm, const int32_t* labels, const int32_t* end, int64_t n, int64_t k,
                              float* S, int32_t* counts, cudaStream_t st, const int* active) {
  if (k <= 0 || n <= 0) return;
  const size_t smem = (size_t)d * sizeof(float);
  static size_t attr_for = 0;
  if (smem > 48 * 1024 && attr_for < smem) {
    MASK_CUDA(cudaFuncSetAttribute(k_update_csr_sorted, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_for = 200 * 1024;
  }
  const int per_sm = smem > 0 ? (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / std::max<size_t>(smem, 1))) : 8;
  const int64_t grid = std::min<int64_t>((n + kSegRows - 1) / kSegRows, (int64_t)num_sms() * per_sm);
  k_update_csr_sorted<<<(unsigned)grid, 256, smem, st>>>(row_ptr, col, val, d, perm, labels, end, n, k, S, counts,
                                                         active);
  MASK_LAUNCH_CHECK();
}

// ====================================================================== K7 finalize
// Warp per prototype.  stat[0] = max over j of ||c_new - c_old||^2 (float bits, atomicMax on
// non-negative floats), stat[1] = number of empty prototypes.  S and counts are zeroed for
// the next pass (unless keep_counts, which leaves counts for the caller to read).
// Last block of a grid (ticket counter, reset by that block): true in exactly one block,
// after every block's earlier global writes/atomics are visible.
__device__ __forceinline__ bool last_block_done(int* ticket) {
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;
    if (last) *ticket = 0;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

__global__ void k_finalize(float* __restrict__ P, float* __restrict__ S, int32_t* __restrict__ counts,
                           int64_t k, int d, uint32_t* __restrict__ stat, int keep_counts,
                           const int* __restrict__ active, LoopCtl lc) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < k; j += warps) {
    if (lc.zero_cnt && lane == 0) lc.zero_cnt[j] = 0;  // label-sort counts of the next pass
    const int32_t cnt = counts[j];
    float disp = 0.f;
    if (cnt > 0) {
      for (int i = lane; i < d; i += 32) {
        const float s = S[j * d + i];
        const float c = __fdiv_rn(s, (float)cnt);
        const float t = c - P[j * d + i];
        disp = fmaf(t, t, disp);
        P[j * d + i] = c;
        S[j * d + i] = 0.f;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) disp += __shfl_xor_sync(0xffffffffu, disp, o);
    if (lane == 0) {
      atomicMax(stat, __float_as_uint(disp));
      if (cnt == 0) atomicAdd(stat + 1, 1u);
      if (!keep_counts) counts[j] = 0;
    }
  }
  // fused loop control (D3 tolerance stop / pass count), formerly a separate 1-thread kernel
  if (lc.ctrl && last_block_done(lc.ctrl + 3) && threadIdx.x == 0) {
    const double disp = sqrt((double)__uint_as_float(*(volatile uint32_t*)stat));
    if (lc.tol > 0.0 && disp <= lc.tol) {
      lc.ctrl[0] = 0;
      lc.ctrl[1] = lc.t + 1;
    } else if (lc.t == lc.T - 1) {
      lc.ctrl[1] = lc.T;
    }
  }
}

// Wide rows (d >= 256, e.g. the dense C4 prototypes with d = 10,000): a block per prototype,
// 16-byte vectors, so the k*d read-modify-write streams at HBM speed instead of a warp walking
// d / 32 scalar iterations.
__global__ void __launch_bounds__(256) k_finalize_wide(float* __restrict__ P, float* __restrict__ S,
                                                       int32_t* __restrict__ counts, int64_t k, int d,
                                                       uint32_t* __restrict__ stat, int keep_counts,
                                                       const int* __restrict__ active, LoopCtl lc) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  __shared__ float red[8];
  for (int64_t j = blockIdx.x; j < k; j += gridDim.x) {
    if (lc.zero_cnt && threadIdx.x == 0) lc.zero_cnt[j] = 0;
    const int32_t cnt = counts[j];
    float disp = 0.f;
    if (cnt > 0) {
      const float fc = (float)cnt;
      float4* P4 = reinterpret_cast<float4*>(P + j * d);
      float4* S4 = reinterpret_cast<float4*>(S + j * d);
      for (int e = threadIdx.x; e < d / 4; e += blockDim.x) {
        const float4 sv = S4[e], pv = P4[e];
        float4 cv;
        cv.x = __fdiv_rn(sv.x, fc);
        cv.y = __fdiv_rn(sv.y, fc);
        cv.z = __fdiv_rn(sv.z, fc);
        cv.w = __fdiv_rn(sv.w, fc);
        float t = cv.x - pv.x;
        disp = fmaf(t, t, disp);
        t = cv.y - pv.y;
        disp = fmaf(t, t, disp);
        t = cv.z - pv.z;
        disp = fmaf(t, t, disp);
        t = cv.w - pv.w;
        disp = fmaf(t, t, disp);
        P4[e] = cv;
        S4[e] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) disp += __shfl_xor_sync(0xffffffffu, disp, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = disp;
    __syncthreads();
    if (threadIdx.x == 0) {
      float tot = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
      atomicMax(stat, __float_as_uint(tot));
      if (cnt == 0) atomicAdd(stat + 1, 1u);
      if (!keep_counts) counts[j] = 0;
    }
    __syncthreads();
  }
  if (lc.ctrl && last_block_done(lc.ctrl + 3) && threadIdx.x == 0) {
    const double dsp = sqrt((double)__uint_as_float(*(volatile uint32_t*)stat));
    if (lc.tol > 0.0 && dsp <= lc.tol) {
      lc.ctrl[0] = 0;
      lc.ctrl[1] = lc.t + 1;
    } else if (lc.t == lc.T - 1) {
      lc.ctrl[1] = lc.T;
    }
  }
}

__global__ void k_finalize64(double* __restrict__ P64, float* __restrict__ P, double* __restrict__ S,
                             int32_t* __restrict__ counts, int64_t k, int d, uint32_t* __restrict__ stat,
                             const int* __restrict__ active, LoopCtl lc) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < k; j += warps) {
    if (lc.zero_cnt && lane == 0) lc.zero_cnt[j] = 0;  // label-sort counts of the next pass
    const int32_t cnt = counts[j];
    double disp = 0.0;
    if (cnt > 0) {
      for (int i = lane; i < d; i += 32) {
        const double c = __ddiv_rn(S[j * d + i], (double)cnt);
        const double t = c - P64[j * d + i];
        disp = fma(t, t, disp);
        P64[j * d + i] = c;
        P[j * d + i] = (float)c;
        S[j * d + i] = 0.0;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) disp += __shfl_xor_sync(0xffffffffu, disp, o);
    if (lane == 0) {
      atomicMax(stat, __float_as_uint((float)disp));
      if (cnt == 0) atomicAdd(stat + 1, 1u);
      counts[j] = 0;
    }
  }
  if (lc.ctrl && last_block_done(lc.ctrl + 3) && threadIdx.x == 0) {
    const double disp = sqrt((double)__uint_as_float(*(volatile uint32_t*)stat));
    if (lc.tol > 0.0 && disp <= lc.tol) {
      lc.ctrl[0] = 0;
      lc.ctrl[1] = lc.t + 1;
    } else if (lc.t == lc.T - 1) {
      lc.ctrl[1] = lc.T;
    }
  }
}

void launch_finalize64(double* P64, float* P, double* S, int32_t* counts, int64_t k, int d, uint32_t* stat,
                       cudaStream_t st, const int* active, LoopCtl lc) {
  k_finalize64<<<grid_for(k * 32, 256), 256, 0, st>>>(P64, P, S, counts, k, d, stat, active, lc);
  MASK_LAUNCH_CHECK();
}

// ====================================================================== D5b farthest-point repair
// SPEC S:128 (reading D5b): the prototypes an update leaves without members, in ascending j,
// are re-seeded at the rows with the largest distance to their prototype in this pass (best[],
// the assignment's d^2), ordered by (distance descending, row ascending).  Runs between the
// update and K7 (which keeps counts == 0 prototypes as they are), so only the re-seeded rows
// are written here; their displacement joins K7's maximum for the tolerance stop.
//
// Ordered compaction of the empty prototypes (single block): emp[0..m) ascending, m_out[0] = m
// (0 when the level already stopped: active == 0).
__global__ void __launch_bounds__(1024) k_empty_list(const int32_t* __restrict__ counts, int64_t k,
                                                     int32_t* __restrict__ emp, int* __restrict__ m_out,
                                                     const int* __restrict__ active) {
  __shared__ int part[1024];
  const int t = threadIdx.x;
  const bool on = !active || *active;
  const int64_t per = (k + blockDim.x - 1) / blockDim.x;
  const int64_t a = t * per, b = a + per < k ? a + per : k;
  int c = 0;
  if (on)
    for (int64_t j = a; j < b; ++j) c += counts[j] == 0;
  part[t] = c;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {
    const int v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int w = part[t] - c;
  if (on)
    for (int64_t j = a; j < b; ++j)
      if (counts[j] == 0) emp[w++] = (int32_t)j;
  if (t == blockDim.x - 1) m_out[0] = part[t];
}

// number of rows whose d^2 (non-negative float, ordered as its bit pattern) is >= thr
__global__ void k_count_ge(const float* __restrict__ best, int64_t n, uint32_t thr,
                           unsigned long long* __restrict__ cnt) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += __float_as_uint(best[i]) >= thr;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

__global__ void k_collect_ge(const float* __restrict__ best, int64_t n, uint32_t thr, int64_t* __restrict__ rows,
                             uint32_t* __restrict__ keys, unsigned long long* __restrict__ cnt, int64_t cap) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t b = __float_as_uint(best[i]);
    if (b >= thr) {
      const unsigned long long at = atomicAdd(cnt, 1ull);
      if ((int64_t)at < cap) {
        rows[at] = i;
        keys[at] = b;
      }
    }
  }
}

// block per re-seeded prototype: P_j <- row (densified for CSR), P64_j likewise; the squared
// displacement (against the FP64 prototype when there is one) into stat[0] (float bits, max)
__global__ void __launch_bounds__(256) k_reseed(const float* __restrict__ X, const int64_t* __restrict__ rp,
                                                const int32_t* __restrict__ col, const float* __restrict__ val,
                                                int d, const int64_t* __restrict__ rows,
                                                const int32_t* __restrict__ emp, float* __restrict__ P,
                                                double* __restrict__ P64, uint32_t* __restrict__ stat) {
  const int64_t j = emp[blockIdx.x], row = rows[blockIdx.x];
  double acc = 0.0;
  if (X) {
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
      const float v = X[row * d + c];
      const double old = P64 ? P64[j * d + c] : (double)P[j * d + c];
      const double t = (double)v - old;
      acc += t * t;
      P[j * d + c] = v;
      if (P64) P64[j * d + c] = (double)v;
    }
  } else {
    // ||new - old||^2 = sum_c old_c^2 + sum_{nz} ((v - old_c)^2 - old_c^2), before overwriting
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
      const double old = (double)P[j * d + c];
      acc += old * old;
    }
    for (int64_t p = rp[row] + threadIdx.x; p < rp[row + 1]; p += blockDim.x) {
      const double old = (double)P[j * d + col[p]];
      const double t = (double)val[p] - old;
      acc += t * t - old * old;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += blockDim.x) P[j * d + c] = 0.f;
    __syncthreads();
    for (int64_t p = rp[row] + threadIdx.x; p < rp[row + 1]; p += blockDim.x) P[j * d + col[p]] = val[p];
  }
  __shared__ double red[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s2 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s2 += red[w];
    atomicMax(stat, __float_as_uint((float)(s2 > 0.0 ? s2 : 0.0)));
  }
}

void reseed_farthest(const float* X, const int64_t* rp, const int32_t* col, const float* val, int d, int64_t n,
                     int64_t k, const float* best, const int32_t* counts, float* P, double* P64, uint32_t* stat,
                     const int* active, cudaStream_t st) {
  if (n <= 0 || k <= 0) return;
  DevBuf<int32_t> emp(k);
  DevBuf<int> m_d(1);
  k_empty_list<<<1, 1024, 0, st>>>(counts, k, emp.p, m_d.p, active);
  MASK_LAUNCH_CHECK();
  int m = 0;
  MASK_CUDA(cudaMemcpyAsync(&m, m_d.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaStreamSynchronize(st));
  if (m <= 0) return;
  if (m > n) m = (int)n;
  // the m-th largest key: largest thr with count(key >= thr) >= m (bisection on the bits)
  DevBuf<unsigned long long> cnt(1);
  auto count_ge = [&](uint32_t thr) {
    MASK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
    k_count_ge<<<grid_for(n, 256, (int64_t)num_sms() * 8), 256, 0, st>>>(best, n, thr, cnt.p);
    MASK_LAUNCH_CHECK();
    unsigned long long h = 0;
    MASK_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    MASK_CUDA(cudaStreamSynchronize(st));
    return h;
  };
  uint32_t lo = 0, hi = 0x7f800001u;  // count(>= lo) = n >= m; count(>= hi) = 0 (finite d^2)
  unsigned long long c_lo = (unsigned long long)n;
  while (hi - lo > 1) {
    const uint32_t mid = lo + (hi - lo) / 2;
    const unsigned long long c = count_ge(mid);
    if (c >= (unsigned long long)m) {
      lo = mid;
      c_lo = c;
    } else {
      hi = mid;
    }
  }
  DevBuf<int64_t> rows(c_lo);
  DevBuf<uint32_t> keys(c_lo);
  MASK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
  k_collect_ge<<<grid_for(n, 256, (int64_t)num_sms() * 8), 256, 0, st>>>(best, n, lo, rows.p, keys.p, cnt.p,
                                                                          (int64_t)c_lo);
  MASK_LAUNCH_CHECK();
  std::vector<int64_t> hr(c_lo);
  std::vector<uint32_t> hk(c_lo);
  MASK_CUDA(cudaMemcpyAsync(hr.data(), rows.p, sizeof(int64_t) * c_lo, cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaMemcpyAsync(hk.data(), keys.p, sizeof(uint32_t) * c_lo, cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaStreamSynchronize(st));
  std::vector<size_t> ord(c_lo);
  for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
    return hk[a] != hk[b] ? hk[a] > hk[b] : hr[a] < hr[b];  // distance descending, row ascending
  });
  std::vector<int64_t> far(m);
  for (int r = 0; r < m; ++r) far[r] = hr[ord[r]];
  DevBuf<int64_t> far_d(m);
  MASK_CUDA(cudaMemcpyAsync(far_d.p, far.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice, st));
  k_reseed<<<(unsigned)m, 256, 0, st>>>(X, rp, col, val, d, far_d.p, emp.p, P, P64, stat);
  MASK_LAUNCH_CHECK();
  MASK_CUDA(cudaStreamSynchronize(st));  // (host vectors and scratch go out of scope)
}

__global__ void k_f32_to_f64(const float* __restrict__ a, int64_t n, double* __restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (double)a[i];
}
void launch_f32_to_f64(const float* a, int64_t n, double* b, cudaStream_t st) {
  if (n <= 0) return;
  k_f32_to_f64<<<grid_for(n, 256), 256, 0, st>>>(a, n, b);
  MASK_LAUNCH_CHECK();
}

void launch_finalize(float* P, float* S, int32_t* counts, int64_t k, int d, uint32_t* stat,
                     int keep_counts, cudaStream_t st, const int* active, LoopCtl lc) {
  if (d >= 256 && d % 4 == 0 && ((uintptr_t)P % 16) == 0 && ((uintptr_t)S % 16) == 0)
    k_finalize_wide<<<grid_for(k, 1, (int64_t)num_sms() * 8), 256, 0, st>>>(P, S, counts, k, d, stat, keep_counts,
                                                                             active, lc);
  else
    k_finalize<<<grid_for(k * 32, 256), 256, 0, st>>>(P, S, counts, k, d, stat, keep_counts, active, lc);
  MASK_LAUNCH_CHECK();
}

// ====================================================================== pass statistics
__global__ void k_pass_stats(const int32_t* __restrict__ cur, const int32_t* __restrict__ prev,
                             const float* __restrict__ best, int64_t n, double* __restrict__ J,
                             unsigned long long* __restrict__ changed, const int* __restrict__ active,
                             LoopCtl lc) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  double s = 0.0;
  unsigned long long c = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    s += (double)best[i];
    c += (cur[i] != prev[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  __shared__ double ss[32];
  __shared__ unsigned long long sc[32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    ss[w] = s;
    sc[w] = c;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    s = lane < nw ? ss[lane] : 0.0;
    c = lane < nw ? sc[lane] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (lane == 0) {
      atomicAdd(J, s);
      atomicAdd(changed, c);
    }
  }
  // fused stop test (single GPU): no label changed -> the update would be a no-op
  if (lc.ctrl && last_block_done(lc.ctrl + 2) && threadIdx.x == 0) {
    if (lc.t > 0 && *(volatile unsigned long long*)changed == 0) {
      lc.ctrl[0] = 0;
      lc.ctrl[1] = lc.t + 1;
    }
  }
}

void launch_pass_stats(const int32_t* cur, const int32_t* prev, const float* best, int64_t n,
                       double* J, unsigned long long* changed, cudaStream_t st, const int* active, LoopCtl lc) {
  if (n <= 0) return;
  k_pass_stats<<<grid_for(n, 256, (int64_t)num_sms() * 4), 256, 0, st>>>(cur, prev, best, n, J,
                                                                         changed, active, lc);
  MASK_LAUNCH_CHECK();
}

// ====================================================================== K10 init gather
// P[j] = Y[idx[j] - row_offset] if that global row is owned by this shard, else zeros (the
// multi-GPU init allreduce sums the owners' copies).
__global__ void k_gather_rows(const float* __restrict__ Y, int d, const int64_t* __restrict__ idx,
                              int64_t k, int64_t row_offset, int64_t n_local, float* __restrict__ P) {
  const int64_t total = k * (int64_t)d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / d;
    const int c = (int)(e - j * d);
    const int64_t r = idx[j] - row_offset;
    P[e] = (r >= 0 && r < n_local) ? Y[r * d + c] : 0.f;
  }
}

void launch_gather_rows(const float* Y, int d, const int64_t* idx, int64_t k, int64_t row_offset,
                        int64_t n_local, float* P, cudaStream_t st) {
  k_gather_rows<<<grid_for(k * d, 256), 256, 0, st>>>(Y, d, idx, k, row_offset, n_local, P);
  MASK_LAUNCH_CHECK();
}

__global__ void k_gather_csr_rows(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                  const float* __restrict__ val, int d,
                                  const int64_t* __restrict__ idx, int64_t k, int64_t row_offset,
                                  int64_t n_local, float* __restrict__ P) {
  // P must be zeroed by the caller; warp per prototype scatters its row's non-zeros.
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < k; j += warps) {
    const int64_t r = idx[j] - row_offset;
    if (r < 0 || r >= n_local) continue;
    for (int64_t p = rp[r] + lane; p < rp[r + 1]; p += 32) P[j * d + col[p]] = val[p];
  }
}

void launch_gather_csr_rows(const int64_t* row_ptr, const int32_t* col, const float* val, int d,
                            const int64_t* idx, int64_t k, int64_t row_offset, int64_t n_local,
                            float* P, cudaStream_t st) {
  k_gather_csr_rows<<<grid_for(k * 32, 256), 256, 0, st>>>(row_ptr, col, val, d, idx, k, row_offset,
                                                           n_local, P);
  MASK_LAUNCH_CHECK();
}

// ====================================================================== K8 child lists
__global__ void k_histogram(const int32_t* __restrict__ labels, int64_t n, int32_t* __restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + labels[i], 1);
}

// Single-block exclusive scan of k counts into offsets[0..k] (k <= a few million).
__global__ void __launch_bounds__(1024) k_scan_offsets(const int32_t* __restrict__ cnt, int64_t k,
                                                       int64_t* __restrict__ offsets,
                                                       int32_t* __restrict__ cursor) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = 0; base < k; base += 1024) {
    const int64_t j = base + threadIdx.x;
    int64_t v = j < k ? cnt[j] : 0;
    int64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    if (w == 0) {
      int64_t t = warp_tot[lane];
      int64_t ti = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int64_t u = __shfl_up_sync(0xffffffffu, ti, o);
        if (lane >= o) ti += u;
      }
      warp_tot[lane] = ti - t;  // exclusive prefix of warp totals
    }
    __syncthreads();
    const int64_t excl = carry + warp_tot[w] + incl - v;
    if (j < k) {
      offsets[j] = excl;
      cursor[j] = (int32_t)excl;
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) offsets[k] = carry;
}

__global__ void k_scatter_members(const int32_t* __restrict__ labels, int64_t n,
                                  int32_t* __restrict__ cursor, int32_t* __restrict__ members) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t pos = atomicAdd(cursor + labels[i], 1);
    members[pos] = (int32_t)i;
  }
}

void launch_children(const int32_t* labels, int64_t n, int64_t k, int64_t* offsets,
                     int32_t* members, int32_t* cursor_ws, cudaStream_t st) {
  MASK_CUDA(cudaMemsetAsync(cursor_ws, 0, sizeof(int32_t) * k, st));
  if (n > 0) k_histogram<<<grid_for(n, 256), 256, 0, st>>>(labels, n, cursor_ws);
  MASK_LAUNCH_CHECK();
  // counts live in cursor_ws; scan writes offsets and resets cursor to the segment starts
  k_scan_offsets<<<1, 1024, 0, st>>>(cursor_ws, k, offsets, cursor_ws);
  MASK_LAUNCH_CHECK();
  if (n > 0) k_scatter_members<<<grid_for(n, 256), 256, 0, st>>>(labels, n, cursor_ws, members);
  MASK_LAUNCH_CHECK();
}

// Counting sort of row indices by label (K1 row order for warp-coherent pruning): perm lists
// the rows of label 0, then label 1, ... (order inside a label unspecified).  Labels outside
// [0, k) are skipped (their rows are appended by nobody: callers pass complete labelings).
__global__ void k_sort_zero(int32_t* __restrict__ cnt, int64_t k, const int* __restrict__ active) {
  if (active && !*active) return;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x)
    cnt[j] = 0;
}
// Positions are visited in the previous pass's sorted order (perm_old, or identity), where
// equal labels are mostly adjacent: a warp aggregates equal labels with __match_any_sync and
// one lane does the atomic for the group, so the count / cursor atomics hit each label about
// once per warp instead of once per row.  copy_to (optional) receives labels[row] (the
// lab_prev <- lab_cur copy of the Lloyd loop, fused here).
__global__ void k_sort_hist(const int32_t* __restrict__ labels, const int32_t* __restrict__ perm_old, int64_t n,
                            int64_t k, int32_t* __restrict__ cnt, int32_t* __restrict__ copy_to,
                            const int* __restrict__ active) {
  if (active && !*active) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t p = base + threadIdx.x;
    int32_t l = -1;
    if (p < n) {
      const int64_t row = perm_old ? (int64_t)__ldg(perm_old + p) : p;
      l = labels[row];
      if (copy_to) copy_to[row] = l;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, l);
    if (l >= 0 && l < k && lane == __ffs(peers) - 1) atomicAdd(cnt + l, __popc(peers));
  }
}
__global__ void __launch_bounds__(1024) k_sort_scan(int32_t* __restrict__ cnt, int64_t k, const int* __restrict__ active) {
  if (active && !*active) return;
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = 0; base < k; base += 1024) {
    const int64_t j = base + threadIdx.x;
    const int32_t v = j < k ? cnt[j] : 0;
    int32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    if (w == 0) {
      const int32_t t = warp_tot[lane];
      int32_t ti = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t u = __shfl_up_sync(0xffffffffu, ti, o);
        if (lane >= o) ti += u;
      }
      warp_tot[lane] = ti - t;
    }
    __syncthreads();
    const int32_t excl = carry + warp_tot[w] + incl - v;
    if (j < k) cnt[j] = excl;  // becomes the scatter cursor
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
}
__global__ void k_sort_scatter(const int32_t* __restrict__ labels, const int32_t* __restrict__ perm_old, int64_t n,
                               int64_t k, int32_t* __restrict__ cursor, int32_t* __restrict__ perm,
                               const int* __restrict__ active) {
  if (active && !*active) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t p = base + threadIdx.x;
    int32_t l = -1;
    int64_t row = 0;
    if (p < n) {
      row = perm_old ? (int64_t)__ldg(perm_old + p) : p;
      l = labels[row];
    }
    const unsigned peers = __match_any_sync(0xffffffffu, l);
    const int leader = __ffs(peers) - 1;
    int32_t pos = 0;
    if (l >= 0 && l < k && lane == leader) pos = atomicAdd(cursor + l, __popc(peers));
    pos = __shfl_sync(0xffffffffu, pos, leader);
    if (l >= 0 && l < k) perm[pos + __popc(peers & ((1u << lane) - 1))] = (int32_t)row;
  }
}

void launch_label_sort(const int32_t* labels, int64_t n, int64_t k, const int32_t* perm_old, int32_t* perm,
                       int32_t* cnt_ws, int32_t* copy_to, cudaStream_t st, const int* active, bool cnt_zeroed) {
  if (n <= 0) return;
  if (!cnt_zeroed) {
    k_sort_zero<<<grid_for(k, 256), 256, 0, st>>>(cnt_ws, k, active);
    MASK_LAUNCH_CHECK();
  }
  const unsigned grid = grid_for(n, 256, (int64_t)num_sms() * 8);
  k_sort_hist<<<grid, 256, 0, st>>>(labels, perm_old, n, k, cnt_ws, copy_to, active);
  MASK_LAUNCH_CHECK();
  k_sort_scan<<<1, 1024, 0, st>>>(cnt_ws, k, active);
  MASK_LAUNCH_CHECK();
  k_sort_scatter<<<grid, 256, 0, st>>>(labels, perm_old, n, k, cnt_ws, perm, active);
  MASK_LAUNCH_CHECK();
}

// ====================================================================== misc
__global__ void k_i64_to_i32(const int64_t* __restrict__ a, int64_t n, int32_t* __restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (int32_t)a[i];
}

void launch_i64_to_i32(const int64_t* a, int64_t n, int32_t* b, cudaStream_t st) {
  if (n <= 0) return;
  k_i64_to_i32<<<grid_for(n, 256), 256, 0, st>>>(a, n, b);
  MASK_LAUNCH_CHECK();
}
__global__ void k_check_finite(const float* __restrict__ v, int64_t count, int32_t* flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(v[i])) *flag = 1;
}

void launch_check_finite(const float* v, int64_t count, int32_t* flag, cudaStream_t st) {
  if (count <= 0) return;
  k_check_finite<<<grid_for(count, 256), 256, 0, st>>>(v, count, flag);
  MASK_LAUNCH_CHECK();
}

__global__ void k_fill(float* p, int64_t count, float v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

void launch_fill(float* p, int64_t count, float v, cudaStream_t st) {
  if (count <= 0) return;
  k_fill<<<grid_for(count, 256), 256, 0, st>>>(p, count, v);
  MASK_LAUNCH_CHECK();
}

// PT[i * k + j] = P[j * d + i] (d x k), used by the sparse assignment.
__global__ void k_transpose(const float* __restrict__ P, int64_t k, int d, float* __restrict__ PT,
                            const int* __restrict__ active) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  __shared__ float tile[32][33];
  const int64_t j0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = j0 + r, i = i0 + threadIdx.x;
    tile[r][threadIdx.x] = (j < k && i < d) ? P[j * d + i] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r, j = j0 + threadIdx.x;
    if (i < d && j < k) PT[i * k + j] = tile[threadIdx.x][r];
  }
}

void launch_transpose(const float* P, int64_t k, int d, float* PT, cudaStream_t st, const int* active) {
  dim3 grid((unsigned)((k + 31) / 32), (unsigned)((d + 31) / 32));
  k_transpose<<<grid, dim3(32, 8), 0, st>>>(P, k, d, PT, active);
  MASK_LAUNCH_CHECK();
}

// CSR structure check on the device (include/mask.h mask_matrix: row_ptr[0] = 0, non-decreasing,
// row_ptr[rows] = nnz, columns strictly increasing within a row and < dim): a warp per row,
// error bits OR-ed into *err (1 = row_ptr, 2 = column range, 4 = column order).
__global__ void k_check_csr(const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t rows,
                            int64_t nnz, int dim, int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  if (blockIdx.x == 0 && threadIdx.x == 0 && (rp[0] != 0 || rp[rows] != nnz)) atomicOr(err, 1);
  int bits = 0;
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const int64_t a = rp[r], b = rp[r + 1];
    if (a < 0 || b < a || b > nnz) {
      bits |= 1;
      continue;
    }
    for (int64_t q = a + lane; q < b; q += 32) {
      const int32_t c = col[q];
      if (c < 0 || c >= dim) bits |= 2;
      if (q > a && col[q - 1] >= c) bits |= 4;
    }
  }
  bits = __reduce_or_sync(0xffffffffu, bits);
  if (lane == 0 && bits) atomicOr(err, bits);
}

void launch_check_csr(const int64_t* rp, const int32_t* col, int64_t rows, int64_t nnz, int dim, int* err,
                      cudaStream_t st) {
  MASK_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
  k_check_csr<<<grid_for(rows * 32, 256), 256, 0, st>>>(rp, col, rows, nnz, dim, err);
  MASK_LAUNCH_CHECK();
}

}  // namespace mask
