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

}  // namespace mask
