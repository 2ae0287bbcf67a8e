// grouped.cu -- K12: the paper's grouped construction (Algorithm 1), SURVEY
// §8(f) NEXT-1.  A layer of n items is split into g = floor(n / lengthGroup) groups (balanced:
// the last n mod g groups hold one extra item, G1) and every group is clustered
// independently with nCentroids k-means prototypes; the g * nCentroids prototypes (group-major)
// are the next layer's items.  One CTA per group runs that group's whole Lloyd loop in shared
// memory (the paper's groups are tiny: lengthGroup 10..110 points in R^2, §5.2):
//
//   init  c_j = the group's first nCentroids items (its chunk order; the data layer's chunks
//         follow the caller's seeded permutation, G1/G3)
//   for t < T: a_i = argmin_j ||y_i - c_j||^2 (FP32 direct, lowest j on ties, D4);
//              stop if t > 0 and no label changed (D3); c_j = mean of its members (FP64
//              sums), empty clusters keep c_j (D5)
//   final assignment; labels are global prototype ids g_i * nCentroids + a_i.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "common.cuh"

namespace mask {

namespace {

__global__ void __launch_bounds__(128) k_group_lloyd(const float* __restrict__ Y, int d,
                                                     const int64_t* __restrict__ perm, int64_t n_items, int64_t g,
                                                     int nc, int T, float* __restrict__ P_out,
                                                     int32_t* __restrict__ labels) {
  extern __shared__ double gsm[];
  const int64_t base = n_items / g, rem = n_items % g;
  const int smax = (int)(base + (rem ? 1 : 0));
  double* sums = gsm;                                                  // [nc][d]
  float* cs = reinterpret_cast<float*>(sums + (size_t)nc * d);        // [nc][d]
  float* xs = cs + (size_t)nc * d;                                     // [smax][d]
  int32_t* cnt = reinterpret_cast<int32_t*>(xs + (size_t)smax * d);   // [nc]
  int32_t* lab = cnt + nc;                                             // [smax]
  int32_t* prv = lab + smax;                                           // [smax]
  for (int64_t gi = blockIdx.x; gi < g; gi += gridDim.x) {
    const int64_t extra = gi - (g - rem) > 0 ? gi - (g - rem) : 0;  // extra-item groups before gi
    const int64_t start = gi * base + extra;
    const int size = (int)(base + (gi >= g - rem ? 1 : 0));
    __syncthreads();
    for (int e = threadIdx.x; e < size * d; e += blockDim.x) {
      const int i = e / d, c = e - i * d;
      const int64_t row = perm ? perm[start + i] : start + i;
      xs[e] = Y[row * d + c];
    }
    for (int i = threadIdx.x; i < size; i += blockDim.x) prv[i] = -1;
    __syncthreads();
    for (int e = threadIdx.x; e < nc * d; e += blockDim.x) cs[e] = xs[e];  // first nc items (G3)
    __syncthreads();
    for (int t = 0;; ++t) {
      // ---- assignment (also the final pass when t == T)
      int changed = 0;
      for (int i = threadIdx.x; i < size; i += blockDim.x) {
        float bv = INFINITY;
        int bj = 0;
        for (int j = 0; j < nc; ++j) {
          float acc = 0.f;
          for (int c = 0; c < d; ++c) {
            const float df = xs[i * d + c] - cs[j * d + c];
            acc = fmaf(df, df, acc);
          }
          if (acc < bv) {  // strict: lowest j on ties
            bv = acc;
            bj = j;
          }
        }
        lab[i] = bj;
        changed |= bj != prv[i];
      }
      const int any = __syncthreads_or(changed);
      if (t == T || (t > 0 && !any)) break;  // final pass done / converged (D3)
      // ---- update: FP64 member sums, counts
      for (int e = threadIdx.x; e < nc * d; e += blockDim.x) sums[e] = 0.0;
      for (int j = threadIdx.x; j < nc; j += blockDim.x) cnt[j] = 0;
      __syncthreads();
      for (int e = threadIdx.x; e < size * d; e += blockDim.x) {
        const int i = e / d, c = e - i * d;
        atomicAdd(sums + (size_t)lab[i] * d + c, (double)xs[e]);
        if (c == 0) atomicAdd(cnt + lab[i], 1);
      }
      __syncthreads();
      for (int e = threadIdx.x; e < nc * d; e += blockDim.x) {
        const int j = e / d;
        if (cnt[j] > 0) cs[e] = (float)(sums[e] / (double)cnt[j]);  // empty keeps (D5)
      }
      for (int i = threadIdx.x; i < size; i += blockDim.x) prv[i] = lab[i];
      __syncthreads();
    }
    // (a converged loop breaks right after an assignment: lab holds the labels of the final cs)
    for (int e = threadIdx.x; e < nc * d; e += blockDim.x) P_out[(gi * nc) * d + e] = cs[e];
    for (int i = threadIdx.x; i < size; i += blockDim.x) {
      const int64_t row = perm ? perm[start + i] : start + i;
      labels[row] = (int32_t)(gi * nc + lab[i]);
    }
  }
}

}  // namespace

size_t group_lloyd_smem(int64_t n_items, int64_t g, int nc, int d) {
  const int64_t smax = n_items / g + (n_items % g ? 1 : 0);
  return (size_t)nc * d * sizeof(double) + (size_t)nc * d * sizeof(float) + (size_t)smax * d * sizeof(float) +
         (size_t)nc * sizeof(int32_t) + 2 * (size_t)smax * sizeof(int32_t);
}

void launch_group_lloyd(const float* Y, int d, const int64_t* perm, int64_t n_items, int64_t g, int nc, int T,
                        float* P_out, int32_t* labels, cudaStream_t st) {
  const size_t smem = group_lloyd_smem(n_items, g, nc, d);
  MASK_REQUIRE(smem <= 200 * 1024, MASK_ERR_UNSUPPORTED,
               "grouped build: a group (items + prototypes + sums) exceeds 200 KB of shared memory");
  if (smem > 48 * 1024) MASK_CUDA(cudaFuncSetAttribute(k_group_lloyd, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int64_t grid = g < (int64_t)num_sms() * 64 ? g : (int64_t)num_sms() * 64;
  k_group_lloyd<<<(unsigned)grid, 128, smem, st>>>(Y, d, perm, n_items, g, nc, T, P_out, labels);
  MASK_LAUNCH_CHECK();
}

}  // namespace mask
