// relocate.cu -- §5.1 relocation bookkeeping between rebuilds (reading G8,
// DESIGN.md): after a grouped build over the data-layer order `order_in` and a beam-1 1-NN
// point search of every point (got[i]), a found point keeps its data-layer group, a missed one
// targets the group of the partition its search reached (level-1 prototype id // nCentroids;
// a search that reached no partition keeps the point in place); the next order lists the
// target groups in order, the points of a group ordered by the iteration's keys.
//
// Groups of the current order: positions split into g balanced groups, the last (n mod g) one
// larger (G1).  The order is a radix sort (sort.cu) of the 64-bit keys (target << 32 | key);
// keys are a permutation rank, so every key is distinct.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace mask {

namespace {

__device__ __forceinline__ int64_t group_of_pos(int64_t p, int64_t n, int64_t g) {
  const int64_t base = n / g, rem = n % g, small = g - rem;  // the first `small` groups hold `base`
  return p < small * base ? p / base : small + (p - small * base) / (base + 1);
}

__global__ void k_reloc_keys(const int64_t* __restrict__ got, const int64_t* __restrict__ order_in,
                             const int64_t* __restrict__ keys, const int32_t* __restrict__ lab1, int64_t n,
                             int64_t g, int n_centroids, uint64_t* __restrict__ comp,
                             int64_t* __restrict__ val, int64_t* __restrict__ reached_out,
                             unsigned long long* __restrict__ misses) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = order_in[p];
    const int64_t gi = got[i];
    const bool found = gi == i;
    const int64_t reached = gi >= 0 ? (int64_t)(lab1[gi] / n_centroids) : -1;
    const int64_t target = (found || reached < 0) ? group_of_pos(p, n, g) : reached;
    comp[p] = ((uint64_t)target << 32) | (uint64_t)(uint32_t)keys[i];
    val[p] = i;
    if (reached_out) reached_out[i] = reached;
    if (!found) atomicAdd(misses, 1ull);
  }
}

}  // namespace

void launch_relocate(const int64_t* got, const int64_t* order_in, const int64_t* keys, const int32_t* lab1, int64_t n,
                     int64_t n_groups, int n_centroids, int64_t* order_out, int64_t* reached_out,
                     unsigned long long* misses, cudaStream_t st) {
  DevBuf<uint64_t> comp(n);
  MASK_CUDA(cudaMemsetAsync(misses, 0, sizeof(unsigned long long), st));
  k_reloc_keys<<<grid_for(n, 256), 256, 0, st>>>(got, order_in, keys, lab1, n, n_groups, n_centroids, comp.p,
                                                 order_out, reached_out, misses);
  MASK_LAUNCH_CHECK();
  radix_sort_pairs(comp.p, order_out, n, 0, 64, st);  // (target, key): distinct keys
}

}  // namespace mask
