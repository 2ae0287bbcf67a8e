// Micro-benchmark: per-SM TMA throughput streaming K1-style B tiles (two 2-D fp32 tensors,
// 128-byte-swizzled boxes of 32 columns x ROWS rows) from an L2-resident prototype array
// through a STAGES-deep mbarrier ring, one CTA per SM, consumer = plain re-arm (no MMA).
// Reports cycles per tile (both boxes) and bytes/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_ubench tools/tma_ubench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ bool try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok)
               : "r"(smem_u32(bar)), "r"(parity)
               : "memory");
  return ok != 0;
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
  while (!try_wait(bar, parity)) {
  }
}

template <int ROWS, int STAGES>
__global__ void k_tma(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int tiles,
                      int tile_rows_total, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[STAGES];
  constexpr int BOX = ROWS * 128, STAGE = 2 * BOX;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    const int ntile_rows = tile_rows_total / ROWS;
    for (int g = 0; g < tiles + STAGES; ++g) {
      if (g >= STAGES) wait(&full[(g - STAGES) % STAGES], ((g - STAGES) / STAGES) & 1);
      if (g < tiles) {
        const int s = g % STAGES;
        uint8_t* dst = smem + s * STAGE;
        const int row = ((g + blockIdx.x * 7) % ntile_rows) * ROWS;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(STAGE)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                smem_u32(dst)),
            "l"(reinterpret_cast<uint64_t>(&ta)), "r"(smem_u32(&full[s])), "r"(0), "r"(row)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                smem_u32(dst + BOX)),
            "l"(reinterpret_cast<uint64_t>(&tb)), "r"(smem_u32(&full[s])), "r"(0), "r"(row)
            : "memory");
      }
    }
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static CUtensorMap make(float* base, int rows, int cols, int width, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)width, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return m;
}

template <int ROWS, int STAGES>
void run(int grid, int cols, int width) {
  const int k = 4608;
  float *a, *b;
  long long* d;
  cudaMalloc(&a, (size_t)k * cols * 4);
  cudaMalloc(&b, (size_t)k * cols * 4);
  cudaMemset(a, 0, (size_t)k * cols * 4);
  cudaMemset(b, 0, (size_t)k * cols * 4);
  cudaMalloc(&d, 8);
  CUtensorMap ta = make(a, k, cols, width, ROWS), tb = make(b, k, cols, width, ROWS);
  auto kern = k_tma<ROWS, STAGES>;
  const int sm = STAGES * 2 * ROWS * 128 + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  const int tiles = 2000;
  kern<<<grid, 32, sm>>>(ta, tb, tiles, k, d);
  kern<<<grid, 32, sm>>>(ta, tb, tiles, k, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double cyc = (double)h / tiles;
  const double bytes = 2.0 * ROWS * width * 4;
  printf("grid %3d rows %3d stages %d cols %d width %2d: %7.1f cyc/tile, %5.1f B/clk/SM (global bytes)  %s\n", grid,
         ROWS, STAGES, cols, width, cyc, bytes / cyc, cudaGetErrorString(e));
  cudaFree(a);
  cudaFree(b);
  cudaFree(d);
}

int main() {
  run<192, 4>(148, 24, 24);
  run<192, 4>(148, 32, 32);
  run<192, 4>(148, 24, 16);
  run<192, 4>(1, 32, 32);
  run<192, 4>(16, 32, 32);
  run<96, 8>(148, 32, 32);
  run<96, 8>(148, 24, 24);
  run<192, 2>(148, 32, 32);
  return 0;
}
