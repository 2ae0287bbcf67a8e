// small_level.cu -- K11: the whole Lloyd loop of a small level in one cooperative launch.
//
// Upper levels are tiny (C2: 4,096 -> 256 and 256 -> 16 items, d = 16): each pass is a few
// microseconds of work, so the per-pass kernel sequence of run_level (assign, stats, sort,
// update, finalize: ~10 launches) was bound by launch latency.  This kernel runs the same
// algorithm (SURVEY §8(c) pseudo-code, the oracle's order) with grid-wide barriers between the
// phases, writing the same per-pass statistics and control words as the multi-kernel loop:
//
//   for t < T:  a <- argmin_j ||y - c_j||^2 (FP32 direct, lowest j on ties, D4)  [P:897-898]
//               J[t] = sum d^2, changed[t] = #(a != a_prev)
//               stop if t > 0 and changed[t] == 0                               (D3)
//               S_j, n_j <- sums (FP64) / counts of the members; c_j <- S_j / n_j if n_j > 0 (D5)
//               fin[2t] = max_j ||c_j' - c_j||^2, fin[2t+1] = #empty; stop if tol > 0 and
//               sqrt(fin[2t]) <= tol                                             (D3)
//   final pass: a <- argmin (stats in slot T+1)
//
// Distances are direct FP32 sums of squares (error ~ d * 2^-24 relative, far inside the
// 1e-5 parity window), so no near-tie re-check is needed.  All blocks are co-resident
// (cudaLaunchCooperativeKernel); the barrier is a counter + generation word in global memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "common.cuh"

#ifndef MASK_K11_THREADS
#define MASK_K11_THREADS 16384  // assignment threads the lanes-per-row split aims for
#endif

namespace mask {

namespace {

struct SmallArgs {
  const float* Y;
  int64_t n;
  int d;
  int64_t k;
  float* P;
  int32_t* lab;
  int32_t* prev;
  float* best;
  double* S;  // FP64 sums (atomics: the summation order varies, the FP32 mean practically never)
  int32_t* counts;
  double* J;
  unsigned long long* changed;
  uint32_t* fin;
  int* ctrl;
  unsigned* bar;  // [0] arrivals, [1] generation (zeroed before the launch)
  int T;
  double tol;
  int tpr;  // threads per row in the assignment phase (power of two <= 32)
  float* P_trace;      // MASK_TRACE_PASSES: (T+1) x k x d prototypes per pass, or nullptr
  int32_t* lab_trace;  // (T+1) x n labels per pass (slot T = the final pass)
};

__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  if (gridDim.x == 1) {  // one block: the block barrier orders its global-memory traffic
    __syncthreads();
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      uint32_t spins = 0;
      while (*gen == g) {
        __nanosleep(32);
        if (++spins > (1u << 26)) __trap();
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// block-wide sums of (double, u64) into global slots
__device__ __forceinline__ void block_stats(double s, unsigned long long c, double* J, unsigned long long* ch) {
  __shared__ double ss[32];
  __shared__ unsigned long long sc[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
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
      atomicAdd(ch, c);
    }
  }
  __syncthreads();
}

constexpr int kSmallSmemFloats = 11264;  // prototypes staged in shared memory up to 44 KB

// row-vs-all-prototypes argmin; C is shared memory (STAGED) or global memory read through L2
// (P changes inside the kernel, so no read-only-cache loads)
template <int D, bool STAGED, bool STRIDED = false>
__device__ __forceinline__ void row_argmin(const float (&x)[D], const float* C, int64_t k, int d, float& bv,
                                           int32_t& bj, int j0 = 0, int jstep = 1) {
  bv = INFINITY;
  bj = 0x7fffffff;
  if (!STRIDED) j0 = 0, jstep = 1;  // compile-time unit stride for the one-lane-per-row case
  for (int64_t j = j0; j < k; j += (STRIDED ? jstep : 1)) {
    const float* cj = C + j * d;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int e = 0; e < D; ++e) {
      if (e < d) {
        const float t = x[e] - (STAGED ? cj[e] : __ldcg(cj + e));
        acc[e & 3] = fmaf(t, t, acc[e & 3]);
      }
    }
    const float v = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    if (v < bv) {  // strict: lowest j on ties (D4)
      bv = v;
      bj = (int32_t)j;
    }
  }
}

// assignment of every row (thread per row, row in registers, prototypes broadcast from shared
// memory when they fit in 44 KB)
template <int D>
__device__ void assign_all(const SmallArgs& a, int slot, float* sP, int tslot) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool staged = a.k * a.d <= kSmallSmemFloats;
  if (a.P_trace)  // P is read-only until the next grid barrier
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.k * a.d; e += stride)
      a.P_trace[(int64_t)tslot * a.k * a.d + e] = __ldcg(a.P + e);
  if (staged)
    for (int64_t e = threadIdx.x; e < a.k * a.d; e += blockDim.x) sP[e] = __ldcg(a.P + e);
  __syncthreads();
  double s = 0.0;
  unsigned long long c = 0;
  // a.tpr consecutive lanes per row (power of two <= 32): lane h of a row scans prototypes
  // h, h + tpr, ... (lowest index on ties within its subset), then the lanes combine by
  // (value, index) -- the same argmin with more threads on the prototypes
  const int S = a.tpr;
  const int lane = threadIdx.x & 31, h = lane & (S - 1);
  const int64_t total = a.n * S;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) - lane;
  for (int64_t base = warp0; base < total; base += stride) {
    const int64_t t = base + lane;
    const bool valid = t < total;
    const int64_t i = valid ? t / S : 0;
    float bv = INFINITY;
    int32_t bj = 0x7fffffff;
    if (valid) {
      float x[D];
#pragma unroll
      for (int e = 0; e < D; ++e) x[e] = e < a.d ? __ldg(a.Y + i * a.d + e) : 0.f;
      if (S == 1) {
        if (staged) row_argmin<D, true>(x, sP, a.k, a.d, bv, bj);
        else row_argmin<D, false>(x, a.P, a.k, a.d, bv, bj);
      } else {
        if (staged) row_argmin<D, true, true>(x, sP, a.k, a.d, bv, bj, h, S);
        else row_argmin<D, false, true>(x, a.P, a.k, a.d, bv, bj, h, S);
      }
    }
    for (int o = 1; o < S; o <<= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int32_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ov < bv || (ov == bv && oj < bj)) {
        bv = ov;
        bj = oj;
      }
    }
    if (valid && h == 0) {
      a.lab[i] = bj;
      if (a.lab_trace) a.lab_trace[(int64_t)tslot * a.n + i] = bj;
      a.best[i] = bv;
      s += (double)bv;
      c += (bj != __ldcg(a.prev + i)) ? 1ull : 0ull;
    }
  }
  block_stats(s, c, a.J + slot, a.changed + slot);
}

template <int D>
__global__ void __launch_bounds__(256) k_small_level(SmallArgs a) {
  __shared__ float sP[kSmallSmemFloats];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int64_t warps = stride >> 5, wid = tid >> 5;
  int t = 0;
  for (; t < a.T; ++t) {
    assign_all<D>(a, t, sP, t);
    grid_barrier(a.bar);
    if (t > 0 && *(volatile unsigned long long*)(a.changed + t) == 0) {  // no label changed: stop
      if (tid == 0) {
        a.ctrl[0] = 0;
        a.ctrl[1] = t + 1;
      }
      break;
    }
    // ---- update: S_j, n_j
    for (int64_t i = tid; i < a.n; i += stride) {
      const int32_t j = __ldcg(a.lab + i);
      double* Sj = a.S + (int64_t)j * a.d;
      for (int e = 0; e < a.d; ++e) atomicAdd(Sj + e, (double)__ldg(a.Y + i * a.d + e));
      atomicAdd(a.counts + j, 1);
      a.prev[i] = j;
    }
    grid_barrier(a.bar);
    // ---- finalize: warp per prototype (IEEE division, empty clusters keep, D5)
    for (int64_t j = wid; j < a.k; j += warps) {
      const int32_t cnt = __ldcg(a.counts + j);
      float disp = 0.f;
      if (cnt > 0) {
        for (int e = lane; e < a.d; e += 32) {
          const float cv = (float)(__ldcg(a.S + j * a.d + e) / (double)cnt);
          const float df = cv - a.P[j * a.d + e];
          disp = fmaf(df, df, disp);
          a.P[j * a.d + e] = cv;
          a.S[j * a.d + e] = 0.0;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) disp += __shfl_xor_sync(0xffffffffu, disp, o);
      if (lane == 0) {
        atomicMax(a.fin + 2 * t, __float_as_uint(disp));
        if (cnt == 0) atomicAdd(a.fin + 2 * t + 1, 1u);
        a.counts[j] = 0;
      }
    }
    grid_barrier(a.bar);
    const double disp = sqrt((double)__uint_as_float(*(volatile uint32_t*)(a.fin + 2 * t)));
    if (a.tol > 0.0 && disp <= a.tol) {  // D3 tolerance stop
      if (tid == 0) {
        a.ctrl[0] = 0;
        a.ctrl[1] = t + 1;
      }
      break;
    }
    if (t == a.T - 1 && tid == 0) a.ctrl[1] = a.T;
  }
  // ---- final assignment with the final prototypes (stats slot T+1)
  assign_all<D>(a, a.T + 1, sP, a.T);
}

}  // namespace

// Fused only where it wins: prototypes staged in shared memory, and little enough work per pass
// that launch latency (not the SIMT distance loop) dominated the per-pass kernels.
bool small_level_supported(int64_t n, int d, int64_t k) {
  return n >= 1 && n <= 65536 && d >= 1 && d <= 64 && k >= 1 && k * d <= kSmallSmemFloats &&
         n * k * d <= ((int64_t)1 << 25);
}

void launch_small_level(const float* Y, int64_t n, int d, int64_t k, float* P, int32_t* lab, int32_t* prev,
                        float* best, double* S, int32_t* counts, double* J, unsigned long long* changed,
                        uint32_t* fin, int* ctrl, unsigned* bar_ws, int T, double tol, cudaStream_t st,
                        float* P_trace, int32_t* lab_trace) {
  SmallArgs a{Y, n, d, k, P, lab, prev, best, S, counts, J, changed, fin, ctrl, bar_ws, T, tol, 1, P_trace, lab_trace};
  MASK_CUDA(cudaMemsetAsync(bar_ws, 0, 2 * sizeof(unsigned), st));
  void* fn;
  if (d <= 4) fn = (void*)k_small_level<4>;
  else if (d <= 8) fn = (void*)k_small_level<8>;
  else if (d <= 16) fn = (void*)k_small_level<16>;
  else if (d <= 32) fn = (void*)k_small_level<32>;
  else fn = (void*)k_small_level<64>;
  int per_sm = 0;
  MASK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
  MASK_REQUIRE(per_sm >= 1, MASK_ERR_CUDA, "small-level kernel cannot be resident");
  // enough blocks for the rows (and the prototypes in the finalize phase), all co-resident
  int64_t want = (std::max<int64_t>(n, k * 32) + 255) / 256;
  // spread each row's prototype scan over tpr lanes until ~16K threads work on the assignment
  // (C2 level 2: 4,096 rows x 256 prototypes -> 4 lanes per row, 64 blocks)
  if (want > 1) {
    while (a.tpr < 32 && n * a.tpr * 2 <= MASK_K11_THREADS && a.tpr * 2 <= k) a.tpr *= 2;
    want = std::max<int64_t>(want, (n * a.tpr + 255) / 256);
  }
  const int64_t cap = (int64_t)per_sm * num_sms();
  const int grid = (int)std::max<int64_t>(1, std::min(want, cap));
  void* args[] = {&a};
  MASK_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(256), args, 0, st));
  MASK_LAUNCH_CHECK();
}

}  // namespace mask
