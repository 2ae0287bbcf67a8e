// Micro-benchmark: issue rate of back-to-back tcgen05.mma (cta_group::1, M=128) on one CTA
// per SM, for kind::tf32 with A from TMEM (TS) or shared memory (SS), and kind::f16 (SS),
// at several N.  Prints cycles per MMA and the implied flops/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_ubench tools/mma_ubench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int CWB>
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  constexpr uint64_t layout = CWB == 128 ? 2 : (CWB == 64 ? 4 : 6);
  constexpr uint64_t sbo = 8 * CWB;
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= layout << 61;
  return d;
}

template <int M, int N, int FMT>  // FMT 2 = tf32 (A,B), 0 = f16
__host__ __device__ constexpr uint32_t idesc() {
  return (1u << 4) | ((uint32_t)FMT << 7) | ((uint32_t)FMT << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok)
                 : "r"(smem_u32(bar)), "r"(parity)
                 : "memory");
}

__device__ __forceinline__ float rndf(uint32_t i) {
  i ^= i >> 16; i *= 0x7feb352dU; i ^= i >> 15; i *= 0x846ca68bU; i ^= i >> 16;
  return (float)(i & 0xFFFFFF) * (1.0f / 16777216.0f) * 20.f - 10.f;
}

template <int N, int MODE, bool RND = false>  // MODE 0 = tf32 TS, 1 = tf32 SS, 2 = f16 SS, 3 = f16 TS
__global__ void k_bench(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<float*>(smem)[i] = RND ? rndf(i + 7919u * blockIdx.x) : 0.f;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (RND && warp < 4) {  // random A in TMEM (columns 256..511), random accumulators
    for (int c = 0; c < 512; c += 8) {
      uint32_t v[8];
      for (int u = 0; u < 8; ++u) v[u] = __float_as_uint(rndf(threadIdx.x * 1000 + c + u));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                       tmem + ((uint32_t)(warp * 32) << 16) + c),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                   : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    constexpr uint32_t ID = MODE >= 2 ? idesc<128, N, 0>() : idesc<128, N, 2>();
    const uint32_t a_s = smem_u32(smem), b_s = smem_u32(smem + 32768);
    const uint64_t da = smem_desc<128>(a_s), db = smem_desc<128>(b_s);
    const uint32_t a_t = tmem + 256 + 32;  // A columns in TMEM (TS mode)
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (MODE == 0)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem),
                     "r"(a_t), "l"(db), "r"(ID), "r"(1)
                     : "memory");
      else if (MODE == 1)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(ID), "r"(1)
                     : "memory");
      else if (MODE == 3)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem),
                     "r"(a_t), "l"(db), "r"(ID), "r"(1)
                     : "memory");
      else
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(ID), "r"(1)
                     : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// Tile loop as in K1's MMA issuer with an infinitely fast epilogue: per tile wait for the
// accumulator buffer's previous use (commit of tile g-NACC), issue MPT MMAs, commit.
template <int N, int MPT, int NACC>
__global__ void k_tiles(int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[NACC];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    for (int a = 0; a < NACC; ++a) mbar_init(&bar[a], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (warp == 1) {
    constexpr uint32_t ID = idesc<128, N, 2>();
    const uint32_t b_s = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int g = 0; g < tiles; ++g) {
      const int acc = g % NACC;
      if (g >= NACC) mbar_wait(&bar[acc], ((g / NACC) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (threadIdx.x == 32) {
        const uint32_t d = tmem + acc * N;
        const uint32_t a_t = tmem + NACC * N;
#pragma unroll
        for (int m = 0; m < MPT; ++m) {
          const uint64_t db = smem_desc<128>(b_s + (m % 3) * 32);
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                       "r"(a_t + (m % 3) * 8), "l"(db), "r"(ID), "r"(m != 0 ? 1 : 0)
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[acc]))
                     : "memory");
      }
      __syncwarp();
    }
    const int last = (tiles - 1) % NACC;
    mbar_wait(&bar[last], ((tiles - 1) / NACC) & 1);
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 32) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// The same tile loop with real consumers: EPI warpgroups wait for the accumulator (tfull),
// tcgen05.ld their BN/EPI columns (x32 chunks), and release it (tempty, one arrive per warp).
template <int N, int MPT, int NACC, int EPI, bool LD>
__global__ void k_tiles_epi(int tiles, long long* out, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t tfull[NACC], tempty[NACC];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (warp == 1) {
    constexpr uint32_t ID = idesc<128, N, 2>();
    const uint32_t b_s = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int g = 0; g < tiles; ++g) {
      const int acc = g % NACC;
      mbar_wait(&tempty[acc], ((g / NACC) & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t d = tmem + acc * N;
        const uint32_t a_t = tmem + NACC * N;
#pragma unroll
        for (int m = 0; m < MPT; ++m) {
          const uint64_t db = smem_desc<128>(b_s + (m % 3) * 32);
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                       "r"(a_t + (m % 3) * 8), "l"(db), "r"(ID), "r"(m != 0 ? 1 : 0)
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&tfull[acc]))
                     : "memory");
      }
      __syncwarp();
    }
    const int last = (tiles - 1) % NACC;
    mbar_wait(&tempty[last], ((tiles - 1) / NACC) & 1);
    long long t1 = clock64();
    if (blockIdx.x == 0 && lane == 0) out[0] = t1 - t0;
  } else if (warp >= 4 && warp < 4 + 4 * EPI) {
    const int wg = (warp - 4) >> 2, q = warp & 3;
    constexpr int COLS = N / EPI;
    int accum = 0;
    for (int g = 0; g < tiles; ++g) {
      const int acc = g % NACC;
      mbar_wait(&tfull[acc], (g / NACC) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (LD) {
        const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + acc * N + wg * COLS;
#pragma unroll
        for (int c = 0; c < COLS / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tb + c * 32, r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int e = 0; e < 32; ++e) accum = min(accum, (int)r[e]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[acc])) : "memory");
    }
    if (accum == 12345) sink[0] = accum;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// Exact K1 persist MMA pattern (3xTF32, KA=24: 2 x-steps x 3 + 1 fold), B from a 4-stage
// ring of [Pb | Ps] chunks (BN x 128 B each), A (big at A0, small at A0+24) in TMEM.
template <int N, int NACC, int A0, int STAGES>
__global__ void k_tiles_k1(int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[NACC];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  constexpr int CHUNK = N * 128, STAGE = 2 * CHUNK;
  for (int i = threadIdx.x; i < STAGES * STAGE / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = rndf(i);
  if (threadIdx.x == 0) {
    for (int a = 0; a < NACC; ++a) mbar_init(&bar[a], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (warp == 1) {
    constexpr uint32_t ID = idesc<128, N, 2>();
    long long t0 = clock64();
    for (int g = 0; g < tiles; ++g) {
      const int acc = g % NACC;
      if (g >= NACC) mbar_wait(&bar[acc], ((g / NACC) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (threadIdx.x == 32) {
        const uint32_t d = tmem + acc * N;
        const uint32_t ab = tmem + A0, as = ab + 24;
        const uint32_t bb = smem_u32(smem + (g % STAGES) * STAGE), bs = bb + CHUNK;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t dbb = smem_desc<128>(bb + ks * 32), dbs = smem_desc<128>(bs + ks * 32);
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                       "r"(as + ks * 8), "l"(dbb), "r"(ID), "r"(ks)
                       : "memory");
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                       "r"(ab + ks * 8), "l"(dbs), "r"(ID), "r"(1)
                       : "memory");
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                       "r"(ab + ks * 8), "l"(dbb), "r"(ID), "r"(1)
                       : "memory");
        }
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                     "r"(ab + 16), "l"(smem_desc<128>(bb + 64)), "r"(ID), "r"(1)
                     : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[acc]))
                     : "memory");
      }
      __syncwarp();
    }
    const int last = (tiles - 1) % NACC;
    mbar_wait(&bar[last], ((tiles - 1) / NACC) & 1);
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 32) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

__device__ __forceinline__ bool try_wait_hint(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void wait_k(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint64_t spins = 0;
  while (!try_wait_hint(addr, parity)) {
    if (++spins > (1ull << 26)) __trap();
  }
}

// k1 pattern with the kernel's control path: a producer warp keeps a STAGES-deep `full` ring
// armed (plain arrives, no data), the issuer waits tempty (committed by MMA completion) and
// full with hinted waits, commits empty + tfull per tile.
template <int N, int NACC, int STAGES, bool HINT, int ISS = 1>
__global__ void k_tiles_ctl(int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t tb[NACC], full[STAGES], empty[STAGES];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int CHUNK = N * 128, STAGE = 2 * CHUNK;
  for (int i = threadIdx.x; i < STAGES * STAGE / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = rndf(i);
  if (threadIdx.x == 0) {
    for (int a = 0; a < NACC; ++a) mbar_init(&tb[a], 1);
    for (int a = 0; a < STAGES; ++a) { mbar_init(&full[a], 1); mbar_init(&empty[a], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      for (int g = 0; g < tiles; ++g) {
        if (HINT) wait_k(&empty[stage], phase ^ 1); else mbar_wait(&empty[stage], phase ^ 1);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[stage])) : "memory");
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= 1 && warp < 1 + ISS) {
    constexpr uint32_t ID = idesc<128, N, 2>();
    long long t0 = clock64();
    for (int g = warp - 1; g < tiles; g += ISS) {
      const int stage = g % STAGES;
      const uint32_t phase = (g / STAGES) & 1;
      const int acc = g % NACC;
      if (HINT) wait_k(&tb[acc], ((g / NACC) & 1) ^ 1); else mbar_wait(&tb[acc], ((g / NACC) & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (HINT) wait_k(&full[stage], phase); else mbar_wait(&full[stage], phase);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t d = tmem + acc * N;
        const uint32_t ab = tmem + 384, as = ab + 24;
        const uint32_t bb = smem_u32(smem + stage * STAGE), bs = bb + CHUNK;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t dbb = smem_desc<128>(bb + ks * 32), dbs = smem_desc<128>(bs + ks * 32);
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                       "r"(as + ks * 8), "l"(dbb), "r"(ID), "r"(ks)
                       : "memory");
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                       "r"(ab + ks * 8), "l"(dbs), "r"(ID), "r"(1)
                       : "memory");
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                       "r"(ab + ks * 8), "l"(dbb), "r"(ID), "r"(1)
                       : "memory");
        }
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                     "r"(ab + 16), "l"(smem_desc<128>(bb + 64)), "r"(ID), "r"(1)
                     : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&empty[stage]))
                     : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&tb[acc]))
                     : "memory");
      }
      __syncwarp();
    }
    const int last = (tiles - 1) % NACC;
    mbar_wait(&tb[last], ((tiles - 1) / NACC) & 1);
    long long t1 = clock64();
    if (blockIdx.x == 0 && lane == 0 && warp == 1) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, int NACC, int STAGES, bool HINT, int ISS = 1>
void run_ctl() {
  long long* d;
  cudaMalloc(&d, 8);
  auto k = k_tiles_ctl<N, NACC, STAGES, HINT, ISS>;
  const int sm = STAGES * 2 * N * 128 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  const int tiles = 2000;
  k<<<148, 128, sm>>>(tiles, d);
  k<<<148, 128, sm>>>(tiles, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("k1 ctl N=%3d NACC=%d STAGES=%d hint=%d issuers=%d: %7.1f cyc/tile (ideal %d)  (%s)\n", N, NACC, STAGES, (int)HINT, ISS,
         (double)h / tiles, 7 * N / 2, cudaGetErrorString(e));
  cudaFree(d);
}

template <int N, int NACC, int A0, int STAGES>
void run_k1(int nthreads) {
  long long* d;
  cudaMalloc(&d, 8);
  auto k = k_tiles_k1<N, NACC, A0, STAGES>;
  const int sm = STAGES * 2 * N * 128 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  const int tiles = 2000;
  k<<<148, nthreads, sm>>>(tiles, d);
  k<<<148, nthreads, sm>>>(tiles, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("k1 pattern N=%3d NACC=%d A0=%d STAGES=%d thr=%d: %7.1f cyc/tile (ideal %d)  (%s)\n", N, NACC, A0, STAGES,
         nthreads, (double)h / tiles, 7 * N / 2, cudaGetErrorString(e));
  cudaFree(d);
}

template <int N, int MPT, int NACC, int EPI, bool LD>
void run_tiles_epi() {
  long long* d;
  int* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 4);
  auto k = k_tiles_epi<N, MPT, NACC, EPI, LD>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int tiles = 2000;
  k<<<148, 128 + 128 * EPI, 64 * 1024>>>(tiles, d, sink);
  k<<<148, 128 + 128 * EPI, 64 * 1024>>>(tiles, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("tiles+epi N=%3d MMAs/tile=%d NACC=%d EPI=%d ld=%d: %7.1f cyc/tile (ideal %d)  (%s)\n", N, MPT, NACC, EPI,
         (int)LD, (double)h / tiles, MPT * N / 2, cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

// tcgen05.ld latency: one warp per lane quarter loads NLD x32 chunks and waits, repeatedly
template <int NLD>
__global__ void k_ldlat(int reps, long long* out, int* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot + ((uint32_t)(warp * 32) << 16);
  int acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint32_t v[NLD][32];
#pragma unroll
    for (int c = 0; c < NLD; ++c) tmem_ld32(tmem + c * 32 + (r & 3) * 64, v[c]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int c = 0; c < NLD; ++c) acc += (int)(v[c][0] ^ v[c][17] ^ v[c][31]);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 123456) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(512));
}

template <int NLD>
void run_ldlat() {
  long long* d;
  int* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 4);
  const int reps = 4000;
  k_ldlat<NLD><<<148, 128>>>(reps, d, sink);
  k_ldlat<NLD><<<148, 128>>>(reps, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("tcgen05.ld %d x 32x32b.x32 + wait::ld: %6.1f cycles per round trip  (%s)\n", NLD, (double)h / reps,
         cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

template <int N, int MPT, int NACC>
void run_tiles() {
  long long* d;
  cudaMalloc(&d, 8);
  auto k = k_tiles<N, MPT, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int tiles = 2000;
  k<<<148, 128, 64 * 1024>>>(tiles, d);
  k<<<148, 128, 64 * 1024>>>(tiles, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("tiles N=%3d MMAs/tile=%d NACC=%d: %7.1f cyc/tile (ideal %d)  (%s)\n", N, MPT, NACC, (double)h / tiles,
         MPT * N / 2, cudaGetErrorString(e));
  cudaFree(d);
}

template <int N, int MODE, bool RND = false>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 8);
  auto k = k_bench<N, MODE, RND>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int reps = 4096;
  k<<<148, 128, 64 * 1024>>>(reps, d);
  k<<<148, 128, 64 * 1024>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const int K = MODE >= 2 ? 16 : 8;
  const double cyc = (double)h / reps;
  printf("%-14s N=%3d: %7.1f cyc/MMA  %6.0f flops/clk/SM  (%s)\n", name, N, cyc, 2.0 * 128 * N * K / cyc,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main(int argc, char** argv) {
  if (argc > 1) {  // f16 TS (K1 3xFP16's MMA) beside tf32 TS, zero and random operands
    run<128, 0>("tf32 TS");
    run<128, 3>("f16 TS");
    run<256, 0>("tf32 TS");
    run<256, 3>("f16 TS");
    run<128, 0, true>("tf32 TS rnd");
    run<128, 3, true>("f16 TS rnd");
    run<128, 2, true>("f16 SS rnd");
    return 0;
  }
  run<128, 0>("tf32 TS");
  run<192, 0>("tf32 TS");
  run<256, 0>("tf32 TS");
  run<128, 1>("tf32 SS");
  run<192, 1>("tf32 SS");
  run<256, 1>("tf32 SS");
  run<128, 2>("f16 SS");
  run<256, 2>("f16 SS");
  run_tiles<192, 7, 2>();
  run_tiles<192, 9, 2>();
  run_tiles<128, 7, 2>();
  run_tiles<128, 7, 3>();
  run_tiles<256, 7, 1>();
  run<192, 0, true>("tf32 TS rnd");
  run<192, 1, true>("tf32 SS rnd");
  run<256, 2, true>("f16 SS rnd");
  run_tiles_epi<192, 7, 2, 3, false>();
  run_tiles_epi<192, 7, 2, 3, true>();
  run_tiles_epi<192, 7, 2, 1, true>();
  run_tiles_epi<128, 7, 2, 2, true>();
  run_k1<192, 2, 384, 1>(128);
  run_k1<192, 2, 384, 4>(128);
  run_k1<192, 2, 384, 4>(640);
  run_k1<192, 2, 416, 4>(128);
  run_ctl<192, 2, 4, false>();
  run_ctl<192, 2, 4, true>();
  run_ctl<192, 2, 4, false, 2>();
  run_ctl<192, 2, 4, true, 2>();
  run_ctl<128, 2, 4, false, 2>();
  run_ldlat<1>();
  run_ldlat<2>();
  run_ldlat<4>();
  return 0;
}
