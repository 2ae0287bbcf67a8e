// assign_tc.cu -- K1: dense assignment on the 5th-generation tensor cores (sm_100a).
//
// For a block of BM = 128 points x_i and every prototype c_j (PAPER.md P:897-898,
// `euclideanDistance` + `searchPosMin`):
//
//     s_ij = ||c_j||^2 - 2 x_i . c_j        a_i = argmin_j s_ij  (lowest j on ties, D4)
//
// (||x_i||^2 is a row constant: it does not move the argmin and is added to the winner
// only: d^2_i = s_i + ||x_i||^2.)  The contraction x . (-2c) runs as 3xTF32 on tcgen05.mma
// kind::tf32 with FP32 accumulation in TMEM:
//
//     x = xb + xs, (-2c) = cb + cs  (xb = rn_tf32(x), xs = rn_tf32(x - xb), same for c)
//     x.(-2c) ~= xs.cb + xb.cs + xb.cb        (representation error <= 2^-22 |x| per term)
//
// Data movement and roles (one CTA per 128-row block, 8 warps):
//   warp 0   TMA producer: the 128 x d A block once (SWIZZLE_128B / 64B K-major chunks of
//            CW fp32 columns), then the B operand (prototype tiles of BN rows, big and small
//            parts) chunk by chunk through a STAGES-deep mbarrier ring;
//   warp 1   MMA issuer (one thread): per K step of 8, three tcgen05.mma into the TMEM
//            accumulator of the current tile; tcgen05.commit frees the smem stage and, after
//            the last chunk of a tile, signals the epilogue; the accumulator is
//            double-buffered (2 x BN TMEM columns) so tile t+1's MMAs overlap tile t's epilogue;
//   warp 2   TMEM allocator;
//   warps 4-7 split the A block in place into (xb, xs) once, then run the epilogue: each
//            thread owns one row (TMEM lane), loads 32 accumulator columns at a time
//            (tcgen05.ld 32x32b.x32), adds ||c_j||^2 and keeps the running best / second-best
//            (value, index).  At the end: label, d^2 = s1 + ||x||^2, and a near-tie flag when
//            s2 - s1 is within the worst-case 3xTF32 error bound (those rows are recomputed
//            exactly by K4).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <cmath>
#include <cstring>
#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "tcgen05.cuh"  // BM, mbarrier / TMA / UMMA / TMEM helpers (mask::tc)


namespace mask {

namespace tc {


// Top-2 of one 32-column chunk of packed keys (bits & mask) | column, in two passes over the
// registers instead of a running top-2 per element (K1 "epilogue"):
//   pass 1: c1 = min_e key_e                                    (3-input mins: 1 ALU op / 2 keys)
//   pass 2: c2 = c1 + 1 + min_e (key_e - c1 - 1) as unsigned    (the minimum itself wraps to
//           0xFFFFFFFF; keys are distinct because they carry the column, so this is the
//           second-smallest key exactly)
// The subtraction is an IMAD (key * one + ~c1, `one` = 1 from a register the compiler cannot
// fold) so it issues on the FMA pipe: the ALU pipe sees 1 LOP3 + 1 three-input min per key,
// against 1 LOP3 + 2.5 min/max per key for the running top-2.
__device__ __forceinline__ void chunk_top2(uint32_t* r, uint32_t mask, uint32_t colbase, uint32_t one, int32_t& c1,
                                           int32_t& c2) {
#pragma unroll
  for (int e = 0; e < 32; ++e)
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r[e]) : "r"(r[e]), "r"(mask), "r"(colbase + (uint32_t)e));
  int32_t m[11];
#pragma unroll
  for (int j = 0; j < 10; ++j)
    m[j] = imin(imin((int32_t)r[3 * j], (int32_t)r[3 * j + 1]), (int32_t)r[3 * j + 2]);
  m[10] = imin((int32_t)r[30], (int32_t)r[31]);
  const int32_t a = imin(imin(m[0], m[1]), m[2]), b = imin(imin(m[3], m[4]), m[5]);
  const int32_t c = imin(imin(m[6], m[7]), m[8]), dd = imin(m[9], m[10]);
  c1 = imin(imin(a, b), imin(c, dd));
  const uint32_t nc = ~(uint32_t)c1;  // -(c1 + 1)
#pragma unroll
  for (int e = 0; e < 32; ++e) asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r[e]) : "r"(r[e]), "r"(one), "r"(nc));
  uint32_t w[11];
#pragma unroll
  for (int j = 0; j < 10; ++j) w[j] = umin(umin(r[3 * j], r[3 * j + 1]), r[3 * j + 2]);
  w[10] = umin(r[30], r[31]);
  const uint32_t ua = umin(umin(w[0], w[1]), w[2]), ub = umin(umin(w[3], w[4]), w[5]);
  const uint32_t uc = umin(umin(w[6], w[7]), w[8]), ud = umin(w[9], w[10]);
  c2 = (int32_t)(umin(umin(ua, ub), umin(uc, ud)) - nc);
}

// Top-3 of a chunk: chunk_top2, then one more pass over the registers (which then hold
// key - c1 - 1, wrapped): key - c2 - 1 = r - (c2 - c1) is the smallest for the third key (c1's and
// c2's own entries wrap to the top), so c3 = c2 + 1 + min.  Only keyed chunks pay for it.
__device__ __forceinline__ void chunk_top3(uint32_t* r, uint32_t mask, uint32_t colbase, uint32_t one, int32_t& c1,
                                           int32_t& c2, int32_t& c3) {
  chunk_top2(r, mask, colbase, one, c1, c2);
  const uint32_t delta = (uint32_t)c2 - (uint32_t)c1;
  uint32_t w[11];
#pragma unroll
  for (int j = 0; j < 10; ++j)
    w[j] = umin(umin(r[3 * j] - delta, r[3 * j + 1] - delta), r[3 * j + 2] - delta);
  w[10] = umin(r[30] - delta, r[31] - delta);
  const uint32_t ua = umin(umin(w[0], w[1]), w[2]), ub = umin(umin(w[3], w[4]), w[5]);
  const uint32_t uc = umin(umin(w[6], w[7]), w[8]), ud = umin(w[9], w[10]);
  c3 = (int32_t)((uint32_t)c2 + 1u + umin(umin(ua, ub), umin(uc, ud)));
}

// merge a chunk's (c1 < c2) into a running (b1 <= b2)
__device__ __forceinline__ void merge_top2(int32_t& b1, int32_t& b2, int32_t c1, int32_t c2) {
  b2 = imin(imin(b2, c2), imax(b1, c1));
  b1 = imin(b1, c1);
}

// development trace (MASK_TC_DEBUG bit 8): %globaltimer stamps of the first CTAs
constexpr int kTraceCtas = 4096;
__device__ long long g_tc_trace[8][kTraceCtas];
constexpr int kPT = 512;
__device__ long long g_pt[9][kPT];
// per-tile trace stamps (development builds with -DMASK_TC_TRACE only)
#if defined(MASK_TC_TRACE)
#define PT_STAMP(cond, row, idx) \
  do {                           \
    if (cond) g_pt[row][idx] = clock64(); \
  } while (0)
#else
#define PT_STAMP(cond, row, idx) \
  do {                           \
    (void)(cond);                \
  } while (0)
#endif
__device__ unsigned long long g_chunk_stats[4];  // debug bit 128: chunks seen / keyed
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Kernel configuration.
//   CW / NKC   K columns per smem chunk of B (32 fp32 = one 128-byte swizzle row) / chunks
//   KA         K columns of the contraction (d, or d + 2 with FOLD), multiple of 8
//   BN         prototypes per tile (MMA N);  NACC TMEM accumulator buffers
//   FOLD       ||x||^2 and ||c||^2 folded into the contraction (small d), packed-key epilogue
//   EPI_WG     epilogue warpgroups (each owns BN / EPI_WG accumulator columns of every tile)
// TMEM: [NACC x BN accumulator columns][KA columns A_big][KA columns A_small]; A lives in TMEM
// (lane = row, column = k), so the tensor core reads only B from shared memory.
template <int CW, int NKC, int KA, int BN, int STAGES, int NACC, bool FOLD, int EPI_WG>
struct Cfg {
  static constexpr int CWB = CW * 4;
  static constexpr int B_CHUNK = BN * CWB;
  static constexpr int STAGE_BYTES = 2 * B_CHUNK;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int NBARS = 2 * STAGES + 2 * NACC + 1;
  static constexpr int SMEM = BAR_OFF + NBARS * 8 + 16 + 1024;  // + alignment slack
  static constexpr int A_COL = NACC * BN;
  static constexpr int AS_COL = A_COL + KA;
  static constexpr int NEED = AS_COL + KA;
  static constexpr int TMEM_COLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static constexpr uint32_t IDESC = idesc_tf32<BM, BN>();
  static constexpr int NTHREADS = 128 + 128 * EPI_WG;
  static_assert(NEED <= 512, "TMEM budget");
  static_assert(KA % 8 == 0 && KA <= NKC * CW, "K layout");
  static_assert(SMEM <= 232448, "shared memory budget");
  static_assert(3 * BM * 4 * EPI_WG <= STAGES * STAGE_BYTES, "merge scratch");
};

template <int CW, int NKC, int KA, int BN, int STAGES, int NACC, bool FOLD, int EPI_WG>
__global__ void __launch_bounds__(128 + 128 * EPI_WG, 1)
    k_assign_tc(const __grid_constant__ CUtensorMap tmBb, const __grid_constant__ CUtensorMap tmBs,
                const float* __restrict__ X, const float* __restrict__ P, const float* __restrict__ cn2,
                const float* __restrict__ xn2, int64_t n, int d, int64_t k, int32_t* __restrict__ labels,
                float* __restrict__ best, int32_t* __restrict__ flag_rows, int32_t* __restrict__ flag_count,
                float err_coef, int dbg,
                const int* __restrict__ active, int2* __restrict__ flag_pair) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
#if !defined(MASK_TC_ABLATE)
  dbg = 0;  // development ablations / trace only in -DMASK_TC_ABLATE builds
#endif
  using C = Cfg<CW, NKC, KA, BN, STAGES, NACC, FOLD, EPI_WG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Bst = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + NACC;
  uint64_t* a_ready = bars + 2 * STAGES + 2 * NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBARS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (int64_t)blockIdx.x * BM;
  const int ntiles = (int)((k + BN - 1) / BN);
  const bool trace = (dbg & 8) && blockIdx.x < kTraceCtas;
  if (trace && threadIdx.x == 0) g_tc_trace[0][blockIdx.x] = gtimer();

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmBb);
    prefetch_tmap(&tmBs);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * EPI_WG * kArrivePerWarp);
    }
    mbar_init(a_ready, 4 * kArrivePerWarp);
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (trace && threadIdx.x == 0) g_tc_trace[1][blockIdx.x] = gtimer();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (B only)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < ntiles; ++t) {
        for (int c = 0; c < NKC; ++c) {
          mbar_wait_spin(&empty[stage], phase ^ 1);
          uint8_t* dst = Bst + stage * C::STAGE_BYTES;
          if (dbg & 4) {  // ablation: no B traffic
            mbar_arrive(&full[stage]);
          } else {
            mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
            tma_load_2d(dst, &tmBb, &full[stage], c * CW, t * BN);
            tma_load_2d(dst + C::B_CHUNK, &tmBs, &full[stage], c * CW, t * BN);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 || warp == 3) {
    // ------------------------------------------------------------ MMA issuers (A from TMEM)
    // warp 1 issues the even tiles, warp 3 the odd ones (see the persistent kernel: the second
    // issuer hides the per-tile control path behind the tensor core's short queue)
    const int par = warp == 1 ? 0 : 1;
    mbar_wait_spin(a_ready, 0);
    tc_fence_after();
    for (int t = par; t < ntiles; t += 2) {
      const int acc = t % NACC;
      mbar_wait_spin(&tempty[acc], ((t / NACC) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
      for (int c = 0; c < NKC; ++c) {
        const int gc = t * NKC + c;  // global chunk index: ring slot and phase
        const int stage = gc % STAGES;
        const uint32_t phase = (uint32_t)((gc / STAGES) & 1);
        mbar_wait_spin(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t bb = smem_u32(Bst + stage * C::STAGE_BYTES);
          const uint32_t bs = bb + C::B_CHUNK;
          const int ks_n = (c == NKC - 1) ? (KA - (NKC - 1) * CW) / 8 : CW / 8;
          for (int ks = 0; ks < ks_n; ++ks) {
            if (dbg & 2) continue;  // ablation: no MMA
            const uint32_t kcol = (uint32_t)(c * CW + ks * 8);
            const uint32_t ab = tmem_base + C::A_COL + kcol, as = tmem_base + C::AS_COL + kcol;
            const uint64_t dbb = smem_desc<C::CWB>(bb + ks * 32), dbs = smem_desc<C::CWB>(bs + ks * 32);
            mma_tf32_ts(d_tmem, as, dbb, C::IDESC, (c | ks) != 0);
            mma_tf32_ts(d_tmem, ab, dbs, C::IDESC, 1u);
            mma_tf32_ts(d_tmem, ab, dbb, C::IDESC, 1u);
          }
          mma_commit(&empty[stage]);
          if (c == NKC - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= kEpiWarp0) {
    constexpr int NEPI = 128 * EPI_WG;
    constexpr int COLS = BN / EPI_WG;
    static_assert(COLS % 32 == 0, "epilogue chunking");
    static_assert(!FOLD, "small d runs the persistent kernel");
    const int et = threadIdx.x - kEpiWarp0 * 32;
    const int wg = et >> 7;
    const int q = warp & 3;          // TMEM lane quarter
    const int rloc = q * 32 + lane;  // row of this thread inside the block
    const int64_t row = row0 + rloc;
    const float xx = row < n ? __ldg(xn2 + row) : 0.f;
    const bool tr0 = trace && et == 0;
    // ------------------------------------------------------------ A -> TMEM (warpgroup 0)
    if (wg == 0) {
      const float* xr = X + row * d;
      const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int g = 0; g < KA; g += 8) {
        uint32_t vb[8], vs[8];
#pragma unroll
        for (int u = 0; u < 8; u += 4) {
          const int col = g + u;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (row < n && col < d) v = __ldg(reinterpret_cast<const float4*>(xr + col));
          const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const float x = e[w];
            const float b = tf32_rn(x);
            vb[u + w] = __float_as_uint(b);
            vs[u + w] = __float_as_uint(tf32_rn(x - b));
          }
        }
        tmem_st8(lane_base + C::A_COL + g, vb);
        tmem_st8(lane_base + C::AS_COL + g, vs);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive_warp(a_ready);
    }
    if (tr0) g_tc_trace[2][blockIdx.x] = gtimer();

    // ------------------------------------------------------------ epilogue
    float g1 = INFINITY, g2 = INFINITY;
    int32_t gi = 0x7fffffff;
    for (int t = 0; t < ntiles; ++t) {
      const int acc = t % NACC;
      // one polling warp per warpgroup, the others on a named barrier (as in the persistent kernel)
      if (q == 0) mbar_wait_spin(&tfull[acc], (t / NACC) & 1);
      asm volatile("bar.sync %0, 128;" ::"r"(2 + wg) : "memory");
      tc_fence_after();
      if (tr0 && t == 0) g_tc_trace[3][blockIdx.x] = gtimer();
      if (tr0 && t == ntiles - 1) g_tc_trace[4][blockIdx.x] = gtimer();
      const int col0 = wg * COLS;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + col0);
      float v1, v2;
      int32_t j1;
      const bool no_ld = dbg & 16;  // ablation: no TMEM loads
      uint32_t r[2][32];
      {
        float b1[4], b2[4];
        int32_t i1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          b1[u] = b2[u] = INFINITY;
          i1[u] = 0;
        }
        if (!no_ld) tmem_ld32(tbase, r[0]);
#pragma unroll
        for (int cc = 0; cc < COLS / 32; ++cc) {
          if (!no_ld) {
            tmem_wait_ld();
            if (cc + 1 < COLS / 32) tmem_ld32(tbase + (cc + 1) * 32, r[(cc + 1) & 1]);
          }
          if (dbg & 1) continue;
          const float4* c4 = reinterpret_cast<const float4*>(cn2 + t * BN + col0 + cc * 32);
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 cv = __ldg(c4 + (i >> 2));
            const float cvv[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float s = __uint_as_float(r[cc & 1][i + u]) + cvv[u];
              const bool lt = s < b1[u];
              b2[u] = fminf(b2[u], fmaxf(b1[u], s));
              b1[u] = fminf(b1[u], s);
              i1[u] = lt ? (cc * 32 + i + u) : i1[u];
            }
          }
        }
        tc_fence_before();
        mbar_arrive_warp(&tempty[acc]);
        v1 = b1[0];
        j1 = i1[0];
#pragma unroll
        for (int u = 1; u < 4; ++u)
          if (b1[u] < v1 || (b1[u] == v1 && i1[u] < j1)) {
            v1 = b1[u];
            j1 = i1[u];
          }
        v2 = INFINITY;
#pragma unroll
        for (int u = 0; u < 4; ++u) v2 = fminf(v2, (b1[u] == v1 && i1[u] == j1) ? b2[u] : b1[u]);
        j1 += col0;
      }
      if (v1 < g1) {  // strict: ties keep the earlier tile (lower prototype index)
        g2 = fminf(g1, v2);
        g1 = v1;
        gi = t * BN + j1;
      } else {
        g2 = fminf(g2, v1);
      }
    }
    // ---- merge the warpgroups' results for each row (lowest index on equal values)
    if (EPI_WG > 1) {
      // scratch [EPI_WG-1][BM] x {g1, g2, gi} in the B stage ring: every MMA (and so every
      // TMA write) has completed once the last tile's accumulator was signalled full
      float* mg1 = reinterpret_cast<float*>(Bst);
      float* mg2 = mg1 + (EPI_WG - 1) * BM;
      int32_t* mgi = reinterpret_cast<int32_t*>(mg2 + (EPI_WG - 1) * BM);
      if (wg > 0) {
        mg1[(wg - 1) * BM + rloc] = g1;
        mg2[(wg - 1) * BM + rloc] = g2;
        mgi[(wg - 1) * BM + rloc] = gi;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(NEPI) : "memory");
      if (wg == 0) {
#pragma unroll
        for (int w = 0; w < EPI_WG - 1; ++w) {
          const float o1 = mg1[w * BM + rloc], o2 = mg2[w * BM + rloc];
          const int32_t oi = mgi[w * BM + rloc];
          if (o1 < g1 || (o1 == g1 && oi < gi)) {
            g2 = fminf(g1, o2);
            g1 = o1;
            gi = oi;
          } else {
            g2 = fminf(g2, o1);
          }
        }
      }
    }
    if (tr0) g_tc_trace[5][blockIdx.x] = gtimer();
    if (wg == 0) {
      bool flag = false;
      if (row < n) {
        if (dbg) gi = gi < 0 ? 0 : (gi >= k ? (int32_t)(k - 1) : gi);  // ablation runs: keep in range
        labels[row] = gi;
        // exact FP32 squared distance of the chosen prototype (direct form, for J and d2_out)
        const float* xr = X + row * d;
        const float* cr = P + (int64_t)gi * d;
        float dd = 0.f;
        for (int i = 0; i < d; i += 4) {
          const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + i));
          const float4 cv = __ldg(reinterpret_cast<const float4*>(cr + i));
          float tt = xv.x - cv.x;
          dd = fmaf(tt, tt, dd);
          tt = xv.y - cv.y;
          dd = fmaf(tt, tt, dd);
          tt = xv.z - cv.z;
          dd = fmaf(tt, tt, dd);
          tt = xv.w - cv.w;
          dd = fmaf(tt, tt, dd);
        }
        best[row] = dd;
        const float cc2 = __ldg(cn2 + gi);
        float thr = err_coef * (xx + cc2);
        flag = (g2 - g1) <= thr;
      }
      const unsigned m = __ballot_sync(0xffffffffu, flag);
      if (m) {
        int base = 0;
        if (lane == 0) base = atomicAdd(flag_count, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (flag) {
          const int pos = base + __popc(m & ((1u << lane) - 1));
          flag_rows[pos] = (int32_t)row;
          if (flag_pair) flag_pair[pos] = make_int2(gi, -1);  // (no third bound: full re-check)
        }
      }
    }
    if (tr0) g_tc_trace[6][blockIdx.x] = gtimer();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS));
    if (trace && lane == 0) g_tc_trace[7][blockIdx.x] = gtimer();
  }
}

// ---------------------------------------------------------------------------------------------
// Persistent variant for the folded (small-d) case.  One CTA per SM walks row blocks
// rb = blockIdx.x, blockIdx.x + gridDim.x, ...  A dedicated loader warpgroup stages the next
// block's A (split, folded columns) into the second of two TMEM A buffers while the current
// block's tiles run, so the per-block prologue (A load) and tail (merge, exact d^2, flags)
// overlap the tensor-core work instead of idling the SM.  Warps: 0 TMA producer, 1 MMA issuer,
// 2 TMEM allocator, 4-7 A loader, 8.. epilogue warpgroups.
//   FOLD  ||x||^2 + ||c||^2 enter the accumulator through one extra K step (small d); else the
//         epilogue adds them (two FADDs per score on the otherwise idle FMA pipe)
//   ABUF  TMEM A buffers (2: the next block's A is staged while the current block runs; 1 for
//         large d, where a block's thousands of tiles dwarf the A reload)
//   NKC   128-byte K chunks per prototype tile (B stage = one chunk of the big and small parts)
//   H16   3xFP16 on kind::f16 (twice the kind::tf32 rate): B and A hold FP16 big / small parts of
//         the scaled operands, 64 K columns per 128-byte chunk, K = 16 per MMA, two halves per
//         TMEM column (K1 "3xFP16")
template <int KA, int BN, int STAGES, int NACC, int EPI_WG, bool FOLD = true, int ABUF = 2, bool H16 = false>
struct PCfg {
  static constexpr int CW = H16 ? 64 : 32, CWB = 128;
  static constexpr int KSTEP = H16 ? 16 : 8;     // K per MMA
  static constexpr int ACOLS = H16 ? KA / 2 : KA;  // TMEM columns of one A part
  static constexpr int NKC = (KA + CW - 1) / CW;
  static constexpr int B_CHUNK = BN * CWB;
  static constexpr int STAGE_BYTES = 2 * B_CHUNK;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int NBARS = 2 * STAGES + 2 * NACC + 10;
  static constexpr int SCRATCH_OFF = BAR_OFF + NBARS * 8 + 16;
  // per-block results of each epilogue warpgroup {s1, s2, j1, j2, s3lb} x BM, double-buffered
  static constexpr int SCRATCH_FLOATS = 2 * 5 * BM * EPI_WG;
  static constexpr int INFO_OFF = SCRATCH_OFF + SCRATCH_FLOATS * 4;  // [2][BM] rows, bounds, ||x||^2
  static constexpr int SMEM = INFO_OFF + 6 * BM * 4 + 1024;
  static constexpr int A_COL = NACC * BN;  // A buffer b: big at A_COL + 2*ACOLS*b, small at + ACOLS
  static constexpr int NEED = A_COL + 2 * ABUF * ACOLS;
  static constexpr int TMEM_COLS = NEED <= 256 ? 256 : 512;
  static constexpr uint32_t IDESC = H16 ? idesc_f16<BM, BN>() : idesc_tf32<BM, BN>();
  static constexpr int NTHREADS = 256 + 128 * EPI_WG;
  static constexpr int EPI0 = 8;  // first epilogue warp
  static constexpr int XSTEPS = FOLD ? KA / 8 - 1 : KA / KSTEP;  // K steps of x (three MMAs each)
  static_assert(!H16 || (!FOLD && KA % 64 == 0), "3xFP16: large d, whole 64-column chunks");
  static_assert(NEED <= 512, "TMEM budget");
  static_assert(KA % 8 == 0 && KA <= NKC * CW, "K layout");
  static_assert(!FOLD || KA <= CW, "folded K fits one chunk");
  static_assert(ABUF == 1 || ABUF == 2, "A buffers");
  static_assert(SMEM <= 232448, "shared memory budget");
};

// MC = 2: the CTAs of a 2-CTA cluster walk the same prototype tiles in lockstep and each loads
// one half of every B stage (big / small part) multicast to both: half the L2 reads of B.
template <int KA, int BN, int STAGES, int NACC, int EPI_WG, bool FOLD, int ABUF, int MC = 1, bool H16 = false>
__global__ void __launch_bounds__(256 + 128 * EPI_WG, 1)
    k_assign_tc_persist(const __grid_constant__ CUtensorMap tmBb, const __grid_constant__ CUtensorMap tmBs,
                        const float* __restrict__ X, const float* __restrict__ P, const float* __restrict__ cn2,
                        const float* __restrict__ xn2, int64_t n, int d, int64_t k, int32_t* __restrict__ labels,
                        float* __restrict__ best, int32_t* __restrict__ flag_rows, int32_t* __restrict__ flag_count,
                        float err_coef, uint32_t key_mask, const int* __restrict__ active,
                        const int32_t* __restrict__ perm, const int32_t* __restrict__ prev_lab,
                        int32_t* __restrict__ lab2, int2* __restrict__ flag_pair, int dbg, float xscale,
                        float dscale, float err_abs) {
  // (H16: xscale = s scales x into FP16 range, B holds s (-2c), dscale = 1 / s^2 undoes both;
  //  err_abs = the score-gap bound's absolute term for FP16 subnormals; TF32: 1, 1, 0)
  if (active && !*active) return;  // level converged: this pass is skipped on the device
#if !defined(MASK_TC_ABLATE)
  dbg = 0;  // development ablations / counters only in -DMASK_TC_ABLATE builds (tools/build_variant.py)
#endif
  using C = PCfg<KA, BN, STAGES, NACC, EPI_WG, FOLD, ABUF, H16>;
  constexpr int COLS = BN / EPI_WG;
  // third-candidate bound for the two-candidate K4 decision: large d only (small d is epilogue-
  // bound and its few flagged rows are cheap to re-scan exactly)
  constexpr bool TRACK3 = !FOLD;
  static_assert(COLS % 32 == 0 && COLS / 32 <= 2, "epilogue chunking (two register buffers)");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Bst = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + NACC;
  uint64_t* afull = bars + 2 * STAGES + 2 * NACC;
  uint64_t* aempty = afull + 2;
  uint64_t* iempty = afull + 4;  // block info (rows, bounds) consumed by the epilogue
  uint64_t* rfull = afull + 6;   // epilogue results of a block ready for the tail
  uint64_t* rempty = afull + 8;  // tail done with a result buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBARS);
  float* scratch = reinterpret_cast<float*>(smem + C::SCRATCH_OFF);
  int32_t* s_row = reinterpret_cast<int32_t*>(smem + C::INFO_OFF);
  int32_t* s_ub = s_row + 2 * BM;
  float* s_xx = reinterpret_cast<float*>(s_ub + 2 * BM);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (int)((k + BN - 1) / BN);
  const int64_t nblocks = (n + BM - 1) / BM;
  // every CTA of a cluster runs the same number of block iterations (a CTA past the last block
  // processes a masked dummy block) so the multicast B stream stays in lockstep
  const int64_t base_cta = (int64_t)(blockIdx.x / MC) * MC;
  const int64_t iters = nblocks > base_cta ? (nblocks - base_cta + gridDim.x - 1) / gridDim.x : 0;
  const uint32_t crank = MC > 1 ? cluster_rank() : 0;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmBb);
    prefetch_tmap(&tmBs);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC);  // every CTA's MMA commit frees the stage in both CTAs
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * EPI_WG * kArrivePerWarp);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&afull[a], 4 * kArrivePerWarp);
      mbar_init(&aempty[a], ntiles >= 2 ? 2 : 1);  // one commit per MMA issuer with tiles in the block
      mbar_init(&iempty[a], 4 * EPI_WG * kArrivePerWarp);
      mbar_init(&rfull[a], 4 * EPI_WG * kArrivePerWarp);
      mbar_init(&rempty[a], 4 * kArrivePerWarp);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  if (MC > 1) cluster_sync_all();  // the partner's barriers are initialised before any multicast
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (B)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int64_t gp = 0;
      const uint64_t pol_b = l2_policy_evict_last();
      for (int64_t it = 0; it < iters; ++it) {
        for (int t = 0; t < ntiles; ++t, ++gp) {
          for (int c = 0; c < C::NKC; ++c) {
            mbar_wait_spin(&empty[stage], phase ^ 1);
            PT_STAMP((dbg & 8) && blockIdx.x == 0 && gp < kPT && c == 0, 8, gp);
            uint8_t* dst = Bst + stage * C::STAGE_BYTES;
            if (dbg & 4) {  // ablation: no B traffic
              mbar_arrive(&full[stage]);
            } else if (MC > 1) {  // this CTA's half (big or small part) to both CTAs
              mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
              if (crank == 0) tma_load_2d_mc(dst, &tmBb, &full[stage], c * C::CW, t * BN, 0x3, pol_b);
              else tma_load_2d_mc(dst + C::B_CHUNK, &tmBs, &full[stage], c * C::CW, t * BN, 0x3, pol_b);
            } else {
              mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
              tma_load_2d_hint(dst, &tmBb, &full[stage], c * C::CW, t * BN, pol_b);
              tma_load_2d_hint(dst + C::B_CHUNK, &tmBs, &full[stage], c * C::CW, t * BN, pol_b);
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1 || warp == 3) {
    // ------------------------------------------------------------ MMA issuers (two warps)
    // Warp 1 issues the even tiles, warp 3 the odd ones (accumulator g % NACC): while
    // one is blocked feeding the tensor core's instruction queue, the other has already passed
    // its barrier waits, so the per-tile control path (commits, two waits) never drains the
    // queue (a single issuer left the pipe idle ~35% of the time at d = 16).
    const int par = warp == 1 ? 0 : 1;
    int g0 = 0;       // first global tile of the block
    int i = 0;       // block iteration of this CTA
    for (int64_t it = 0; it < iters; ++it, ++i, g0 += ntiles) {
      const int first = (int)((g0 & 1) == par ? 0 : 1);  // this issuer's first tile of the block
      const int ab = i % ABUF;
      // every block's afull phase is consumed, also by an issuer without tiles in it (k <= BN):
      // with one A buffer a skipped phase would let the next parity wait pass a phase early
      mbar_wait_spin(&afull[ab], (i / ABUF) & 1);
      tc_fence_after();
      if (first >= ntiles) continue;
      const int last = first + (ntiles - 1 - first) / 2 * 2;
      const uint32_t a_big = tmem_base + C::A_COL + 2 * C::ACOLS * ab, a_small = a_big + C::ACOLS;
      for (int t = first; t < ntiles; t += 2) {
        const int g = g0 + t;
        const int acc = (int)(g % NACC);
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        mbar_wait_spin(&tempty[acc], ((g / NACC) & 1) ^ 1);
        tc_fence_after();
        const bool ptr = (dbg & 8) && blockIdx.x == 0 && lane == 0 && g < kPT;
        PT_STAMP(ptr, 0, g);
#pragma unroll
        for (int c = 0; c < C::NKC; ++c) {
          const int64_t gc = (int64_t)g * C::NKC + c;  // global chunk: ring slot and phase
          const int stage = (int)(gc % STAGES);
          const uint32_t phase = (uint32_t)((gc / STAGES) & 1);
          mbar_wait_spin(&full[stage], phase);
          tc_fence_after();
          if (c == 0) PT_STAMP(ptr, 1, g);
          if (lane == 0) {
            const uint32_t bb = smem_u32(Bst + stage * C::STAGE_BYTES);
            const uint32_t bs = bb + C::B_CHUNK;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const int s8 = c * 4 + ks;  // global K step
              if (s8 >= KA / C::KSTEP || (dbg & 2)) break;  // (dbg 2, ablation: no MMA)
              const uint64_t dbb = smem_desc<C::CWB>(bb + ks * 32);
              if constexpr (H16) {  // K step s8 = 16 halves = 8 TMEM columns, 32 bytes of B
                const uint64_t dbs = smem_desc<C::CWB>(bs + ks * 32);
                mma_f16_ts(d_tmem, a_small + s8 * 8, dbb, C::IDESC, s8 != 0);
                mma_f16_ts(d_tmem, a_big + s8 * 8, dbs, C::IDESC, 1u);
                mma_f16_ts(d_tmem, a_big + s8 * 8, dbb, C::IDESC, 1u);
              } else if (s8 < C::XSTEPS) {
                const uint64_t dbs = smem_desc<C::CWB>(bs + ks * 32);
                mma_tf32_ts(d_tmem, a_small + s8 * 8, dbb, C::IDESC, s8 != 0);
                mma_tf32_ts(d_tmem, a_big + s8 * 8, dbs, C::IDESC, 1u);
                mma_tf32_ts(d_tmem, a_big + s8 * 8, dbb, C::IDESC, 1u);
              } else {
                // fold step: ||c||^2 + ||x||^2 from exact 1-products of the split norms (one MMA)
                mma_tf32_ts(d_tmem, a_big + s8 * 8, dbb, C::IDESC, 1u);
              }
            }
            if (MC > 1) mma_commit_mc(&empty[stage], 0x3);
            else mma_commit(&empty[stage]);
            if (c == C::NKC - 1) {
              mma_commit(&tfull[acc]);
              // this issuer's MMAs on the block's A are done (aempty counts one arrive per issuer
              // that has tiles in the block)
              if (t == last) mma_commit(&aempty[ab]);
            }
          }
          __syncwarp();
        }
        PT_STAMP(ptr, 7, g);
      }
    }
  } else if (warp >= 4 && warp < C::EPI0) {
    // ------------------------------------------------------------ A loader (one thread per row)
    // Also publishes, per block, each row's index (through `perm`) and its pruning bound:
    // with the previous pass's best and second-best prototypes a1 != a2, the exact FP32
    // U = max(d^2(x, c_a1), d^2(x, c_a2)) bounds the true second-best distance, so the two
    // smallest 3xTF32 scores are <= U + (score error) and any 32-column chunk whose raw
    // minimum exceeds that bound holds neither (K1 "bound-pruned epilogue").
    // The same warpgroup runs each block's tail one block later (merge of the epilogue
    // warpgroups' top-2, labels, exact FP32 d^2 of the winner, near-tie flags), so the epilogue
    // warpgroups go straight on to the next block's tiles.
    const int q = warp & 3;
    const int rloc = q * 32 + lane;
    const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
    auto tail = [&](int ib) {  // block iteration ib of this CTA
      const int tb = ib & 1;
      mbar_wait_sleep(&rfull[tb], (ib >> 1) & 1);
      const float* r1 = scratch + tb * 5 * BM * EPI_WG;
      const float* r2 = r1 + BM * EPI_WG;
      const int32_t* ri = reinterpret_cast<const int32_t*>(r2 + BM * EPI_WG);
      const int32_t* ri2 = ri + BM * EPI_WG;
      const float* r3 = reinterpret_cast<const float*>(ri2 + BM * EPI_WG);
      float g1 = r1[rloc], g2 = r2[rloc], g3 = r3[rloc];
      int32_t gi = ri[rloc], gi2 = ri2[rloc];
#pragma unroll
      for (int w = 1; w < EPI_WG; ++w) {  // lowest index on equal values
        const float o1 = r1[w * BM + rloc], o2 = r2[w * BM + rloc], o3 = r3[w * BM + rloc];
        const int32_t oi = ri[w * BM + rloc], oi2 = ri2[w * BM + rloc];
        // third-smallest lower bound of the union (merge path of two sorted triples)
        g3 = fminf(fminf(g3, o3), fminf(fmaxf(g1, o2), fmaxf(g2, o1)));
        if (o1 < g1 || (o1 == g1 && oi < gi)) {
          if (g1 <= o2) {
            g2 = g1;
            gi2 = gi;
          } else {
            g2 = o2;
            gi2 = oi2;
          }
          g1 = o1;
          gi = oi;
        } else if (o1 < g2) {
          g2 = o1;
          gi2 = oi;
        }
      }
      const int64_t row = s_row[tb * BM + rloc];
      mbar_arrive_warp(&rempty[tb]);
      bool flag = false, pair = false;
      if (row < n) {
        if (dbg) gi = gi < 0 ? 0 : (gi >= k ? (int32_t)(k - 1) : gi);  // ablation runs: keep in range
        labels[row] = gi;
        if (lab2) lab2[row] = gi2;
        const float* xr = X + row * d;
        const float* cr = P + (int64_t)gi * d;
        float dd = 0.f;
        for (int c = 0; c < d; c += 4) {
          const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + c));
          const float4 cv = __ldg(reinterpret_cast<const float4*>(cr + c));
          float tt = xv.x - cv.x;
          dd = fmaf(tt, tt, dd);
          tt = xv.y - cv.y;
          dd = fmaf(tt, tt, dd);
          tt = xv.z - cv.z;
          dd = fmaf(tt, tt, dd);
          tt = xv.w - cv.w;
          dd = fmaf(tt, tt, dd);
        }
        best[row] = dd;
        const float xx = __ldg(xn2 + row);
        const float thr = err_coef * (xx + __ldg(cn2 + gi)) + ldexpf(fmaxf(fabsf(g2), fabsf(g1)), -14) + err_abs;
        flag = (g2 - g1) <= thr;
        // a flagged row whose every other score (lower bound g3: keyed chunks' third-smallest,
        // skipped chunks' minima) lies beyond the window (x 1.25: the window already holds twice the score error) has exactly two candidates:
        // K4 decides between them exactly, no re-scan
        pair = flag && gi2 >= 0 && gi2 < k && gi2 != gi && (g3 - g1) > 1.25f * thr;
      }
      const unsigned msk = __ballot_sync(0xffffffffu, flag);
      if (msk) {
        int base = 0;
        if (lane == 0) base = atomicAdd(flag_count, __popc(msk));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (flag) {
          const int pos = base + __popc(msk & ((1u << lane) - 1));
          flag_rows[pos] = (int32_t)row;
          if (flag_pair) flag_pair[pos] = make_int2(gi, pair ? gi2 : -1);
        }
      }
    };
    int i = 0;
    for (int64_t it = 0; it < iters; ++it, ++i) {
      const int64_t rb = blockIdx.x + it * gridDim.x;  // (>= nblocks: a masked dummy block)
      const int ab = i % ABUF;  // TMEM A buffer
      const int ib = i & 1;     // block info slot
      mbar_wait_sleep(&aempty[ab], ((i / ABUF) & 1) ^ 1);
      mbar_wait_sleep(&iempty[ib], ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      const bool ptr = (dbg & 8) && blockIdx.x == 0 && rloc == 0 && i < 512;
      PT_STAMP(ptr, 5, i);
      const int64_t pos = rb * BM + rloc;
      const int64_t row = pos < n ? (perm ? (int64_t)__ldg(perm + pos) : pos) : n;
      const float xx = row < n ? __ldg(xn2 + row) : 0.f;
      const float* xr = X + row * d;
      constexpr int KX = FOLD ? KA - 8 : KA;  // x columns (d rounded up to 8); [KX, KA) is the fold step
      float ub = INFINITY;
      if (prev_lab && row < n) {
        const int32_t a1 = __ldg(prev_lab + row), a2 = lab2[row];
        if (a1 >= 0 && a1 < k && a2 >= 0 && a2 < k && a1 != a2) {
          const float* c1 = P + (int64_t)a1 * d;
          const float* c2 = P + (int64_t)a2 * d;
          float s1 = 0.f, s2 = 0.f;
          for (int c = 0; c < d; c += 4) {
            const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + c));
            const float4 u = __ldg(reinterpret_cast<const float4*>(c1 + c));
            const float4 w = __ldg(reinterpret_cast<const float4*>(c2 + c));
            float t;
            t = xv.x - u.x; s1 = fmaf(t, t, s1); t = xv.x - w.x; s2 = fmaf(t, t, s2);
            t = xv.y - u.y; s1 = fmaf(t, t, s1); t = xv.y - w.y; s2 = fmaf(t, t, s2);
            t = xv.z - u.z; s1 = fmaf(t, t, s1); t = xv.z - w.z; s2 = fmaf(t, t, s2);
            t = xv.w - u.w; s1 = fmaf(t, t, s1); t = xv.w - w.w; s2 = fmaf(t, t, s2);
          }
          const float U = fmaxf(s1, s2);
          // ||c_j|| <= ||x|| + sqrt(U) for every j with d^2 <= U; doubled error coefficient
          const float cm = sqrtf(xx) + sqrtf(U);
          ub = (U + 2.f * err_coef * (xx + cm * cm) + err_abs) * (1.f + 0x1p-12f) + 0x1p-100f;
        }
      }
      s_row[ib * BM + rloc] = (int32_t)row;
      s_ub[ib * BM + rloc] = __float_as_int(ub);
      s_xx[ib * BM + rloc] = xx;
      if ((dbg & 32) && i >= 2) {  // ablation: keep the stale A block (no TMEM stores)
        tc_fence_before();
        mbar_arrive_warp(&afull[ab]);
        tail(i - 1);
        continue;
      }
      const uint32_t a_big = lane_base + C::A_COL + 2 * C::ACOLS * ab, a_small = a_big + C::ACOLS;
      if constexpr (H16) {
        // 16 columns of s x -> FP16 big / small parts, two halves per TMEM column
#pragma unroll 1
        for (int g16 = 0; g16 < KA; g16 += 16) {
          uint32_t vb[8], vs[8];
#pragma unroll
          for (int u = 0; u < 16; u += 4) {
            const int col = g16 + u;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row < n && col < d) v = __ldg(reinterpret_cast<const float4*>(xr + col));
            const float e[4] = {v.x * xscale, v.y * xscale, v.z * xscale, v.w * xscale};
#pragma unroll
            for (int w = 0; w < 4; w += 2) {
              const __half b0 = __float2half_rn(e[w]), b1 = __float2half_rn(e[w + 1]);
              const __half s0 = __float2half_rn(e[w] - __half2float(b0)), s1 = __float2half_rn(e[w + 1] - __half2float(b1));
              vb[(u + w) >> 1] = (uint32_t)__half_as_ushort(b0) | ((uint32_t)__half_as_ushort(b1) << 16);
              vs[(u + w) >> 1] = (uint32_t)__half_as_ushort(s0) | ((uint32_t)__half_as_ushort(s1) << 16);
            }
          }
          tmem_st8(a_big + g16 / 2, vb);
          tmem_st8(a_small + g16 / 2, vs);
        }
      } else
#pragma unroll
      for (int g8 = 0; g8 < KA; g8 += 8) {
        uint32_t vb[8], vs[8];
#pragma unroll
        for (int u = 0; u < 8; u += 4) {
          const int col = g8 + u;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (row < n && col < d) v = __ldg(reinterpret_cast<const float4*>(xr + col));
          const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const float b = tf32_rn(e[w]);
            vb[u + w] = __float_as_uint(b);
            vs[u + w] = __float_as_uint(tf32_rn(e[w] - b));
          }
        }
        if (FOLD && g8 == KX) {  // fold step: [1, 1, xx_b, xx_s] . [cn2_b, cn2_s, 1, 1] (big parts only)
          const float hb = tf32_rn(xx);
          vb[0] = vb[1] = __float_as_uint(1.0f);
          vb[2] = __float_as_uint(hb);
          vb[3] = __float_as_uint(tf32_rn(xx - hb));
          vb[4] = vb[5] = vb[6] = vb[7] = 0u;
        }
        tmem_st8(a_big + g8, vb);
        if (g8 < KX) tmem_st8(a_small + g8, vs);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive_warp(&afull[ab]);
      PT_STAMP(ptr, 6, i);
      if (i >= 1) tail(i - 1);
    }
    if (i >= 1) tail(i - 1);
  } else if (warp >= C::EPI0) {
    // ------------------------------------------------------------ epilogue warpgroups
    const int et = threadIdx.x - C::EPI0 * 32;
    const int wg = et >> 7;
    const int q = warp & 3;
    const int rloc = q * 32 + lane;
    int g = 0;
    int i = 0;
    unsigned long long st_seen = 0, st_keyed = 0;
    for (int64_t it = 0; it < iters; ++it, ++i) {
      const int ab = i % ABUF, ib = i & 1;
      mbar_wait_spin(&afull[ab], (i / ABUF) & 1);  // block info published with the A block
      const int32_t ubk = s_ub[ib * BM + rloc];
      const float xx = FOLD ? 0.f : s_xx[ib * BM + rloc];
      mbar_arrive_warp(&iempty[ib]);
      float g1 = INFINITY, g2 = INFINITY, g3 = INFINITY;  // g3: lower bound of the third-smallest
      int32_t gi = 0x7fffffff, gi2 = -1;
      int32_t smin = 0x7fffffff;  // smallest raw key of the chunks this row skipped
      for (int t = 0; t < ntiles; ++t, ++g) {
        const int acc = (int)(g % NACC);
        // polled, not suspended: the accumulator round trip (MMA -> epilogue -> MMA) must fit in
        // one tile of tensor-core work, and a suspended waiter wakes hundreds of cycles late.
        // One warp per warpgroup polls; the other three wait on a named barrier (no issue slots,
        // no traffic on the barrier unit the MMA issuers' own waits go through).
#if !defined(MASK_TC_ALL_POLL)
        if (q == 0) mbar_wait_spin(&tfull[acc], (g / NACC) & 1);
        asm volatile("bar.sync %0, 128;" ::"r"(2 + wg) : "memory");
#else
        mbar_wait_spin(&tfull[acc], (g / NACC) & 1);
#endif
        tc_fence_after();
        const bool ptr = (dbg & 8) && blockIdx.x == 0 && lane == 0 && q == 0 && g < 512;
        PT_STAMP(ptr && wg == 0, 2, g);
        const int col0 = wg * COLS;
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + col0);
        uint32_t r[2][32];
        if (dbg & 64) {  // ablation: no TMEM loads, no epilogue
          tc_fence_before();
          mbar_arrive_warp(&tempty[acc]);
          PT_STAMP(ptr && wg == 0, 3, g);
          PT_STAMP(ptr && wg == EPI_WG - 1, 4, g);
          continue;
        }
        // all of this warpgroup's columns into registers, then release the accumulator before
        // any arithmetic (the MMAs of tile g + NACC may start while this tile is reduced)
#pragma unroll
        for (int cc = 0; cc < COLS / 32; ++cc) tmem_ld32(tbase + cc * 32, r[cc]);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive_warp(&tempty[acc]);
        PT_STAMP(ptr && wg == 0, 3, g);
        PT_STAMP(ptr && wg == EPI_WG - 1, 4, g);
        // running top-2 keys of this tile; k2 starts at the pruning bound (low byte 0xFF marks
        // "no element": real keys carry a column < COLS in that byte)
        if (!FOLD) {
          // the d^2 estimate: accumulator (-2 x.c) + ||c_j||^2 + ||x||^2 (FMA pipe; cn2 is padded
          // with +inf beyond k, so pad columns never win)
#pragma unroll
          for (int cc = 0; cc < COLS / 32; ++cc) {
            const float4* c4 = reinterpret_cast<const float4*>(cn2 + (int64_t)t * BN + col0 + cc * 32);
#pragma unroll
            for (int e4 = 0; e4 < 8; ++e4) {
              const float4 cv = __ldg(c4 + e4);
              // (dscale = 1 for TF32: fmaf(D, 1, c) rounds like D + c)
              r[cc][4 * e4 + 0] = __float_as_uint(fmaf(__uint_as_float(r[cc][4 * e4 + 0]), dscale, cv.x) + xx);
              r[cc][4 * e4 + 1] = __float_as_uint(fmaf(__uint_as_float(r[cc][4 * e4 + 1]), dscale, cv.y) + xx);
              r[cc][4 * e4 + 2] = __float_as_uint(fmaf(__uint_as_float(r[cc][4 * e4 + 2]), dscale, cv.z) + xx);
              r[cc][4 * e4 + 3] = __float_as_uint(fmaf(__uint_as_float(r[cc][4 * e4 + 3]), dscale, cv.w) + xx);
            }
          }
        }
        int32_t k1 = 0x7fffffff;
        int32_t k2 = imin(ubk, __float_as_int(g2)) | 0xFF;
        // the tile's keyed elements alone (no bound marker): second smallest t2 and a lower bound t3
        // of the third (a chunk's exact top-2 (c1, c2) stands for (c1, c2, >= c2))
        int32_t t2 = 0x7fffffff, t3 = 0x7fffffff;
#pragma unroll
        for (int cc = 0; cc < COLS / 32; ++cc) {
          if (dbg & 1) {  // ablation: no epilogue arithmetic
            if (cc == 0) k1 = (int32_t)r[0][0] & 0xFFFFFF00;
            continue;
          }
#if !defined(MASK_TC_NO_PRUNE)
          // pass 0: raw minimum of the chunk (3-input mins, 0.5 ALU op per key); the chunk is
          // keyed and merged only if some row of the warp may have a key below its k2
          const uint32_t* rr = r[cc & 1];
          int32_t m[11];
#pragma unroll
          for (int j = 0; j < 10; ++j) m[j] = imin(imin((int32_t)rr[3 * j], (int32_t)rr[3 * j + 1]), (int32_t)rr[3 * j + 2]);
          m[10] = imin((int32_t)rr[30], (int32_t)rr[31]);
          const int32_t c0 = imin(imin(imin(m[0], m[1]), imin(m[2], m[3])),
                                  imin(imin(imin(m[4], m[5]), imin(m[6], m[7])), imin(imin(m[8], m[9]), m[10])));
          const bool need = __any_sync(0xffffffffu, c0 <= k2);
          if (dbg & 128) {
            ++st_seen;
            st_keyed += need ? 1 : 0;
          }
          if (!need || (dbg & 256)) {  // dbg 256 (ablation): never key
            if constexpr (TRACK3) smin = imin(smin, c0);
            continue;
          }
#endif
          int32_t c1, c2;
          if constexpr (TRACK3) {
            int32_t c3;
            chunk_top3(r[cc & 1], key_mask, (uint32_t)(cc * 32), key_mask >> 31, c1, c2, c3);
            // merge path of sorted triples (k1, t2, t3) and (c1, c2, c3) (old values on the right)
            t3 = imin(imin(t3, c3), imin(imax(k1, c2), imax(t2, c1)));
            t2 = imin(imin(t2, c2), imax(k1, c1));
          } else {
            chunk_top2(r[cc & 1], key_mask, (uint32_t)(cc * 32), key_mask >> 31, c1, c2);
          }
          merge_top2(k1, k2, c1, c2);
        }
        if constexpr (TRACK3) {  // lower bound of the block's third-smallest so far (merge path)
          const float v1 = k1 != 0x7fffffff ? __int_as_float(k1 & 0xFFFFFF00) : INFINITY;
          const float v2 = t2 != 0x7fffffff ? __int_as_float(t2 & 0xFFFFFF00) : INFINITY;
          const float v3 = t3 != 0x7fffffff ? __int_as_float(t3 & 0xFFFFFF00) : INFINITY;
          g3 = fminf(fminf(g3, v3), fminf(fmaxf(g1, v2), fmaxf(g2, v1)));
        }
        if (k1 != 0x7fffffff) {
          const float v1 = __int_as_float(k1 & 0xFFFFFF00);
          const int32_t j1 = t * BN + col0 + (k1 & 0xFF);
          const bool real2 = (k2 & 0xFF) != 0xFF;
          const float v2 = real2 ? __int_as_float(k2 & 0xFFFFFF00) : INFINITY;
          const int32_t j2 = real2 ? t * BN + col0 + (k2 & 0xFF) : -1;
          if (v1 < g1) {  // strict: ties keep the earlier tile (lower prototype index)
            if (g1 <= v2) {
              g2 = g1;
              gi2 = gi;
            } else {
              g2 = v2;
              gi2 = j2;
            }
            g1 = v1;
            gi = j1;
          } else if (v1 < g2) {
            g2 = v1;
            gi2 = j1;
          }
        }
      }
      // hand this warpgroup's per-row top-2 to the tail (loader warpgroup)
      mbar_wait_spin(&rempty[ib], ((i >> 1) & 1) ^ 1);
      float* r1 = scratch + ib * 5 * BM * EPI_WG;
      float* r2 = r1 + BM * EPI_WG;
      int32_t* ri = reinterpret_cast<int32_t*>(r2 + BM * EPI_WG);
      int32_t* ri2 = ri + BM * EPI_WG;
      float* r3 = reinterpret_cast<float*>(ri2 + BM * EPI_WG);
      r1[wg * BM + rloc] = g1;
      r2[wg * BM + rloc] = g2;
      ri[wg * BM + rloc] = gi;
      ri2[wg * BM + rloc] = gi2;
      // raw keys order as floats only when non-negative: a negative skipped minimum (a d^2 estimate
      // below 0, i.e. a row on a prototype) gives no bound
      const float sm = __int_as_float(smin);
      r3[wg * BM + rloc] = TRACK3 ? fminf(g3, smin == 0x7fffffff ? INFINITY : (sm < 0.f ? -INFINITY : sm))
                                  : -INFINITY;  // (no bound: flagged rows re-scanned)
      mbar_arrive_warp(&rfull[ib]);
    }
    if ((dbg & 128) && lane == 0) {
      atomicAdd(&g_chunk_stats[0], st_seen);
      atomicAdd(&g_chunk_stats[1], st_keyed);
    }
  }
  tc_fence_before();
  if (MC > 1) cluster_sync_all();  // no CTA leaves while its partner may still signal its barriers
  else __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS));
  }
}

// development trace of the persistent kernel (MASK_TC_DEBUG bit 8): clock64 stamps of CTA 0,
// per tile g: [0] MMA issuer past tempty, [1] past full, [2] epilogue (wg0) past tfull,
// [3] wg0 release, [4] last wg release; per block i: [5] loader start, [6] loader done
void dump_ptrace() {
  static long long h[9][kPT];
  if (cudaDeviceSynchronize() != cudaSuccess) return;
  if (cudaMemcpyFromSymbol(h, g_pt, sizeof(h)) != cudaSuccess) return;
  fprintf(stderr, "[ptrace] tile: tma_issue tempty_ok full_ok issue_done | epi_start wg0_rel last_rel (cycles rel. to full_ok of the tile)\n");
  for (int g = 40; g < 64; ++g)
    fprintf(stderr, "  %3d: %6lld %6lld %6lld %6lld | %6lld %6lld %6lld | dfull %lld\n", g, h[8][g] - h[1][g], h[0][g] - h[1][g], 0ll,
            h[7][g] - h[1][g], h[2][g] - h[1][g], h[3][g] - h[1][g], h[4][g] - h[1][g], h[1][g] - h[1][g - 1]);
  for (int i = 1; i < 6; ++i)
    fprintf(stderr, "  block %d loader start %lld dur %lld (rel. tile %d full_ok)\n", i, h[5][i] - h[1][0], h[6][i] - h[5][i], 0);
  fprintf(stderr, "  full_ok deltas tiles 1..%d:", kPT - 1);
  for (int g = 1; g < 140; ++g) fprintf(stderr, "%s%lld", g % 22 == 0 ? " | " : " ", h[1][g] - h[1][g - 1]);
  fprintf(stderr, "\n  total tiles 0..139: %lld cycles\n", h[1][139] - h[1][0]);
}

// Host dump of the development trace: per-phase medians (us) over the traced CTAs.
void dump_trace(int nctas) {
  static long long h[8][kTraceCtas];
  if (cudaDeviceSynchronize() != cudaSuccess) return;
  if (cudaMemcpyFromSymbol(h, g_tc_trace, sizeof(h)) != cudaSuccess) return;
  const int m = nctas < kTraceCtas ? nctas : kTraceCtas;
  long long t0 = h[0][0], tend = 0;
  for (int i = 0; i < m; ++i) {
    t0 = h[0][i] < t0 ? h[0][i] : t0;
    tend = h[7][i] > tend ? h[7][i] : tend;
  }
  const char* names[7] = {"setup", "A_to_tmem", "wait_first_tile", "tiles(all but last)", "last_tile+merge",
                          "outputs", "teardown"};
  fprintf(stderr, "[tc trace] %d CTAs span %.1f us; per-CTA phase medians (us):", m, (tend - t0) / 1e3);
  for (int p = 0; p < 7; ++p) {
    std::vector<long long> v;
    for (int i = 0; i < m; ++i) v.push_back(h[p + 1][i] - h[p][i]);
    std::sort(v.begin(), v.end());
    fprintf(stderr, " %s=%.2f", names[p], v[v.size() / 2] / 1e3);
  }
  std::vector<long long> tot;
  for (int i = 0; i < m; ++i) tot.push_back(h[7][i] - h[0][i]);
  std::sort(tot.begin(), tot.end());
  fprintf(stderr, " total=%.2f\n", tot[tot.size() / 2] / 1e3);
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  MASK_REQUIRE(fn != nullptr, MASK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2-D fp32 row-major [rows x cols] tensor map with a {box_cols x box_rows} box.
// `width` <= cols limits the columns actually read (the rest of the box is zero-filled by the
// TMA unit without memory traffic).
CUtensorMap make_map(const float* base, int64_t rows, int cols, int box_cols, int box_rows, int width) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)(width > 0 ? width : cols), (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = box_cols * 4 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : box_cols * 4 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                     : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MASK_REQUIRE(r == CUDA_SUCCESS, MASK_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

CUtensorMap make_map16(const void* base, int64_t rows, int cols, int box_cols, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  MASK_REQUIRE(box_cols * 2 == 128, MASK_ERR_CUDA, "make_map16: 128-byte rows only");
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MASK_REQUIRE(r == CUDA_SUCCESS, MASK_ERR_CUDA, "cuTensorMapEncodeTiled (fp16) failed (" + std::to_string((int)r) + ")");
  return m;
}

#ifndef MASK_TC_EPI_WG
#define MASK_TC_EPI_WG 4
#endif

// development ablations (MASK_TC_DEBUG bits: 1 = no epilogue math, 2 = no MMA, 4 = no B loads,
// 8 = phase trace, 16 = no TMEM loads)
inline int tc_debug_mode() {
  static int mode = [] {
    const char* e = getenv("MASK_TC_DEBUG");
    return e ? atoi(e) : 0;
  }();
  return mode;
}

template <int CW, int NKC, int KA, int BN, int STAGES, int NACC, bool FOLD, int EPI_WG>
void launch_cfg(const float* X, int64_t n, int d, int kc, int64_t k_rows, const float* P, const float* Pb,
                const float* Ps, const float* cn2, int64_t k, const float* xn2, int32_t* labels, float* best,
                int32_t* flag_rows, int32_t* flag_count, float err_coef, cudaStream_t st,
                const int* active, int2* flag_pair) {
  using C = Cfg<CW, NKC, KA, BN, STAGES, NACC, FOLD, EPI_WG>;
  const CUtensorMap tBb = make_map(Pb, k_rows, kc, CW, BN);
  const CUtensorMap tBs = make_map(Ps, k_rows, kc, CW, BN);
  auto kern = k_assign_tc<CW, NKC, KA, BN, STAGES, NACC, FOLD, EPI_WG>;
  static bool attr_set = false;
  if (!attr_set) {
    MASK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  const unsigned grid = (unsigned)((n + BM - 1) / BM);
  kern<<<grid, C::NTHREADS, C::SMEM, st>>>(tBb, tBs, X, P, cn2, xn2, n, d, k, labels, best, flag_rows, flag_count,
                                           err_coef, tc_debug_mode(), active, flag_pair);
  MASK_LAUNCH_CHECK();
  if (tc_debug_mode() & 8) dump_trace((int)grid);
}

template <int KA, int BN, int STAGES, int NACC, int EPI_WG, bool FOLD = true, int ABUF = 2, int MC = 1,
          bool H16 = false>
void launch_persist(const float* X, int64_t n, int d, int kc, int64_t k_rows, const float* P, const void* Pb,
                    const void* Ps, const float* cn2, int64_t k, const float* xn2, int32_t* labels, float* best,
                    int32_t* flag_rows, int32_t* flag_count, float err_coef, cudaStream_t st, const int* active,
                    const int32_t* perm, const int32_t* prev_lab, int32_t* lab2, int2* flag_pair,
                    float xscale = 1.f, float dscale = 1.f, float err_abs = 0.f) {
  using C = PCfg<KA, BN, STAGES, NACC, EPI_WG, FOLD, ABUF, H16>;
  CUtensorMap tBb, tBs;
  if constexpr (H16) {  // FP16 [k_rows x KA] big / small parts
    tBb = make_map16(Pb, k_rows, KA, C::CW, BN);
    tBs = make_map16(Ps, k_rows, KA, C::CW, BN);
  } else {
    tBb = make_map(static_cast<const float*>(Pb), k_rows, kc, C::CW, BN);
    // the small part is only read by the x steps (KA - 8 columns); the fold step uses Pb alone
#if defined(MASK_TC_PS_TRIM)
    tBs = make_map(static_cast<const float*>(Ps), k_rows, kc, C::CW, BN, FOLD ? KA - 8 : 0);
#else
    tBs = make_map(static_cast<const float*>(Ps), k_rows, kc, C::CW, BN);
#endif
  }
  auto kern = k_assign_tc_persist<KA, BN, STAGES, NACC, EPI_WG, FOLD, ABUF, MC, H16>;
  static bool attr_set = false;
  if (!attr_set) {
    MASK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    if (MC > 1) MASK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
    attr_set = true;
  }
  const int64_t nblocks = (n + BM - 1) / BM;
  unsigned grid = (unsigned)(nblocks < num_sms() ? nblocks : num_sms());
  if (MC > 1) {
    grid = (grid + MC - 1) / MC * MC;  // whole clusters (a CTA without blocks runs masked dummies)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(C::NTHREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = MC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MASK_CUDA(cudaLaunchKernelEx(&cfg, kern, tBb, tBs, X, P, cn2, xn2, n, d, k, labels, best, flag_rows, flag_count,
                                 err_coef, 0xFFFFFF00u, active, perm, prev_lab, lab2, flag_pair, tc_debug_mode(),
                                 xscale, dscale, err_abs));
  } else {
    kern<<<grid, C::NTHREADS, C::SMEM, st>>>(tBb, tBs, X, P, cn2, xn2, n, d, k, labels, best, flag_rows, flag_count,
                                             err_coef, 0xFFFFFF00u, active, perm, prev_lab, lab2, flag_pair,
                                             tc_debug_mode(), xscale, dscale, err_abs);
  }
  MASK_LAUNCH_CHECK();
  if (tc_debug_mode() & 8) dump_ptrace();
  if (tc_debug_mode() & 128) {
    unsigned long long h[4] = {0, 0, 0, 0};
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, g_chunk_stats, sizeof(h));
    fprintf(stderr, "[chunks] seen %llu keyed %llu (%.1f%%)\n", h[0], h[1], 100.0 * h[1] / (h[0] ? h[0] : 1));
    const unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_chunk_stats, z, sizeof(z));
  }
}

}  // namespace tc

bool tc_supported(int64_t n, int d, int64_t k) {
  (void)k;
  if (const char* e = getenv("MASK_DISABLE_TC")) {
    if (e[0] == '1') return false;
  }
  return n >= 1 && d >= 4 && d <= 128 && d % 4 == 0;
}

// B operand columns: d rounded up to 8 (zero columns beyond d); small d (d <= 24, folded) holds
// one more K step of 8 after the x columns, [||c||^2 big, ||c||^2 small, 1, 1, 0...]
// Small d pads the rows to 32 columns (128 bytes): the TMA streams whole, aligned 128-byte
// swizzle rows ~2.4x faster than 96-byte rows with an out-of-bounds tail (tools/tma_ubench.cu).
int tc_operand_cols(int d) { return d <= 24 ? 32 : ((d + 7) / 8) * 8; }
// rows of the B operand arrays: padded to whole 256-prototype tiles (pad rows never win)
int64_t tc_operand_rows(int64_t k) { return (k + 255) / 256 * 256 + 256; }

// Worst-case error coefficient of the 3xTF32 score, doubled for a gap of two scores:
// representation (<= 2^-20 |x||c| summed over the three products and the dropped xs.cs)
// + FP32 accumulation of 3*ceil(K/8) partial sums (<= 3 ceil(K/8) 2^-24 sum|x_i c_i|) + the
// final rounding, bounded with |x||c| <= (|x|^2+|c|^2)/2.
bool tc_legacy_large_d() {
  static const bool v = [] {
    const char* e = getenv("MASK_TC_LEGACY");
    return e && e[0] == '1';
  }();
  return v;
}

float tc_err_coef(int d) {
  const double ks = std::ceil(tc_operand_cols(d) / 8.0);
  const double per = std::ldexp(1.0, -20) + 3.0 * ks * std::ldexp(1.0, -24) + std::ldexp(1.0, -22);
  return (float)(2.0 * per);
}

void launch_assign_tc(const float* X, int64_t n, int d, const float* P, const float* Pb, const float* Ps,
                      const float* cn2, int64_t k, const float* xn2, int32_t* labels, float* best,
                      int32_t* flag_rows, int32_t* flag_count, cudaStream_t st, const int* active,
                      const int32_t* perm, const int32_t* prev_lab, int32_t* lab2, int2* flag_pair,
                      const void* Hb, const void* Hs, float h16_scale, float h16_err_abs) {
  const float coef = tc_err_coef(d);
  const int kc = tc_operand_cols(d);
  const int64_t kr = tc_operand_rows(k);
  // small d (FOLD): epilogue-bound; 192-prototype tiles, two TMEM accumulators (2 x 192 + 2 x
  // KA columns), three epilogue warpgroups of 64 columns (best of the measured variants)
  // small d (fold): epilogue-heavy; persistent CTAs, 192-prototype tiles, two TMEM
  // accumulators, three epilogue warpgroups of 64 columns (best of the measured variants)
#ifndef MASK_TC_P_BN
#define MASK_TC_P_BN 192
#define MASK_TC_P_STAGES 4
#define MASK_TC_P_NACC 2
#define MASK_TC_P_EPI 3
#endif
  if (d <= 8)
    tc::launch_persist<16, MASK_TC_P_BN, MASK_TC_P_STAGES, MASK_TC_P_NACC, MASK_TC_P_EPI>(
        X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best, flag_rows, flag_count, coef, st, active, perm,
        prev_lab, lab2, flag_pair);
  else if (d <= 16) {
    static const int var = [] {  // development A/B of the d = 16 tiling (MASK_TC_D16=1/2)
      const char* e = getenv("MASK_TC_D16");
      return e ? atoi(e) : 0;
    }();
    if (var == 1)  // three accumulators of 128 columns
      tc::launch_persist<24, 128, 4, 3, 2>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best, flag_rows,
                                           flag_count, coef, st, active, perm, prev_lab, lab2, flag_pair);
    else if (var == 2)  // three accumulators of 128 columns, four epilogue warpgroups of 32 columns
      tc::launch_persist<24, 128, 4, 3, 4>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best, flag_rows,
                                           flag_count, coef, st, active, perm, prev_lab, lab2, flag_pair);
    else if (var == 3)  // the default tiling with B multicast over 2-CTA clusters
      tc::launch_persist<24, MASK_TC_P_BN, MASK_TC_P_STAGES, MASK_TC_P_NACC, MASK_TC_P_EPI, true, 2, 2>(
          X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best, flag_rows, flag_count, coef, st, active, perm,
          prev_lab, lab2, flag_pair);
    else if (var == 4)  // three accumulators + multicast
      tc::launch_persist<24, 128, 4, 3, 2, true, 2, 2>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best,
                                                       flag_rows, flag_count, coef, st, active, perm, prev_lab, lab2,
                                                       flag_pair);
    else
      tc::launch_persist<24, MASK_TC_P_BN, MASK_TC_P_STAGES, MASK_TC_P_NACC, MASK_TC_P_EPI>(
          X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best, flag_rows, flag_count, coef, st, active, perm,
          prev_lab, lab2, flag_pair);
  }
  else if (d <= 24)
    tc::launch_persist<32, MASK_TC_P_BN, MASK_TC_P_STAGES, MASK_TC_P_NACC, MASK_TC_P_EPI>(
        X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best, flag_rows, flag_count, coef, st, active, perm,
        prev_lab, lab2, flag_pair);
  else if (tc_legacy_large_d()) {  // MASK_TC_LEGACY=1: the round-1 one-CTA-per-block kernel (A/B runs)
    if (d <= 32)
      tc::launch_cfg<32, 1, 32, 192, 4, 2, false, 3>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best, flag_rows,
                                                     flag_count, coef, st, active, flag_pair);
    else if (d <= 64)
      tc::launch_cfg<32, 2, 64, 128, 6, 3, false, 2>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best, flag_rows,
                                                     flag_count, coef, st, active, flag_pair);
    else if (d <= 96)
      tc::launch_cfg<32, 3, 96, 128, 6, 2, false, 2>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best, flag_rows,
                                                     flag_count, coef, st, active, flag_pair);
    else
      tc::launch_cfg<32, 4, 128, 128, 6, 2, false, 2>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best,
                                                      flag_rows, flag_count, coef, st, active, flag_pair);
  } else {
    // d > 24: the persistent kernel without the fold step (||c||^2 + ||x||^2 added by the
    // epilogue, two more roundings: + 2^-21 (||x||^2 + ||c||^2) on the gap bound), the same
    // raw-minimum / bound-pruned epilogue and label-sorted rows as small d.  K = d rounded up
    // to a whole 32-column chunk (zero columns add exact zeros)
    const float c2 = coef + std::ldexp(1.0f, -21);
    if (d <= 32)
      tc::launch_persist<32, 192, 4, 2, 3, false, 2>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best,
                                                     flag_rows, flag_count, c2, st, active, perm, prev_lab, lab2,
                                                     flag_pair);
    else if (d <= 64) {
      // three accumulators (one A buffer): the extra tile of slack between the MMAs and the
      // epilogue measured 32.5 -> 30.6 ms (n = 1e6, k = 65,536) and 349 -> 318 ms per C3 pass;
      // MASK_TC_D64=1 / 2 select the two-accumulator / 192-wide variants (development A/B)
      static const int var = [] {
        const char* e = getenv("MASK_TC_D64");
        return e ? atoi(e) : 0;
      }();
      // 3xFP16 tiling: four epilogue warpgroups of 32 columns (the MMAs take half the TF32 time,
      // so the epilogue needs the extra warps: C3 rows, n = 2e6, 63.6 -> 47.4 ms per pass; the
      // TF32 tiling at twice the rate: 50.4 ms).  MASK_TC_H16V selects development variants
      static const int hv = [] {
        const char* e = getenv("MASK_TC_H16V");
        return e ? atoi(e) : 2;
      }();
      const float ds = 1.f / (h16_scale * h16_scale);
      if (Hb && hv == 1)
        tc::launch_persist<64, 192, 4, 2, 3, false, 2, 1, true>(
            X, n, d, kc, kr, P, Hb, Hs, cn2, k, xn2, labels, best, flag_rows, flag_count, 2.f * c2, st, active, perm,
            prev_lab, lab2, flag_pair, h16_scale, ds, h16_err_abs);
      else if (Hb && hv == 2)  // (default)
        tc::launch_persist<64, 128, 6, 3, 4, false, 1, 1, true>(
            X, n, d, kc, kr, P, Hb, Hs, cn2, k, xn2, labels, best, flag_rows, flag_count, 2.f * c2, st, active, perm,
            prev_lab, lab2, flag_pair, h16_scale, ds, h16_err_abs);
      else if (Hb && hv == 3)
        tc::launch_persist<64, 192, 4, 2, 3, false, 1, 1, true>(
            X, n, d, kc, kr, P, Hb, Hs, cn2, k, xn2, labels, best, flag_rows, flag_count, 2.f * c2, st, active, perm,
            prev_lab, lab2, flag_pair, h16_scale, ds, h16_err_abs);
      else if (Hb && hv == 5)  // the default tiling with B multicast over 2-CTA clusters
        tc::launch_persist<64, 128, 6, 3, 4, false, 1, 2, true>(
            X, n, d, kc, kr, P, Hb, Hs, cn2, k, xn2, labels, best, flag_rows, flag_count, 2.f * c2, st, active, perm,
            prev_lab, lab2, flag_pair, h16_scale, ds, h16_err_abs);
      else if (Hb && hv == 6)  // more accumulator slack: 96-wide tiles, four accumulators
        tc::launch_persist<64, 96, 8, 4, 3, false, 1, 1, true>(
            X, n, d, kc, kr, P, Hb, Hs, cn2, k, xn2, labels, best, flag_rows, flag_count, 2.f * c2, st, active, perm,
            prev_lab, lab2, flag_pair, h16_scale, ds, h16_err_abs);
      else if (Hb && hv == 7)  // 64-wide tiles, six accumulators
        tc::launch_persist<64, 64, 8, 6, 2, false, 1, 1, true>(
            X, n, d, kc, kr, P, Hb, Hs, cn2, k, xn2, labels, best, flag_rows, flag_count, 2.f * c2, st, active, perm,
            prev_lab, lab2, flag_pair, h16_scale, ds, h16_err_abs);
      else if (Hb && hv == 4)
        tc::launch_persist<64, 128, 6, 3, 2, false, 2, 1, true>(
            X, n, d, kc, kr, P, Hb, Hs, cn2, k, xn2, labels, best, flag_rows, flag_count, 2.f * c2, st, active, perm,
            prev_lab, lab2, flag_pair, h16_scale, ds, h16_err_abs);
      else if (Hb)  // 3xFP16 (kind::f16): the TF32 tiling at twice the MMA rate
        tc::launch_persist<64, 128, 6, 3, 2, false, 1, 1, true>(
            X, n, d, kc, kr, P, Hb, Hs, cn2, k, xn2, labels, best, flag_rows, flag_count, 2.f * c2, st, active, perm,
            prev_lab, lab2, flag_pair, h16_scale, ds, h16_err_abs);
      else if (var == 0)
        tc::launch_persist<64, 128, 6, 3, 2, false, 1>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best,
                                                       flag_rows, flag_count, c2, st, active, perm, prev_lab, lab2,
                                                       flag_pair);
      else if (var == 3)  // multicast B over 2-CTA clusters
        tc::launch_persist<64, 128, 6, 3, 2, false, 1, 2>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best,
                                                          flag_rows, flag_count, c2, st, active, perm, prev_lab, lab2,
                                                          flag_pair);
      else if (var == 2)
        tc::launch_persist<64, 192, 4, 2, 3, false, 1>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best,
                                                       flag_rows, flag_count, c2, st, active, perm, prev_lab, lab2,
                                                       flag_pair);
      else
        tc::launch_persist<64, 128, 6, 2, 2, false, 2>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best,
                                                       flag_rows, flag_count, c2, st, active, perm, prev_lab, lab2,
                                                       flag_pair);  // MASK_TC_D64=1
    }
    else if (d <= 96)
      tc::launch_persist<96, 128, 6, 2, 2, false, 1>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best,
                                                     flag_rows, flag_count, c2, st, active, perm, prev_lab, lab2,
                                                     flag_pair);
    else if (Hb && d == 128 && getenv("MASK_TC_H16V") && atoi(getenv("MASK_TC_H16V")) == 1)
      tc::launch_persist<128, 192, 4, 2, 3, false, 1, 1, true>(
          X, n, d, kc, kr, P, Hb, Hs, cn2, k, xn2, labels, best, flag_rows, flag_count, 2.f * c2, st, active, perm,
          prev_lab, lab2, flag_pair, h16_scale, 1.f / (h16_scale * h16_scale), h16_err_abs);
    else if (Hb && d == 128 && getenv("MASK_TC_H16V") && atoi(getenv("MASK_TC_H16V")) == 2)
      tc::launch_persist<128, 128, 6, 3, 4, false, 1, 1, true>(
          X, n, d, kc, kr, P, Hb, Hs, cn2, k, xn2, labels, best, flag_rows, flag_count, 2.f * c2, st, active, perm,
          prev_lab, lab2, flag_pair, h16_scale, 1.f / (h16_scale * h16_scale), h16_err_abs);
    else if (Hb && d == 128 && getenv("MASK_TC_H16V") && atoi(getenv("MASK_TC_H16V")) == 3)
      tc::launch_persist<128, 128, 6, 3, 2, false, 1, 1, true>(
          X, n, d, kc, kr, P, Hb, Hs, cn2, k, xn2, labels, best, flag_rows, flag_count, 2.f * c2, st, active, perm,
          prev_lab, lab2, flag_pair, h16_scale, 1.f / (h16_scale * h16_scale), h16_err_abs);
    else if (Hb && d == 128 && getenv("MASK_TC_H16V") && atoi(getenv("MASK_TC_H16V")) == 4)
      tc::launch_persist<128, 128, 6, 2, 4, false, 1, 1, true>(
          X, n, d, kc, kr, P, Hb, Hs, cn2, k, xn2, labels, best, flag_rows, flag_count, 2.f * c2, st, active, perm,
          prev_lab, lab2, flag_pair, h16_scale, 1.f / (h16_scale * h16_scale), h16_err_abs);
    else if (Hb && d == 128)
      tc::launch_persist<128, 128, 6, 2, 2, false, 1, 1, true>(
          X, n, d, kc, kr, P, Hb, Hs, cn2, k, xn2, labels, best, flag_rows, flag_count, 2.f * c2, st, active, perm,
          prev_lab, lab2, flag_pair, h16_scale, 1.f / (h16_scale * h16_scale), h16_err_abs);
    else
      tc::launch_persist<128, 128, 6, 2, 2, false, 1>(X, n, d, kc, kr, P, Pb, Ps, cn2, k, xn2, labels, best,
                                                      flag_rows, flag_count, c2, st, active, perm, prev_lab, lab2,
                                                     flag_pair);
  }
}

// ---------------------------------------------------------------------------------------------
// 3xFP16 operands (K1 H16).  Per level: max |x| -> the power-of-two scale s with max |s x| in
// (2^11, 2^12] (|s (-2c)| <= 2^13: prototypes are member means).  Per pass: the split
// s (-2c) = big + small in FP16 (from the FP64 prototypes when the level keeps them).
__global__ void k_maxabs(const float* __restrict__ X, int64_t cnt, unsigned* __restrict__ out) {
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(X[i]));
  const unsigned u = __reduce_max_sync(0xffffffffu, __float_as_uint(m));  // (non-negative floats order as uints)
  if ((threadIdx.x & 31) == 0 && u) atomicMax(out, u);
}

bool tc_h16_enabled() {  // default on; MASK_TC_H16=0 keeps 3xTF32 everywhere (A/B runs)
  static const bool v = [] {
    const char* e = getenv("MASK_TC_H16");
    return !(e && e[0] == '0');
  }();
  return v;
}

float h16_level_scale(const float* X, int64_t cnt, float* maxabs_out, cudaStream_t st) {
  unsigned* dv = nullptr;
  MASK_CUDA(cudaMallocAsync(&dv, sizeof(unsigned), st));
  MASK_CUDA(cudaMemsetAsync(dv, 0, sizeof(unsigned), st));
  if (cnt > 0) {
    k_maxabs<<<grid_for(cnt, 256, (int64_t)num_sms() * 8), 256, 0, st>>>(X, cnt, dv);
    MASK_LAUNCH_CHECK();
  }
  unsigned h = 0;
  MASK_CUDA(cudaMemcpyAsync(&h, dv, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  MASK_CUDA(cudaFreeAsync(dv, st));
  MASK_CUDA(cudaStreamSynchronize(st));
  float m = 0.f;
  std::memcpy(&m, &h, sizeof(m));
  *maxabs_out = m;
  if (!(m > 0.f) || !std::isfinite(m)) return 1.f;
  int e = 0;
  std::frexp(m, &e);  // m = f 2^e, f in [0.5, 1)
  return std::ldexp(1.0f, 12 - e);
}

template <typename T>
__global__ void k_prep_h16(const T* __restrict__ P, int64_t k, int d, float s, __half* __restrict__ Hb,
                           __half* __restrict__ Hs, const int* __restrict__ active) {
  if (active && !*active) return;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < k * d; e += (int64_t)gridDim.x * blockDim.x) {
    const double m2 = -2.0 * (double)P[e] * (double)s;
    const __half b = __float2half_rn((float)m2);
    Hb[e] = b;
    Hs[e] = __float2half_rn((float)(m2 - (double)__half2float(b)));
  }
}

void launch_prep_h16(const float* P, const double* P64, int64_t k, int d, float s, void* Hb, void* Hs, cudaStream_t st,
                     const int* active) {
  if (k <= 0) return;
  const unsigned grid = grid_for(k * d, 256, (int64_t)num_sms() * 16);
  if (P64)
    k_prep_h16<double><<<grid, 256, 0, st>>>(P64, k, d, s, static_cast<__half*>(Hb), static_cast<__half*>(Hs), active);
  else
    k_prep_h16<float><<<grid, 256, 0, st>>>(P, k, d, s, static_cast<__half*>(Hb), static_cast<__half*>(Hs), active);
  MASK_LAUNCH_CHECK();
}

}  // namespace mask
