// assign_csr_tc.cu -- K3T: sparse (CSR) assignment with the hot columns on the tensor cores
// (the high-dimensional sparse workload of PAPER.md §4.3; BASELINE.json configs[3]).
//
//   s_ij = ||c_j||^2 - 2 sum_{p in nz(i)} v_p c_j[col_p]          (D12; ||x_i||^2 is a row
//   constant, added back to the winner: d^2 = s + ||x_i||^2), a_i = argmin_j s_ij (lowest j, D4)
//
// The non-zeros of a row split by column into the H most frequent ("hot") columns of the level
// and the rest ("tail"):  x.(-2c) = xh.(-2c_h) + sum_{tail} (-2 v_p) c[col_p].
//   hot:  a dense n x H block Xh (built once per level) times the hot slice of the prototypes,
//         3xTF32 on tcgen05.mma (A = Xh split big/small in TMEM, B = the split -2 c_h streamed
//         by TMA), FP32 accumulation in TMEM -- K1's pipeline with d = H;
//   tail: the epilogue stages each 128 x BN accumulator tile in shared memory and then walks the
//         rows warp by warp: lane l owns prototypes j0 + 4l .. 4l + 3, adds the row's tail
//         non-zeros through the transposed prototypes PT (one coalesced 512-byte row slice per
//         non-zero) and ||c_j||^2, and folds the tile's (s, j) minimum into the row's running key.
// Zipf column popularity: at C4 the 128 hot columns hold 58 % of the
// non-zeros; the tail (42 %) stays on the SIMT load path, the hot part costs ~18 % of the
// tensor pipe.  DESIGN.md §6 "K3T".
//
// Roles (one CTA per 128-row block; 2 control warps + EPI_WG epilogue warpgroups):
//   warp 0      TMA producer of the B chunks (big + small, 32 K columns each) through a ring;
//   warp 1      TMEM allocator (512 columns: 2 x BN accumulators + H big + H small), then the MMA
//               issuer (one elected lane), A from TMEM, accumulators double-buffered;
//   warps 2..   epilogue (4 EPI_WG warps; warp w reads TMEM lane quarter w % 4): warpgroup 0 first splits the Xh block into TMEM; then per tile every
//               epilogue warp copies its 32 x 32 accumulator quarter to shared memory (double-
//               buffered), one named barrier, and each warp finishes BM / (4 EPI_WG) rows.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "tcgen05.cuh"

namespace mask {
namespace k3t {
using namespace tc;

constexpr int H = 128;               // hot columns (A big + small = 2H TMEM columns)
constexpr int BN = 128;              // prototypes per tile
constexpr int CW = 32;               // K columns per B chunk (one 128-byte swizzle row)
constexpr int NKC = H / CW;
constexpr int STAGES = 2;
constexpr int NACC = 2;
constexpr int EPI_WG = 4;
constexpr int NEW = 4 * EPI_WG;      // epilogue warps
constexpr int RPW = BM / NEW;        // rows finished per epilogue warp and tile
constexpr int kEpi0 = 2;             // first epilogue warp (warps 0, 1: TMA producer, TMEM + MMA)
constexpr int NTHREADS = 32 * kEpi0 + 32 * NEW;
constexpr int CWB = CW * 4;
constexpr int B_CHUNK = BN * CWB;
constexpr int STAGE_BYTES = 2 * B_CHUNK;
constexpr int DS = BN + 4;           // padded row stride (floats) of a staged tile: conflict-free
constexpr int D_FLOATS = BM * DS;
constexpr int D_OFF = STAGES * STAGE_BYTES;
constexpr int BAR_OFF = D_OFF + 2 * D_FLOATS * 4;  // two staged tiles (one barrier per tile)
constexpr int NBARS = 2 * STAGES + 2 * NACC + 1;
constexpr int G = 8;                 // tail loads in flight per warp and group
constexpr int SMEM = BAR_OFF + NBARS * 8 + 16 + 1024;
constexpr int A_COL = NACC * BN;
constexpr int AS_COL = A_COL + H;
constexpr int TMEM_COLS = 512;
constexpr uint32_t IDESC = idesc_tf32<BM, BN>();
static_assert(AS_COL + H <= TMEM_COLS, "TMEM budget");
static_assert(SMEM <= 232448, "shared memory budget");
static_assert(BN == 128 && NEW * RPW == BM && RPW <= 32 && EPI_WG <= BN / 32, "epilogue layout");

// order-preserving float -> uint32 (total order of the finite values and +-inf)
__device__ __forceinline__ uint32_t ord(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord(uint32_t k) { return __uint_as_float((k & 0x80000000u) ? (k ^ 0x80000000u) : ~k); }
__device__ __forceinline__ uint64_t key_of(float s, uint32_t j) { return ((uint64_t)ord(s) << 32) | j; }
__device__ __forceinline__ uint64_t kmin(uint64_t a, uint64_t b) { return b < a ? b : a; }

__global__ void __launch_bounds__(NTHREADS, 1)
    k_assign_csr_tc(const __grid_constant__ CUtensorMap tmBb, const __grid_constant__ CUtensorMap tmBs,
                    const float* __restrict__ Xh, const int64_t* __restrict__ rp, const int2* __restrict__ tail,
                    const int32_t* __restrict__ ntail, const float* __restrict__ PT, int64_t kp,
                    const float* __restrict__ cn2, const float* __restrict__ xn2, int64_t n, int64_t k,
                    int32_t* __restrict__ labels, float* __restrict__ best, const int* __restrict__ active) {
  if (active && !*active) return;  // level converged: this pass is skipped on the device
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Bst = smem;
  float* Dsm = reinterpret_cast<float*>(smem + D_OFF);  // two staged 128 x BN accumulator tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + NACC;
  uint64_t* a_ready = bars + 2 * STAGES + 2 * NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBARS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (int64_t)blockIdx.x * BM;
  const int ntiles = (int)((k + BN - 1) / BN);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmBb);
    prefetch_tmap(&tmBs);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], NEW * kArrivePerWarp);
    }
    mbar_init(a_ready, 4 * kArrivePerWarp);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (B)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < ntiles; ++t) {
        for (int c = 0; c < NKC; ++c) {
          mbar_wait_spin(&empty[stage], phase ^ 1);
          uint8_t* dst = Bst + stage * STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(dst, &tmBb, &full[stage], c * CW, t * BN);
          tma_load_2d(dst + B_CHUNK, &tmBs, &full[stage], c * CW, t * BN);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (A from TMEM)
    // one issuer for every tile, in ring order: the tensor pipe is ~1/5 busy here (the epilogue
    // binds), and a second issuer a whole tile ahead could read a ring slot two phases early
    mbar_wait_spin(a_ready, 0);
    tc_fence_after();
    for (int t = 0; t < ntiles; ++t) {
      const int acc = t % NACC;
      mbar_wait_spin(&tempty[acc], ((t / NACC) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
      for (int c = 0; c < NKC; ++c) {
        const int gc = t * NKC + c;
        const int stage = gc % STAGES;
        const uint32_t phase = (uint32_t)((gc / STAGES) & 1);
        mbar_wait_spin(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t bb = smem_u32(Bst + stage * STAGE_BYTES);
          const uint32_t bs = bb + B_CHUNK;
#pragma unroll
          for (int ks = 0; ks < CW / 8; ++ks) {
            const uint32_t kcol = (uint32_t)(c * CW + ks * 8);
            const uint32_t ab = tmem_base + A_COL + kcol, as = tmem_base + AS_COL + kcol;
            const uint64_t dbb = smem_desc<CWB>(bb + ks * 32), dbs = smem_desc<CWB>(bs + ks * 32);
            mma_tf32_ts(d_tmem, as, dbb, IDESC, (c | ks) != 0);
            mma_tf32_ts(d_tmem, ab, dbs, IDESC, 1u);
            mma_tf32_ts(d_tmem, ab, dbb, IDESC, 1u);
          }
          mma_commit(&empty[stage]);
          if (c == NKC - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else {
    const int et = threadIdx.x - kEpi0 * 32;
    const int wg = et >> 7;
    const int ew = et >> 5;          // epilogue warp 0 .. NEW-1
    const int q = warp & 3;          // TMEM lane quarter
    const int rloc = q * 32 + lane;  // row of this thread in the TMEM / staging phase
    // ------------------------------------------------------------ Xh -> TMEM (warpgroup 0)
    if (wg == 0) {
      const int64_t row = row0 + rloc;
      const float* xr = Xh + row * H;
      const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int g = 0; g < H; g += 8) {
        uint32_t vb[8], vs[8];
#pragma unroll
        for (int u = 0; u < 8; u += 4) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (row < n) v = __ldg(reinterpret_cast<const float4*>(xr + g + u));
          const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const float b = tf32_rn(e[w]);
            vb[u + w] = __float_as_uint(b);
            vs[u + w] = __float_as_uint(tf32_rn(e[w] - b));
          }
        }
        tmem_st8(lane_base + A_COL + g, vb);
        tmem_st8(lane_base + AS_COL + g, vs);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive_warp(a_ready);
    }
    // this warp's rows: rr_i = ew + NEW i (i < RPW); lane i keeps row rr_i's tail range and key
    int64_t my_p0 = 0;
    int my_nt = 0;
    uint64_t my_key = ~0ull;
    if (lane < RPW && ew + NEW * lane < BM) {
      const int64_t row = row0 + ew + NEW * lane;
      if (row < n) {
        my_p0 = rp[row];
        my_nt = ntail[row];
      }
    }
    const int64_t inblk = n - row0 < BM ? n - row0 : BM;
    const int64_t nr_ = (inblk - ew + NEW - 1) / NEW;
    const int nrows = nr_ <= 0 ? 0 : (nr_ >= RPW ? RPW : (int)nr_);
    for (int t = 0; t < ntiles; ++t) {
      const int acc = t % NACC;
      float* D = Dsm + (t & 1) * D_FLOATS;
      // ---- stage the accumulator tile: warp (wg, q) copies TMEM lanes 32q.. x 32-column chunks
      // wg, wg + EPI_WG, ..  (double-buffered: the barrier of tile t + 1 orders tile t's readers
      // before tile t + 2's writers)
      if (q == 0) mbar_wait_spin(&tfull[acc], (t / NACC) & 1);
      asm volatile("bar.sync %0, 128;" ::"r"(2 + wg) : "memory");
      tc_fence_after();
      for (int cc = wg; cc < BN / 32; cc += EPI_WG) {
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + cc * 32), r);
        tmem_wait_ld();
        float4* dst = reinterpret_cast<float4*>(D + rloc * DS + cc * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          dst[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]), __uint_as_float(r[4 * i + 2]),
                               __uint_as_float(r[4 * i + 3]));
      }
      tc_fence_before();
      mbar_arrive_warp(&tempty[acc]);
      asm volatile("bar.sync 1, %0;" ::"n"(32 * NEW) : "memory");
      // ---- finish this warp's rows: tail non-zeros (G coalesced 512-byte PT slices in flight),
      // + ||c||^2, tile minimum
      const int64_t j0 = (int64_t)t * BN;
      const float4 cv = __ldg(reinterpret_cast<const float4*>(cn2 + j0) + lane);
      const float* ptl = PT + j0 + 4 * lane;
#pragma unroll 1
      for (int i = 0; i < nrows; ++i) {
        float4 a = *reinterpret_cast<const float4*>(D + (ew + NEW * i) * DS + 4 * lane);
        const int64_t p0 = __shfl_sync(0xffffffffu, my_p0, i);
        const int nt = __shfl_sync(0xffffffffu, my_nt, i);
        for (int e0 = 0; e0 < nt; e0 += 32) {
          const int m = min(32, nt - e0);
          const int2 ent = lane < m ? __ldg(tail + p0 + e0 + lane) : make_int2(0, 0);
          for (int g = 0; g < m; g += G) {
            float4 pv[G];
            float vv[G];
#pragma unroll
            for (int u = 0; u < G; ++u) {
              const int c = __shfl_sync(0xffffffffu, ent.x, g + u);
              vv[u] = __int_as_float(__shfl_sync(0xffffffffu, ent.y, g + u));
              pv[u] = g + u < m ? __ldg(reinterpret_cast<const float4*>(ptl + (int64_t)c * kp))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < G; ++u) {
              a.x = fmaf(vv[u], pv[u].x, a.x);
              a.y = fmaf(vv[u], pv[u].y, a.y);
              a.z = fmaf(vv[u], pv[u].z, a.z);
              a.w = fmaf(vv[u], pv[u].w, a.w);
            }
          }
        }
        const uint32_t jl = (uint32_t)(j0 + 4 * lane);
        uint64_t key = kmin(kmin(key_of(a.x + cv.x, jl), key_of(a.y + cv.y, jl + 1)),
                            kmin(key_of(a.z + cv.z, jl + 2), key_of(a.w + cv.w, jl + 3)));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) key = kmin(key, __shfl_xor_sync(0xffffffffu, key, o));
        if (lane == i) my_key = kmin(my_key, key);
      }
    }
    if (lane < RPW && ew + NEW * lane < BM) {
      const int64_t row = row0 + ew + NEW * lane;
      if (row < n) {
        const uint32_t j = (uint32_t)(my_key & 0xffffffffu);
        labels[row] = (int32_t)j;
        if (best) best[row] = fmaxf(unord((uint32_t)(my_key >> 32)) + __ldg(xn2 + row), 0.f);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
}

// ---------------------------------------------------------------------------------------------
// Per level (the data do not change across passes): the dense hot block Xh [n x H] (slot order of
// `colslot`, zeros elsewhere), the tail non-zeros {col, -2 v} compacted to the front of each
// row's CSR segment (CSR order kept), their count, and ||x||^2 (FP32, CSR order as K3).
// One warp per row.
__global__ void k3t_build_level(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                const float* __restrict__ val, int64_t n, const int16_t* __restrict__ colslot,
                                float* __restrict__ Xh, int2* __restrict__ tail, int32_t* __restrict__ ntail,
                                float* __restrict__ xn2) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const int64_t p0 = rp[r], p1 = rp[r + 1];
    float* xr = Xh + r * H;
    for (int h = lane; h < H; h += 32) xr[h] = 0.f;
    __syncwarp();
    float xx = 0.f;
    int cnt = 0;
    for (int64_t pb = p0; pb < p1; pb += 32) {
      const int64_t p = pb + lane;
      int32_t c = 0;
      float v = 0.f;
      int s = -1;
      if (p < p1) {
        c = col[p];
        v = val[p];
        xx = fmaf(v, v, xx);
        s = colslot[c];
      }
      const unsigned tb = __ballot_sync(0xffffffffu, p < p1 && s < 0);
      if (p < p1) {
        if (s >= 0) xr[s] = v;
        else tail[p0 + cnt + __popc(tb & ((1u << lane) - 1u))] = make_int2(c, __float_as_int(-2.f * v));
      }
      cnt += __popc(tb);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xx += __shfl_xor_sync(0xffffffffu, xx, o);
    if (lane == 0) {
      ntail[r] = cnt;
      xn2[r] = xx;
    }
  }
}

// Per pass: ||c_j||^2 (FP64 sum, +inf beyond k), the split hot slice -2 c_j[hotcols] = big +
// small (TF32 parts; zero for an unused slot and beyond k).  One warp per prototype row.
__global__ void k3t_prep_protos(const float* __restrict__ P, int64_t k, int64_t k_rows, int d,
                                const int32_t* __restrict__ hotcols, float* __restrict__ Hb, float* __restrict__ Hs,
                                float* __restrict__ cn2, const int* __restrict__ active) {
  if (active && !*active) return;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < k_rows; j += warps) {
    if (j >= k) {
      for (int h = lane; h < H; h += 32) Hb[j * H + h] = Hs[j * H + h] = 0.f;
      if (lane == 0) cn2[j] = INFINITY;
      continue;
    }
    const float* pr = P + j * d;
    double s = 0.0;
    for (int i = lane; i < d; i += 32) {
      const double c = pr[i];
      s += c * c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) cn2[j] = (float)s;
    for (int h = lane; h < H; h += 32) {
      const int32_t c = hotcols[h];
      const double m2 = c >= 0 ? -2.0 * (double)pr[c] : 0.0;
      const float b = tf32_rn((float)m2);
      Hb[j * H + h] = b;
      Hs[j * H + h] = tf32_rn((float)(m2 - (double)b));
    }
  }
}

// PT[c * kp + j] = P[j * d + c] (zero for k <= j < kp): 32 x 32 tiles through shared memory.
__global__ void k3t_transpose(const float* __restrict__ P, int64_t k, int64_t kp, int d, float* __restrict__ PT,
                              const int* __restrict__ active) {
  if (active && !*active) return;
  __shared__ float tile[32][33];
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
    const int64_t j = j0 + yy;
    const int c = c0 + threadIdx.x;
    tile[yy][threadIdx.x] = (j < k && c < d) ? P[j * d + c] : 0.f;
  }
  __syncthreads();
  for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
    const int c = c0 + yy;
    const int64_t j = j0 + threadIdx.x;
    if (c < d && j < kp) PT[(int64_t)c * kp + j] = tile[threadIdx.x][yy];
  }
}

}  // namespace k3t

int64_t csr_tc_rows(int64_t k) { return (k + k3t::BN - 1) / k3t::BN * k3t::BN; }
int csr_tc_hot() { return k3t::H; }

void launch_csr_tc_level(const int64_t* rp, const int32_t* col, const float* val, int64_t n, const int16_t* colslot,
                         float* Xh, int2* tail, int32_t* ntail, float* xn2, cudaStream_t st) {
  if (n <= 0) return;
  k3t::k3t_build_level<<<grid_for(n * 32, 256, (int64_t)num_sms() * 16), 256, 0, st>>>(rp, col, val, n, colslot, Xh,
                                                                                         tail, ntail, xn2);
  MASK_LAUNCH_CHECK();
}

void launch_csr_tc_prep(const float* P, int64_t k, int d, const int32_t* hotcols, float* Hb, float* Hs, float* cn2,
                        float* PT, cudaStream_t st, const int* active) {
  const int64_t kr = csr_tc_rows(k);
  k3t::k3t_prep_protos<<<grid_for(kr * 32, 256), 256, 0, st>>>(P, k, kr, d, hotcols, Hb, Hs, cn2, active);
  MASK_LAUNCH_CHECK();
  dim3 grid((unsigned)(kr / 32), (unsigned)((d + 31) / 32));
  k3t::k3t_transpose<<<grid, dim3(32, 8), 0, st>>>(P, k, kr, d, PT, active);
  MASK_LAUNCH_CHECK();
}

void launch_assign_csr_tc(const float* Xh, const int64_t* rp, const int2* tail, const int32_t* ntail, const float* xn2,
                          int64_t n, const float* Hb, const float* Hs, const float* PT, const float* cn2, int64_t k,
                          int32_t* labels, float* best, cudaStream_t st, const int* active) {
  using namespace k3t;
  if (n <= 0) return;
  const int64_t kr = csr_tc_rows(k);
  const CUtensorMap tBb = tc::make_map(Hb, kr, H, CW, BN);
  const CUtensorMap tBs = tc::make_map(Hs, kr, H, CW, BN);
  static bool attr = false;
  if (!attr) {
    MASK_CUDA(cudaFuncSetAttribute(k_assign_csr_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    attr = true;
  }
  const unsigned grid = (unsigned)((n + BM - 1) / BM);
  k_assign_csr_tc<<<grid, NTHREADS, SMEM, st>>>(tBb, tBs, Xh, rp, tail, ntail, PT, kr, cn2, xn2, n, k, labels, best,
                                                active);
  MASK_LAUNCH_CHECK();
}

}  // namespace mask
