// cluster.cu -- K14: the paper's distributed mode (§3.4 "Indexing distributed
// datasets").  Every node (one GPU) builds its own index
// over its own rows with no communication; the coordinator records "just the top level
// centroids from each node"; a query is sent either to all nodes or only to
// "nodes that have centroids whose distance to the target query object is lower than a given
// threshold epsilon", and the nodes' answers are merged.
//
//   route:  routed[q * W + n] = 1 iff min over registered centroids c of node n of
//           ||q - c||^2 < eps^2 (strict, reading C1; FP32 direct sums like K9), or eps = inf
//   merge:  per query, the k best of the W node answers (each sorted by (d^2, id), padded
//           with (-1, +inf)) by (d^2, node, id) (reading C3)
//
// Both are tiny next to the per-node descent (K9): routing is Q x R distances with R = the
// registry size (W * k_L rows), merging touches W * k candidates per query.  One warp per
// query for routing (lanes over registry rows, node flags set with plain byte stores: every
// writer stores the same 1); one thread per query for the W-way merge.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "common.cuh"

namespace mask {

namespace {

constexpr int kRouteWarps = 8;

__global__ void __launch_bounds__(kRouteWarps * 32)
    k_route_dense(const float* __restrict__ reg, const int32_t* __restrict__ node_of, int64_t R, int W,
                  const float* __restrict__ Q, int64_t nq, int d, float eps2, int all,
                  uint8_t* __restrict__ routed) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = warp; q < nq; q += nwarps) {
    uint8_t* out = routed + q * W;
    for (int n = lane; n < W; n += 32) out[n] = all ? 1 : 0;
    if (all) continue;
    __syncwarp();
    const float* qv = Q + q * d;
    for (int64_t j = lane; j < R; j += 32) {
      const float* c = reg + j * d;
      float s = 0.f;
      for (int i = 0; i < d; ++i) {
        const float t = __ldg(qv + i) - __ldg(c + i);
        s = fmaf(t, t, s);
      }
      if (s < eps2) out[node_of[j]] = 1;
    }
  }
}

// CSR queries: ||q - c||^2 = ||c||^2 + sum_{p in nz(q)} (q_p^2 - 2 q_p c[col_p]) (D12)
__global__ void __launch_bounds__(kRouteWarps * 32)
    k_route_csr(const float* __restrict__ reg, const float* __restrict__ reg_n2, const int32_t* __restrict__ node_of,
                int64_t R, int W, int d, const int64_t* __restrict__ qrp, const int32_t* __restrict__ qcol,
                const float* __restrict__ qval, int64_t nq, float eps2, int all, uint8_t* __restrict__ routed) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = warp; q < nq; q += nwarps) {
    uint8_t* out = routed + q * W;
    for (int n = lane; n < W; n += 32) out[n] = all ? 1 : 0;
    if (all) continue;
    __syncwarp();
    const int64_t p0 = qrp[q], p1 = qrp[q + 1];
    float qq = 0.f;
    for (int64_t p = p0; p < p1; ++p) qq = fmaf(qval[p], qval[p], qq);
    for (int64_t j = lane; j < R; j += 32) {
      const float* c = reg + j * (int64_t)d;
      float s = 0.f;
      for (int64_t p = p0; p < p1; ++p) s = fmaf(qval[p], __ldg(c + qcol[p]), s);
      if (reg_n2[j] + qq - 2.f * s < eps2) out[node_of[j]] = 1;
    }
  }
}

__global__ void k_reg_norms(const float* __restrict__ reg, int64_t R, int d, float* __restrict__ n2) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < R; j += nwarps) {
    float s = 0.f;
    for (int i = lane; i < d; i += 32) s = fmaf(reg[j * d + i], reg[j * d + i], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) n2[j] = s;
  }
}

constexpr int kMaxNodes = 64;

// ids/d2: W blocks of nq x k (node-major), each row sorted by (d^2, id), padding (-1, +inf) last
__global__ void k_merge(const int64_t* __restrict__ ids, const float* __restrict__ d2, int W, int64_t nq, int k,
                        int64_t* __restrict__ ids_out, float* __restrict__ d2_out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  uint8_t head[kMaxNodes];
  for (int n = 0; n < W; ++n) head[n] = 0;
  const int64_t blk = nq * k;
  for (int r = 0; r < k; ++r) {
    int bn = -1;
    float bd = INFINITY;
    int64_t bi = -1;
    for (int n = 0; n < W; ++n) {  // ascending n: strict < keeps the lowest node on (d^2) ties
      if (head[n] >= k) continue;
      const int64_t e = n * blk + q * k + head[n];
      const int64_t ci = ids[e];
      if (ci < 0) continue;  // this node's answer is exhausted
      const float cd = d2[e];
      if (bn < 0 || cd < bd) {
        bn = n;
        bd = cd;
        bi = ci;
      }
    }
    if (bn >= 0) ++head[bn];
    ids_out[q * k + r] = bi;
    d2_out[q * k + r] = bn >= 0 ? bd : INFINITY;
  }
}

}  // namespace

void launch_route_dense(const float* reg, const int32_t* node_of, int64_t R, int W, const float* Q, int64_t nq, int d,
                        float eps2, bool all, uint8_t* routed, cudaStream_t st) {
  if (nq <= 0) return;
  const int64_t blocks = (nq + kRouteWarps - 1) / kRouteWarps;
  const unsigned grid = (unsigned)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  k_route_dense<<<grid, kRouteWarps * 32, 0, st>>>(reg, node_of, R, W, Q, nq, d, eps2, all ? 1 : 0, routed);
  MASK_LAUNCH_CHECK();
}

void launch_route_csr(const float* reg, float* reg_n2, const int32_t* node_of, int64_t R, int W, int d,
                      const int64_t* qrp, const int32_t* qcol, const float* qval, int64_t nq, float eps2, bool all,
                      uint8_t* routed, cudaStream_t st) {
  if (nq <= 0) return;
  if (!all && R > 0) {
    const int64_t b = (R + 7) / 8;
    k_reg_norms<<<(unsigned)(b < 4096 ? b : 4096), 256, 0, st>>>(reg, R, d, reg_n2);
    MASK_LAUNCH_CHECK();
  }
  const int64_t blocks = (nq + kRouteWarps - 1) / kRouteWarps;
  const unsigned grid = (unsigned)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
  k_route_csr<<<grid, kRouteWarps * 32, 0, st>>>(reg, reg_n2, node_of, R, W, d, qrp, qcol, qval, nq, eps2,
                                                 all ? 1 : 0, routed);
  MASK_LAUNCH_CHECK();
}

void launch_merge(const int64_t* ids, const float* d2, int W, int64_t nq, int k, int64_t* ids_out, float* d2_out,
                  cudaStream_t st) {
  MASK_REQUIRE(W >= 1 && W <= kMaxNodes, MASK_ERR_ARG, "merge: n_nodes must be in [1, 64]");
  if (nq <= 0) return;
  k_merge<<<(unsigned)((nq + 127) / 128), 128, 0, st>>>(ids, d2, W, nq, k, ids_out, d2_out);
  MASK_LAUNCH_CHECK();
}

}  // namespace mask
