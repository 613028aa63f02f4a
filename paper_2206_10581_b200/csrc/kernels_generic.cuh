// kernels_generic.cuh -- the shape-agnostic path: any d, ranks and factors.
// One thread per output element with fixed-order (ascending) contractions;
// level products are materialised.  It is the correctness baseline for the
// fused fast path and serves every config the fast path does not cover
// (e.g. the reference's tiny test shapes).
//
// Level k (0-based) of the plan holds the distinct prefixes (i_1..i_{k+1});
// a level-k node's product P_k is rows[k] x cols[k]  (= N_{k+1} x R_{k+1}),
// P_k = P_{k-1}[parent] (rows[k] x R_k) . G_k[i_{k+1}] (R_k x n_k R_{k+1})
// -- the chain of reconstruct_padded_into (tt_embedding.cpp:39-71) with
// shared prefixes computed once.
#pragma once
#include "common.cuh"

namespace tt {

struct LevelBufs {
  float* P[TT_MAXD];    // level-k products (k = 1..d-2)
  float* dP[TT_MAXD];   // level-k gradients of P_k (k = 0..d-1; dP[d-1] = unique upstream rows)
  float* dPc[TT_MAXD];  // per-child contributions to dP[k-1] (k = 1..d-1)
};

// A operand of level k for node `nd`: P_{k-1}[parent], or the core-0 slice.
__device__ __forceinline__ const float* level_A(const DevCfg& c, const float* params, const LevelBufs& L,
                                                const int* parent_k, const int* digit0, int k, int nd) {
  int p = parent_k[nd];
  if (k == 1) return params + c.core_off[0] + (int64_t)digit0[p] * c.slice[0];
  return L.P[k - 1] + (int64_t)p * c.rows[k] * c.R[k];
}

// forward, level k >= 1
__global__ void k_gen_fwd_level(DevCfg c, int k, const float* __restrict__ params, LevelBufs L,
                                const int* __restrict__ counts, const int* __restrict__ digit_k,
                                const int* __restrict__ parent_k, const int* __restrict__ digit0,
                                const int* __restrict__ seg, const int* __restrict__ spos,
                                float* __restrict__ out, const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  const int cnt = ld_count(&counts[k]);
  const int64_t rows = c.rows[k], cols = c.cols[k], K = c.R[k];
  const int64_t per = rows * cols;
  const int64_t total = (int64_t)cnt * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int nd = (int)(t / per);
    const int64_t e = t - (int64_t)nd * per;
    const int64_t a = e / cols, col = e - a * cols;
    const float* A = level_A(c, params, L, parent_k, digit0, k, nd) + a * K;
    const float* S = params + c.core_off[k] + (int64_t)digit_k[nd] * c.slice[k] + col;
    float acc = 0.f;
    for (int64_t r = 0; r < K; ++r) acc = fmaf(A[r], S[r * cols], acc);
    if (k + 1 < c.d) {
      L.P[k][t] = acc;
    } else if (e < c.emb_dim) {  // output column j = e (R_d = 1), truncated (tt_embedding.cpp:122)
      for (int s = seg[nd], se = seg[nd + 1]; s < se; ++s) out[(int64_t)spos[s] * c.emb_dim + e] = acc;
    }
  }
}

// dP[d-1][u][j] = sum over the ID's batch positions (ascending) of the
// upstream row, zero-padded beyond emb_dim (autodiff.cpp:96-97).
__global__ void k_gen_dy(DevCfg c, const float* __restrict__ up, const int* __restrict__ counts,
                         const int* __restrict__ seg, const int* __restrict__ spos, float* __restrict__ dY,
                         const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  const int U = ld_count(&counts[c.d - 1]);
  const int64_t per = c.npad, total = (int64_t)U * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(t / per);
    const int64_t j = t - (int64_t)u * per;
    float acc = 0.f;
    if (j < c.emb_dim)
      for (int s = seg[u], se = seg[u + 1]; s < se; ++s) acc += up[(int64_t)spos[s] * c.emb_dim + j];
    dY[t] = acc;
  }
}

// dPc[k][nd] (rows x R_k) = dP[k][nd] (rows x cols) . G_k[i]^T
__global__ void k_gen_bwd_input(DevCfg c, int k, const float* __restrict__ params, LevelBufs L,
                                const int* __restrict__ counts, const int* __restrict__ digit_k,
                                const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  const int cnt = ld_count(&counts[k]);
  const int64_t rows = c.rows[k], cols = c.cols[k], K = c.R[k];
  const int64_t per = rows * K, total = (int64_t)cnt * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int nd = (int)(t / per);
    const int64_t e = t - (int64_t)nd * per;
    const int64_t a = e / K, r = e - a * K;
    const float* dP = L.dP[k] + (int64_t)nd * rows * cols + a * cols;
    const float* S = params + c.core_off[k] + (int64_t)digit_k[nd] * c.slice[k] + r * cols;
    float acc = 0.f;
    for (int64_t q = 0; q < cols; ++q) acc = fmaf(dP[q], S[q], acc);
    L.dPc[k][t] = acc;
  }
}

// dG_k[v] (R_k x cols) = sum over the digit-v group (node order) of
// A_nd^T . dP[k][nd]; one thread per (v, r, col); a fixed-order segmented
// reduction, no atomics.  Writes only touched slices.
__global__ void k_gen_bwd_weight(DevCfg c, int k, const float* __restrict__ params, LevelBufs L,
                                 const int* __restrict__ goff, const int* __restrict__ order,
                                 const int* __restrict__ parent_k, const int* __restrict__ digit0,
                                 float* __restrict__ grads, const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  const int64_t rows = c.rows[k], cols = c.cols[k], K = c.R[k];
  const int64_t per = K * cols, total = c.m[k] * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(t / per);
    const int64_t e = t - (int64_t)v * per;
    const int64_t r = e / cols, col = e - r * cols;
    const int g0 = goff[v], g1 = goff[v + 1];
    if (g0 == g1) continue;
    float acc = 0.f;
    for (int gi = g0; gi < g1; ++gi) {
      const int nd = order[gi];
      const float* A = level_A(c, params, L, parent_k, digit0, k, nd);
      const float* dP = L.dP[k] + (int64_t)nd * rows * cols + col;
      for (int64_t a = 0; a < rows; ++a) acc = fmaf(A[a * K + r], dP[a * cols], acc);
    }
    grads[c.core_off[k] + (int64_t)v * c.slice[k] + e] = acc;
  }
}

// dP[k-1][p] = sum of dPc[k][children of p] (children contiguous, ascending)
__global__ void k_gen_reduce_children(DevCfg c, int k, LevelBufs L, const int* __restrict__ counts,
                                      const int* __restrict__ cstart_km1, const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  const int cnt = ld_count(&counts[k - 1]);
  const int64_t per = c.rows[k] * c.R[k], total = (int64_t)cnt * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(t / per);
    const int64_t e = t - (int64_t)p * per;
    float acc = 0.f;
    for (int ch = cstart_km1[p], ce = cstart_km1[p + 1]; ch < ce; ++ch) acc += L.dPc[k][(int64_t)ch * per + e];
    L.dP[k - 1][t] = acc;
  }
}

// dG_0[i_1] = dP[0][node] (level-0 nodes are distinct digits)
__global__ void k_gen_bwd_core0(DevCfg c, LevelBufs L, const int* __restrict__ counts,
                                const int* __restrict__ digit0, float* __restrict__ grads, const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  const int cnt = ld_count(&counts[0]);
  const int64_t per = c.cols[0], total = (int64_t)cnt * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int nd = (int)(t / per);
    const int64_t e = t - (int64_t)nd * per;
    grads[c.core_off[0] + (int64_t)digit0[nd] * c.slice[0] + e] = L.dP[0][t];
  }
}

// touch counters: tc[k][v] = nodes with digit v at level k (0 = untouched);
// all levels in one launch (blockIdx.y = level)
struct GoffPtrs {
  const int* goff[TT_MAXD];
};
__global__ void k_touch_counters(DevCfg c, GoffPtrs gp, float* __restrict__ grads, int accumulate,
                                 const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  const int k = blockIdx.y;
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= c.m[k]) return;
  const int* goff = gp.goff[k];
  const float cnt = (float)(goff[v + 1] - goff[v]);
  float* tc = grads + c.tc_off[k] + v;
  *tc = accumulate ? *tc + cnt : cnt;
}

}  // namespace tt
