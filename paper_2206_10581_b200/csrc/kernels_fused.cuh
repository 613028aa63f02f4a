// kernels_fused.cuh -- the fused fast path for the last two cores.
//
// Level F = d-2 (0-based) holds the distinct prefixes (i_1..i_{d-1}).  Its
// products P_F = P_{F-1}[parent] . G_F[i_{d-1}] are grouped by the digit
// i_{d-1}, so every node of a group multiplies the SAME core slice: a group is
// one GEMM  C (rows x NC) = A (rows x K) . S (K x NC)  with
//   rows = (#nodes) x RP,  RP = prod_{p<F} n_p,  K = R_F,  NC = n_F R_{F+1},
// where A stacks the parents' products (the core-0 slices when F = 1).  One
// CTA owns a (group, column block) unit: the BN-column block of the slice is
// staged once in shared memory (cp.async) and reused by every row tile of the
// group; a tile is BM = 64 rows; 256 threads each own a register micro-tile;
// the contraction is warp-level FFMA (fp32) out of shared memory.
//
// Forward epilogue: the last level (R_d = 1) is applied straight from the C
// tile in shared memory -- for every distinct ID under the tile's nodes,
// out[(a, j_F, j_l)] = sum_r C[a][(j_F, r)] G_{d-1}[r, i_d, j_l] -- and the
// row is written to every batch position holding that ID.  The C tile is also
// saved (P_F) for the backward (the autograd pattern; no recompute).
//
// Backward per unit: for each row tile
//   W_u  (R_{F+1} x n_l)  = P_F[u's prefix]^T . dY_u    (dG_{d-1} partials)
//   dC   (rows x BN)      = sum_u dY_u . G_{d-1}[i_d(u)]^T   (dP_F)
//   dG_F block (K x BN)  += A^T . dC                  (registers, whole group)
//   dA   (rows x K)       = dC . S_block^T              (dP_{F-1} partials)
// so dG_F needs no atomics (one CTA per slice column block), and the W / dA
// partials are reduced afterwards by sorted segmented reductions in a fixed
// order (k_fused_reduce_last, k_fused_reduce_children).
#pragma once
#include "common.cuh"

namespace tt {

constexpr int FB_THREADS = 256;
constexpr int FB_BM = 64;
constexpr int FB_CH = 16;  // distinct IDs staged per chunk in the backward

struct FusedShape {
  int ok;
  int F;       // fused level (d-2)
  int K;       // R_F
  int BN;      // column block
  int ncb;     // NC / BN
  int NC;      // n_F R_{F+1}
  int RP;      // rows per node at level F
  int R2;      // R_{F+1}
  int NL;      // n_{d-1}
  int nF;      // n_F
  int BNj;     // BN / R2
  int OUT;     // RP * BNj * NL outputs per ID per column block
  size_t smem_fwd, smem_bwd;
};

struct FusedBufs {
  float* Psave = nullptr;  // [capk[F]][RP][NC]
  float* W = nullptr;      // [capk[d-1]][ncb][R2*NL]
  float* dPc = nullptr;    // [capk[F]][ncb][RP*K]
  int64_t cap_nodes = 0, cap_ids = 0;
};

inline void free_fused(FusedBufs& b) {
  cudaFree(b.Psave);
  cudaFree(b.W);
  cudaFree(b.dPc);
  b = FusedBufs{};
}

struct FusedArgs {
  DevCfg c;
  int F, ncb, RP, R2, NL, nF, BNj, OUT, NC;
  const float* params;
  const float* Aprev;       // P_{F-1} buffer (F >= 2) or nullptr (F == 1: core-0 slices)
  const int* digitF;        // level-F node digits
  const int* parentF;       // level-F node parents
  const int* digit0;        // level-0 digits (F == 1)
  const int* goffF;         // group offsets over level-F digits
  const int* orderF;        // level-F nodes in digit order
  const int* cstartF;       // level-F node -> range of distinct IDs
  const int* digitL;        // digits i_d of the distinct IDs
  const int* seg;           // distinct ID -> sorted batch slots
  const int* spos;          // sorted slot -> batch position
  float* out;               // forward rows (nullptr: no row output)
  float* Psave;
  const float* up;          // backward upstream rows
  float* W;
  float* dPc;
  float* grads;
  const DevStatus* st;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

__device__ __forceinline__ const float* fused_A(const FusedArgs& a, int node) {
  const int p = a.parentF[node];
  if (a.F == 1) return a.params + a.c.core_off[0] + (int64_t)a.digit0[p] * a.c.slice[0];
  return a.Aprev + (int64_t)p * a.RP * a.c.R[a.F];
}

// Stage the (K x BN) column block cb of slice g of core F: Bs[k][n], row stride SB.
template <int K, int BN>
__device__ __forceinline__ void load_slice_block(const FusedArgs& a, int g, int cb, float* Bs) {
  constexpr int SB = BN + 4;
  const float* src = a.params + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F] + cb * BN;
  for (int i = threadIdx.x; i < K * BN / 4; i += FB_THREADS) {
    const int k = i / (BN / 4), q = i - k * (BN / 4);
    cp_async16(Bs + k * SB + q * 4, src + (int64_t)k * a.NC + q * 4);
  }
}

// Per-tile node list and the prefix of their distinct-ID counts.
__device__ __forceinline__ int tile_nodes(const FusedArgs& a, int t0, int nn, int* s_node, int* s_pref) {
  if (threadIdx.x < 32) {
    int run = 0;
    for (int base = 0; base < nn; base += 32) {
      const int j = base + threadIdx.x;
      int node = 0, cnt = 0;
      if (j < nn) {
        node = a.orderF[t0 + j];
        cnt = a.cstartF[node + 1] - a.cstartF[node];
      }
      int x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if ((int)lane_id() >= o) x += y;
      }
      if (j < nn) {
        s_node[j] = node;
        s_pref[j] = run + x - cnt;
      }
      run += __shfl_sync(0xffffffffu, x, 31);
    }
    if (threadIdx.x == 0) s_pref[nn] = run;
  }
  __syncthreads();
  return s_pref[nn];
}

// flat ID index f in [0, total) of the tile -> (node_local j, distinct ID u)
__device__ __forceinline__ int find_node(const int* s_pref, int nn, int f) {
  int lo = 0, hi = nn - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_pref[mid] <= f) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ---------------------------------------------------------------------------
template <int K, int BN>
__global__ void __launch_bounds__(FB_THREADS, 1) k_fused_fwd(FusedArgs a) {
  constexpr int BM = FB_BM, SB = BN + 4, SA = BM + 4, TN = BN / 32;
  extern __shared__ __align__(16) float smem[];
  float* Bs = smem;             // [K][SB]
  float* As = Bs + K * SB;      // [K][SA]  (A transposed)
  float* Cs = As + K * SA;      // [BM][SB]
  int* s_node = (int*)(Cs + BM * SB);
  int* s_pref = s_node + BM + 1;

  if (tt_failed(a.st)) return;
  const int g = blockIdx.x / a.ncb, cb = blockIdx.x - (blockIdx.x / a.ncb) * a.ncb;
  const int g0 = a.goffF[g], g1 = a.goffF[g + 1];
  if (g0 == g1) return;
  load_slice_block<K, BN>(a, g, cb, Bs);
  asm volatile("cp.async.commit_group;\n" ::);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int RP = a.RP, npt = BM / RP;
  const int m0 = warp * 8;
  const int64_t emb = a.c.emb_dim;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];

  for (int t0 = g0; t0 < g1; t0 += npt) {
    const int nn = min(npt, g1 - t0);
    const int total_ids = tile_nodes(a, t0, nn, s_node, s_pref);
    // A tile, transposed: As[k][j*RP + r]
    for (int i = threadIdx.x; i < BM * K; i += FB_THREADS) {
      const int m = i / K, k = i - m * K;
      const int j = m / RP;
      float v = 0.f;
      if (j < nn) v = fused_A(a, s_node[j])[(m - j * RP) * K + k];
      As[k * SA + m] = v;
    }
    cp_async_wait_all();
    __syncthreads();

    float acc[8][TN];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
#pragma unroll 4
    for (int k = 0; k < K; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(As + k * SA + m0);
      const float4 a1 = *reinterpret_cast<const float4*>(As + k * SA + m0 + 4);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float bv[TN];
      if constexpr (TN >= 4) {
#pragma unroll
        for (int q = 0; q < TN / 4; ++q) {
          const float4 b = *reinterpret_cast<const float4*>(Bs + k * SB + q * 128 + lane * 4);
          bv[q * 4 + 0] = b.x; bv[q * 4 + 1] = b.y; bv[q * 4 + 2] = b.z; bv[q * 4 + 3] = b.w;
        }
      } else {
        const float2 b = *reinterpret_cast<const float2*>(Bs + k * SB + lane * 2);
        bv[0] = b.x; bv[1] = b.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    // C -> shared (epilogue) and -> saved P_F (backward)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = m0 + i;
      const int j = m / RP;
      float* crow = Cs + m * SB;
      float* prow = (a.Psave && j < nn)
                        ? a.Psave + ((int64_t)s_node[j] * RP + (m - j * RP)) * a.NC + cb * BN : nullptr;
      if constexpr (TN >= 4) {
#pragma unroll
        for (int q = 0; q < TN / 4; ++q) {
          const float4 v = make_float4(acc[i][q * 4], acc[i][q * 4 + 1], acc[i][q * 4 + 2], acc[i][q * 4 + 3]);
          *reinterpret_cast<float4*>(crow + q * 128 + lane * 4) = v;
          if (prow) *reinterpret_cast<float4*>(prow + q * 128 + lane * 4) = v;
        }
      } else {
        const float2 v = make_float2(acc[i][0], acc[i][1]);
        *reinterpret_cast<float2*>(crow + lane * 2) = v;
        if (prow) *reinterpret_cast<float2*>(prow + lane * 2) = v;
      }
    }
    __syncthreads();
    // last level straight from the C tile
    if (a.out) {
      const int OUT = a.OUT, R2 = a.R2, NL = a.NL, BNj = a.BNj;
      for (int f = threadIdx.x; f < total_ids * OUT; f += FB_THREADS) {
        const int idf = f / OUT, o = f - idf * OUT;
        const int j = find_node(s_pref, nn, idf);
        const int u = a.cstartF[s_node[j]] + (idf - s_pref[j]);
        const int ar = o / (BNj * NL), rem = o - ar * (BNj * NL);
        const int jf = rem / NL, jl = rem - jf * NL;
        const float* crow = Cs + (j * RP + ar) * SB + jf * R2;
        const float* gl = Gl + (int64_t)a.digitL[u] * sliceL + jl;
        float v = 0.f;
        for (int r = 0; r < R2; ++r) v = fmaf(crow[r], __ldg(gl + r * NL), v);
        const int64_t col = ((int64_t)(ar * a.nF + cb * BNj + jf)) * NL + jl;
        if (col < emb)
          for (int s = a.seg[u], se = a.seg[u + 1]; s < se; ++s) a.out[(int64_t)a.spos[s] * emb + col] = v;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
template <int K, int BN>
__global__ void __launch_bounds__(FB_THREADS, 1) k_fused_bwd(FusedArgs a) {
  constexpr int BM = FB_BM, SB = BN + 4, SA = K + 4, TN = BN / 32, TK = K / 8;
  constexpr int KG = K < 16 ? K : 16, MG = FB_THREADS / KG, TKA = K / KG, TMA = BM / MG;
  extern __shared__ __align__(16) float smem[];
  float* Bs = smem;               // [K][SB]
  float* As = Bs + K * SB;        // [BM][SA]  (A row-major)
  float* Cs = As + BM * SA;       // [BM][SB]  C, then dC
  float* Ys = Cs + BM * SB;       // [FB_CH][OUT] staged dY
  int* s_node = (int*)(Ys + FB_CH * 256);
  int* s_pref = s_node + BM + 1;

  if (tt_failed(a.st)) return;
  const int g = blockIdx.x / a.ncb, cb = blockIdx.x - (blockIdx.x / a.ncb) * a.ncb;
  const int g0 = a.goffF[g], g1 = a.goffF[g + 1];
  if (g0 == g1) return;
  load_slice_block<K, BN>(a, g, cb, Bs);
  asm volatile("cp.async.commit_group;\n" ::);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int RP = a.RP, npt = BM / RP;
  const int OUT = a.OUT, R2 = a.R2, NL = a.NL, BNj = a.BNj;
  const int64_t emb = a.c.emb_dim;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];
  const int WE = R2 * NL;

  float gacc[TK][TN];
#pragma unroll
  for (int i = 0; i < TK; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) gacc[i][j] = 0.f;

  for (int t0 = g0; t0 < g1; t0 += npt) {
    const int nn = min(npt, g1 - t0);
    const int total_ids = tile_nodes(a, t0, nn, s_node, s_pref);
    // A tile row-major; saved C tile
    for (int i = threadIdx.x; i < BM * K; i += FB_THREADS) {
      const int m = i / K, k = i - m * K;
      const int j = m / RP;
      As[m * SA + k] = j < nn ? fused_A(a, s_node[j])[(m - j * RP) * K + k] : 0.f;
    }
    for (int i = threadIdx.x; i < BM * BN / 4; i += FB_THREADS) {
      const int m = i / (BN / 4), q = i - m * (BN / 4);
      const int j = m / RP;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j < nn)
        v = *reinterpret_cast<const float4*>(a.Psave + ((int64_t)s_node[j] * RP + (m - j * RP)) * a.NC + cb * BN + q * 4);
      *reinterpret_cast<float4*>(Cs + m * SB + q * 4) = v;
    }
    cp_async_wait_all();
    __syncthreads();

    // pass 1: W_u = C^T dY_u for every distinct ID of the tile
    for (int c0 = 0; c0 < total_ids; c0 += FB_CH) {
      const int nc = min(FB_CH, total_ids - c0);
      for (int f = threadIdx.x; f < nc * OUT; f += FB_THREADS) {
        const int ci = f / OUT, o = f - ci * OUT;
        const int j = find_node(s_pref, nn, c0 + ci);
        const int u = a.cstartF[s_node[j]] + (c0 + ci - s_pref[j]);
        const int ar = o / (BNj * NL), rem = o - ar * (BNj * NL);
        const int jf = rem / NL, jl = rem - jf * NL;
        const int64_t col = ((int64_t)(ar * a.nF + cb * BNj + jf)) * NL + jl;
        float v = 0.f;
        if (col < emb)
          for (int s = a.seg[u], se = a.seg[u + 1]; s < se; ++s) v += a.up[(int64_t)a.spos[s] * emb + col];
        Ys[ci * OUT + o] = v;
      }
      __syncthreads();
      for (int f = threadIdx.x; f < nc * WE; f += FB_THREADS) {
        const int ci = f / WE, e = f - ci * WE;
        const int r = e / NL, jl = e - r * NL;
        const int j = find_node(s_pref, nn, c0 + ci);
        const int u = a.cstartF[s_node[j]] + (c0 + ci - s_pref[j]);
        float v = 0.f;
        for (int ar = 0; ar < RP; ++ar)
          for (int jf = 0; jf < BNj; ++jf)
            v = fmaf(Cs[(j * RP + ar) * SB + jf * R2 + r], Ys[ci * OUT + (ar * BNj + jf) * NL + jl], v);
        a.W[((int64_t)u * a.ncb + cb) * WE + e] = v;
      }
      __syncthreads();
    }
    // pass 2: dC (overwrites C) = sum over the node's IDs of dY_u G_l(u)^T
    for (int i = threadIdx.x; i < BM * BN; i += FB_THREADS) Cs[(i / BN) * SB + (i % BN)] = 0.f;
    __syncthreads();
    for (int c0 = 0; c0 < total_ids; c0 += FB_CH) {
      const int nc = min(FB_CH, total_ids - c0);
      for (int f = threadIdx.x; f < nc * OUT; f += FB_THREADS) {
        const int ci = f / OUT, o = f - ci * OUT;
        const int j = find_node(s_pref, nn, c0 + ci);
        const int u = a.cstartF[s_node[j]] + (c0 + ci - s_pref[j]);
        const int ar = o / (BNj * NL), rem = o - ar * (BNj * NL);
        const int jf = rem / NL, jl = rem - jf * NL;
        const int64_t col = ((int64_t)(ar * a.nF + cb * BNj + jf)) * NL + jl;
        float v = 0.f;
        if (col < emb)
          for (int s = a.seg[u], se = a.seg[u + 1]; s < se; ++s) v += a.up[(int64_t)a.spos[s] * emb + col];
        Ys[ci * OUT + o] = v;
      }
      __syncthreads();
      const int jlo = find_node(s_pref, nn, c0), jhi = find_node(s_pref, nn, c0 + nc - 1);
      const int rows = (jhi - jlo + 1) * RP;
      for (int i = threadIdx.x; i < rows * BN; i += FB_THREADS) {
        const int mm = i / BN, n = i - mm * BN;
        const int m = jlo * RP + mm;
        const int j = m / RP, ar = m - j * RP;
        const int jf = n / R2, r = n - jf * R2;
        const int u0 = max(s_pref[j], c0), u1 = min(s_pref[j + 1], c0 + nc);
        float v = Cs[m * SB + n];
        for (int f = u0; f < u1; ++f) {
          const int u = a.cstartF[s_node[j]] + (f - s_pref[j]);
          const float* gl = Gl + (int64_t)a.digitL[u] * sliceL + r * NL;
          const float* y = Ys + (f - c0) * OUT + (ar * BNj + jf) * NL;
          for (int jl = 0; jl < NL; ++jl) v = fmaf(y[jl], __ldg(gl + jl), v);
        }
        Cs[m * SB + n] = v;
      }
      __syncthreads();
    }
    // dG_F block += A^T dC  (k rows warp*TK.., columns as in the forward)
#pragma unroll 2
    for (int m = 0; m < BM; ++m) {
      float av[TK];
#pragma unroll
      for (int q = 0; q < TK; q += 4) {
        if constexpr (TK >= 4) {
          const float4 t = *reinterpret_cast<const float4*>(As + m * SA + warp * TK + q);
          av[q] = t.x; av[q + 1] = t.y; av[q + 2] = t.z; av[q + 3] = t.w;
        }
      }
      if constexpr (TK < 4) {
#pragma unroll
        for (int q = 0; q < TK; ++q) av[q] = As[m * SA + warp * TK + q];
      }
      float bv[TN];
      if constexpr (TN >= 4) {
#pragma unroll
        for (int q = 0; q < TN / 4; ++q) {
          const float4 b = *reinterpret_cast<const float4*>(Cs + m * SB + q * 128 + lane * 4);
          bv[q * 4 + 0] = b.x; bv[q * 4 + 1] = b.y; bv[q * 4 + 2] = b.z; bv[q * 4 + 3] = b.w;
        }
      } else {
        const float2 b = *reinterpret_cast<const float2*>(Cs + m * SB + lane * 2);
        bv[0] = b.x; bv[1] = b.y;
      }
#pragma unroll
      for (int i = 0; i < TK; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) gacc[i][j] = fmaf(av[i], bv[j], gacc[i][j]);
    }
    // dA = dC . S_block^T  -> per-(node, column block) partials
    {
      const int kg = threadIdx.x % KG, mg = threadIdx.x / KG;
      float dacc[TMA][TKA];
#pragma unroll
      for (int i = 0; i < TMA; ++i)
#pragma unroll
        for (int j = 0; j < TKA; ++j) dacc[i][j] = 0.f;
#pragma unroll 2
      for (int n = 0; n < BN; n += 4) {
        float4 cv[TMA], bv[TKA];
#pragma unroll
        for (int i = 0; i < TMA; ++i) cv[i] = *reinterpret_cast<const float4*>(Cs + (mg + MG * i) * SB + n);
#pragma unroll
        for (int j = 0; j < TKA; ++j) bv[j] = *reinterpret_cast<const float4*>(Bs + (kg + KG * j) * SB + n);
#pragma unroll
        for (int i = 0; i < TMA; ++i)
#pragma unroll
          for (int j = 0; j < TKA; ++j) {
            dacc[i][j] = fmaf(cv[i].x, bv[j].x, dacc[i][j]);
            dacc[i][j] = fmaf(cv[i].y, bv[j].y, dacc[i][j]);
            dacc[i][j] = fmaf(cv[i].z, bv[j].z, dacc[i][j]);
            dacc[i][j] = fmaf(cv[i].w, bv[j].w, dacc[i][j]);
          }
      }
#pragma unroll
      for (int i = 0; i < TMA; ++i) {
        const int m = mg + MG * i;
        const int j = m / RP;
        if (j >= nn) continue;
        float* dst = a.dPc + ((int64_t)s_node[j] * a.ncb + cb) * RP * K + (m - j * RP) * K;
#pragma unroll
        for (int jj = 0; jj < TKA; ++jj) dst[kg + KG * jj] = dacc[i][jj];
      }
    }
    __syncthreads();
  }
  // the group's dG_F column block (one writer per slice block: no atomics)
  float* gdst = a.grads + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F] + cb * BN;
#pragma unroll
  for (int i = 0; i < TK; ++i) {
    float* row = gdst + (int64_t)(warp * TK + i) * a.NC;
    if constexpr (TN >= 4) {
#pragma unroll
      for (int q = 0; q < TN / 4; ++q)
        *reinterpret_cast<float4*>(row + q * 128 + lane * 4) =
            make_float4(gacc[i][q * 4], gacc[i][q * 4 + 1], gacc[i][q * 4 + 2], gacc[i][q * 4 + 3]);
    } else {
      *reinterpret_cast<float2*>(row + lane * 2) = make_float2(gacc[i][0], gacc[i][1]);
    }
  }
}

// dG_{d-1}[v] = sum over the digit-v IDs (group order) and column blocks of W
__global__ void k_fused_reduce_last(DevCfg c, int ncb, int WE, const int* __restrict__ goffL,
                                    const int* __restrict__ orderL, const float* __restrict__ W,
                                    float* __restrict__ grads, const DevStatus* st) {
  if (tt_failed(st)) return;
  const int v = blockIdx.x;
  const int g0 = goffL[v], g1 = goffL[v + 1];
  if (g0 == g1) return;
  for (int e = threadIdx.x; e < WE; e += blockDim.x) {
    float acc = 0.f;
    for (int gi = g0; gi < g1; ++gi) {
      const float* w = W + (int64_t)orderL[gi] * ncb * WE + e;
      for (int cbi = 0; cbi < ncb; ++cbi) acc += w[cbi * WE];
    }
    grads[c.core_off[c.d - 1] + (int64_t)v * c.slice[c.d - 1] + e] = acc;
  }
}

// dP_{F-1}[p] (or dG_0 when F == 1) = sum over children and column blocks of dPc
__global__ void k_fused_reduce_children(DevCfg c, int F, int ncb, int per, const int* __restrict__ counts,
                                        const int* __restrict__ cstart_pm1, const int* __restrict__ digit0,
                                        const float* __restrict__ dPc, float* __restrict__ dst,
                                        const DevStatus* st) {
  if (tt_failed(st)) return;
  const int cnt = ld_count(&counts[F - 1]);
  const int64_t total = (int64_t)cnt * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(t / per);
    const int e = (int)(t - (int64_t)p * per);
    float acc = 0.f;
    for (int ch = cstart_pm1[p], ce = cstart_pm1[p + 1]; ch < ce; ++ch) {
      const float* src = dPc + (int64_t)ch * ncb * per + e;
      for (int cbi = 0; cbi < ncb; ++cbi) acc += src[cbi * per];
    }
    if (F == 1)
      dst[c.core_off[0] + (int64_t)digit0[p] * c.slice[0] + e] = acc;
    else
      dst[t] = acc;
  }
}

// Shape admission for the fused path (host).
inline bool fused_plan_shape(const DevCfg& c, FusedShape* s) {
  *s = FusedShape{};
  if (c.d < 3) return false;
  const int F = c.d - 2;
  const int64_t K = c.R[F], NC = c.cols[F], R2 = c.R[F + 1], NL = c.n[c.d - 1], RP = c.rows[F];
  int BN = 0;
  if (K == 16 && NC % 64 == 0 && 64 % R2 == 0) BN = 64;
  if (K == 32 && NC % 128 == 0 && 128 % R2 == 0) BN = 128;
  if (K == 64 && NC % 256 == 0 && 256 % R2 == 0) BN = 256;
  if (K == 64 && !BN && NC % 128 == 0 && 128 % R2 == 0) BN = 128;
  if (K == 128 && NC % 128 == 0 && 128 % R2 == 0) BN = 128;
  if (!BN) return false;
  if (RP > FB_BM || FB_BM % RP) return false;
  const int64_t OUT = RP * (BN / R2) * NL;
  if (OUT > 256 || R2 * NL > 4096) return false;
  for (int k = 0; k < c.d; ++k)
    if (c.core_off[k] % 4 || c.slice[k] % 4) return false;
  s->ok = 1;
  s->F = F;
  s->K = (int)K;
  s->BN = BN;
  s->NC = (int)NC;
  s->ncb = (int)(NC / BN);
  s->RP = (int)RP;
  s->R2 = (int)R2;
  s->NL = (int)NL;
  s->nF = (int)c.n[F];
  s->BNj = (int)(BN / R2);
  s->OUT = (int)OUT;
  const int SB = BN + 4;
  s->smem_fwd = sizeof(float) * ((size_t)K * SB + (size_t)K * (FB_BM + 4) + (size_t)FB_BM * SB) +
                sizeof(int) * (2 * FB_BM + 4);
  s->smem_bwd = sizeof(float) * ((size_t)K * SB + (size_t)FB_BM * (K + 4) + (size_t)FB_BM * SB + FB_CH * 256) +
                sizeof(int) * (2 * FB_BM + 4);
  return true;
}

}  // namespace tt
