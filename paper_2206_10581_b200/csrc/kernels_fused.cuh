// kernels_fused.cuh -- the fused fast path for the last two cores.
//
// Level F = d-2 (0-based) holds the distinct prefixes (i_1..i_{d-1}).  Its
// products P_F = P_{F-1}[parent] . G_F[i_{d-1}] are grouped by the digit
// i_{d-1}, so every node of a group multiplies the SAME core slice: a group is
// one GEMM  C (rows x NC) = A (rows x K) . S (K x NC)  with
//   rows = (#nodes) x RP,  RP = prod_{p<F} n_p,  K = R_F,  NC = n_F R_{F+1},
// where A stacks the parents' products (the core-0 slices when F = 1).  One
// CTA owns a (group, column block) unit: the K x BN block of the slice is
// staged once in shared memory (cp.async) and reused by every 64-row tile of
// the group; A tiles arrive by cp.async (double-buffered in the forward);
// 256 threads each own a register micro-tile and contract with warp-level
// FFMA (fp32) out of shared memory.  Ranks are uniform on this path
// (R_{F+1} = R_F = K).
//
// Forward epilogue: the last level (R_d = 1) is applied from the C tile in
// shared memory -- for every distinct ID under the tile's nodes,
// out[(a, j_F, j_l)] = sum_r C[a][(j_F, r)] G_{d-1}[r, i_d, j_l] (slices staged
// transposed in shared memory) -- and written to the ID's batch positions
// (IDs with more than HEAVY_POS positions go through Yu and the balanced
// k_scatter_heavy).  The C tile is saved (P_F) for the backward.
//
// Backward per unit, for each row tile (C-tile load overlapped with compute):
//   dC   (rows x BN)      = sum_u dY_u . G_{d-1}[i_d(u)]^T        (dP_F)
//   dG_F block (K x BN)  += A^T . dC      (registers across the whole group)
//   dA   (rows x K)       = dC . S_block^T  -> dP_{F-1} partials
//   W_u  (K x n_l)        = C_u^T . dY_u    -> dG_{d-1} partials
// dG_F needs no atomics (one CTA per slice column block); the W / dA partials
// are reduced by sorted segmented reductions in a fixed order
// (k_fused_reduce_last, k_fused_reduce_children).
#pragma once
#include "common.cuh"
#include "kernels_rows.cuh"

namespace tt {

constexpr int FB_THREADS = 256;
constexpr int FB_BM = 64;
constexpr int FB_SMEM_MAX = 227 * 1024;

struct FusedShape {
  int ok;
  int F;       // fused level (d-2)
  int K;       // R_F = R_{F+1}
  int BN;      // column block
  int ncb;     // NC / BN
  int NC;      // n_F R_{F+1}
  int RP;      // rows per node at level F
  int NL;      // n_{d-1}
  int nF;      // n_F
  int BNj;     // BN / K
  int OUT;     // RP * BNj * NL outputs per ID per column block
  int CHF, CHB;            // distinct IDs staged per chunk (fwd / bwd)
  size_t smem_fwd, smem_bwd;
};

struct FusedBufs {
  float* Psave = nullptr;  // [capk[F]][RP][NC]
  float* W = nullptr;      // [capk[d-1]][ncb][K*NL]
  float* dPc = nullptr;    // [capk[F]][ncb][RP*K]
  float* dY = nullptr;     // [capk[d-1]][npad]   upstream summed per distinct ID
  float* Yu = nullptr;     // [capk[d-1]][npad]   rows of heavy IDs
  float* part = nullptr;   // [chunks][2][npad]   k_dy_chunks partials
  int64_t cap_nodes = 0, cap_ids = 0, cap_chunks = 0;
};

inline void free_fused(FusedBufs& b) {
  cudaFree(b.Psave);
  cudaFree(b.W);
  cudaFree(b.dPc);
  cudaFree(b.dY);
  cudaFree(b.Yu);
  cudaFree(b.part);
  b = FusedBufs{};
}

struct FusedArgs {
  DevCfg c;
  int F, ncb, RP, NL, nF, BNj, OUT, NC, CH;
  const float* params;
  const float* Abase;       // core-0 parameters (F == 1) or the P_{F-1} buffer
  const int* parentF;       // level-F node parents
  const int* digit0;        // level-0 digits (F == 1)
  const int* goffF;         // group offsets over level-F digits
  const int* orderF;        // level-F nodes in digit order
  const int* cstartF;       // level-F node -> range of distinct IDs
  const int* digitL;        // digits i_d of the distinct IDs
  const int* seg;           // distinct ID -> sorted batch slots
  const int* spos;          // sorted slot -> batch position
  float* out;               // forward rows (nullptr: no row output)
  float* Yu;
  float* Psave;
  const float* dY;
  float* W;
  float* dPc;
  float* grads;
  const DevStatus* st;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Stage the (K x BN) column block cb of slice g of core F: Bs[k][n], row stride SB.
template <int K, int BN, int SB>
__device__ __forceinline__ void load_slice_block(const FusedArgs& a, int g, int cb, float* Bs) {
  const float* src = a.params + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F] + cb * BN;
  for (int i = threadIdx.x; i < K * BN / 4; i += FB_THREADS) {
    const int k = i / (BN / 4), q = i - k * (BN / 4);
    cp_async16(Bs + k * SB + q * 4, src + (int64_t)k * a.NC + q * 4);
  }
}

// Node list of the tile starting at group slot t0: node ids, prefix of their
// distinct-ID counts, and each node's A-block offset.  Ends with a barrier.
__device__ __forceinline__ int tile_nodes(const FusedArgs& a, int t0, int nn, int* s_node, int* s_pref,
                                          int64_t* s_aoff) {
  if (threadIdx.x < 32) {
    int run = 0;
    for (int base = 0; base < nn; base += 32) {
      const int j = base + threadIdx.x;
      int node = 0, cnt = 0;
      if (j < nn) {
        node = a.orderF[t0 + j];
        cnt = a.cstartF[node + 1] - a.cstartF[node];
        const int p = a.parentF[node];
        s_aoff[j] = a.F == 1 ? a.c.core_off[0] + (int64_t)a.digit0[p] * a.c.slice[0]
                             : (int64_t)p * a.RP * a.c.R[a.F];
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

// A tile (BM x K, row-major, stride K) by cp.async; rows past the tile's
// nodes are zero-filled.
template <int K>
__device__ __forceinline__ void load_A_tile(const FusedArgs& a, int nn, const int64_t* s_aoff, float* As) {
  const int RP = a.RP;
  for (int i = threadIdx.x; i < FB_BM * K / 4; i += FB_THREADS) {
    const int m = i / (K / 4), q = i - m * (K / 4);
    const int j = m / RP;
    float* dst = As + m * K + q * 4;
    if (j < nn) cp_async16(dst, a.Abase + s_aoff[j] + (m - j * RP) * K + q * 4);
    else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// flat distinct-ID index f of the tile -> node_local j (s_pref is ascending)
__device__ __forceinline__ int find_node(const int* s_pref, int nn, int f) {
  int lo = 0, hi = nn - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_pref[mid] <= f) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Stage the last-core slices of IDs [c0, c0+nc) of the tile, transposed:
// Gs[(ci*NL + jl)*(K+1) + r] = G_{d-1}[r, i_d(u), jl]; also s_u/s_j.
template <int K>
__device__ __forceinline__ void stage_ids(const FusedArgs& a, int c0, int nc, int nn, const int* s_node,
                                          const int* s_pref, int* s_u, int* s_j, float* Gs, bool want_g) {
  for (int ci = threadIdx.x; ci < nc; ci += FB_THREADS) {
    const int j = find_node(s_pref, nn, c0 + ci);
    s_j[ci] = j;
    s_u[ci] = a.cstartF[s_node[j]] + (c0 + ci - s_pref[j]);
  }
  __syncthreads();
  if (!want_g) return;
  const int NL = a.NL;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];
  for (int i = threadIdx.x; i < nc * K * NL; i += FB_THREADS) {
    const int ci = i / (K * NL), e = i - ci * (K * NL);
    const int r = e / NL, jl = e - r * NL;
    Gs[(ci * NL + jl) * (K + 1) + r] = __ldg(Gl + (int64_t)a.digitL[s_u[ci]] * sliceL + e);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
template <int K, int BN>
__global__ void __launch_bounds__(FB_THREADS, 1) k_fused_fwd(FusedArgs a) {
  constexpr int BM = FB_BM, SB = BN + 4, TN = BN / 32;
  extern __shared__ __align__(16) float smem[];
  float* Bs = smem;                      // [K][SB]
  float* As0 = Bs + K * SB;              // [2][BM][K]
  float* Cs = As0 + 2 * BM * K;          // [BM][BN]
  float* Gs = Cs + BM * BN;              // [CH][NL][K+1]
  int64_t* s_aoff = reinterpret_cast<int64_t*>(Gs + a.CH * a.NL * (K + 1) + ((a.CH * a.NL * (K + 1)) & 1));
  int* s_node = reinterpret_cast<int*>(s_aoff + 2 * BM);   // [2][BM]
  int* s_pref = s_node + 2 * BM;                           // [2][BM+1]
  int* s_u = s_pref + 2 * (BM + 1);                        // [CH]
  int* s_j = s_u + a.CH;                                   // [CH]

  if (tt_failed(a.st)) return;
  const int g = blockIdx.x / a.ncb, cb = blockIdx.x - g * a.ncb;
  const int g0 = a.goffF[g], g1 = a.goffF[g + 1];
  if (g0 == g1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int RP = a.RP, npt = BM / RP, NL = a.NL, BNj = a.BNj, nF = a.nF;
  const int m0 = warp * 8;
  const int64_t emb = a.c.emb_dim, npad = a.c.npad;

  load_slice_block<K, BN, SB>(a, g, cb, Bs);
  int nn = min(npt, g1 - g0);
  tile_nodes(a, g0, nn, s_node, s_pref, s_aoff);
  load_A_tile<K>(a, nn, s_aoff, As0);
  cp_async_commit();

  int buf = 0;
  for (int t0 = g0; t0 < g1; t0 += npt, buf ^= 1) {
    const int t1 = t0 + npt;
    const int nn1 = min(npt, g1 - t1);
    int* nd = s_node + buf * BM;
    int* pf = s_pref + buf * (BM + 1);
    if (t1 < g1) {  // prefetch the next tile's nodes and A
      tile_nodes(a, t1, nn1, s_node + (buf ^ 1) * BM, s_pref + (buf ^ 1) * (BM + 1), s_aoff + (buf ^ 1) * BM);
      load_A_tile<K>(a, nn1, s_aoff + (buf ^ 1) * BM, As0 + (buf ^ 1) * BM * K);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* As = As0 + buf * BM * K;

    float acc[8][TN];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
#pragma unroll 2
    for (int kk = 0; kk < K; kk += 4) {
      float4 av[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) av[i] = *reinterpret_cast<const float4*>(As + (m0 + i) * K + kk);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        float bv[TN];
        if constexpr (TN >= 4) {
#pragma unroll
          for (int q = 0; q < TN / 4; ++q) {
            const float4 b = *reinterpret_cast<const float4*>(Bs + (kk + t) * SB + q * 128 + lane * 4);
            bv[q * 4 + 0] = b.x; bv[q * 4 + 1] = b.y; bv[q * 4 + 2] = b.z; bv[q * 4 + 3] = b.w;
          }
        } else {
          const float2 b = *reinterpret_cast<const float2*>(Bs + (kk + t) * SB + lane * 2);
          bv[0] = b.x; bv[1] = b.y;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float x = t == 0 ? av[i].x : t == 1 ? av[i].y : t == 2 ? av[i].z : av[i].w;
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(x, bv[j], acc[i][j]);
        }
      }
    }
    const int cur_nn = min(npt, g1 - t0);
    // C -> shared (epilogue) and -> saved P_F (backward)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = m0 + i;
      const int j = m / RP;
      float* crow = Cs + m * BN;
      float* prow = (a.Psave && j < cur_nn)
                        ? a.Psave + ((int64_t)nd[j] * RP + (m - j * RP)) * a.NC + cb * BN : nullptr;
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
      const int total_ids = pf[cur_nn];
      for (int c0 = 0; c0 < total_ids; c0 += a.CH) {
        const int nc = min(a.CH, total_ids - c0);
        stage_ids<K>(a, c0, nc, cur_nn, nd, pf, s_u, s_j, Gs, true);
        const int per_row = nc * NL;
        for (int f = threadIdx.x; f < RP * BNj * per_row; f += FB_THREADS) {
          const int rc = f / per_row, e = f - rc * per_row;  // rc = (ar, jf); e = (ci, jl)
          const int ci = e / NL, jl = e - ci * NL;
          const int ar = rc / BNj, jf = rc - ar * BNj;
          const int u = s_u[ci];
          const float* crow = Cs + (s_j[ci] * RP + ar) * BN + jf * K;
          const float* gcol = Gs + (ci * NL + jl) * (K + 1);
          float v = 0.f;
#pragma unroll 16
          for (int r = 0; r < K; ++r) v = fmaf(crow[r], gcol[r], v);
          const int64_t col = ((int64_t)(ar * nF + cb * BNj + jf)) * NL + jl;
          const int s0 = a.seg[u], s1 = a.seg[u + 1];
          if (s1 - s0 > HEAVY_POS) {
            a.Yu[(int64_t)u * npad + col] = v;
          } else if (col < emb) {
            for (int s = s0; s < s1; ++s) a.out[(int64_t)a.spos[s] * emb + col] = v;
          }
        }
        __syncthreads();
      }
    }
  }
}

// ---------------------------------------------------------------------------
template <int K, int BN>
__global__ void __launch_bounds__(FB_THREADS, 1) k_fused_bwd(FusedArgs a) {
  constexpr int BM = FB_BM, SB = BN + 4, TN = BN / 32, TK = K / 8;
  constexpr int KG = K < 16 ? K : 16, MG = FB_THREADS / KG, TKA = K / KG, TMA = BM / MG;
  extern __shared__ __align__(16) float smem[];
  float* Bs = smem;               // [K][SB]
  float* As = Bs + K * SB;        // [BM][K]
  float* Cs = As + BM * K;        // [BM][BN]  saved C (for W)
  float* Ds = Cs + BM * BN;       // [BM][BN]  dC
  float* Ys = Ds + BM * BN;       // [CH][OUT]
  float* Gs = Ys + a.CH * a.OUT;  // [CH][NL][K+1]
  int64_t* s_aoff = reinterpret_cast<int64_t*>(Gs + a.CH * a.NL * (K + 1) + ((a.CH * a.NL * (K + 1) + a.CH * a.OUT) & 1));
  int* s_node = reinterpret_cast<int*>(s_aoff + BM);
  int* s_pref = s_node + BM;
  int* s_u = s_pref + BM + 1;
  int* s_j = s_u + a.CH;

  if (tt_failed(a.st)) return;
  const int g = blockIdx.x / a.ncb, cb = blockIdx.x - g * a.ncb;
  const int g0 = a.goffF[g], g1 = a.goffF[g + 1];
  if (g0 == g1) return;
  load_slice_block<K, BN, SB>(a, g, cb, Bs);
  cp_async_commit();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int RP = a.RP, npt = BM / RP, NL = a.NL, BNj = a.BNj, nF = a.nF, OUT = a.OUT, CH = a.CH;
  const int64_t npad = a.c.npad;
  const int WE = K * NL;

  float gacc[TK][TN];
#pragma unroll
  for (int i = 0; i < TK; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) gacc[i][j] = 0.f;

  for (int t0 = g0; t0 < g1; t0 += npt) {
    const int nn = min(npt, g1 - t0);
    const int total_ids = tile_nodes(a, t0, nn, s_node, s_pref, s_aoff);
    load_A_tile<K>(a, nn, s_aoff, As);
    cp_async_commit();
    for (int i = threadIdx.x; i < BM * BN / 4; i += FB_THREADS) {  // saved C tile (for W, used last)
      const int m = i / (BN / 4), q = i - m * (BN / 4);
      const int j = m / RP;
      float* dst = Cs + m * BN + q * 4;
      if (j < nn) cp_async16(dst, a.Psave + ((int64_t)s_node[j] * RP + (m - j * RP)) * a.NC + cb * BN + q * 4);
      else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    cp_async_commit();
    for (int i = threadIdx.x; i < BM * BN / 4; i += FB_THREADS)
      reinterpret_cast<float4*>(Ds)[i] = make_float4(0.f, 0.f, 0.f, 0.f);

    // dC = sum over each node's IDs of dY_u G_l(u)^T
    for (int c0 = 0; c0 < total_ids; c0 += CH) {
      const int nc = min(CH, total_ids - c0);
      stage_ids<K>(a, c0, nc, nn, s_node, s_pref, s_u, s_j, Gs, true);
      for (int i = threadIdx.x; i < nc * OUT / 4; i += FB_THREADS) {
        const int ci = i / (OUT / 4), q = i - ci * (OUT / 4);
        const int ar = (q * 4) / (BNj * NL), w = q * 4 - ar * (BNj * NL);
        *reinterpret_cast<float4*>(Ys + ci * OUT + q * 4) = *reinterpret_cast<const float4*>(
            a.dY + (int64_t)s_u[ci] * npad + ((int64_t)ar * nF + cb * BNj) * NL + w);
      }
      __syncthreads();
      const int jlo = s_j[0], jhi = s_j[nc - 1];
      const int rows = (jhi - jlo + 1) * RP;
      for (int i = threadIdx.x; i < rows * BN; i += FB_THREADS) {
        const int mm = i / BN, n = i - mm * BN;
        const int m = jlo * RP + mm;
        const int j = m / RP, ar = m - j * RP;
        const int jf = n / K, r = n - jf * K;
        const int f0 = max(s_pref[j], c0) - c0, f1 = min(s_pref[j + 1], c0 + nc) - c0;
        float v = Ds[m * BN + n];
        for (int ci = f0; ci < f1; ++ci) {
          const float* y = Ys + ci * OUT + (ar * BNj + jf) * NL;
          const float* gc = Gs + ci * NL * (K + 1) + r;
          for (int jl = 0; jl < NL; ++jl) v = fmaf(y[jl], gc[jl * (K + 1)], v);
        }
        Ds[m * BN + n] = v;
      }
      __syncthreads();
    }
    cp_async_wait<1>();  // slice block + A tile landed (C may still be in flight)
    __syncthreads();
    // dG_F block += A^T dC
#pragma unroll 2
    for (int m = 0; m < BM; ++m) {
      float av[TK];
      if constexpr (TK >= 4) {
#pragma unroll
        for (int q = 0; q < TK; q += 4) {
          const float4 t = *reinterpret_cast<const float4*>(As + m * K + warp * TK + q);
          av[q] = t.x; av[q + 1] = t.y; av[q + 2] = t.z; av[q + 3] = t.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < TK; ++q) av[q] = As[m * K + warp * TK + q];
      }
      float bv[TN];
      if constexpr (TN >= 4) {
#pragma unroll
        for (int q = 0; q < TN / 4; ++q) {
          const float4 b = *reinterpret_cast<const float4*>(Ds + m * BN + q * 128 + lane * 4);
          bv[q * 4 + 0] = b.x; bv[q * 4 + 1] = b.y; bv[q * 4 + 2] = b.z; bv[q * 4 + 3] = b.w;
        }
      } else {
        const float2 b = *reinterpret_cast<const float2*>(Ds + m * BN + lane * 2);
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
        for (int i = 0; i < TMA; ++i) cv[i] = *reinterpret_cast<const float4*>(Ds + (mg + MG * i) * BN + n);
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
    cp_async_wait<0>();  // saved C tile
    __syncthreads();
    // W_u = C_u^T dY_u  (per distinct ID, this column block's share)
    for (int c0 = 0; c0 < total_ids; c0 += CH) {
      const int nc = min(CH, total_ids - c0);
      stage_ids<K>(a, c0, nc, nn, s_node, s_pref, s_u, s_j, Gs, false);
      for (int i = threadIdx.x; i < nc * OUT / 4; i += FB_THREADS) {
        const int ci = i / (OUT / 4), q = i - ci * (OUT / 4);
        const int ar = (q * 4) / (BNj * NL), w = q * 4 - ar * (BNj * NL);
        *reinterpret_cast<float4*>(Ys + ci * OUT + q * 4) = *reinterpret_cast<const float4*>(
            a.dY + (int64_t)s_u[ci] * npad + ((int64_t)ar * nF + cb * BNj) * NL + w);
      }
      __syncthreads();
      for (int f = threadIdx.x; f < nc * WE; f += FB_THREADS) {
        const int ci = f / WE, e = f - ci * WE;
        const int r = e / NL, jl = e - r * NL;
        const int j = s_j[ci];
        float v = 0.f;
        for (int ar = 0; ar < RP; ++ar)
          for (int jf = 0; jf < BNj; ++jf)
            v = fmaf(Cs[(j * RP + ar) * BN + jf * K + r], Ys[ci * OUT + (ar * BNj + jf) * NL + jl], v);
        a.W[((int64_t)s_u[ci] * a.ncb + cb) * WE + e] = v;
      }
      __syncthreads();
    }
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
  const int npair = (g1 - g0) * ncb;
  for (int e = threadIdx.x; e < WE; e += blockDim.x) {
    float acc = 0.f;
    int q = 0;
    for (; q + 8 <= npair; q += 8) {  // (member, column block) pairs in fixed order
      float x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int gi = g0 + (q + i) / ncb, cbi = (q + i) - ((q + i) / ncb) * ncb;
        x[i] = W[((int64_t)orderL[gi] * ncb + cbi) * WE + e];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) acc += x[i];
    }
    for (; q < npair; ++q) {
      const int gi = g0 + q / ncb, cbi = q - (q / ncb) * ncb;
      acc += W[((int64_t)orderL[gi] * ncb + cbi) * WE + e];
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
    const int n0 = cstart_pm1[p] * ncb, n1 = cstart_pm1[p + 1] * ncb;  // (child, cb) pairs are contiguous
    float acc = 0.f;
    int q = n0;
    for (; q + 8 <= n1; q += 8) {
      float x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = dPc[(int64_t)(q + i) * per + e];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc += x[i];
    }
    for (; q < n1; ++q) acc += dPc[(int64_t)q * per + e];
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
  if (R2 != K) return false;
  int BN = 0;
  if (K == 16 && NC % 64 == 0) BN = 64;
  if (K == 32 && NC % 128 == 0) BN = 128;
  if (K == 64 && NC % 256 == 0) BN = 256;
  if (K == 64 && !BN && NC % 128 == 0) BN = 128;
  if (K == 128 && NC % 128 == 0) BN = 128;
  if (!BN) return false;
  if (RP > FB_BM || FB_BM % RP) return false;
  const int64_t OUT = RP * (BN / K) * NL;
  if (OUT % 4 || NL > 16) return false;
  if (c.emb_dim % 4 || c.npad % 4 || c.npad > 512) return false;
  for (int k = 0; k < c.d; ++k)
    if (c.core_off[k] % 4 || c.slice[k] % 4) return false;
  s->ok = 1;
  s->F = F;
  s->K = (int)K;
  s->BN = BN;
  s->NC = (int)NC;
  s->ncb = (int)(NC / BN);
  s->RP = (int)RP;
  s->NL = (int)NL;
  s->nF = (int)c.n[F];
  s->BNj = (int)(BN / K);
  s->OUT = (int)OUT;
  const size_t SB = BN + 4;
  const size_t ints = sizeof(int64_t) * 2 * FB_BM + sizeof(int) * (6 * FB_BM + 8) + 16;
  const size_t base_f = sizeof(float) * (K * SB + 2 * FB_BM * K + FB_BM * BN) + ints;
  const size_t base_b = sizeof(float) * (K * SB + FB_BM * K + 2 * FB_BM * BN) + ints;
  const size_t per_f = sizeof(float) * NL * (K + 1) + 2 * sizeof(int);
  const size_t per_b = sizeof(float) * (NL * (K + 1) + OUT) + 2 * sizeof(int);
  if (base_f + 4 * per_f > (size_t)FB_SMEM_MAX || base_b + 4 * per_b > (size_t)FB_SMEM_MAX) return false;
  s->CHF = (int)std::min<size_t>(32, (FB_SMEM_MAX - base_f) / per_f);
  s->CHB = (int)std::min<size_t>(32, (FB_SMEM_MAX - base_b) / per_b);
  s->smem_fwd = base_f + s->CHF * per_f;
  s->smem_bwd = base_b + s->CHB * per_b;
  return true;
}

}  // namespace tt
