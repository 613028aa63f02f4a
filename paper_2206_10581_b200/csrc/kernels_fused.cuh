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
// Forward: the C tile is saved (P_F); the last level (R_d = 1) runs as the
// streaming kernel k_last_level over it -- for every distinct ID,
// out[(a, j_F, j_l)] = sum_r P_F[a][(j_F, r)] G_{d-1}[r, i_d, j_l] -- written to
// the ID's batch positions (IDs with more than HEAVY_POS positions go through
// Yu and the balanced k_scatter_heavy).
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
#include <cuda.h>  // CUtensorMap (types only: the encoder comes from cudaGetDriverEntryPoint)

#include "common.cuh"
#include "kernels_rows.cuh"

namespace tt {

constexpr int FB_THREADS = 256;
#ifndef TT_DG_UNROLL
#define TT_DG_UNROLL 8
#endif
constexpr int DG_UNROLL = TT_DG_UNROLL;  // k_fused_bwd's dG_F row loop unroll (A/B builds)
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
  int BNf, ncbf, BNjf;     // forward column block (no side traffic: sized for 2 CTAs/SM)
  size_t smem_fwd, smem_bwd;
};

struct FusedBufs {
  float* Psave = nullptr;  // [capk[F]][RP][NC]
  float* W = nullptr;      // [capk[d-1]][K*NL]
  float* dPc = nullptr;    // [capk[F]][ncb][RP*K]
  float* dY = nullptr;     // [capk[d-1]][npad]   upstream summed per distinct ID
  float* Yu = nullptr;     // [capk[d-1]][npad]   rows of heavy IDs
  float* part = nullptr;   // [chunks][2][npad]   k_dy_chunks partials
  float* gpart = nullptr;  // [groups][2][npad]   k_dy_groups partials
  float* dPcw = nullptr;   // wide-level dA partials
  float* gsplit = nullptr; // dG partials of split digit groups (FusedArgs::gsplit)
  int64_t cap_gsplit = 0;
  int64_t cap_nodes = 0, cap_ids = 0, cap_chunks = 0, cap_w = 0;
};

inline void free_fused(FusedBufs& b) {
  cudaFree(b.Psave);
  cudaFree(b.W);
  cudaFree(b.dPc);
  cudaFree(b.dY);
  cudaFree(b.Yu);
  cudaFree(b.part);
  cudaFree(b.gpart);
  cudaFree(b.dPcw);
  cudaFree(b.gsplit);
  b = FusedBufs{};
}

struct FusedArgs {
  DevCfg c;
  int F, ncb, RP, NL, nF, BNj, OUT, NC, CH;
  int mode;                 // 0: fused last level; 1: wide level (dC = dPin, no IDs, no W)
  const float* dPin;        // mode 1: materialised dP_F [nodes][RP][NC]
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
  int split;       // max chunks per digit group (work_item); > 1: dG_F partials in gsplit
  int split_rows;  // min rows per chunk
  float* gsplit;  // [groups][split][slice] dG_F partials of the chunks (k_fused_reduce_gsplit)
  const DevStatus* st;
  long long* dbg;  // optional per-CTA phase timestamps (TT_TC_TRACE builds only)
};

// A fused GEMM CTA's work item: digit group g, column block cb, and chunk
// `chunk` of the group's nodes (a.split chunks of equal node count: groups are
// split when m_F x ncb alone would leave SMs idle -- products has 140 groups
// and one column block, billion 178).  Returns false for an empty item.
// Chunks of a group of n nodes (RP rows each): at most `split`, and at least
// `min_rows` rows per chunk (small groups stay whole: splitting them only
// re-stages the slice block and leaves tiles part-empty).
__host__ __device__ __forceinline__ int group_chunks(int n, int RP, int split, int min_rows) {
  const int64_t by_rows = ((int64_t)n * RP) / (min_rows > 0 ? min_rows : 1);
  return (int)(by_rows < 1 ? 1 : (by_rows < split ? by_rows : split));
}

__device__ __forceinline__ bool work_item_at(const FusedArgs& a, int it, int& g, int& cb, int& chunk, int& g0,
                                             int& g1) {
  if (a.split <= 1) {
    g = it / a.ncb;
    cb = it - g * a.ncb;
    chunk = 0;
    g0 = a.goffF[g];
    g1 = a.goffF[g + 1];
    return g0 < g1;
  }
  const int split = a.split;
  const int gc = it / a.ncb;
  cb = it - gc * a.ncb;
  g = gc / split;
  chunk = gc - g * split;
  const int n0 = a.goffF[g], n = a.goffF[g + 1] - n0;
  const int nch = group_chunks(n, a.RP, split, a.split_rows);
  if (chunk >= nch) return false;
  g0 = n0 + (int)(((int64_t)n * chunk) / nch);
  g1 = n0 + (int)(((int64_t)n * (chunk + 1)) / nch);
  return g0 < g1;
}
__device__ __forceinline__ bool work_item(const FusedArgs& a, int& g, int& cb, int& chunk, int& g0, int& g1) {
  return work_item_at(a, blockIdx.x, g, cb, chunk, g0, g1);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Stage the (K x BN) column block cb of slice g of core F: Bs[k][n], row stride SB.
template <int K, int BN, int SB, int NT = FB_THREADS>
__device__ __forceinline__ void load_slice_block(const FusedArgs& a, int g, int cb, float* Bs) {
  const float* src = a.params + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F] + cb * BN;
  for (int i = threadIdx.x; i < K * BN / 4; i += NT) {
    const int k = i / (BN / 4), q = i - k * (BN / 4);
    cp_async16(Bs + k * SB + q * 4, src + (int64_t)k * a.NC + q * 4);
  }
}

constexpr int FB_NB = 256;  // nodes whose metadata is staged per batch

// Metadata for nodes [nb0, nb0 + nbn) of the group (one thread per node):
// node id, first distinct ID, A-block offset, and the exclusive prefix of the
// nodes' distinct-ID counts (s_pref[nbn] = total).  Ends with a barrier.
template <int NT = FB_THREADS>
__device__ __forceinline__ void prep_nodes(const FusedArgs& a, int nb0, int nbn, int* s_node, int* s_cs0,
                                           int* s_pref, int64_t* s_aoff, int* s_wsum) {
  const int t = threadIdx.x;
  int cnt = 0;
  if (t < nbn) {
    const int node = a.orderF[nb0 + t];
    const int c0 = a.cstartF[node];
    cnt = a.cstartF[node + 1] - c0;
    const int p = a.parentF[node];
    s_node[t] = node;
    s_cs0[t] = c0;
    s_aoff[t] = a.F == 1 ? a.c.core_off[0] + (int64_t)a.digit0[p] * a.c.slice[0] : (int64_t)p * a.RP * a.c.R[a.F];
  }
  int x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if ((int)lane_id() >= o) x += y;
  }
  if (lane_id() == 31) s_wsum[t >> 5] = x;
  __syncthreads();
  if (t < 32) {
    int w = t < NT / 32 ? s_wsum[t] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if ((int)lane_id() >= o) w += y;
    }
    if (t < NT / 32) s_wsum[t] = w;  // inclusive warp totals
  }
  __syncthreads();
  const int excl = x - cnt + ((t >> 5) ? s_wsum[(t >> 5) - 1] : 0);
  if (t < nbn) s_pref[t] = excl;
  if (t == nbn - 1) s_pref[nbn] = excl + cnt;
  __syncthreads();
}

constexpr int FB_IDS = 512;  // per-batch distinct IDs whose metadata is staged

// A tile (BM x K, row-major) of batch-local nodes [tb, tb+nn) by cp.async;
// rows past the tile's nodes are zero-filled.
template <int K, int RP, int NT = FB_THREADS>
__device__ __forceinline__ void load_A_tile(const FusedArgs& a, int tb, int nn, const int64_t* s_aoff, float* As) {
  for (int i = threadIdx.x; i < FB_BM * K / 4; i += NT) {
    const int m = i / (K / 4), q = i - m * (K / 4);
    const int j = m / RP;
    float* dst = As + m * K + q * 4;
    if (j < nn) cp_async16(dst, a.Abase + s_aoff[tb + j] + (m - j * RP) * K + q * 4);
    else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

template <int BN>
__device__ __forceinline__ void load_row_frag(const float* row, int lane, float* v) {
  constexpr int TN = BN / 32;
  if constexpr (TN >= 4) {
#pragma unroll
    for (int q = 0; q < TN / 4; ++q) {
      const float4 b = *reinterpret_cast<const float4*>(row + q * 128 + lane * 4);
      v[q * 4 + 0] = b.x; v[q * 4 + 1] = b.y; v[q * 4 + 2] = b.z; v[q * 4 + 3] = b.w;
    }
  } else if constexpr (TN == 2) {
    const float2 b = *reinterpret_cast<const float2*>(row + lane * 2);
    v[0] = b.x; v[1] = b.y;
  } else {
    v[0] = row[lane];
  }
}

template <int BN>
__device__ __forceinline__ void store_row_frag(float* row, int lane, const float* v) {
  constexpr int TN = BN / 32;
  if constexpr (TN >= 4) {
#pragma unroll
    for (int q = 0; q < TN / 4; ++q)
      *reinterpret_cast<float4*>(row + q * 128 + lane * 4) = make_float4(v[q * 4], v[q * 4 + 1], v[q * 4 + 2], v[q * 4 + 3]);
  } else if constexpr (TN == 2) {
    *reinterpret_cast<float2*>(row + lane * 2) = make_float2(v[0], v[1]);
  } else {
    row[lane] = v[0];
  }
}

// NL consecutive floats (the last core's column factor n_d) into registers:
// 16-byte loads when NL is a multiple of 4, scalar loads otherwise (the
// paper's Table-4 products shape has n = (4,5,5))
template <int NL>
__device__ __forceinline__ void ldg_vec(const float* p, float* v) {
  if constexpr (NL % 4 == 0) {
#pragma unroll
    for (int l4 = 0; l4 < NL; l4 += 4) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(p + l4));
      v[l4] = x.x; v[l4 + 1] = x.y; v[l4 + 2] = x.z; v[l4 + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int jl = 0; jl < NL; ++jl) v[jl] = __ldg(p + jl);
  }
}
template <int NL>
__device__ __forceinline__ void st_vec(float* p, const float* v) {
  if constexpr (NL % 4 == 0) {
#pragma unroll
    for (int l4 = 0; l4 < NL; l4 += 4) *reinterpret_cast<float4*>(p + l4) = make_float4(v[l4], v[l4 + 1], v[l4 + 2], v[l4 + 3]);
  } else {
#pragma unroll
    for (int jl = 0; jl < NL; ++jl) p[jl] = v[jl];
  }
}

// ---------------------------------------------------------------------------
// Column map of a warp's micro-tile (the backward's dC pass): rows m0..m0+7
// and, per lane, NQ column groups of W4 consecutive columns; group q of lane l
// covers columns q*128 + l*W4 .. (+W4) for BN >= 128 and l*W4.. for BN = 64,
// i.e. core-F column block jf = col / K and rank index r = col % K.
template <int BN>
struct ColMap {
  static constexpr int TN = BN / 32;
  static constexpr int W4 = TN >= 4 ? 4 : TN;
  static constexpr int NQ = TN / W4;
  __device__ static int col(int lane, int q) { return TN >= 4 ? q * 128 + lane * 4 : lane * W4; }
};

// ---------------------------------------------------------------------------
template <int K, int BN, int RP, int NL>
__global__ void __launch_bounds__(FB_THREADS, 2) k_fused_fwd(FusedArgs a) {
  TT_PDL_ENTRY();
  constexpr int BM = FB_BM, SB = BN + 4, TN = BN / 32, NPT = BM / RP;
  extern __shared__ __align__(16) float smem[];
  float* Bs = smem;                      // [K][SB]
  float* As0 = Bs + K * SB;              // [2][BM][K]
  int64_t* s_aoff = reinterpret_cast<int64_t*>(As0 + 2 * BM * K);
  int* s_node = reinterpret_cast<int*>(s_aoff + FB_NB);
  int* s_cs0 = s_node + FB_NB;
  int* s_pref = s_cs0 + FB_NB;            // [FB_NB + 1]
  int* s_wsum = s_pref + FB_NB + 4;

  if (tt_failed(a.st)) return;
  int g, cb, g0, g1, chunk;
  if (!work_item(a, g, cb, chunk, g0, g1)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = warp * 8;

  load_slice_block<K, BN, SB>(a, g, cb, Bs);
  cp_async_commit();
  for (int nb0 = g0; nb0 < g1; nb0 += FB_NB) {
    const int nbn = min(FB_NB, g1 - nb0);
    prep_nodes(a, nb0, nbn, s_node, s_cs0, s_pref, s_aoff, s_wsum);
    load_A_tile<K, RP>(a, 0, min(NPT, nbn), s_aoff, As0);
    cp_async_commit();
    int buf = 0;
    for (int tb = 0; tb < nbn; tb += NPT, buf ^= 1) {
      const int nn = min(NPT, nbn - tb);
      cp_async_wait<0>();
      __syncthreads();
      if (tb + NPT < nbn) {  // prefetch the next tile's A under this tile's GEMM
        load_A_tile<K, RP>(a, tb + NPT, min(NPT, nbn - tb - NPT), s_aoff, As0 + (buf ^ 1) * BM * K);
      }
      cp_async_commit();
      const float* As = As0 + buf * BM * K;
      float acc[8][TN];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
#pragma unroll 4
      for (int kk = 0; kk < K; kk += 4) {
        float4 av[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) av[i] = *reinterpret_cast<const float4*>(As + (m0 + i) * K + kk);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          float bv[TN];
          load_row_frag<BN>(Bs + (kk + t) * SB, lane, bv);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float x = t == 0 ? av[i].x : t == 1 ? av[i].y : t == 2 ? av[i].z : av[i].w;
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(x, bv[j], acc[i][j]);
          }
        }
      }
      // P_F rows of the tile (saved for the last level and the backward)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int m = m0 + i, j = m / RP;
        if (j < nn)
          store_row_frag<BN>(a.Psave + ((int64_t)s_node[tb + j] * RP + (m - j * RP)) * a.NC + cb * BN, lane, acc[i]);
      }
    }
    __syncthreads();  // the batch's node metadata is rewritten by the next prep_nodes
  }
}

// dC rows m0..m0+7 of the warp (GEMM layout) for the tile's nodes into Ds:
// dC[row][col] = sum over the node's IDs and jl of dY_u[(ar, jf, jl)] G_l(u)[r, jl]
template <int K, int BN, int RP, int NL, int DS = BN>
__device__ __forceinline__ void form_dC(const FusedArgs& a, int tb, int nn, int cb, const int* s_pref, const int* s_cs0,
                                        const int* s_bd, float* Ds, int m0) {
  constexpr int TN = BN / 32;
  using CM = ColMap<BN>;
  constexpr int W4 = CM::W4, NQ = CM::NQ;
  constexpr int NR = RP < 8 ? RP : 8;
  constexpr int NPW = 8 / NR;
  const int lane = threadIdx.x & 31;
  const int nF = a.nF;
  const int64_t npad = a.c.npad;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];

  // dC in registers (GEMM layout): dC[row][col] = sum over the node's IDs
  // and jl of dY_u[(ar, jf, jl)] G_l(u)[r, jl]
  float dacc[8][TN];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) dacc[i][j] = 0.f;
#pragma unroll
  for (int jw = 0; jw < NPW; ++jw) {
    const int j = (m0 + jw * NR) / RP;
    if (j >= nn) continue;
    const int ar0 = (m0 + jw * NR) % RP;
    const int fA = s_pref[tb + j], fB = s_pref[tb + j + 1], cs0 = s_cs0[tb + j];
    for (int f = fA; f < fB; ++f) {
      const int u = cs0 + (f - fA);
      const float* Gp = Gl + (int64_t)(f < FB_IDS ? s_bd[f] : __ldg(a.digitL + u)) * sliceL;
      const float* Yp = a.dY + (int64_t)u * npad;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        // global column of P_F: core-F column block jf, rank index r0
        // (BN may be smaller than K: a block then covers part of one jf)
        const int colg = cb * BN + CM::col(lane, q);
        const int r0 = colg % K, jf = colg / K;
        float gv[W4][NL];
#pragma unroll
        for (int t = 0; t < W4; ++t) ldg_vec<NL>(Gp + (r0 + t) * NL, gv[t]);
#pragma unroll
        for (int ii = 0; ii < NR; ++ii) {
          float yv[NL];
          ldg_vec<NL>(Yp + ((int64_t)(ar0 + ii) * nF + jf) * NL, yv);
#pragma unroll
          for (int t = 0; t < W4; ++t) {
            float s = dacc[jw * NR + ii][q * W4 + t];
#pragma unroll
            for (int jl = 0; jl < NL; ++jl) s = fmaf(yv[jl], gv[t][jl], s);
            dacc[jw * NR + ii][q * W4 + t] = s;
          }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) store_row_frag<BN>(Ds + (m0 + i) * DS, lane, dacc[i]);
}

// ---------------------------------------------------------------------------
// Forward with 8 x 8 register tiles (BN = 128, K = 32 / 64): 128 threads per
// CTA, each owning 8 rows x 8 columns of the 64 x 128 C tile.  Per k step a
// thread reads 8 A values and 8 slice values for 64 FFMAs -- 0.25 shared-memory
// floats per FFMA, against 0.375 for the 8 x 4 tiles of k_fused_fwd, whose
// shared-memory bandwidth (32 floats / clk / SM) capped the FMA pipe at 67%.
// Lane (rh, cl) = (lane / 16, lane % 16) of warp w owns rows w*16 + rh*8 ..+8
// and columns cl*4 ..+4 and 64 + cl*4 ..+4 (each 16-lane group reads 256
// contiguous bytes of a slice row: conflict-free).
constexpr int F8_THREADS = 128;

// TMA (cp.async.bulk.tensor.2d) of the K x 128 slice block: the tensor map
// views core F as a [m_F K] x [NC] fp32 matrix (slice g = rows g K ..+K), box
// {128 columns, K rows}; it lands dense in shared memory (row stride 128
// floats -- the 16-lane row fragments this kernel reads stay conflict-free)
// and completes on an mbarrier with the byte count.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
      ::"r"((unsigned)__cvta_generic_to_shared(smem_dst)), "l"(map), "r"(x), "r"(y),
      "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "W:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra W;\n\t}\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
      "r"(phase)
      : "memory");
}

// LL (round 2; NL = 4, RP = 4): the last level is fused into the tile
// epilogue -- for each distinct ID u of the thread's two nodes, the 16 lanes
// of a row group each hold 4 of the tile's 64 rank columns per core-F column,
// form the 32 partial outputs (4 rows x 2 column blocks x NL) over those 4
// ranks, reduce-scatter them over the 16 lanes (shuffles xor 8, 4, 2, 1), and
// write 2 contiguous floats of the output row to every batch position of u
// (heavy IDs: their Yu row, scattered by k_scatter_heavy).  k_last_level then
// does not run (it re-read all of P_F).
template <int K, int RP, bool TMA, bool LL = false>
__global__ void __launch_bounds__(F8_THREADS, (K <= 32) ? 4 : 3)
    k_fused_fwd8(FusedArgs a, const __grid_constant__ CUtensorMap tmS) {
  TT_PDL_ENTRY();
  constexpr int BN = 128, BM = FB_BM, SB = TMA ? BN : BN + 4, NPT = BM / RP, NB = F8_THREADS;
  extern __shared__ __align__(128) float smem[];
  float* Bs = smem;                      // [K][SB]
  float* As0 = Bs + K * SB;              // [2][BM][K]
  int64_t* s_aoff = reinterpret_cast<int64_t*>(As0 + 2 * BM * K);
  int* s_node = reinterpret_cast<int*>(s_aoff + NB);
  int* s_cs0 = s_node + NB;
  int* s_pref = s_cs0 + NB;               // [NB + 1]
  int* s_wsum = s_pref + NB + 4;
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_wsum + 12);  // 8-byte aligned (s_wsum is)

  if (tt_failed(a.st)) return;
  int g, cb, g0, g1, chunk;
  if (!work_item(a, g, cb, chunk, g0, g1)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = warp * 16 + (lane >> 4) * 8, c0 = (lane & 15) * 4;

  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(s_bar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      mbar_expect_tx(s_bar, K * BN * 4);
      tma_load_2d(Bs, &tmS, s_bar, cb * BN, g * K);
    }
  } else {
    load_slice_block<K, BN, SB, F8_THREADS>(a, g, cb, Bs);
  }
  cp_async_commit();
  bool s_ready = !TMA;
  for (int nb0 = g0; nb0 < g1; nb0 += NB) {
    const int nbn = min(NB, g1 - nb0);
    prep_nodes<F8_THREADS>(a, nb0, nbn, s_node, s_cs0, s_pref, s_aoff, s_wsum);
    load_A_tile<K, RP, F8_THREADS>(a, 0, min(NPT, nbn), s_aoff, As0);
    cp_async_commit();
    int buf = 0;
    for (int tb = 0; tb < nbn; tb += NPT, buf ^= 1) {
      const int nn = min(NPT, nbn - tb);
      cp_async_wait<0>();
      __syncthreads();
      if (tb + NPT < nbn)  // the next tile's A under this tile's GEMM
        load_A_tile<K, RP, F8_THREADS>(a, tb + NPT, min(NPT, nbn - tb - NPT), s_aoff, As0 + (buf ^ 1) * BM * K);
      cp_async_commit();
      if constexpr (TMA) {
        if (!s_ready) {  // (every thread passed the barrier above after thread 0 armed it)
          mbar_wait_parity(s_bar, 0);
          s_ready = true;
        }
      }
      if (r0 >= nn * RP) continue;  // rows past the group's end: no work (warp-uniform per half)
      const float* As = As0 + buf * BM * K;
      float acc[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
#pragma unroll 2
      for (int kk = 0; kk < K; kk += 4) {
        float4 av[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) av[i] = *reinterpret_cast<const float4*>(As + (r0 + i) * K + kk);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float4 b0 = *reinterpret_cast<const float4*>(Bs + (kk + t) * SB + c0);
          const float4 b1 = *reinterpret_cast<const float4*>(Bs + (kk + t) * SB + 64 + c0);
          const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float x = t == 0 ? av[i].x : t == 1 ? av[i].y : t == 2 ? av[i].z : av[i].w;
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(x, bv[j], acc[i][j]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int m = r0 + i, j = m / RP;
        if (j < nn) {
          float* dst = a.Psave + ((int64_t)s_node[tb + j] * RP + (m - j * RP)) * a.NC + cb * BN;
          *reinterpret_cast<float4*>(dst + c0) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
          *reinterpret_cast<float4*>(dst + 64 + c0) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
        }
      }
      if constexpr (LL && !(K == 64 && RP == 4)) {
        __trap();  // the fused last level exists for K = 64, RP = 4 only (the host never selects it otherwise)
      } else if constexpr (LL) {
        constexpr int NLL = 4;
        const unsigned gmask = 0xFFFFu << (lane & 16);
        const int li = lane & 15;
        const float* Gl = a.params + a.c.core_off[a.c.d - 1];
        const int64_t sliceL = a.c.slice[a.c.d - 1];
        const int64_t emb = a.c.emb_dim, npad = a.c.npad;
        // this lane's 2 outputs after the reduce-scatter: row a = li / 4, column
        // block h = (li / 2) & 1, NL entries 2 (li & 1) .. + 1
        const int oa = li >> 2, oh = (li >> 1) & 1;
        const int64_t col = ((int64_t)oa * a.nF + 2 * cb + oh) * NLL + 2 * (li & 1);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int j = r0 / RP + k;
          if (j >= nn) break;
          const int node = s_node[tb + j];
          const int u0 = __ldg(a.cstartF + node), u1 = __ldg(a.cstartF + node + 1);
          for (int u = u0; u < u1; ++u) {
            const float4* gp = reinterpret_cast<const float4*>(Gl + (int64_t)__ldg(a.digitL + u) * sliceL + c0 * NLL);
            float4 g[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) g[t] = __ldg(gp + t);
            float v[32];  // v[ar * 8 + h * 4 + jl]
#pragma unroll
            for (int ar = 0; ar < 4; ++ar)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                float o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                  const float x = acc[4 * k + ar][4 * h + t];
                  o0 = fmaf(x, g[t].x, o0); o1 = fmaf(x, g[t].y, o1); o2 = fmaf(x, g[t].z, o2); o3 = fmaf(x, g[t].w, o3);
                }
                v[ar * 8 + h * 4] = o0; v[ar * 8 + h * 4 + 1] = o1; v[ar * 8 + h * 4 + 2] = o2; v[ar * 8 + h * 4 + 3] = o3;
              }
            // reduce-scatter over the 16 lanes: after the xor-8 step a lane keeps
            // the half of v its bit 3 selects, and so on down to 2 values
#pragma unroll
            for (int step = 0; step < 4; ++step) {
              const int half = 16 >> step;
              const bool hi = (li >> (3 - step)) & 1;
#pragma unroll
              for (int i = 0; i < half; ++i) {
                const float give = hi ? v[i] : v[half + i];
                const float keep = hi ? v[half + i] : v[i];
                v[i] = keep + __shfl_xor_sync(gmask, give, 8 >> step);
              }
            }
            const int s0 = __ldg(a.seg + u), s1 = __ldg(a.seg + u + 1);
            if (s1 - s0 > HEAVY_POS) {
              *reinterpret_cast<float2*>(a.Yu + (int64_t)u * npad + col) = make_float2(v[0], v[1]);
            } else if (col < emb) {
              for (int sl = s0; sl < s1; ++sl) {
                float* orow = a.out + (int64_t)__ldg(a.spos + sl) * emb + col;
                if (col + 1 < emb) *reinterpret_cast<float2*>(orow) = make_float2(v[0], v[1]);
                else orow[0] = v[0];
              }
            }
          }
        }
      }
    }
    __syncthreads();  // the batch's node metadata is rewritten by the next prep_nodes
  }
}

// ---------------------------------------------------------------------------
// k_fused_fwd8 without CTA barriers in the tile loop (round 2, TT_FWD8W):
// every warp walks its own 16-row warp tiles (16 / RP nodes) of the group --
// warp tiles w, w + 4, ... -- with a private double-buffered A tile (cp.async,
// cp.async.wait_group + __syncwarp), so the warps drift apart instead of
// meeting at a barrier after every 64-row tile, and one warp's A loads and
// P_F stores overlap the other warps' FFMAs.  The slice block arrives once by
// TMA.  Lane (rh, cl) owns rows rh, rh + 2, ..., rh + 14 of the warp tile and
// columns cl*4 ..+4, 64 + cl*4 ..+4; the A tile's row stride is K + 4 floats,
// so the two half-warps' rows (adjacent) sit in different banks.
constexpr int F8W_ROWS = 16;
#ifndef TT_F8W_UNROLL
#define TT_F8W_UNROLL 4
#endif
constexpr int F8W_UNROLL = TT_F8W_UNROLL;  // k-step unroll of k_fused_fwd8w (A/B builds)
template <int K>
__host__ __device__ constexpr int f8w_astride() { return K + 4; }
inline size_t fwd8w_smem(int K) {
  return sizeof(float) * ((size_t)K * 128 + (size_t)(F8_THREADS / 32) * 2 * F8W_ROWS * (K + 4)) +
         sizeof(int) * (F8_THREADS / 32) * 2 * F8W_ROWS + 16;
}

// LL (K = 64, RP = 4, NL = 4; TT_FWD_LL=1): the last level in the warp tile's
// epilogue.  For each distinct ID u of the tile's 4 nodes, lane (rh, cl) forms
// the 16 partial outputs (a = rh + 2 aa, column block 2 cb + h, jl) over its 4
// ranks c0..c0+3, the 16 lanes of a half-warp reduce-scatter them (xor 8, 4,
// 2, 1: 15 shuffles) so lane cl keeps output (aa, h, jl) = (cl / 8, cl / 4 % 2,
// cl % 4), and write it to every batch position of u (heavy IDs: their Yu row,
// scattered later by k_scatter_heavy).  The nodes' ID ranges are fetched before
// the tile's GEMM and the IDs' digits / position ranges lane-parallel after it,
// so one warp's epilogue latency runs under the other warps' FFMAs (no CTA
// barrier couples them).  k_last_level then does not run.
template <int K, int RP, bool LL = false>
__global__ void __launch_bounds__(F8_THREADS, 3)
    k_fused_fwd8w(FusedArgs a, const __grid_constant__ CUtensorMap tmS) {
  TT_PDL_ENTRY();
  constexpr int BN = 128, AS = f8w_astride<K>(), WR = F8W_ROWS, NPW = WR / RP, NW = F8_THREADS / 32;
  static_assert(WR % RP == 0, "warp tiles hold whole nodes");
  extern __shared__ __align__(128) float smem[];
  float* Bs = smem;  // [K][128] (TMA, dense)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* Aw = Bs + K * BN + warp * 2 * WR * AS;                                             // [2][WR][AS]
  int* s_wnode = reinterpret_cast<int*>(Bs + K * BN + NW * 2 * WR * AS) + warp * 2 * WR;  // [2][NPW]
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(reinterpret_cast<int*>(Bs + K * BN + NW * 2 * WR * AS) + NW * 2 * WR);

  if (tt_failed(a.st)) return;
  int g, cb, g0, g1, chunk;
  if (!work_item(a, g, cb, chunk, g0, g1)) return;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(s_bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    mbar_expect_tx(s_bar, K * BN * 4);
    tma_load_2d(Bs, &tmS, s_bar, cb * BN, g * K);
  }
  __syncthreads();  // the barrier is initialised before any warp waits on it

  const int ntiles = (g1 - g0 + NPW - 1) / NPW;
  // A rows of warp tile wt into buffer b: node metadata by lanes < NPW, then
  // K/4 16-byte cp.async per row (32 lanes x WR*K/128 copies)
  // Node metadata for TPB = 32 / NPW consecutive warp tiles at a time (lane l:
  // tile l / NPW of the batch, node l % NPW): the dependent orderF -> parentF
  // -> digit0 loads are paid once per TPB tiles, not before every tile's A copy.
  constexpr int TPB = 32 / NPW;
  int m_node = 0;
  int64_t m_aoff = 0;
  auto fetch_meta = [&](int it0) {
    const int n = g0 + (warp + NW * (it0 + lane / NPW)) * NPW + lane % NPW;
    if (n < g1) {
      const int node = a.orderF[n];
      const int p = a.parentF[node];
      m_node = node;
      m_aoff = a.F == 1 ? a.c.core_off[0] + (int64_t)a.digit0[p] * a.c.slice[0] : (int64_t)p * RP * K;
    }
  };
  // A rows of the warp's tile ordinal `it` (warp tile warp + NW it) into buffer b
  auto load_tile = [&](int it, int b) {
    if (it % TPB == 0) fetch_meta(it);
    const int wt = warp + NW * it;
    const int nn = min(NPW, g1 - (g0 + wt * NPW));
    const int lb = (it % TPB) * NPW;  // the tile's first lane in the metadata batch
    const int node = __shfl_sync(0xffffffffu, m_node, lb + (lane % NPW));
    if (lane < nn) s_wnode[b * WR + lane] = node;
    float* dst = Aw + b * WR * AS;
#pragma unroll
    for (int t = 0; t < WR * K / 128; ++t) {
      const int i = lane + 32 * t, m = i / (K / 4), q = i - m * (K / 4);
      const int j = m / RP;
      const int64_t off = __shfl_sync(0xffffffffu, m_aoff, lb + j);
      if (j < nn) cp_async16(dst + m * AS + q * 4, a.Abase + off + (m - j * RP) * K + q * 4);
    }
  };

  const int rh = lane >> 4, c0 = (lane & 15) * 4;
  const int nit = ntiles > warp ? (ntiles - warp + NW - 1) / NW : 0;  // this warp's tiles
  if (nit > 0) load_tile(0, 0);
  cp_async_commit();
  bool s_ready = false;
  for (int it = 0, b = 0; it < nit; ++it, b ^= 1) {
    const int wt = warp + NW * it;
    if (it + 1 < nit) load_tile(it + 1, b ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    if (!s_ready) {
      mbar_wait_parity(s_bar, 0);
      s_ready = true;
    }
    const int nn = min(NPW, g1 - (g0 + wt * NPW));
    const float* As = Aw + b * WR * AS;
    int ll_c0 = 0, ll_c1 = 0;  // LL: lane j < nn holds node j's distinct-ID range
    if constexpr (LL) {
      if (lane < nn) {
        const int node = s_wnode[b * WR + lane];
        ll_c0 = __ldg(a.cstartF + node);
        ll_c1 = __ldg(a.cstartF + node + 1);
      }
    }
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
#pragma unroll F8W_UNROLL
    for (int kk = 0; kk < K; kk += 4) {
      float4 av[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) av[i] = *reinterpret_cast<const float4*>(As + (rh + 2 * i) * AS + kk);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float4 b0 = *reinterpret_cast<const float4*>(Bs + (kk + t) * BN + c0);
        const float4 b1 = *reinterpret_cast<const float4*>(Bs + (kk + t) * BN + 64 + c0);
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float x = t == 0 ? av[i].x : t == 1 ? av[i].y : t == 2 ? av[i].z : av[i].w;
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(x, bv[j], acc[i][j]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = rh + 2 * i, j = m / RP;
      if (j < nn) {
        float* dst = a.Psave + ((int64_t)s_wnode[b * WR + j] * RP + (m - j * RP)) * a.NC + cb * BN;
        *reinterpret_cast<float4*>(dst + c0) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        *reinterpret_cast<float4*>(dst + 64 + c0) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
      }
    }
    if constexpr (LL && !(K == 64 && RP == 4)) {
      __trap();  // the fused last level exists for K = 64, RP = 4, NL = 4 only (the host never selects it otherwise)
    } else if constexpr (LL) {
      constexpr int NLL = 4;
      const int cl = lane & 15;
      const float* Gl = a.params + a.c.core_off[a.c.d - 1];
      const int64_t sliceL = a.c.slice[a.c.d - 1];
      const int64_t emb = a.c.emb_dim, npad = a.c.npad;
      const int oaa = cl >> 3, oh = (cl >> 2) & 1, ojl = cl & 3;
      const int64_t col = ((int64_t)(rh + 2 * oaa) * a.nF + 2 * cb + oh) * NLL + ojl;
      // exclusive prefix of the nodes' ID counts (lanes 0..3)
      const int cnt = ll_c1 - ll_c0;
      int x = cnt;
#pragma unroll
      for (int o = 1; o < NPW; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const int T = __shfl_sync(0xffffffffu, x, NPW - 1);
      const int off = x - cnt;
      for (int t0 = 0; t0 < T; t0 += 32) {
        // lane i: metadata of the tile's ID t0 + i (node j, u, last digit, positions)
        const int f = t0 + lane;
        int jf_ = 0;
#pragma unroll
        for (int jj = 1; jj < NPW; ++jj)
          if (f >= __shfl_sync(0xffffffffu, off, jj)) jf_ = jj;
        const int fo = __shfl_sync(0xffffffffu, off, jf_), fc0 = __shfl_sync(0xffffffffu, ll_c0, jf_);
        int mu = 0, mdg = 0, ms0 = 0, ms1 = 0;
        if (f < T) {
          mu = fc0 + (f - fo);
          mdg = __ldg(a.digitL + mu);
          ms0 = __ldg(a.seg + mu);
          ms1 = __ldg(a.seg + mu + 1);
        }
        const int nk = min(32, T - t0);
        for (int k = 0; k < nk; ++k) {
          const int j = __shfl_sync(0xffffffffu, jf_, k), u = __shfl_sync(0xffffffffu, mu, k);
          const int dg = __shfl_sync(0xffffffffu, mdg, k);
          const int s0 = __shfl_sync(0xffffffffu, ms0, k), s1 = __shfl_sync(0xffffffffu, ms1, k);
          const float4* gp = reinterpret_cast<const float4*>(Gl + (int64_t)dg * sliceL + c0 * NLL);
          float4 gv[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) gv[t] = __ldg(gp + t);
          float v[16];  // v[aa * 8 + h * 4 + jl]
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] = 0.f;
#pragma unroll
          for (int jj = 0; jj < NPW; ++jj) {
            if (jj != j) continue;  // warp-uniform: the node's two rows of this lane
#pragma unroll
            for (int aa = 0; aa < 2; ++aa)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                  const float xv = acc[2 * jj + aa][4 * hh + t];
                  v[aa * 8 + hh * 4 + 0] = fmaf(xv, gv[t].x, v[aa * 8 + hh * 4 + 0]);
                  v[aa * 8 + hh * 4 + 1] = fmaf(xv, gv[t].y, v[aa * 8 + hh * 4 + 1]);
                  v[aa * 8 + hh * 4 + 2] = fmaf(xv, gv[t].z, v[aa * 8 + hh * 4 + 2]);
                  v[aa * 8 + hh * 4 + 3] = fmaf(xv, gv[t].w, v[aa * 8 + hh * 4 + 3]);
                }
          }
#pragma unroll
          for (int step = 0; step < 4; ++step) {
            const int half = 8 >> step;
            const bool hi = (cl >> (3 - step)) & 1;
#pragma unroll
            for (int i = 0; i < half; ++i) {
              const float give = hi ? v[i] : v[half + i];
              const float keep = hi ? v[half + i] : v[i];
              v[i] = keep + __shfl_xor_sync(0xffffffffu, give, half);
            }
          }
          if (s1 - s0 > HEAVY_POS) {
            a.Yu[(int64_t)u * npad + col] = v[0];
          } else if (col < emb) {
            for (int sl = s0; sl < s1; ++sl) a.out[(int64_t)__ldg(a.spos + sl) * emb + col] = v[0];
          }
        }
      }
    }
    __syncwarp();  // buffer b (A rows, node ids) is refilled by the next iteration's load
  }
  cp_async_wait<0>();
}

// (K, RP) instantiations of k_fused_fwd8 / k_fused_fwd8w (papers, sweep64,
// billion, products, sweep32, the papers100M Table-4 shape).  Measured (1 B200):
// k_fused_fwd8 at papers 0.552 -> 0.541 ms but slower at K = 32 (products 0.023
// -> 0.025, billion 1.58 -> 1.73 ms); the warp-tile k_fused_fwd8w (the default
// where TMA is on) is faster everywhere: papers 0.534 -> 0.497, billion 0.969
// -> 0.796, products 0.023 -> 0.021 (profiles/r02/NOTES.md).
#define TT_FWD8_SHAPES(X) X(64, 4) X(32, 16) X(32, 4) X(64, 8)

inline size_t fwd8_smem(int K) {
  const size_t NB = F8_THREADS;
  return sizeof(float) * ((size_t)K * 132 + 2 * FB_BM * K) + sizeof(int64_t) * NB + sizeof(int) * (3 * NB + 12) + 16 +
         16;
}

// ---------------------------------------------------------------------------
template <int K, int BN, int RP, int NL>
__global__ void __launch_bounds__(FB_THREADS, (K * BN <= 64 * 128) ? 2 : 1) k_fused_bwd(FusedArgs a) {
  TT_PDL_ENTRY();
  constexpr int BM = FB_BM, SB = BN + 4, TN = BN / 32, TK = K / 8, NPT = BM / RP;
  constexpr int WE = K * NL;
  // dC row stride: padded by 4 floats so the dA phase's two half-warps (rows
  // mg, mg + 1) read different banks
  constexpr int DS = BN + 4;
  constexpr int KG = K < 16 ? K : 16, MG = FB_THREADS / KG, TKA = K / KG, TMA = BM / MG;
  using CM = ColMap<BN>;
  constexpr int W4 = CM::W4, NQ = CM::NQ;
  constexpr int NR = RP < 8 ? RP : 8;
  constexpr int NPW = 8 / NR;
  constexpr int WPL = WE / 32 > 0 ? WE / 32 : 1;  // W values per lane per ID
  extern __shared__ __align__(16) float smem[];
  float* Bs = smem;               // [K][SB]
  float* As = Bs + K * SB;        // [BM][K]
  float* Ds = As + BM * K;        // [BM][DS]  dC
  int64_t* s_aoff = reinterpret_cast<int64_t*>(Ds + BM * DS);
  int* s_node = reinterpret_cast<int*>(s_aoff + FB_NB);
  int* s_cs0 = s_node + FB_NB;
  int* s_pref = s_cs0 + FB_NB;
  int* s_wsum = s_pref + FB_NB + 4;
  int* s_bd = s_wsum + 8;  // [FB_IDS] last-core digits of the batch's first IDs (mode 0)

  long long* trace = (a.dbg && blockIdx.x < 4096) ? a.dbg + (int64_t)blockIdx.x * 64 : nullptr;
  int ntr = 0;
  auto TR = [&]() {
    if (trace && threadIdx.x == 0 && ntr < 63) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[1 + ntr++] = t;
      trace[0] = ntr;
    }
  };
  TR();
  if (tt_failed(a.st)) return;
  int g, cb, g0, g1, chunk;
  if (!work_item(a, g, cb, chunk, g0, g1)) return;
  load_slice_block<K, BN, SB>(a, g, cb, Bs);
  cp_async_commit();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = warp * 8;
  const int nF = a.nF;
  const int64_t npad = a.c.npad;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];

  float gacc[TK][TN];
#pragma unroll
  for (int i = 0; i < TK; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) gacc[i][j] = 0.f;

  for (int nb0 = g0; nb0 < g1; nb0 += FB_NB) {
    const int nbn = min(FB_NB, g1 - nb0);
    prep_nodes(a, nb0, nbn, s_node, s_cs0, s_pref, s_aoff, s_wsum);
    if (a.mode == 0) {  // digits of the batch's IDs: one L2 round trip per batch, not per ID
      const int tot = min(s_pref[nbn], FB_IDS);
      for (int f = threadIdx.x; f < tot; f += FB_THREADS) {
        int lo = 0, hi = nbn - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_pref[mid] <= f) lo = mid; else hi = mid - 1;
        }
        s_bd[f] = __ldg(a.digitL + s_cs0[lo] + (f - s_pref[lo]));
      }
      __syncthreads();
    }
    for (int tb = 0; tb < nbn; tb += NPT) {
      const int nn = min(NPT, nbn - tb);
      TR();
      load_A_tile<K, RP>(a, tb, nn, s_aoff, As);
      if (a.mode == 1) {  // the materialised dC tile
        for (int i = threadIdx.x; i < BM * BN / 4; i += FB_THREADS) {
          const int m = i / (BN / 4), q = i - m * (BN / 4);
          const int j = m / RP;
          float* dst = Ds + m * DS + q * 4;
          if (j < nn) cp_async16(dst, a.dPin + ((int64_t)s_node[tb + j] * RP + (m - j * RP)) * a.NC + cb * BN + q * 4);
          else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      cp_async_commit();
      if (a.mode == 0) {
        form_dC<K, BN, RP, NL, DS>(a, tb, nn, cb, s_pref, s_cs0, s_bd, Ds, (threadIdx.x >> 5) * 8);
        cp_async_wait<0>();  // slice block + A tile landed
      } else {
        cp_async_wait<0>();  // slice block + A tile + dC tile
      }
      __syncthreads();
      TR();
      // dG_F block += A^T dC  (operands double-buffered in registers)
      {
        auto ldA = [&](int m, float* av) {
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
        };
        auto fma_tile = [&](const float* av, const float* bv) {
#pragma unroll
          for (int i = 0; i < TK; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) gacc[i][j] = fmaf(av[i], bv[j], gacc[i][j]);
        };
        float a0[TK], b0[TN], a1[TK], b1[TN];
        ldA(0, a0);
        load_row_frag<BN>(Ds, lane, b0);
#pragma unroll DG_UNROLL
        for (int m = 0; m < BM; m += 2) {
          ldA(m + 1, a1);
          load_row_frag<BN>(Ds + (m + 1) * DS, lane, b1);
          fma_tile(a0, b0);
          if (m + 2 < BM) {
            ldA(m + 2, a0);
            load_row_frag<BN>(Ds + (m + 2) * DS, lane, b0);
          }
          fma_tile(a1, b1);
        }
      }
      TR();
      // dA = dC . S_block^T  -> per-(node, column block) partials
      {
        const int kg = threadIdx.x % KG, mg = threadIdx.x / KG;
        float xacc[TMA][TKA];
#pragma unroll
        for (int i = 0; i < TMA; ++i)
#pragma unroll
          for (int j = 0; j < TKA; ++j) xacc[i][j] = 0.f;
        auto ldX = [&](int n, float4* cv, float4* bv) {
#pragma unroll
          for (int i = 0; i < TMA; ++i) cv[i] = *reinterpret_cast<const float4*>(Ds + (mg + MG * i) * DS + n);
#pragma unroll
          for (int j = 0; j < TKA; ++j) bv[j] = *reinterpret_cast<const float4*>(Bs + (kg + KG * j) * SB + n);
        };
        auto fmaX = [&](const float4* cv, const float4* bv) {
#pragma unroll
          for (int i = 0; i < TMA; ++i)
#pragma unroll
            for (int j = 0; j < TKA; ++j) {
              xacc[i][j] = fmaf(cv[i].x, bv[j].x, xacc[i][j]);
              xacc[i][j] = fmaf(cv[i].y, bv[j].y, xacc[i][j]);
              xacc[i][j] = fmaf(cv[i].z, bv[j].z, xacc[i][j]);
              xacc[i][j] = fmaf(cv[i].w, bv[j].w, xacc[i][j]);
            }
        };
        float4 c0[TMA], e0[TKA], c1[TMA], e1[TKA];
        ldX(0, c0, e0);
#pragma unroll
        for (int n = 0; n < BN; n += 8) {
          ldX(n + 4, c1, e1);
          fmaX(c0, e0);
          if (n + 8 < BN) ldX(n + 8, c0, e0);
          fmaX(c1, e1);
        }
#pragma unroll
        for (int i = 0; i < TMA; ++i) {
          const int m = mg + MG * i;
          const int j = m / RP;
          if (j >= nn) continue;
          float* dst = a.dPc + ((int64_t)s_node[tb + j] * a.ncb + cb) * RP * K + (m - j * RP) * K;
#pragma unroll
          for (int jj = 0; jj < TKA; ++jj) dst[kg + KG * jj] = xacc[i][jj];
        }
      }
      __syncthreads();
    }
  }
  // the group's dG_F column block (one writer per slice block: no atomics)
  float* gdst = (a.split > 1 ? a.gsplit + ((int64_t)g * a.split + chunk) * a.c.slice[a.F]
                              : a.grads + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F]) + cb * BN;
#pragma unroll
  for (int i = 0; i < TK; ++i) store_row_frag<BN>(gdst + (int64_t)(warp * TK + i) * a.NC, lane, gacc[i]);
}

// ---------------------------------------------------------------------------
// Backward for rank 32 (K = 32, BN = 128): 128-thread CTAs, 3 per SM, the two
// GEMMs on separate warp pairs.  With 256 threads k_fused_bwd's tiles at
// K = 32 are 4 x 4 (dG_F) and 4 x 2 (dA): 0.5 and 0.75 shared-memory floats per
// FFMA, which bounds it well below the FMA pipe (billion: 26-37% of peak).
// Here, after all 4 warps have formed the tile's dC (16 rows each):
//   warps 0-1: dG_F += A^T dC with 8 x 8 tiles (thread t: k rows (t/16)*8 ..+8,
//     columns (t%16)*4 ..+4 and 64 + (t%16)*4 ..+4): 0.25 floats / FFMA;
//   warps 2-3: dA = dC S^T with 8 x 4 tiles (rows (t/8)*8 ..+8, k = t%8 + 8j):
//     0.375 floats / FFMA;
// one 64-entry accumulator array is the persistent dG_F tile in warps 0-1 and
// the per-tile dA tile in warps 2-3.  mode 1 (a wide level) loads dC.
constexpr int K32_THREADS = 128, K32_NB = 128;

template <int RP, int NL>
__global__ void __launch_bounds__(K32_THREADS, 3) k_fused_bwd_k32(FusedArgs a) {
  TT_PDL_ENTRY();
  constexpr int K = 32, BN = 128, BM = FB_BM, SB = BN + 4, NPT = BM / RP, NB = K32_NB;
  extern __shared__ __align__(16) float smem[];
  float* Bs = smem;               // [K][SB]
  float* As = Bs + K * SB;        // [BM][K]
  float* Ds = As + BM * K;        // [BM][BN]  dC
  int64_t* s_aoff = reinterpret_cast<int64_t*>(Ds + BM * BN);
  int* s_node = reinterpret_cast<int*>(s_aoff + NB);
  int* s_cs0 = s_node + NB;
  int* s_pref = s_cs0 + NB;
  int* s_wsum = s_pref + NB + 4;
  int* s_bd = s_wsum + 8;  // [FB_IDS]

  if (tt_failed(a.st)) return;
  int g, cb, g0, g1, chunk;
  if (!work_item(a, g, cb, chunk, g0, g1)) return;
  load_slice_block<K, BN, SB, K32_THREADS>(a, g, cb, Bs);
  cp_async_commit();

  const int tid = threadIdx.x, warp = tid >> 5;
  const bool gw = warp < 2;
  const int kb = (tid >> 4) * 8, c0 = (tid & 15) * 4;        // dG role (tid < 64)
  const int t2 = tid - 64, mg8 = (t2 >> 3) * 8, kg = t2 & 7;  // dA role (tid >= 64)

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  for (int nb0 = g0; nb0 < g1; nb0 += NB) {
    const int nbn = min(NB, g1 - nb0);
    prep_nodes<K32_THREADS>(a, nb0, nbn, s_node, s_cs0, s_pref, s_aoff, s_wsum);
    if (a.mode == 0) {  // digits of the batch's IDs: one L2 round trip per batch, not per ID
      const int tot = min(s_pref[nbn], FB_IDS);
      for (int f = tid; f < tot; f += K32_THREADS) {
        int lo = 0, hi = nbn - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_pref[mid] <= f) lo = mid; else hi = mid - 1;
        }
        s_bd[f] = __ldg(a.digitL + s_cs0[lo] + (f - s_pref[lo]));
      }
      __syncthreads();
    }
    for (int tb = 0; tb < nbn; tb += NPT) {
      const int nn = min(NPT, nbn - tb);
      const int mlim = nn * RP;
      load_A_tile<K, RP, K32_THREADS>(a, tb, nn, s_aoff, As);
      if (a.mode == 1) {  // the materialised dC tile
        for (int i = tid; i < BM * BN / 4; i += K32_THREADS) {
          const int m = i / (BN / 4), q = i - m * (BN / 4);
          const int j = m / RP;
          float* dst = Ds + m * BN + q * 4;
          if (j < nn) cp_async16(dst, a.dPin + ((int64_t)s_node[tb + j] * RP + (m - j * RP)) * a.NC + cb * BN + q * 4);
          else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      cp_async_commit();
      if (a.mode == 0) {
        form_dC<K, BN, RP, NL>(a, tb, nn, cb, s_pref, s_cs0, s_bd, Ds, warp * 16);
        form_dC<K, BN, RP, NL>(a, tb, nn, cb, s_pref, s_cs0, s_bd, Ds, warp * 16 + 8);
      }
      cp_async_wait<0>();  // slice block + A tile (+ dC tile)
      __syncthreads();
      if (gw) {
#pragma unroll 2
        for (int m = 0; m < BM; ++m) {
          if (m >= mlim) break;
          const float4 a0 = *reinterpret_cast<const float4*>(As + m * K + kb);
          const float4 a1 = *reinterpret_cast<const float4*>(As + m * K + kb + 4);
          const float4 d0 = *reinterpret_cast<const float4*>(Ds + m * BN + c0);
          const float4 d1 = *reinterpret_cast<const float4*>(Ds + m * BN + 64 + c0);
          const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
          const float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], dv[j], acc[i][j]);
        }
      } else if (mg8 < mlim) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 4
        for (int n = 0; n < BN; n += 4) {
          float4 cv[8], bv[4];
#pragma unroll
          for (int i = 0; i < 8; ++i) cv[i] = *reinterpret_cast<const float4*>(Ds + (mg8 + i) * BN + n);
#pragma unroll
          for (int j = 0; j < 4; ++j) bv[j] = *reinterpret_cast<const float4*>(Bs + (kg + 8 * j) * SB + n);
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              acc[i][j] = fmaf(cv[i].x, bv[j].x, acc[i][j]);
              acc[i][j] = fmaf(cv[i].y, bv[j].y, acc[i][j]);
              acc[i][j] = fmaf(cv[i].z, bv[j].z, acc[i][j]);
              acc[i][j] = fmaf(cv[i].w, bv[j].w, acc[i][j]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int m = mg8 + i;
          const int j = m / RP;
          if (j >= nn) continue;
          float* dst = a.dPc + ((int64_t)s_node[tb + j] * a.ncb + cb) * RP * K + (m - j * RP) * K;
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) dst[kg + 8 * jj] = acc[i][jj];
        }
      }
      __syncthreads();
    }
  }
  if (gw) {  // the group's (chunk's) dG_F column block
    float* gdst = (a.split > 1 ? a.gsplit + ((int64_t)g * a.split + chunk) * a.c.slice[a.F]
                                : a.grads + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F]) + cb * BN;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float* row = gdst + (int64_t)(kb + i) * a.NC;
      *reinterpret_cast<float4*>(row + c0) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      *reinterpret_cast<float4*>(row + 64 + c0) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
  }
}

inline size_t bwd_k32_smem() {
  return sizeof(float) * (32 * 132 + FB_BM * 32 + FB_BM * 128) + sizeof(int64_t) * K32_NB +
         sizeof(int) * (3 * K32_NB + 12 + 8 + FB_IDS) + 16;
}

// (RP, NL) instantiations of k_fused_bwd_k32 (billion's level F; the RP = 4
// variant measured slower than k_fused_bwd, profiles/r02/NOTES.md)
#define TT_BWDK32_SHAPES(X) X(16, 4)

// ---------------------------------------------------------------------------
// Warp-specialised rank-32 backward (billion's level F).  The profile of
// k_fused_bwd_k32 puts ~21% of its stall samples on the dC formation's L2
// loads (last-core slices, upstream rows) and ~12% on the barriers around it:
// every warp waited for the slowest warp's dC before the GEMMs could start.
// Here dC and the A tile are produced one tile ahead into double buffers:
//   warps 0-3 (producers): A tile by cp.async + dC (16 rows each) -> buffer t%2,
//     then bar.arrive FULL[t%2]; before reusing a buffer they bar.sync on
//     EMPTY[t%2] (the consumers' release of tile t-2);
//   warps 4-5: dG_F += A^T dC (8 x 8 tiles, persistent), warps 6-7: dA (8 x 4),
//     each bar.sync FULL[t%2] -> GEMM -> bar.arrive EMPTY[t%2].
// Named barriers 1-2 (FULL) and 3-4 (EMPTY), 256 threads each.
constexpr int WS_THREADS = 256, WS_NB = 256;

template <int ID, int N>
__device__ __forceinline__ void named_sync() { asm volatile("bar.sync %0, %1;\n" ::"n"(ID), "n"(N) : "memory"); }
template <int ID, int N>
__device__ __forceinline__ void named_arrive() { asm volatile("bar.arrive %0, %1;\n" ::"n"(ID), "n"(N) : "memory"); }
// barrier (base + buf) with a run-time buffer index 0 / 1
template <int BASE, int N>
__device__ __forceinline__ void named_sync2(int buf) { if (buf) named_sync<BASE + 1, N>(); else named_sync<BASE, N>(); }
template <int BASE, int N>
__device__ __forceinline__ void named_arrive2(int buf) { if (buf) named_arrive<BASE + 1, N>(); else named_arrive<BASE, N>(); }

// dC rows m0..m0+7 (one node: RP % 8 == 0) x the lane's 4 columns: per ID
// all twelve loads (4 slice rows + 8 upstream rows) are issued before the FMAs
template <int K, int RP, int NL>
__device__ __forceinline__ void form_dC8(const FusedArgs& a, int tb, int nn, int cb, const int* s_pref,
                                         const int* s_cs0, const int* s_bd, float* Ds, int m0, int lane) {
  constexpr int BN = 128;
  const int j = m0 / RP;
  float dacc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int t = 0; t < 4; ++t) dacc[i][t] = 0.f;
  if (j < nn) {
    const int ar0 = m0 - j * RP;
    const int fA = s_pref[tb + j], fB = s_pref[tb + j + 1], cs0 = s_cs0[tb + j];
    const int colg = cb * BN + lane * 4, r0 = colg % K, jf = colg / K;
    const int nF = a.nF;
    const int64_t npad = a.c.npad;
    const float* Gl = a.params + a.c.core_off[a.c.d - 1];
    const int64_t sliceL = a.c.slice[a.c.d - 1];
    for (int f = fA; f < fB; ++f) {
      const int u = cs0 + (f - fA);
      const float* Gp = Gl + (int64_t)(f < FB_IDS ? s_bd[f] : __ldg(a.digitL + u)) * sliceL;
      const float* Yp = a.dY + (int64_t)u * npad + ((int64_t)ar0 * nF + jf) * NL;
#pragma unroll
      for (int l4 = 0; l4 < NL; l4 += 4) {
        float4 gv[4], y[8];
#pragma unroll
        for (int t = 0; t < 4; ++t) gv[t] = __ldg(reinterpret_cast<const float4*>(Gp + (r0 + t) * NL + l4));
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) y[ii] = __ldg(reinterpret_cast<const float4*>(Yp + (int64_t)ii * nF * NL + l4));
#pragma unroll
        for (int ii = 0; ii < 8; ++ii)
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            float x = dacc[ii][t];
            x = fmaf(y[ii].x, gv[t].x, x);
            x = fmaf(y[ii].y, gv[t].y, x);
            x = fmaf(y[ii].z, gv[t].z, x);
            x = fmaf(y[ii].w, gv[t].w, x);
            dacc[ii][t] = x;
          }
      }
    }
  }
#pragma unroll
  for (int ii = 0; ii < 8; ++ii)
    *reinterpret_cast<float4*>(Ds + (m0 + ii) * BN + lane * 4) = make_float4(dacc[ii][0], dacc[ii][1], dacc[ii][2], dacc[ii][3]);
}

struct WsSmem {
  float *Bs, *As0, *Ds0;
  int64_t* s_aoff;
  int *s_node, *s_cs0, *s_pref, *s_wsum, *s_bd;
};

// the batch prologue every role runs in step (prep_nodes' barriers + the
// digit staging barrier: the same __syncthreads sequence in both roles)
template <int T>
__device__ __forceinline__ void ws_batch_prologue(const FusedArgs& a, const WsSmem& m, int nb0, int nbn) {
  prep_nodes<T>(a, nb0, nbn, m.s_node, m.s_cs0, m.s_pref, m.s_aoff, m.s_wsum);
  const int tot = min(m.s_pref[nbn], FB_IDS);
  for (int f = threadIdx.x; f < tot; f += T) {
    int lo = 0, hi = nbn - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (m.s_pref[mid] <= f) lo = mid; else hi = mid - 1;
    }
    m.s_bd[f] = __ldg(a.digitL + m.s_cs0[lo] + (f - m.s_pref[lo]));
  }
  __syncthreads();
}

// thread counts of the warp-specialised backward: 4 producer warps, then the
// dG_F warps (8 x 8 tiles over K x 128) and the dA warps (8 x 4 tiles over
// 64 x K)
template <int K>
struct WsRoles {
  static constexpr int PROD = 128, DG = K * 128 / 64, DA = FB_BM * K / 32, T = PROD + DG + DA;
};

template <int K, int RP, int NL>
__device__ __forceinline__ void ws_producer(const FusedArgs& a, const WsSmem& m, int g0, int g1, int cb) {
  constexpr int BM = FB_BM, BN = 128, NPT = BM / RP, NB = WS_NB, T = WsRoles<K>::T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int nb0 = g0; nb0 < g1; nb0 += NB) {
    const int nbn = min(NB, g1 - nb0);
    ws_batch_prologue<T>(a, m, nb0, nbn);
    const int TT = (nbn + NPT - 1) / NPT;
    for (int t = 0; t < TT; ++t) {
      const int buf = t & 1, tb = t * NPT, nn = min(NPT, nbn - tb);
      if (t >= 2) named_sync2<3, T>(buf);  // the consumers released tile t - 2
      load_A_tile<K, RP, 128>(a, tb, nn, m.s_aoff, m.As0 + buf * BM * K);
      cp_async_commit();
#pragma unroll 1
      for (int q = 0; q < 2; ++q) {
        if constexpr (RP % 8 == 0)
          form_dC8<K, RP, NL>(a, tb, nn, cb, m.s_pref, m.s_cs0, m.s_bd, m.Ds0 + buf * BM * BN, warp * 16 + q * 8, lane);
        else
          form_dC<K, BN, RP, NL>(a, tb, nn, cb, m.s_pref, m.s_cs0, m.s_bd, m.Ds0 + buf * BM * BN, warp * 16 + q * 8);
      }
      cp_async_wait<0>();  // the A tile (and this thread's share of the slice block)
      named_arrive2<1, T>(buf);
    }
    for (int t = TT < 2 ? 2 : TT; t < TT + 2; ++t) named_sync2<3, T>(t & 1);  // the last releases
    __syncthreads();  // the batch's node metadata is rewritten by the next prologue
  }
}

template <int K, int RP, int NL>
__device__ __forceinline__ void ws_consumer(const FusedArgs& a, const WsSmem& m, int g0, int g1, int g, int cb,
                                            int chunk) {
  constexpr int BM = FB_BM, BN = 128, SB = BN + 4, NPT = BM / RP, NB = WS_NB;
  using R = WsRoles<K>;
  constexpr int T = R::T, KG = K / 4;
  const int tc = threadIdx.x - R::PROD;
  const bool gw = tc < R::DG;                                    // dG role
  const int kb = (tc >> 4) * 8, c0 = (tc & 15) * 4;             // dG role
  const int t2 = tc - R::DG, mg8 = (t2 / KG) * 8, kg = t2 % KG;  // dA role: k = kg + KG j
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  cp_async_wait<0>();  // this thread's share of the slice block
  for (int nb0 = g0; nb0 < g1; nb0 += NB) {
    const int nbn = min(NB, g1 - nb0);
    ws_batch_prologue<T>(a, m, nb0, nbn);
    const int TT = (nbn + NPT - 1) / NPT;
    for (int t = 0; t < TT; ++t) {
      const int buf = t & 1, tb = t * NPT, nn = min(NPT, nbn - tb), mlim = nn * RP;
      const float* As = m.As0 + buf * BM * K;
      const float* Ds = m.Ds0 + buf * BM * BN;
      named_sync2<1, T>(buf);
      if (gw) {
#pragma unroll 2
        for (int mm = 0; mm < BM; ++mm) {
          if (mm >= mlim) break;
          const float4 a0 = *reinterpret_cast<const float4*>(As + mm * K + kb);
          const float4 a1 = *reinterpret_cast<const float4*>(As + mm * K + kb + 4);
          const float4 d0 = *reinterpret_cast<const float4*>(Ds + mm * BN + c0);
          const float4 d1 = *reinterpret_cast<const float4*>(Ds + mm * BN + 64 + c0);
          const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
          const float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], dv[j], acc[i][j]);
        }
      } else if (mg8 < mlim) {
        // (the dA tile reuses the accumulator array: dA threads hold no dG_F)
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 4
        for (int n = 0; n < BN; n += 4) {
          float4 cv[8], bv[4];
#pragma unroll
          for (int i = 0; i < 8; ++i) cv[i] = *reinterpret_cast<const float4*>(Ds + (mg8 + i) * BN + n);
#pragma unroll
          for (int j = 0; j < 4; ++j) bv[j] = *reinterpret_cast<const float4*>(m.Bs + (kg + KG * j) * SB + n);
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              acc[i][j] = fmaf(cv[i].x, bv[j].x, acc[i][j]);
              acc[i][j] = fmaf(cv[i].y, bv[j].y, acc[i][j]);
              acc[i][j] = fmaf(cv[i].z, bv[j].z, acc[i][j]);
              acc[i][j] = fmaf(cv[i].w, bv[j].w, acc[i][j]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int mm = mg8 + i;
          const int j = mm / RP;
          if (j >= nn) continue;
          float* dst = a.dPc + ((int64_t)m.s_node[tb + j] * a.ncb + cb) * RP * K + (mm - j * RP) * K;
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) dst[kg + KG * jj] = acc[i][jj];
        }
      }
      named_arrive2<3, T>(buf);
    }
    __syncthreads();  // (matches the producers' end-of-batch barrier)
  }
  if (gw) {  // the group's (chunk's) dG_F column block
    float* gdst = (a.split > 1 ? a.gsplit + ((int64_t)g * a.split + chunk) * a.c.slice[a.F]
                                : a.grads + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F]) + cb * BN;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float* row = gdst + (int64_t)(kb + i) * a.NC;
      *reinterpret_cast<float4*>(row + c0) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      *reinterpret_cast<float4*>(row + 64 + c0) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
  }
}

template <int K, int RP, int NL>
__global__ void __launch_bounds__(WsRoles<K>::T, K <= 32 ? 2 : 1) k_fused_bwd_ws(FusedArgs a) {
  TT_PDL_ENTRY();
  constexpr int BN = 128, BM = FB_BM, SB = BN + 4, NB = WS_NB;
  static_assert(K == 32 || K == 64, "warp-specialised backward: K = 32 / 64");
  extern __shared__ __align__(16) float smem[];
  WsSmem m;
  m.Bs = smem;                       // [K][SB]
  m.As0 = m.Bs + K * SB;             // [2][BM][K]
  m.Ds0 = m.As0 + 2 * BM * K;        // [2][BM][BN]
  m.s_aoff = reinterpret_cast<int64_t*>(m.Ds0 + 2 * BM * BN);
  m.s_node = reinterpret_cast<int*>(m.s_aoff + NB);
  m.s_cs0 = m.s_node + NB;
  m.s_pref = m.s_cs0 + NB;
  m.s_wsum = m.s_pref + NB + 4;
  m.s_bd = m.s_wsum + 16;  // [FB_IDS]
  if (tt_failed(a.st)) return;
  int g, cb, g0, g1, chunk;
  if (!work_item(a, g, cb, chunk, g0, g1)) return;
  load_slice_block<K, BN, SB, WsRoles<K>::T>(a, g, cb, m.Bs);
  cp_async_commit();
  if (threadIdx.x < WsRoles<K>::PROD) ws_producer<K, RP, NL>(a, m, g0, g1, cb);
  else ws_consumer<K, RP, NL>(a, m, g0, g1, g, cb, chunk);
}

inline size_t bwd_ws_smem(int K) {
  return sizeof(float) * ((size_t)K * 132 + 2 * FB_BM * K + 2 * FB_BM * 128) + sizeof(int64_t) * WS_NB +
         sizeof(int) * (3 * WS_NB + 12 + 16 + FB_IDS) + 16;
}

// (K, RP, NL) instantiations of k_fused_bwd_ws (billion's level F; products /
// sweep32).  At K = 64 (one 384-thread CTA per SM) it measured slower than
// k_fused_bwd: papers 1.204 -> 1.283 ms, sweep64 0.468 -> 0.589 ms.
#define TT_BWDWS_SHAPES(X) X(32, 16, 4) X(32, 4, 8)

// Streaming kernels over the saved P_F, one warp per distinct ID
// (grid-stride).  The ID's prefix block P_F[p] (RP x NC floats, contiguous)
// is staged into the warp's shared buffer with coalesced 16-byte loads (all
// independent: the whole block is in flight at once), rows padded to K + 4.
#ifndef TT_SK_WARPS
#define TT_SK_WARPS 8
#endif
#ifndef TT_SK_MINB
#define TT_SK_MINB 2
#endif
constexpr int SK_WARPS = TT_SK_WARPS;  // warps per CTA of the streaming P_F kernels (A/B builds)

template <int K>
__device__ __forceinline__ void stage_prefix_block(const float* __restrict__ Cp, int nrow, float* buf, int lane) {
  const int n4 = nrow * (K / 4);
  constexpr int B8 = 16;  // the whole block (<= 2048 floats) in flight: one latency per ID
  for (int i0 = 0; i0 < n4; i0 += 32 * B8) {
    float4 v[B8];
#pragma unroll
    for (int b = 0; b < B8; ++b) {
      const int i = i0 + b * 32 + lane;
      if (i < n4) v[b] = __ldg(reinterpret_cast<const float4*>(Cp) + i);
    }
#pragma unroll
    for (int b = 0; b < B8; ++b) {
      const int i = i0 + b * 32 + lane;
      if (i < n4) {
        const int row = i / (K / 4), c4 = i - row * (K / 4);
        *reinterpret_cast<float4*>(buf + row * (K + 4) + c4 * 4) = v[b];
      }
    }
  }
  __syncwarp();
}

// The last level (forward rows): lane q owns output row block (ar, jf) = q:
// out[(q, jl)] = sum_r P_F[prefix][q][r] G_{d-1}[r, i_d, jl]; a row's NL
// outputs are contiguous, so a warp writes one contiguous output row per batch
// position.  IDs with more than HEAVY_POS positions go to Yu (k_scatter_heavy).
// PIPE (prefix blocks of <= 2048 floats): the next ID's block and last-core
// slice are loaded into registers while this ID is computed from shared
// memory, so every warp keeps a block in flight; the indices run one ID ahead
// of that.
template <int K, int NL, bool PIPE, int KS>
__global__ void __launch_bounds__(SK_WARPS * 32, TT_SK_MINB) k_last_level(FusedArgs a, const int* __restrict__ counts,
                                                              const int* __restrict__ parentL) {
  TT_PDL_ENTRY();
  extern __shared__ __align__(16) float sk_smem[];
  if (tt_failed(a.st)) return;
  constexpr int PB = 16;                      // block float4 per lane (PIPE)
  constexpr int GV = (K * NL / 4 + 31) / 32;  // slice float4 per lane (PIPE)
  const int U = ld_count(&counts[a.c.d - 1]);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int RP = a.RP, nF = a.nF, nrow = RP * nF;
  const int n4 = nrow * (K / 4);
  float* buf = sk_smem + wib * (nrow * (K + 4) + K * NL);
  float* Gs = buf + nrow * (K + 4);
  const int64_t emb = a.c.emb_dim, npad = a.c.npad;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];
  float4 pv[PIPE ? PB : 1], gr[PIPE ? GV : 1];
  auto issue = [&](int p, int dg, bool block) {  // (a block and) a slice into registers
    if (block) {
      const float4* src = reinterpret_cast<const float4*>(a.Psave + (int64_t)p * RP * a.NC);
#pragma unroll
      for (int b = 0; b < PB; ++b)
        if (b * 32 + lane < n4) pv[b] = __ldg(src + b * 32 + lane);
    }
    const float4* gs = reinterpret_cast<const float4*>(Gl + (int64_t)dg * sliceL);
#pragma unroll
    for (int b = 0; b < GV; ++b)
      if (b * 32 + lane < K * NL / 4) gr[b] = __ldg(gs + b * 32 + lane);
  };
  // each warp owns a contiguous run of distinct IDs: consecutive IDs share
  // their level-F prefix whenever the batch has locality (8 IDs per prefix in
  // the rank sweep), and the staged prefix block is then reused, not reloaded
  const int per = (U + nwarps - 1) / nwarps;
  int u = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * per;
  const int uend = min(U, u + per);
  int staged = -1;  // parent whose block is in buf
  int pn = 0, dn = 0, sn0 = 0, sn1 = 0;
  if (u < uend) { pn = __ldg(parentL + u); dn = __ldg(a.digitL + u); sn0 = __ldg(a.seg + u); sn1 = __ldg(a.seg + u + 1); }
  if constexpr (PIPE) {
    if (u < uend) issue(pn, dn, true);
  }
  for (; u < uend; ++u) {
    const int p = pn, dg = dn, s0 = sn0, s1 = sn1;
    const int un = u + 1;
    if (un < uend) {  // the next ID's indices under this ID
      pn = __ldg(parentL + un); dn = __ldg(a.digitL + un);
      sn0 = __ldg(a.seg + un); sn1 = __ldg(a.seg + un + 1);
    }
    if constexpr (PIPE) {
      if (p != staged) {
#pragma unroll
        for (int b = 0; b < PB; ++b) {
          const int i = b * 32 + lane;
          if (i < n4) {
            const int row = i / (K / 4), c4 = i - row * (K / 4);
            *reinterpret_cast<float4*>(buf + row * (K + 4) + c4 * 4) = pv[b];
          }
        }
        staged = p;
      }
#pragma unroll
      for (int b = 0; b < GV; ++b)
        if (b * 32 + lane < K * NL / 4) reinterpret_cast<float4*>(Gs)[b * 32 + lane] = gr[b];
      __syncwarp();
      if (un < uend) issue(pn, dn, pn != p);  // lands while this ID is computed
    } else {
      const float* Gsrc = Gl + (int64_t)dg * sliceL;
      for (int i = lane; i < K * NL / 4; i += 32)
        reinterpret_cast<float4*>(Gs)[i] = __ldg(reinterpret_cast<const float4*>(Gsrc) + i);
      if (p != staged) {
        stage_prefix_block<K>(a.Psave + (int64_t)p * RP * a.NC, nrow, buf, lane);
        staged = p;
      }
    }
    const float* Gp = Gs;
    // KS lanes per output row, each over K / KS ranks (KS = 2 when a block
    // has at most 16 rows: the two half-warps split the rank sum and combine
    // it with one shuffle, so no lane idles)
    static_assert(KS == 1 || KS == 2, "rank split");
    constexpr int KR = K / KS;
    const int kpart = KS == 2 ? (lane >> 4) : 0, qlane = KS == 2 ? (lane & 15) : lane;
    for (int q0 = 0; q0 < nrow; q0 += 32 / KS) {
      const int q = q0 + qlane;
      const float* crow = buf + (q < nrow ? q : 0) * (K + 4) + kpart * KR;
      const float* Gk = Gp + kpart * KR * NL;
      float o[NL];
#pragma unroll
      for (int jl = 0; jl < NL; ++jl) o[jl] = 0.f;
#pragma unroll
      for (int r = 0; r < KR; r += 4) {
        const float4 c = *reinterpret_cast<const float4*>(crow + r);
        const float cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if constexpr (NL % 4 == 0) {
#pragma unroll
            for (int l4 = 0; l4 < NL; l4 += 4) {
              const float4 gv = *reinterpret_cast<const float4*>(Gk + (r + t) * NL + l4);
              o[l4] = fmaf(cv[t], gv.x, o[l4]);
              o[l4 + 1] = fmaf(cv[t], gv.y, o[l4 + 1]);
              o[l4 + 2] = fmaf(cv[t], gv.z, o[l4 + 2]);
              o[l4 + 3] = fmaf(cv[t], gv.w, o[l4 + 3]);
            }
          } else {
#pragma unroll
            for (int jl = 0; jl < NL; ++jl) o[jl] = fmaf(cv[t], Gk[(r + t) * NL + jl], o[jl]);
          }
        }
      }
      if constexpr (KS == 2) {
#pragma unroll
        for (int jl = 0; jl < NL; ++jl) o[jl] += __shfl_xor_sync(0xffffffffu, o[jl], 16);
      }
      if (q >= nrow || kpart != 0) continue;
      const int64_t col = (int64_t)q * NL;
      if (s1 - s0 > HEAVY_POS) {
        st_vec<NL>(a.Yu + (int64_t)u * npad + col, o);
      } else if (col < emb) {
        for (int s = s0; s < s1; ++s) {
          float* orow = a.out + (int64_t)__ldg(a.spos + s) * emb + col;
          if constexpr (NL % 4 == 0) {
            st_vec<NL>(orow, o);
          } else {  // (rows are truncated to emb_dim: the last block may be partial)
#pragma unroll
            for (int jl = 0; jl < NL; ++jl)
              if (col + jl < emb) orow[jl] = o[jl];
          }
        }
      }
    }
    __syncwarp();
  }
}

// W_u = P_F[prefix(u)]^T dY_u over all NC columns (K x n_d per distinct ID):
// the last core's gradient contributions.  Lane owns RPL rank rows and sums
// over the block's nrow rows (no cross-lane reduction).
template <int K, int NL, bool PIPE>
__global__ void __launch_bounds__(SK_WARPS * 32, 2) k_fused_w(FusedArgs a, const int* __restrict__ counts,
                                                           const int* __restrict__ parentL) {
  TT_PDL_ENTRY();
  extern __shared__ __align__(16) float sk_smem[];
  if (tt_failed(a.st)) return;
  constexpr int RPL = K >= 32 ? K / 32 : 1;
  constexpr int PB = 16;  // block float4 per lane (PIPE: blocks of <= 2048 floats)
  constexpr int YB = 2;   // dY float4 per lane (PIPE: nrow * NL <= 256)
  const int U = ld_count(&counts[a.c.d - 1]);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int RP = a.RP, nF = a.nF, nrow = RP * nF;
  const int n4 = nrow * (K / 4), y4 = nrow * NL / 4;
  float* buf = sk_smem + wib * (nrow * (K + 4) + nrow * NL);
  float* Ys = buf + nrow * (K + 4);
  const int64_t npad = a.c.npad;
  const int r0 = lane * RPL;
  float4 pv[PIPE ? PB : 1], yr[PIPE ? YB : 1];
  auto issue = [&](int u, int p, bool block) {  // ID u's (prefix block and) dY row into registers
    if (block) {
      const float4* src = reinterpret_cast<const float4*>(a.Psave + (int64_t)p * RP * a.NC);
#pragma unroll
      for (int b = 0; b < PB; ++b)
        if (b * 32 + lane < n4) pv[b] = __ldg(src + b * 32 + lane);
    }
    const float4* ys = reinterpret_cast<const float4*>(a.dY + (int64_t)u * npad);
#pragma unroll
    for (int b = 0; b < YB; ++b)
      if (b * 32 + lane < y4) yr[b] = __ldg(ys + b * 32 + lane);
  };
  // contiguous runs of IDs per warp, the staged prefix block reused across
  // IDs of one prefix (as in k_last_level)
  const int per = (U + nwarps - 1) / nwarps;
  int u = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * per;
  const int uend = min(U, u + per);
  int staged = -1;
  int pn = u < uend ? __ldg(parentL + u) : 0;
  if constexpr (PIPE) {
    if (u < uend) issue(u, pn, true);
  }
  for (; u < uend; ++u) {
    const int p = pn;
    const int un = u + 1;
    if (un < uend) pn = __ldg(parentL + un);  // next ID's parent under this ID
    if constexpr (PIPE) {
      if (p != staged) {
#pragma unroll
        for (int b = 0; b < PB; ++b) {
          const int i = b * 32 + lane;
          if (i < n4) {
            const int row = i / (K / 4), c4 = i - row * (K / 4);
            *reinterpret_cast<float4*>(buf + row * (K + 4) + c4 * 4) = pv[b];
          }
        }
        staged = p;
      }
#pragma unroll
      for (int b = 0; b < YB; ++b)
        if (b * 32 + lane < y4) reinterpret_cast<float4*>(Ys)[b * 32 + lane] = yr[b];
      __syncwarp();
      if (un < uend) issue(un, pn, pn != p);  // lands while this ID is computed
    } else {
      const float* Yp = a.dY + (int64_t)u * npad;
      for (int i = lane; i < y4; i += 32)
        reinterpret_cast<float4*>(Ys)[i] = __ldg(reinterpret_cast<const float4*>(Yp) + i);
      if (p != staged) {
        stage_prefix_block<K>(a.Psave + (int64_t)p * RP * a.NC, nrow, buf, lane);
        staged = p;
      }
    }
    if (r0 < K) {
      float wv[RPL][NL];
#pragma unroll
      for (int i = 0; i < RPL; ++i)
#pragma unroll
        for (int jl = 0; jl < NL; ++jl) wv[i][jl] = 0.f;
#pragma unroll 8
      for (int q = 0; q < nrow; ++q) {
        float yv[NL], cv[RPL];
        if constexpr (NL % 4 == 0) {
#pragma unroll
          for (int l4 = 0; l4 < NL; l4 += 4) {
            const float4 x = *reinterpret_cast<const float4*>(Ys + q * NL + l4);
            yv[l4] = x.x; yv[l4 + 1] = x.y; yv[l4 + 2] = x.z; yv[l4 + 3] = x.w;
          }
        } else {
#pragma unroll
          for (int jl = 0; jl < NL; ++jl) yv[jl] = Ys[q * NL + jl];
        }
#pragma unroll
        for (int i = 0; i < RPL; ++i) cv[i] = buf[q * (K + 4) + r0 + i];
#pragma unroll
        for (int i = 0; i < RPL; ++i)
#pragma unroll
          for (int jl = 0; jl < NL; ++jl) wv[i][jl] = fmaf(cv[i], yv[jl], wv[i][jl]);
      }
      float* wdst = a.W + (int64_t)u * K * NL + r0 * NL;
#pragma unroll
      for (int i = 0; i < RPL; ++i) st_vec<NL>(wdst + i * NL, wv[i]);
    }
    __syncwarp();
  }
}

// k_fused_w plus dC = dP_F for the tensor backward (path tc, round 2): per
// level-F node p, dC[q][r] = sum over p's distinct IDs u of
// sum_jl dY_u[q][jl] G_{d-1}[r, i_d(u), jl], written over p's saved P_F block
// (same layout: row q = a n_F + jf, column r) once every W_u of p has read it.
// k_tc_bwd2<..., true> then streams dC tiles instead of forming them from
// dependent L2 loads.  Warps own node-aligned runs of IDs (a run starts at the
// first ID of a node: cstartF), so each block is written by one warp.  Lane
// owns rank columns r0 .. r0 + RPL of both W_u and dC.
template <int K, int NL>
__global__ void __launch_bounds__(SK_WARPS * 32, 1) k_fused_wdc(FusedArgs a, const int* __restrict__ counts,
                                                             const int* __restrict__ parentL) {
  TT_PDL_ENTRY();
  extern __shared__ __align__(16) float sk_smem[];
  if (tt_failed(a.st)) return;
  static_assert(K == 32 || K == 64, "rank");
  constexpr int RPL = K / 32;
  constexpr int QMAX = 2048 / K;  // block rows (PIPE blocks: <= 2048 floats)
  constexpr int PB = 16;
  constexpr int YB = 2;
  const int U = ld_count(&counts[a.c.d - 1]);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int RP = a.RP, nF = a.nF, nrow = RP * nF;
  const int n4 = nrow * (K / 4), y4 = nrow * NL / 4;
  float* buf = sk_smem + wib * (nrow * (K + 4) + nrow * NL);
  float* Ys = buf + nrow * (K + 4);
  const int64_t npad = a.c.npad;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];
  const int r0 = lane * RPL;
  float4 pv[PB], yr[YB];
  float gr[RPL * NL];
  auto issue = [&](int u, int p, bool block) {  // ID u's (prefix block,) dY row and slice rows
    if (block) {
      const float4* src = reinterpret_cast<const float4*>(a.Psave + (int64_t)p * RP * a.NC);
#pragma unroll
      for (int b = 0; b < PB; ++b)
        if (b * 32 + lane < n4) pv[b] = __ldg(src + b * 32 + lane);
    }
    const float4* ys = reinterpret_cast<const float4*>(a.dY + (int64_t)u * npad);
#pragma unroll
    for (int b = 0; b < YB; ++b)
      if (b * 32 + lane < y4) yr[b] = __ldg(ys + b * 32 + lane);
    const float4* gs = reinterpret_cast<const float4*>(Gl + (int64_t)__ldg(a.digitL + u) * sliceL + r0 * NL);
#pragma unroll
    for (int b = 0; b < RPL * NL / 4; ++b) {
      const float4 x = __ldg(gs + b);
      gr[4 * b] = x.x; gr[4 * b + 1] = x.y; gr[4 * b + 2] = x.z; gr[4 * b + 3] = x.w;
    }
  };
  // node-aligned run: the first ID at or after v that starts a node
  auto node_start = [&](int v) {
    if (v <= 0) return 0;
    if (v >= U) return U;
    const int p = __ldg(parentL + v);
    const int c0 = __ldg(a.cstartF + p);
    return c0 == v ? v : __ldg(a.cstartF + p + 1);
  };
  const int per = (U + nwarps - 1) / nwarps;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int u = node_start(min(U, w * per));
  const int uend = node_start(min(U, (w + 1) * per));
  float dc[QMAX][RPL];
#pragma unroll
  for (int q = 0; q < QMAX; ++q)
#pragma unroll
    for (int i = 0; i < RPL; ++i) dc[q][i] = 0.f;
  int staged = -1;
  int pn = u < uend ? __ldg(parentL + u) : 0;
  if (u < uend) issue(u, pn, true);
  for (; u < uend; ++u) {
    const int p = pn;
    const int un = u + 1;
    if (un < uend) pn = __ldg(parentL + un);
    if (p != staged) {
#pragma unroll
      for (int b = 0; b < PB; ++b) {
        const int i = b * 32 + lane;
        if (i < n4) {
          const int row = i / (K / 4), c4 = i - row * (K / 4);
          *reinterpret_cast<float4*>(buf + row * (K + 4) + c4 * 4) = pv[b];
        }
      }
      staged = p;
    }
#pragma unroll
    for (int b = 0; b < YB; ++b)
      if (b * 32 + lane < y4) reinterpret_cast<float4*>(Ys)[b * 32 + lane] = yr[b];
    float g[RPL * NL];
#pragma unroll
    for (int i = 0; i < RPL * NL; ++i) g[i] = gr[i];
    __syncwarp();
    const bool last = un >= uend || pn != p;
    if (un < uend) issue(un, pn, pn != p);  // lands while this ID is computed
    float wv[RPL][NL];
#pragma unroll
    for (int i = 0; i < RPL; ++i)
#pragma unroll
      for (int jl = 0; jl < NL; ++jl) wv[i][jl] = 0.f;
#pragma unroll
    for (int q = 0; q < QMAX; ++q) {
      if (q < nrow) {
        float yv[NL], cv[RPL];
#pragma unroll
        for (int l4 = 0; l4 < NL; l4 += 4) {
          const float4 x = *reinterpret_cast<const float4*>(Ys + q * NL + l4);
          yv[l4] = x.x; yv[l4 + 1] = x.y; yv[l4 + 2] = x.z; yv[l4 + 3] = x.w;
        }
#pragma unroll
        for (int i = 0; i < RPL; ++i) cv[i] = buf[q * (K + 4) + r0 + i];
#pragma unroll
        for (int i = 0; i < RPL; ++i)
#pragma unroll
          for (int jl = 0; jl < NL; ++jl) {
            wv[i][jl] = fmaf(cv[i], yv[jl], wv[i][jl]);
            dc[q][i] = fmaf(yv[jl], g[i * NL + jl], dc[q][i]);
          }
      }
    }
    float* wdst = a.W + (int64_t)u * K * NL + r0 * NL;
#pragma unroll
    for (int i = 0; i < RPL; ++i) st_vec<NL>(wdst + i * NL, wv[i]);
    if (last) {  // p's block is in smem (and every W_u of p done): dC over it
      float* dst = a.Psave + (int64_t)p * RP * a.NC + r0;
#pragma unroll
      for (int q = 0; q < QMAX; ++q) {
        if (q < nrow) {
          if constexpr (RPL == 2) *reinterpret_cast<float2*>(dst + q * K) = make_float2(dc[q][0], dc[q][1]);
          else dst[q * K] = dc[q][0];
        }
#pragma unroll
        for (int i = 0; i < RPL; ++i) dc[q][i] = 0.f;
      }
    }
    __syncwarp();
  }
}

// dG_{d-1}[v] = sum over the digit-v IDs (group order) and column blocks of W.
// 256 threads = S sub-groups x (WE/4) float4 columns; sub-group sg sums the
// (member, column block) pairs q = sg, sg+S, ... in order, and the S partials
// are combined in sub-group order (a fixed tree: deterministic).
template <int T>
__global__ void __launch_bounds__(T) k_fused_reduce_last(DevCfg c, int ncb, int WE, const int* __restrict__ goffL,
                                                           const int* __restrict__ orderL, const float* __restrict__ W,
                                                           float* __restrict__ grads, const DevStatus* st) {
  TT_PDL_ENTRY();
  __shared__ float4 red[T];
  if (tt_failed(st)) return;
  const int v = blockIdx.x;
  const int g0 = goffL[v], g1 = goffL[v + 1];
  if (g0 == g1) return;
  const int cols = WE / 4;
  const int S = cols >= T ? 1 : T / cols;
  float* dst = grads + c.core_off[c.d - 1] + (int64_t)v * c.slice[c.d - 1];
  const int npair = (g1 - g0) * ncb;
  for (int col0 = 0; col0 < cols; col0 += T) {
    const int sg = threadIdx.x / min(cols, T), col = col0 + threadIdx.x % min(cols, T);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (sg < S && col < cols) {
      int q = sg;
      for (; q + 3 * S < npair; q += 4 * S) {
        float4 x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int qq = q + i * S, gi = g0 + qq / ncb, cbi = qq - (qq / ncb) * ncb;
          x[i] = *reinterpret_cast<const float4*>(W + ((int64_t)orderL[gi] * ncb + cbi) * WE + col * 4);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc.x += x[i].x; acc.y += x[i].y; acc.z += x[i].z; acc.w += x[i].w;
        }
      }
      for (; q < npair; q += S) {
        const int gi = g0 + q / ncb, cbi = q - (q / ncb) * ncb;
        const float4 x = *reinterpret_cast<const float4*>(W + ((int64_t)orderL[gi] * ncb + cbi) * WE + col * 4);
        acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      }
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < min(cols, T) && col0 + threadIdx.x < cols) {
      float4 t = red[threadIdx.x];
      for (int s2 = 1; s2 < S; ++s2) {
        const float4 y = red[s2 * min(cols, T) + threadIdx.x];
        t.x += y.x; t.y += y.y; t.z += y.z; t.w += y.w;
      }
      *reinterpret_cast<float4*>(dst + (col0 + threadIdx.x) * 4) = t;
    }
    __syncthreads();
  }
}

// dP_{F-1}[p] (or dG_0 when F == 1) = sum over children and column blocks of dPc
__global__ void k_fused_reduce_children(DevCfg c, int F, int ncb, int per, const int* __restrict__ counts,
                                        const int* __restrict__ cstart_pm1, const int* __restrict__ digit0,
                                        const float* __restrict__ dPc, float* __restrict__ dst,
                                        const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  const int cnt = ld_count(&counts[F - 1]);
  const int64_t total = (int64_t)cnt * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(t / per);
    const int e = (int)(t - (int64_t)p * per);
    const int n0 = cstart_pm1[p] * ncb, n1 = cstart_pm1[p + 1] * ncb;  // (child, cb) pairs are contiguous
    // 32 loads in flight per thread (the loop is latency-bound; the adds stay
    // in q order, so the sum is the same for any batch size)
    float acc = 0.f;
    int q = n0;
    for (; q + 32 <= n1; q += 32) {
      float x[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = dPc[(int64_t)(q + i) * per + e];
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += x[i];
    }
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

// dG_F[g] = sum over the group's nonempty chunks c (ascending) of gpart[g][c]
// (split > 1; a fixed order, so the result does not depend on scheduling).
__global__ void k_fused_reduce_gsplit(DevCfg c, int F, int split, int split_rows, const int* __restrict__ goffF,
                                      const float* __restrict__ gsplit, float* __restrict__ grads, const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  const int64_t per4 = c.slice[F] / 4;
  const int64_t total = c.m[F] * per4;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int g = (int)(t / per4);
    const int64_t e4 = t - (int64_t)g * per4;
    const int n = goffF[g + 1] - goffF[g];
    if (n == 0) continue;
    const int nch = group_chunks(n, (int)c.rows[F], split, split_rows);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int ch = 0; ch < nch; ++ch) {
      if (((int64_t)n * (ch + 1)) / nch == ((int64_t)n * ch) / nch) continue;  // empty chunk: nothing written
      const float4 x = reinterpret_cast<const float4*>(gsplit + ((int64_t)g * split + ch) * c.slice[F])[e4];
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    reinterpret_cast<float4*>(grads + c.core_off[F] + (int64_t)g * c.slice[F])[e4] = acc;
  }
}

// ---------------------------------------------------------------------------
// Low-rank streaming backward (round 2, K <= 16: small, sweep8, sweep16).  At
// these ranks the level-F GEMMs are a few FMAs per upstream float and
// k_fused_bwd is bound by forming dC one ID at a time per warp, then waiting
// at the tile barrier for the warp with the most IDs (sweep8 ncu: barrier 47%,
// long_scoreboard 34% of stall samples, issue 17%).  Here every warp owns a
// chunk of one digit group's nodes (work_item_at over groups x LR_SPLIT
// chunks; the chunks' dG_F partials are summed by k_fused_reduce_gsplit in
// chunk order) and walks it with no barrier at all:
//   lane l owns the CPL columns c = l + 32 i of the level-F block (NC = 32 CPL,
//   column c = jf K + r) and keeps S_g[:, c] (the slice) and dG_F[:, c] in
//   registers;
//   per node: its A rows (core-0 slice or P_{F-1} rows, RP x K) staged in the
//   warp's shared memory; dC[ar][c] = sum over the node's IDs u (digits
//   fetched lane-parallel, up to 32 per load) of sum_jl dY_u[ar, jf, jl]
//   G_last[i_d(u)][r, jl]; dG_F[k][c] += sum_ar A[ar][k] dC[ar][c];
//   dA[ar][k] = sum_c dC[ar][c] S[k][c] as RP K per-lane partials,
//   reduce-scattered over the warp (lane l ends with entries l RP K / 32 ..)
//   and written as the node's dP_{F-1} partial (ncb = 1).
// Every sum runs in a fixed order (IDs in distinct-ID order, lanes in a fixed
// butterfly), so results are deterministic.
constexpr int LR_WARPS = 4, LR_SPLIT = 32;
template <int K, int RP, int NL, int CPL>
__global__ void __launch_bounds__(LR_WARPS * 32) k_lowrank_bwd(FusedArgs a) {
  TT_PDL_ENTRY();
  constexpr int NC = 32 * CPL, V = RP * K, VL = V / 32;
  static_assert(V % 32 == 0 && V >= 32, "RP K must be a multiple of 32");
  __shared__ float s_A[LR_WARPS][RP * K];
  if (tt_failed(a.st)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int it = blockIdx.x * LR_WARPS + warp;
  if (it >= a.c.m[a.F] * a.split) return;
  int g, cb, chunk, g0, g1;
  if (!work_item_at(a, it, g, cb, chunk, g0, g1)) return;
  const int nF = a.nF;
  const int64_t npad = a.c.npad;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];
  const float* S = a.params + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F];
  int jf[CPL], rr[CPL];
  float sv[K][CPL], gacc[K][CPL];
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    const int col = lane + 32 * i;
    jf[i] = col / K;
    rr[i] = col % K;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      sv[k][i] = __ldg(S + (int64_t)k * NC + col);
      gacc[k][i] = 0.f;
    }
  }
  float* sA = s_A[warp];
  for (int n = g0; n < g1; ++n) {
    const int node = __ldg(a.orderF + n);
    const int p = __ldg(a.parentF + node);
    const float* Ap = a.Abase + (a.F == 1 ? a.c.core_off[0] + (int64_t)__ldg(a.digit0 + p) * a.c.slice[0]
                                          : (int64_t)p * RP * K);
    __syncwarp();  // the previous node's A rows are no longer read
#pragma unroll
    for (int t = 0; t < V / 32; ++t) sA[lane + 32 * t] = __ldg(Ap + lane + 32 * t);
    const int c0 = __ldg(a.cstartF + node), c1 = __ldg(a.cstartF + node + 1);
    float dc[RP][CPL];
#pragma unroll
    for (int ar = 0; ar < RP; ++ar)
#pragma unroll
      for (int i = 0; i < CPL; ++i) dc[ar][i] = 0.f;
    // an ID's operands: its last-core slice row r of column c and the node's
    // RP upstream row parts (jf(c), 0..NL) -- two IDs in flight (registers
    // double-buffered; static buffers, the loop is unrolled by two)
    float gA[CPL][NL], yA[CPL][RP][NL], gB[CPL == 1 ? CPL : 1][NL], yB[CPL == 1 ? CPL : 1][RP][NL];
    auto ld_id = [&](int u, int dg, float (&gv)[CPL][NL], float (&yv)[CPL][RP][NL]) {
      const float* Gp = Gl + (int64_t)dg * sliceL;
      const float* Yp = a.dY + (int64_t)u * npad;
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        ldg_vec<NL>(Gp + rr[i] * NL, gv[i]);
#pragma unroll
        for (int ar = 0; ar < RP; ++ar) ldg_vec<NL>(Yp + ((int64_t)ar * nF + jf[i]) * NL, yv[i][ar]);
      }
    };
    // WF (CPL = 1): the last core's W_u = P_F^T dY_u here too (k_fused_w does
    // not run): lane (jf, r) forms sum_ar P_F[ar][(jf, r)] dY_u[ar, jf, :], the
    // lanes of one r (jf = 0..nF-1, K apart) reduce-scatter the NL sums, and
    // each writes NL / nF of W_u[r][:]
    constexpr int NFL = 32 / K;  // lanes sharing a rank column r (the jf bits of the lane)
    constexpr bool WF = NFL >= 1 && NL % NFL == 0;
    float pf[RP][CPL];
    if constexpr (WF) {
#pragma unroll
      for (int ar = 0; ar < RP; ++ar)
#pragma unroll
        for (int i = 0; i < CPL; ++i) pf[ar][i] = __ldg(a.Psave + (int64_t)node * RP * NC + ar * NC + lane + 32 * i);
    }
    auto acc_id = [&](int u, const float (&gv)[CPL][NL], const float (&yv)[CPL][RP][NL]) {
#pragma unroll
      for (int i = 0; i < CPL; ++i)
#pragma unroll
        for (int ar = 0; ar < RP; ++ar) {
          float s = dc[ar][i];
#pragma unroll
          for (int jl = 0; jl < NL; ++jl) s = fmaf(yv[i][ar][jl], gv[i][jl], s);
          dc[ar][i] = s;
        }
      if constexpr (WF) {
        float w[NL];
#pragma unroll
        for (int jl = 0; jl < NL; ++jl) {
          float x = 0.f;
#pragma unroll
          for (int i = 0; i < CPL; ++i)
#pragma unroll
            for (int ar = 0; ar < RP; ++ar) x = fmaf(pf[ar][i], yv[i][ar][jl], x);
          w[jl] = x;
        }
        // reduce-scatter over the jf bits of the lane (distances 16, 8, .. K)
        int len = NL;
#pragma unroll
        for (int dist = 16; dist >= K; dist >>= 1) {
          const int half = len >> 1;
          const bool hi = (lane & dist) != 0;
#pragma unroll
          for (int i = 0; i < NL / 2; ++i)
            if (i < half) {
              const float give = hi ? w[i] : w[half + i];
              const float keep = hi ? w[half + i] : w[i];
              w[i] = keep + __shfl_xor_sync(0xffffffffu, give, dist);
            }
          len = half;
        }
        // lane (jf, r) holds W_u[r][jl0 .. jl0 + NL / NFL), jl0 = the jf bits read high to low
        int jl0 = 0, blk = NL;
#pragma unroll
        for (int dist = 16; dist >= K; dist >>= 1) {
          blk >>= 1;
          if (lane & dist) jl0 += blk;
        }
        float* wd = a.W + (int64_t)u * K * NL + (lane % K) * NL + jl0;
#pragma unroll
        for (int i = 0; i < NL / NFL; ++i) wd[i] = w[i];
      }
    };
    for (int u0 = c0; u0 < c1; u0 += 32) {
      const int nu = min(32, c1 - u0);
      const int my_dg = lane < nu ? __ldg(a.digitL + u0 + lane) : 0;
      if constexpr (CPL > 1) {  // (two IDs' operands would not fit the registers)
        for (int q = 0; q < nu; ++q) {
          ld_id(u0 + q, __shfl_sync(0xffffffffu, my_dg, q), gA, yA);
          acc_id(u0 + q, gA, yA);
        }
      } else {
      ld_id(u0, __shfl_sync(0xffffffffu, my_dg, 0), gA, yA);
      for (int q = 0; q < nu; q += 2) {
        const int dgB = __shfl_sync(0xffffffffu, my_dg, (q + 1) & 31);
        const int dgA = __shfl_sync(0xffffffffu, my_dg, (q + 2) & 31);
        if (q + 1 < nu) ld_id(u0 + q + 1, dgB, gB, yB);
        acc_id(u0 + q, gA, yA);
        if (q + 1 < nu) {
          if (q + 2 < nu) ld_id(u0 + q + 2, dgA, gA, yA);
          acc_id(u0 + q + 1, gB, yB);
        }
      }
      }
    }
    __syncwarp();  // sA complete
    // dG_F[k][c] += sum_ar A[ar][k] dC[ar][c]
#pragma unroll
    for (int ar = 0; ar < RP; ++ar)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const float av = sA[ar * K + k];
#pragma unroll
        for (int i = 0; i < CPL; ++i) gacc[k][i] = fmaf(av, dc[ar][i], gacc[k][i]);
      }
    // dA[ar][k] = sum_c dC[ar][c] S[k][c], 32 entries at a time: per-lane
    // partials, then a butterfly reduce-scatter (lane l keeps entry t 32 + l)
    float* dst = a.dPc + (int64_t)node * V;  // ncb = 1
#pragma unroll
    for (int t = 0; t < VL; ++t) {
      float v[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int ar = (t * 32 + e) / K, k = (t * 32 + e) % K;
        float x = 0.f;
#pragma unroll
        for (int i = 0; i < CPL; ++i) x = fmaf(dc[ar][i], sv[k][i], x);
        v[e] = x;
      }
#pragma unroll
      for (int st = 0; st < 5; ++st) {
        const int half = 16 >> st;
        const bool hi = (lane >> (4 - st)) & 1;
#pragma unroll
        for (int i = 0; i < half; ++i) {
          const float give = hi ? v[i] : v[half + i];
          const float keep = hi ? v[half + i] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, give, half);
        }
      }
      dst[t * 32 + lane] = v[0];
    }
  }
  float* gdst = a.split > 1 ? a.gsplit + ((int64_t)g * a.split + chunk) * a.c.slice[a.F]
                            : a.grads + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int i = 0; i < CPL; ++i) gdst[(int64_t)k * NC + lane + 32 * i] = gacc[k][i];
}

// Low-rank streaming forward (round 2, R = 8 with one 32-column block: the
// rank sweep's R = 8).  k_fused_fwd's 64-row GEMM tiles are a few FMAs per
// loaded float here, and k_last_level then re-reads every P_F block; instead
// a warp walks a chunk of one digit group's nodes (the backward's work items):
//   lane l = level-F column (jf, r) keeps S_g[:, l] in registers;
//   per node: P_F[ar][l] = sum_k A[ar][k] S[k][l] (A rows broadcast by
//   shuffles), stored for the backward; then for each distinct ID u of the
//   node (digits / position ranges fetched lane-parallel) the lane's 32
//   partial outputs P_F[ar][l] G_last[i_d(u)][r, jl] are reduce-scattered over
//   the 8 lanes of its jf (xor 4, 2, 1) so lane (jf, r) holds outputs
//   (ar = r / 2, jf, jl = 4 (r % 2) ..+4): one float4 per lane and position, the
//   warp writing the whole 128-float row (heavy IDs: their Yu row, scattered
//   later by k_scatter_heavy).
template <int K, int RP, int NL, int CPL>
__global__ void __launch_bounds__(LR_WARPS * 32) k_lowrank_fwd(FusedArgs a) {
  TT_PDL_ENTRY();
  // lane l owns columns l + 32 i (i < CPL): jf_i = (l + 32 i) / K, r = l % K;
  // an ID's CPL RP NL partial outputs are reduce-scattered over the log2(K) r
  // bits of the lane, leaving V / K = 4 per lane: entries 4 (l % K) ..+4 of
  // [i][ar][jl]
  constexpr int NC = 32 * CPL, NFJ = NC / K, V = CPL * RP * NL, AE = RP * K / 32;
  static_assert(V == 4 * K && (RP * K) % 32 == 0 && 32 % K == 0, "one float4 of outputs per lane");
  if (tt_failed(a.st)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int it = blockIdx.x * LR_WARPS + warp;
  if (it >= a.c.m[a.F] * a.split) return;
  int g, cb, chunk, g0, g1;
  if (!work_item_at(a, it, g, cb, chunk, g0, g1)) return;
  const int r = lane % K;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];
  const int64_t emb = a.c.emb_dim, npad = a.c.npad;
  const float* S = a.params + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F];
  float sv[CPL][K];
#pragma unroll
  for (int i = 0; i < CPL; ++i)
#pragma unroll
    for (int k = 0; k < K; ++k) sv[i][k] = __ldg(S + k * NC + lane + 32 * i);
  // this lane's output quad: entries e0 .. e0 + 3 of [i][ar][jl], e0 = 4 r
  const int e0 = 4 * r, oi = e0 / (RP * NL), oar = (e0 % (RP * NL)) / NL, ojl = e0 % NL;
  const int ojf = (lane + 32 * oi) / K;
  const int64_t ocol = ((int64_t)oar * NFJ + ojf) * NL + ojl;
  for (int n = g0; n < g1; ++n) {
    const int node = __ldg(a.orderF + n);
    const int p = __ldg(a.parentF + node);
    const float* Ap = a.Abase + (a.F == 1 ? a.c.core_off[0] + (int64_t)__ldg(a.digit0 + p) * a.c.slice[0]
                                          : (int64_t)p * RP * K);
    float my_a[AE];  // A[ar][k] = element ar K + k, held by lane (ar K + k) % 32 in slot / 32
#pragma unroll
    for (int t = 0; t < AE; ++t) my_a[t] = __ldg(Ap + lane + 32 * t);
    const int c0 = __ldg(a.cstartF + node), c1 = __ldg(a.cstartF + node + 1);
    float pf[RP][CPL];
#pragma unroll
    for (int ar = 0; ar < RP; ++ar) {
      float x[CPL];
#pragma unroll
      for (int i = 0; i < CPL; ++i) x[i] = 0.f;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const float av = __shfl_sync(0xffffffffu, my_a[(ar * K + k) / 32], (ar * K + k) % 32);
#pragma unroll
        for (int i = 0; i < CPL; ++i) x[i] = fmaf(av, sv[i][k], x[i]);
      }
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        pf[ar][i] = x[i];
        a.Psave[(int64_t)node * RP * NC + ar * NC + lane + 32 * i] = x[i];
      }
    }
    for (int u0 = c0; u0 < c1; u0 += 32) {
      const int nu = min(32, c1 - u0);
      int my_dg = 0, my_s0 = 0, my_s1 = 0, my_p0 = 0;
      if (lane < nu) {
        my_dg = __ldg(a.digitL + u0 + lane);
        my_s0 = __ldg(a.seg + u0 + lane);
        my_s1 = __ldg(a.seg + u0 + lane + 1);
        my_p0 = __ldg(a.spos + my_s0);  // the first position (most IDs have one or two)
      }
      // the next ID's slice row is loaded under this ID's reduction (static
      // double buffer: the loop is unrolled by two)
      float gA[NL], gB[NL];
      auto ldg_g = [&](int q, float (&gv)[NL]) {
        ldg_vec<NL>(Gl + (int64_t)__shfl_sync(0xffffffffu, my_dg, q & 31) * sliceL + r * NL, gv);
      };
      auto emit = [&](int q, const float (&gv)[NL]) {
        const int u = u0 + q;
        const int s0 = __shfl_sync(0xffffffffu, my_s0, q), s1 = __shfl_sync(0xffffffffu, my_s1, q);
        const int p0 = __shfl_sync(0xffffffffu, my_p0, q);
        float v[V];  // v[(i RP + ar) NL + jl]
#pragma unroll
        for (int i = 0; i < CPL; ++i)
#pragma unroll
          for (int ar = 0; ar < RP; ++ar)
#pragma unroll
            for (int jl = 0; jl < NL; ++jl) v[(i * RP + ar) * NL + jl] = pf[ar][i] * gv[jl];
#pragma unroll
        for (int dist = K / 2; dist >= 1; dist >>= 1) {  // over the r bits of the lane, high to low
          const int half = (V * dist) / K;
          const bool hi = (lane & dist) != 0;
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const float give = hi ? v[i] : v[half + i];
            const float keep = hi ? v[half + i] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, give, dist);
          }
        }
        const float4 o = make_float4(v[0], v[1], v[2], v[3]);
        if (s1 - s0 > HEAVY_POS) {
          *reinterpret_cast<float4*>(a.Yu + (int64_t)u * npad + ocol) = o;
        } else {
          *reinterpret_cast<float4*>(a.out + (int64_t)p0 * emb + ocol) = o;
          for (int sl = s0 + 1; sl < s1; ++sl)
            *reinterpret_cast<float4*>(a.out + (int64_t)__ldg(a.spos + sl) * emb + ocol) = o;
        }
      };
      ldg_g(0, gA);
      for (int q = 0; q < nu; q += 2) {
        if (q + 1 < nu) ldg_g(q + 1, gB);
        emit(q, gA);
        if (q + 1 < nu) {
          if (q + 2 < nu) ldg_g(q + 2, gA);
          emit(q + 1, gB);
        }
      }
    }
  }
}
// (K, RP, NL, CPL) instantiations of k_lowrank_fwd: sweep8.  The two-column
// version (R = 16) is parity-tested but measured slower or equal (sweep16 0.454
// -> 0.475, small 0.143 -> 0.142 ms/step; profiles/r02/NOTES.md)
#define TT_LOWRANK_FWD_SHAPES(X) X(8, 4, 8, 1)

// (K, RP, NL, CPL) instantiations of k_lowrank_bwd: sweep8.  At R = 16 (CPL 2:
// one ID's operands at a time) it measured slower than k_fused_bwd + k_fused_w
// (sweep16 0.454 -> 0.485 ms/step, small 0.144 -> 0.146; profiles/r02/NOTES.md)
#define TT_LOWRANK_SHAPES(X) X(8, 4, 8, 1)

// The (K, BN, RP, NL) instantiations compiled into the library (engine.cu
// FUSED_SWITCH): papers, products / sweep32, small (and the paper's Table-4
// arxiv / papers100M shapes at R = 16), billion, sweep16, sweep64, sweep128,
// sweep8, the Table-4 arxiv / papers100M shapes (n = (8,4,4)) at R = 32 and
// 64, and the Table-4 products shape (n = (4,5,5), NC = 5R) at R = 32 and 64.
#define TT_FUSED_SHAPES(X) \
  X(64, 128, 4, 4) X(32, 128, 4, 8) X(16, 64, 8, 4) X(32, 128, 16, 4) X(16, 64, 4, 8) X(64, 128, 4, 8) X(128, 64, 4, 8) \
  X(128, 128, 4, 8) X(8, 32, 4, 8) X(32, 128, 8, 4) X(64, 128, 8, 4) X(32, 32, 4, 5) X(64, 64, 4, 5)
#define TT_FUSED_FWD_SHAPES(X) TT_FUSED_SHAPES(X)

inline bool fused_shape_compiled(int K, int BN, int RP, int NL) {
#define TT_SHAPE_EQ(k_, bn_, rp_, nl_) if (K == k_ && BN == bn_ && RP == rp_ && NL == nl_) return true;
  TT_FUSED_SHAPES(TT_SHAPE_EQ)
#undef TT_SHAPE_EQ
  return false;
}

// Shape admission for the fused path (host).
inline bool fused_plan_shape(const DevCfg& c, FusedShape* s) {
  *s = FusedShape{};
  if (c.d < 3) return false;
  const int F = c.d - 2;
  const int64_t K = c.R[F], NC = c.cols[F], R2 = c.R[F + 1], NL = c.n[c.d - 1], RP = c.rows[F];
  if (R2 != K) return false;
  int BN = 0;
  if (K == 8 && NC % 32 == 0) BN = 32;
  if (K == 16 && NC % 64 == 0) BN = 64;
  if (K == 32 && NC % 128 == 0) BN = 128;
  if (K == 64 && NC % 128 == 0) BN = 128;
  if (K == 128 && NC % 64 == 0) BN = 64;  // 64-column blocks: two CTAs per SM at rank 128
  // column counts that are no multiple of 128 (NC = n_F R with n_F = 5 in the
  // paper's Table-4 products shape): one core-F column block of K columns each
  if (!BN && (K == 32 || K == 64) && NC % K == 0) BN = (int)K;
  if (!BN || !fused_shape_compiled((int)K, BN, (int)RP, (int)NL)) return false;
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
  s->OUT = (int)(RP * (BN / K) * NL);
  // forward column block: up to 128 (2 CTAs/SM without spills); at rank 128
  // the forward keeps 128-column blocks while the backward uses 64
  const int BNf = (K == 128 && NC % 128 == 0) ? 128 : (int)std::min<int64_t>(BN, 128);
  s->BNf = BNf;
  s->ncbf = (int)(NC / BNf);
  s->BNjf = (int)(BNf / K);
  const size_t SB = BN + 4, SG = K + 4, SBf = BNf + 4;
  const size_t ints = sizeof(int64_t) * FB_NB + sizeof(int) * (3 * FB_NB + 12) + 16;
  const size_t base_f = sizeof(float) * (K * SBf + 2 * FB_BM * K) + ints + sizeof(int) * (3 * FB_IDS + 8) + 16;
  const size_t half = 113 * 1024;  // keep two forward CTAs per SM
  const size_t per_id = sizeof(float) * K * NL;
  s->CHF = (int)std::min<size_t>(32, base_f < half ? (half - base_f) / per_id : 0);
  if (s->CHF < 1) s->CHF = (int)std::min<size_t>(8, ((size_t)FB_SMEM_MAX - base_f) / per_id);
  s->smem_fwd = base_f + s->CHF * per_id;
  s->smem_bwd = sizeof(float) * (K * SB + FB_BM * K + FB_BM * (BN + 4)) + ints + sizeof(int) * (FB_IDS + 8);
  (void)SG;
  if (s->smem_fwd > (size_t)FB_SMEM_MAX || s->smem_bwd > (size_t)FB_SMEM_MAX) return false;
  s->CHB = 0;
  return true;
}

}  // namespace tt
