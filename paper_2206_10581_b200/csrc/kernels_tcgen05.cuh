// kernels_tcgen05.cuh -- the optional tensor-core path (path "tc"): the
// level-F GEMMs of the fused kernels on the 5th-generation tensor cores
// (tcgen05.mma, accumulators in TMEM), FP32-accurate through the BF16x3
// scheme of tc_sm100.cuh.  Same work units (one CTA per (digit group g,
// column block cb)), same inputs and outputs as k_fused_fwd / k_fused_bwd
// (kernels_fused.cuh): P_F saved for the backward, dP_{F-1} partials per
// (node, column block), dG_F written once per slice block (no atomics).
//
// Rows are processed in tiles of 128 (= 128 / RP nodes of the group):
//   forward   C (128 x BN)  = A (128 x K) . S (K x BN)          M=128, N=BN
//   backward  dG_F^T (BN x K) += dC^T (BN x 128) . A (128 x K)  M=BN=128, N=K  (TMEM across the group)
//             dA (128 x K)     = dC (128 x BN) . S^T (BN x K)    M=128, N=K
// where dC = dP_F is formed on the CUDA cores (FFMA) from the upstream rows
// summed per distinct ID and the last core's slices.  Every operand tile is
// one core-matrix plane triple in shared memory (tc_sm100.cuh): A and S are
// written once and read as K-major or MN-major as each product needs; dC is
// written once and read as both dC (K-major) and dC^T (MN-major).
#pragma once
#include "kernels_fused.cuh"
#include "tc_sm100.cuh"

namespace tt {

constexpr int TC_BM = 128;

struct TcShape {
  int ok;
  int BNf, ncbf;  // forward column block
  int BNb, ncbb;  // backward column block (= 128)
  size_t smem_fwd, smem_bwd;
};

// metadata area shared by both kernels (node batch of FB_NB)
constexpr size_t TC_META = sizeof(int64_t) * FB_NB + sizeof(int) * (3 * FB_NB + 12) + 64;

template <int K, int BN>
constexpr size_t tc_fwd_smem() {
  return 3 * (size_t)K * BN * 2 + 3 * (size_t)TC_BM * K * 2 + TC_META;
}
template <int K, int BN>
constexpr size_t tc_bwd_smem() {
  return 3 * (size_t)K * BN * 2 + 3 * (size_t)TC_BM * K * 2 + 3 * (size_t)TC_BM * BN * 2 + TC_META;
}

// S block (K x BN) of slice g, column block cb -> planes [K rows][BN cols]
template <int K, int BN>
__device__ __forceinline__ void tc_stage_slice(const FusedArgs& a, int g, int cb, uint8_t* p0, uint8_t* p1,
                                               uint8_t* p2) {
  const float* src = a.params + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F] + cb * BN;
  for (int u = threadIdx.x; u < K * BN / 8; u += FB_THREADS) {
    const int k = u / (BN / 8), c0 = (u - k * (BN / 8)) * 8;
    const float4 x0 = __ldg(reinterpret_cast<const float4*>(src + (int64_t)k * a.NC + c0));
    const float4 x1 = __ldg(reinterpret_cast<const float4*>(src + (int64_t)k * a.NC + c0 + 4));
    const float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    tc::store_split8(p0, p1, p2, k, c0, BN, x);
  }
}

// A tile: rows m = j*RP + a of the batch-local nodes [tb, tb+nn) -> planes [128][K]
template <int K, int RP>
__device__ __forceinline__ void tc_stage_A(const FusedArgs& a, int tb, int nn, const int64_t* s_aoff, uint8_t* p0,
                                           uint8_t* p1, uint8_t* p2) {
  for (int u = threadIdx.x; u < TC_BM * K / 8; u += FB_THREADS) {
    const int m = u / (K / 8), k0 = (u - m * (K / 8)) * 8;
    const int j = m / RP;
    float x[8];
    if (j < nn) {
      const float* src = a.Abase + s_aoff[tb + j] + (m - j * RP) * K + k0;
      const float4 x0 = __ldg(reinterpret_cast<const float4*>(src));
      const float4 x1 = __ldg(reinterpret_cast<const float4*>(src + 4));
      x[0] = x0.x; x[1] = x0.y; x[2] = x0.z; x[3] = x0.w; x[4] = x1.x; x[5] = x1.y; x[6] = x1.z; x[7] = x1.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = 0.f;
    }
    tc::store_split8(p0, p1, p2, m, k0, K, x);
  }
}

// ---------------------------------------------------------------------------
// Forward: P_F tiles on the tensor pipe, saved to Psave.
template <int K, int BN, int RP>
__global__ void __launch_bounds__(FB_THREADS, 1) k_tc_fwd(FusedArgs a) {
  static_assert(BN % 16 == 0 && BN <= 256 && K % 16 == 0 && TC_BM % RP == 0, "tcgen05 forward shape");
  constexpr int NPT = TC_BM / RP;
  constexpr uint32_t TCOLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  extern __shared__ __align__(128) uint8_t tsm[];
  uint8_t* S0 = tsm;
  uint8_t* S1 = S0 + K * BN * 2;
  uint8_t* S2 = S1 + K * BN * 2;
  uint8_t* A0 = S2 + K * BN * 2;
  uint8_t* A1 = A0 + TC_BM * K * 2;
  uint8_t* A2 = A1 + TC_BM * K * 2;
  int64_t* s_aoff = reinterpret_cast<int64_t*>(A2 + TC_BM * K * 2);
  int* s_node = reinterpret_cast<int*>(s_aoff + FB_NB);
  int* s_cs0 = s_node + FB_NB;
  int* s_pref = s_cs0 + FB_NB;
  int* s_wsum = s_pref + FB_NB + 4;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;

  if (tt_failed(a.st)) return;
  const int g = blockIdx.x / a.ncb, cb = blockIdx.x - g * a.ncb;
  const int g0 = a.goffF[g], g1 = a.goffF[g + 1];
  if (g0 == g1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tc::tmem_alloc<TCOLS>(&tslot);
  if (threadIdx.x == 32) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  tc_stage_slice<K, BN>(a, g, cb, S0, S1, S2);
  uint32_t phase = 0;
  const uint32_t idesc = tc::idesc_bf16(TC_BM, BN, 0, 1);
  for (int nb0 = g0; nb0 < g1; nb0 += FB_NB) {
    const int nbn = min(FB_NB, g1 - nb0);
    prep_nodes(a, nb0, nbn, s_node, s_cs0, s_pref, s_aoff, s_wsum);
    for (int tb = 0; tb < nbn; tb += NPT) {
      const int nn = min(NPT, nbn - tb);
      tc_stage_A<K, RP>(a, tb, nn, s_aoff, A0, A1, A2);
      tc::fence_async_smem();
      tc::before_sync();
      __syncthreads();
      tc::after_sync();
      const uint32_t tm = tslot;
      if (threadIdx.x == 0) {
        const tc::Operand oa = tc::kmajor(tc::smem_u32(A0), tc::smem_u32(A1), tc::smem_u32(A2), K);
        const tc::Operand ob = tc::mnmajor(tc::smem_u32(S0), tc::smem_u32(S1), tc::smem_u32(S2), BN);
        tc::mma_x3(tm, oa, ob, K, idesc, false);
        tc::commit(&bar);
      }
      __syncwarp();
      tc::mbar_wait(&bar, phase);
      phase ^= 1;
      tc::after_sync();
      // epilogue: warp w reads TMEM lanes 32*(w%4).. (tile rows), columns half w/4
      const int m = 32 * (warp & 3) + lane;
      const int j = m / RP;
      const int c_lo = (warp >> 2) * (BN / 2);
      float* dst = j < nn ? a.Psave + ((int64_t)s_node[tb + j] * RP + (m - j * RP)) * a.NC + cb * BN : nullptr;
#pragma unroll 1
      for (int c = c_lo; c < c_lo + BN / 2; c += 16) {
        float v[16];
        tc::tmem_ld16(tm + ((uint32_t)(32 * (warp & 3)) << 16) + c, v);
        if (dst) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<float4*>(dst + c + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
      }
      tc::before_sync();
      __syncthreads();  // TMEM drained and A planes free before the next tile
    }
  }
  if (warp == 0) tc::tmem_free<TCOLS>(tslot);
}

// ---------------------------------------------------------------------------
// Backward: dC on the CUDA cores, dG_F^T and dA on the tensor pipe.
template <int K, int BN, int RP, int NL>
__global__ void __launch_bounds__(FB_THREADS, 1) k_tc_bwd(FusedArgs a) {
  static_assert(BN == 128 && K % 16 == 0 && K <= 128 && TC_BM % RP == 0 && RP % 4 == 0, "tcgen05 backward shape");
  constexpr int NPT = TC_BM / RP;
  constexpr uint32_t TCOLS = 2 * K <= 64 ? 64 : 2 * K <= 128 ? 128 : 256;
  extern __shared__ __align__(128) uint8_t tsm[];
  uint8_t* S0 = tsm;
  uint8_t* S1 = S0 + K * BN * 2;
  uint8_t* S2 = S1 + K * BN * 2;
  uint8_t* A0 = S2 + K * BN * 2;
  uint8_t* A1 = A0 + TC_BM * K * 2;
  uint8_t* A2 = A1 + TC_BM * K * 2;
  uint8_t* D0 = A2 + TC_BM * K * 2;
  uint8_t* D1 = D0 + TC_BM * BN * 2;
  uint8_t* D2 = D1 + TC_BM * BN * 2;
  int64_t* s_aoff = reinterpret_cast<int64_t*>(D2 + TC_BM * BN * 2);
  int* s_node = reinterpret_cast<int*>(s_aoff + FB_NB);
  int* s_cs0 = s_node + FB_NB;
  int* s_pref = s_cs0 + FB_NB;
  int* s_wsum = s_pref + FB_NB + 4;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;

  if (tt_failed(a.st)) return;
  const int g = blockIdx.x / a.ncb, cb = blockIdx.x - g * a.ncb;
  const int g0 = a.goffF[g], g1 = a.goffF[g + 1];
  if (g0 == g1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tc::tmem_alloc<TCOLS>(&tslot);
  if (threadIdx.x == 32) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  tc_stage_slice<K, BN>(a, g, cb, S0, S1, S2);
  const int nF = a.nF;
  const int64_t npad = a.c.npad;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];
  const uint32_t id_g = tc::idesc_bf16(BN, K, 1, 1);      // dG^T = dC^T . A
  const uint32_t id_a = tc::idesc_bf16(TC_BM, K, 0, 0);   // dA = dC . S^T
  uint32_t phase = 0;
  int tiles = 0;
  for (int nb0 = g0; nb0 < g1; nb0 += FB_NB) {
    const int nbn = min(FB_NB, g1 - nb0);
    prep_nodes(a, nb0, nbn, s_node, s_cs0, s_pref, s_aoff, s_wsum);
    for (int tb = 0; tb < nbn; tb += NPT, ++tiles) {
      const int nn = min(NPT, nbn - tb);
      tc_stage_A<K, RP>(a, tb, nn, s_aoff, A0, A1, A2);
      // dC units: 4 rows of one node x 8 columns (one core-F column block jf)
#pragma unroll 1
      for (int unit = threadIdx.x; unit < (TC_BM / 4) * (BN / 8); unit += FB_THREADS) {
        const int rg = unit / (BN / 8), c8 = unit - rg * (BN / 8);
        const int m0 = rg * 4, j = m0 / RP, a0 = m0 - j * RP;
        const int col0 = cb * BN + c8 * 8, jf = col0 / K, r0 = col0 - jf * K;
        float acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int t = 0; t < 8; ++t) acc[i][t] = 0.f;
        if (j < nn) {
          const int fA = s_pref[tb + j], fB = s_pref[tb + j + 1], cs0 = s_cs0[tb + j];
          for (int f = fA; f < fB; ++f) {
            const int u = cs0 + (f - fA);
            const float* Gp = Gl + (int64_t)__ldg(a.digitL + u) * sliceL + r0 * NL;
            float gv[8][NL];
#pragma unroll
            for (int t = 0; t < 8; ++t)
#pragma unroll
              for (int l4 = 0; l4 < NL; l4 += 4) {
                const float4 x = __ldg(reinterpret_cast<const float4*>(Gp + t * NL + l4));
                gv[t][l4] = x.x; gv[t][l4 + 1] = x.y; gv[t][l4 + 2] = x.z; gv[t][l4 + 3] = x.w;
              }
            const float* Yp = a.dY + (int64_t)u * npad + ((int64_t)a0 * nF + jf) * NL;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float yv[NL];
#pragma unroll
              for (int l4 = 0; l4 < NL; l4 += 4) {
                const float4 x = __ldg(reinterpret_cast<const float4*>(Yp + (int64_t)i * nF * NL + l4));
                yv[l4] = x.x; yv[l4 + 1] = x.y; yv[l4 + 2] = x.z; yv[l4 + 3] = x.w;
              }
#pragma unroll
              for (int t = 0; t < 8; ++t) {
                float s = acc[i][t];
#pragma unroll
                for (int jl = 0; jl < NL; ++jl) s = fmaf(yv[jl], gv[t][jl], s);
                acc[i][t] = s;
              }
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) tc::store_split8(D0, D1, D2, m0 + i, c8 * 8, BN, acc[i]);
      }
      tc::fence_async_smem();
      tc::before_sync();
      __syncthreads();
      tc::after_sync();
      const uint32_t tm = tslot;
      if (threadIdx.x == 0) {
        const uint32_t d0 = tc::smem_u32(D0), d1 = tc::smem_u32(D1), d2 = tc::smem_u32(D2);
        const tc::Operand dcT = tc::mnmajor(d0, d1, d2, BN);  // A operand (m = col, k = row)
        const tc::Operand aB = tc::mnmajor(tc::smem_u32(A0), tc::smem_u32(A1), tc::smem_u32(A2), K);
        tc::mma_x3(tm, dcT, aB, TC_BM, id_g, tiles > 0);
        const tc::Operand dcK = tc::kmajor(d0, d1, d2, BN);   // A operand (m = row, k = col)
        const tc::Operand sT = tc::kmajor(tc::smem_u32(S0), tc::smem_u32(S1), tc::smem_u32(S2), BN);
        tc::mma_x3(tm + K, dcK, sT, BN, id_a, false);
        tc::commit(&bar);
      }
      __syncwarp();
      tc::mbar_wait(&bar, phase);
      phase ^= 1;
      tc::after_sync();
      // dA epilogue -> dPc[(node, cb)][a][r]
      {
        const int m = 32 * (warp & 3) + lane;
        const int j = m / RP;
        const int c_lo = (warp >> 2) * (K / 2);
        float* dst = j < nn ? a.dPc + ((int64_t)s_node[tb + j] * a.ncb + cb) * RP * K + (m - j * RP) * K : nullptr;
#pragma unroll 1
        for (int c = c_lo; c < c_lo + K / 2; c += 16) {
          float v[16];
          tc::tmem_ld16(tm + ((uint32_t)(32 * (warp & 3)) << 16) + K + c, v);
          if (dst) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              *reinterpret_cast<float4*>(dst + c + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
        }
      }
      tc::before_sync();
      __syncthreads();
    }
  }
  // dG_F block: TMEM lane = column of the block, TMEM column = rank index r
  tc::after_sync();
  {
    const uint32_t tm = tslot;
    const int col = 32 * (warp & 3) + lane;
    const int r_lo = (warp >> 2) * (K / 2);
    float* gdst = a.grads + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F] + cb * BN + col;
#pragma unroll 1
    for (int r = r_lo; r < r_lo + K / 2; r += 16) {
      float v[16];
      tc::tmem_ld16(tm + ((uint32_t)(32 * (warp & 3)) << 16) + r, v);
#pragma unroll
      for (int i = 0; i < 16; ++i) gdst[(int64_t)(r + i) * a.NC] = v[i];
    }
  }
  tc::before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<TCOLS>(tslot);
}

// (K, BNf, RP, NL) instantiations of the tensor-core path
#define TT_TC_SHAPES(X) X(64, 128, 4, 4) X(32, 128, 4, 8) X(32, 128, 16, 4) X(64, 128, 4, 8)

inline bool tc_plan_shape(const FusedShape& f, TcShape* t) {
  *t = TcShape{};
  bool ok = false;
#define TT_TC_EQ(k_, bn_, rp_, nl_) \
  if (f.K == k_ && f.RP == rp_ && f.NL == nl_ && f.NC % bn_ == 0 && f.NC % 128 == 0) ok = true;
  TT_TC_SHAPES(TT_TC_EQ)
#undef TT_TC_EQ
  if (!ok) return false;
  t->BNf = 128;
  t->ncbf = f.NC / 128;
  t->BNb = 128;
  t->ncbb = f.NC / 128;
  t->smem_fwd = 3 * (size_t)f.K * 128 * 2 + 3 * (size_t)TC_BM * f.K * 2 + TC_META;
  // at most two forward CTAs per SM (TMEM: 2 x 128 columns)
  t->smem_fwd = std::max<size_t>(t->smem_fwd, 80 * 1024);
  t->smem_bwd = 3 * (size_t)f.K * 128 * 2 + 3 * (size_t)TC_BM * f.K * 2 + 3 * (size_t)TC_BM * 128 * 2 + TC_META;
  t->ok = t->smem_bwd <= (size_t)FB_SMEM_MAX;
  return t->ok;
}

}  // namespace tt
