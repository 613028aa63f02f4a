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

// Plane writers map 8 consecutive threads to the 8 rows of one core matrix
// (unit u: row-in-core = u % 8), so each 16-byte store phase covers 128
// contiguous bytes -- no bank conflicts.

// S block (K x BN) of slice g, column block cb -> planes [K rows][BN cols]
template <int K, int BN, int T>
__device__ __forceinline__ void tc_stage_slice(const FusedArgs& a, int g, int cb, uint8_t* p0, uint8_t* p1,
                                               uint8_t* p2) {
  const float* src = a.params + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F] + cb * BN;
  for (int u = threadIdx.x; u < K * BN / 8; u += T) {
    const int cc = (u >> 3) % (BN / 8), k = ((u >> 3) / (BN / 8)) * 8 + (u & 7), c0 = cc * 8;
    const float4 x0 = __ldg(reinterpret_cast<const float4*>(src + (int64_t)k * a.NC + c0));
    const float4 x1 = __ldg(reinterpret_cast<const float4*>(src + (int64_t)k * a.NC + c0 + 4));
    const float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    tc::store_split8(p0, p1, p2, k, c0, BN, x);
  }
}

// A tile: rows m = j*RP + a of the batch-local nodes [tb, tb+nn) -> planes
// [128][K].  Loading (to registers) and storing (split into the planes) are
// separate so the next tile's global loads are in flight under the current
// tile's MMA and epilogue.
template <int K, int T>
struct ATileRegs {
  static constexpr int N = TC_BM * K / 8 / T;  // units per thread
  static_assert(N >= 1, "A tile smaller than the block");
  float4 v[N][2];
};

template <int K, int RP, int T>
__device__ __forceinline__ void tc_load_A(const FusedArgs& a, int tb, int nn, const int64_t* s_aoff,
                                          ATileRegs<K, T>& r) {
#pragma unroll
  for (int i = 0; i < ATileRegs<K, T>::N; ++i) {
    const int u = threadIdx.x + i * T;
    const int kc = (u >> 3) % (K / 8), m = ((u >> 3) / (K / 8)) * 8 + (u & 7);
    const int j = m / RP;
    if (j < nn) {
      const float* src = a.Abase + s_aoff[tb + j] + (m - j * RP) * K + kc * 8;
      r.v[i][0] = __ldg(reinterpret_cast<const float4*>(src));
      r.v[i][1] = __ldg(reinterpret_cast<const float4*>(src + 4));
    } else {
      r.v[i][0] = r.v[i][1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

template <int K, int T>
__device__ __forceinline__ void tc_store_A(const ATileRegs<K, T>& r, uint8_t* p0, uint8_t* p1, uint8_t* p2) {
#pragma unroll
  for (int i = 0; i < ATileRegs<K, T>::N; ++i) {
    const int u = threadIdx.x + i * T;
    const int kc = (u >> 3) % (K / 8), m = ((u >> 3) / (K / 8)) * 8 + (u & 7);
    const float x[8] = {r.v[i][0].x, r.v[i][0].y, r.v[i][0].z, r.v[i][0].w,
                        r.v[i][1].x, r.v[i][1].y, r.v[i][1].z, r.v[i][1].w};
    tc::store_split8(p0, p1, p2, m, kc * 8, K, x);
  }
}

// Node metadata of nodes [nb0, nb0 + nbn) of the group (kernels_fused.cuh
// prep_nodes for a block of T threads).  Ends with a barrier.
template <int T>
__device__ __forceinline__ void tc_prep_nodes(const FusedArgs& a, int nb0, int nbn, int* s_node, int* s_cs0,
                                              int* s_pref, int64_t* s_aoff, int* s_wsum) {
  static_assert(T >= FB_NB && T <= 1024, "one thread per staged node");
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
    int w = t < T / 32 ? s_wsum[t] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if ((int)lane_id() >= o) w += y;
    }
    if (t < T / 32) s_wsum[t] = w;
  }
  __syncthreads();
  const int excl = x - cnt + ((t >> 5) ? s_wsum[(t >> 5) - 1] : 0);
  if (t < nbn) s_pref[t] = excl;
  if (t == nbn - 1) s_pref[nbn] = excl + cnt;
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Forward: P_F tiles on the tensor pipe, saved to Psave.  512 threads, one
// CTA per SM.  The epilogue is store-bound (P_F is 666 MB at papers): warp w
// drains TMEM lanes 32(w%4).. x columns 32(w/4).. of the accumulator, turns
// its 32 x 32 chunk around in shared memory and writes 4 full 128-byte row
// segments per store instruction (a TMEM lane per thread would write 32 rows
// x 16 bytes per instruction, 8x the L2 requests).
constexpr int TCF_THREADS = 512;
constexpr int TCF_ES = 36;  // epilogue staging row stride (floats): conflict-free 16-byte stores and loads
template <int K, int BN>
constexpr size_t tc_fwd_smem_bytes() {
  return 3 * (size_t)K * BN * 2 + 3 * (size_t)TC_BM * K * 2 + (size_t)(TCF_THREADS / 32) * 32 * TCF_ES * 4 + TC_META;
}

template <int K, int BN, int RP>
__global__ void __launch_bounds__(TCF_THREADS, 1) k_tc_fwd(FusedArgs a) {
  static_assert(BN == 128 && K % 16 == 0 && TC_BM % RP == 0, "tcgen05 forward shape");
  constexpr int T = TCF_THREADS;
  constexpr int NPT = TC_BM / RP;
  constexpr uint32_t TCOLS = BN;
  extern __shared__ __align__(128) uint8_t tsm[];
  uint8_t* S0 = tsm;
  uint8_t* S1 = S0 + K * BN * 2;
  uint8_t* S2 = S1 + K * BN * 2;
  uint8_t* A0 = S2 + K * BN * 2;
  uint8_t* A1 = A0 + TC_BM * K * 2;
  uint8_t* A2 = A1 + TC_BM * K * 2;
  float* Es = reinterpret_cast<float*>(A2 + TC_BM * K * 2);  // [16 warps][32][TCF_ES]
  int64_t* s_aoff = reinterpret_cast<int64_t*>(Es + (T / 32) * 32 * TCF_ES);
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
  tc_stage_slice<K, BN, T>(a, g, cb, S0, S1, S2);
  uint32_t phase = 0;
  const uint32_t idesc = tc::idesc_bf16(TC_BM, BN, 0, 1);
  ATileRegs<K, T> ar;
  const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
  const int ccol = (warp >> 2) * 32;          // this warp's 32 accumulator columns
  float* Ew = Es + warp * 32 * TCF_ES;
  for (int nb0 = g0; nb0 < g1; nb0 += FB_NB) {
    const int nbn = min(FB_NB, g1 - nb0);
    tc_prep_nodes<T>(a, nb0, nbn, s_node, s_cs0, s_pref, s_aoff, s_wsum);
    tc_load_A<K, RP, T>(a, 0, min(NPT, nbn), s_aoff, ar);
    for (int tb = 0; tb < nbn; tb += NPT) {
      const int nn = min(NPT, nbn - tb);
      if (!(a.mode & 8)) tc_store_A<K, T>(ar, A0, A1, A2);
      tc::fence_async_smem();
      tc::before_sync();
      __syncthreads();  // A planes written; the previous tile's TMEM reads done
      tc::after_sync();
      const uint32_t tm = tslot;
      if (threadIdx.x == 0) {
        const tc::Operand oa = tc::kmajor(tc::smem_u32(A0), tc::smem_u32(A1), tc::smem_u32(A2), K);
        const tc::Operand ob = tc::mnmajor(tc::smem_u32(S0), tc::smem_u32(S1), tc::smem_u32(S2), BN);
        if (!(a.mode & 2)) tc::mma_x3<K / 16>(tm, oa, ob, idesc, false);
        tc::commit(&bar);
      }
      __syncwarp();
      if (tb + NPT < nbn && !(a.mode & 8)) tc_load_A<K, RP, T>(a, tb + NPT, min(NPT, nbn - tb - NPT), s_aoff, ar);
      tc::mbar_wait(&bar, phase);
      phase ^= 1;
      tc::after_sync();
      // epilogue: TMEM (row = lane) -> staging -> 4 rows x 128 B per store
      {
        float v[16];
        tc::tmem_ld16(tm + lane_base + ccol, v);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<float4*>(Ew + lane * TCF_ES + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        tc::tmem_ld16(tm + lane_base + ccol + 16, v);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<float4*>(Ew + lane * TCF_ES + 16 + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        __syncwarp();
        const int c4 = (lane & 7) * 4;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = (lane >> 3) + 4 * i;     // row within the warp's 32
          const int m = 32 * (warp & 3) + r;     // tile row
          const int j = m / RP;
          const float4 x = *reinterpret_cast<const float4*>(Ew + r * TCF_ES + c4);
          if (j < nn && !(a.mode & 4))
            *reinterpret_cast<float4*>(a.Psave + ((int64_t)s_node[tb + j] * RP + (m - j * RP)) * a.NC + cb * BN +
                                       ccol + c4) = x;
        }
        __syncwarp();
      }
      tc::before_sync();
    }
    tc::before_sync();
    __syncthreads();
  }
  if (warp == 0) tc::tmem_free<TCOLS>(tslot);
}

// ---------------------------------------------------------------------------
// Backward: dC on the CUDA cores, dG_F^T and dA on the tensor pipe.  512
// threads (16 warps) per CTA: the CUDA-core half of a tile is a chain of
// dependent L2 loads (ID digit -> last-core slice), so latency is hidden by
// warps, and one CTA holds the whole 192 KB operand set per SM.
constexpr int TCB_THREADS = 512;

template <int K, int BN, int RP, int NL>
__global__ void __launch_bounds__(TCB_THREADS, 1) k_tc_bwd(FusedArgs a) {
  TT_PDL_ENTRY();
  static_assert(BN == 128 && K % 16 == 0 && K <= 128 && TC_BM % RP == 0 && RP % 4 == 0, "tcgen05 backward shape");
  constexpr int T = TCB_THREADS;
  constexpr int NPT = TC_BM / RP;
  // TMEM: dG_F^T [0, K) + dA [K, 2K)
  constexpr uint32_t TCOLS = 2 * K <= 64 ? 64 : 2 * K <= 128 ? 128 : 256;
  constexpr int EC = K / 4;  // epilogue columns per warp (16 warps = 4 lane quadrants x 4 column slices)
  static_assert(EC == 8 || EC == 16, "epilogue column slice");
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
  const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;  // TMEM lane quadrant of this warp
  const int eslice = (warp >> 2) * EC;
  if (warp == 0) tc::tmem_alloc<TCOLS>(&tslot);
  if (threadIdx.x == 32) {
    tc::mbar_init(&bar, 2);  // two issuers commit per tile (dG_F^T and dA)
    tc::fence_mbar_init();
  }
  tc_stage_slice<K, BN, T>(a, g, cb, S0, S1, S2);
  const int nF = a.nF;
  const int64_t npad = a.c.npad;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];
  const uint32_t id_g = tc::idesc_bf16(BN, K, 1, 1);      // dG^T = dC^T . A
  const uint32_t id_a = tc::idesc_bf16(TC_BM, K, 0, 0);   // dA = dC . S^T
  uint32_t phase = 0;
  int tiles = 0;
  ATileRegs<K, T> ar;
  // dC unit of this thread: 4 rows of one node x 8 columns (one core-F
  // column block jf).  unit bits: [0,2) column chunk low, [2] row group low,
  // [3,5) column chunk high, [5,9) row group high; with the rows of a unit
  // stored in rotated order (rot = unit % 4) the 8 threads of a store phase
  // write 8 distinct rows of one core-matrix column: conflict-free.
  static_assert((TC_BM / 4) * (BN / 8) == T, "one dC unit per thread");
  const int unit = threadIdx.x;
  const int c8 = (unit & 3) + 4 * ((unit >> 3) & 3);
  const int rg = ((unit >> 2) & 1) + 2 * (unit >> 5);
  const int rot = unit & 3;
  const int m0 = rg * 4, uj = m0 / RP, a0 = m0 - uj * RP;
  const int col0 = cb * BN + c8 * 8, jf = col0 / K, r0 = col0 - jf * K;
  // dC(t) of this thread's unit into registers (loads + FFMA): issued for
  // tile t+1 while the tensor pipe works on tile t
  auto compute_dC = [&](int tb, int nn, float (&acc)[4][8]) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[i][t] = 0.f;
    if (uj >= nn || (a.mode & 16)) return;
    const int fA = s_pref[tb + uj], fB = (a.mode & 64) ? min(s_pref[tb + uj + 1], s_pref[tb + uj] + 1) : s_pref[tb + uj + 1], cs0 = s_cs0[tb + uj];
    for (int f = fA; f < fB; ++f) {
      const int u = cs0 + (f - fA);
      const float* Gp = Gl + (int64_t)__ldg(a.digitL + u) * sliceL + r0 * NL;
      const float* Yp = a.dY + (int64_t)u * npad + ((int64_t)a0 * nF + jf) * NL;
      float yv[4][NL];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int ii = (i + rot) & 3;
#pragma unroll
        for (int l4 = 0; l4 < NL; l4 += 4) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(Yp + (int64_t)ii * nF * NL + l4));
          yv[i][l4] = x.x; yv[i][l4 + 1] = x.y; yv[i][l4 + 2] = x.z; yv[i][l4 + 3] = x.w;
        }
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        float gv[NL];
#pragma unroll
        for (int l4 = 0; l4 < NL; l4 += 4) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(Gp + t * NL + l4));
          gv[l4] = x.x; gv[l4 + 1] = x.y; gv[l4 + 2] = x.z; gv[l4 + 3] = x.w;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float s = acc[i][t];
#pragma unroll
          for (int jl = 0; jl < NL; ++jl) s = fmaf(yv[i][jl], gv[jl], s);
          acc[i][t] = s;
        }
      }
    }
  };
  float acc[4][8];
  const int em = 32 * (warp & 3) + lane;  // epilogue row (TMEM lane)
  const int emj = em / RP, ema = em - emj * RP;
  // dA rows of a finished tile: accumulator `buf` -> dPc[(node, cb)][a][r]
  auto epilogue = [&](uint32_t tm, int buf, float* dst) {
    float v[EC];
    if constexpr (EC == 16) tc::tmem_ld16(tm + lane_base + K + buf * K + eslice, v);
    else tc::tmem_ld8(tm + lane_base + K + buf * K + eslice, v);
    if (dst) {
#pragma unroll
      for (int q = 0; q < EC / 4; ++q)
        *reinterpret_cast<float4*>(dst + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  };
  for (int nb0 = g0; nb0 < g1; nb0 += FB_NB) {
    const int nbn = min(FB_NB, g1 - nb0);
    tc_prep_nodes<T>(a, nb0, nbn, s_node, s_cs0, s_pref, s_aoff, s_wsum);
    tc_load_A<K, RP, T>(a, 0, min(NPT, nbn), s_aoff, ar);
    compute_dC(0, min(NPT, nbn), acc);
    for (int tb = 0; tb < nbn; tb += NPT, ++tiles) {
      const int nn = min(NPT, nbn - tb);
      if (!(a.mode & 8)) tc_store_A<K, T>(ar, A0, A1, A2);
      if (!(a.mode & 32)) {
#pragma unroll
        for (int i = 0; i < 4; ++i) tc::store_split8(D0, D1, D2, m0 + ((i + rot) & 3), c8 * 8, BN, acc[i]);
      }
      tc::fence_async_smem();
      tc::before_sync();
      __syncthreads();
      tc::after_sync();
      const uint32_t tm = tslot;
      // the next tile's A loads go out first (they land while the issuers
      // below block on the tensor pipe's queue)
      const bool more = tb + NPT < nbn;
      if (more && !(a.mode & 8)) tc_load_A<K, RP, T>(a, tb + NPT, min(NPT, nbn - tb - NPT), s_aoff, ar);
      // two issuers in different warps (the products write separate TMEM
      // accumulators): issuing blocks while the tensor pipe's queue is full,
      // so each product's 48 MMAs hold up only its own warp
      if (threadIdx.x == 0) {  // dG_F^T += dC^T . A   (accumulated over the group)
        const tc::Operand dcT = tc::mnmajor(tc::smem_u32(D0), tc::smem_u32(D1), tc::smem_u32(D2), BN);
        const tc::Operand aB = tc::mnmajor(tc::smem_u32(A0), tc::smem_u32(A1), tc::smem_u32(A2), K);
        if (!(a.mode & 2)) tc::mma_x3<TC_BM / 16>(tm, dcT, aB, id_g, tiles > 0);
        tc::commit(&bar);
      } else if (threadIdx.x == 32) {  // dA = dC . S^T
        const tc::Operand dcK = tc::kmajor(tc::smem_u32(D0), tc::smem_u32(D1), tc::smem_u32(D2), BN);
        const tc::Operand sT = tc::kmajor(tc::smem_u32(S0), tc::smem_u32(S1), tc::smem_u32(S2), BN);
        if (!(a.mode & 2)) tc::mma_x3<BN / 16>(tm + K, dcK, sT, id_a, false);
        tc::commit(&bar);
      }
      __syncwarp();
      float* dst = (emj < nn && !(a.mode & 4))
                       ? a.dPc + ((int64_t)s_node[tb + emj] * a.ncb + cb) * RP * K + ema * K + eslice
                       : nullptr;
      // under this tile's MMAs: the next tile's dC unit (no TMEM access -- a
      // tcgen05.ld issued now would queue behind the MMAs)
      if (more) compute_dC(tb + NPT, min(NPT, nbn - tb - NPT), acc);
      tc::mbar_wait(&bar, phase);  // planes free for the next tile
      phase ^= 1;
      tc::after_sync();
      epilogue(tm, 0, dst);
      tc::before_sync();
    }
    tc::before_sync();
    __syncthreads();
  }
  // dG_F block: TMEM lane = column of the block, TMEM column = rank index r
  tc::after_sync();
  {
    const uint32_t tm = tslot;
    const int col = 32 * (warp & 3) + lane;
    float* gdst = a.grads + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F] + cb * BN + col;
    float v[EC];
    if constexpr (EC == 16) tc::tmem_ld16(tm + lane_base + eslice, v);
    else tc::tmem_ld8(tm + lane_base + eslice, v);
#pragma unroll
    for (int i = 0; i < EC; ++i) gdst[(int64_t)(eslice + i) * a.NC] = v[i];
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
  t->smem_fwd = 3 * (size_t)f.K * 128 * 2 + 3 * (size_t)TC_BM * f.K * 2 +
                (size_t)(TCF_THREADS / 32) * 32 * TCF_ES * 4 + TC_META;
  t->smem_bwd = 3 * (size_t)f.K * 128 * 2 + 3 * (size_t)TC_BM * f.K * 2 + 3 * (size_t)TC_BM * 128 * 2 + TC_META;
  t->ok = t->smem_bwd <= (size_t)FB_SMEM_MAX;
  return t->ok;
}

}  // namespace tt
