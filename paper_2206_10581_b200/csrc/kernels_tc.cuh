// kernels_tc.cuh -- the optional tensor-core path (path "tf32x3").
//
// The level-F GEMMs of the fused kernels on warp-level mma.sync m16n8k8 TF32
// with the 3xTF32 split: x = hi + lo with hi = tf32(x), lo = tf32(x - hi),
// a.b ~= hi_a.hi_b + hi_a.lo_b + lo_a.hi_b (the dropped lo.lo term is ~2^-22
// relative), accumulated in fp32 -- fp32-level accuracy on the tensor pipe.
// Measured on this B200: mma.sync TF32 275 TFLOP/s vs 72.5 FFMA, so 3 passes
// still beat FFMA and, above all, replace 32 FFMA issue slots by one MMA.
// The slice block is split once per unit into hi/lo planes in shared memory;
// A fragments are split on the fly.  Same data flow, epilogue semantics and
// outputs as k_fused_fwd (kernels_fused.cuh); only the contraction differs.
#pragma once
#include "kernels_fused.cuh"

namespace tt {

__device__ __forceinline__ uint32_t f2tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void split3(float x, uint32_t& hi, uint32_t& lo) {
  hi = f2tf32(x);
  lo = f2tf32(x - __uint_as_float(hi));
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// A tile (BM x K) by cp.async into rows of stride SA (padded for conflict-free
// fragment loads); rows past the tile's nodes are zero-filled.
template <int K, int RP, int SA>
__device__ __forceinline__ void load_A_tile_pad(const FusedArgs& a, int tb, int nn, const int64_t* s_aoff, float* As) {
  for (int i = threadIdx.x; i < FB_BM * K / 4; i += FB_THREADS) {
    const int m = i / (K / 4), q = i - m * (K / 4);
    const int j = m / RP;
    float* dst = As + m * SA + q * 4;
    if (j < nn) cp_async16(dst, a.Abase + s_aoff[tb + j] + (m - j * RP) * K + q * 4);
    else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Forward on the tensor pipe.  8 warps = 4 (rows) x 2 (column halves); a warp
// owns 16 rows x K columns = one core-F column block jf, i.e. every rank index
// r of its rows, so the last-level contraction over r stays inside the warp
// (16 r per lane, then a 4-lane butterfly).
template <int K, int BN, int RP, int NL>
__global__ void __launch_bounds__(FB_THREADS, 2) k_fused_fwd_tc(FusedArgs a) {
  static_assert(BN == 2 * K && K % 8 == 0 && RP == 4 && NL == 4, "tensor-core forward: papers-type shape only");
  constexpr int BM = FB_BM, SB2 = BN + 4, SA = K + 4, NPT = BM / RP, BNJ = BN / K;
  constexpr int NT = K / 8;  // n8 tiles per warp (its K columns)
  extern __shared__ __align__(16) float smem[];
  float2* Bhl = reinterpret_cast<float2*>(smem);   // [K][SB2] (hi, lo) pairs: one LDS.64 per element
  float* As0 = smem + 2 * K * SB2;                 // [2][BM][SA]
  int64_t* s_aoff = reinterpret_cast<int64_t*>(As0 + 2 * BM * SA);
  int* s_node = reinterpret_cast<int*>(s_aoff + FB_NB);
  int* s_cs0 = s_node + FB_NB;
  int* s_pref = s_cs0 + FB_NB;
  int* s_wsum = s_pref + FB_NB + 4;

  if (tt_failed(a.st)) return;
  const int g = blockIdx.x / a.ncb, cb = blockIdx.x - g * a.ncb;
  const int g0 = a.goffF[g], g1 = a.goffF[g + 1];
  if (g0 == g1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp & 3, wn = warp >> 2;
  const int gq = lane >> 2, tq = lane & 3;
  const int rm = wm * 16, cn0 = wn * K;
  const int64_t emb = a.c.emb_dim, npad = a.c.npad;
  const int nF = a.nF;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];

  // raw slice block -> (A staging area) -> split once into interleaved hi/lo pairs
  load_slice_block<K, BN, BN>(a, g, cb, As0);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int i = threadIdx.x; i < K * BN; i += FB_THREADS) {
    const int k = i / BN, n = i - k * BN;
    uint32_t hi, lo;
    split3(As0[i], hi, lo);
    Bhl[k * SB2 + n] = make_float2(__uint_as_float(hi), __uint_as_float(lo));
  }
  __syncthreads();

  for (int nb0 = g0; nb0 < g1; nb0 += FB_NB) {
    const int nbn = min(FB_NB, g1 - nb0);
    prep_nodes(a, nb0, nbn, s_node, s_cs0, s_pref, s_aoff, s_wsum);
    load_A_tile_pad<K, RP, SA>(a, 0, min(NPT, nbn), s_aoff, As0);
    cp_async_commit();
    int buf = 0;
    for (int tb = 0; tb < nbn; tb += NPT, buf ^= 1) {
      const int nn = min(NPT, nbn - tb);
      cp_async_wait<0>();
      __syncthreads();
      if (tb + NPT < nbn) {
        load_A_tile_pad<K, RP, SA>(a, tb + NPT, min(NPT, nbn - tb - NPT), s_aoff, As0 + (buf ^ 1) * BM * SA);
        cp_async_commit();
      }
      const float* As = As0 + buf * BM * SA;
      float acc[NT][4];
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[j][e] = 0.f;
#pragma unroll 2
      for (int kk = 0; kk < K; kk += 8) {
        uint32_t ah[4], al[4];
        split3(As[(rm + gq) * SA + kk + tq], ah[0], al[0]);
        split3(As[(rm + gq + 8) * SA + kk + tq], ah[1], al[1]);
        split3(As[(rm + gq) * SA + kk + tq + 4], ah[2], al[2]);
        split3(As[(rm + gq + 8) * SA + kk + tq + 4], ah[3], al[3]);
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int n = cn0 + j * 8 + gq;
          const float2 p0 = Bhl[(kk + tq) * SB2 + n], p1 = Bhl[(kk + tq + 4) * SB2 + n];
          const uint32_t bh0 = __float_as_uint(p0.x), bh1 = __float_as_uint(p1.x);
          const uint32_t bl0 = __float_as_uint(p0.y), bl1 = __float_as_uint(p1.y);
          mma_tf32(acc[j], al, bh0, bh1);
          mma_tf32(acc[j], ah, bl0, bl1);
          mma_tf32(acc[j], ah, bh0, bh1);
        }
      }
      // rows of this lane: R0 = rm + gq (acc[..][0..1]), R1 = R0 + 8 (acc[..][2..3])
      const int R0 = rm + gq;
      if (a.Psave) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int m = R0 + 8 * h, j = m / RP;
          if (j < nn) {
            float* prow = a.Psave + ((int64_t)s_node[tb + j] * RP + (m - j * RP)) * a.NC + cb * BN + cn0 + 2 * tq;
#pragma unroll
            for (int jt = 0; jt < NT; ++jt)
              *reinterpret_cast<float2*>(prow + jt * 8) = make_float2(acc[jt][2 * h], acc[jt][2 * h + 1]);
          }
        }
      }
      if (!a.out) continue;
      // last level: per row half h, per distinct ID of its node
      const int jf = cb * BNJ + wn;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = R0 + 8 * h, j = m / RP, ar = m - j * RP;
        const bool live = j < nn;
        const int fA = live ? s_pref[tb + j] : 0, cnt = live ? s_pref[tb + j + 1] - fA : 0;
        const int cs0 = live ? s_cs0[tb + j] : 0;
        int maxc = cnt;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) maxc = max(maxc, __shfl_xor_sync(0xffffffffu, maxc, o));
        for (int f = 0; f < maxc; ++f) {
          const bool act = f < cnt;
          const int u = act ? cs0 + f : cs0;
          float v[NL];
#pragma unroll
          for (int jl = 0; jl < NL; ++jl) v[jl] = 0.f;
          if (act) {
            const float* Gp = Gl + (int64_t)__ldg(a.digitL + u) * sliceL;
#pragma unroll
            for (int jt = 0; jt < NT; ++jt)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const float4 gv = __ldg(reinterpret_cast<const float4*>(Gp + (jt * 8 + 2 * tq + e) * NL));
                const float c = acc[jt][2 * h + e];
                v[0] = fmaf(c, gv.x, v[0]);
                v[1] = fmaf(c, gv.y, v[1]);
                v[2] = fmaf(c, gv.z, v[2]);
                v[3] = fmaf(c, gv.w, v[3]);
              }
          }
          transpose_reduce<NL, 4>(v, lane);  // lane tq ends with jl = tq
          if (act) {
            const int jl = tq;
            const int64_t col = ((int64_t)(ar * nF + jf)) * NL + jl;
            const int s0 = __ldg(a.seg + u), s1 = __ldg(a.seg + u + 1);
            if (s1 - s0 > HEAVY_POS) {
              a.Yu[(int64_t)u * npad + col] = v[0];
            } else if (col < emb) {
              for (int s = s0; s < s1; ++s) a.out[(int64_t)__ldg(a.spos + s) * emb + col] = v[0];
            }
          }
        }
      }
    }
  }
}

}  // namespace tt
