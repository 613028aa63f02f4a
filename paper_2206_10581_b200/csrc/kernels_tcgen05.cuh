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

// metadata area of the backward (node batch of FB_NB)
constexpr size_t TC_META = sizeof(int64_t) * FB_NB + sizeof(int) * (3 * FB_NB + 12) + 64;

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
// Forward: P_F tiles on the tensor pipe, saved to Psave.  Persistent (one
// CTA per SM) and warp-specialised; the roles are coupled by mbarriers only:
//   warps 0-7   loaders, two sets of four.  Set s owns A stage s (tiles
//               t % 2 == s): thread (w % 4, lane) loads row m = 32 (w % 4) +
//               lane of its tile (all K), splits it into three BF16 slices and
//               writes them to TMEM with tcgen05.st -- A never touches shared
//               memory, so the tensor pipe reads only S from it.  The next
//               tile's row loads are in flight while the other set's tile is
//               on the tensor pipe.  Both sets stage half of each item's S
//               block (K x BN) into the shared-memory S ring.
//   warps 8-15  epilogue: accumulator lanes 32 (w % 4).. x columns
//               64 ((w - 8) / 4).. drained to registers (the accumulator is
//               released at once), turned around in shared memory, written as
//               4 full 128-byte row segments per store instruction.
//   warp 16     one thread issues the six-product MMAs (A from TMEM).
// TMEM: accumulators 2 x BN columns, then A slices 2 stages x 3 x K/2.
// Work items (digit group g, column block cb) are dealt round-robin over the
// CTAs, so the ncb items of a group run at the same time on neighbouring CTAs
// and share their A rows in L2.
// Experiment bits (FusedArgs::mode, TT_TC_VARIANT): 2 no MMAs, 4 no P_F
// stores, 8 no A loads.
constexpr int TCF_LOADERS = 8;   // two sets of four warps
constexpr int TCF_EPI = 8;
constexpr int TCF_THREADS = 32 * (TCF_LOADERS + TCF_EPI + 1);
constexpr int TCF_ES = 132;  // epilogue staging row stride (floats): 128 columns + pad, conflict-free 16-byte stores
// dynamic shared memory: forward = S ring (2 stages x 3 slices of K x BN)
// + the epilogue's staging rows; backward = S, A and dC planes + metadata
inline size_t tc_fwd_smem(int K, int BN) {
  return 2 * 3 * (size_t)K * BN * 2 + (size_t)4 * 32 * TCF_ES * 4;
}

// Work item `it` of the persistent forward: (digit group g, column block cb,
// chunk of the group's nodes) -- the same chunking as the FFMA kernels'
// work_item (a.split chunks at most, a.split_rows rows at least); g0 / n =
// the chunk's first node (in group order) and node count (0: empty item).
__device__ __forceinline__ void tc_item(const FusedArgs& a, int it, int& g, int& cb, int& g0, int& n) {
  if (a.split <= 1) {  // (the common case: no chunk arithmetic, no 64-bit divisions)
    g = it / a.ncb;
    cb = it - g * a.ncb;
    g0 = a.goffF[g];
    n = a.goffF[g + 1] - g0;
    return;
  }
  const int split = a.split;
  const int gc = it / a.ncb;
  cb = it - gc * a.ncb;
  g = gc / split;
  const int chunk = gc - g * split;
  const int n0 = a.goffF[g], ng = a.goffF[g + 1] - n0;
  const int nch = group_chunks(ng, a.RP, split, a.split_rows);
  if (chunk >= nch) { g0 = n0; n = 0; return; }
  g0 = n0 + (int)(((int64_t)ng * chunk) / nch);
  n = n0 + (int)(((int64_t)ng * (chunk + 1)) / nch) - g0;
}

// A CTA's static tile schedule: items it = blockIdx.x + k * gridDim.x, tiles
// of npt nodes (tb = first node of the tile within the item's node range)
struct TileCursor {
  int it, g0, n, tb;
  __device__ __forceinline__ void seek(const FusedArgs& a, int nitems) {
    while (it < nitems) {
      int g, cb;
      tc_item(a, it, g, cb, g0, n);
      if (tb < n) return;
      it += gridDim.x;
      tb = 0;
    }
  }
  __device__ __forceinline__ void advance(const FusedArgs& a, int nitems, int npt) {
    tb += npt;
    seek(a, nitems);
  }
};

template <int K, int BN, int RP>
__global__ void __launch_bounds__(TCF_THREADS, 1) k_tc_fwd(FusedArgs a) {
  TT_PDL_ENTRY();  // under programmatic dependent launch: the plan must be complete
  static_assert(BN == 128 && K % 32 == 0 && K <= 64 && TC_BM % RP == 0 && 32 % RP == 0, "tcgen05 forward shape");
  constexpr int NPT = TC_BM / RP;                 // nodes per tile
  constexpr uint32_t SPL = (uint32_t)K * BN * 2;  // bytes per S slice plane
  constexpr uint32_t ACOLS = K / 2;               // TMEM columns per A slice
  extern __shared__ __align__(128) uint8_t tsm[];
  float* Es = reinterpret_cast<float*>(tsm + 2 * 3 * SPL);
  __shared__ uint64_t s_full[2], s_empty[2], a_full[2], a_empty[2], c_full[2], c_empty[2];
  __shared__ uint32_t tslot;

  if (tt_failed(a.st)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tc::tmem_alloc<512>(&tslot);
  if (threadIdx.x == 32) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s_full[i], TCF_LOADERS);
      tc::mbar_init(&s_empty[i], 1);
      tc::mbar_init(&a_full[i], TCF_LOADERS / 2);
      tc::mbar_init(&a_empty[i], 1);
      tc::mbar_init(&c_full[i], 1);
      tc::mbar_init(&c_empty[i], TCF_EPI);
    }
    tc::fence_mbar_init();
  }
  tc::before_sync();
  __syncthreads();
  tc::after_sync();
  const uint32_t tm = tslot;
  const uint32_t tacc = tm, ta = tm + 2 * BN;
  const int nitems = (int)a.c.m[a.F] * a.ncb * (a.split > 1 ? a.split : 1);
  // TT_TC_TRACE=2: per-tile %globaltimer stamps, 256 per role and CTA:
  // [0] MMA issued, [1] epilogue has the accumulator, [2] epilogue done,
  // [3] A stage handed over by the loaders
  long long* trace = (a.dbg && blockIdx.x < 256) ? a.dbg + (int64_t)blockIdx.x * 1024 : nullptr;
  auto TR = [&](int role, uint32_t t) {
    if (trace && t < 256) {
      long long x;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(x));
      trace[role * 256 + t] = x;
    }
  };

  if (warp < TCF_LOADERS) {
    // ---------------- loaders ----------------
    const int set = warp >> 2, q = warp & 3;
    const int m = 32 * q + lane, jm = m / RP, am = m - jm * RP;
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    const int su = (int)(threadIdx.x & 127);  // thread within the set
    uint32_t t = 0, i = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      int g, cb, g0, n;
      tc_item(a, it, g, cb, g0, n);
      if (n == 0) continue;
      {  // half of the S block (rows k of the set's half) into S stage i % 2
        const int s = i & 1;
        tc::mbar_wait(&s_empty[s], ((i >> 1) & 1) ^ 1);
        uint8_t* S0 = tsm + s * 3 * SPL;
        const float* src = a.params + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F] + cb * BN;
        constexpr int UH = K * BN / 16;  // units (8 values) per set
#pragma unroll
        for (int uu = 0; uu < UH / 128; ++uu) {
          const int u = set * UH + su + uu * 128;
          const int cc = (u >> 3) % (BN / 8), k = ((u >> 3) / (BN / 8)) * 8 + (u & 7), c0 = cc * 8;
          const float4 x0 = __ldg(reinterpret_cast<const float4*>(src + (int64_t)k * a.NC + c0));
          const float4 x1 = __ldg(reinterpret_cast<const float4*>(src + (int64_t)k * a.NC + c0 + 4));
          const float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
          tc::store_split8(S0, S0 + SPL, S0 + 2 * SPL, k, c0, BN, x);
        }
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&s_full[s]);
        ++i;
      }
      for (int tb = 0; tb < n; tb += NPT, ++t) {
        if ((int)(t & 1) != set) continue;
        const int nn = min(NPT, n - tb);
        float x[K];
        if (jm < nn && !(a.mode & 8)) {
          const int node = __ldg(a.orderF + g0 + tb + jm);
          const int p = __ldg(a.parentF + node);
          const int64_t aoff = a.F == 1 ? a.c.core_off[0] + (int64_t)__ldg(a.digit0 + p) * a.c.slice[0]
                                        : (int64_t)p * RP * a.c.R[a.F];
          const float4* src = reinterpret_cast<const float4*>(a.Abase + aoff + am * K);
#pragma unroll
          for (int v = 0; v < K / 4; ++v) {
            const float4 y = __ldg(src + v);
            x[4 * v] = y.x; x[4 * v + 1] = y.y; x[4 * v + 2] = y.z; x[4 * v + 3] = y.w;
          }
        } else {
#pragma unroll
          for (int v = 0; v < K; ++v) x[v] = 0.f;
        }
        tc::mbar_wait(&a_empty[set], ((t >> 1) & 1) ^ 1);  // the (t/2)-th use of this set's stage
        tc::after_sync();
        const uint32_t base = ta + set * 3 * ACOLS + lane_off;
#pragma unroll
        for (int c = 0; c < K / 16; ++c) {  // 8 columns (16 values) per slice per step
          uint32_t p0[8], p1[8], p2[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) tc::split3(x[16 * c + 2 * v], x[16 * c + 2 * v + 1], p0[v], p1[v], p2[v]);
          tc::tmem_st8(base + 8 * c, p0);
          tc::tmem_st8(base + ACOLS + 8 * c, p1);
          tc::tmem_st8(base + 2 * ACOLS + 8 * c, p2);
        }
        tc::tmem_st_wait();
        tc::before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&a_full[set]);
        if (threadIdx.x == 0 || threadIdx.x == 128) TR(3, t);
      }
    }
  } else if (warp < TCF_LOADERS + TCF_EPI) {
    // ---------------- epilogue ----------------
    const int q = warp & 3, h = (warp - TCF_LOADERS) >> 2;
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    float* Ew = Es + q * 32 * TCF_ES;  // the quadrant's 32 staging rows (shared by its two warps)
    // the node ids of the next tile are loaded while this tile is drained
    const int jl0 = 32 * q / RP;
    auto tile_node = [&](const TileCursor& c) {
      return (c.it < nitems && lane < 32 / RP && jl0 + lane < min(NPT, c.n - c.tb))
                 ? __ldg(a.orderF + c.g0 + c.tb + jl0 + lane)
                 : 0;
    };
    // one tile: accumulator stage t % 2 -> Psave rows of the tile's nodes
    // (node ids in `mynode`, one per lane, loaded a tile ahead)
    auto drain = [&](uint32_t t, const TileCursor& c, int mynode) {
      const int cb = c.it % a.ncb;  // (it = (g * split + chunk) * ncb + cb)
      const int nn = min(NPT, c.n - c.tb);
      const int st = t & 1;
      tc::mbar_wait(&c_full[st], (t >> 1) & 1);
      tc::after_sync();
      if (threadIdx.x == 32 * TCF_LOADERS) TR(1, t);
      uint32_t v[64];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) tc::tmem_ld16_async(tacc + st * BN + lane_off + 64 * h + 16 * cc, v + 16 * cc);
      tc::tmem_ld_wait();
      tc::before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&c_empty[st]);
      // row (32 q + lane) of the tile: warps (q, h = 0) and (q, h = 1) write
      // the two 64-column halves of its staging row, then warp h = 0 issues
      // one 512-byte bulk (TMA) store of the row to its Psave segment (the
      // TMA unit's per-operation cost makes 512-byte copies twice as fast as
      // 256-byte ones).  The staging row is rewritten once the previous
      // tile's copy has read it (named barrier per quadrant, 64 threads).
      if (h == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      asm volatile("bar.sync %0, 64;\n" ::"r"(1 + q) : "memory");
      float* er = Ew + lane * TCF_ES + 64 * h;
#pragma unroll
      for (int qq = 0; qq < 16; ++qq)
        *reinterpret_cast<float4*>(er + 4 * qq) = make_float4(__uint_as_float(v[4 * qq]), __uint_as_float(v[4 * qq + 1]),
                                                              __uint_as_float(v[4 * qq + 2]), __uint_as_float(v[4 * qq + 3]));
      tc::fence_async_smem();
      asm volatile("bar.sync %0, 64;\n" ::"r"(1 + q) : "memory");
      if (h == 0) {
        const int jl = lane / RP;
        const int node = __shfl_sync(0xffffffffu, mynode, jl);
        if (jl0 + jl < nn && !(a.mode & 4)) {
          float* dst = a.Psave + ((int64_t)node * RP + (lane - jl * RP)) * a.NC + cb * BN;
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;\n" ::"l"(dst),
                       "r"(tc::smem_u32(Ew + lane * TCF_ES))
                       : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
      if (threadIdx.x == 32 * TCF_LOADERS) TR(2, t);
    };
    // unrolled by two with alternating node registers: a register copy of a
    // pending load would wait for it
    TileCursor cur{(int)blockIdx.x, 0, 0, 0};
    cur.seek(a, nitems);
    TileCursor nxt = cur;
    if (nxt.it < nitems) nxt.advance(a, nitems, NPT);
    int nodeA = tile_node(cur), nodeB = 0;
    uint32_t t = 0;
    while (cur.it < nitems) {
      nodeB = tile_node(nxt);
      drain(t++, cur, nodeA);
      cur = nxt;
      if (nxt.it < nitems) nxt.advance(a, nitems, NPT);
      if (cur.it >= nitems) break;
      nodeA = tile_node(nxt);
      drain(t++, cur, nodeB);
      cur = nxt;
      if (nxt.it < nitems) nxt.advance(a, nitems, NPT);
    }
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  } else if (lane == 0) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = tc::idesc_bf16(TC_BM, BN, 0, 1);
    uint32_t t = 0, i = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      int g, cb, g0, n;
      tc_item(a, it, g, cb, g0, n);
      if (n == 0) continue;
      const int s = i & 1;
      tc::mbar_wait(&s_full[s], (i >> 1) & 1);
      uint8_t* S0 = tsm + s * 3 * SPL;
      const tc::Operand ob = tc::mnmajor(tc::smem_u32(S0), tc::smem_u32(S0 + SPL), tc::smem_u32(S0 + 2 * SPL), BN);
      for (int tb = 0; tb < n; tb += NPT, ++t) {
        const int st = t & 1;
        tc::mbar_wait(&a_full[st], (t >> 1) & 1);
        tc::mbar_wait(&c_empty[st], ((t >> 1) & 1) ^ 1);
        tc::after_sync();
        TR(0, t);
        if (!(a.mode & 2)) tc::mma_x3_ts<K / 16>(tacc + st * BN, ta + st * 3 * ACOLS, ob, idesc, false);
        tc::commit(&a_empty[st]);
        tc::commit(&c_full[st]);
      }
      tc::commit(&s_empty[s]);
      ++i;
    }
  }
  tc::before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tm);
}

// ---------------------------------------------------------------------------
// Backward: dC on the CUDA cores, dG_F^T and dA on the tensor pipe.  512
// threads (16 warps) per CTA: the CUDA-core half of a tile is a chain of
// dependent L2 loads (ID digit -> last-core slice), so latency is hidden by
// warps, and one CTA holds the whole 192 KB operand set per SM.
constexpr int TCB_THREADS = 512;
inline size_t tc_bwd_smem(int K, int BN) {
  return 3 * (size_t)K * BN * 2 + 3 * (size_t)TC_BM * K * 2 + 3 * (size_t)TC_BM * BN * 2 + TC_META;
}

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
  int g, cb, g0, g1, chunk;
  if (!work_item(a, g, cb, chunk, g0, g1)) return;
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
    float* gdst = (a.split > 1 ? a.gsplit + ((int64_t)g * a.split + chunk) * a.c.slice[a.F]
                                : a.grads + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F]) + cb * BN + col;
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

// ---------------------------------------------------------------------------
// Backward, persistent (round 2, the default at K <= 64): the same tiles and
// products as k_tc_bwd, with
//   * a warp of its own (warp 8) that only issues the MMAs: in k_tc_bwd the
//     two issuing threads sat in dC-forming warps, and an issue that blocks on
//     a full tensor-pipe queue delayed their warps' next dC unit, so the MMAs
//     added to the tile time instead of running under the dC formation.  Nine
//     warps keep 168 registers per thread (17 warps would cap it at 96: five
//     warps on one SM sub-partition), so each of the 256 worker threads forms
//     two dC units of one node, column chunks c8 and c8 + 8 -- the same IDs and
//     last-core rows, two upstream column blocks: one latency chain, twice the
//     FMAs;
//   * dA double-buffered in TMEM: tile t's dA epilogue runs under tile t+1's
//     MMAs (TMEM: dG_F^T [0, K), dA [K, 2K) and [2K, 3K));
//   * one CTA per SM walking the items it = blockIdx.x + k * gridDim.x, with
//     the node metadata of the next node batch staged into the other of two
//     buffers and the next tile's A rows and dC units formed under the current
//     tile's MMAs across item boundaries: the per-item prologue (node
//     metadata chain, first tile) no longer stands alone on the SM.
// Per tile: wait MMA(t-1) -> [new item: drain dG_F^T of the last item,
// stage the slice block] -> store A(t), dC(t) planes -> barrier -> issue
// MMA(t) | dA epilogue of t-1, next batch's metadata, A(t+1) loads, dC(t+1).
constexpr int TCB2_WORKERS = 256;
constexpr int TCB2_THREADS = TCB2_WORKERS + 32;
constexpr size_t TC_META2 = 2 * (sizeof(int64_t) * FB_NB + sizeof(int) * (3 * FB_NB + 8)) + sizeof(int) * 40 + 64;
inline size_t tc_bwd2_smem(int K, int BN) {
  return 3 * (size_t)K * BN * 2 + 3 * (size_t)TC_BM * K * 2 + 3 * (size_t)TC_BM * BN * 2 + TC_META2;
}

struct BwdCursor {
  int it, g, cb, chunk, g0, g1, nb0, nbn, tb;
  // first non-empty item at or after `it` (stride gridDim.x); false: none left
  __device__ __forceinline__ bool seek_item(const FusedArgs& a, int nitems) {
    for (; it < nitems; it += gridDim.x)
      if (work_item_at(a, it, g, cb, chunk, g0, g1)) {
        nb0 = g0;
        nbn = min(FB_NB, g1 - g0);
        tb = 0;
        return true;
      }
    return false;
  }
  // next tile; sets new_batch / new_item
  __device__ __forceinline__ bool advance(const FusedArgs& a, int nitems, int npt, bool& new_batch, bool& new_item) {
    tb += npt;
    new_batch = new_item = false;
    if (tb < nbn) return true;
    new_batch = true;
    nb0 += FB_NB;
    tb = 0;
    if (nb0 < g1) {
      nbn = min(FB_NB, g1 - nb0);
      return true;
    }
    new_item = true;
    it += gridDim.x;
    return seek_item(a, nitems);
  }
};

// dC tile of the LDC variant: 128 rows x BN columns of the dC blocks that
// k_fused_wdc wrote over P_F, 8 units of 8 floats per worker thread, unit u:
// column chunk (u / 8) % (BN / 8), row 8 (u / 8 / (BN / 8)) + u % 8
template <int BN>
struct DTileRegs {
  static constexpr int N = TC_BM * BN / 8 / TCB2_WORKERS;
  float4 v[N][2];
};

template <int K, int BN, int RP, int NL, bool LDC>
__global__ void __launch_bounds__(TCB2_THREADS, 1) k_tc_bwd2(FusedArgs a) {
  TT_PDL_ENTRY();
  static_assert(BN == 128 && K % 16 == 0 && K <= 64 && 64 % K == 0 && TC_BM % RP == 0 && RP % 4 == 0,
                "tcgen05 backward shape");
  constexpr int W = TCB2_WORKERS;  // warps 0-7: dC, planes, epilogues; warp 8: MMA issue
  constexpr int NPT = TC_BM / RP;
  constexpr uint32_t TCOLS = 3 * K <= 128 ? 128 : 256;
  constexpr int EC = K / 2;  // epilogue columns per warp (8 warps = 4 lane quadrants x 2 column halves)
  static_assert(EC == 16 || EC == 32, "epilogue column slice");
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
  int64_t* s_aoff = reinterpret_cast<int64_t*>(D2 + TC_BM * BN * 2);  // [2][FB_NB]
  int* s_node = reinterpret_cast<int*>(s_aoff + 2 * FB_NB);           // [2][FB_NB]
  int* s_cs0 = s_node + 2 * FB_NB;                                    // [2][FB_NB]
  int* s_pref = s_cs0 + 2 * FB_NB;                                    // [2][FB_NB + 8]
  int* s_wsum = s_pref + 2 * (FB_NB + 8);                             // [40]
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;

  if (tt_failed(a.st)) return;
  const int nitems = (int)a.c.m[a.F] * a.ncb * (a.split > 1 ? a.split : 1);
  BwdCursor cur;
  cur.it = blockIdx.x;
  if (!cur.seek_item(a, nitems)) return;
  // TT_TC_TRACE=1: thread 0's clock cycles per phase, summed per CTA into
  // a.dbg[blockIdx.x * 16 + phase] (scripts/tc_trace.py with BWD2=1)
  const bool trace = a.dbg != nullptr && threadIdx.x == 0;
  long long ph[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tlast = clock64();
  auto mark = [&](int k) {
    if (trace) {
      const long long now = clock64();
      ph[k] += now - tlast;
      tlast = now;
    }
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool worker = threadIdx.x < W;
  const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
  const int eslice = ((warp >> 2) & 1) * EC;
  if (warp == 0) tc::tmem_alloc<TCOLS>(&tslot);
  if (threadIdx.x == 32) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  const int nF = a.nF;
  const int64_t npad = a.c.npad;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];
  const uint32_t id_g = tc::idesc_bf16(BN, K, 1, 1);
  const uint32_t id_a = tc::idesc_bf16(TC_BM, K, 0, 0);
  ATileRegs<K, W> ar;
  // this thread's dC units: unit0 = thread index with a 0 inserted at bit 4,
  // unit1 = unit0 | 16 (column chunk c8 + 8, same rows); k_tc_bwd's unit bit
  // layout, so each 8-thread store phase stays conflict-free
  const int x = threadIdx.x & (W - 1);
  const int unit = (x & 15) | ((x >> 4) << 5);
  const int c8 = (unit & 3) + 4 * ((unit >> 3) & 3);  // < 8
  const int rg = ((unit >> 2) & 1) + 2 * (unit >> 5);
  const int rot = unit & 3;
  const int m0 = rg * 4, uj = m0 / RP, a0 = m0 - uj * RP;
  constexpr int JF1 = 64 / K;  // unit1's core-F column block offset
  auto compute_dC = [&](const int* pref, const int* cs0s, int cb, int tb, int nn, float (&acc)[2][4][8]) {
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[v][i][t] = 0.f;
    if (uj >= nn || (a.mode & 16)) return;
    const int col0 = cb * BN + c8 * 8, jf = col0 / K, r0 = col0 - jf * K;
    const int fA = pref[tb + uj], fB = pref[tb + uj + 1], cs0 = cs0s[tb + uj];
    for (int f = fA; f < fB; ++f) {
      const int u = cs0 + (f - fA);
      const float* Gp = Gl + (int64_t)__ldg(a.digitL + u) * sliceL + r0 * NL;
      const float* Yp = a.dY + (int64_t)u * npad + ((int64_t)a0 * nF + jf) * NL;
      float yv[2][4][NL];
#pragma unroll
      for (int v = 0; v < 2; ++v)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int ii = (i + rot) & 3;
#pragma unroll
          for (int l4 = 0; l4 < NL; l4 += 4) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(Yp + (int64_t)ii * nF * NL + v * JF1 * NL + l4));
            yv[v][i][l4] = q.x; yv[v][i][l4 + 1] = q.y; yv[v][i][l4 + 2] = q.z; yv[v][i][l4 + 3] = q.w;
          }
        }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        float gv[NL];
#pragma unroll
        for (int l4 = 0; l4 < NL; l4 += 4) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(Gp + t * NL + l4));
          gv[l4] = q.x; gv[l4 + 1] = q.y; gv[l4 + 2] = q.z; gv[l4 + 3] = q.w;
        }
#pragma unroll
        for (int v = 0; v < 2; ++v)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float s = acc[v][i][t];
#pragma unroll
            for (int jl = 0; jl < NL; ++jl) s = fmaf(yv[v][i][jl], gv[jl], s);
            acc[v][i][t] = s;
          }
      }
    }
  };
  const int em = 32 * (warp & 3) + lane;  // epilogue row (TMEM lane)
  const int emj = em / RP, ema = em - emj * RP;
  auto tmem_row = [&](uint32_t taddr, float (&v)[EC]) {
    if constexpr (EC == 32) {
      uint32_t r[32];
      tc::tmem_ld16_async(taddr, r);
      tc::tmem_ld16_async(taddr + 16, r + 16);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
    } else {
      tc::tmem_ld16(taddr, v);
    }
  };
  // dG_F^T of a finished item -> its slice block (or its chunk's partial)
  auto drain_dG = [&](uint32_t tm, int g, int cb, int chunk) {
    const int col = 32 * (warp & 3) + lane;
    float* gdst = (a.split > 1 ? a.gsplit + ((int64_t)g * a.split + chunk) * a.c.slice[a.F]
                                : a.grads + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F]) + cb * BN + col;
    float v[EC];
    tmem_row(tm + lane_base + eslice, v);
#pragma unroll
    for (int i = 0; i < EC; ++i) gdst[(int64_t)(eslice + i) * a.NC] = v[i];
  };
  auto drain_dA = [&](uint32_t tm, int buf, float* dst) {
    float v[EC];
    tmem_row(tm + lane_base + K + buf * K + eslice, v);
    if (dst && !(a.mode & 4)) {
#pragma unroll
      for (int q = 0; q < EC / 4; ++q)
        *reinterpret_cast<float4*>(dst + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  };
  auto store_dC = [&](const float (&acc)[2][4][8]) {
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int i = 0; i < 4; ++i) tc::store_split8(D0, D1, D2, m0 + ((i + rot) & 3), (c8 + 8 * v) * 8, BN, acc[v][i]);
  };

  // prologue: first item's slice block, first batch's metadata, first tile
  if (worker) tc_stage_slice<K, BN, W>(a, cur.g, cur.cb, S0, S1, S2);
  int mb = 0;
  tc_prep_nodes<TCB2_THREADS>(a, cur.nb0, cur.nbn, s_node, s_cs0, s_pref, s_aoff, s_wsum);
  float acc[2][4][8];
  DTileRegs<BN> dr;
  auto load_dC = [&](const int* nodes, int cb, int tb, int nn) {
#pragma unroll
    for (int i = 0; i < DTileRegs<BN>::N; ++i) {
      const int u = x + i * W;
      const int kc = (u >> 3) % (BN / 8), m = ((u >> 3) / (BN / 8)) * 8 + (u & 7);
      const int j = m / RP;
      if (j < nn) {
        const float* src = a.Psave + ((int64_t)nodes[tb + j] * RP + (m - j * RP)) * a.NC + cb * BN + kc * 8;
        dr.v[i][0] = __ldg(reinterpret_cast<const float4*>(src));
        dr.v[i][1] = __ldg(reinterpret_cast<const float4*>(src + 4));
      } else {
        dr.v[i][0] = dr.v[i][1] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  };
  if (worker) {
    tc_load_A<K, RP, W>(a, 0, min(NPT, cur.nbn), s_aoff, ar);
    if constexpr (LDC) load_dC(s_node, cur.cb, 0, min(NPT, cur.nbn));
    else compute_dC(s_pref, s_cs0, cur.cb, 0, min(NPT, cur.nbn), acc);
  }
  mark(8);
  bool first_of_item = true;
  int pg = cur.g, pcb = cur.cb, pchunk = cur.chunk;  // item of the last issued tile
  float* dst_prev = nullptr;
  uint32_t t = 0;
  for (;;) {
    const int nn = min(NPT, cur.nbn - cur.tb);
    if (t > 0) {
      tc::mbar_wait(&bar, (t - 1) & 1);  // MMA(t-1) done: planes free, dA(t-1) ready
      tc::after_sync();
      mark(0);
      if (first_of_item && worker) {
        drain_dG(tslot, pg, pcb, pchunk);
        tc_stage_slice<K, BN, W>(a, cur.g, cur.cb, S0, S1, S2);
      }
      mark(1);
    }
    if (worker) {
      if (!(a.mode & 8)) tc_store_A<K, W>(ar, A0, A1, A2);
      if constexpr (LDC) {
#pragma unroll
        for (int i = 0; i < DTileRegs<BN>::N; ++i) {
          const int u = x + i * W;
          const int kc = (u >> 3) % (BN / 8), m = ((u >> 3) / (BN / 8)) * 8 + (u & 7);
          const float v8[8] = {dr.v[i][0].x, dr.v[i][0].y, dr.v[i][0].z, dr.v[i][0].w,
                               dr.v[i][1].x, dr.v[i][1].y, dr.v[i][1].z, dr.v[i][1].w};
          tc::store_split8(D0, D1, D2, m, kc * 8, BN, v8);
        }
      } else {
        store_dC(acc);
      }
    }
    mark(2);
    tc::fence_async_smem();
    tc::before_sync();
    __syncthreads();
    tc::after_sync();
    mark(3);
    const uint32_t tm = tslot;
    if (!worker) {
      if (lane == 0) {
        if (!(a.mode & 2)) {
          const tc::Operand dcT = tc::mnmajor(tc::smem_u32(D0), tc::smem_u32(D1), tc::smem_u32(D2), BN);
          const tc::Operand aB = tc::mnmajor(tc::smem_u32(A0), tc::smem_u32(A1), tc::smem_u32(A2), K);
          tc::mma_x3<TC_BM / 16>(tm, dcT, aB, id_g, !first_of_item);
          const tc::Operand dcK = tc::kmajor(tc::smem_u32(D0), tc::smem_u32(D1), tc::smem_u32(D2), BN);
          const tc::Operand sT = tc::kmajor(tc::smem_u32(S0), tc::smem_u32(S1), tc::smem_u32(S2), BN);
          tc::mma_x3<BN / 16>(tm + K + (t & 1) * K, dcK, sT, id_a, false);
        }
        tc::commit(&bar);
      }
      __syncwarp();
    } else if (t > 0) {
      drain_dA(tm, (t - 1) & 1, dst_prev);
    }
    mark(4);
    const int* nodes = s_node + mb * FB_NB;
    dst_prev = (worker && emj < nn) ? a.dPc + ((int64_t)nodes[cur.tb + emj] * a.ncb + cur.cb) * RP * K + ema * K + eslice
                                    : nullptr;
    pg = cur.g;
    pcb = cur.cb;
    pchunk = cur.chunk;
    bool new_batch, new_item;
    if (!cur.advance(a, nitems, NPT, new_batch, new_item)) break;
    first_of_item = new_item;
    if (new_batch) {
      mb ^= 1;
      tc_prep_nodes<TCB2_THREADS>(a, cur.nb0, cur.nbn, s_node + mb * FB_NB, s_cs0 + mb * FB_NB,
                                  s_pref + mb * (FB_NB + 8), s_aoff + mb * FB_NB, s_wsum);
    }
    mark(5);
    if (worker) {
      const int nn2 = min(NPT, cur.nbn - cur.tb);
      if (!(a.mode & 8)) tc_load_A<K, RP, W>(a, cur.tb, nn2, s_aoff + mb * FB_NB, ar);
      if constexpr (LDC) {
        if (!(a.mode & 16)) load_dC(s_node + mb * FB_NB, cur.cb, cur.tb, nn2);
      } else {
        compute_dC(s_pref + mb * (FB_NB + 8), s_cs0 + mb * FB_NB, cur.cb, cur.tb, nn2, acc);
      }
    }
    mark(6);
    ++t;
  }
  // last tile: its dA, then the last item's dG_F
  tc::mbar_wait(&bar, t & 1);
  tc::after_sync();
  if (worker) {
    drain_dA(tslot, t & 1, dst_prev);
    drain_dG(tslot, pg, pcb, pchunk);
  }
  mark(9);
  if (trace) {
    ph[7] = t + 1;
    for (int k = 0; k < 12; ++k) a.dbg[blockIdx.x * 16 + k] = ph[k];
  }
  tc::before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<TCOLS>(tslot);
}

// ---------------------------------------------------------------------------
// Backward with both dC operands in TMEM (round 2, TT_TCBWD=4; dC formed by
// k_fused_wdc over the saved P_F blocks).  The tensor pipe alternates
//   dG_F^T(t) = dC(t)^T . A(t)   (A operand dC^T from TMEM, B = A planes)
//   dA(t)     = dC(t) . S^T      (A operand dC from TMEM, B = S planes)
// and each half's operands are rewritten while the other half runs:
// dC^T(t+1) and A(t+1) as soon as dG_F^T(t) completes (under dA(t)), dC(t+1)
// and the drain of dA(t) as soon as dA(t) completes (under dG_F^T(t+1)).
// The dC tiles arrive by TMA: per node and 32-column chunk one
// cp.async.bulk.tensor.2d box {32 floats, RP rows} of the saved blocks, with
// the 128-byte swizzle (address-based: a box may start at any 512-byte
// offset, scripts/micro/tma_swz.cu), into two raw tile buffers; so the
// converters read both layouts from shared memory without bank conflicts
// (column reads: one wavefront; row reads: four per 512 bytes).
// TMEM (512 columns): dC [0, 192) (lane = tile row, 3 slices x BN/2),
// dC^T [192, 384) (lane = block column, 3 slices x 128/2), dG_F^T [384, 384+K),
// dA [448, 448+K).
// Warps 0 .. 4 CW - 1 convert (quadrant w % 4, part h = w / 4 of CW: dC^T rows
// RW h.., dC columns RW h.., accumulator columns K / CW h..; RW = 128 / CW);
// warp 4 CW issues the MMAs; warp 4 CW + 1 is the producer: node metadata of
// a tile, its TMA boxes, L2 prefetch of its A rows and of each new item's
// slice block.  CW = 2; CW = 4 (16 converter warps at 96 registers) measured
// slower (papers 1.452 -> 1.515 ms/step).
constexpr int TCB3_CW = 2;                  // converter warps per TMEM lane quadrant
constexpr int TCB3_CONV = 4 * TCB3_CW;
constexpr int TCB3_THREADS = 32 * (TCB3_CONV + 2);
constexpr int TCB3_RAW = TC_BM * 128 * 4;  // one raw dC tile (fp32, 4 chunks of 128 rows x 128 bytes)
inline size_t tc_bwd3_smem(int K, int BN) {
  return 1024 + 2 * (size_t)TCB3_RAW + 3 * (size_t)K * BN * 2 + 3 * (size_t)TC_BM * K * 2 + 2 * 32 * 8 + 128;
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
      ::"r"((unsigned)__cvta_generic_to_shared(smem_dst)), "l"(map), "r"(x), "r"(y), "r"(z),
      "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

template <int K, int BN, int RP, int NL>
__global__ void __launch_bounds__(TCB3_THREADS, 1) k_tc_bwd3(FusedArgs a, const __grid_constant__ CUtensorMap tmP) {
  TT_PDL_ENTRY();
  static_assert(BN == 128 && (K == 32 || K == 64) && TC_BM % RP == 0 && RP >= 4 && 64 % RP == 0, "shape");
  constexpr int NPT = TC_BM / RP;
  constexpr uint32_t T_DC = 0, T_DCT = 192, T_DG = 384, T_DA = 448;
  constexpr int CW = TCB3_CW;
  constexpr int EC = K / CW;     // accumulator columns per converter warp
  constexpr int RW = TC_BM / CW;  // dC^T rows / dC columns per converter warp
  static_assert(EC % 8 == 0 && RW % 32 == 0, "converter split");
  constexpr int NA = TC_BM * K / 8 / (32 * TCB3_CONV);  // A units (8 values) per converter thread
  extern __shared__ uint8_t tsm_raw[];
  // 1024-byte aligned base (the swizzle atom); raw buffers first
  uint8_t* base = tsm_raw + ((1024 - (tc::smem_u32(tsm_raw) & 1023)) & 1023);
  uint8_t* RAW = base;  // [2][4 chunks][128 rows][128 B], swizzled
  uint8_t* S0 = RAW + 2 * TCB3_RAW;
  uint8_t* S1 = S0 + K * BN * 2;
  uint8_t* S2 = S1 + K * BN * 2;
  uint8_t* A0 = S2 + K * BN * 2;
  uint8_t* A1 = A0 + TC_BM * K * 2;
  uint8_t* A2 = A1 + TC_BM * K * 2;
  int* r_node = reinterpret_cast<int*>(A2 + TC_BM * K * 2);  // [2][32]
  int* r_aoff = r_node + 64;                                 // [2][32] (float offsets < 2^31)
  uint64_t* bars = reinterpret_cast<uint64_t*>(r_aoff + 64);
  uint64_t* b_gt = bars;
  uint64_t* b_c = bars + 1;
  uint64_t* b_gdone = bars + 2;
  uint64_t* b_ddone = bars + 3;
  uint64_t* b_full = bars + 4;   // [2]
  uint64_t* b_empty = bars + 6;  // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);

  if (tt_failed(a.st)) return;
  const int nitems = (int)a.c.m[a.F] * a.ncb * (a.split > 1 ? a.split : 1);
  BwdCursor cur;
  cur.it = blockIdx.x;
  if (!cur.seek_item(a, nitems)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 2 * TCB3_RAW / 16; i += TCB3_THREADS)
    reinterpret_cast<uint4*>(RAW)[i] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // (ordered before the TMA writes)
  if (warp == 0) tc::tmem_alloc<512>(tslot);
  if (threadIdx.x == 32) {
    tc::mbar_init(b_gt, TCB3_CONV);
    tc::mbar_init(b_c, TCB3_CONV);
    tc::mbar_init(b_gdone, 1);
    tc::mbar_init(b_ddone, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&b_full[i], 1);
      tc::mbar_init(&b_empty[i], TCB3_CONV);
    }
    tc::fence_mbar_init();
  }
  tc::before_sync();
  __syncthreads();
  tc::after_sync();
  const uint32_t tm = *tslot;

  if (warp == TCB3_CONV + 1) {
    // ---------------- producer: metadata, TMA boxes, L2 prefetch ----------------
    // a tile's metadata is fetched (and its A rows and slice block
    // prefetched into L2) while the producer waits for the buffer of the
    // tile before it, so the TMA boxes go out as soon as a buffer frees
    int last_it = -1;
    auto fetch = [&](const BwdCursor& c, int& nn, int& node, int& aoff) {
      nn = min(NPT, c.nbn - c.tb);
      node = aoff = 0;
      if (lane < nn) {
        node = __ldg(a.orderF + c.nb0 + c.tb + lane);
        const int p = __ldg(a.parentF + node);
        aoff = (int)(a.F == 1 ? a.c.core_off[0] + (int64_t)__ldg(a.digit0 + p) * a.c.slice[0]
                              : (int64_t)p * RP * a.c.R[a.F]);
        prefetch_l2(a.Abase + aoff, RP * K * 4);
      }
      if (c.it != last_it) {
        last_it = c.it;
        const float* sb = a.params + a.c.core_off[a.F] + (int64_t)c.g * a.c.slice[a.F] + c.cb * BN;
        for (int k = lane; k < K; k += 32) prefetch_l2(sb + (int64_t)k * a.NC, BN * 4);
      }
    };
    BwdCursor c = cur;
    uint32_t tau = 0;
    int nn, node, aoff;
    fetch(c, nn, node, aoff);
    for (;;) {
      const int sl = tau & 1;
      tc::mbar_wait_sleep(&b_empty[sl], ((tau >> 1) & 1) ^ 1);  // (parked: not latency-critical)
      if (lane < nn) {
        r_node[sl * 32 + lane] = node;
        r_aoff[sl * 32 + lane] = aoff;
      }
      __syncwarp();
      if (lane == 0) mbar_expect_tx(&b_full[sl], (a.mode & 16) ? 0u : (unsigned)(nn * RP * 512));
      __syncwarp();
      if (lane < nn && !(a.mode & 16))  // the node's RP rows x BN columns: one 3-D box [4 chunks][RP][32]
        tma_load_3d(RAW + sl * TCB3_RAW + lane * RP * 512, &tmP, &b_full[sl], 0, node * RP, c.cb * (BN / 32));
      bool nb, ni;
      if (!c.advance(a, nitems, NPT, nb, ni)) break;
      fetch(c, nn, node, aoff);
      ++tau;
    }
  } else if (warp == TCB3_CONV) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t id_g = tc::idesc_bf16(BN, K, 0, 1);     // dG^T = dC^T (TMEM) . A
      const uint32_t id_a = tc::idesc_bf16(TC_BM, K, 0, 0);  // dA = dC (TMEM) . S^T
      const tc::Operand aB = tc::mnmajor(tc::smem_u32(A0), tc::smem_u32(A1), tc::smem_u32(A2), K);
      const tc::Operand sT = tc::kmajor(tc::smem_u32(S0), tc::smem_u32(S1), tc::smem_u32(S2), BN);
      BwdCursor c = cur;
      uint32_t t = 0;
      bool first = true;
      for (;;) {
        tc::mbar_wait(b_gt, t & 1);
        tc::after_sync();
        if (!(a.mode & 2)) tc::mma_x3_ts<TC_BM / 16>(tm + T_DG, tm + T_DCT, aB, id_g, !first);
        tc::commit(b_gdone);
        tc::mbar_wait(b_c, t & 1);
        tc::after_sync();
        if (!(a.mode & 2)) tc::mma_x3_ts<BN / 16>(tm + T_DA, tm + T_DC, sT, id_a, false);
        tc::commit(b_ddone);
        bool nb, ni;
        if (!c.advance(a, nitems, NPT, nb, ni)) break;
        first = ni;
        ++t;
      }
    }
    __syncwarp();
  } else {
    // ---------------- converters ----------------
    const int q = warp & 3, h = warp >> 2;
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    const int x = threadIdx.x;     // 0 .. 255
    const int cc = 32 * q + lane;  // block column (dC^T lane) / tile row (dC lane)
#ifdef TT_BWD3_TRACE  // thread 0's cycles per phase, summed into a.dbg[blockIdx.x * 16 + k] (TT_TC_TRACE=1)
    const bool trace = a.dbg != nullptr && threadIdx.x == 0;
    long long ph[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tlast = clock64();
    auto mark = [&](int k) {
      if (trace) {
        const long long now = clock64();
        ph[k] += now - tlast;
        tlast = now;
      }
    };
#else
    auto mark = [](int) {};
#endif
    auto ld_acc = [&](uint32_t taddr, uint32_t (&r)[EC]) {
      if constexpr (EC >= 16) {
#pragma unroll
        for (int i = 0; i < EC / 16; ++i) tc::tmem_ld16_async(taddr + 16 * i, r + 16 * i);
        tc::tmem_ld_wait();
      } else {
        float f[8];
        tc::tmem_ld8(taddr, f);
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = __float_as_uint(f[i]);
      }
    };
    auto drain_dG = [&](int g, int cb, int chunk) {
      float* gdst = (a.split > 1 ? a.gsplit + ((int64_t)g * a.split + chunk) * a.c.slice[a.F]
                                  : a.grads + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F]) + cb * BN + cc;
      uint32_t r[EC];
      ld_acc(tm + lane_off + T_DG + h * EC, r);
#pragma unroll
      for (int i = 0; i < EC; ++i) gdst[(int64_t)(h * EC + i) * a.NC] = __uint_as_float(r[i]);
    };
    auto drain_dA = [&](float* dst) {
      uint32_t da[EC];
      ld_acc(tm + lane_off + T_DA + h * EC, da);
      if (dst) {
#pragma unroll
        for (int v = 0; v < EC / 4; ++v)
          reinterpret_cast<float4*>(dst)[v] = make_float4(__uint_as_float(da[4 * v]), __uint_as_float(da[4 * v + 1]),
                                                          __uint_as_float(da[4 * v + 2]), __uint_as_float(da[4 * v + 3]));
      }
    };
    BwdCursor c = cur;
    uint32_t t = 0;
    bool first = true;
    int pg = 0, pcb = 0, pchunk = 0;
    float* dst_prev = nullptr;
    // A rows of tile tt into registers: issued under the previous tile's dC
    // conversion when tile tt's buffer has landed by then, else after it
    float4 av[NA][2];
    auto load_A = [&](uint32_t tt, int nn) {
      const int sl = tt & 1;
      tc::mbar_wait(&b_full[sl], (tt >> 1) & 1);
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        const int u = x + i * 32 * TCB3_CONV;
        const int kc = (u >> 3) % (K / 8), m = ((u >> 3) / (K / 8)) * 8 + (u & 7), j = m / RP;
        av[i][0] = av[i][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < nn) {
          const float* src = a.Abase + r_aoff[sl * 32 + j] + (m - j * RP) * K + kc * 8;
          av[i][0] = __ldg(reinterpret_cast<const float4*>(src));
          av[i][1] = __ldg(reinterpret_cast<const float4*>(src + 4));
        }
      }
    };
    load_A(0, min(NPT, c.nbn - c.tb));
    bool a_ready = true;  // av holds tile t's A rows
    for (;;) {
      const int sl = t & 1;
      const int nn = min(NPT, c.nbn - c.tb);
      mark(8);
      const uint8_t* raw = RAW + sl * TCB3_RAW;
      mark(0);
      // (B) after dG_F^T(t-1): [new item: drain dG_F^T], write A(t) and dC^T(t)
      if (t > 0) {
        tc::mbar_wait(b_gdone, (t - 1) & 1);
        tc::after_sync();
      }
      mark(1);
      if (first && t > 0) drain_dG(pg, pcb, pchunk);
      mark(9);
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        const int u = x + i * 32 * TCB3_CONV;
        const int kc = (u >> 3) % (K / 8), m = ((u >> 3) / (K / 8)) * 8 + (u & 7);
        const float v8[8] = {av[i][0].x, av[i][0].y, av[i][0].z, av[i][0].w,
                             av[i][1].x, av[i][1].y, av[i][1].z, av[i][1].w};
        tc::store_split8<true>(A0, A1, A2, m, kc * 8, K, v8);
      }
      // raw tile layout (one 3-D box per node): 128-byte line
      // L(m, qc) = (m / RP) 4 RP + qc RP + m % RP, 16-byte unit u at
      // L 128 + ((u ^ (L & 7)) << 4)
      // Rows past the tile's nodes hold finite stale values (the buffers are
      // zeroed at entry): their A rows are zero, so they add nothing to dG_F,
      // and their dA rows are not stored -- no per-element predicates.
      {
        // column cc = 32 q + lane of chunk q; rows RW h + k, k < RW: line
        // Lb + (k / RP) 4 RP + k % RP with Lb = (RW h / RP) 4 RP + q RP, and
        // L & 7 = (q RP + k % RP) & 7 -- a per-thread offset table xo
        const uint8_t* colp = raw + (lane & 3) * 4 + ((RW * h / RP) * 4 * RP + q * RP) * 128;
        const int c16 = lane >> 2;
        constexpr int NX = RP < 8 ? RP : 8;
        int xo[NX];
#pragma unroll
        for (int r = 0; r < NX; ++r) xo[r] = (c16 ^ ((q * RP + r) & 7)) << 4;
        auto at = [&](int k) {
          return *reinterpret_cast<const float*>(colp + ((k / RP) * 4 * RP + k % RP) * 128 + xo[(k % RP) % NX]);
        };
#pragma unroll
        for (int ch = 0; ch < RW / 16; ++ch) {
          uint32_t w0[8], w1[8], w2[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) tc::split3t(at(16 * ch + 2 * i), at(16 * ch + 2 * i + 1), w0[i], w1[i], w2[i]);
          const uint32_t col = tm + lane_off + T_DCT + (RW / 2) * h + 8 * ch;
          tc::tmem_st8(col, w0);
          tc::tmem_st8(col + 64, w1);
          tc::tmem_st8(col + 128, w2);
        }
      }
      tc::tmem_st_wait();
      tc::fence_async_smem();
      tc::before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(b_gt);
      mark(2);
      // the next tile, and its A rows now if its buffer is already in
      BwdCursor nx = c;
      bool nb, ni;
      const bool more = nx.advance(a, nitems, NPT, nb, ni);
      a_ready = false;
      if (more && tc::mbar_test(&b_full[(t + 1) & 1], ((t + 1) >> 1) & 1)) {
        load_A(t + 1, min(NPT, nx.nbn - nx.tb));
        a_ready = true;
      }
      // dA destination of tile t (row cc)
      float* dst_cur;
      {
        const int j = cc / RP;
        dst_cur = (j < nn && !(a.mode & 4))
                      ? a.dPc + ((int64_t)r_node[sl * 32 + j] * a.ncb + c.cb) * RP * K + (cc - j * RP) * K + h * EC
                      : nullptr;
      }
      mark(3);
      // (D) after dA(t-1): drain and store it, [new item: stage S], write dC(t)
      uint32_t da[EC];  // dA(t-1): read before dA(t) may overwrite it, stored after dC(t) is handed over
      if (t > 0) {
        tc::mbar_wait(b_ddone, (t - 1) & 1);
        tc::after_sync();
        mark(4);
        ld_acc(tm + lane_off + T_DA + h * EC, da);
      }
      mark(6);
      if (first) tc_stage_slice<K, BN, 32 * TCB3_CONV>(a, c.g, c.cb, S0, S1, S2);
      {
        // row cc, columns RW h .. RW h + RW - 1 = 32-column chunks (RW / 32) h ..
#pragma unroll
        for (int hc = 0; hc < RW / 32; ++hc) {
          const int L = (cc / RP) * 4 * RP + ((RW / 32) * h + hc) * RP + (cc % RP);
          const uint8_t* rowp = raw + L * 128;
          const int sw = L & 7;
#pragma unroll
          for (int uu = 0; uu < 2; ++uu) {  // 16 columns per step
            float v[16];
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4) {
              const int u = 4 * uu + k4;
              const float4 y = *reinterpret_cast<const float4*>(rowp + ((u ^ sw) << 4));
              v[4 * k4] = y.x; v[4 * k4 + 1] = y.y; v[4 * k4 + 2] = y.z; v[4 * k4 + 3] = y.w;
            }
            uint32_t w0[8], w1[8], w2[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) tc::split3t(v[2 * i], v[2 * i + 1], w0[i], w1[i], w2[i]);
            const uint32_t col = tm + lane_off + T_DC + (RW / 2) * h + 16 * hc + 8 * uu;
            tc::tmem_st8(col, w0);
            tc::tmem_st8(col + 64, w1);
            tc::tmem_st8(col + 128, w2);
          }
        }
      }
      tc::tmem_st_wait();
      tc::fence_async_smem();
      tc::before_sync();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(b_c);
        tc::mbar_arrive(&b_empty[sl]);  // raw tile and metadata slot consumed
      }
      mark(5);
      if (t > 0 && dst_prev) {
#pragma unroll
        for (int v = 0; v < EC / 4; ++v)
          reinterpret_cast<float4*>(dst_prev)[v] = make_float4(__uint_as_float(da[4 * v]), __uint_as_float(da[4 * v + 1]),
                                                               __uint_as_float(da[4 * v + 2]), __uint_as_float(da[4 * v + 3]));
      }
      dst_prev = dst_cur;
      pg = c.g;
      pcb = c.cb;
      pchunk = c.chunk;
      if (!more) break;
      c = nx;
      first = ni;
      ++t;
      if (!a_ready) load_A(t, min(NPT, c.nbn - c.tb));
    }
    // the last tile's dA, the last item's dG_F
    tc::mbar_wait(b_ddone, t & 1);
    tc::after_sync();
    drain_dA(dst_prev);
    drain_dG(pg, pcb, pchunk);
    mark(9);
#ifdef TT_BWD3_TRACE
    if (trace) {
      ph[7] = t + 1;
      for (int k = 0; k < 12; ++k) a.dbg[blockIdx.x * 16 + k] = ph[k];
    }
#endif
  }
  tc::before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tm);
}

// ---------------------------------------------------------------------------
// Backward at rank 128 (the rank sweep's R = 128): 64-column blocks, so the
// BF16x3 planes fit in 192 KB (S 48 KB, A 96 KB, dC 48 KB; 128-column blocks
// would need 288 KB).  dG_F is accumulated untransposed, M = 128 (k) x N = 64
// (columns) with A^T read MN-major, since an M = 64 dG_F^T accumulator has a
// different TMEM lane layout; dA = dC . S^T is M = 128 (rows) x N = 128 (k).
// dC unit: 2 rows of one node x 8 columns per thread (512 units); thread bits
// [0] c8 low, [1] row pair, [2] node low, [3,5) c8 high, [5,9) node high, and
// row i of the pair stored in rotated order i ^ (c8 & 1), so the 8 threads of
// a store phase write 8 distinct rows of a core matrix: conflict-free.
// The forward at rank 128 runs the FFMA kernel (the forward's TMEM budget,
// 2 x 128 accumulator + 2 x 3 x 64 A columns, exceeds 512).
template <int RP, int NL>
__global__ void __launch_bounds__(TCB_THREADS, 1) k_tc_bwd128(FusedArgs a) {
  TT_PDL_ENTRY();
  constexpr int K = 128, BN = 64, T = TCB_THREADS;
  static_assert(RP == 4, "rank-128 tensor backward: 4 rows per node");
  constexpr int NPT = TC_BM / RP;
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
  int g, cb, g0, g1, chunk;
  if (!work_item(a, g, cb, chunk, g0, g1)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
  if (warp == 0) tc::tmem_alloc<256>(&tslot);
  if (threadIdx.x == 32) {
    tc::mbar_init(&bar, 2);
    tc::fence_mbar_init();
  }
  tc_stage_slice<K, BN, T>(a, g, cb, S0, S1, S2);
  const int nF = a.nF;
  const int64_t npad = a.c.npad;
  const float* Gl = a.params + a.c.core_off[a.c.d - 1];
  const int64_t sliceL = a.c.slice[a.c.d - 1];
  const uint32_t id_g = tc::idesc_bf16(K, BN, 1, 1);     // dG = A^T . dC   (M = 128 k, N = 64 cols)
  const uint32_t id_a = tc::idesc_bf16(TC_BM, K, 0, 0);  // dA = dC . S^T   (M = 128 rows, N = 128 k)
  uint32_t phase = 0;
  int tiles = 0;
  ATileRegs<K, T> ar;
  const int t = threadIdx.x;
  const int c8 = (t & 1) | (((t >> 3) & 3) << 1);
  const int hh = (t >> 1) & 1;
  const int uj = ((t >> 2) & 1) | ((t >> 5) << 1);
  const int rot = c8 & 1;
  const int a0 = 2 * hh;  // the unit's first row within its node
  const int colg = cb * BN + c8 * 8, jf = colg / K, r0 = colg - jf * K;
  auto compute_dC = [&](int tb, int nn, float (&acc)[2][8]) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[i][q] = 0.f;
    if (uj >= nn) return;
    const int fA = s_pref[tb + uj], fB = s_pref[tb + uj + 1], cs0 = s_cs0[tb + uj];
    for (int f = fA; f < fB; ++f) {
      const int u = cs0 + (f - fA);
      const float* Gp = Gl + (int64_t)__ldg(a.digitL + u) * sliceL + r0 * NL;
      const float* Yp = a.dY + (int64_t)u * npad + ((int64_t)a0 * nF + jf) * NL;
      float yv[2][NL];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int ii = i ^ rot;
#pragma unroll
        for (int l4 = 0; l4 < NL; l4 += 4) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(Yp + (int64_t)ii * nF * NL + l4));
          yv[i][l4] = x.x; yv[i][l4 + 1] = x.y; yv[i][l4 + 2] = x.z; yv[i][l4 + 3] = x.w;
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float gv[NL];
#pragma unroll
        for (int l4 = 0; l4 < NL; l4 += 4) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(Gp + q * NL + l4));
          gv[l4] = x.x; gv[l4 + 1] = x.y; gv[l4 + 2] = x.z; gv[l4 + 3] = x.w;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          float sacc = acc[i][q];
#pragma unroll
          for (int jl = 0; jl < NL; ++jl) sacc = fmaf(yv[i][jl], gv[jl], sacc);
          acc[i][q] = sacc;
        }
      }
    }
  };
  float acc[2][8];
  const int em = 32 * (warp & 3) + lane;  // epilogue row (TMEM lane)
  const int emj = em / RP, ema = em - emj * RP;
  const int esl = (warp >> 2) * 32;       // dA epilogue: 32 of the 128 k columns
  for (int nb0 = g0; nb0 < g1; nb0 += FB_NB) {
    const int nbn = min(FB_NB, g1 - nb0);
    tc_prep_nodes<T>(a, nb0, nbn, s_node, s_cs0, s_pref, s_aoff, s_wsum);
    tc_load_A<K, RP, T>(a, 0, min(NPT, nbn), s_aoff, ar);
    compute_dC(0, min(NPT, nbn), acc);
    for (int tb = 0; tb < nbn; tb += NPT, ++tiles) {
      const int nn = min(NPT, nbn - tb);
      tc_store_A<K, T>(ar, A0, A1, A2);
#pragma unroll
      for (int i = 0; i < 2; ++i) tc::store_split8(D0, D1, D2, 4 * uj + a0 + (i ^ rot), c8 * 8, BN, acc[i]);
      tc::fence_async_smem();
      tc::before_sync();
      __syncthreads();
      tc::after_sync();
      const uint32_t tm = tslot;
      const bool more = tb + NPT < nbn;
      if (more) tc_load_A<K, RP, T>(a, tb + NPT, min(NPT, nbn - tb - NPT), s_aoff, ar);
      if (threadIdx.x == 0) {  // dG += A^T . dC   (accumulated over the group)
        const tc::Operand aT = tc::mnmajor(tc::smem_u32(A0), tc::smem_u32(A1), tc::smem_u32(A2), K);
        const tc::Operand dcB = tc::mnmajor(tc::smem_u32(D0), tc::smem_u32(D1), tc::smem_u32(D2), BN);
        tc::mma_x3<TC_BM / 16>(tm, aT, dcB, id_g, tiles > 0);
        tc::commit(&bar);
      } else if (threadIdx.x == 32) {  // dA = dC . S^T
        const tc::Operand dcK = tc::kmajor(tc::smem_u32(D0), tc::smem_u32(D1), tc::smem_u32(D2), BN);
        const tc::Operand sT = tc::kmajor(tc::smem_u32(S0), tc::smem_u32(S1), tc::smem_u32(S2), BN);
        tc::mma_x3<BN / 16>(tm + BN, dcK, sT, id_a, false);
        tc::commit(&bar);
      }
      __syncwarp();
      float* dst = emj < nn ? a.dPc + ((int64_t)s_node[tb + emj] * a.ncb + cb) * RP * K + ema * K + esl : nullptr;
      if (more) compute_dC(tb + NPT, min(NPT, nbn - tb - NPT), acc);
      tc::mbar_wait(&bar, phase);  // planes free for the next tile
      phase ^= 1;
      tc::after_sync();
      {
        float v[16];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          tc::tmem_ld16(tm + lane_base + BN + esl + 16 * h2, v);
          if (dst) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              *reinterpret_cast<float4*>(dst + 16 * h2 + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
        }
      }
      tc::before_sync();
    }
    tc::before_sync();
    __syncthreads();
  }
  // dG_F block: TMEM lane = k, column = n of the block
  tc::after_sync();
  {
    const uint32_t tm = tslot;
    const int k = 32 * (warp & 3) + lane, n0 = (warp >> 2) * 16;
    float* gdst = (a.split > 1 ? a.gsplit + ((int64_t)g * a.split + chunk) * a.c.slice[a.F]
                                : a.grads + a.c.core_off[a.F] + (int64_t)g * a.c.slice[a.F]) +
                  (int64_t)k * a.NC + cb * BN + n0;
    float v[16];
    tc::tmem_ld16(tm + lane_base + n0, v);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      *reinterpret_cast<float4*>(gdst + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
  tc::before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<256>(tslot);
}

// (RP, NL) instantiations of the rank-128 tensor backward (sweep128)
#define TT_TC128_SHAPES(X) X(4, 8)

// (K, BNf, RP, NL) instantiations of the tensor-core path
#define TT_TC_SHAPES(X) X(64, 128, 4, 4) X(32, 128, 4, 8) X(32, 128, 16, 4) X(64, 128, 4, 8)

inline bool tc_plan_shape(const FusedShape& f, TcShape* t) {
  *t = TcShape{};
  bool ok = false;
  if (f.K == 128) {  // FFMA forward + k_tc_bwd128 (64-column blocks)
#define TT_TC128_EQ(rp_, nl_) if (f.RP == rp_ && f.NL == nl_ && f.NC % 64 == 0) ok = true;
    TT_TC128_SHAPES(TT_TC128_EQ)
#undef TT_TC128_EQ
    if (!ok) return false;
    t->BNf = 0;
    t->ncbf = 0;
    t->BNb = 64;
    t->ncbb = f.NC / 64;
    t->smem_fwd = 0;
    t->smem_bwd = 3 * (size_t)128 * 64 * 2 + 3 * (size_t)TC_BM * 128 * 2 + 3 * (size_t)TC_BM * 64 * 2 + TC_META;
    t->ok = t->smem_bwd <= (size_t)FB_SMEM_MAX;
    return t->ok;
  }
#define TT_TC_EQ(k_, bn_, rp_, nl_) \
  if (f.K == k_ && f.RP == rp_ && f.NL == nl_ && f.NC % bn_ == 0 && f.NC % 128 == 0) ok = true;
  TT_TC_SHAPES(TT_TC_EQ)
#undef TT_TC_EQ
  if (!ok) return false;
  t->BNf = 128;
  t->ncbf = f.NC / 128;
  t->BNb = 128;
  t->ncbb = f.NC / 128;
  t->smem_fwd = tc_fwd_smem(f.K, 128);
  t->smem_bwd = tc_bwd_smem(f.K, 128);
  t->ok = t->smem_bwd <= (size_t)FB_SMEM_MAX;
  return t->ok;
}

}  // namespace tt
