// kernels_rows.cuh -- balanced row movement between batch positions and
// distinct IDs (HBM bound, fully coalesced 16-byte accesses).
//
// * k_dy_chunks / k_dy_spans: dY[u] = sum of the upstream rows at the ID's
//   batch positions, in ascending position order (the stable sort's slot
//   order) -- the duplicate additivity of backward_lookup
//   (autodiff.cpp:76-116).  The sorted slots are cut into fixed
//   32-slot chunks, one warp each, so a Zipf-hot ID with 10^4 positions is
//   spread over many warps instead of serialising one; segments crossing
//   chunk boundaries are finished by k_dy_spans in chunk order.  The
//   summation order depends only on the batch, never on scheduling.
// * k_scatter_heavy: copies the rows of IDs with many positions (deferred by
//   the forward epilogue) to every position, one thread per 16 bytes.
#pragma once
#include "common.cuh"

namespace tt {

constexpr int DY_CHUNK = 32;
constexpr int HEAVY_POS = 8;  // IDs with more positions are scattered by k_scatter_heavy

// uid1[s] = (distinct index of sorted slot s) + 1  (the inclusive unique scan);
// NV = ceil(npad / 128) float4 column groups per lane (1, 2 or 4)
template <int NV>
__global__ void __launch_bounds__(256) k_dy_chunks(const float* __restrict__ up, int B, int64_t emb, int64_t npad,
                                                   const int* __restrict__ uid1, const int* __restrict__ spos,
                                                   const int* __restrict__ seg, float* __restrict__ dY,
                                                   float* __restrict__ part, const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int lo = warp * DY_CHUNK;
  if (lo >= B) return;
  const int hi = min(lo + DY_CHUNK, B);
  const int my_s = lo + lane;
  const int my_u = my_s < hi ? uid1[my_s] - 1 : -1;
  const int my_p = my_s < hi ? spos[my_s] : 0;
  constexpr int nv = NV;
  float4 acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  int cur = __shfl_sync(0xffffffffu, my_u, 0);
  auto flush = [&](int u) {
    const int s0 = seg[u], s1 = seg[u + 1];
    float* dst;
    if (s0 >= lo && s1 <= hi) dst = dY + (int64_t)u * npad;
    else dst = part + ((int64_t)warp * 2 + (s0 < lo ? 0 : 1)) * npad;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int64_t c = (int64_t)v * 128 + lane * 4;
      if (v < nv && c < npad) *reinterpret_cast<float4*>(dst + c) = acc[v];
      acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  // rows are loaded PF at a time (independent 16-byte loads in flight), then
  // summed in slot order
  constexpr int PF = NV <= 2 ? 8 : 4;
  for (int i0 = 0; i0 < hi - lo; i0 += PF) {
    float4 x[PF][NV];
#pragma unroll
    for (int b = 0; b < PF; ++b) {
      const int p = __shfl_sync(0xffffffffu, my_p, (i0 + b) & 31);
      const float* row = up + (int64_t)p * emb;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int64_t c = (int64_t)v * 128 + lane * 4;
        if (i0 + b < hi - lo && v < nv && c < emb) x[b][v] = __ldg(reinterpret_cast<const float4*>(row + c));
      }
    }
#pragma unroll
    for (int b = 0; b < PF; ++b) {
      if (i0 + b >= hi - lo) break;
      const int u = __shfl_sync(0xffffffffu, my_u, i0 + b);
      if (u != cur) {
        flush(cur);
        cur = u;
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int64_t c = (int64_t)v * 128 + lane * 4;
        if (v < nv && c < emb) {
          acc[v].x += x[b][v].x; acc[v].y += x[b][v].y; acc[v].z += x[b][v].z; acc[v].w += x[b][v].w;
        }
      }
    }
  }
  flush(cur);
}

// Level 1 of the span reduction: warp per group of 32 chunks.  A chunk's
// head partial part[c][0] continues the ID of its first slot when that ID
// started in an earlier chunk; runs of equal IDs are summed in chunk order.
// A run holding all of an ID's continuation chunks completes dY[u] (tail
// partial of its first chunk + run); otherwise it is kept per group:
// gpart[G][0] if the ID's continuations began before the group, else
// gpart[G][1] (it continues after the group).
__global__ void __launch_bounds__(256) k_dy_groups(int B, int64_t npad, const int* __restrict__ uid1,
                                                   const int* __restrict__ seg, const float* __restrict__ part,
                                                   float* __restrict__ gpart, float* __restrict__ dY,
                                                   const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  const int G = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nchunks = (B + DY_CHUNK - 1) / DY_CHUNK;
  const int cbase = G * 32;
  if (cbase >= nchunks) return;
  const int my_c = cbase + lane;
  int my_u = -1;
  if (my_c < nchunks) {
    const int u = uid1[my_c * DY_CHUNK] - 1;
    if (seg[u] < my_c * DY_CHUNK) my_u = u;  // head partial continues u
  }
  const unsigned valid = __ballot_sync(0xffffffffu, my_u >= 0);
  if (!valid) return;
  const int nv = (int)((npad + 127) / 128);
  float4 acc[4];
  int cur = -1;
  // a run that holds all of u's continuation chunks is seeded with the tail
  // partial of u's first chunk (strict chunk order) and completes dY[u].
  // Per lane (chunk), the run facts of its ID are loaded in parallel before
  // the serial walk: whether a run here completes dY[u], whether u's
  // continuations began before this group, and u's first chunk.
  int my_first = 0, my_flags = 0;
  if (my_u >= 0) {
    const int c0 = seg[my_u] / DY_CHUNK, c1 = (seg[my_u + 1] - 1) / DY_CHUNK;
    my_first = c0;
    const bool complete = !(c0 + 1 < cbase) && !(c1 > cbase + 31);
    my_flags = (complete ? 1 : 0) | (c0 + 1 < cbase ? 2 : 0);
  }
  int cur_flags = 0;
  auto emit = [&](int u) {
    float* dst = (cur_flags & 1) ? dY + (int64_t)u * npad : gpart + ((int64_t)G * 2 + ((cur_flags & 2) ? 0 : 1)) * npad;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t c = (int64_t)v * 128 + lane * 4;
      if (v < nv && c < npad) *reinterpret_cast<float4*>(dst + c) = acc[v];
    }
  };
  for (int i = 0; i < 32; ++i) {
    const int u = __shfl_sync(0xffffffffu, my_u, i);
    const int fl = __shfl_sync(0xffffffffu, my_flags, i), first = __shfl_sync(0xffffffffu, my_first, i);
    if (u != cur) {
      if (cur >= 0) emit(cur);
      cur = u;
      cur_flags = fl;
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (u >= 0 && (fl & 1)) {
        const float* head = part + ((int64_t)first * 2 + 1) * npad;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int64_t c = (int64_t)v * 128 + lane * 4;
          if (v < nv && c < npad) acc[v] = *reinterpret_cast<const float4*>(head + c);
        }
      }
    }
    if (u < 0) continue;
    const float* src = part + ((int64_t)(cbase + i) * 2) * npad;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t c = (int64_t)v * 128 + lane * 4;
      if (v < nv && c < npad) {
        const float4 x = *reinterpret_cast<const float4*>(src + c);
        acc[v].x += x.x; acc[v].y += x.y; acc[v].z += x.z; acc[v].w += x.w;
      }
    }
  }
  if (cur >= 0) emit(cur);
}

// Level 2: IDs whose continuation chunks cross group boundaries:
// dY[u] = tail(c0) + gpart[G0][1] + sum_{G0<G<G1} gpart[G][0] + gpart[G1][0].
__global__ void __launch_bounds__(256) k_dy_spans(const int* __restrict__ counts, int d, int64_t npad,
                                                  const int* __restrict__ seg, const float* __restrict__ part,
                                                  const float* __restrict__ gpart, float* __restrict__ dY,
                                                  const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  const int U = ld_count(&counts[d - 1]);
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  // each lane tests one ID (32 per step); the warp then finishes the IDs
  // that span several chunk groups, in lane order
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int ub = warp * 32; ub < U; ub += nwarps * 32) {
    const int mu = ub + lane;
    int mc0 = 0, mc1 = 0;
    if (mu < U) {
      mc0 = seg[mu] / DY_CHUNK;
      mc1 = (seg[mu + 1] - 1) / DY_CHUNK;
    }
    // k_dy_groups completes IDs within one chunk or one group
    unsigned todo = __ballot_sync(0xffffffffu, mu < U && mc0 != mc1 && (mc0 + 1) / 32 != mc1 / 32);
    while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const int u = ub + src;
    const int c0 = __shfl_sync(0xffffffffu, mc0, src), c1 = __shfl_sync(0xffffffffu, mc1, src);
    const int G0 = (c0 + 1) / 32, G1 = c1 / 32;
    for (int64_t c = lane * 4; c < npad; c += 128) {
      float4 acc = *reinterpret_cast<const float4*>(part + ((int64_t)c0 * 2 + 1) * npad + c);
      float4 x = *reinterpret_cast<const float4*>(gpart + ((int64_t)G0 * 2 + 1) * npad + c);
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      for (int g = G0 + 1; g <= G1; ++g) {
        x = *reinterpret_cast<const float4*>(gpart + ((int64_t)g * 2) * npad + c);
        acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      }
      *reinterpret_cast<float4*>(dY + (int64_t)u * npad + c) = acc;
    }
    }
  }
}

// out[pos] = Yu[u] for the slots of heavy IDs (more than HEAVY_POS positions).
// Warp per 32 sorted slots: the lanes look up their slot's ID, segment and
// position in parallel, then the warp copies the ID's row (loaded once per run
// of equal IDs; a heavy ID's slots are contiguous) to each heavy slot's
// position, 16 bytes per lane.
__global__ void __launch_bounds__(256) k_scatter_heavy(int B, int64_t emb, int64_t npad, const int* __restrict__ uid1,
                                                       const int* __restrict__ spos, const int* __restrict__ seg,
                                                       const float* __restrict__ Yu, float* __restrict__ out,
                                                       const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nv = (int)((emb + 127) / 128);  // float4 column groups per lane (emb <= 512)
  for (int base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < B; base += nwarps * 32) {
    const int s = base + lane;
    int u = -1, pos = 0;
    if (s < B) {
      u = uid1[s] - 1;
      if (seg[u + 1] - seg[u] > HEAVY_POS) pos = spos[s];
      else u = -1;
    }
    unsigned todo = __ballot_sync(0xffffffffu, u >= 0);
    int cu = -1;
    float4 row[4];
    while (todo) {
      const int i = __ffs(todo) - 1;
      todo &= todo - 1;
      const int uu = __shfl_sync(0xffffffffu, u, i), p = __shfl_sync(0xffffffffu, pos, i);
      if (uu != cu) {
        cu = uu;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int64_t c = (int64_t)v * 128 + lane * 4;
          if (v < nv && c < emb) row[v] = *reinterpret_cast<const float4*>(Yu + (int64_t)uu * npad + c);
        }
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int64_t c = (int64_t)v * 128 + lane * 4;
        if (v < nv && c < emb) *reinterpret_cast<float4*>(out + (int64_t)p * emb + c) = row[v];
      }
    }
  }
}

}  // namespace tt
