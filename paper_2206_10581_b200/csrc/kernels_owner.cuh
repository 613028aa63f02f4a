// kernels_owner.cuh -- device side of ID-owner sharding (the
// scheme that keeps cross-GPU dedupe): rank r of P owns the level-F digits
// [floor(m_F r / P), floor(m_F (r+1) / P)) -- and with them every ID, every
// level-F prefix and every G_F slice with such a digit.  Each rank buckets its
// position shard's IDs by owner (a stable radix sort on the owner rank), the
// engine's NCCL communicator moves IDs / rows between ranks (engine.cu,
// tt_owner_*), and these kernels gather and scatter the rows.
#pragma once
#include "common.cuh"

namespace tt {

// owner rank of every local ID (and range validation against num_nodes, the
// minimum bad position recorded as in k_decompose_validate); invalid IDs are
// routed to the local rank (the batch fails as a whole anyway)
__global__ void k_owner_of(const int64_t* __restrict__ idx, int64_t B, DevCfg c, int F, int P, int self,
                           unsigned* __restrict__ owner, int* __restrict__ pos, DevStatus* st) {
  TT_PDL_ENTRY();
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int64_t id = idx[b];
  const bool bad = id < 0 || id >= c.num_nodes;
  const unsigned ballot = __ballot_sync(__activemask(), bad);
  if (ballot && bad && (ballot & lanemask_lt()) == 0) atomicMin(&st->bad_pos, (unsigned long long)b);
  unsigned o = (unsigned)self;
  if (!bad) {
    const int64_t digit = (id / c.S[F]) % c.m[F];
    o = (unsigned)(((digit + 1) * P - 1) / c.m[F]);
  }
  owner[b] = o;
  pos[b] = (int)b;
}

// counts[r] = number of sorted owner keys equal to r (P small: one thread per rank)
__global__ void k_owner_counts(const unsigned* __restrict__ sorted_owner, int B, int P, int* __restrict__ counts) {
  TT_PDL_ENTRY();
  const int r = threadIdx.x;
  if (r >= P) return;
  auto lower = [&](unsigned v) {
    int lo = 0, hi = B;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sorted_owner[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  counts[r] = lower((unsigned)r + 1) - lower((unsigned)r);
}

// dst[i] = src[perm[i]] for i < n (IDs into owner order)
__global__ void k_gather_ids(const int64_t* __restrict__ src, const int* __restrict__ perm, int n,
                             int64_t* __restrict__ dst) {
  TT_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}

// rows (N floats, N % 4 == 0): gather dst[i] = src[perm[i]] or scatter
// dst[perm[i]] = src[i]; one warp per row
template <bool SCATTER>
__global__ void k_permute_rows(const float* __restrict__ src, const int* __restrict__ perm, int n, int64_t N,
                               float* __restrict__ dst) {
  TT_PDL_ENTRY();
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w; i < n; i += nw) {
    const int64_t p = perm[i];
    const float4* s = reinterpret_cast<const float4*>(src + (SCATTER ? i : p) * N);
    float4* d = reinterpret_cast<float4*>(dst + (SCATTER ? p : i) * N);
    for (int64_t q = lane; q < N / 4; q += 32) d[q] = s[q];
  }
}

}  // namespace tt
