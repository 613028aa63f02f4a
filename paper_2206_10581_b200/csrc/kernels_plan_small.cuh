// kernels_plan_small.cuh -- the whole K1 + K2 plan in ONE CTA for small
// batches (B <= PS_MAXB).  The multi-kernel plan (kernels_plan.cuh) is ~19
// dependent launches; for a few thousand IDs each launch is mostly latency
// (~4 us inside a CUDA graph), so at small (B = 4,096) the plan was half of the
// training step.  Here one 1024-thread CTA validates, sorts, uniques and builds
// every level in shared memory, with __syncthreads between phases, and writes
// exactly the buffers the multi-kernel plan writes (the fused kernels cannot
// tell the two apart; tests/test_gpu_parity.py checks the plan bit-exactly):
//   skeys / spos (stable sort by ID, ties by position), flag (inclusive unique
//   scan), uniq / seg, counts, per level digit / parent / first / cstart, the
//   per-level digit order (stable by node) and group offsets.
// Sorting: stable LSD radix sort of packed 64-bit values (key << 13 | index)
// on the key bits, 8-bit digits; each warp owns a contiguous segment, ranks
// its 32-value chunks in order with __match_any_sync, and scatters through
// per-(digit, warp) offsets from a block-wide scan -- stable by construction.
#pragma once
#include "common.cuh"

namespace tt {

constexpr int PS_THREADS = 1024, PS_WARPS = PS_THREADS / 32, PS_MAXB = 8192, PS_IBITS = 13;
constexpr int PS_DBITS = 9, PS_NB = 1 << PS_DBITS;  // radix digits of up to 9 bits (18-bit IDs: 2 passes)
constexpr unsigned long long PS_IMASK = (1ull << PS_IBITS) - 1;
// dynamic shared memory: two value buffers + the (digit, warp) offset table
// (reused as the levels' first-ID tables) + bucket starts + scan scratch
constexpr size_t PS_SMEM = sizeof(unsigned long long) * 2 * PS_MAXB + sizeof(int) * (PS_WARPS * PS_NB + PS_NB + 64);

struct PlanSmallArgs {
  DevCfg c;
  const int64_t* idx;
  int B;
  const int* perm;
  int idbits;
  int64_t cap;
  unsigned long long* skeys;
  int* spos;
  int* flag;
  unsigned long long* uniq;
  int* seg;
  int* counts;  // [TT_MAXD] + counts[TT_MAXD] = B
  int* digit;
  int* parent;
  int* first;
  int* cstart;
  unsigned* sdig[TT_MAXD];
  int* order[TT_MAXD];
  int* goff[TT_MAXD];
  DevStatus* st;
  long long* dbg;  // TT_PS_TRACE=1: clock64 at the end of each phase (thread 0), else nullptr
};

// exclusive block scan of one int per thread (1024 threads); total in *tot
__device__ __forceinline__ int ps_block_excl(int v, int* wsum, int* tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    wsum[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const int excl = x - v + (warp ? wsum[warp - 1] : 0);
  if (threadIdx.x == PS_THREADS - 1) *tot = excl + v;
  __syncthreads();
  return excl;
}

// stable LSD sort of a[0, n) on bits [lo, hi) of the values; returns the buffer
// holding the result (a or b)
// (bits per pass: PS_DBITS; a sort of at most PS_DBITS bits is one pass, and
// then bstart[d] = the first output slot of digit d, if bstart is given)
__device__ unsigned long long* ps_sort(unsigned long long* a, unsigned long long* b, int n, int lo, int hi, int* H,
                                       int* wsum, int* tot, int* bstart = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int segn = (n + PS_WARPS - 1) / PS_WARPS;
  const int s0 = min(n, warp * segn), s1 = min(n, s0 + segn);
  constexpr int EPT = PS_WARPS * PS_NB / PS_THREADS;  // offset-table entries per thread
  for (int shift = lo; shift < hi; shift += PS_DBITS) {
    const int bits = min(PS_DBITS, hi - shift);
    const unsigned long long dm = (1ull << bits) - 1;
    for (int i = threadIdx.x; i < PS_WARPS * PS_NB; i += PS_THREADS) H[i] = 0;
    __syncthreads();
    for (int i = s0 + lane; i < s1; i += 32) atomicAdd(&H[warp * PS_NB + (int)((a[i] >> shift) & dm)], 1);
    __syncthreads();
    // offsets in (digit, warp) order: entry e = d * 32 + w, EPT entries per thread
    int v[EPT], t = 0;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int e = threadIdx.x * EPT + j, d = e >> 5, w = e & 31;
      v[j] = H[w * PS_NB + d];
      t += v[j];
    }
    int run = ps_block_excl(t, wsum, tot);
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int e = threadIdx.x * EPT + j, d = e >> 5, w = e & 31;
      H[w * PS_NB + d] = run;
      if (bstart && w == 0) bstart[d] = run;
      run += v[j];
    }
    __syncthreads();
    for (int c0 = s0; c0 < s1; c0 += 32) {
      const int i = c0 + lane;
      const bool ok = i < s1;
      const unsigned long long x = ok ? a[i] : 0ull;
      const int d = ok ? (int)((x >> shift) & dm) : PS_NB + lane;  // invalid lanes match nobody
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const int rank = __popc(peers & lanemask_lt());
      const int off = ok ? H[warp * PS_NB + d] : 0;
      __syncwarp();
      if (ok) {
        b[off + rank] = x;
        if (rank == 0) H[warp * PS_NB + d] = off + __popc(peers);
      }
      __syncwarp();
    }
    __syncthreads();
    unsigned long long* tmp = a;
    a = b;
    b = tmp;
  }
  return a;
}

// inclusive scan of flags f(i), i < n, 8 contiguous items per thread (n <= 8192);
// out[i] = inclusive count; returns the total
template <class Flag>
__device__ __forceinline__ int ps_scan_flags(int n, Flag f, int* out, int* wsum, int* tot) {
  const int i0 = threadIdx.x * 8;
  int fl[8], t = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    fl[j] = (i0 + j < n) ? f(i0 + j) : 0;
    t += fl[j];
  }
  int run = ps_block_excl(t, wsum, tot);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    run += fl[j];
    if (i0 + j < n) out[i0 + j] = run;
  }
  __syncthreads();
  return *tot;
}

__global__ void __launch_bounds__(PS_THREADS, 1) k_plan_small(PlanSmallArgs p) {
  TT_PDL_ENTRY();
  extern __shared__ __align__(16) unsigned long long ps_smem[];
  unsigned long long* A = ps_smem;
  unsigned long long* Bf = A + PS_MAXB;
  int* H = reinterpret_cast<int*>(Bf + PS_MAXB);
  int* bst = H + PS_WARPS * PS_NB;  // [PS_NB] bucket starts of a one-pass sort
  int* wsum = bst + PS_NB;
  int* tot = wsum + 40;
  const DevCfg& c = p.c;
  const int d = c.d, B = p.B;
  const int64_t cap = p.cap;
  int nmark = 0;
  auto mark = [&]() {
    if (p.dbg && threadIdx.x == 0) p.dbg[nmark] = clock64();
    ++nmark;
  };
  mark();

  // K1: validate, key = (relabelled) id, packed with the position
  for (int b = threadIdx.x; b < B; b += PS_THREADS) {
    const int64_t id = p.idx[b];
    const bool bad = id < 0 || id >= c.num_nodes;
    if (bad) atomicMin(&p.st->bad_pos, (unsigned long long)b);
    const unsigned long long key = bad ? 0ull : (unsigned long long)(p.perm ? (int64_t)__ldg(p.perm + id) : id);
    A[b] = (key << PS_IBITS) | (unsigned long long)b;
  }
  if (threadIdx.x == 0) p.counts[TT_MAXD] = B;
  __syncthreads();
  if (*(volatile unsigned long long*)&p.st->bad_pos != TT_NO_POS) {  // the batch fails as a whole
    if (threadIdx.x < d) p.counts[threadIdx.x] = 0;
    return;
  }
  mark();  // 1: validate
  // K2: stable sort by id, ties by position
  unsigned long long* S = ps_sort(A, Bf, B, PS_IBITS, PS_IBITS + p.idbits, H, wsum, tot);
  mark();  // 2: sort
  for (int s = threadIdx.x; s < B; s += PS_THREADS) {
    p.skeys[s] = S[s] >> PS_IBITS;
    p.spos[s] = (int)(S[s] & PS_IMASK);
  }
  __syncthreads();
  // unique IDs: flag = inclusive scan of "key differs from the previous slot"
  const int U = ps_scan_flags(
      B, [&](int s) { return (s == 0 || (S[s] >> PS_IBITS) != (S[s - 1] >> PS_IBITS)) ? 1 : 0; }, p.flag, wsum, tot);
  for (int s = threadIdx.x; s < B; s += PS_THREADS) {
    if (s == 0 || (S[s] >> PS_IBITS) != (S[s - 1] >> PS_IBITS)) {
      const int u = p.flag[s] - 1;
      p.uniq[u] = S[s] >> PS_IBITS;
      p.seg[u] = s;
    }
  }
  if (threadIdx.x == 0) {
    p.counts[d - 1] = U;
    p.seg[U] = B;
  }
  __syncthreads();
  mark();  // 3: sorted keys out, unique
  // levels 0..d-2: prefix flags over the distinct IDs (scans in the sort
  // buffers, which are free now: level k in Lc, level k-1 in Lp; the IDs'
  // level-k prefixes in Q, 32-bit when the IDs fit)
  int* Lp = reinterpret_cast<int*>(A);
  int* Lc = Lp + PS_MAXB;
  unsigned long long* Q = Bf;  // [U] level-k prefix of every distinct ID
  // first distinct ID of every node of levels k - 1 and k (the sort table is
  // free here): cstart without a round trip through p.first
  int* Fp = H;
  int* Fc = H + PS_MAXB;
  const bool id32 = c.num_nodes <= 0xFFFFFFFFll;
  for (int k = 0; k + 1 < d; ++k) {
    const unsigned long long Sk = (unsigned long long)c.S[k];
    for (int u = threadIdx.x; u < U; u += PS_THREADS)
      Q[u] = id32 ? (unsigned long long)((unsigned)p.uniq[u] / (unsigned)Sk) : p.uniq[u] / Sk;
    __syncthreads();
    const int nk = ps_scan_flags(
        U, [&](int u) { return (u == 0 || Q[u] != Q[u - 1]) ? 1 : 0; }, Lc, wsum, tot);
    for (int u = threadIdx.x; u < U; u += PS_THREADS) {
      const unsigned long long q = Q[u];
      if (u == 0 || q != Q[u - 1]) {
        const int node = Lc[u] - 1;
        const int dg = id32 ? (int)((unsigned)q % (unsigned)c.m[k]) : (int)(q % (unsigned long long)c.m[k]);
        p.digit[k * cap + node] = dg;
        p.first[k * cap + node] = u;
        Fc[node] = u;
        p.parent[k * cap + node] = k ? Lp[u] - 1 : -1;
        if (k == 0) {
          p.order[0][node] = node;
          p.sdig[0][node] = (unsigned)dg;
          // level 0 is in digit order: goff[0][v] = first node with digit >= v
          const int prev = u == 0 ? -1 : (int)(id32 ? (unsigned)Q[u - 1] % (unsigned)c.m[0] : Q[u - 1] % (unsigned long long)c.m[0]);
          for (int v = prev + 1; v <= dg; ++v) p.goff[0][v] = node;
        }
      }
    }
    if (threadIdx.x == 0) p.counts[k] = nk;
    if (k == 0 && threadIdx.x < 32) {  // digits past the last node's: goff = n_0
      const int last = id32 ? (int)((unsigned)Q[U - 1] % (unsigned)c.m[0]) : (int)(Q[U - 1] % (unsigned long long)c.m[0]);
      for (int v = last + 1 + threadIdx.x; v <= c.m[0]; v += 32) p.goff[0][v] = nk;
    }
    __syncthreads();
    if (k >= 1) {  // children of level k-1: the level-k node of each one's first ID
      const int np = p.counts[k - 1];
      for (int n = threadIdx.x; n <= np; n += PS_THREADS)
        p.cstart[(k - 1) * (cap + 1) + n] = n == np ? nk : Lc[Fp[n]] - 1;
    }
    __syncthreads();
    int* t = Lp;
    Lp = Lc;
    Lc = t;
    t = Fp;
    Fp = Fc;
    Fc = t;
  }
  mark();  // 4: prefix levels
  {  // the last level: the distinct IDs themselves
    const int k = d - 1;
    for (int u = threadIdx.x; u < U; u += PS_THREADS) {
      p.digit[k * cap + u] = id32 ? (int)((unsigned)p.uniq[u] % (unsigned)c.m[k]) : (int)(p.uniq[u] % (unsigned long long)c.m[k]);
      p.first[k * cap + u] = u;
      p.parent[k * cap + u] = Lp[u] - 1;
    }
    const int np = p.counts[k - 1];
    for (int n = threadIdx.x; n <= np; n += PS_THREADS)
      p.cstart[(k - 1) * (cap + 1) + n] = n == np ? U : p.first[(k - 1) * cap + n];
  }
  __syncthreads();
  mark();  // 5: last level
  // per-level digit order (stable by node index) for levels 1..d-1: one
  // one-pass sort over all levels at once on (level, digit) when the nodes fit
  // the buffer and the key fits one radix digit; its bucket starts are the
  // group offsets
  int tot_nodes = 0, dmax = 1;
  for (int k = 1; k < d; ++k) {
    tot_nodes += p.counts[k];
    while ((1ll << dmax) < c.m[k]) ++dmax;
  }
  int lbits = 0;
  while ((1 << lbits) < d - 1) ++lbits;
  if (tot_nodes <= PS_MAXB && dmax + lbits <= PS_DBITS) {
    int off = 0;
    for (int k = 1; k < d; ++k) {
      const int nk = p.counts[k];
      for (int n = threadIdx.x; n < nk; n += PS_THREADS)
        A[off + n] = (((unsigned long long)(k - 1) << dmax | (unsigned long long)p.digit[k * cap + n]) << PS_IBITS) |
                     (unsigned long long)n;
      off += nk;
    }
    __syncthreads();
    unsigned long long* O = ps_sort(A, Bf, tot_nodes, PS_IBITS, PS_IBITS + dmax + lbits, H, wsum, tot, bst);
    off = 0;
    for (int k = 1; k < d; ++k) {
      const int nk = p.counts[k];
      const unsigned dmask = (1u << dmax) - 1;
      for (int n = threadIdx.x; n < nk; n += PS_THREADS) {
        const unsigned long long x = O[off + n];
        p.sdig[k][n] = (unsigned)(x >> PS_IBITS) & dmask;
        p.order[k][n] = (int)(x & PS_IMASK);
      }
      for (int v = threadIdx.x; v <= c.m[k]; v += PS_THREADS)
        p.goff[k][v] = v == c.m[k] ? nk : bst[((k - 1) << dmax) | v] - off;
      off += nk;
    }
    __syncthreads();
    mark();  // 6: digit orders + group offsets
    mark();  // 7
    if (p.dbg && threadIdx.x == 0) p.dbg[15] = nmark;
    return;
  }
  for (int k = 1; k < d; ++k) {
    const int nk = p.counts[k];
    int dbits = 1;
    while ((1ll << dbits) < c.m[k]) ++dbits;
    for (int n = threadIdx.x; n < nk; n += PS_THREADS)
      A[n] = ((unsigned long long)p.digit[k * cap + n] << PS_IBITS) | (unsigned long long)n;
    __syncthreads();
    unsigned long long* O = ps_sort(A, Bf, nk, PS_IBITS, PS_IBITS + dbits, H, wsum, tot);
    for (int n = threadIdx.x; n < nk; n += PS_THREADS) {
      p.sdig[k][n] = (unsigned)(O[n] >> PS_IBITS);
      p.order[k][n] = (int)(O[n] & PS_IMASK);
    }
    __syncthreads();
  }
  mark();  // 6: digit orders
  // group offsets: goff[k][v] = first slot whose sorted digit >= v
  for (int k = 0; k < d; ++k) {
    const int nk = p.counts[k];
    const unsigned* sd = p.sdig[k];
    for (int v = threadIdx.x; v <= c.m[k]; v += PS_THREADS) {
      int lo = 0, hi = nk;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((int)sd[mid] < v) lo = mid + 1; else hi = mid;
      }
      p.goff[k][v] = lo;
    }
  }
  __syncthreads();
  mark();  // 7: group offsets
  if (p.dbg && threadIdx.x == 0) p.dbg[15] = nmark;
}

}  // namespace tt
