// kernels_plan.cuh -- K1 (decompose + validate) and K2 (radix sort, unique,
// prefix levels, digit groups).  Integer work: HBM/latency bound, no tensor
// cores.  Every count that depends on the batch's content stays on the
// device; grids are sized by host-known upper bounds and kernels read the
// live count, so the whole plan is stream-ordered (graph-capturable) with no
// host round trip.
#pragma once
#include "common.cuh"

namespace tt {

// ---------------------------------------------------------------------------
// K1: validate every index (tt_embedding.cpp:112-117, autodiff.cpp:57-60) and
// emit (key, position) pairs.  The minimum offending position is recorded
// (the reference reports the first in input order).
// perm (optional): the node relabelling of a hierarchical reorder
// (graph.cpp:218-252 apply_permutation): row perm[id] serves id.  Validation
// is on the caller's id.
__global__ void k_decompose_validate(const int64_t* __restrict__ idx, int64_t B, int64_t num_nodes,
                                     unsigned long long* __restrict__ keys, int* __restrict__ pos,
                                     DevStatus* st, const int* __restrict__ perm, int* __restrict__ nB) {
  TT_PDL_ENTRY();
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b == 0) *nB = (int)B;  // the batch size as a device count
  if (b >= B) return;
  int64_t id = idx[b];
  bool bad = id < 0 || id >= num_nodes;
  unsigned ballot = __ballot_sync(__activemask(), bad);
  if (ballot) {
    // lowest bad lane of the warp reports: one atomic per warp
    if (bad && (ballot & lanemask_lt()) == 0) atomicMin(&st->bad_pos, (unsigned long long)b);
  }
  keys[b] = bad ? 0ull : (unsigned long long)(perm ? (int64_t)__ldg(perm + id) : id);
  pos[b] = (int)b;
}

// ---------------------------------------------------------------------------
// Stable LSD radix sort of (key, int value) pairs, up to 11-bit digits per
// pass and three kernels per pass: per-tile digit histograms; a column scan
// (one thread per digit) turning them into per-tile exclusive offsets plus
// digit totals; a scatter whose blocks scan the digit totals, rank their keys
// stably with warp match_any peers and write.  Counts stay on the device.
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_PER_WARP = 128;
constexpr int RS_TILE = RS_WARPS * RS_PER_WARP;  // 1024 keys per tile (>= 148 tiles at B = 256k)
constexpr int RS_MAXBITS = 11;
constexpr int RS_MAXBINS = 1 << RS_MAXBITS;
constexpr size_t RS_SCATTER_SMEM = sizeof(int) * ((size_t)RS_WARPS * RS_MAXBINS + RS_MAXBINS + 64);

__device__ __forceinline__ int rs_count(const int* n_dev, int n_host) { return n_dev ? ld_count(n_dev) : n_host; }

// One launch sorts up to TT_MAXD independent arrays (blockIdx.y selects the
// array): the ID sort uses one, the per-level digit sorts of the plan run
// batched in a single pass.
template <class K>
struct RSBatch {
  const K* kin[TT_MAXD];
  const int* vin[TT_MAXD];  // nullptr: the value is the key's index
  K* kout[TT_MAXD];
  int* vout[TT_MAXD];
  const int* n_dev[TT_MAXD];
  int* hist[TT_MAXD];       // [tiles][bins] per-tile histograms -> exclusive column prefixes
  int* tot[TT_MAXD];        // [bins] digit totals
  int n_host;
};

// per-tile digit histogram -> hist[tile * bins + digit]
template <class K>
__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(RSBatch<K> rb, int shift, int nbits) {
  TT_PDL_ENTRY();
  __shared__ int cnt[RS_MAXBINS];
  const int y = blockIdx.y;
  const K* __restrict__ keys = rb.kin[y];
  int* __restrict__ hist = rb.hist[y];
  const int n = rs_count(rb.n_dev[y], rb.n_host);
  const int base = blockIdx.x * RS_TILE;
  if (base >= n) return;
  const int bins = 1 << nbits;
  const unsigned mask = bins - 1;
  for (int i = threadIdx.x; i < bins; i += RS_THREADS) cnt[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < RS_TILE; i += RS_THREADS) {
    const int g = base + i;
    if (g < n) atomicAdd(&cnt[(int)((keys[g] >> shift) & mask)], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bins; i += RS_THREADS) hist[blockIdx.x * bins + i] = cnt[i];
}

// hist[t][d] <- sum_{t' < t} hist[t'][d];  tot[d] = sum_t hist[t][d].
// A block owns 32 digits (lanes) x 8 tile segments (warps): each thread sums
// its segment with independent loads, the 8 segment totals are scanned in
// shared memory, then each thread rewrites its segment as prefixes.
constexpr int RS_CS_SEG = 8;
template <class K>
__global__ void __launch_bounds__(32 * RS_CS_SEG) k_rs_colscan(RSBatch<K> rb, int nbits) {
  TT_PDL_ENTRY();
  __shared__ int part[RS_CS_SEG][33];
  int* __restrict__ hist = rb.hist[blockIdx.y];
  int* __restrict__ tot = rb.tot[blockIdx.y];
  const int* n_dev = rb.n_dev[blockIdx.y];
  const int n_host = rb.n_host;
  const int bins = 1 << nbits;
  const int lane = threadIdx.x & 31, seg = threadIdx.x >> 5;
  const int dgt = blockIdx.x * 32 + lane;
  const int n = rs_count(n_dev, n_host);
  const int ntiles = (n + RS_TILE - 1) / RS_TILE;
  const int per = (ntiles + RS_CS_SEG - 1) / RS_CS_SEG;
  const int t0 = min(ntiles, seg * per), t1 = min(ntiles, t0 + per);
  int sum = 0;
  if (dgt < bins) {
    int t = t0;
    for (; t + 8 <= t1; t += 8) {
      int h[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) h[i] = hist[(t + i) * bins + dgt];
#pragma unroll
      for (int i = 0; i < 8; ++i) sum += h[i];
    }
    for (; t < t1; ++t) sum += hist[t * bins + dgt];
  }
  part[seg][lane] = sum;
  __syncthreads();
  int run = 0;
  for (int q = 0; q < seg; ++q) run += part[q][lane];
  if (dgt >= bins) return;
  int t = t0;
  for (; t + 8 <= t1; t += 8) {
    int h[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = hist[(t + i) * bins + dgt];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      hist[(t + i) * bins + dgt] = run;
      run += h[i];
    }
  }
  for (; t < t1; ++t) {
    const int h = hist[t * bins + dgt];
    hist[t * bins + dgt] = run;
    run += h;
  }
  if (seg == RS_CS_SEG - 1) tot[dgt] = run;
}

template <class K>
__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(RSBatch<K> rb, int shift, int nbits) {
  TT_PDL_ENTRY();
  const int y = blockIdx.y;
  const K* __restrict__ kin = rb.kin[y];
  const int* __restrict__ vin = rb.vin[y];
  K* __restrict__ kout = rb.kout[y];
  int* __restrict__ vout = rb.vout[y];
  const int* n_dev = rb.n_dev[y];
  const int n_host = rb.n_host;
  const int* __restrict__ colpre = rb.hist[y];
  const int* __restrict__ tot = rb.tot[y];
  extern __shared__ int rs_smem[];
  int* cnt = rs_smem;                            // [RS_WARPS][bins]
  const int bins = 1 << nbits;
  int* base = cnt + RS_WARPS * bins;             // [bins]
  int* wsum = base + bins;                       // [RS_WARPS]
  const int n = rs_count(n_dev, n_host);
  const int tile = blockIdx.x;
  if (tile * RS_TILE >= n) return;
  const unsigned mask = bins - 1;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // exclusive scan of the digit totals, plus this tile's column prefix
  constexpr int DPT = RS_MAXBINS / RS_THREADS;  // digits per thread (<= 8)
  int tv[DPT];
  int my = 0;
#pragma unroll
  for (int q = 0; q < DPT; ++q) {
    const int dgt = threadIdx.x * DPT + q;
    tv[q] = dgt < bins ? tot[dgt] : 0;
    my += tv[q];
  }
  int x = my;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  for (int i = threadIdx.x; i < RS_WARPS * bins; i += RS_THREADS) cnt[i] = 0;
  __syncthreads();
  int run = x - my;
  for (int i = 0; i < w; ++i) run += wsum[i];
#pragma unroll
  for (int q = 0; q < DPT; ++q) {
    const int dgt = threadIdx.x * DPT + q;
    if (dgt < bins) base[dgt] = run + colpre[tile * bins + dgt];
    run += tv[q];
  }
  // per-warp digit counts of this tile
  const int wbase = tile * RS_TILE + w * RS_PER_WARP;
  for (int r = 0; r < RS_PER_WARP / 32; ++r) {
    const int g = wbase + r * 32 + lane;
    const int dig = g < n ? (int)((kin[g] >> shift) & mask) : RS_MAXBINS + lane;
    const unsigned peers = __match_any_sync(0xffffffffu, dig);
    if (g < n && lane == 31 - __clz(peers)) cnt[w * bins + dig] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int dgt = threadIdx.x; dgt < bins; dgt += RS_THREADS) {
    int rr = base[dgt];
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ++ww) {
      const int c = cnt[ww * bins + dgt];
      cnt[ww * bins + dgt] = rr;
      rr += c;
    }
  }
  __syncthreads();
  for (int r = 0; r < RS_PER_WARP / 32; ++r) {
    const int g = wbase + r * 32 + lane;
    const K key = g < n ? kin[g] : (K)0;
    const int dig = g < n ? (int)((key >> shift) & mask) : RS_MAXBINS + lane;
    const unsigned peers = __match_any_sync(0xffffffffu, dig);
    if (g < n) {
      const int dst = cnt[w * bins + dig] + __popc(peers & lanemask_lt());
      kout[dst] = key;
      vout[dst] = vin ? vin[g] : g;
    }
    __syncwarp();
    if (g < n && lane == 31 - __clz(peers)) cnt[w * bins + dig] += __popc(peers);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// In-place inclusive scan of `narr` int arrays (stride apart) whose live
// length is *n_dev.  Three phases: per-block scan, scan of block totals,
// add-back.
constexpr int SC_THREADS = 256;
constexpr int SC_ITEMS = 8;
constexpr int SC_BLOCK = SC_THREADS * SC_ITEMS;

__device__ __forceinline__ int block_excl_scan_256(int t, int* wsum, int& total) {
  int x = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane_id() >= (unsigned)o) x += y;
  }
  if (lane_id() == 31) wsum[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    int w = threadIdx.x < SC_THREADS / 32 ? wsum[threadIdx.x] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane_id() >= (unsigned)o) w += y;
    }
    if (threadIdx.x < SC_THREADS / 32) wsum[threadIdx.x] = w;
  }
  __syncthreads();
  total = wsum[SC_THREADS / 32 - 1];
  int r = (x - t) + ((threadIdx.x >> 5) ? wsum[(threadIdx.x >> 5) - 1] : 0);
  __syncthreads();
  return r;
}

// Values to scan: read from the array (keys == nullptr), or group-start flags
// formed here from sorted keys -- 1 where keys[s] / div[y] changes (array y):
// div 1 gives the unique-ID flags, div S_k the level-k prefix flags.
struct ScanFlags {
  const unsigned long long* keys;
  unsigned long long div[TT_MAXD];
};

// Single-pass inclusive scan (chained scan with decoupled look-back): block
// tickets in launch order, each block publishes its aggregate (state 1) and,
// once its prefix is known, its inclusive prefix (state 2) in a 64-bit status
// word; a block walks back over its predecessors' words until it meets an
// inclusive prefix.  status[narr][nblk] and ticket[narr] are zeroed before
// the launch.  Blocks only wait on lower tickets, which belong to blocks
// already running, so the scan cannot deadlock.
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_onepass(int* __restrict__ a, int64_t stride, const int* n_dev,
                                                             unsigned long long* __restrict__ status,
                                                             unsigned long long* __restrict__ ticket, int nblk,
                                                             ScanFlags sf) {
  TT_PDL_ENTRY();
  __shared__ int wsum[SC_THREADS / 32];
  __shared__ int s_blk, s_prefix;
  if (threadIdx.x == 0) s_blk = (int)atomicAdd(ticket + blockIdx.y, 1ull);
  __syncthreads();
  const int blk = s_blk;
  const int n = ld_count(n_dev);
  if (blk * SC_BLOCK >= n) return;  // later tickets are past n as well
  int* arr = a + blockIdx.y * stride;
  unsigned long long* stt = status + (int64_t)blockIdx.y * nblk;
  const int i0 = blk * SC_BLOCK + threadIdx.x * SC_ITEMS;
  int v[SC_ITEMS];
  int t = 0;
  const unsigned long long dv = sf.div[blockIdx.y];
  if (sf.keys) {  // flags: key prefix (key / dv) differs from the previous slot's; one division per slot
    auto q = [&](int s) { return dv == 1 ? sf.keys[s] : sf.keys[s] / dv; };
    unsigned long long prev = (i0 > 0 && i0 - 1 < n) ? q(i0 - 1) : ~0ull;
#pragma unroll
    for (int j = 0; j < SC_ITEMS; ++j) {
      const int s = i0 + j;
      int f = 0;
      if (s < n) {
        const unsigned long long cur = q(s);
        f = (s == 0 || cur != prev) ? 1 : 0;
        prev = cur;
      }
      t += f;
      v[j] = t;
    }
  } else {
#pragma unroll
    for (int j = 0; j < SC_ITEMS; ++j) {
      const int s = i0 + j;
      t += s < n ? arr[s] : 0;
      v[j] = t;
    }
  }
  int total;
  const int off = block_excl_scan_256(t, wsum, total);
  if (threadIdx.x < 32) {  // warp 0: publish, then look back 32 predecessors at a time
    const int lane = threadIdx.x;
    int prefix = 0;
    if (blk == 0) {
      if (lane == 0) st_release_u64(stt, (2ull << 62) | (unsigned)total);
    } else {
      if (lane == 0) st_release_u64(stt + blk, (1ull << 62) | (unsigned)total);
      for (int hi = blk - 1; hi >= 0; hi -= 32) {
        const int i = hi - lane;  // lane 0 = nearest predecessor
        unsigned long long w = 2ull << 62;  // past block 0: contributes nothing
        if (i >= 0) {
          do {
            w = ld_acquire_u64(stt + i);
          } while ((w >> 62) == 0);
        }
        const unsigned incl = __ballot_sync(0xffffffffu, i >= 0 && (w >> 62) == 2);
        const int stop = incl ? __ffs(incl) - 1 : 31;  // nearest inclusive prefix in the window
        int x = (lane <= stop && i >= 0) ? (int)(unsigned)(w & 0xffffffffull) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        prefix += x;
        if (incl) break;
      }
      if (lane == 0) st_release_u64(stt + blk, (2ull << 62) | (unsigned)(prefix + total));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  const int base = off + s_prefix;
#pragma unroll
  for (int j = 0; j < SC_ITEMS; ++j)
    if (i0 + j < n) arr[i0 + j] = v[j] + base;
}

// ---------------------------------------------------------------------------
// unique IDs over the sorted keys (flags formed inside k_scan_onepass)
// After the inclusive scan: uniq[u] = key, seg[u] = first sorted slot.
// counts[d-1] = U, seg[U] = B.
__global__ void k_unique_emit(const unsigned long long* __restrict__ skey, int B, const int* __restrict__ scan,
                              unsigned long long* __restrict__ uniq, int* __restrict__ seg,
                              int* __restrict__ counts, int d, const DevStatus* st) {
  TT_PDL_ENTRY();
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= B) return;
  if (tt_failed(st)) {
    if (s == 0)
      for (int k = 0; k < d; ++k) counts[k] = 0;
    return;
  }
  int u = scan[s] - 1;
  if (s == 0 || skey[s] != skey[s - 1]) {
    uniq[u] = skey[s];
    seg[u] = s;
  }
  if (s == B - 1) {
    counts[d - 1] = u + 1;
    seg[u + 1] = B;
  }
}

// Node arrays per level (0-based k): digit, parent, first unique.  Level d-1
// nodes are the unique IDs themselves.
// Level 0 nodes are already in digit order and distinct: their group order is
// the identity and their sorted digits are their digits (order0 / sdig0).
__global__ void k_level_emit(DevCfg c, const unsigned long long* __restrict__ uniq, int* __restrict__ counts,
                             const int* __restrict__ scan /*[k][cap] inclusive*/, int64_t cap,
                             int* __restrict__ digit /*[k][cap]*/, int* __restrict__ parent,
                             int* __restrict__ first, int* __restrict__ order0, unsigned* __restrict__ sdig0) {
  TT_PDL_ENTRY();
  const int U = ld_count(&counts[c.d - 1]);
  int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= U) return;
  unsigned long long key = uniq[u], prev = u ? uniq[u - 1] : 0;
  for (int k = 0; k + 1 < c.d; ++k) {
    unsigned long long S = (unsigned long long)c.S[k];
    unsigned long long p = key / S;
    if (u == 0 || p != prev / S) {
      int node = scan[k * cap + u] - 1;
      const int dg = (int)(p % (unsigned long long)c.m[k]);
      digit[k * cap + node] = dg;
      first[k * cap + node] = u;
      if (k == 0) {
        order0[node] = node;
        sdig0[node] = (unsigned)dg;
      }
      parent[k * cap + node] = k ? scan[(k - 1) * cap + u] - 1 : -1;
    }
    if (u == U - 1) counts[k] = scan[k * cap + u];
  }
  const int k = c.d - 1;
  digit[k * cap + u] = (int)(key % (unsigned long long)c.m[k]);
  first[k * cap + u] = u;
  parent[k * cap + u] = scan[(k - 1) * cap + u] - 1;
}

// child ranges: level-k node n owns level-(k+1) nodes [cs[n], cs[n+1]).
__global__ void k_children(DevCfg c, const int* __restrict__ counts, const int* __restrict__ scan, int64_t cap,
                           const int* __restrict__ first, int* __restrict__ cstart /*[k][cap+1]*/) {
  TT_PDL_ENTRY();
  const int k = blockIdx.y;  // 0 .. d-2
  const int cnt = ld_count(&counts[k]);
  int nd = blockIdx.x * blockDim.x + threadIdx.x;
  if (nd > cnt) return;
  int* cs = cstart + k * (cap + 1);
  if (nd == cnt) {
    cs[nd] = ld_count(&counts[k + 1]);
    return;
  }
  int u = first[k * cap + nd];
  cs[nd] = (k + 1 == c.d - 1) ? u : scan[(k + 1) * cap + u] - 1;
}

// copy node digits into sort keys (values = node index)
__global__ void k_digits_to_keys(const int* __restrict__ digit, const int* n_dev, unsigned* __restrict__ keys,
                                 int* __restrict__ vals) {
  TT_PDL_ENTRY();
  const int n = ld_count(n_dev);
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = (unsigned)digit[i];
  vals[i] = i;
}

struct GroupOffArgs {
  const unsigned* sdig[TT_MAXD];
  int* goff[TT_MAXD];
  int m[TT_MAXD];
  int shift[TT_MAXD];  // sorted keys are (digit << shift) | refinement
};

// Level-F sort keys with a secondary refinement: (digit << 2) | min(#IDs - 1, 3).
// Inside a digit group the level-F nodes then come ordered by their number of
// distinct IDs, so a GEMM tile holds nodes of similar dC cost: the tile's dC
// phase lasts as long as its most expensive node, and mixing one 4-ID node
// into a tile of 1-ID nodes stalls every other thread at the tile barrier.
__global__ void k_levelF_keys(const int* __restrict__ counts, int F, const int* __restrict__ digitF,
                              const int* __restrict__ cstartF, unsigned* __restrict__ keys) {
  TT_PDL_ENTRY();
  const int n = ld_count(&counts[F]);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int nid = cstartF[i + 1] - cstartF[i];
  keys[i] = ((unsigned)digitF[i] << 2) | (unsigned)min(nid - 1, 3);
}

// all levels at once: blockIdx.y = level
__global__ void k_group_offsets_all(GroupOffArgs ga, const int* __restrict__ counts) {
  TT_PDL_ENTRY();
  const int k = blockIdx.y;
  const int n = ld_count(&counts[k]);
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v > ga.m[k]) return;
  const unsigned* sd = ga.sdig[k];
  const int sh = ga.shift[k];
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((int)(sd[mid] >> sh) < v) lo = mid + 1; else hi = mid;
  }
  ga.goff[k][v] = lo;
}

// goff[v] = first slot whose sorted digit >= v, v in [0, m]
__global__ void k_group_offsets(const unsigned* __restrict__ sdig, const int* n_dev, int m, int* __restrict__ goff) {
  TT_PDL_ENTRY();
  const int n = ld_count(n_dev);
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v > m) return;
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if ((int)sdig[mid] < v) lo = mid + 1; else hi = mid;
  }
  goff[v] = lo;
}

}  // namespace tt
