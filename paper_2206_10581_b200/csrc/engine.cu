// engine.cu -- host side of the B200 TT-embedding engine and its C-ABI
// (include/tt_engine.h).  One handle per GPU owns the device cores,
// gradients, optimizer state and the per-batch plan; every hot-path call is
// stream-ordered and host-sync free (counts that depend on the batch stay on
// the device), so a whole training step can be captured in a CUDA graph.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>
#include <utility>

#include "../../include/tt_engine.h"
#include "comm.cuh"
#include "common.cuh"
#include "kernels_fused.cuh"
#include "kernels_generic.cuh"
#include "kernels_init.cuh"
#include "kernels_owner.cuh"
#include "kernels_plan.cuh"
#include "kernels_plan_small.cuh"
#include "kernels_rows.cuh"
#include "kernels_tcgen05.cuh"
#include "kernels_update.cuh"

using namespace tt;

namespace {

thread_local std::string g_err;
// staging slots of the pipelined host-buffer steps: three, so the host can keep
// a step's upload queued while it waits for the download of the step before
// (with two, that wait coupled the copy engines: 3.12 vs 2.8 ms at papers)
constexpr int TT_HOST_SLOTS = 3;
long long* g_trace_buf = nullptr;  // TT_TC_TRACE: last backward's per-CTA timestamps
thread_local int64_t g_err_pos = -1;
thread_local int64_t g_err_val = 0;

int fail(int code, const std::string& msg, int64_t pos = -1, int64_t val = 0) {
  g_err = msg;
  g_err_pos = pos;
  g_err_val = val;
  return code;
}

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? TT_ERR_NOMEM : TT_ERR_CUDA,           \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                    \
  } while (0)

int64_t bitlen(uint64_t v) {
  int64_t b = 0;
  while (v) { ++b; v >>= 1; }
  return b;
}

int grid_for(int64_t total, int threads = 256, int64_t cap = 148 * 32) {
  int64_t g = (total + threads - 1) / threads;
  if (g < 1) g = 1;
  return (int)std::min<int64_t>(g, cap);
}

}  // namespace

struct tt_engine {
  tt_config_c cfg{};
  DevCfg dc{};
  int device = 0;
  int nsm = 148;
  cudaStream_t own = nullptr;

  // parameters / gradients / optimizer state (device layout)
  float* params = nullptr;
  float* grads = nullptr;  // nparams values + touch counters (own or bound)
  float* own_grads = nullptr;
  int64_t ntc = 0;         // number of touch counters (sum of m_k)
  float* s1 = nullptr;
  float* s2 = nullptr;
  float* snap = nullptr;  // tt_cores_snapshot
  int* perm = nullptr;    // tt_set_permutation (node relabelling), int32 on the device
  long long* d_step = nullptr;
  DevStatus* st = nullptr;
  int opt_kind = TT_OPT_SGD;
  double lr = 1e-3, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  bool dense = false;

  // plan (capacity grows, never shrinks)
  int64_t cap = 0;
  int64_t B = 0;
  const int64_t* last_idx = nullptr;
  unsigned long long *keys_a = nullptr, *keys_b = nullptr, *skeys = nullptr, *uniq = nullptr;
  int *pos_a = nullptr, *pos_b = nullptr, *spos = nullptr;
  int* hist = nullptr;
  int* flag = nullptr;
  int* seg = nullptr;
  int* counts = nullptr;
  int* d_B = nullptr;
  int* lflags = nullptr;
  int *digit = nullptr, *parent = nullptr, *first = nullptr, *cstart = nullptr;
  unsigned* gk[TT_MAXD][2] = {};
  int* gv[TT_MAXD][2] = {};
  int* order[TT_MAXD] = {};
  unsigned* sdig[TT_MAXD] = {};
  int* goff[TT_MAXD] = {};
  unsigned long long* scan_status = nullptr;  // single-pass scan: [narr][nblk] status words + [narr] tickets
  LevelBufs L{};
  int64_t capk[TT_MAXD] = {};
  FusedBufs F{};

  // host-entry staging
  int64_t stage_cap = 0;
  int64_t* st_idx = nullptr;
  float* st_out = nullptr;
  float* st_up = nullptr;
  // host-entry copy streams: the upstream upload overlaps the plan + forward,
  // the row download overlaps the backward + update
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_up = nullptr, ev_fwd = nullptr, ev_in = nullptr;

  // pipelined host-buffer steps (tt_train_step_submit / _wait): staging slots
  // so that later steps' uploads run under a step's compute and download
  struct HostSlot {
    int64_t cap = 0, B = 0;
    int64_t* idx = nullptr;
    float* up = nullptr;
    float* out = nullptr;
    const int64_t* h_idx = nullptr;
    DevStatus* h_st = nullptr;  // pinned: the device status right after the step
    cudaEvent_t ev_idx = nullptr, ev_up = nullptr, ev_fwd = nullptr, ev_done = nullptr, ev_out = nullptr;
    bool busy = false, has_out = false;
  } hs[TT_HOST_SLOTS];
  int hs_next = 0, hs_head = 0, hs_count = 0;

  // profiling (tt_set_profiling): event pairs per slot
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev[8];
  std::vector<cudaEvent_t> ev_pool;

  // bookkeeping
  bool plan_valid = false;
  bool psave_valid = false;
  bool ll_fused = false;
  bool lr_w = false;  // the last backward's k_lowrank_bwd also formed W_u (k_fused_w skipped)
  cudaStream_t s_aux = nullptr;  // side stream: k_fused_w beside the level-F backward (TT_AUX_STREAM)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // the last forward's GEMM also wrote the output rows (k_fused_fwd8<..., LL>)  // Psave holds P_F (false once k_fused_wdc wrote dC over it)
  int64_t cores_version = 0, plan_version = -1;
  int64_t batch_count = 0;
  int64_t launches = 0;
  int path_pref = 0;   // 0 auto, 1 generic
  int last_path = 0;
  bool fused_ok = false;
  FusedShape fs{};
  int level_shift_F = 0;  // level-F sort keys carry an ID-count class in their low bits
  bool tc_ok = false;  // tensor-core (tcgen05) kernels exist for this shape
  TcShape ts{};

  // data parallelism (tt_comm_init*, tt_allreduce_grads): NCCL communicator,
  // its stream, and the events that order the gradient all-reduce against
  // the backward -- ev_gF is recorded right after the level-F GEMM kernel
  // (which alone writes dG_F, 63 of the 64 MB at papers), so that segment's
  // all-reduce overlaps the backward's remaining kernels
  ncclComm_t comm = nullptr;
  bool own_comm = false;
  int rank = 0, nranks = 1;
  cudaStream_t s_comm = nullptr;
  cudaEvent_t ev_gF = nullptr, ev_bwd = nullptr, ev_comm = nullptr;
  bool gF_ready = false;

  // ID-owner sharding (tt_owner_*): the last owner-routed batch
  struct Owner {
    int64_t cap = 0, cap_r = 0;
    unsigned *ka = nullptr, *kb = nullptr;
    int *va = nullptr, *vb = nullptr;
    int* perm = nullptr;      // local positions in owner order (va or vb)
    int64_t* sid = nullptr;   // local IDs in owner order
    int* d_counts = nullptr;  // [P] local IDs per owner
    int* d_all = nullptr;     // [P][P] all ranks' counts
    unsigned long long* d_gbad = nullptr;
    int* h_all = nullptr;     // pinned [P][P] + 2 ints of the global bad position
    int64_t* rid = nullptr;   // received IDs (owner side)
    float *rout = nullptr, *back = nullptr, *sup = nullptr, *rup = nullptr;
    std::vector<int64_t> soff, roff, send, recv;
    int64_t B = 0, Bown = 0;
    bool valid = false;
  } ow;

  // TMA tensor maps of the cores for the fused forward (level k -> [m_k R_k] x
  // [n_k R_{k+1}] fp32 view of core k, box {128, R_k})
  CUtensorMap tmap[TT_MAXD] = {};
  bool tmap_ok[TT_MAXD] = {};
  CUtensorMap ps_tmap = {};  // saved P_F / dC blocks as [rows][NC] fp32, box {32, RP}, 128-byte swizzle
  const void* ps_tmap_ptr = nullptr;
  int64_t ps_tmap_rows = 0;

  // the level-F GEMM kernels of the last forward / backward (tt_main_kernels)
  const char* fwd_kernel = "";
  const char* bwd_kernel = "";
};

namespace {

cudaEvent_t ev_get(tt_engine* h) {
  if (!h->ev_pool.empty()) {
    cudaEvent_t e = h->ev_pool.back();
    h->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// RAII phase timer: records a start/stop event pair on `s` when profiling
struct Phase {
  tt_engine* h;
  int slot;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  Phase(tt_engine* h_, int slot_, cudaStream_t s_) : h(h_), slot(slot_), s(s_) {
    if (h->profiling) {
      a = ev_get(h);
      cudaEventRecord(a, s);
    }
  }
  ~Phase() {
    if (a) {
      cudaEvent_t b = ev_get(h);
      cudaEventRecord(b, s);
      h->prof_ev[slot].push_back({a, b});
    }
  }
};

void free_plan(tt_engine* h) {
  void* ptrs[] = {h->keys_a, h->keys_b, h->uniq, h->pos_a, h->pos_b, h->hist, h->flag, h->seg,
                  h->lflags, h->digit, h->parent, h->first, h->cstart, h->scan_status};
  for (void* p : ptrs) cudaFree(p);
  for (int k = 0; k < TT_MAXD; ++k) {
    for (int j = 0; j < 2; ++j) { cudaFree(h->gk[k][j]); cudaFree(h->gv[k][j]); h->gk[k][j] = nullptr; h->gv[k][j] = nullptr; }
    cudaFree(h->goff[k]); h->goff[k] = nullptr;
    h->sdig[k] = nullptr; h->order[k] = nullptr;
    cudaFree(h->L.P[k]); cudaFree(h->L.dP[k]); cudaFree(h->L.dPc[k]);
    h->L.P[k] = h->L.dP[k] = h->L.dPc[k] = nullptr;
  }
  free_fused(h->F);
  h->keys_a = h->keys_b = h->uniq = nullptr;
  h->pos_a = h->pos_b = h->hist = h->flag = h->seg = h->lflags = nullptr;
  h->digit = h->parent = h->first = h->cstart = nullptr;
  h->scan_status = nullptr;
  h->cap = 0;
}

template <class T>
cudaError_t dalloc(T** p, int64_t count) {
  return cudaMalloc((void**)p, sizeof(T) * (size_t)std::max<int64_t>(count, 1));
}

int ensure_plan(tt_engine* h, int64_t B) {
  if (B <= h->cap) return TT_OK;
  free_plan(h);
  const int64_t cap = std::max<int64_t>(B, 1024);
  const DevCfg& c = h->dc;
  const int d = c.d;
  const int64_t ntiles = (cap + RS_TILE - 1) / RS_TILE;
  CU(dalloc(&h->keys_a, cap));
  CU(dalloc(&h->keys_b, cap));
  CU(dalloc(&h->uniq, cap));
  CU(dalloc(&h->pos_a, cap));
  CU(dalloc(&h->pos_b, cap));
  CU(dalloc(&h->hist, (int64_t)TT_MAXD * (ntiles + 1) * RS_MAXBINS));  // rs_hist slots
  CU(dalloc(&h->flag, cap));
  CU(dalloc(&h->seg, cap + 1));
  CU(dalloc(&h->lflags, (int64_t)d * cap));
  CU(dalloc(&h->digit, (int64_t)d * cap));
  CU(dalloc(&h->parent, (int64_t)d * cap));
  CU(dalloc(&h->first, (int64_t)d * cap));
  CU(dalloc(&h->cstart, (int64_t)d * (cap + 1)));
  const int64_t nblk = (cap + SC_BLOCK - 1) / SC_BLOCK;
  CU(dalloc(&h->scan_status, (nblk + 1) * TT_MAXD));
  int64_t prod = 1;
  for (int k = 0; k < d; ++k) {
    prod = (prod > (int64_t)1 << 40) ? prod : prod * c.m[k];
    h->capk[k] = std::min<int64_t>(cap, prod);
    CU(dalloc(&h->gk[k][0], cap));
    CU(dalloc(&h->gk[k][1], cap));
    CU(dalloc(&h->gv[k][0], cap));
    CU(dalloc(&h->gv[k][1], cap));
    CU(dalloc(&h->goff[k], c.m[k] + 1));
  }
  h->cap = cap;
  return TT_OK;
}

// generic-path level buffers (allocated on first generic use)
int ensure_generic(tt_engine* h) {
  const DevCfg& c = h->dc;
  for (int k = 0; k < c.d; ++k) {
    if (k >= 1 && k + 1 < c.d && !h->L.P[k]) CU(dalloc(&h->L.P[k], h->capk[k] * c.rows[k] * c.cols[k]));
    if (!h->L.dP[k]) CU(dalloc(&h->L.dP[k], h->capk[k] * c.rows[k] * c.cols[k]));
    if (k >= 1 && !h->L.dPc[k]) CU(dalloc(&h->L.dPc[k], h->capk[k] * c.rows[k] * c.R[k]));
  }
  return TT_OK;
}

// Programmatic stream serialisation (PDL, default on; TT_PDL=0 turns it off):
// the next kernel is scheduled while the previous one drains and waits
// (griddepcontrol.wait, TT_PDL_ENTRY, first statement of every kernel) for
// its completion -- 0.147 -> 0.130 ms for the eager plan at papers.  (An
// earlier race on the tensor path was k_tc_fwd missing that entry wait.)
// Not used under stream capture unless TT_PDL_GRAPH=1: the replayed graph
// already launches back to back, and programmatic edges measured slower there.
// Diagnostic switches, read once per process (all off by default):
//   TT_TC_VARIANT / TT_TC_BVARIANT = bit mask handed to the tcgen05 forward /
//     backward as FusedArgs::mode to skip parts of the work for attribution
//     (2 MMAs, 4 epilogue stores, 8 A staging, 16 dC formation, 32 dC planes,
//     64 one ID per node); results are wrong while set (scripts/tc_variants.sh);
//   TT_TC_TRACE = 1: per-CTA phase timestamps of the backward GEMM kernels,
//     2: per-tile role stamps of the tcgen05 forward (tt_debug_trace,
//     scripts/tc_trace.py).
// The forward's variant bits are 2 MMAs, 4 P_F stores, 8 A loads.
struct DiagEnv {
  int tc_fwd_variant = 0, tc_bwd_variant = 0;
  int trace = 0;  // 1: backward, 2: forward
  DiagEnv() {
    if (const char* e = getenv("TT_TC_VARIANT")) tc_fwd_variant = atoi(e);
    if (const char* e = getenv("TT_TC_BVARIANT")) tc_bwd_variant = atoi(e);
    if (const char* e = getenv("TT_TC_TRACE")) trace = atoi(e);
  }
};
const DiagEnv& diag() {
  static const DiagEnv d;
  return d;
}

// Programmatic dependent launch on eager launches (default; TT_PDL=0 turns it
// off).  Every kernel opens with TT_PDL_ENTRY (griddepcontrol.wait before any
// read of its predecessor's output).
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("TT_PDL");
    return !(e && *e == '0');
  }();
  return on;
}
// TT_PDL_GRAPH=1: also under stream capture (programmatic edges in the graph;
// measured slower for the replayed step, so off by default)
bool pdl_graph_enabled() {
  static const bool on = [] {
    const char* e = getenv("TT_PDL_GRAPH");
    return e && *e && *e != '0';
  }();
  return on;
}

template <typename... KArgs, typename... Args>
void tt_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  cfg.numAttrs = (pdl_enabled() && (cs == cudaStreamCaptureStatusNone || pdl_graph_enabled())) ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#define LAUNCH(kernel, grid, block, smem, stream, ...)                          \
  do {                                                                          \
    tt_launch(kernel, dim3(grid), dim3(block), (size_t)(smem), (stream), __VA_ARGS__); \
    ++h->launches;                                                              \
  } while (0)

// The dynamic shared-memory opt-in is a per-device attribute of the function:
// one bit per device that has it (an engine on a second GPU of the process
// must set it again).
template <class K>
void rs_set_attrs(int device) {
  static std::atomic<unsigned long long> done{0};  // bit per device (devices 0..63)
  const unsigned long long bit = 1ull << (device & 63);
  if (device >= 64 || !(done.load() & bit)) {
    cudaFuncSetAttribute(k_rs_scatter<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RS_SCATTER_SMEM);
    done.fetch_or(bit);
  }
}

// hist/tot region of sort slot y: (ntiles + 1) * RS_MAXBINS ints each
int* rs_hist(tt_engine* h, int y, int ntiles) { return h->hist + (int64_t)y * (ntiles + 1) * RS_MAXBINS; }

template <class K>
K* radix_sort(tt_engine* h, cudaStream_t s, K* ka, int* va, K* kb, int* vb, const int* n_dev, int n_host,
              int64_t nmax, int nbits, int** vout) {
  const int ntiles = (int)((nmax + RS_TILE - 1) / RS_TILE);
  const int passes = (nbits + RS_MAXBITS - 1) / RS_MAXBITS;
  K* kin = ka; K* kout = kb;
  int* vin = va; int* vo = vb;
  rs_set_attrs<K>(h->device);
  int shift = 0;
  for (int p = 0; p < passes; ++p) {
    const int bits = (nbits - shift + (passes - p) - 1) / (passes - p);  // split evenly
    const int bins = 1 << bits;
    RSBatch<K> rb{};
    rb.kin[0] = kin; rb.vin[0] = vin; rb.kout[0] = kout; rb.vout[0] = vo; rb.n_dev[0] = n_dev;
    rb.hist[0] = rs_hist(h, 0, ntiles);
    rb.tot[0] = rb.hist[0] + (int64_t)ntiles * RS_MAXBINS;
    rb.n_host = n_host;
    LAUNCH(k_rs_hist<K>, ntiles, RS_THREADS, 0, s, rb, shift, bits);
    LAUNCH(k_rs_colscan<K>, (bins + 31) / 32, 32 * RS_CS_SEG, 0, s, rb, bits);
    const size_t smem = sizeof(int) * ((size_t)RS_WARPS * bins + bins + 64);
    LAUNCH(k_rs_scatter<K>, ntiles, RS_THREADS, smem, s, rb, shift, bits);
    std::swap(kin, kout);
    std::swap(vin, vo);
    shift += bits;
  }
  *vout = vin;
  return kin;
}

// The plan's per-level digit sorts (levels 1..d-1) in one pass for all levels
// at once (3 launches instead of 4 per level): stable by node index.
// Requires every m_k <= 2^RS_MAXBITS.
// TT_COUNT_ORDER=0: level-F nodes in plain digit order (no ID-count refinement)
bool count_order_enabled() {
  static const bool on = [] {
    const char* e = getenv("TT_COUNT_ORDER");
    return !(e && *e == '0');
  }();
  return on;
}

void sort_levels(tt_engine* h, cudaStream_t s) {
  const DevCfg& c = h->dc;
  const int d = c.d;
  const int64_t cap = h->cap;
  const int ntiles = (int)((cap + RS_TILE - 1) / RS_TILE);
  int nbits = 1;
  for (int k = 1; k < d; ++k) nbits = std::max<int>(nbits, (int)bitlen((uint64_t)(c.m[k] - 1)));
  // the fused level F sorts on (digit, ID-count class) when the key still
  // fits one radix pass (k_levelF_keys)
  const int F = d - 2;
  h->level_shift_F = 0;
  if (F >= 1 && count_order_enabled() && bitlen((uint64_t)(c.m[F] - 1)) + 2 <= RS_MAXBITS) {
    h->level_shift_F = 2;
    nbits = std::max<int>(nbits, (int)bitlen((uint64_t)(c.m[F] - 1)) + 2);
    LAUNCH(k_levelF_keys, grid_for(cap, 256, INT_MAX), 256, 0, s, (const int*)h->counts, F,
           (const int*)(h->digit + F * cap), (const int*)(h->cstart + F * (cap + 1)), h->gk[F][0]);
  }
  rs_set_attrs<unsigned>(h->device);
  RSBatch<unsigned> rb{};
  for (int k = 1; k < d; ++k) {
    const int y = k - 1;
    rb.kin[y] = (k == F && h->level_shift_F) ? h->gk[F][0] : reinterpret_cast<const unsigned*>(h->digit + k * cap);
    rb.vin[y] = nullptr;
    rb.kout[y] = h->gk[k][1];
    rb.vout[y] = h->gv[k][1];
    rb.n_dev[y] = h->counts + k;
    rb.hist[y] = rs_hist(h, 1 + y, ntiles);
    rb.tot[y] = rb.hist[y] + (int64_t)ntiles * RS_MAXBINS;
    h->sdig[k] = h->gk[k][1];
    h->order[k] = h->gv[k][1];
  }
  rb.n_host = 0;
  const int bins = 1 << nbits;
  LAUNCH(k_rs_hist<unsigned>, dim3(ntiles, d - 1), RS_THREADS, 0, s, rb, 0, nbits);
  LAUNCH(k_rs_colscan<unsigned>, dim3((bins + 31) / 32, d - 1), 32 * RS_CS_SEG, 0, s, rb, nbits);
  const size_t smem = sizeof(int) * ((size_t)RS_WARPS * bins + bins + 64);
  LAUNCH(k_rs_scatter<unsigned>, dim3(ntiles, d - 1), RS_THREADS, smem, s, rb, 0, nbits);
}

// TT_PLAN_SMALL=0 keeps the multi-kernel plan for small batches too
bool plan_small_enabled() {
  static const bool on = [] {
    const char* e = getenv("TT_PLAN_SMALL");
    return !(e && *e == '0');
  }();
  return on;
}

// one memset (status words + tickets) and one single-pass scan kernel
void scan_inclusive(tt_engine* h, cudaStream_t s, int* a, int64_t stride, int narr, const int* n_dev, int64_t nmax,
                    const ScanFlags& sf) {
  const int nblk = (int)((nmax + SC_BLOCK - 1) / SC_BLOCK);
  unsigned long long* status = h->scan_status;
  unsigned long long* ticket = status + (int64_t)narr * nblk;
  cudaMemsetAsync(status, 0, sizeof(unsigned long long) * ((size_t)narr * nblk + narr), s);
  LAUNCH(k_scan_onepass, dim3(nblk, narr), SC_THREADS, 0, s, a, stride, n_dev, status, ticket, nblk, sf);
}

// the device status into mapped host memory (UVA: the host pointer is valid
// on the device)
__global__ void k_status_to_host(const DevStatus* st, DevStatus* host) {
  TT_PDL_ENTRY();
  volatile DevStatus* h = host;
  h->bad_pos = st->bad_pos;
  h->bad_core = st->bad_core;
  __threadfence_system();
}

__global__ void k_reset_status(DevStatus* st, int which) {
  TT_PDL_ENTRY();
  if (which & 1) st->bad_pos = TT_NO_POS;
  if (which & 2) st->bad_core = INT_MAX;
}

// Build the plan for a batch: validate, sort, unique, prefix levels, groups.
int build_plan(tt_engine* h, const int64_t* d_idx, int64_t B, cudaStream_t s) {
  int rc = ensure_plan(h, B);
  if (rc) return rc;
  Phase ph(h, 0, s);
  const DevCfg& c = h->dc;
  const int d = c.d;
  const int64_t cap = h->cap;
  h->B = B;
  h->last_idx = d_idx;
  h->d_B = h->counts + TT_MAXD;
  const int idbits = (int)std::max<int64_t>(1, bitlen((uint64_t)(c.num_nodes - 1)));
  if (B <= PS_MAXB && idbits + PS_IBITS <= 64 && plan_small_enabled()) {
    // the whole plan in one CTA (kernels_plan_small.cuh)
    PlanSmallArgs ps{};
    ps.c = c;
    ps.idx = d_idx;
    ps.B = (int)B;
    ps.perm = h->perm;
    ps.idbits = idbits;
    ps.cap = cap;
    ps.skeys = h->keys_b;
    ps.spos = h->pos_b;
    ps.flag = h->flag;
    ps.uniq = h->uniq;
    ps.seg = h->seg;
    ps.counts = h->counts;
    ps.digit = h->digit;
    ps.parent = h->parent;
    ps.first = h->first;
    ps.cstart = h->cstart;
    for (int k = 0; k < d; ++k) {
      ps.sdig[k] = k == 0 ? h->gk[0][0] : h->gk[k][1];
      ps.order[k] = k == 0 ? h->gv[0][0] : h->gv[k][1];
      ps.goff[k] = h->goff[k];
      h->sdig[k] = ps.sdig[k];
      h->order[k] = ps.order[k];
    }
    ps.st = h->st;
    if (getenv("TT_PS_TRACE")) {  // diagnostics: phase clocks of k_plan_small (tt_debug_trace)
      static long long* ps_trace = nullptr;
      if (!ps_trace) cudaMalloc(&ps_trace, sizeof(long long) * 4096 * 64);
      ps.dbg = ps_trace;
      g_trace_buf = ps_trace;
    }
    CU(cudaFuncSetAttribute(k_plan_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PS_SMEM));
    LAUNCH(k_plan_small, 1, PS_THREADS, PS_SMEM, s, ps);
    h->skeys = h->keys_b;
    h->spos = h->pos_b;
    return TT_OK;
  }
  LAUNCH(k_decompose_validate, grid_for(B, 256, INT_MAX), 256, 0, s, d_idx, B, c.num_nodes, h->keys_a, h->pos_a, h->st,
         (const int*)h->perm, h->counts + TT_MAXD);
  h->skeys = radix_sort<unsigned long long>(h, s, h->keys_a, h->pos_a, h->keys_b, h->pos_b, nullptr, (int)B, B,
                                            idbits, &h->spos);
  ScanFlags uf{};
  uf.keys = h->skeys;
  uf.div[0] = 1;  // unique-ID flags
  scan_inclusive(h, s, h->flag, 0, 1, h->d_B, B, uf);
  LAUNCH(k_unique_emit, grid_for(B, 256, INT_MAX), 256, 0, s, h->skeys, (int)B, h->flag, h->uniq, h->seg, h->counts,
         d, h->st);
  const int* U = h->counts + (d - 1);
  ScanFlags lf{};
  lf.keys = h->uniq;
  for (int k = 0; k + 1 < d; ++k) lf.div[k] = (unsigned long long)c.S[k];  // level-k prefix flags
  scan_inclusive(h, s, h->lflags, cap, d - 1, U, B, lf);
  // level nodes; level 0 is already digit-sorted and distinct (identity group order)
  LAUNCH(k_level_emit, grid_for(B, 256, INT_MAX), 256, 0, s, c, h->uniq, h->counts, h->lflags, cap, h->digit,
         h->parent, h->first, h->gv[0][0], h->gk[0][0]);
  h->order[0] = h->gv[0][0];
  h->sdig[0] = h->gk[0][0];
  LAUNCH(k_children, dim3(grid_for(B + 1, 256, INT_MAX), d - 1), 256, 0, s, c, h->counts, h->lflags, cap, h->first,
         h->cstart);

  bool batched = true;
  for (int k = 1; k < d; ++k) batched = batched && bitlen((uint64_t)(c.m[k] - 1)) <= RS_MAXBITS;
  if (batched) {
    sort_levels(h, s);
  } else {
    for (int k = 1; k < d; ++k) {
      LAUNCH(k_digits_to_keys, grid_for(B, 256, INT_MAX), 256, 0, s, h->digit + k * cap, h->counts + k, h->gk[k][0],
             h->gv[k][0]);
      const int nb = (int)std::max<int64_t>(1, bitlen((uint64_t)(c.m[k] - 1)));
      h->sdig[k] = radix_sort<unsigned>(h, s, h->gk[k][0], h->gv[k][0], h->gk[k][1], h->gv[k][1], h->counts + k, 0,
                                        h->capk[k], nb, &h->order[k]);
    }
  }
  GroupOffArgs ga{};
  int64_t mmax = 0;
  for (int k = 0; k < d; ++k) {
    ga.sdig[k] = h->sdig[k];
    ga.goff[k] = h->goff[k];
    ga.m[k] = (int)c.m[k];
    ga.shift[k] = (batched && k == d - 2) ? h->level_shift_F : 0;
    mmax = std::max<int64_t>(mmax, c.m[k]);
  }
  LAUNCH(k_group_offsets_all, dim3(grid_for(mmax + 1, 256, INT_MAX), d), 256, 0, s, ga, h->counts);
  return TT_OK;
}

int gen_forward(tt_engine* h, float* d_out, cudaStream_t s) {
  int rc = ensure_generic(h);
  if (rc) return rc;
  const DevCfg& c = h->dc;
  const int64_t cap = h->cap;
  for (int k = 1; k < c.d; ++k) {
    if (k == c.d - 1 && !d_out) break;  // backward-only plan: the last level's rows are not needed
    const int64_t total = h->capk[k] * c.rows[k] * c.cols[k];
    LAUNCH(k_gen_fwd_level, grid_for(total), 256, 0, s, c, k, h->params, h->L, h->counts, h->digit + k * cap,
           h->parent + k * cap, h->digit, h->seg, h->spos, d_out, h->st);
  }
  return TT_OK;
}

int gen_backward(tt_engine* h, const float* d_up, cudaStream_t s) {
  int rc = ensure_generic(h);
  if (rc) return rc;
  const DevCfg& c = h->dc;
  const int d = c.d;
  const int64_t cap = h->cap;
  LAUNCH(k_gen_dy, grid_for(h->capk[d - 1] * c.npad), 256, 0, s, c, d_up, h->counts, h->seg, h->spos,
         h->L.dP[d - 1], h->st);
  for (int k = d - 1; k >= 1; --k) {
    LAUNCH(k_gen_bwd_input, grid_for(h->capk[k] * c.rows[k] * c.R[k]), 256, 0, s, c, k, h->params, h->L, h->counts,
           h->digit + k * cap, h->st);
    LAUNCH(k_gen_bwd_weight, grid_for(c.m[k] * c.R[k] * c.cols[k]), 256, 0, s, c, k, h->params, h->L, h->goff[k],
           h->order[k], h->parent + k * cap, h->digit, h->grads, h->st);
    LAUNCH(k_gen_reduce_children, grid_for(h->capk[k - 1] * c.rows[k] * c.R[k]), 256, 0, s, c, k, h->L, h->counts,
           h->cstart + (k - 1) * (cap + 1), h->st);
  }
  LAUNCH(k_gen_bwd_core0, grid_for(h->capk[0] * c.cols[0]), 256, 0, s, c, h->L, h->counts, h->digit, h->grads,
         h->st);
  return TT_OK;
}

int ensure_fused(tt_engine* h) {
  const DevCfg& c = h->dc;
  const FusedShape& f = h->fs;
  FusedBufs& b = h->F;
  const int64_t nodes = h->capk[f.F], ids = h->capk[c.d - 1], chunks = (h->cap + DY_CHUNK - 1) / DY_CHUNK;
  if (b.cap_nodes >= nodes && b.cap_ids >= ids && b.cap_chunks >= chunks) return TT_OK;
  free_fused(b);
  CU(dalloc(&b.Psave, nodes * f.RP * f.NC));
  CU(dalloc(&b.dPc, nodes * f.ncb * f.RP * f.K));
  CU(dalloc(&b.W, ids * f.K * f.NL));
  CU(dalloc(&b.dY, ids * c.npad));
  CU(dalloc(&b.Yu, ids * c.npad));
  CU(dalloc(&b.part, chunks * 2 * c.npad));
  CU(dalloc(&b.gpart, ((chunks + 31) / 32) * 2 * c.npad));
  b.cap_nodes = nodes;
  b.cap_ids = ids;
  b.cap_chunks = chunks;
  return TT_OK;
}

FusedArgs fused_args(tt_engine* h, float* d_out) {
  const DevCfg& c = h->dc;
  const FusedShape& f = h->fs;
  const int64_t cap = h->cap;
  FusedArgs a{};
  a.c = c;
  a.F = f.F; a.ncb = f.ncb; a.RP = f.RP; a.NL = f.NL; a.nF = f.nF; a.BNj = f.BNj; a.OUT = f.OUT; a.NC = f.NC;
  a.params = h->params;
  a.Abase = f.F >= 2 ? h->L.P[f.F - 1] : h->params;
  a.parentF = h->parent + f.F * cap;
  a.digit0 = h->digit;
  a.goffF = h->goff[f.F];
  a.orderF = h->order[f.F];
  a.cstartF = h->cstart + f.F * (cap + 1);
  a.digitL = h->digit + (c.d - 1) * cap;
  a.seg = h->seg;
  a.spos = h->spos;
  a.out = d_out;
  a.Yu = h->F.Yu;
  a.Psave = h->F.Psave;
  a.dY = h->F.dY;
  a.W = h->F.W;
  a.dPc = h->F.dPc;
  a.grads = h->grads;
  a.st = h->st;
  return a;
}

#define FUSED_LAUNCH_T(KER, SMEM, GRID, THREADS, S, ARGS)                                    \
  do {                                                                                       \
    CU(cudaFuncSetAttribute(KER, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(SMEM)));   \
    tt_launch(KER, dim3(GRID), dim3(THREADS), (size_t)(SMEM), (S), ARGS);                     \
    ++h->launches;                                                                           \
  } while (0)
#define FUSED_LAUNCH(KER, SMEM, GRID, S, ARGS) FUSED_LAUNCH_T(KER, SMEM, GRID, FB_THREADS, S, ARGS)

#define FUSED_CASE_F(k_, bn_, rp_, nl_) \
  else if (f.K == k_ && f.BNf == bn_ && f.RP == rp_ && f.NL == nl_) FUSED_LAUNCH((k_fused_fwd<k_, bn_, rp_, nl_>), f.smem_fwd, grid, s, a);
#define FUSED_CASE_B(k_, bn_, rp_, nl_) \
  else if (f.K == k_ && f.BN == bn_ && f.RP == rp_ && f.NL == nl_) FUSED_LAUNCH((k_fused_bwd<k_, bn_, rp_, nl_>), f.smem_bwd, grid, s, a);

// TT_FWD8W=0 keeps the CTA-synchronous k_fused_fwd8 (tile barriers) instead of
// the warp-private-tile k_fused_fwd8w
bool fwd8w_enabled() {
  static const bool on = [] {
    const char* e = getenv("TT_FWD8W");
    return !(e && *e == '0');
  }();
  return on;
}

// TT_FWD8=0 selects the 8 x 4-tile forward (k_fused_fwd) where the 8 x 8 one exists
bool fwd8_enabled() {
  static const bool on = [] {
    const char* e = getenv("TT_FWD8");
    return !(e && *e == '0');
  }();
  return on;
}

// Chunks per digit group for a fused GEMM launch of `grid` = groups x column
// blocks CTAs: enough CTAs for ~3 waves of 2 per SM (products: 140 groups x
// 1 block -> 7 chunks each; billion: 178 -> 5; papers: 1924 -> 1).  TT_SPLIT
// overrides (1 = one CTA per (group, column block)).
// Chunks are only worth it for large groups: an empty CTA (a chunk a small
// group does not have) still costs a CTA slot, measured at ~10 us per launch
// at products / small.  The host bounds a group's rows by
// min(B, prod_{p<=F} m_p) / m_F x RP (the level-F prefixes of the batch) and
// splits only when that bound allows min_rows x 2 rows per chunk
// (profiles/r02/NOTES.md: billion 7.45 -> 5.7 ms; products / small / sweeps
// slower when split).
int split_for(tt_engine* h, int grid, int level, bool fwd) {
  static const int env = [] {
    const char* e = getenv("TT_SPLIT");
    return e && *e ? atoi(e) : 0;
  }();
  static const int env_f = [] {  // forward only (A/B of the forward's wave tail)
    const char* e = getenv("TT_SPLIT_FWD");
    return e && *e ? atoi(e) : 0;
  }();
  if (fwd && env_f > 0) return env_f;
  if (env > 0) return env;
  const DevCfg& c = h->dc;
  long double prefixes = 1;
  for (int k = 0; k <= level; ++k) prefixes *= (long double)c.m[k];
  const long double nodes = std::min<long double>((long double)h->B, prefixes) / (long double)c.m[level];
  const long double rows = nodes * (long double)c.rows[level];
  // ranks <= 16: the backward is bound by forming dC (latency of the
  // last-core slices and upstream rows; the GEMMs are tiny), so more CTAs pay
  // even for small groups (sweep8 / sweep16: profiles/r02/NOTES.md)
  const int min_rows = fwd ? 4096 : (c.R[level] <= 16 ? 128 : 1024);
  const int by_rows = (int)std::min<long double>(16.0L, rows / min_rows);
  const int target = h->nsm * 9;  // (billion: 8 chunks per group -- 4.89 vs 5.18 ms at 5; 12 and 16 no better)
  const int by_grid = std::max(1, std::min(16, (target + grid - 1) / grid));
  return std::max(1, std::min(by_rows, by_grid));
}

// TT_BWDK32 = bit mask of the RP values using k_fused_bwd_k32 (1: RP 4, 2: RP 16);
// default 2: billion's level-F backward 2.75 -> 2.44 ms, while at RP 4
// (products 0.068 -> 0.087 ms, sweep32 0.262 -> 0.324) k_fused_bwd is faster
bool bwdk32_enabled(int rp) {
  static const int mask = [] {
    const char* e = getenv("TT_BWDK32");
    return e && *e ? atoi(e) : 2;
  }();
  return (rp == 4 && (mask & 1)) || (rp == 16 && (mask & 2));
}

// TT_TCBWD: the tensor backward at K <= 64.
//   4 (default at K = 64): k_fused_wdc forms dC = dP_F (with the last core's
//     W_u) over the saved P_F blocks; k_tc_bwd3 stages it by TMA and keeps both
//     dC operands in TMEM (papers 1.62 -> 1.45 ms/step, sweep64 1.05 -> 0.75);
//   1 (default at K = 32): k_tc_bwd, one CTA per item, dC formed in the kernel
//     (billion 3.70 vs 4.12 and products 0.258 vs 0.267 with mode 4: there
//     the extra pass over P_F costs more than the kernel saves);
//   2: the persistent k_tc_bwd2 forming dC itself (0.764 vs 0.765 ms at papers);
//   3: k_fused_wdc + k_tc_bwd2 streaming dC through registers (slower).
// Phase split of k_tc_bwd2 (scripts/tc_bwd2_phases.py): ~17.5k cycles per
// 128-row tile against 4.6k of MMAs -- its roles run one after another.
int tcbwd_mode(const FusedShape& f) {
  static const int m = [] {
    const char* e = getenv("TT_TCBWD");
    return e && *e ? atoi(e) : 0;
  }();
  return m ? m : (f.K == 64 ? 4 : 1);
}
// TT_FWD_LL=1: the FFMA forward writes the output rows itself
// (k_fused_fwd8<..., LL>) instead of k_last_level re-reading P_F.  Off: at
// papers the forward went 0.534 -> 0.915 ms for the 0.147 ms it saves (the
// per-ID epilogue -- slice loads, a 16-lane reduce-scatter, position writes --
// runs serially after every tile and stalls the GEMM), step 2.355 -> 2.600.
bool fwd_ll_enabled() {
  static const bool on = [] {
    const char* e = getenv("TT_FWD_LL");
    return e && *e == '1';
  }();
  return on;
}

// The FFMA backward loads dC formed by k_fused_wdc (mode 1) instead of
// forming it per tile: TT_FFMA_WDC=1 always, 0 never; default at K = 64 with
// NL = 8 (the rank sweep's R = 64: 8 IDs per level-F node, 8-wide last-core
// rows, 0.987 -> 0.856 ms/step).  Measured slower where dC per node is cheap:
// papers 2.359 -> 2.391, products 0.276 -> 0.284, billion (K = 32) 4.90 -> 5.45.
bool ffma_wdc_enabled(const FusedShape& f) {
  static const int m = [] {
    const char* e = getenv("TT_FFMA_WDC");
    return e && *e ? atoi(e) : -1;
  }();
  return m >= 0 ? m == 1 : (f.K == 64 && f.NL == 8);
}
// TT_AUX_STREAM=1: k_fused_w on a side stream beside the level-F backward.
// Off: the two time-share the SMs rather than overlap (papers 2.359 -> 2.357,
// billion 4.898 -> 4.875, products 0.275 -> 0.319 ms/step)
bool aux_stream_enabled() {
  static const bool on = [] {
    const char* e = getenv("TT_AUX_STREAM");
    return e && *e == '1';
  }();
  return on;
}

// k_fused_wdc's shape condition (PIPE blocks, K in {32, 64})
static bool wdc_ok(const FusedShape& f) {
  return (f.K == 32 || f.K == 64) && (int64_t)f.RP * f.nF * f.K <= 2048 && (int64_t)f.RP * f.nF * f.NL <= 256 &&
         f.NL % 4 == 0;
}

// TT_BWDWS = bit mask of the level-F shapes using the warp-specialised
// backward (1: K = 32 with RP = 16, 2: K = 32 with RP = 4; default 1); 0
// selects k_fused_bwd_k32 / k_fused_bwd
bool bwdws_enabled(int K, int RP) {
  static const int mask = [] {
    const char* e = getenv("TT_BWDWS");
    return e && *e ? atoi(e) : 1;
  }();
  return K == 32 && ((RP == 16 && (mask & 1)) || (RP == 4 && (mask & 2)));
}

int split_rows_env(bool fwd, int dflt) {
  static const int f = [] { const char* e = getenv("TT_SPLIT_ROWS_FWD"); return e && *e ? atoi(e) : 0; }();
  static const int b = [] { const char* e = getenv("TT_SPLIT_ROWS_BWD"); return e && *e ? atoi(e) : 0; }();
  const int v = fwd ? f : b;
  return v > 0 ? v : dflt;
}

// TT_TMA=0 stages the forward's slice block by cp.async instead of TMA
bool tma_enabled() {
  static const bool on = [] {
    const char* e = getenv("TT_TMA");
    return !(e && *e == '0');
  }();
  return on;
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  return encode;
}

// The tensor map of the saved level-F blocks (k_tc_bwd3's dC boxes): rows
// node * RP + a of NC fp32 columns, viewed as [NC / 32][rows][32] so that one
// box {32, RP, 4} is a node's 128-column block; 128-byte swizzle
bool psave_tmap(tt_engine* h) {
  const FusedShape& f = h->fs;
  const int64_t rows = h->F.cap_nodes * f.RP;
  if (h->ps_tmap_ptr == h->F.Psave && h->ps_tmap_rows == rows) return true;
  auto encode = tmap_encoder();
  if (!encode) return false;
  // 3-D view [NC / 32 chunks][rows][32]: one box = a node's RP rows x 128 columns
  const cuuint64_t dims[3] = {32, (cuuint64_t)rows, (cuuint64_t)(f.NC / 32)};
  const cuuint64_t strides[2] = {(cuuint64_t)f.NC * sizeof(float), 32 * sizeof(float)};
  const cuuint32_t box[3] = {32, (cuuint32_t)f.RP, 4};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(&h->ps_tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, h->F.Psave, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  h->ps_tmap_ptr = h->F.Psave;
  h->ps_tmap_rows = rows;
  return true;
}

// The tensor map of core k for TMA loads of (K x 128) slice blocks; false
// when the driver entry point is unavailable (the cp.async kernel runs).
bool core_tmap(tt_engine* h, int k) {
  if (h->tmap_ok[k]) return true;
  auto encode = tmap_encoder();
  if (!encode) return false;
  const DevCfg& c = h->dc;
  const cuuint64_t dims[2] = {(cuuint64_t)c.cols[k], (cuuint64_t)(c.m[k] * c.R[k])};
  const cuuint64_t strides[1] = {(cuuint64_t)c.cols[k] * sizeof(float)};
  const cuuint32_t box[2] = {128, (cuuint32_t)c.R[k]};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&h->tmap[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, h->params + c.core_off[k], dims, strides,
                            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  h->tmap_ok[k] = r == CUDA_SUCCESS;
  return h->tmap_ok[k];
}

// TT_LRBWD=0 keeps k_fused_bwd at ranks <= 16 instead of the low-rank
// streaming backward k_lowrank_bwd
bool lrbwd_enabled() {
  static const bool on = [] {
    const char* e = getenv("TT_LRBWD");
    return !(e && *e == '0');
  }();
  return on;
}

bool lrfwd_shape(const FusedShape& f) {
#define LRF_EQ(k_, rp_, nl_, cpl_) if (f.K == k_ && f.RP == rp_ && f.NL == nl_ && f.NC == 32 * cpl_) return true;
  TT_LOWRANK_FWD_SHAPES(LRF_EQ)
#undef LRF_EQ
  return false;
}

int fused_dispatch(tt_engine* h, bool fwd, const FusedArgs& a0, int grid0, cudaStream_t s) {
  const FusedShape& f = h->fs;
  FusedArgs a = a0;
  const int groups = grid0 / a.ncb;
  if (!fwd && a.mode == 0 && a.ncb == 1 && f.K <= 16 && lrbwd_enabled()) {
    // low-rank streaming backward: one warp per (digit group, chunk of >= 1 node)
    a.split = LR_SPLIT;
    a.split_rows = f.RP;
    const int64_t need = (int64_t)groups * a.split * h->dc.slice[a.F];
    if (h->F.cap_gsplit < need) {
      cudaFree(h->F.gsplit);
      h->F.gsplit = nullptr;
      h->F.cap_gsplit = 0;
      CU(dalloc(&h->F.gsplit, need));
      h->F.cap_gsplit = need;
    }
    a.gsplit = h->F.gsplit;
    const int lgrid = (int)(((int64_t)groups * a.split + LR_WARPS - 1) / LR_WARPS);
#define LR_CASE(k_, rp_, nl_, cpl_)                                                              \
    if (f.K == k_ && f.RP == rp_ && f.NL == nl_ && f.NC == 32 * cpl_) {                          \
      LAUNCH((k_lowrank_bwd<k_, rp_, nl_, cpl_>), lgrid, LR_WARPS * 32, 0, s, a);                 \
      h->lr_w = (32 / f.K) >= 1 && f.NL % (32 / f.K) == 0;                                       \
      LAUNCH(k_fused_reduce_gsplit, grid_for((int64_t)groups * h->dc.slice[a.F] / 4, 256, 148 * 8), 256, 0, s, h->dc, \
             a.F, a.split, a.split_rows, a.goffF, (const float*)a.gsplit, a.grads, a.st);      \
      h->bwd_kernel = "k_lowrank_bwd";                                                           \
      return TT_OK;                                                                              \
    }
    TT_LOWRANK_SHAPES(LR_CASE)
#undef LR_CASE
    a.split = 0;  // (no instantiation: the general kernels below)
    a.gsplit = nullptr;
  }
  a.split = split_for(h, grid0, a.F, fwd);
  // min rows per chunk: the forward (a short GEMM per tile, then stores) only
  // pays off with long chunks; the backward (dC formation latency-bound) with
  // short ones (measured: profiles/r02/NOTES.md)
  a.split_rows = fwd ? split_rows_env(true, 1024) : split_rows_env(false, 128);
  const int grid = grid0 * a.split;
  if (!fwd && a.split > 1) {  // dG_F partials of the chunks, reduced below in a fixed order
    const int64_t need = (int64_t)groups * a.split * h->dc.slice[a.F];
    if (h->F.cap_gsplit < need) {
      cudaFree(h->F.gsplit);
      h->F.gsplit = nullptr;
      h->F.cap_gsplit = 0;
      CU(dalloc(&h->F.gsplit, need));
      h->F.cap_gsplit = need;
    }
    a.gsplit = h->F.gsplit;
  }
  if (!fwd && f.BN == 128 && a.mode == 0 && bwdws_enabled(f.K, f.RP)) {
#define BWDWS_CASE(k_, rp_, nl_)                                                                 \
  if (f.K == k_ && f.RP == rp_ && f.NL == nl_) {                                                 \
    FUSED_LAUNCH_T((k_fused_bwd_ws<k_, rp_, nl_>), bwd_ws_smem(k_), grid, WsRoles<k_>::T, s, a);  \
    h->bwd_kernel = "k_fused_bwd_ws";                                                            \
    if (a.split > 1)                                                                             \
      LAUNCH(k_fused_reduce_gsplit, grid_for((int64_t)groups * h->dc.slice[a.F] / 4, 256, 148 * 8), 256, 0, s, h->dc, \
             a.F, a.split, a.split_rows, a.goffF, (const float*)a.gsplit, a.grads, a.st);      \
    return TT_OK;                                                                                \
  }
    TT_BWDWS_SHAPES(BWDWS_CASE)
#undef BWDWS_CASE
  }
  if (!fwd && f.K == 32 && f.BN == 128 && bwdk32_enabled(f.RP)) {
#define BWDK32_CASE(rp_, nl_)                                                                    \
  if (f.RP == rp_ && f.NL == nl_) {                                                              \
    FUSED_LAUNCH_T((k_fused_bwd_k32<rp_, nl_>), bwd_k32_smem(), grid, K32_THREADS, s, a);         \
    h->bwd_kernel = "k_fused_bwd_k32";                                                           \
    if (a.split > 1)                                                                             \
      LAUNCH(k_fused_reduce_gsplit, grid_for((int64_t)groups * h->dc.slice[a.F] / 4, 256, 148 * 8), 256, 0, s, h->dc, \
             a.F, a.split, a.split_rows, a.goffF, (const float*)a.gsplit, a.grads, a.st);      \
    return TT_OK;                                                                                \
  }
    TT_BWDK32_SHAPES(BWDK32_CASE)
#undef BWDK32_CASE
  }
  if (fwd && f.BNf == 128 && fwd8_enabled()) {
#define FWD8_CASE(k_, rp_)                                                                       \
  if (f.K == k_ && f.RP == rp_) {                                                                \
    bool w8 = false;                                                                             \
    if (a.out && tma_enabled() && core_tmap(h, a.F) && fwd8w_enabled()) { /* last level fused */  \
      CU(cudaFuncSetAttribute((k_fused_fwd8w<k_, rp_, true>), cudaFuncAttributeMaxDynamicSharedMemorySize, \
                              (int)fwd8w_smem(k_)));                                              \
      tt_launch((k_fused_fwd8w<k_, rp_, true>), dim3(grid), dim3(F8_THREADS), fwd8w_smem(k_), s, a, h->tmap[a.F]); \
      h->ll_fused = true;                                                                        \
      w8 = true;                                                                                 \
    } else if (a.out && tma_enabled() && core_tmap(h, a.F)) { /* last level fused (fused_forward decided) */ \
      CU(cudaFuncSetAttribute((k_fused_fwd8<k_, rp_, true, true>), cudaFuncAttributeMaxDynamicSharedMemorySize, \
                              (int)fwd8_smem(k_)));                                               \
      tt_launch((k_fused_fwd8<k_, rp_, true, true>), dim3(grid), dim3(F8_THREADS), fwd8_smem(k_), s, a, h->tmap[a.F]); \
      h->ll_fused = true;                                                                        \
    } else if (tma_enabled() && core_tmap(h, a.F) && fwd8w_enabled()) {                         \
      CU(cudaFuncSetAttribute((k_fused_fwd8w<k_, rp_>), cudaFuncAttributeMaxDynamicSharedMemorySize, \
                              (int)fwd8w_smem(k_)));                                              \
      tt_launch((k_fused_fwd8w<k_, rp_>), dim3(grid), dim3(F8_THREADS), fwd8w_smem(k_), s, a, h->tmap[a.F]); \
      w8 = true;                                                                                 \
    } else if (tma_enabled() && core_tmap(h, a.F)) {                                             \
      CU(cudaFuncSetAttribute((k_fused_fwd8<k_, rp_, true>), cudaFuncAttributeMaxDynamicSharedMemorySize, \
                              (int)fwd8_smem(k_)));                                               \
      tt_launch((k_fused_fwd8<k_, rp_, true>), dim3(grid), dim3(F8_THREADS), fwd8_smem(k_), s, a, h->tmap[a.F]); \
    } else {                                                                                     \
      CU(cudaFuncSetAttribute((k_fused_fwd8<k_, rp_, false>), cudaFuncAttributeMaxDynamicSharedMemorySize, \
                              (int)fwd8_smem(k_)));                                               \
      tt_launch((k_fused_fwd8<k_, rp_, false>), dim3(grid), dim3(F8_THREADS), fwd8_smem(k_), s, a, h->tmap[a.F]); \
    }                                                                                            \
    ++h->launches;                                                                               \
    if (a.mode == 0) h->fwd_kernel = w8 ? "k_fused_fwd8w" : "k_fused_fwd8";                      \
    return TT_OK;                                                                                \
  }
    TT_FWD8_SHAPES(FWD8_CASE)
#undef FWD8_CASE
  }
  if (fwd) {
    if (false) {
    }
    TT_FUSED_FWD_SHAPES(FUSED_CASE_F)
    else return fail(TT_ERR_ARG, "fused path: forward shape not compiled");
    if (a.mode == 0) h->fwd_kernel = "k_fused_fwd";
  } else {
    if (false) {
    }
    TT_FUSED_SHAPES(FUSED_CASE_B)
    else return fail(TT_ERR_ARG, "fused path: backward shape not compiled");
    if (a.mode == 0) h->bwd_kernel = "k_fused_bwd";
    if (a.split > 1)
      LAUNCH(k_fused_reduce_gsplit, grid_for((int64_t)groups * h->dc.slice[a.F] / 4, 256, 148 * 8), 256, 0, s, h->dc, a.F,
             a.split, a.split_rows, a.goffF, (const float*)a.gsplit, a.grads, a.st);
  }
  return TT_OK;
}

// Wide (materialised) level k < F on the fused kernels: C = P_{k-1} . G_k is
// written to L.P[k] (forward), dC = L.dP[k] (backward).  Requires a compiled
// (K, BN, RP, *) instantiation; otherwise the generic kernels run.
struct WideShape {
  bool ok = false;
  FusedShape f{};
};

WideShape wide_shape(const DevCfg& c, int k) {
  WideShape w;
  const int64_t K = c.R[k], NC = c.cols[k], RP = c.rows[k];
  int BN = 0;
  if (K == 16 && NC % 64 == 0) BN = 64;
  if (K == 32 && NC % 128 == 0) BN = 128;
  if (K == 64 && NC % 128 == 0) BN = 128;
  if (K == 128 && NC % 128 == 0) BN = 128;
  if (!BN || RP > FB_BM || FB_BM % RP || c.R[k + 1] != K) return w;
  int nl = 0;
  for (int cand : {4, 8})
    if (fused_shape_compiled((int)K, BN, (int)RP, cand) || fused_shape_compiled((int)K, BN * 2, (int)RP, cand)) nl = cand;
  if (!nl) return w;
  FusedShape& f = w.f;
  f.ok = 1; f.F = k; f.K = (int)K; f.NC = (int)NC; f.RP = (int)RP; f.NL = nl; f.nF = (int)c.n[k];
  f.BN = BN; f.ncb = (int)(NC / BN); f.BNj = BN / (int)K; f.OUT = 0;
  f.BNf = std::min(BN, 128); f.ncbf = (int)(NC / f.BNf); f.BNjf = f.BNf / (int)K;
  const size_t ints = sizeof(int64_t) * FB_NB + sizeof(int) * (3 * FB_NB + 12) + 16;
  f.smem_fwd = sizeof(float) * (K * (f.BNf + 4) + 2 * FB_BM * K) + ints + sizeof(int) * (3 * FB_IDS + 8) + 16;
  f.CHF = 0;
  f.smem_bwd = sizeof(float) * (K * (BN + 4) + FB_BM * K + FB_BM * (BN + 4)) + ints + sizeof(int) * (FB_IDS + 8);
  // the instantiation list pairs (K, BN) -- make sure the forward/backward kernels exist
  bool fwd_ok = false, bwd_ok = false;
#define TT_CHECK_F(k_, bn_, rp_, nl_) if (K == k_ && f.BNf == bn_ && RP == rp_ && nl == nl_) fwd_ok = true;
#define TT_CHECK_B(k_, bn_, rp_, nl_) if (K == k_ && BN == bn_ && RP == rp_ && nl == nl_) bwd_ok = true;
  TT_FUSED_FWD_SHAPES(TT_CHECK_F)
  TT_FUSED_SHAPES(TT_CHECK_B)
#undef TT_CHECK_F
#undef TT_CHECK_B
  w.ok = fwd_ok && bwd_ok;
  return w;
}

FusedArgs wide_args(tt_engine* h, int k, const FusedShape& f) {
  FusedArgs a = fused_args(h, nullptr);
  const int64_t cap = h->cap;
  a.F = k; a.ncb = f.ncb; a.RP = f.RP; a.NL = f.NL; a.nF = f.nF; a.BNj = f.BNj; a.OUT = 0; a.NC = f.NC;
  a.Abase = k >= 2 ? h->L.P[k - 1] : h->params;
  a.parentF = h->parent + k * cap;
  a.goffF = h->goff[k];
  a.orderF = h->order[k];
  a.cstartF = h->cstart + k * (cap + 1);
  a.Psave = h->L.P[k];
  a.out = nullptr;
  a.mode = 1;
  a.dPin = h->L.dP[k];
  return a;
}

int wide_dispatch(tt_engine* h, const FusedShape& f, bool fwd, const FusedArgs& a, int grid, cudaStream_t s) {
  FusedShape saved = h->fs;
  h->fs = f;
  int rc = fused_dispatch(h, fwd, a, grid, s);
  h->fs = saved;
  return rc;
}

bool use_tc(tt_engine* h);

int fused_forward(tt_engine* h, float* d_out, cudaStream_t s) {
  const DevCfg& c = h->dc;
  const FusedShape& f = h->fs;
  int rc = ensure_fused(h);
  if (rc) return rc;
  if (f.F >= 2) {
    rc = ensure_generic(h);
    if (rc) return rc;
    const int64_t cap = h->cap;
    for (int k = 1; k < f.F; ++k) {
      const WideShape w = wide_shape(c, k);
      if (w.ok) {
        FusedArgs wa = wide_args(h, k, w.f);
        wa.CH = 0;
        wa.ncb = w.f.ncbf;
        wa.BNj = w.f.BNjf;
        rc = wide_dispatch(h, w.f, true, wa, (int)(c.m[k] * w.f.ncbf), s);
        if (rc) return rc;
        continue;
      }
      const int64_t total = h->capk[k] * c.rows[k] * c.cols[k];
      LAUNCH(k_gen_fwd_level, grid_for(total), 256, 0, s, c, k, h->params, h->L, h->counts, h->digit + k * cap,
             h->parent + k * cap, h->digit, h->seg, h->spos, nullptr, h->st);
    }
  }
  // the fused kernel computes P_F (saved); the last level runs as a streaming
  // kernel over it (k_last_level), then heavy rows are scattered
  FusedArgs a = fused_args(h, nullptr);
  a.CH = 0;
  a.ncb = f.ncbf;
  a.BNj = f.BNjf;
  h->ll_fused = false;
  // TT_FWD_LL=1: the FFMA forward at K = 64, RP = 4, NL = 4 (papers) writes the
  // output rows itself (k_fused_fwd8<..., LL>; measured slower, off by default)
  if (d_out && !use_tc(h) && fwd_ll_enabled() && f.K == 64 && f.RP == 4 && f.NL == 4 && f.BNf == 128 &&
      c.emb_dim % 2 == 0)
    a.out = d_out;
  {
    Phase ph(h, 1, s);
    if (use_tc(h) && f.K == 128) {  // rank 128: the FFMA forward, the tcgen05 backward
      rc = fused_dispatch(h, true, a, (int)(c.m[f.F] * f.ncbf), s);
      h->last_path = 2;
    } else if (use_tc(h)) {
      a.ncb = h->ts.ncbf;
      a.mode = diag().tc_fwd_variant;
      static long long* trace_fwd = nullptr;
      if (diag().trace == 2) {  // TT_TC_TRACE=2: trace the forward instead of the backward
        if (!trace_fwd) cudaMalloc(&trace_fwd, sizeof(long long) * 4096 * 64);
        cudaMemsetAsync(trace_fwd, 0, sizeof(long long) * 4096 * 64, s);
        a.dbg = trace_fwd;
        g_trace_buf = trace_fwd;
      }
      // persistent: one CTA per SM over the (group, column block) items
      static int sms = 0;
      if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      }
      // chunks of large digit groups as in the FFMA kernels (billion: 178 items
      // alone leave the persistent CTAs unevenly loaded)
      a.split = split_for(h, (int)(c.m[f.F] * h->ts.ncbf), f.F, true);
      a.split_rows = split_rows_env(true, 1024);
      const int grid = (int)std::min<int64_t>(c.m[f.F] * h->ts.ncbf * a.split, sms);
      if (false) {
      }
#define TT_TC_FWD_CASE(k_, bn_, rp_, nl_) \
  else if (f.K == k_ && f.RP == rp_ && f.NL == nl_) FUSED_LAUNCH_T((k_tc_fwd<k_, bn_, rp_>), h->ts.smem_fwd, grid, TCF_THREADS, s, a);
      TT_TC_SHAPES(TT_TC_FWD_CASE)
#undef TT_TC_FWD_CASE
      h->fwd_kernel = "k_tc_fwd";
      h->last_path = 2;
    } else if (d_out && lrbwd_enabled() && f.K <= 16 && f.ncbf == 1 &&
               c.emb_dim == (int64_t)f.RP * f.nF * f.NL && c.npad % 4 == 0 && lrfwd_shape(f)) {
      // low-rank streaming forward with the last level (k_lowrank_fwd): a warp
      // per chunk of a digit group's nodes, as the low-rank backward
      FusedArgs al = a;
      al.out = d_out;
      al.split = 4 * LR_SPLIT;  // (no dG_F partials here: chunks of ~1 node keep every warp's ID chain short)
      al.split_rows = f.RP;
      const int groups = (int)c.m[f.F];
      const int lgrid = (int)(((int64_t)groups * al.split + LR_WARPS - 1) / LR_WARPS);
      if (false) {
      }
#define LRF_CASE(k_, rp_, nl_, cpl_) \
  else if (f.K == k_ && f.RP == rp_ && f.NL == nl_ && f.NC == 32 * cpl_) LAUNCH((k_lowrank_fwd<k_, rp_, nl_, cpl_>), lgrid, LR_WARPS * 32, 0, s, al);
      TT_LOWRANK_FWD_SHAPES(LRF_CASE)
#undef LRF_CASE
      h->ll_fused = true;
      h->fwd_kernel = "k_lowrank_fwd";
      rc = TT_OK;
    } else {
      rc = fused_dispatch(h, true, a, (int)(c.m[f.F] * f.ncbf), s);
    }
  }
  if (rc) return rc;
  if (d_out && !h->ll_fused) {
    FusedArgs o = fused_args(h, d_out);
    const int d = c.d;
    const int64_t cap = h->cap;
#define TT_LL_CASE(k_, bn_, rp_, nl_) \
  else if (f.K == k_ && f.NL == nl_ && f.BN == bn_ && f.RP == rp_) { \
    const size_t sm_ = sizeof(float) * SK_WARPS * (f.RP * f.nF * (k_ + 4) + k_ * nl_); \
    const bool pipe_ = (int64_t)f.RP * f.nF * k_ <= 2048, split_ = f.RP * f.nF <= 16; \
    if (pipe_ && split_) { \
      CU(cudaFuncSetAttribute((k_last_level<k_, nl_, true, 2>), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_)); \
      LAUNCH((k_last_level<k_, nl_, true, 2>), 148 * 8, SK_WARPS * 32, sm_, s, o, h->counts, h->parent + (d - 1) * cap); \
    } else if (pipe_) { \
      CU(cudaFuncSetAttribute((k_last_level<k_, nl_, true, 1>), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_)); \
      LAUNCH((k_last_level<k_, nl_, true, 1>), 148 * 8, SK_WARPS * 32, sm_, s, o, h->counts, h->parent + (d - 1) * cap); \
    } else { \
      CU(cudaFuncSetAttribute((k_last_level<k_, nl_, false, 1>), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_)); \
      LAUNCH((k_last_level<k_, nl_, false, 1>), 148 * 8, SK_WARPS * 32, sm_, s, o, h->counts, h->parent + (d - 1) * cap); \
    } \
  }
    if (false) {
    }
    TT_FUSED_SHAPES(TT_LL_CASE)
#undef TT_LL_CASE
  }
  if (d_out)
    LAUNCH(k_scatter_heavy, grid_for((h->B + 31) / 32 * 32, 256, 148 * 8), 256, 0, s, (int)h->B, c.emb_dim, c.npad, h->flag,
           h->spos, h->seg, h->F.Yu, d_out, h->st);
  h->psave_valid = true;
  return TT_OK;
}

int fused_backward(tt_engine* h, const float* d_up, cudaStream_t s) {
  const DevCfg& c = h->dc;
  const FusedShape& f = h->fs;
  const int d = c.d;
  const int64_t cap = h->cap;
  const int64_t chunks = (h->B + DY_CHUNK - 1) / DY_CHUNK;
  if (c.npad <= 128)
    LAUNCH(k_dy_chunks<1>, (int)((chunks + 7) / 8), 256, 0, s, d_up, (int)h->B, c.emb_dim, c.npad, h->flag, h->spos,
           h->seg, h->F.dY, h->F.part, h->st);
  else if (c.npad <= 256)
    LAUNCH(k_dy_chunks<2>, (int)((chunks + 7) / 8), 256, 0, s, d_up, (int)h->B, c.emb_dim, c.npad, h->flag, h->spos,
           h->seg, h->F.dY, h->F.part, h->st);
  else
    LAUNCH(k_dy_chunks<4>, (int)((chunks + 7) / 8), 256, 0, s, d_up, (int)h->B, c.emb_dim, c.npad, h->flag, h->spos,
           h->seg, h->F.dY, h->F.part, h->st);
  LAUNCH(k_dy_groups, (int)(((chunks + 31) / 32 + 7) / 8), 256, 0, s, (int)h->B, c.npad, h->flag, h->seg, h->F.part,
         h->F.gpart, h->F.dY, h->st);
  LAUNCH(k_dy_spans, grid_for(h->capk[d - 1] * 32, 256, 148 * 8), 256, 0, s, h->counts, d, c.npad, h->seg, h->F.part,
         h->F.gpart, h->F.dY, h->st);
  FusedArgs a = fused_args(h, nullptr);
  a.CH = f.CHB;
  a.mode = 0;
  int rc;
  bool wdc_done = false;  // W_u already formed (k_fused_wdc)
  h->lr_w = false;
  // W_u = P_F^T dY_u (k_fused_w) needs only dY and P_F: with TT_AUX_STREAM=1 it
  // runs on a side stream beside the level-F backward, joined before its
  // reduction
  const int WE = f.K * f.NL;
  auto launch_w = [&](cudaStream_t st) -> int {
    FusedArgs aw = a;
    aw.mode = 0;
    if (false) {
    }
#define TT_W_CASE(k_, bn_, rp_, nl_) \
  else if (f.K == k_ && f.NL == nl_ && f.BN == bn_ && f.RP == rp_) { \
    const size_t sm_ = sizeof(float) * SK_WARPS * (f.RP * f.nF * (k_ + 4) + f.RP * f.nF * nl_); \
    if ((int64_t)f.RP * f.nF * k_ <= 2048 && (int64_t)f.RP * f.nF * nl_ <= 256) { \
      CU(cudaFuncSetAttribute((k_fused_w<k_, nl_, true>), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_)); \
      LAUNCH((k_fused_w<k_, nl_, true>), 148 * 8, SK_WARPS * 32, sm_, st, aw, h->counts, h->parent + (d - 1) * cap); \
    } else { \
      CU(cudaFuncSetAttribute((k_fused_w<k_, nl_, false>), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_)); \
      LAUNCH((k_fused_w<k_, nl_, false>), 148 * 8, SK_WARPS * 32, sm_, st, aw, h->counts, h->parent + (d - 1) * cap); \
    } \
  }
    TT_FUSED_SHAPES(TT_W_CASE)
#undef TT_W_CASE
    return TT_OK;
  };
  const bool tc_wdc = h->last_path == 2 && f.K != 128 && (tcbwd_mode(f) == 3 || tcbwd_mode(f) == 4) && wdc_ok(f);
  const bool ffma_wdc = h->last_path != 2 && ffma_wdc_enabled(f) && wdc_ok(f);
  const bool w_side = aux_stream_enabled() && !tc_wdc && !ffma_wdc;
  if (w_side) {
    if (!h->s_aux) {
      CU(cudaStreamCreateWithFlags(&h->s_aux, cudaStreamNonBlocking));
      CU(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    }
    CU(cudaEventRecord(h->ev_fork, s));
    CU(cudaStreamWaitEvent(h->s_aux, h->ev_fork, 0));
    int rcw = launch_w(h->s_aux);
    if (rcw) return rcw;
    CU(cudaEventRecord(h->ev_join, h->s_aux));
  }
  {
    Phase ph(h, 2, s);
    if (h->last_path == 2 && f.K == 128) {
      a.ncb = h->ts.ncbb;
      a.split = split_for(h, (int)(c.m[f.F] * h->ts.ncbb), f.F, false);
      a.split_rows = split_rows_env(false, 128);
      if (a.split > 1) {
        const int64_t need = c.m[f.F] * a.split * c.slice[f.F];
        if (h->F.cap_gsplit < need) {
          cudaFree(h->F.gsplit);
          h->F.gsplit = nullptr;
          h->F.cap_gsplit = 0;
          CU(dalloc(&h->F.gsplit, need));
          h->F.cap_gsplit = need;
        }
        a.gsplit = h->F.gsplit;
      }
      const int grid = (int)(c.m[f.F] * h->ts.ncbb * a.split);
      rc = TT_OK;
      if (false) {
      }
#define TT_TC128_CASE(rp_, nl_) \
  else if (f.RP == rp_ && f.NL == nl_) FUSED_LAUNCH_T((k_tc_bwd128<rp_, nl_>), h->ts.smem_bwd, grid, TCB_THREADS, s, a);
      TT_TC128_SHAPES(TT_TC128_CASE)
#undef TT_TC128_CASE
      if (a.split > 1)
        LAUNCH(k_fused_reduce_gsplit, grid_for(c.m[f.F] * c.slice[f.F] / 4, 256, 148 * 8), 256, 0, s, c, f.F, a.split,
               a.split_rows, a.goffF, (const float*)a.gsplit, a.grads, a.st);
      h->bwd_kernel = "k_tc_bwd128";
    } else if (h->last_path == 2) {
      a.ncb = h->ts.ncbb;
      a.mode = diag().tc_bwd_variant;
      static long long* trace_buf = nullptr;
      if (diag().trace == 1) {
        if (!trace_buf) cudaMalloc(&trace_buf, sizeof(long long) * 4096 * 64);
        cudaMemsetAsync(trace_buf, 0, sizeof(long long) * 4096 * 64, s);
        a.dbg = trace_buf;
        g_trace_buf = trace_buf;
      }
      a.split = split_for(h, (int)(c.m[f.F] * h->ts.ncbb), f.F, false);
      a.split_rows = split_rows_env(false, 128);
      if (a.split > 1) {
        const int64_t need = c.m[f.F] * a.split * c.slice[f.F];
        if (h->F.cap_gsplit < need) {
          cudaFree(h->F.gsplit);
          h->F.gsplit = nullptr;
          h->F.cap_gsplit = 0;
          CU(dalloc(&h->F.gsplit, need));
          h->F.cap_gsplit = need;
        }
        a.gsplit = h->F.gsplit;
      }
      const int grid = (int)(c.m[f.F] * h->ts.ncbb * a.split);
      rc = TT_OK;
      const int mode = tcbwd_mode(f);
      if ((mode == 3 || mode == 4) && wdc_ok(f)) {
        const int64_t cap = h->cap;
        const size_t sm_ = sizeof(float) * SK_WARPS * (f.RP * f.nF * (f.K + 4) + f.RP * f.nF * f.NL);
        if (false) {
        }
#define TT_WDC_CASE(k_, nl_)                                                                                        \
  else if (f.K == k_ && f.NL == nl_) {                                                                              \
    CU(cudaFuncSetAttribute((k_fused_wdc<k_, nl_>), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_));       \
    LAUNCH((k_fused_wdc<k_, nl_>), h->nsm, SK_WARPS * 32, sm_, s, a, h->counts, h->parent + (d - 1) * cap);    \
  }
        TT_WDC_CASE(64, 4) TT_WDC_CASE(64, 8) TT_WDC_CASE(32, 4) TT_WDC_CASE(32, 8)
#undef TT_WDC_CASE
        wdc_done = true;
        h->psave_valid = false;
        const int pgrid = std::min(grid, h->nsm);
        if (mode == 4 && psave_tmap(h)) {
          const size_t smem3 = tc_bwd3_smem(f.K, 128);
          if (false) {
          }
#define TT_TC_BWD4_CASE(k_, bn_, rp_, nl_)                                                                   \
  else if (f.K == k_ && f.RP == rp_ && f.NL == nl_) {                                                        \
    CU(cudaFuncSetAttribute((k_tc_bwd3<k_, 128, rp_, nl_>), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3)); \
    tt_launch((k_tc_bwd3<k_, 128, rp_, nl_>), dim3(pgrid), dim3(TCB3_THREADS), smem3, s, a, h->ps_tmap);    \
    ++h->launches;                                                                                           \
  }
          TT_TC_SHAPES(TT_TC_BWD4_CASE)
#undef TT_TC_BWD4_CASE
          h->bwd_kernel = "k_tc_bwd3";
        } else {
          const size_t smem2 = tc_bwd2_smem(f.K, 128);
          if (false) {
          }
#define TT_TC_BWD3_CASE(k_, bn_, rp_, nl_) \
  else if (f.K == k_ && f.RP == rp_ && f.NL == nl_) FUSED_LAUNCH_T((k_tc_bwd2<k_, 128, rp_, nl_, true>), smem2, pgrid, TCB2_THREADS, s, a);
          TT_TC_SHAPES(TT_TC_BWD3_CASE)
#undef TT_TC_BWD3_CASE
          h->bwd_kernel = "k_tc_bwd2";
        }
      } else if (mode == 2) {
        const int pgrid = std::min(grid, h->nsm);
        const size_t smem2 = tc_bwd2_smem(f.K, 128);
        if (false) {
        }
#define TT_TC_BWD2_CASE(k_, bn_, rp_, nl_) \
  else if (f.K == k_ && f.RP == rp_ && f.NL == nl_) FUSED_LAUNCH_T((k_tc_bwd2<k_, 128, rp_, nl_, false>), smem2, pgrid, TCB2_THREADS, s, a);
        TT_TC_SHAPES(TT_TC_BWD2_CASE)
#undef TT_TC_BWD2_CASE
        h->bwd_kernel = "k_tc_bwd2";
      } else {
        if (false) {
        }
#define TT_TC_BWD_CASE(k_, bn_, rp_, nl_) \
  else if (f.K == k_ && f.RP == rp_ && f.NL == nl_) FUSED_LAUNCH_T((k_tc_bwd<k_, 128, rp_, nl_>), h->ts.smem_bwd, grid, TCB_THREADS, s, a);
        TT_TC_SHAPES(TT_TC_BWD_CASE)
#undef TT_TC_BWD_CASE
        h->bwd_kernel = "k_tc_bwd";
      }
      if (a.split > 1)
        LAUNCH(k_fused_reduce_gsplit, grid_for(c.m[f.F] * c.slice[f.F] / 4, 256, 148 * 8), 256, 0, s, c, f.F, a.split,
               a.split_rows, a.goffF, (const float*)a.gsplit, a.grads, a.st);
    } else {
      static long long* trace_buf2 = nullptr;
      if (diag().trace == 1) {
        if (!trace_buf2) cudaMalloc(&trace_buf2, sizeof(long long) * 4096 * 64);
        cudaMemsetAsync(trace_buf2, 0, sizeof(long long) * 4096 * 64, s);
        a.dbg = trace_buf2;
        g_trace_buf = trace_buf2;
      }
      if (ffma_wdc_enabled(f) && wdc_ok(f)) {  // dC (and W_u) streamed over P_F first; the GEMM kernel loads dC
        const int64_t cap = h->cap;
        const size_t sm_ = sizeof(float) * SK_WARPS * (f.RP * f.nF * (f.K + 4) + f.RP * f.nF * f.NL);
        if (false) {
        }
#define TT_WDC_CASE(k_, nl_)                                                                                        \
  else if (f.K == k_ && f.NL == nl_) {                                                                              \
    CU(cudaFuncSetAttribute((k_fused_wdc<k_, nl_>), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_));       \
    LAUNCH((k_fused_wdc<k_, nl_>), h->nsm, SK_WARPS * 32, sm_, s, a, h->counts, h->parent + (d - 1) * cap);        \
  }
        TT_WDC_CASE(64, 4) TT_WDC_CASE(64, 8) TT_WDC_CASE(32, 4) TT_WDC_CASE(32, 8)
#undef TT_WDC_CASE
        wdc_done = true;
        h->psave_valid = false;
        a.mode = 1;
        a.dPin = h->F.Psave;
      }
      rc = fused_dispatch(h, false, a, (int)(c.m[f.F] * f.ncb), s);
    }
  }
  if (rc) return rc;
  if (h->comm) {  // dG_F is final here: its all-reduce may start (tt_allreduce_grads)
    CU(cudaEventRecord(h->ev_gF, s));
    h->gF_ready = true;
  }
  Phase ph_aux(h, 3, s);
  if (w_side) {
    CU(cudaStreamWaitEvent(s, h->ev_join, 0));
  } else if (!wdc_done && !h->lr_w) {
    rc = launch_w(s);
    if (rc) return rc;
  }
  // wide W rows (128+ float4 columns): 1024 threads, so several sub-groups
  // split each digit group's rows
  if (WE / 4 >= 128)
    LAUNCH(k_fused_reduce_last<1024>, (int)c.m[d - 1], 1024, 0, s, c, 1, WE, h->goff[d - 1], h->order[d - 1], h->F.W,
           h->grads, h->st);
  else
    LAUNCH(k_fused_reduce_last<256>, (int)c.m[d - 1], 256, 0, s, c, 1, WE, h->goff[d - 1], h->order[d - 1], h->F.W,
           h->grads, h->st);
  const int per = f.RP * f.K;
  float* dst = f.F == 1 ? h->grads : h->L.dP[f.F - 1];
  // 128-thread blocks: twice the blocks of a parent-per-block grid, a smaller
  // tail over the SMs (each block streams a contiguous run of partials)
  LAUNCH(k_fused_reduce_children, grid_for(h->capk[f.F - 1] * per, 128, 148 * 64), 128, 0, s, c, f.F, f.ncb, per,
         h->counts, h->cstart + (f.F - 1) * (cap + 1), h->digit, h->F.dPc, dst, h->st);
  for (int k = f.F - 1; k >= 1; --k) {
    const WideShape w = wide_shape(c, k);
    if (w.ok) {
      if (!h->F.dPcw || h->F.cap_w < h->capk[k] * w.f.ncb * w.f.RP * w.f.K) {
        cudaFree(h->F.dPcw);
        h->F.cap_w = h->capk[k] * w.f.ncb * w.f.RP * w.f.K;
        CU(dalloc(&h->F.dPcw, h->F.cap_w));
      }
      FusedArgs wa = wide_args(h, k, w.f);
      wa.dPc = h->F.dPcw;
      rc = wide_dispatch(h, w.f, false, wa, (int)(c.m[k] * w.f.ncb), s);
      if (rc) return rc;
      const int wper = w.f.RP * w.f.K;
      float* wdst = k == 1 ? h->grads : h->L.dP[k - 1];
      LAUNCH(k_fused_reduce_children, grid_for(h->capk[k - 1] * wper), 256, 0, s, c, k, w.f.ncb, wper, h->counts,
             h->cstart + (k - 1) * (cap + 1), h->digit, h->F.dPcw, wdst, h->st);
      continue;
    }
    LAUNCH(k_gen_bwd_input, grid_for(h->capk[k] * c.rows[k] * c.R[k]), 256, 0, s, c, k, h->params, h->L, h->counts,
           h->digit + k * cap, h->st);
    LAUNCH(k_gen_bwd_weight, grid_for(c.m[k] * c.R[k] * c.cols[k]), 256, 0, s, c, k, h->params, h->L, h->goff[k],
           h->order[k], h->parent + k * cap, h->digit, h->grads, h->st);
    LAUNCH(k_gen_reduce_children, grid_for(h->capk[k - 1] * c.rows[k] * c.R[k]), 256, 0, s, c, k, h->L, h->counts,
           h->cstart + (k - 1) * (cap + 1), h->st);
  }
  if (f.F >= 2 && !wide_shape(c, 1).ok)
    LAUNCH(k_gen_bwd_core0, grid_for(h->capk[0] * c.cols[0]), 256, 0, s, c, h->L, h->counts, h->digit, h->grads,
           h->st);
  return TT_OK;
}

void touch_counters(tt_engine* h, cudaStream_t s) {
  const DevCfg& c = h->dc;
  GoffPtrs gp{};
  int64_t mmax = 0;
  for (int k = 0; k < c.d; ++k) {
    gp.goff[k] = h->goff[k];
    mmax = std::max<int64_t>(mmax, c.m[k]);
  }
  LAUNCH(k_touch_counters, dim3(grid_for(mmax, 256, INT_MAX), c.d), 256, 0, s, c, gp, h->grads, 0, h->st);
}

bool use_fused(tt_engine* h) { return h->path_pref != 1 && h->fused_ok; }
bool use_tc(tt_engine* h) { return h->path_pref == 2 && h->tc_ok; }

int do_forward(tt_engine* h, const int64_t* d_idx, int64_t B, float* d_out, cudaStream_t s, bool write_out) {
  LAUNCH(k_reset_status, 1, 1, 0, s, h->st, 1);
  int rc = build_plan(h, d_idx, B, s);
  if (rc) return rc;
  if (use_fused(h)) {
    h->last_path = 1;
    rc = fused_forward(h, write_out ? d_out : nullptr, s);
  } else {
    rc = gen_forward(h, write_out ? d_out : nullptr, s);
    h->last_path = 0;
  }
  if (rc) return rc;
  h->plan_valid = true;
  h->plan_version = h->cores_version;
  CU(cudaGetLastError());
  return TT_OK;
}

int do_backward(tt_engine* h, const float* d_up, cudaStream_t s) {
  h->gF_ready = false;
  if (h->dense) CU(cudaMemsetAsync(h->grads, 0, sizeof(float) * (size_t)(h->dc.nparams + h->ntc), s));
  int rc;
  if (h->last_path >= 1 && !h->psave_valid) {  // a second backward of one forward: P_F again
    rc = fused_forward(h, nullptr, s);
    if (rc) return rc;
  }
  if (h->last_path >= 1)
    rc = fused_backward(h, d_up, s);
  else
    rc = gen_backward(h, d_up, s);
  if (rc) return rc;
  touch_counters(h, s);
  h->batch_count = h->B;
  CU(cudaGetLastError());
  return TT_OK;
}

int set_cfg(tt_engine* h, const tt_config_c* in) {
  h->cfg = *in;
  DevCfg& c = h->dc;
  memset(&c, 0, sizeof(c));
  c.d = in->d;
  c.num_nodes = in->num_nodes;
  c.emb_dim = in->emb_dim;
  c.npad = 1;
  for (int k = 0; k < c.d; ++k) {
    c.m[k] = in->row_factors[k];
    c.n[k] = in->col_factors[k];
    c.npad *= c.n[k];
  }
  for (int k = 0; k <= c.d; ++k) c.R[k] = in->ranks[k];
  int64_t acc = 1;
  for (int k = c.d - 1; k >= 0; --k) { c.S[k] = acc; acc *= c.m[k]; }
  acc = 1;
  int64_t off = 0;
  for (int k = 0; k < c.d; ++k) {
    c.rows[k] = acc;
    acc *= c.n[k];
    c.cols[k] = c.n[k] * c.R[k + 1];
    c.slice[k] = c.R[k] * c.cols[k];
    c.core_off[k] = off;
    off += c.m[k] * c.slice[k];
  }
  c.nparams = off;
  int64_t toff = off;
  for (int k = 0; k < c.d; ++k) { c.tc_off[k] = toff; toff += c.m[k]; }
  h->ntc = toff - off;
  return TT_OK;
}

int validate_cfg(const tt_config_c* c, std::string* why) {
  auto bad = [&](const char* m) { if (why) *why = m; return TT_ERR_ARG; };
  if (!c) return bad("TTConfig: null config");
  if (c->num_nodes <= 0) return bad("TTConfig: num_nodes must be positive");
  if (c->emb_dim <= 0) return bad("TTConfig: emb_dim must be positive");
  if (c->d < 2) return bad("TTConfig: need at least 2 cores");
  if (c->d > TT_MAX_CORES) return bad("TTConfig: at most TT_MAX_CORES cores supported");
  if (c->ranks[0] != 1 || c->ranks[c->d] != 1) return bad("TTConfig: boundary ranks R_0 and R_d must be 1");
  for (int k = 0; k <= c->d; ++k)
    if (c->ranks[k] <= 0) return bad("TTConfig: ranks must be positive");
  long double pr = 1, pc = 1;
  for (int k = 0; k < c->d; ++k) {
    if (c->row_factors[k] <= 0 || c->col_factors[k] <= 0) return bad("TTConfig: factors must be positive");
    pr *= c->row_factors[k];
    pc *= c->col_factors[k];
  }
  if (pr < c->num_nodes) return bad("TTConfig: prod(row_factors) < num_nodes");
  if (pc < c->emb_dim) return bad("TTConfig: prod(col_factors) < emb_dim");
  if (pr > 9.0e18L) return bad("TTConfig: prod(row_factors) overflows int64");
  return TT_OK;
}

// index into the reference layout (R_{k-1}, m, n, R_k) from the device
// layout [m][R_{k-1}][n][R_k]
inline int64_t dev_index(const DevCfg& c, int k, int64_t r, int64_t i, int64_t j, int64_t s) {
  return ((i * c.R[k] + r) * c.n[k] + j) * c.R[k + 1] + s;
}

template <class T>
void to_device_layout(const DevCfg& c, const T* const* cores, std::vector<float>& out) {
  out.assign((size_t)c.nparams, 0.f);
  for (int k = 0; k < c.d; ++k) {
    const T* src = cores[k];
    float* dst = out.data() + c.core_off[k];
    int64_t e = 0;
    for (int64_t r = 0; r < c.R[k]; ++r)
      for (int64_t i = 0; i < c.m[k]; ++i)
        for (int64_t j = 0; j < c.n[k]; ++j)
          for (int64_t s = 0; s < c.R[k + 1]; ++s) dst[dev_index(c, k, r, i, j, s)] = (float)src[e++];
  }
}

template <class T>
void from_device_layout(const DevCfg& c, const std::vector<float>& in, T* const* cores, const float* tc) {
  for (int k = 0; k < c.d; ++k) {
    T* dst = cores[k];
    const float* src = in.data() + c.core_off[k];
    int64_t e = 0;
    for (int64_t r = 0; r < c.R[k]; ++r)
      for (int64_t i = 0; i < c.m[k]; ++i) {
        const bool live = !tc || tc[c.tc_off[k] - c.nparams + i] > 0.f;
        for (int64_t j = 0; j < c.n[k]; ++j)
          for (int64_t s = 0; s < c.R[k + 1]; ++s) dst[e++] = live ? (T)src[dev_index(c, k, r, i, j, s)] : (T)0;
      }
  }
}

int ensure_stage(tt_engine* h, int64_t B) {
  if (B <= h->stage_cap) return TT_OK;
  cudaFree(h->st_idx); cudaFree(h->st_out); cudaFree(h->st_up);
  const int64_t cap = std::max<int64_t>(B, 1024);
  CU(dalloc(&h->st_idx, cap));
  CU(dalloc(&h->st_out, cap * h->dc.emb_dim));
  CU(dalloc(&h->st_up, cap * h->dc.emb_dim));
  h->stage_cap = cap;
  return TT_OK;
}

int read_status(tt_engine* h, cudaStream_t s) {
  CU(cudaStreamSynchronize(s));
  DevStatus st;
  CU(cudaMemcpy(&st, h->st, sizeof(st), cudaMemcpyDeviceToHost));
  if (st.bad_pos != TT_NO_POS) {
    int64_t val = 0;
    if (h->last_idx) cudaMemcpy(&val, h->last_idx + st.bad_pos, sizeof(val), cudaMemcpyDeviceToHost);
    LAUNCH(k_reset_status, 1, 1, 0, s, h->st, 3);
    CU(cudaStreamSynchronize(s));
    h->plan_valid = false;
    return fail(TT_ERR_INDEX,
                "lookup_batch: index " + std::to_string(val) + " at batch position " +
                    std::to_string((long long)st.bad_pos) + " out of [0, " + std::to_string(h->dc.num_nodes) + ")",
                (int64_t)st.bad_pos, val);
  }
  if (st.bad_core != INT_MAX) {
    LAUNCH(k_reset_status, 1, 1, 0, s, h->st, 2);
    CU(cudaStreamSynchronize(s));
    return fail(TT_ERR_NONFINITE,
                "apply_update: non-finite gradient in core " + std::to_string(st.bad_core) + "; update rejected",
                st.bad_core);
  }
  return TT_OK;
}

}  // namespace

// ============================================================================
extern "C" {

int tt_config_validate(const tt_config_c* cfg) {
  std::string why;
  int rc = validate_cfg(cfg, &why);
  return rc ? fail(rc, why) : TT_OK;
}

int64_t tt_count_params(const tt_config_c* cfg) {
  if (validate_cfg(cfg, nullptr)) return -1;
  int64_t t = 0;
  for (int k = 0; k < cfg->d; ++k)
    t += cfg->ranks[k] * cfg->row_factors[k] * cfg->col_factors[k] * cfg->ranks[k + 1];
  return t;
}

int tt_engine_create(const tt_config_c* cfg, int device, tt_engine** out) {
  if (!out) return fail(TT_ERR_ARG, "tt_engine_create: null output handle");
  *out = nullptr;
  std::string why;
  if (validate_cfg(cfg, &why)) return fail(TT_ERR_ARG, why);
  CU(cudaSetDevice(device));
  tt_engine* h = new tt_engine();
  h->device = device;
  set_cfg(h, cfg);
  cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, device);
  auto cleanup = [&](int code) { tt_engine_destroy(h); return code; };
  if (cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking) != cudaSuccess) return cleanup(fail(TT_ERR_CUDA, "stream"));
  if (dalloc(&h->params, h->dc.nparams) || dalloc(&h->own_grads, h->dc.nparams + h->ntc) ||
      dalloc(&h->d_step, 1) || dalloc(&h->st, 1) || dalloc(&h->counts, 2 * TT_MAXD))
    return cleanup(fail(TT_ERR_NOMEM, "tt_engine_create: device allocation failed"));
  h->grads = h->own_grads;
  cudaMemset(h->params, 0, sizeof(float) * (size_t)h->dc.nparams);
  cudaMemset(h->grads, 0, sizeof(float) * (size_t)(h->dc.nparams + h->ntc));
  cudaMemset(h->d_step, 0, sizeof(long long));
  cudaMemset(h->counts, 0, sizeof(int) * 2 * TT_MAXD);
  DevStatus st0{TT_NO_POS, INT_MAX, 0};
  cudaMemcpy(h->st, &st0, sizeof(st0), cudaMemcpyHostToDevice);
  h->fused_ok = fused_plan_shape(h->dc, &h->fs) &&
                h->fs.smem_bwd <= 227 * 1024 && h->fs.smem_fwd <= 227 * 1024;
  h->tc_ok = h->fused_ok && tc_plan_shape(h->fs, &h->ts);
  if (cudaGetLastError() != cudaSuccess) return cleanup(fail(TT_ERR_CUDA, "tt_engine_create: CUDA error"));
  *out = h;
  return TT_OK;
}

void tt_engine_destroy(tt_engine* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->own) cudaStreamSynchronize(h->own);
  free_plan(h);
  for (auto& v : h->prof_ev)
    for (auto& pr : v) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  void* ptrs[] = {h->params, h->own_grads, h->snap, h->s1, h->s2, h->d_step, h->st, h->counts, h->st_idx, h->st_out, h->st_up,
                  h->perm};
  for (void* p : ptrs) cudaFree(p);
  for (auto& sl : h->hs) {
    for (cudaEvent_t e : {sl.ev_done, sl.ev_out})
      if (e) cudaEventSynchronize(e);
    cudaFree(sl.idx); cudaFree(sl.up); cudaFree(sl.out);
    if (sl.h_st) cudaFreeHost(sl.h_st);
    for (cudaEvent_t e : {sl.ev_idx, sl.ev_up, sl.ev_fwd, sl.ev_done, sl.ev_out})
      if (e) cudaEventDestroy(e);
  }
  {
    auto& o = h->ow;
    void* ptrs2[] = {o.ka, o.kb, o.va, o.vb, o.sid, o.d_counts, o.d_all, o.d_gbad, o.rid, o.rout, o.back, o.sup, o.rup};
    for (void* p : ptrs2) cudaFree(p);
    if (o.h_all) cudaFreeHost(o.h_all);
  }
  if (h->own) cudaStreamDestroy(h->own);
  if (h->s_comm) { cudaStreamSynchronize(h->s_comm); cudaStreamDestroy(h->s_comm); }
  for (cudaEvent_t e : {h->ev_gF, h->ev_bwd, h->ev_comm})
    if (e) cudaEventDestroy(e);
  if (h->comm && h->own_comm && nccl().ok) nccl().CommDestroy(h->comm);
  if (h->s_h2d) { cudaStreamSynchronize(h->s_h2d); cudaStreamDestroy(h->s_h2d); }
  if (h->s_d2h) { cudaStreamSynchronize(h->s_d2h); cudaStreamDestroy(h->s_d2h); }
  if (h->s_aux) {
    cudaStreamSynchronize(h->s_aux);
    cudaStreamDestroy(h->s_aux);
    cudaEventDestroy(h->ev_fork);
    cudaEventDestroy(h->ev_join);
  }
  for (cudaEvent_t e : {h->ev_up, h->ev_fwd, h->ev_in})
    if (e) cudaEventDestroy(e);
  delete h;
}

int tt_set_cores_f64(tt_engine* h, const double* const* cores) {
  if (!h || !cores) return fail(TT_ERR_ARG, "tt_set_cores: null argument");
  std::vector<float> buf;
  to_device_layout(h->dc, cores, buf);
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(h->params, buf.data(), buf.size() * sizeof(float), cudaMemcpyHostToDevice));
  ++h->cores_version;
  return TT_OK;
}

int tt_set_cores_f32(tt_engine* h, const float* const* cores) {
  if (!h || !cores) return fail(TT_ERR_ARG, "tt_set_cores: null argument");
  std::vector<float> buf;
  to_device_layout(h->dc, cores, buf);
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(h->params, buf.data(), buf.size() * sizeof(float), cudaMemcpyHostToDevice));
  ++h->cores_version;
  return TT_OK;
}

int tt_get_cores_f64(tt_engine* h, double* const* cores) {
  if (!h || !cores) return fail(TT_ERR_ARG, "tt_get_cores: null argument");
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  std::vector<float> buf((size_t)h->dc.nparams);
  CU(cudaMemcpy(buf.data(), h->params, buf.size() * sizeof(float), cudaMemcpyDeviceToHost));
  from_device_layout(h->dc, buf, cores, nullptr);
  return TT_OK;
}

int tt_get_cores_f32(tt_engine* h, float* const* cores) {
  if (!h || !cores) return fail(TT_ERR_ARG, "tt_get_cores: null argument");
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  std::vector<float> buf((size_t)h->dc.nparams);
  CU(cudaMemcpy(buf.data(), h->params, buf.size() * sizeof(float), cudaMemcpyDeviceToHost));
  from_device_layout(h->dc, buf, cores, nullptr);
  return TT_OK;
}

int tt_get_core_grads_f64(tt_engine* h, double* const* grads, int64_t* batch_count) {
  if (!h || !grads) return fail(TT_ERR_ARG, "tt_get_core_grads: null argument");
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  std::vector<float> buf((size_t)(h->dc.nparams + h->ntc));
  CU(cudaMemcpy(buf.data(), h->grads, buf.size() * sizeof(float), cudaMemcpyDeviceToHost));
  from_device_layout(h->dc, buf, grads, buf.data() + h->dc.nparams);
  if (batch_count) *batch_count = h->batch_count;
  return TT_OK;
}

// Optimizer state in the reference layout (R_{k-1}, m_k, n_k, R_k): s1 is the
// Adagrad accumulator / Adam first moment, s2 the Adam second moment (NULL
// where the optimizer has none).  A checkpoint of these plus the cores and the
// step counter resumes training bit-exactly (the reference has no resume,
// SPEC.md:102; tt_io.py writes them next to the TTE1 core file).
// Node relabelling: after a hierarchical reorder
// (partition.cpp:428-552 -> graph.cpp:218-252 apply_permutation) node v's row
// is perm[v]; with a permutation set, every lookup / backward maps its IDs
// through it on the device.  perm must be a bijection on [0, num_nodes);
// NULL (or n == 0) clears it.
// init_ortho_core (initializer.cpp:103-132) on the device: fp64 cores in the
// reference layout, written to host buffers (the caller sets them into an
// engine, as the reference's initializer returns a TTEmbedding).
int tt_ortho_cores_f64(const tt_config_c* cfgc, int device, uint64_t seed, double target_scale,
                       double* const* cores, int64_t* bad) {
  std::string why;
  if (validate_cfg(cfgc, &why)) return fail(TT_ERR_ARG, why);
  if (!cores) return fail(TT_ERR_ARG, "tt_ortho_cores_f64: null output");
  const int d = cfgc->d;
  for (int k = 0; k < d; ++k) {
    const int64_t count = cfgc->col_factors[k] * cfgc->ranks[k];
    const int64_t dim = cfgc->row_factors[k] * cfgc->ranks[k + 1];
    if (count > dim) {
      if (bad) { bad[0] = k; bad[1] = count; bad[2] = dim; }
      return fail(TT_ERR_ARG, "ortho-core init infeasible at core " + std::to_string(k) + ": needs " +
                                  std::to_string(count) + " orthonormal vectors of length " + std::to_string(dim) +
                                  " (require n_k*R_{k-1} <= m_k*R_k)", k, count);
    }
  }
  if (target_scale < 0.0) return fail(TT_ERR_ARG, "target_scale must be positive");  // 0: no rescaling
  CU(cudaSetDevice(device));
  const double c = target_scale > 0.0 ? std::pow(target_scale, 1.0 / (2.0 * d)) : 1.0;
  for (int k = 0; k < d; ++k) {
    const int64_t rp = cfgc->ranks[k], rn = cfgc->ranks[k + 1], m = cfgc->row_factors[k], n = cfgc->col_factors[k];
    const int64_t count = n * rp, dim = m * rn;
    double *Q = nullptr, *dots = nullptr, *sc = nullptr;
    CU(cudaMalloc(&Q, sizeof(double) * (size_t)(count * dim)));
    CU(cudaMalloc(&dots, sizeof(double) * (size_t)std::max<int64_t>(count, 1)));
    CU(cudaMalloc(&sc, sizeof(double)));
    auto cleanup = [&] { cudaFree(Q); cudaFree(dots); cudaFree(sc); };
    const int gdim = (int)std::min<int64_t>((dim + 255) / 256, 148 * 8);
    for (int64_t i = 0; i < count; ++i) {
      double* v = Q + i * dim;
      bool placed = false;
      for (int attempt = 0; attempt < 8 && !placed; ++attempt) {
        k_gs_draw<<<gdim, 256>>>(v, dim, (unsigned long long)seed, k, (int)i, attempt);
        k_gs_sumsq<<<1, 256>>>(v, dim, sc);
        double raw2 = 0, nrm2 = 0;
        if (cudaMemcpy(&raw2, sc, sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) { cleanup(); return fail(TT_ERR_CUDA, "ortho init"); }
        for (int pass = 0; pass < 2 && i > 0; ++pass) {
          k_gs_dots<<<(int)i, 256>>>(Q, v, dim, dots);
          k_gs_axpy<<<gdim, 256>>>(Q, v, dim, dots, (int)i);
        }
        k_gs_sumsq<<<1, 256>>>(v, dim, sc);
        if (cudaMemcpy(&nrm2, sc, sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) { cleanup(); return fail(TT_ERR_CUDA, "ortho init"); }
        const double raw = std::sqrt(raw2), nrm = std::sqrt(nrm2);
        if (nrm > 1e-10 * raw && nrm > 0.0) {
          k_gs_scale<<<gdim, 256>>>(v, dim, 1.0 / nrm);
          placed = true;
        }
      }
      if (!placed) {
        cleanup();
        return fail(TT_ERR_STATE, "gram_schmidt_rows: degenerate draws for vector " + std::to_string(i) + " after 8 retries");
      }
    }
    std::vector<double> hq((size_t)(count * dim));
    const cudaError_t e = cudaMemcpy(hq.data(), Q, sizeof(double) * hq.size(), cudaMemcpyDeviceToHost);
    cleanup();
    if (e != cudaSuccess) return fail(TT_ERR_CUDA, std::string("ortho init: ") + cudaGetErrorString(e));
    // vector (r, j) becomes the slice G_k(r, :, j, :), reshaped (m, R_k)
    double* core = cores[k];
    for (int64_t r = 0; r < rp; ++r)
      for (int64_t j = 0; j < n; ++j) {
        const double* vec = hq.data() + (r * n + j) * dim;
        for (int64_t i2 = 0; i2 < m; ++i2)
          for (int64_t s2 = 0; s2 < rn; ++s2) core[((r * m + i2) * n + j) * rn + s2] = c * vec[i2 * rn + s2];
      }
  }
  return TT_OK;
}

int tt_set_permutation(tt_engine* h, const int64_t* perm, int64_t n) {
  if (!h) return fail(TT_ERR_ARG, "tt_set_permutation: null handle");
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  if (!perm || n == 0) {
    cudaFree(h->perm);
    h->perm = nullptr;
    h->plan_valid = false;
    return TT_OK;
  }
  if (n != h->dc.num_nodes) return fail(TT_ERR_ARG, "apply_permutation: permutation size mismatch");
  if (n > INT_MAX) return fail(TT_ERR_ARG, "tt_set_permutation: more than 2^31 nodes");
  std::vector<int> p32((size_t)n);
  std::vector<unsigned char> seen((size_t)n, 0);
  for (int64_t v = 0; v < n; ++v) {
    const int64_t t = perm[v];
    if (t < 0 || t >= n || seen[(size_t)t])
      return fail(TT_ERR_ARG, "tt_set_permutation: not a permutation of [0, num_nodes) (entry " + std::to_string(v) + ")");
    seen[(size_t)t] = 1;
    p32[(size_t)v] = (int)t;
  }
  if (!h->perm) CU(dalloc(&h->perm, n));
  CU(cudaMemcpy(h->perm, p32.data(), sizeof(int) * (size_t)n, cudaMemcpyHostToDevice));
  h->plan_valid = false;
  return TT_OK;
}

int tt_opt_state_get_f64(tt_engine* h, double* const* s1, double* const* s2, int64_t* step) {
  if (!h) return fail(TT_ERR_ARG, "tt_opt_state_get: null handle");
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  std::vector<float> buf((size_t)h->dc.nparams);
  if (s1 && h->s1) {
    CU(cudaMemcpy(buf.data(), h->s1, buf.size() * sizeof(float), cudaMemcpyDeviceToHost));
    from_device_layout(h->dc, buf, s1, nullptr);
  }
  if (s2 && h->s2) {
    CU(cudaMemcpy(buf.data(), h->s2, buf.size() * sizeof(float), cudaMemcpyDeviceToHost));
    from_device_layout(h->dc, buf, s2, nullptr);
  }
  if (step) {
    long long v = 0;
    CU(cudaMemcpy(&v, h->d_step, sizeof(v), cudaMemcpyDeviceToHost));
    *step = v;
  }
  return TT_OK;
}

int tt_opt_state_set_f64(tt_engine* h, const double* const* s1, const double* const* s2, int64_t step) {
  if (!h) return fail(TT_ERR_ARG, "tt_opt_state_set: null handle");
  if (step < 0) return fail(TT_ERR_ARG, "tt_opt_state_set: negative step");
  if ((s1 && !h->s1) || (s2 && !h->s2))
    return fail(TT_ERR_STATE, "tt_opt_state_set: the configured optimizer has no such state (call tt_opt_init)");
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  std::vector<float> buf;
  if (s1) {
    to_device_layout(h->dc, s1, buf);
    CU(cudaMemcpy(h->s1, buf.data(), buf.size() * sizeof(float), cudaMemcpyHostToDevice));
  }
  if (s2) {
    to_device_layout(h->dc, s2, buf);
    CU(cudaMemcpy(h->s2, buf.data(), buf.size() * sizeof(float), cudaMemcpyHostToDevice));
  }
  const long long v = step;
  CU(cudaMemcpy(h->d_step, &v, sizeof(v), cudaMemcpyHostToDevice));
  return TT_OK;
}

int tt_cores_snapshot(tt_engine* h, void* stream) {
  if (!h) return fail(TT_ERR_ARG, "tt_cores_snapshot: null handle");
  CU(cudaSetDevice(h->device));
  if (!h->snap) CU(dalloc(&h->snap, h->dc.nparams));
  CU(cudaMemcpyAsync(h->snap, h->params, sizeof(float) * (size_t)h->dc.nparams, cudaMemcpyDeviceToDevice,
                     (cudaStream_t)stream));
  return TT_OK;
}

int tt_cores_restore(tt_engine* h, void* stream) {
  if (!h) return fail(TT_ERR_ARG, "tt_cores_restore: null handle");
  if (!h->snap) return fail(TT_ERR_STATE, "tt_cores_restore: no snapshot");
  CU(cudaSetDevice(h->device));
  CU(cudaMemcpyAsync(h->params, h->snap, sizeof(float) * (size_t)h->dc.nparams, cudaMemcpyDeviceToDevice,
                     (cudaStream_t)stream));
  ++h->cores_version;
  return TT_OK;
}

int tt_set_core_grads_f64(tt_engine* h, const double* const* grads, int64_t batch_count) {
  if (!h || !grads) return fail(TT_ERR_ARG, "tt_set_core_grads: null argument");
  std::vector<float> buf;
  to_device_layout(h->dc, grads, buf);
  buf.resize((size_t)(h->dc.nparams + h->ntc), 1.f);  // all slices touched
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(h->grads, buf.data(), buf.size() * sizeof(float), cudaMemcpyHostToDevice));
  h->batch_count = batch_count;
  return TT_OK;
}

int tt_opt_init(tt_engine* h, int kind, double lr, double beta1, double beta2, double eps) {
  if (!h) return fail(TT_ERR_ARG, "tt_opt_init: null handle");
  if (kind < 0 || kind > 2) return fail(TT_ERR_ARG, "tt_opt_init: unknown optimizer kind");
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  h->opt_kind = kind;
  h->lr = lr;
  h->beta1 = beta1 > 0 ? beta1 : 0.9;
  h->beta2 = beta2 > 0 ? beta2 : 0.999;
  h->eps = eps > 0 ? eps : (kind == TT_OPT_ADAGRAD ? 1e-10 : 1e-8);
  // state buffers are kept (zeroed) when the kind needs them, so device
  // pointers captured in a CUDA graph stay valid across re-initialisation
  if (kind == TT_OPT_SGD) { cudaFree(h->s1); h->s1 = nullptr; }
  if (kind != TT_OPT_ADAM) { cudaFree(h->s2); h->s2 = nullptr; }
  if (kind != TT_OPT_SGD) {
    if (!h->s1) CU(dalloc(&h->s1, h->dc.nparams));
    CU(cudaMemset(h->s1, 0, sizeof(float) * (size_t)h->dc.nparams));
  }
  if (kind == TT_OPT_ADAM) {
    if (!h->s2) CU(dalloc(&h->s2, h->dc.nparams));
    CU(cudaMemset(h->s2, 0, sizeof(float) * (size_t)h->dc.nparams));
  }
  CU(cudaMemset(h->d_step, 0, sizeof(long long)));
  return TT_OK;
}

int tt_opt_set_hparams(tt_engine* h, double lr, double beta1, double beta2, double eps) {
  if (!h) return fail(TT_ERR_ARG, "tt_opt_set_hparams: null handle");
  h->lr = lr;
  h->beta1 = beta1 > 0 ? beta1 : 0.9;
  h->beta2 = beta2 > 0 ? beta2 : 0.999;
  h->eps = eps > 0 ? eps : (h->opt_kind == TT_OPT_ADAGRAD ? 1e-10 : 1e-8);
  return TT_OK;
}

int tt_opt_get_step(tt_engine* h, int64_t* step) {
  if (!h || !step) return fail(TT_ERR_ARG, "tt_opt_get_step: null argument");
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  long long v = 0;
  CU(cudaMemcpy(&v, h->d_step, sizeof(v), cudaMemcpyDeviceToHost));
  *step = v;
  return TT_OK;
}

int tt_forward(tt_engine* h, const int64_t* d_idx, int64_t B, float* d_out, void* stream) {
  if (!h) return fail(TT_ERR_ARG, "tt_forward: null handle");
  if (B < 0 || B > INT_MAX / 2) return fail(TT_ERR_ARG, "tt_forward: batch size out of range");
  if (B > 0 && (!d_idx || !d_out)) return fail(TT_ERR_ARG, "tt_forward: null device buffer");
  CU(cudaSetDevice(h->device));
  if (B == 0) { h->plan_valid = false; return TT_OK; }  // empty batch -> 0 x N
  return do_forward(h, d_idx, B, d_out, (cudaStream_t)stream, true);
}

int tt_backward(tt_engine* h, const int64_t* d_idx, int64_t B, const float* d_up, void* stream) {
  if (!h) return fail(TT_ERR_ARG, "tt_backward: null handle");
  CU(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (B < 0 || B > INT_MAX / 2) return fail(TT_ERR_ARG, "backward_lookup: upstream rows != index count");
  if (B > 0 && !d_up) return fail(TT_ERR_ARG, "backward_lookup: null upstream buffer");
  if (d_idx == nullptr) {
    if (!h->plan_valid || h->plan_version != h->cores_version || B != h->B)
      return fail(TT_ERR_STATE, "tt_backward: no matching forward plan (run tt_forward on this batch first)");
  } else {
    if (B == 0) {
      CU(cudaMemsetAsync(h->grads, 0, sizeof(float) * (size_t)(h->dc.nparams + h->ntc), s));
      h->batch_count = 0;
      return TT_OK;
    }
    int rc = do_forward(h, d_idx, B, nullptr, s, false);
    if (rc) return rc;
  }
  return do_backward(h, d_up, s);
}

static int step_impl(tt_engine* h, cudaStream_t s, bool global_reject);

int tt_step(tt_engine* h, void* stream) {
  if (!h) return fail(TT_ERR_ARG, "tt_step: null handle");
  CU(cudaSetDevice(h->device));
  return step_impl(h, (cudaStream_t)stream, false);
}

// the update kernels; global_reject: the non-finite check's verdict is
// min-reduced over the communicator before any core changes, so every rank
// applies or rejects the step together (owner sharding: a rank's gradient
// covers its own G_F slices only)
static int step_impl(tt_engine* h, cudaStream_t s, bool global_reject) {
  const DevCfg& c = h->dc;
  Phase ph(h, 4, s);
  LAUNCH(k_reset_status, 1, 1, 0, s, h->st, 2);
  bool vec4 = true;
  for (int k = 0; k < c.d; ++k) vec4 = vec4 && c.core_off[k] % 4 == 0 && c.slice[k] % 4 == 0;
  const int64_t work = vec4 ? c.nparams / 4 : c.nparams;
  LAUNCH(k_check_finite, grid_for(work), 256, 0, s, c, h->grads, vec4 ? 1 : 0, h->st);
  if (global_reject && h->comm) {
    const ncclResult_t r = nccl().AllReduce(&h->st->bad_core, &h->st->bad_core, 1, ncclInt32, ncclMin, h->comm, s);
    if (r != ncclSuccess) return fail(TT_ERR_CUDA, std::string("ncclAllReduce: ") + nccl().GetErrorString(r));
  }
  const float lr = (float)h->lr, b1 = (float)h->beta1, b2 = (float)h->beta2, ep = (float)h->eps;
  if (h->opt_kind == TT_OPT_SGD)
    LAUNCH(k_update<0>, grid_for(work), 256, 0, s, c, h->params, h->grads, h->s1, h->s2, vec4 ? 1 : 0, lr, b1, b2,
           ep, h->d_step, h->st);
  else if (h->opt_kind == TT_OPT_ADAM)
    LAUNCH(k_update<1>, grid_for(work), 256, 0, s, c, h->params, h->grads, h->s1, h->s2, vec4 ? 1 : 0, lr, b1, b2,
           ep, h->d_step, h->st);
  else
    LAUNCH(k_update<2>, grid_for(work), 256, 0, s, c, h->params, h->grads, h->s1, h->s2, vec4 ? 1 : 0, lr, b1, b2,
           ep, h->d_step, h->st);
  LAUNCH(k_commit_step, 1, 1, 0, s, h->d_step, h->st);
  ++h->cores_version;
  CU(cudaGetLastError());
  return TT_OK;
}

int tt_sync(tt_engine* h, void* stream) {
  if (!h) return fail(TT_ERR_ARG, "tt_sync: null handle");
  CU(cudaSetDevice(h->device));
  return read_status(h, (cudaStream_t)stream);
}

int tt_lookup_batch(tt_engine* h, const int64_t* h_idx, int64_t B, float* h_out) {
  if (!h) return fail(TT_ERR_ARG, "lookup_batch: null handle");
  if (B < 0) return fail(TT_ERR_ARG, "lookup_batch: negative batch");
  if (B == 0) return TT_OK;
  if (!h_idx || !h_out) return fail(TT_ERR_ARG, "lookup_batch: null buffer");
  CU(cudaSetDevice(h->device));
  int rc = ensure_stage(h, B);
  if (rc) return rc;
  CU(cudaMemcpyAsync(h->st_idx, h_idx, sizeof(int64_t) * B, cudaMemcpyHostToDevice, h->own));
  rc = tt_forward(h, h->st_idx, B, h->st_out, h->own);
  if (rc) return rc;
  rc = read_status(h, h->own);
  if (rc) return rc;
  CU(cudaMemcpyAsync(h_out, h->st_out, sizeof(float) * B * h->dc.emb_dim, cudaMemcpyDeviceToHost, h->own));
  CU(cudaStreamSynchronize(h->own));
  return TT_OK;
}

int tt_backward_lookup(tt_engine* h, const int64_t* h_idx, int64_t B, const float* h_up) {
  if (!h) return fail(TT_ERR_ARG, "backward_lookup: null handle");
  if (B < 0) return fail(TT_ERR_ARG, "backward_lookup: negative batch");
  CU(cudaSetDevice(h->device));
  if (B == 0) {  // CoreGradients::zeros with batch_count 0 (autodiff.cpp:40-46)
    CU(cudaMemsetAsync(h->grads, 0, sizeof(float) * (size_t)(h->dc.nparams + h->ntc), h->own));
    CU(cudaStreamSynchronize(h->own));
    h->batch_count = 0;
    return TT_OK;
  }
  if (!h_idx || !h_up) return fail(TT_ERR_ARG, "backward_lookup: null buffer");
  int rc = ensure_stage(h, B);
  if (rc) return rc;
  CU(cudaMemcpyAsync(h->st_idx, h_idx, sizeof(int64_t) * B, cudaMemcpyHostToDevice, h->own));
  CU(cudaMemcpyAsync(h->st_up, h_up, sizeof(float) * B * h->dc.emb_dim, cudaMemcpyHostToDevice, h->own));
  rc = tt_backward(h, h->st_idx, B, h->st_up, h->own);
  if (rc) return rc;
  rc = read_status(h, h->own);
  if (rc == TT_ERR_INDEX) g_err = "backward_lookup" + g_err.substr(g_err.find(':'));
  return rc;
}

int tt_apply_update(tt_engine* h) {
  if (!h) return fail(TT_ERR_ARG, "apply_update: null handle");
  int rc = tt_step(h, h->own);
  if (rc) return rc;
  return read_status(h, h->own);
}

int tt_train_step_host(tt_engine* h, const int64_t* h_idx, int64_t B, const float* h_up, float* h_out) {
  if (!h) return fail(TT_ERR_ARG, "tt_train_step_host: null handle");
  if (B <= 0 || !h_idx || !h_up) return fail(TT_ERR_ARG, "tt_train_step_host: empty batch or null buffer");
  CU(cudaSetDevice(h->device));
  int rc = ensure_stage(h, B);
  if (rc) return rc;
  if (!h->s_h2d) {
    CU(cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&h->ev_up, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_fwd, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
  }
  cudaStream_t s = h->own;
  const size_t rows = sizeof(float) * (size_t)B * (size_t)h->dc.emb_dim;
  // the compute stream's previous work (and any earlier reader of st_up /
  // st_out) is ordered before this step's copies
  // the indices go first: host-to-device copies share a copy engine, and the
  // plan + forward must not queue behind the 128 MB upstream upload
  CU(cudaMemcpyAsync(h->st_idx, h_idx, sizeof(int64_t) * B, cudaMemcpyHostToDevice, s));
  CU(cudaEventRecord(h->ev_in, s));
  CU(cudaStreamWaitEvent(h->s_h2d, h->ev_in, 0));
  CU(cudaMemcpyAsync(h->st_up, h_up, rows, cudaMemcpyHostToDevice, h->s_h2d));  // under plan + forward
  CU(cudaEventRecord(h->ev_up, h->s_h2d));
  // on any error below, the copies already queued (the upstream upload, the
  // row download) may still be reading / writing the caller's host buffers:
  // drain all three streams before returning
  auto drained = [&](int code) {
    cudaStreamSynchronize(h->s_h2d);
    cudaStreamSynchronize(h->s_d2h);
    cudaStreamSynchronize(s);
    return code;
  };
#define CU_D(call)                                                                        \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) return drained(fail(TT_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_))); \
  } while (0)
  rc = tt_forward(h, h->st_idx, B, h->st_out, s);
  if (rc) return drained(rc);
  if (h_out) {  // rows go back under the backward + update
    CU_D(cudaEventRecord(h->ev_fwd, s));
    CU_D(cudaStreamWaitEvent(h->s_d2h, h->ev_fwd, 0));
    CU_D(cudaMemcpyAsync(h_out, h->st_out, rows, cudaMemcpyDeviceToHost, h->s_d2h));
  }
  CU_D(cudaStreamWaitEvent(s, h->ev_up, 0));
  rc = tt_backward(h, nullptr, B, h->st_up, s);
  if (rc) return drained(rc);
  rc = tt_step(h, s);
  if (rc) return drained(rc);
#undef CU_D
  CU(cudaStreamSynchronize(h->s_d2h));
  CU(cudaStreamSynchronize(h->s_h2d));
  return read_status(h, s);
}

// ---- data parallelism over NCCL ---------------------------
namespace {
int nccl_fail(const char* what, ncclResult_t r) {
  return fail(TT_ERR_CUDA, std::string(what) + ": " + (nccl().ok ? nccl().GetErrorString(r) : nccl().why));
}

int comm_attach(tt_engine* h, ncclComm_t comm, bool own, int rank, int nranks) {
  CU(cudaSetDevice(h->device));
  if (!h->s_comm) {
    CU(cudaStreamCreateWithFlags(&h->s_comm, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&h->ev_gF, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_bwd, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_comm, cudaEventDisableTiming));
  }
  if (h->comm && h->own_comm) nccl().CommDestroy(h->comm);
  h->comm = comm;
  h->own_comm = own;
  h->rank = rank;
  h->nranks = nranks;
  h->dense = true;  // every rank's buffer holds its full local gradient: the sum is the global one
  h->gF_ready = false;
  return TT_OK;
}
}  // namespace

int tt_nccl_unique_id(void* out, int64_t nbytes) {
  if (!out || nbytes < (int64_t)sizeof(ncclUniqueId)) return fail(TT_ERR_ARG, "tt_nccl_unique_id: need 128 bytes");
  if (!nccl().ok) return fail(TT_ERR_CUDA, nccl().why);
  ncclUniqueId id;
  const ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
  memcpy(out, &id, sizeof(id));
  return TT_OK;
}

int tt_comm_init_rank(tt_engine* h, const void* unique_id, int rank, int nranks) {
  if (!h || !unique_id) return fail(TT_ERR_ARG, "tt_comm_init_rank: null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(TT_ERR_ARG, "tt_comm_init_rank: bad rank / nranks");
  if (!nccl().ok) return fail(TT_ERR_CUDA, nccl().why);
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  const ncclResult_t r = nccl().CommInitRank(&comm, nranks, id, rank);
  if (r != ncclSuccess) return nccl_fail("ncclCommInitRank", r);
  return comm_attach(h, comm, true, rank, nranks);
}

int tt_comm_init(tt_engine* h, void* nccl_comm, int rank, int nranks) {
  if (!h) return fail(TT_ERR_ARG, "tt_comm_init: null handle");
  if (!nccl_comm) {  // detach
    CU(cudaSetDevice(h->device));
    CU(cudaDeviceSynchronize());
    if (h->comm && h->own_comm && nccl().ok) nccl().CommDestroy(h->comm);
    h->comm = nullptr;
    h->own_comm = false;
    h->rank = 0;
    h->nranks = 1;
    h->dense = false;
    return TT_OK;
  }
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(TT_ERR_ARG, "tt_comm_init: bad rank / nranks");
  if (!nccl().ok) return fail(TT_ERR_CUDA, nccl().why);
  return comm_attach(h, (ncclComm_t)nccl_comm, false, rank, nranks);
}

int tt_allreduce_grads(tt_engine* h, void* stream) {
  if (!h) return fail(TT_ERR_ARG, "tt_allreduce_grads: null handle");
  if (!h->comm) return fail(TT_ERR_STATE, "tt_allreduce_grads: no communicator (tt_comm_init first)");
  CU(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  const DevCfg& c = h->dc;
  const size_t total = (size_t)(c.nparams + h->ntc);
  const auto& api = nccl();
  ncclResult_t r;
  CU(cudaEventRecord(h->ev_bwd, s));
  if (h->gF_ready && h->last_path >= 1) {
    // dG_F (the fused level, written only by the GEMM kernel) was final at
    // ev_gF: its all-reduce overlaps the backward's auxiliary kernels; the
    // rest of the buffer (the other cores and the touch counters) follows
    // the whole backward
    const int F = h->fs.F;
    const size_t o0 = (size_t)c.core_off[F], o1 = (size_t)(c.core_off[F] + c.m[F] * c.slice[F]);
    CU(cudaStreamWaitEvent(h->s_comm, h->ev_gF, 0));
    r = api.AllReduce(h->grads + o0, h->grads + o0, o1 - o0, ncclFloat32, ncclSum, h->comm, h->s_comm);
    if (r != ncclSuccess) return nccl_fail("ncclAllReduce", r);
    CU(cudaStreamWaitEvent(h->s_comm, h->ev_bwd, 0));
    if (o0 > 0) {
      r = api.AllReduce(h->grads, h->grads, o0, ncclFloat32, ncclSum, h->comm, h->s_comm);
      if (r != ncclSuccess) return nccl_fail("ncclAllReduce", r);
    }
    r = api.AllReduce(h->grads + o1, h->grads + o1, total - o1, ncclFloat32, ncclSum, h->comm, h->s_comm);
    if (r != ncclSuccess) return nccl_fail("ncclAllReduce", r);
  } else {
    CU(cudaStreamWaitEvent(h->s_comm, h->ev_bwd, 0));
    r = api.AllReduce(h->grads, h->grads, total, ncclFloat32, ncclSum, h->comm, h->s_comm);
    if (r != ncclSuccess) return nccl_fail("ncclAllReduce", r);
  }
  h->gF_ready = false;
  CU(cudaEventRecord(h->ev_comm, h->s_comm));
  CU(cudaStreamWaitEvent(s, h->ev_comm, 0));
  return TT_OK;
}

// ---- pipelined host-buffer steps ------------------------------------------
int tt_train_step_wait(tt_engine* h) {
  if (!h) return fail(TT_ERR_ARG, "tt_train_step_wait: null handle");
  if (h->hs_count == 0) return TT_OK;
  CU(cudaSetDevice(h->device));
  auto& sl = h->hs[h->hs_head];
  h->hs_head = (h->hs_head + 1) % TT_HOST_SLOTS;
  --h->hs_count;
  sl.busy = false;
  CU(cudaEventSynchronize(sl.ev_done));
  if (sl.has_out) CU(cudaEventSynchronize(sl.ev_out));  // (ev_done follows the slot's uploads)
  DevStatus st;
  memcpy(&st, (const void*)sl.h_st, sizeof(st));
  if (st.bad_pos != TT_NO_POS) {
    const int64_t val = sl.h_idx ? sl.h_idx[st.bad_pos] : 0;
    h->plan_valid = false;
    return fail(TT_ERR_INDEX,
                "lookup_batch: index " + std::to_string(val) + " at batch position " +
                    std::to_string((long long)st.bad_pos) + " out of [0, " + std::to_string(h->dc.num_nodes) + ")",
                (int64_t)st.bad_pos, val);
  }
  if (st.bad_core != INT_MAX)
    return fail(TT_ERR_NONFINITE,
                "apply_update: non-finite gradient in core " + std::to_string(st.bad_core) + "; update rejected",
                st.bad_core);
  return TT_OK;
}

int tt_train_step_submit(tt_engine* h, const int64_t* h_idx, int64_t B, const float* h_up, float* h_out) {
  if (!h) return fail(TT_ERR_ARG, "tt_train_step_submit: null handle");
  if (B <= 0 || !h_idx || !h_up) return fail(TT_ERR_ARG, "tt_train_step_submit: empty batch or null buffer");
  CU(cudaSetDevice(h->device));
  if (h->hs_count == TT_HOST_SLOTS) {  // every slot in flight: retire the oldest first
    int rc = tt_train_step_wait(h);
    if (rc) return rc;
  }
  if (!h->s_h2d) {
    CU(cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&h->ev_up, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_fwd, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
  }
  auto& sl = h->hs[h->hs_next];
  const int64_t N = h->dc.emb_dim;
  if (sl.cap < B) {
    cudaFree(sl.idx); cudaFree(sl.up); cudaFree(sl.out);
    sl.idx = nullptr; sl.up = nullptr; sl.out = nullptr; sl.cap = 0;
    CU(dalloc(&sl.idx, B));
    CU(dalloc(&sl.up, B * N));
    CU(dalloc(&sl.out, B * N));
    sl.cap = B;
  }
  if (!sl.ev_idx) {
    for (cudaEvent_t* e : {&sl.ev_idx, &sl.ev_up, &sl.ev_fwd, &sl.ev_done, &sl.ev_out})
      CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    CU(cudaHostAlloc(&sl.h_st, sizeof(DevStatus), cudaHostAllocMapped));
  }
  cudaStream_t s = h->own;
  const size_t rows = sizeof(float) * (size_t)B * (size_t)N;
  // uploads on the copy stream: the indices first (the plan needs them), the
  // upstream behind them -- both may run under the previous step's compute
  CU(cudaMemcpyAsync(sl.idx, h_idx, sizeof(int64_t) * B, cudaMemcpyHostToDevice, h->s_h2d));
  CU(cudaEventRecord(sl.ev_idx, h->s_h2d));
  CU(cudaMemcpyAsync(sl.up, h_up, rows, cudaMemcpyHostToDevice, h->s_h2d));
  CU(cudaEventRecord(sl.ev_up, h->s_h2d));
  CU(cudaStreamWaitEvent(s, sl.ev_idx, 0));
  int rc = tt_forward(h, sl.idx, B, sl.out, s);
  if (rc) { cudaStreamSynchronize(h->s_h2d); cudaStreamSynchronize(s); return rc; }
  sl.has_out = h_out != nullptr;
  if (h_out) {  // rows go back under the backward + update (and the next step's upload)
    CU(cudaEventRecord(sl.ev_fwd, s));
    CU(cudaStreamWaitEvent(h->s_d2h, sl.ev_fwd, 0));
    CU(cudaMemcpyAsync(h_out, sl.out, rows, cudaMemcpyDeviceToHost, h->s_d2h));
    CU(cudaEventRecord(sl.ev_out, h->s_d2h));
  }
  CU(cudaStreamWaitEvent(s, sl.ev_up, 0));
  rc = tt_backward(h, nullptr, B, sl.up, s);
  if (!rc) rc = tt_step(h, s);
  if (rc) { cudaStreamSynchronize(h->s_h2d); cudaStreamSynchronize(h->s_d2h); cudaStreamSynchronize(s); return rc; }
  // the step's status goes to host memory by a one-thread kernel writing
  // mapped (zero-copy) pinned memory: a 16-byte cudaMemcpy here would queue on
  // the device-to-host copy engine behind the 134 MB row download and hold the
  // compute stream (the next step's forward) until it finished -- measured
  // 3.67 -> 2.8 ms per pipelined step at papers
  LAUNCH(k_status_to_host, 1, 1, 0, s, (const DevStatus*)h->st, sl.h_st);
  CU(cudaEventRecord(sl.ev_done, s));
  sl.B = B;
  sl.h_idx = h_idx;
  sl.busy = true;
  h->hs_next = (h->hs_next + 1) % TT_HOST_SLOTS;
  ++h->hs_count;
  return TT_OK;
}

void* tt_engine_stream(tt_engine* h) { return h ? (void*)h->own : nullptr; }

const char* tt_main_kernel(tt_engine* h, int backward) {
  if (!h) return "";
  return backward ? h->bwd_kernel : h->fwd_kernel;
}

// ---- ID-owner sharding over the handle's NCCL communicator ------------------
namespace {
int owner_alloc(tt_engine* h, int64_t B) {
  auto& o = h->ow;
  const int P = h->nranks;
  const int64_t N = h->dc.emb_dim;
  if (!o.d_counts) {
    CU(dalloc(&o.d_counts, P));
    CU(dalloc(&o.d_all, (int64_t)P * P));
    CU(dalloc(&o.d_gbad, 1));
    CU(cudaMallocHost(&o.h_all, sizeof(int) * ((size_t)P * P + 2)));
  }
  if (o.cap < B) {
    void* ptrs[] = {o.ka, o.kb, o.va, o.vb, o.sid, o.back, o.sup};
    for (void* p : ptrs) cudaFree(p);
    o.ka = o.kb = nullptr; o.va = o.vb = nullptr; o.sid = nullptr; o.back = o.sup = nullptr; o.cap = 0;
    CU(dalloc(&o.ka, B)); CU(dalloc(&o.kb, B)); CU(dalloc(&o.va, B)); CU(dalloc(&o.vb, B));
    CU(dalloc(&o.sid, B)); CU(dalloc(&o.back, B * N)); CU(dalloc(&o.sup, B * N));
    o.cap = B;
  }
  return TT_OK;
}

int owner_recv_alloc(tt_engine* h, int64_t R) {
  auto& o = h->ow;
  if (o.cap_r >= R) return TT_OK;
  const int64_t N = h->dc.emb_dim;
  cudaFree(o.rid); cudaFree(o.rout); cudaFree(o.rup);
  o.rid = nullptr; o.rout = o.rup = nullptr; o.cap_r = 0;
  CU(dalloc(&o.rid, R)); CU(dalloc(&o.rout, R * N)); CU(dalloc(&o.rup, R * N));
  o.cap_r = R;
  return TT_OK;
}

// grouped point-to-point exchange: send counts[p] elements at offsets soff to
// every p, receive rcounts[p] at roff (elem = `width` values of `type`)
int owner_exchange(tt_engine* h, const void* sbuf, const std::vector<int64_t>& soff, const std::vector<int64_t>& scnt,
                   void* rbuf, const std::vector<int64_t>& roff, const std::vector<int64_t>& rcnt, size_t esize,
                   int64_t width, ncclDataType_t type, cudaStream_t s) {
  const auto& api = nccl();
  ncclResult_t r = api.GroupStart();
  for (int p = 0; p < h->nranks && r == ncclSuccess; ++p) {
    if (scnt[p]) r = api.Send((const char*)sbuf + soff[p] * width * esize, (size_t)(scnt[p] * width), type, p, h->comm, s);
    if (r == ncclSuccess && rcnt[p])
      r = api.Recv((char*)rbuf + roff[p] * width * esize, (size_t)(rcnt[p] * width), type, p, h->comm, s);
  }
  const ncclResult_t e = api.GroupEnd();
  if (r != ncclSuccess || e != ncclSuccess)
    return fail(TT_ERR_CUDA, std::string("owner exchange: ") + api.GetErrorString(r != ncclSuccess ? r : e));
  return TT_OK;
}
}  // namespace

int tt_owner_forward(tt_engine* h, const int64_t* d_idx, int64_t B, float* d_out, void* stream) {
  if (!h) return fail(TT_ERR_ARG, "tt_owner_forward: null handle");
  if (!h->comm) return fail(TT_ERR_STATE, "tt_owner_forward: no communicator (tt_comm_init first)");
  if (B < 0 || B > INT_MAX / 2) return fail(TT_ERR_ARG, "tt_owner_forward: batch size out of range");
  if (B > 0 && (!d_idx || !d_out)) return fail(TT_ERR_ARG, "tt_owner_forward: null device buffer");
  if (h->dc.emb_dim % 4) return fail(TT_ERR_ARG, "tt_owner_forward: emb_dim must be a multiple of 4");
  CU(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  auto& o = h->ow;
  o.valid = false;
  const int P = h->nranks, F = std::max(h->dc.d - 2, 0);
  int rc = ensure_plan(h, std::max<int64_t>(B, 1));  // (the radix sort's histogram slots)
  if (rc) return rc;
  rc = owner_alloc(h, std::max<int64_t>(B, 1));
  if (rc) return rc;
  const int64_t N = h->dc.emb_dim;
  LAUNCH(k_reset_status, 1, 1, 0, s, h->st, 1);
  if (B > 0) {
    LAUNCH(k_owner_of, grid_for(B, 256, INT_MAX), 256, 0, s, d_idx, B, h->dc, F, P, h->rank, o.ka, o.va, h->st);
    const int nbits = std::max<int>(1, (int)bitlen((uint64_t)(P - 1)));
    unsigned* sk = radix_sort<unsigned>(h, s, o.ka, o.va, o.kb, o.vb, nullptr, (int)B, B, nbits, &o.perm);
    LAUNCH(k_owner_counts, 1, 32 * ((P + 31) / 32), 0, s, (const unsigned*)sk, (int)B, P, o.d_counts);
  } else {
    CU(cudaMemsetAsync(o.d_counts, 0, sizeof(int) * P, s));
  }
  const auto& api = nccl();
  ncclResult_t r = api.AllGather(o.d_counts, o.d_all, (size_t)P, ncclInt32, h->comm, s);
  if (r == ncclSuccess) r = api.AllReduce(&h->st->bad_pos, o.d_gbad, 1, ncclUint64, ncclMin, h->comm, s);
  if (r != ncclSuccess) return fail(TT_ERR_CUDA, std::string("owner counts: ") + api.GetErrorString(r));
  // the one host round trip of a routed step: NCCL's point-to-point calls take
  // host-side counts (the P x P matrix, 4 P^2 bytes)
  CU(cudaMemcpyAsync(o.h_all, o.d_all, sizeof(int) * P * P, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(o.h_all + P * P, o.d_gbad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  unsigned long long gbad;
  memcpy(&gbad, o.h_all + P * P, sizeof(gbad));
  if (gbad != TT_NO_POS) {
    DevStatus st;
    CU(cudaMemcpy(&st, h->st, sizeof(st), cudaMemcpyDeviceToHost));
    LAUNCH(k_reset_status, 1, 1, 0, s, h->st, 1);
    CU(cudaStreamSynchronize(s));
    if (st.bad_pos != TT_NO_POS) {
      int64_t val = 0;
      cudaMemcpy(&val, d_idx + st.bad_pos, sizeof(val), cudaMemcpyDeviceToHost);
      return fail(TT_ERR_INDEX,
                  "lookup_batch: index " + std::to_string(val) + " at batch position " +
                      std::to_string((long long)st.bad_pos) + " out of [0, " + std::to_string(h->dc.num_nodes) + ")",
                  (int64_t)st.bad_pos, val);
    }
    return fail(TT_ERR_INDEX, "lookup_batch: an index out of range on another rank; batch rejected", -1, 0);
  }
  o.send.assign(P, 0); o.recv.assign(P, 0); o.soff.assign(P + 1, 0); o.roff.assign(P + 1, 0);
  for (int p = 0; p < P; ++p) {
    o.send[p] = o.h_all[h->rank * P + p];
    o.recv[p] = o.h_all[p * P + h->rank];
    o.soff[p + 1] = o.soff[p] + o.send[p];
    o.roff[p + 1] = o.roff[p] + o.recv[p];
  }
  o.B = B;
  o.Bown = o.roff[P];
  rc = owner_recv_alloc(h, std::max<int64_t>(o.Bown, 1));
  if (rc) return rc;
  if (B > 0) LAUNCH(k_gather_ids, grid_for(B, 256, INT_MAX), 256, 0, s, d_idx, (const int*)o.perm, (int)B, o.sid);
  rc = owner_exchange(h, o.sid, o.soff, o.send, o.rid, o.roff, o.recv, sizeof(int64_t), 1, ncclInt64, s);
  if (rc) return rc;
  if (o.Bown > 0) {
    rc = do_forward(h, o.rid, o.Bown, o.rout, s, true);
    if (rc) return rc;
  } else {
    h->plan_valid = false;
  }
  // rows back to the ranks that asked, then to their batch positions
  rc = owner_exchange(h, o.rout, o.roff, o.recv, o.back, o.soff, o.send, sizeof(float), N, ncclFloat32, s);
  if (rc) return rc;
  if (B > 0)
    LAUNCH(k_permute_rows<true>, grid_for(B * 32, 256, 148 * 8), 256, 0, s, (const float*)o.back, (const int*)o.perm,
           (int)B, N, d_out);
  o.valid = true;
  CU(cudaGetLastError());
  return TT_OK;
}

int tt_owner_backward(tt_engine* h, const float* d_up, void* stream) {
  if (!h) return fail(TT_ERR_ARG, "tt_owner_backward: null handle");
  auto& o = h->ow;
  if (!h->comm || !o.valid) return fail(TT_ERR_STATE, "tt_owner_backward: no matching tt_owner_forward");
  if (o.B > 0 && !d_up) return fail(TT_ERR_ARG, "tt_owner_backward: null upstream buffer");
  CU(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t N = h->dc.emb_dim;
  const DevCfg& c = h->dc;
  if (o.B > 0)
    LAUNCH(k_permute_rows<false>, grid_for(o.B * 32, 256, 148 * 8), 256, 0, s, d_up, (const int*)o.perm, (int)o.B, N,
           o.sup);
  int rc = owner_exchange(h, o.sup, o.soff, o.send, o.rup, o.roff, o.recv, sizeof(float), N, ncclFloat32, s);
  if (rc) return rc;
  if (o.Bown > 0) {
    if (!h->plan_valid || h->plan_version != h->cores_version)
      return fail(TT_ERR_STATE, "tt_owner_backward: the cores changed since tt_owner_forward");
    rc = do_backward(h, o.rup, s);
    if (rc) return rc;
  } else {  // nothing owned this step: CoreGradients::zeros (autodiff.cpp:40-46)
    CU(cudaMemsetAsync(h->grads, 0, sizeof(float) * (size_t)(c.nparams + h->ntc), s));
    h->batch_count = 0;
  }
  // the replicated cores' gradients (every core but F, and their touch
  // counters) are summed over the ranks; the owned G_F slices never move
  const int F = std::max(c.d - 2, 0);
  const int64_t g0 = c.core_off[F], g1 = c.core_off[F] + c.m[F] * c.slice[F];
  const int64_t t0 = c.tc_off[F], t1 = c.tc_off[F] + c.m[F], tend = c.nparams + h->ntc;
  const int64_t spans[3][2] = {{0, g0}, {g1, t0}, {t1, tend}};
  for (auto& sp : spans) {
    if (sp[1] <= sp[0]) continue;
    const ncclResult_t r =
        nccl().AllReduce(h->grads + sp[0], h->grads + sp[0], (size_t)(sp[1] - sp[0]), ncclFloat32, ncclSum, h->comm, s);
    if (r != ncclSuccess) return fail(TT_ERR_CUDA, std::string("ncclAllReduce: ") + nccl().GetErrorString(r));
  }
  CU(cudaGetLastError());
  return TT_OK;
}

int tt_owner_step(tt_engine* h, void* stream) {
  if (!h) return fail(TT_ERR_ARG, "tt_owner_step: null handle");
  if (!h->comm) return fail(TT_ERR_STATE, "tt_owner_step: no communicator");
  CU(cudaSetDevice(h->device));
  return step_impl(h, (cudaStream_t)stream, true);
}

int64_t tt_owner_rows(tt_engine* h) { return h ? h->ow.Bown : -1; }

int tt_grad_buffer(tt_engine* h, float** d_ptr, int64_t* count) {
  if (!h || !d_ptr || !count) return fail(TT_ERR_ARG, "tt_grad_buffer: null argument");
  *d_ptr = h->grads;
  *count = h->dc.nparams + h->ntc;
  return TT_OK;
}

int tt_bind_grad_buffer(tt_engine* h, float* d_ptr, int64_t count) {
  if (!h) return fail(TT_ERR_ARG, "tt_bind_grad_buffer: null handle");
  const int64_t need = h->dc.nparams + h->ntc;
  if (d_ptr && count < need) return fail(TT_ERR_ARG, "tt_bind_grad_buffer: buffer too small");
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  float* target = d_ptr ? d_ptr : h->own_grads;
  if (target != h->grads) {
    CU(cudaMemcpy(target, h->grads, sizeof(float) * (size_t)need, cudaMemcpyDeviceToDevice));
    h->grads = target;
  }
  return TT_OK;
}

int tt_set_dense_grads(tt_engine* h, int on) {
  if (!h) return fail(TT_ERR_ARG, "tt_set_dense_grads: null handle");
  h->dense = on != 0;
  return TT_OK;
}

int tt_plan_stats(tt_engine* h, int64_t* out) {
  if (!h || !out) return fail(TT_ERR_ARG, "tt_plan_stats: null argument");
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  int c[TT_MAXD];
  CU(cudaMemcpy(c, h->counts, sizeof(int) * h->dc.d, cudaMemcpyDeviceToHost));
  for (int k = 0; k < h->dc.d; ++k) out[k] = c[k];
  return TT_OK;
}

int64_t tt_plan_digits(tt_engine* h, int64_t* ids, int32_t* digits, int64_t capn) {
  if (!h || !h->cap) return -1;
  if (cudaSetDevice(h->device) || cudaDeviceSynchronize()) return -1;
  const int d = h->dc.d;
  int c[TT_MAXD];
  cudaMemcpy(c, h->counts, sizeof(int) * d, cudaMemcpyDeviceToHost);
  const int64_t U = c[d - 1];
  if (U > capn) return U;
  std::vector<unsigned long long> uq(U);
  std::vector<int> dig((size_t)d * h->cap), par((size_t)d * h->cap);
  cudaMemcpy(uq.data(), h->uniq, sizeof(unsigned long long) * U, cudaMemcpyDeviceToHost);
  cudaMemcpy(dig.data(), h->digit, sizeof(int) * dig.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(par.data(), h->parent, sizeof(int) * par.size(), cudaMemcpyDeviceToHost);
  for (int64_t u = 0; u < U; ++u) {
    ids[u] = (int64_t)uq[u];
    int64_t node = u;
    for (int k = d - 1; k >= 0; --k) {
      digits[u * d + k] = dig[(size_t)k * h->cap + node];
      node = par[(size_t)k * h->cap + node];
    }
  }
  return U;
}

int64_t tt_plan_sorted(tt_engine* h, int64_t* keys, int32_t* pos, int64_t capn) {
  if (!h || !h->cap) return -1;
  if (cudaSetDevice(h->device) || cudaDeviceSynchronize()) return -1;
  if (h->B > capn) return h->B;
  std::vector<unsigned long long> k((size_t)h->B);
  cudaMemcpy(k.data(), h->skeys, sizeof(unsigned long long) * h->B, cudaMemcpyDeviceToHost);
  cudaMemcpy(pos, h->spos, sizeof(int) * h->B, cudaMemcpyDeviceToHost);
  for (int64_t i = 0; i < h->B; ++i) keys[i] = (int64_t)k[i];
  return h->B;
}

int64_t tt_launch_count(tt_engine* h) { return h ? h->launches : -1; }

// debug: copy the tcgen05 backward's per-CTA phase timestamps (TT_TC_TRACE)
int64_t tt_debug_trace(long long* out, int64_t n) {
  if (!g_trace_buf) return 0;
  cudaDeviceSynchronize();
  n = std::min<int64_t>(n, 4096 * 64);
  cudaMemcpy(out, g_trace_buf, sizeof(long long) * n, cudaMemcpyDeviceToHost);
  return n;
}

int tt_set_profiling(tt_engine* h, int on) {
  if (!h) return fail(TT_ERR_ARG, "tt_set_profiling: null handle");
  h->profiling = on != 0;
  return TT_OK;
}

int tt_profile_read(tt_engine* h, double* ms, int64_t* counts, int nslots) {
  if (!h || !ms || !counts) return fail(TT_ERR_ARG, "tt_profile_read: null argument");
  CU(cudaSetDevice(h->device));
  CU(cudaDeviceSynchronize());
  for (int k = 0; k < nslots && k < 8; ++k) {
    double t = 0;
    for (auto& pr : h->prof_ev[k]) {
      float x = 0;
      cudaEventElapsedTime(&x, pr.first, pr.second);
      t += x;
      h->ev_pool.push_back(pr.first);
      h->ev_pool.push_back(pr.second);
    }
    ms[k] = t;
    counts[k] = (int64_t)h->prof_ev[k].size();
    h->prof_ev[k].clear();
  }
  return TT_OK;
}

int tt_set_path(tt_engine* h, int path) {
  if (!h || path < 0 || path > 2) return fail(TT_ERR_ARG, "tt_set_path: bad argument");
  h->path_pref = path;
  h->plan_valid = false;
  return TT_OK;
}

int tt_last_path(tt_engine* h) { return h ? h->last_path : -1; }

int64_t tt_last_error_position(void) { return g_err_pos; }
int64_t tt_last_error_value(void) { return g_err_val; }
const char* tt_last_error(void) { return g_err.c_str(); }

double tt_ffma_outer_tflops(int device, int iters) {
  if (cudaSetDevice(device) != cudaSuccess) return -1.0;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  cudaMalloc(&out, sizeof(float) * nsm * 8);
  const int blocks = nsm * 4;
  k_ffma_outer<<<blocks, 256>>>(out, 16, 1.0f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_ffma_outer<<<blocks, 256>>>(out, iters, 1.0f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  const double flops = 2.0 * 64 * (double)iters * 256.0 * blocks;
  return ms > 0 ? flops / (ms * 1e-3) / 1e12 : -1.0;
}

double tt_ffma_peak_tflops(int device, int iters) {
  if (cudaSetDevice(device) != cudaSuccess) return -1.0;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  cudaMalloc(&out, sizeof(float) * nsm * 8);
  const int blocks = nsm * 8;
  k_ffma_peak<<<blocks, 256>>>(out, 16, 1.0001f, 0.5f);  // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_ffma_peak<<<blocks, 256>>>(out, iters, 1.0001f, 0.5f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  const double flops = 2.0 * 8 * 16 * (double)iters * 256.0 * blocks;
  return ms > 0 ? flops / (ms * 1e-3) / 1e12 : -1.0;
}

}  // extern "C"
