/*
 * tt_engine.h -- C-ABI of the B200-native tensor-train embedding engine.
 *
 * This is the drop-in boundary for the reference's lookup/training hot path
 * (namespace ttgnn, /root/reference/proj/core).  The reference has no FFI
 * layer; its "operator API" is free functions over value types.  Each entry
 * point below names the reference interface it replaces.  Plain pointers and
 * sizes only; no torch or CUDA types appear in the signatures (streams are
 * passed as `void*` holding a cudaStream_t, NULL = legacy default stream).
 *
 * Errors: every call returns a tt_status.  The reference throws
 * std::invalid_argument (TT_ERR_ARG) and std::out_of_range (TT_ERR_INDEX) and
 * rejects non-finite gradients before mutating anything (TT_ERR_NONFINITE).
 * Device-side errors of the asynchronous calls are deferred: the batch is
 * failed as a whole (no output row and no gradient is written) and the error
 * is returned by tt_sync() / the next synchronous call.  tt_last_error()
 * returns a thread-local message in the reference's wording.
 *
 * Threading: one handle per GPU; calls on a handle are serialised by the
 * caller (SPEC.md:100,222 -- readers concurrent, updates exclusive).
 */
#ifndef TT_ENGINE_H
#define TT_ENGINE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TT_MAX_CORES 8

typedef enum {
  TT_OK = 0,
  TT_ERR_ARG = 1,       /* std::invalid_argument: config / shape / misuse     */
  TT_ERR_INDEX = 2,     /* std::out_of_range: index outside [0, num_nodes)     */
  TT_ERR_NONFINITE = 3, /* apply_update: non-finite gradient, update rejected  */
  TT_ERR_CUDA = 4,      /* CUDA runtime failure                                */
  TT_ERR_STATE = 5,     /* saved-plan backward without a matching forward      */
  TT_ERR_NOMEM = 6
} tt_status;

typedef enum { TT_OPT_SGD = 0, TT_OPT_ADAM = 1, TT_OPT_ADAGRAD = 2 } tt_opt_kind;

/* TTConfig (tt_config.hpp:33-52): d cores, core k of shape
 * (ranks[k], row_factors[k], col_factors[k], ranks[k+1]). */
typedef struct {
  int64_t num_nodes;
  int64_t emb_dim;
  int32_t d;
  int32_t reserved_;
  int64_t row_factors[TT_MAX_CORES];
  int64_t col_factors[TT_MAX_CORES];
  int64_t ranks[TT_MAX_CORES + 1];
} tt_config_c;

typedef struct tt_engine tt_engine;

/* ---- configuration (tt_config.cpp) --------------------------------------- */
/* TTConfig::validate (tt_config.cpp:92-113). */
int tt_config_validate(const tt_config_c* cfg);
/* count_params (tt_config.cpp:204-208); -1 on an invalid config. */
int64_t tt_count_params(const tt_config_c* cfg);

/* ---- lifetime ------------------------------------------------------------- */
/* TTEmbedding::zeros (tt_embedding.cpp:73-81): cores live on `device`,
 * zero-filled; optimizer defaults to SGD lr=1e-3 until tt_opt_init. */
int tt_engine_create(const tt_config_c* cfg, int device, tt_engine** out);
void tt_engine_destroy(tt_engine* h);

/* ---- cores: host buffers in the reference layout (R_{k-1}, m_k, n_k, R_k),
 * row-major, one pointer per core (TTEmbedding::cores, tt_embedding.hpp:30-32).
 * The device layout is private. */
int tt_set_cores_f64(tt_engine* h, const double* const* cores);
int tt_set_cores_f32(tt_engine* h, const float* const* cores);
int tt_get_cores_f64(tt_engine* h, double* const* cores);
int tt_get_cores_f32(tt_engine* h, float* const* cores);

/* ---- optimizer: OptimizerState::make (autodiff.cpp:120-133) + Adagrad ------
 * SGD: G -= lr g; Adam: bias-corrected (autodiff.cpp:135-145);
 * Adagrad: h += g^2, G -= lr g / (sqrt(h) + eps), h0 = 0.  Resets state and
 * the step counter.  Non-positive beta/eps arguments select the defaults
 * (0.9, 0.999, 1e-8; Adagrad eps 1e-10). */
int tt_opt_init(tt_engine* h, int kind, double lr, double beta1, double beta2, double eps);
int tt_opt_get_step(tt_engine* h, int64_t* step); /* synchronises */
/* Hyper-parameters only (apply_update reads opt.learning_rate etc. on every
 * call, autodiff.cpp:147-173): moments and step are kept, so a learning-rate
 * schedule does not reset the optimizer.  Takes effect for the next tt_step. */
int tt_opt_set_hparams(tt_engine* h, double lr, double beta1, double beta2, double eps);

/* ---- hot path: device buffers, stream-ordered, asynchronous ---------------
 * tt_forward  ~ lookup_batch (tt_embedding.cpp:110-125): d_out is
 *   batch x emb_dim row-major fp32; row b = embedding of d_indices[b].
 * tt_backward ~ backward_lookup (autodiff.cpp:48-118): gradients (a sum over
 *   rows, no 1/B) stay in the handle.  d_indices == NULL reuses the plan and
 *   saved activations of the last tt_forward (the autograd pattern); the cores
 *   must not have changed since (else TT_ERR_STATE).
 * tt_step     ~ apply_update (autodiff.cpp:147-173): all-or-nothing; a
 *   non-finite gradient leaves cores, optimizer state and step untouched. */
int tt_forward(tt_engine* h, const int64_t* d_indices, int64_t batch, float* d_out, void* stream);
int tt_backward(tt_engine* h, const int64_t* d_indices, int64_t batch, const float* d_grad_out,
                void* stream);
int tt_step(tt_engine* h, void* stream);
/* Waits for `stream`, returns (and clears) the first deferred error. */
int tt_sync(tt_engine* h, void* stream);

/* Device-side checkpoint of the cores: snapshot copies the parameters to a
 * handle-owned buffer, restore copies them back (stream-ordered).  Optimizer
 * state and step are not touched. */
int tt_cores_snapshot(tt_engine* h, void* stream);
int tt_cores_restore(tt_engine* h, void* stream);

/* ---- host-buffer entry points (synchronous; the reference call shapes) ---- */
int tt_lookup_batch(tt_engine* h, const int64_t* h_indices, int64_t batch, float* h_out);
int tt_backward_lookup(tt_engine* h, const int64_t* h_indices, int64_t batch,
                       const float* h_upstream);
int tt_apply_update(tt_engine* h);
/* One training step through host memory: upload indices and upstream,
 * forward (result copied to h_out, may be NULL), backward on the saved plan,
 * update.  The upstream upload runs on its own copy stream under the plan and
 * forward, and the row download under the backward and update (pinned host
 * buffers make both asynchronous).  Returns after the step has completed. */
int tt_train_step_host(tt_engine* h, const int64_t* h_indices, int64_t batch,
                       const float* h_upstream, float* h_out);

/* The same step, pipelined across calls: tt_train_step_submit enqueues one
 * step (uploads on a copy stream, compute on the handle's stream, the row
 * download on a second copy stream) into one of three staging slots and
 * returns at once; tt_train_step_wait retires the oldest submitted step and
 * returns its status (TT_ERR_INDEX / TT_ERR_NONFINITE as tt_sync would).  With
 * steps in flight, step t+1's host-to-device copies run under step t's compute
 * and device-to-host copy (as a data loader feeding a training loop would);
 * steps still run in submission order on the cores.  Host buffers must stay
 * valid until the step is retired; a submit with every slot busy retires the
 * oldest first. */
int tt_train_step_submit(tt_engine* h, const int64_t* h_indices, int64_t batch, const float* h_upstream,
                         float* h_out);
int tt_train_step_wait(tt_engine* h);
/* The handle's own CUDA stream (the host-buffer calls run on it). */
void* tt_engine_stream(tt_engine* h);
/* Name of the level-F GEMM kernel the last forward (backward != 0: backward)
 * launched, e.g. "k_fused_fwd8", "k_fused_bwd_ws", "k_tc_bwd" ("" if none). */
const char* tt_main_kernel(tt_engine* h, int backward);

/* Dense gradients in the reference layout (CoreGradients, autodiff.hpp:29-34);
 * untouched slices read as exactly 0.  batch_count may be NULL. */
int tt_get_core_grads_f64(tt_engine* h, double* const* grads, int64_t* batch_count);

/* Uploads caller-built gradients (reference layout, e.g. a CoreGradients a
 * test constructed); every slice counts as touched by the next update. */
int tt_set_core_grads_f64(tt_engine* h, const double* const* grads, int64_t batch_count);

/* init_ortho_core (initializer.cpp:103-132) computed on `device` in fp64:
 * per core, n_k R_{k-1} orthonormal vectors of length m_k R_k (Gram-Schmidt
 * with one re-orthogonalisation pass), vector (r, j) -> slice G_k(r,:,j,:),
 * all cores scaled by target_scale^(1/2d) when target_scale > 0.  Writes
 * host buffers in the reference layout (set them with tt_set_cores_f64).
 * Infeasible ranks: TT_ERR_ARG and, if `bad` is non-NULL,
 * bad = {core, vectors needed, vector length} (InfeasibleRanksError). */
int tt_ortho_cores_f64(const tt_config_c* cfg, int device, uint64_t seed, double target_scale,
                       double* const* cores, int64_t* bad);

/* Node relabelling (graph.cpp:218-252 apply_permutation after a hierarchical
 * reorder): with a permutation set, ID v is served by row perm[v] in every
 * lookup and backward (mapped on the device; range checks stay on v).  perm
 * is a host array of num_nodes entries, a bijection on [0, num_nodes); NULL
 * clears it.  TT_ERR_ARG on a size mismatch or a non-permutation. */
int tt_set_permutation(tt_engine* h, const int64_t* perm, int64_t n);

/* Optimizer state (checkpoint / resume; absent in the reference).
 * Reference layout per core; s1 = Adagrad accumulator or Adam first moment,
 * s2 = Adam second moment; NULL skips an array.  `step` is the update count. */
int tt_opt_state_get_f64(tt_engine* h, double* const* s1, double* const* s2, int64_t* step);
int tt_opt_state_set_f64(tt_engine* h, const double* const* s1, const double* const* s2, int64_t step);

/* ---- data-parallel plumbing ------------------------------------------------
 * The gradient buffer is one contiguous fp32 array: every core's gradient
 * (device layout) followed by one touch counter per core slice.  With
 * dense mode on, tt_backward zero-fills it first so that a sum all-reduce
 * (NCCL over NVLink, issued by the caller on the same stream) yields the
 * global gradient and the union of touched slices. */
int tt_grad_buffer(tt_engine* h, float** d_ptr, int64_t* count);
int tt_set_dense_grads(tt_engine* h, int on);
/* Makes the engine use caller-owned device memory (>= the count that
 * tt_grad_buffer reports, same device) as its gradient buffer, e.g. a tensor
 * a torch.distributed NCCL all-reduce operates on.  NULL restores the
 * engine's own buffer. */
int tt_bind_grad_buffer(tt_engine* h, float* d_ptr, int64_t count);

/* NCCL data parallelism, position sharding: the batch is
 * sharded by position, cores are replicated, and the one exchange step is a
 * sum all-reduce of the gradient buffer between tt_backward and tt_step.
 *   tt_nccl_unique_id     ncclGetUniqueId into `out` (>= 128 bytes), on one
 *                         rank; the caller ships it to the others;
 *   tt_comm_init_rank     creates the handle's own ncclComm_t (ncclCommInitRank);
 *   tt_comm_init          attaches a caller-owned ncclComm_t (NULL detaches);
 *   tt_allreduce_grads    enqueues the all-reduce on the handle's comm stream,
 *                         ordered after the backward on `stream` and before
 *                         anything later on `stream`.  The level-F core's
 *                         gradient (the fused GEMM's output, 63 of 64 MB at
 *                         papers) is all-reduced as soon as that kernel ends,
 *                         overlapping the backward's remaining kernels; the
 *                         other cores and the touch counters follow.
 * Attaching a communicator turns dense gradients on.  NCCL is resolved at run
 * time (dlopen of libnccl.so.2, reusing a copy the process already loaded);
 * without it these return TT_ERR_CUDA. */
int tt_nccl_unique_id(void* out, int64_t nbytes);
int tt_comm_init_rank(tt_engine* h, const void* unique_id, int rank, int nranks);
int tt_comm_init(tt_engine* h, void* nccl_comm, int rank, int nranks);
int tt_allreduce_grads(tt_engine* h, void* stream);

/* NCCL data parallelism, ID-owner sharding (keeps the dedupe that
 * position sharding loses across ranks): rank r owns the level-F digits
 * [floor(m_F r / P), floor(m_F (r+1) / P)) of core F = d-2 -- every ID,
 * level-F prefix and G_F slice with such a digit.
 *   tt_owner_forward   buckets this rank's batch by owner (stable radix
 *                      sort), exchanges the IDs (ncclSend/Recv groups), runs
 *                      the owner's forward on what it received (every prefix
 *                      once in the job) and sends the rows back to their
 *                      batch positions.  One host round trip per call: the
 *                      P x P count matrix the point-to-point calls size from.
 *                      An out-of-range index on any rank fails the batch on
 *                      every rank (TT_ERR_INDEX).
 *   tt_owner_backward  routes the upstream rows to the owners, runs the
 *                      owner's backward on the forward's plan, and sum
 *                      all-reduces the replicated cores' gradients (every
 *                      core but F, with their touch counters); the owned G_F
 *                      slices and their optimizer state never cross NVLink.
 *   tt_owner_step      tt_step with the non-finite verdict min-reduced over
 *                      the ranks first (all apply or all reject).
 *   tt_owner_rows      IDs this rank received in the last tt_owner_forward. */
int tt_owner_forward(tt_engine* h, const int64_t* d_indices, int64_t batch, float* d_out, void* stream);
int tt_owner_backward(tt_engine* h, const float* d_grad_out, void* stream);
int tt_owner_step(tt_engine* h, void* stream);
int64_t tt_owner_rows(tt_engine* h);

/* ---- introspection -------------------------------------------------------- */
/* Distinct prefixes (i_1..i_l), l = 1..d, of the last planned batch
 * (unique_per_level[d-1] = distinct IDs).  Synchronises. */
int tt_plan_stats(tt_engine* h, int64_t* unique_per_level);
/* Per-level digits of the last planned batch's distinct IDs, sorted
 * ascending (digits[u*d + k] = i_{k+1}); returns U.  Synchronises. */
int64_t tt_plan_digits(tt_engine* h, int64_t* ids_out, int32_t* digits_out, int64_t cap);
/* The last planned batch's stable sort: keys (IDs) ascending and their batch
 * positions (ties in position order); returns B.  Synchronises. */
int64_t tt_plan_sorted(tt_engine* h, int64_t* keys_out, int32_t* pos_out, int64_t cap);
/* Per-phase device timing with CUDA events recorded on the launching stream:
 * slot 0 plan (K1+K2), 1 forward main kernel(s), 2 backward main kernel(s),
 * 3 backward auxiliary kernels, 4 update (K5).  tt_profile_read synchronises
 * and returns total milliseconds and event-pair counts per slot, then resets. */
int tt_set_profiling(tt_engine* h, int on);
int tt_profile_read(tt_engine* h, double* ms, int64_t* counts, int nslots);
/* Kernel launches issued by this handle since creation. */
int64_t tt_launch_count(tt_engine* h);
/* Debug: per-CTA phase timestamps of the last backward GEMM launch when the
 * process runs with TT_TC_TRACE=1 (scripts/tc_trace.py); returns the number
 * of int64 values copied (0 when tracing is off). */
int64_t tt_debug_trace(long long* out, int64_t n);
/* Selects the kernel family: 0 = auto (fused FFMA fast path where the shapes
 * allow), 1 = generic path only, 2 = fused with the optional tensor-core
 * (tcgen05, BF16x3 split, FP32 accumulation) contraction where compiled for
 * the shape (reported separately). */
int tt_set_path(tt_engine* h, int path);
/* Which path the last forward used (0 generic, 1 fused FFMA, 2 fused tcgen05). */
int tt_last_path(tt_engine* h);
/* Batch position (TT_ERR_INDEX) or core (TT_ERR_NONFINITE) of the last error. */
int64_t tt_last_error_position(void);
/* Offending index value of the last TT_ERR_INDEX. */
int64_t tt_last_error_value(void);
const char* tt_last_error(void);

/* FP32 FFMA throughput microbenchmark (the roofline denominator): runs
 * `iters` dependent-chain FFMA loops on every SM and returns TFLOP/s. */
double tt_ffma_peak_tflops(int device, int iters);
/* The same with GEMM-shaped 3-register FFMAs (8x8 register outer product per
 * thread): the FFMA rate an SGEMM-style micro-kernel can reach. */
double tt_ffma_outer_tflops(int device, int iters);

#ifdef __cplusplus
}
#endif

#endif /* TT_ENGINE_H */
