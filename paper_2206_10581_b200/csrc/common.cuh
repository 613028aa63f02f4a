// common.cuh -- shared device-side definitions for the TT engine (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define TT_MAXD 8

// Configuration passed by value to every kernel.  Core k (0-based) has shape
// (R[k], m[k], n[k], R[k+1]); on the device it is stored slice-major,
// [m_k][R_k][n_k][R_{k+1}], so slice G_k(:, i, :, :) is one contiguous
// R_k x (n_k R_{k+1}) matrix (the reference layout is (R,m,n,R),
// tt_embedding.hpp:28-32, whose slices are strided).
struct DevCfg {
  int d;
  int pad_;
  int64_t num_nodes, emb_dim, npad;      // npad = prod(n)
  int64_t m[TT_MAXD], n[TT_MAXD], R[TT_MAXD + 1];
  int64_t S[TT_MAXD];        // S[k] = prod_{p>k} m_p (suffix radix), S[d-1] = 1
  int64_t rows[TT_MAXD];     // rows[k] = prod_{p<k} n_p  (A rows per node at level k)
  int64_t cols[TT_MAXD];     // cols[k] = n_k R_{k+1}
  int64_t slice[TT_MAXD];    // slice size R_k n_k R_{k+1}
  int64_t core_off[TT_MAXD]; // offset of core k in the parameter buffer
  int64_t tc_off[TT_MAXD];   // offset of core k's touch counters (after all grads)
  int64_t nparams;           // total parameters
};

// Deferred device-side error record.
struct DevStatus {
  unsigned long long bad_pos;  // min out-of-range batch position, ~0 if none
  int bad_core;                // min core with a non-finite gradient, INT_MAX if none
  int pad_;
};

#define TT_NO_POS 0xFFFFFFFFFFFFFFFFull

// Programmatic dependent launch: every kernel is launched with programmatic
// stream serialisation (engine.cu tt_launch), lets its dependent grid be
// scheduled once all of its CTAs are resident, and waits for the full
// completion (and memory visibility) of the grid before it before touching
// any data.  The dependency semantics are those of plain stream order; only
// the launch latency between consecutive kernels overlaps.
#define TT_PDL_ENTRY()                                         \
  do {                                                         \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    asm volatile("griddepcontrol.wait;" ::: "memory");         \
  } while (0)

__device__ __forceinline__ bool tt_failed(const DevStatus* st) {
  return *(volatile const unsigned long long*)&st->bad_pos != TT_NO_POS;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <class T>
__device__ __forceinline__ T ld_count(const T* p) { return *(volatile const T*)p; }
