// kernels_update.cuh -- K5: all-or-nothing optimizer update
// (apply_update, autodiff.cpp:147-173) on the device-layout parameters.
//
// Phase 1 checks every gradient entry of every touched slice for NaN/Inf and
// records the first offending core; phase 2 applies SGD / Adagrad to touched
// slices only (identical to the dense update for these optimizers: g = 0
// leaves p and h bit-identical) or Adam densely (its moments decay
// everywhere), and does nothing at all if phase 1 found a bad entry.  The
// step counter lives on the device and advances only on success.
// HBM bound: SGD moves 12 B/param touched, Adagrad 20 B, Adam 28 B.
#pragma once
#include <limits.h>
#include "common.cuh"

namespace tt {

__device__ __forceinline__ int core_of(const DevCfg& c, int64_t e) {
  int k = 0;
#pragma unroll 1
  while (k + 1 < c.d && e >= c.core_off[k + 1]) ++k;
  return k;
}

__global__ void k_check_finite(DevCfg c, const float* __restrict__ grads, DevStatus* st) {
  if (tt_failed(st)) return;
  int bad = INT_MAX;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < c.nparams; e += (int64_t)gridDim.x * blockDim.x) {
    const float g = grads[e];
    if (!isfinite(g)) {
      const int k = core_of(c, e);
      const int64_t v = (e - c.core_off[k]) / c.slice[k];
      if (grads[c.tc_off[k] + v] > 0.f && k < bad) bad = k;
    }
  }
  if (bad != INT_MAX) atomicMin(&st->bad_core, bad);
}

// kind: 0 SGD, 1 Adam, 2 Adagrad.  Vectorised float4 path where a 4-group
// stays inside one slice (slice sizes are multiples of 4 at every BASELINE
// config; the scalar tail handles the rest).
__global__ void k_update(DevCfg c, float* __restrict__ p, const float* __restrict__ grads,
                         float* __restrict__ s1, float* __restrict__ s2, int kind, float lr, float b1, float b2,
                         float eps, const long long* __restrict__ step_ptr, const DevStatus* st) {
  if (tt_failed(st) || ld_count(&st->bad_core) != INT_MAX) return;
  const long long step = *step_ptr + 1;
  float bc1 = 1.f, bc2 = 1.f;
  if (kind == 1) {
    bc1 = (float)(1.0 - pow((double)b1, (double)step));
    bc2 = (float)(1.0 - pow((double)b2, (double)step));
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < c.nparams; e += (int64_t)gridDim.x * blockDim.x) {
    const float g = grads[e];
    if (kind != 1) {
      const int k = core_of(c, e);
      const int64_t v = (e - c.core_off[k]) / c.slice[k];
      if (!(grads[c.tc_off[k] + v] > 0.f)) continue;
    }
    if (kind == 0) {
      p[e] = p[e] - lr * g;
    } else if (kind == 2) {
      const float h = s1[e] + g * g;
      s1[e] = h;
      p[e] = p[e] - lr * g / (sqrtf(h) + eps);
    } else {
      const float m = b1 * s1[e] + (1.f - b1) * g;
      const float v = b2 * s2[e] + (1.f - b2) * g * g;
      s1[e] = m;
      s2[e] = v;
      p[e] = p[e] - lr * (m / bc1) / (sqrtf(v / bc2) + eps);
    }
  }
}

__global__ void k_commit_step(long long* step_ptr, const DevStatus* st) {
  if (!tt_failed(st) && ld_count(&st->bad_core) == INT_MAX) *step_ptr += 1;
}

// zero the gradient values of the slices touched by the current batch only
__global__ void k_zero_grads(float* __restrict__ g, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    g[e] = 0.f;
}

// FFMA throughput microbenchmark: 8 independent chains per thread.
__global__ void __launch_bounds__(256) k_ffma_peak(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 1234.5f) out[blockIdx.x] = s;
}

}  // namespace tt
