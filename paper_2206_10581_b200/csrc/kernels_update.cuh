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

// core index and slice of flat parameter e (d <= 8, unrolled compares)
__device__ __forceinline__ void locate(const DevCfg& c, int64_t e, int& k, int64_t& v) {
  k = 0;
#pragma unroll
  for (int q = 1; q < TT_MAXD; ++q)
    if (q < c.d && e >= c.core_off[q]) k = q;
  v = (e - c.core_off[k]) / c.slice[k];
}

// Vectorised over 4-element groups when every core offset and slice size is a
// multiple of 4 (then a group never straddles slices); scalar otherwise.
__global__ void k_check_finite(DevCfg c, const float* __restrict__ grads, int vec4, DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st)) return;
  int bad = INT_MAX;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  if (vec4) {
    // four independent 16-byte loads per thread per step
    const int64_t n4 = c.nparams / 4;
    for (int64_t q0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q0 < n4; q0 += 4 * step) {
      float4 g[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (q0 + i * step < n4) g[i] = reinterpret_cast<const float4*>(grads)[q0 + i * step];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t q = q0 + i * step;
        if (q < n4 && !(isfinite(g[i].x) && isfinite(g[i].y) && isfinite(g[i].z) && isfinite(g[i].w))) {
          int k;
          int64_t v;
          locate(c, q * 4, k, v);
          if (grads[c.tc_off[k] + v] > 0.f && k < bad) bad = k;
        }
      }
    }
  } else {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < c.nparams; e += step) {
      if (!isfinite(grads[e])) {
        int k;
        int64_t v;
        locate(c, e, k, v);
        if (grads[c.tc_off[k] + v] > 0.f && k < bad) bad = k;
      }
    }
  }
  if (bad != INT_MAX) atomicMin(&st->bad_core, bad);
}

template <int KIND>
__device__ __forceinline__ void upd1(float& p, float g, float& h, float& v2, float lr, float b1, float b2, float eps,
                                     float bc1, float bc2) {
  if (KIND == 0) {
    p = p - lr * g;
  } else if (KIND == 2) {
    h = h + g * g;
    p = p - lr * g / (sqrtf(h) + eps);
  } else {
    h = b1 * h + (1.f - b1) * g;
    v2 = b2 * v2 + (1.f - b2) * g * g;
    p = p - lr * (h / bc1) / (sqrtf(v2 / bc2) + eps);
  }
}

// KIND: 0 SGD, 1 Adam (dense), 2 Adagrad (touched slices only; identical to
// the dense update since g = 0 leaves p and h bit-identical).
template <int KIND>
__global__ void k_update(DevCfg c, float* __restrict__ p, const float* __restrict__ grads, float* __restrict__ s1,
                         float* __restrict__ s2, int vec4, float lr, float b1, float b2, float eps,
                         const long long* __restrict__ step_ptr, const DevStatus* st) {
  TT_PDL_ENTRY();
  if (tt_failed(st) || ld_count(&st->bad_core) != INT_MAX) return;
  float bc1 = 1.f, bc2 = 1.f;
  if (KIND == 1) {
    const long long step = *step_ptr + 1;
    bc1 = (float)(1.0 - pow((double)b1, (double)step));
    bc2 = (float)(1.0 - pow((double)b2, (double)step));
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float dummy = 0.f;
  if (vec4) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < c.nparams / 4; q += stride) {
      int k;
      int64_t v;
      locate(c, q * 4, k, v);
      const bool touched = grads[c.tc_off[k] + v] > 0.f;
      if (KIND != 1 && !touched) continue;
      // Adam runs densely; a slice this batch did not touch has g = 0 (the
      // buffer may still hold an earlier batch's values there)
      const float4 g = touched ? reinterpret_cast<const float4*>(grads)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 pv = reinterpret_cast<float4*>(p)[q];
      float4 hv = KIND != 0 ? reinterpret_cast<float4*>(s1)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 vv = KIND == 1 ? reinterpret_cast<float4*>(s2)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
      upd1<KIND>(pv.x, g.x, hv.x, vv.x, lr, b1, b2, eps, bc1, bc2);
      upd1<KIND>(pv.y, g.y, hv.y, vv.y, lr, b1, b2, eps, bc1, bc2);
      upd1<KIND>(pv.z, g.z, hv.z, vv.z, lr, b1, b2, eps, bc1, bc2);
      upd1<KIND>(pv.w, g.w, hv.w, vv.w, lr, b1, b2, eps, bc1, bc2);
      reinterpret_cast<float4*>(p)[q] = pv;
      if (KIND != 0) reinterpret_cast<float4*>(s1)[q] = hv;
      if (KIND == 1) reinterpret_cast<float4*>(s2)[q] = vv;
    }
  } else {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < c.nparams; e += stride) {
      int k;
      int64_t v;
      locate(c, e, k, v);
      const bool touched = grads[c.tc_off[k] + v] > 0.f;
      if (KIND != 1 && !touched) continue;
      float h = KIND != 0 ? s1[e] : 0.f, v2 = KIND == 1 ? s2[e] : 0.f;
      upd1<KIND>(p[e], touched ? grads[e] : 0.f, KIND != 0 ? s1[e] : dummy, KIND == 1 ? s2[e] : dummy, lr, b1, b2, eps,
                 bc1, bc2);
      (void)h;
      (void)v2;
    }
  }
}

__global__ void k_commit_step(long long* step_ptr, const DevStatus* st) {
  TT_PDL_ENTRY();
  if (!tt_failed(st) && ld_count(&st->bad_core) == INT_MAX) *step_ptr += 1;
}

// zero the gradient values of the slices touched by the current batch only
__global__ void k_zero_grads(float* __restrict__ g, int64_t n) {
  TT_PDL_ENTRY();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    g[e] = 0.f;
}

// FFMA throughput microbenchmark: 8 independent chains per thread.
__global__ void __launch_bounds__(256) k_ffma_peak(float* out, int iters, float a, float b) {
  TT_PDL_ENTRY();
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

// GEMM-like FFMA microbenchmark: an 8x8 register outer product per thread
// (3-register FFMAs, operands reused as in an SGEMM micro-kernel).
__global__ void __launch_bounds__(256) k_ffma_outer(float* out, int iters, float s0) {
  TT_PDL_ENTRY();
  float a[8], b[8], acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = s0 + threadIdx.x * 0.001f + i;
    b[i] = s0 - i * 0.5f;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      a[i] = __int_as_float(__float_as_int(a[i]) ^ 1);
      b[i] = __int_as_float(__float_as_int(b[i]) ^ 2);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) s += acc[i][j];
  if (s == 1234.5f) out[blockIdx.x] = s;
}

}  // namespace tt
