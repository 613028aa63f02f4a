// kernels_init.cuh -- the ortho-core initializer on the device (SURVEY 8f
// row f3; init_ortho_core, initializer.cpp:103-132).
//
// Core k needs count = n_k R_{k-1} orthonormal vectors of length
// dim = m_k R_k.  They are drawn i.i.d. N(0, 1) from a counter-based,
// portable generator (splitmix64 + Box-Muller of (seed, core, vector, attempt,
// element)).  The reference's std::mt19937_64 + std::normal_distribution
// stream is implementation-defined, so the draws are not the reference's.
// They are orthonormalised in fp64 by Gram-Schmidt with one
// re-orthogonalisation pass (classical projections per pass -- CGS2, which
// reaches the reference's MGS2 orthogonality, gram_schmidt_rows
// initializer.cpp:54-80, and parallelises over the previous vectors) and the
// reference's bounded redraw of degenerate vectors.
#pragma once
#include "common.cuh"

namespace tt {

__device__ __forceinline__ unsigned long long gs_mix(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// v[j] = N(0,1) draw for (seed, core, row, attempt, j)
__global__ void k_gs_draw(double* __restrict__ v, int64_t dim, unsigned long long seed, int core, int row,
                          int attempt) {
  TT_PDL_ENTRY();
  const unsigned long long key =
      gs_mix(seed ^ gs_mix(((unsigned long long)core << 48) ^ ((unsigned long long)row << 8) ^ (unsigned)attempt));
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < dim; j += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long a = gs_mix(key ^ (2 * (unsigned long long)j));
    const unsigned long long b = gs_mix(key ^ (2 * (unsigned long long)j + 1));
    const double u1 = ((double)(a >> 11) + 1.0) * (1.0 / 9007199254740992.0);  // (0, 1]
    const double u2 = (double)(b >> 11) * (1.0 / 9007199254740992.0);
    v[j] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925 * u2);
  }
}

// block-wide sum of a double (256 threads)
__device__ __forceinline__ double gs_block_sum(double x, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

// dots[p] = <Q[p], v>, p < nprev (one block per previous vector; fixed order)
__global__ void __launch_bounds__(256) k_gs_dots(const double* __restrict__ Q, const double* __restrict__ v, int64_t dim,
                                                 double* __restrict__ dots) {
  TT_PDL_ENTRY();
  __shared__ double red[8];
  const int p = blockIdx.x;
  const double* q = Q + (int64_t)p * dim;
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < dim; j += blockDim.x) s += q[j] * v[j];
  s = gs_block_sum(s, red);
  if (threadIdx.x == 0) dots[p] = s;
}

// v -= sum_p dots[p] Q[p]  (one classical projection pass)
__global__ void k_gs_axpy(const double* __restrict__ Q, double* __restrict__ v, int64_t dim,
                          const double* __restrict__ dots, int nprev) {
  TT_PDL_ENTRY();
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < dim; j += (int64_t)gridDim.x * blockDim.x) {
    double x = v[j];
    for (int p = 0; p < nprev; ++p) x -= dots[p] * Q[(int64_t)p * dim + j];
    v[j] = x;
  }
}

// out[0] = |v|^2 (one block)
__global__ void __launch_bounds__(256) k_gs_sumsq(const double* __restrict__ v, int64_t dim, double* __restrict__ out) {
  TT_PDL_ENTRY();
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < dim; j += blockDim.x) s += v[j] * v[j];
  s = gs_block_sum(s, red);
  if (threadIdx.x == 0) out[0] = s;
}

__global__ void k_gs_scale(double* __restrict__ v, int64_t dim, double inv) {
  TT_PDL_ENTRY();
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < dim; j += (int64_t)gridDim.x * blockDim.x)
    v[j] *= inv;
}

}  // namespace tt
