// tc_probe_ts.cu -- validates the TMEM-A form of the BF16x3 product
// (tc_sm100.cuh mma_x3_ts): D (128 x N) = A (128 x 64, written to TMEM with
// tcgen05.st, one row per lane) . B (64 x N, shared memory, K- or MN-major),
// against an fp64 host product.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_probe_ts tc_probe_ts.cu
#include <cstdio>
#include <cmath>
#include <vector>
#include <random>
#include "../../paper_2206_10581_b200/csrc/tc_sm100.cuh"

using namespace tt::tc;

constexpr int M = 128, K = 64;

template <int N>
__global__ void probe(const float* A, const float* B, float* D, int b_mn) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* pb[3];
  for (int i = 0; i < 3; ++i) pb[i] = sm + i * (N * K * 2);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  const int bR = b_mn ? K : N, bC = b_mn ? N : K;
  for (int u = t; u < bR * bC / 8; u += blockDim.x) {
    const int r = u / (bC / 8), c0 = (u % (bC / 8)) * 8;
    float x[8];
    for (int i = 0; i < 8; ++i) {
      const int n = b_mn ? c0 + i : r, k = b_mn ? r : c0 + i;
      x[i] = B[k * N + n];
    }
    store_split8(pb[0], pb[1], pb[2], r, c0, bC, x);
  }
  if (t < 32) tmem_alloc<512>(&tslot);
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_async_smem();
  before_sync();
  __syncthreads();
  after_sync();
  const uint32_t tm = tslot;
  const uint32_t ta = tm + N;  // A slices at columns N, N + 32, N + 64
  {
    const int m = 32 * w + l;  // TMEM lane = row
    uint32_t s[3][32];
    for (int k = 0; k < K; k += 2) split3(A[m * K + k], A[m * K + k + 1], s[0][k / 2], s[1][k / 2], s[2][k / 2]);
    for (int p = 0; p < 3; ++p) {
      uint32_t lo[16], hi[16];
      for (int i = 0; i < 16; ++i) { lo[i] = s[p][i]; hi[i] = s[p][16 + i]; }
      tmem_st16(ta + ((uint32_t)(32 * w) << 16) + p * (K / 2), lo);
      tmem_st16(ta + ((uint32_t)(32 * w) << 16) + p * (K / 2) + 16, hi);
    }
    tmem_st_wait();
  }
  before_sync();
  __syncthreads();
  after_sync();
  if (t == 0) {
    Operand ob = b_mn ? mnmajor(smem_u32(pb[0]), smem_u32(pb[1]), smem_u32(pb[2]), bC)
                      : kmajor(smem_u32(pb[0]), smem_u32(pb[1]), smem_u32(pb[2]), bC);
    mma_x3_ts<K / 16>(tm, ta, ob, idesc_bf16(M, N, 0, b_mn), false);
    commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  after_sync();
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tm + ((uint32_t)(32 * w) << 16) + c, v);
    for (int i = 0; i < 16; ++i) D[(32 * w + l) * N + c + i] = v[i];
  }
  before_sync();
  __syncthreads();
  if (t < 32) tmem_free<512>(tm);
}

template <int N>
int run(int b_mn) {
  std::mt19937 g(77 + N + 13 * b_mn);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<float> A(M * K), B(K * N), D(M * N);
  for (auto& x : A) x = nd(g);
  for (auto& x : B) x = nd(g);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xFF, D.size() * 4);
  const int smem = 3 * N * K * 2;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N><<<1, 128, smem>>>(dA, dB, dD, b_mn);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("N=%d b_mn=%d CUDA error %s\n", N, b_mn, cudaGetErrorString(e)); return 1; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double worst = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0, sa = 0;
      for (int k = 0; k < K; ++k) { s += (double)A[m * K + k] * B[k * N + n]; sa += fabs((double)A[m * K + k] * B[k * N + n]); }
      const double err = fabs(D[m * N + n] - s) / sa;
      if (!(err <= worst)) worst = err;
    }
  printf("TMEM-A N=%3d b_mn=%d  max|err|/sum|ab| = %.3e  D[0]=%f\n", N, b_mn, worst, D[0]);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return worst < 1e-6 ? 0 : 1;
}

int main() {
  int bad = 0;
  for (int b = 0; b < 2; ++b) { bad += run<64>(b); bad += run<128>(b); bad += run<256>(b); }
  printf(bad ? "FAIL %d\n" : "ALL OK\n", bad);
  return bad;
}
