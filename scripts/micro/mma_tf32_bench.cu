// Microbenchmark: legacy warp-level mma.sync m16n8k8 TF32 throughput on this GPU
// (is a 3xTF32 register-fragment path worth it versus FFMA?).  Build/run:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a mma_tf32_bench.cu -o /tmp/mma && /tmp/mma
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, int iters) {
  unsigned a0 = __float_as_uint(1.0f + threadIdx.x), a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  unsigned b0 = __float_as_uint(0.5f), b1 = b0 + 7;
  float c[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 1.2345f) out[0] = s;
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* o; cudaMalloc(&o, 4);
  for (int warps : {4, 8, 16}) {
    int blocks = nsm * 2, iters = 4096;
    k<<<blocks, warps * 32>>>(o, 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<blocks, warps * 32>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 8 * 8.0 * iters * warps * blocks;
    printf("warps/block %2d: mma.sync tf32 %.1f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
