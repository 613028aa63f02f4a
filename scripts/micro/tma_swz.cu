// Does a SWIZZLE_128B TMA box of 4 rows land at a 512-byte (not 1024-byte)
// aligned shared-memory offset, and is its swizzle a function of the shared
// address (chunk ^= (addr >> 7) & 7)?  nvcc -gencode arch=compute_100a,code=sm_100a tma_swz.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void k(const __grid_constant__ CUtensorMap map, float* out, int nbox, const int* rows, const int* offs) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 8192 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = -1.f;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nbox * 512));
    for (int i = 0; i < nbox; ++i) {
      unsigned dst = (unsigned)__cvta_generic_to_shared(sm + offs[i]);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(dst), "l"(&map), "r"(0), "r"(rows[i]), "r"(b) : "memory");
    }
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(b));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8192 / 4; i += blockDim.x) out[i] = reinterpret_cast<float*>(sm)[i];
}

int main() {
  const int R = 64, C = 32;
  float h[R * C];
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = r * 100 + c;
  float* d; cudaMalloc(&d, sizeof(h)); cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
  cuuint64_t strides[1] = {C * 4};
  cuuint32_t box[2] = {32, 4}, es[2] = {1, 1};
  CUresult e = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)e);
  // boxes: rows 8..11 -> smem 0, rows 20..23 -> smem 512, rows 40..43 -> smem 1536
  int hrows[3] = {8, 20, 40}, hoffs[3] = {0, 512, 1536};
  int *drows, *doffs; cudaMalloc(&drows, 12); cudaMalloc(&doffs, 12);
  cudaMemcpy(drows, hrows, 12, cudaMemcpyHostToDevice); cudaMemcpy(doffs, hoffs, 12, cudaMemcpyHostToDevice);
  float* dout; cudaMalloc(&dout, 8192);
  k<<<1, 128, 8192>>>(map, dout, 3, drows, doffs);
  cudaError_t ce = cudaDeviceSynchronize();
  printf("kernel %s\n", cudaGetErrorString(ce));
  float o[2048]; cudaMemcpy(o, dout, 8192, cudaMemcpyDeviceToHost);
  int bad = 0, checked = 0;
  for (int b = 0; b < 3; ++b)
    for (int rr = 0; rr < 4; ++rr)
      for (int c = 0; c < 32; ++c) {
        const int addr = hoffs[b] + rr * 128;  // logical row start
        const int chunk = c / 4, phys = chunk ^ ((addr >> 7) & 7);
        const float v = o[(addr + phys * 16 + (c % 4) * 4) / 4];
        ++checked;
        if (v != (hrows[b] + rr) * 100 + c) ++bad;
      }
  printf("address-based swizzle: %d / %d mismatches\n", bad, checked);
  return 0;
}
