// tmem_shapes.cu -- which (TMEM lane, column) each thread receives from the
// tcgen05.ld shapes 32x32b / 16x64b / 16x128b / 16x256b (values written with
// 32x32b stores: lane*1000 + column).
#include <cstdio>
#include <cstdint>
#include "../../paper_2206_10581_b200/csrc/tc_sm100.cuh"
using namespace tt::tc;

__global__ void k(int* out) {
  __shared__ uint32_t slot;
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  if (w == 0) tmem_alloc<64>(&slot);
  before_sync(); __syncthreads(); after_sync();
  const uint32_t tm = slot;
  // each warp writes its lane quadrant: lane 32w+l, columns 0..15
  uint32_t v[16];
  for (int c = 0; c < 16; ++c) v[c] = (32 * w + l) * 1000 + c;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
               :: "r"(tm + ((uint32_t)(32 * w) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                  "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  before_sync(); __syncthreads(); after_sync();
  if (w == 0) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int i = 0; i < 4; ++i) out[l * 8 + i] = r[i];
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];\n" : "=r"(r[0]), "=r"(r[1]) : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int i = 0; i < 2; ++i) out[256 + l * 8 + i] = r[i];
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];\n" : "=r"(r[0]) : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    out[512 + l * 8] = r[0];
  }
  before_sync(); __syncthreads();
  if (w == 0) tmem_free<64>(tm);
}

int main() {
  int* d; cudaMalloc(&d, 4096 * 4); cudaMemset(d, 0xff, 4096 * 4);
  k<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  int h[4096]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[3] = {"16x256b", "16x128b", "16x64b"};
  int cnt[3] = {4, 2, 1};
  for (int s = 0; s < 3; ++s) {
    printf("%s:\n", nm[s]);
    for (int l = 0; l < 32; ++l) {
      printf("  t%02d:", l);
      for (int i = 0; i < cnt[s]; ++i) { int v = h[s * 256 + l * 8 + i]; printf(" (lane %d col %d)", v / 1000, v % 1000); }
      printf("\n");
    }
  }
  return 0;
}
