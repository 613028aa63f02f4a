// tc_rate.cu -- throughput of the BF16 tcgen05.mma shapes the TT kernels use,
// from the no-swizzle core-matrix planes (tc_sm100.cuh): cycles per MMA for
// M=128 and N in {64,128,256}, K-major / MN-major operands, one CTA per SM.
#include <cstdio>
#include "../../paper_2206_10581_b200/csrc/tc_sm100.cuh"
using namespace tt::tc;

template <int N>
__global__ void rate(long long* out, int reps, int a_mn, int b_mn) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x;
  for (int i = t; i < (128 * 128 + N * 128) * 2 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (t < 32) tmem_alloc<256>(&slot);
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_async_smem(); before_sync(); __syncthreads(); after_sync();
  const uint32_t tm = slot;
  long long c0 = clock64();
  if (t == 0) {
    const uint32_t A = smem_u32(sm), B = smem_u32(sm + 128 * 128 * 2);
    Operand oa = a_mn ? mnmajor(A, A, A, 128) : kmajor(A, A, A, 128);  // A: 128 x 128 (K = 128)
    Operand ob = b_mn ? mnmajor(B, B, B, N) : kmajor(B, B, B, 128);
    const uint32_t id = idesc_bf16(128, N, a_mn, b_mn);
    for (int r = 0; r < reps; ++r) {
      for (int k = 0; k < 8; ++k) {
        const uint64_t da = sdesc(oa.plane[0] + k * oa.kstep, oa.lbo, oa.sbo);
        const uint64_t db = sdesc(ob.plane[0] + k * ob.kstep, ob.lbo, ob.sbo);
        mma_bf16(tm, da, db, id, 1u);
      }
    }
    commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  long long c1 = clock64();
  if (t == 0) out[blockIdx.x] = c1 - c0;
  before_sync(); __syncthreads();
  if (t < 32) tmem_free<256>(tm);
}

template <int N>
void run(int a_mn, int b_mn) {
  long long* d; cudaMalloc(&d, 148 * 8);
  const int smem = (128 * 128 + N * 128) * 2;
  cudaFuncSetAttribute(rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 200;
  rate<N><<<148, 128, smem>>>(d, 4, a_mn, b_mn);
  rate<N><<<148, 128, smem>>>(d, reps, a_mn, b_mn);
  cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0; for (int i = 0; i < 148; ++i) cyc += h[i]; cyc /= 148;
  const double per = cyc / (reps * 8.0);
  const double macs = 128.0 * N * 16;
  printf("M=128 N=%3d a_mn=%d b_mn=%d: %.1f cycles/MMA  (%.0f MAC/clk/SM, floor %d cyc; smem %.0f B/clk)\n", N, a_mn, b_mn,
         per, macs / per, 128 * N / 256, (128 * 16 * 2 + N * 16 * 2) / per);
  cudaFree(d);
}

int main() {
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) { run<64>(a, b); run<128>(a, b); run<256>(a, b); }
  return 0;
}
