// tc_rate.cu -- throughput of the BF16 tcgen05.mma shapes the TT kernels use,
// from the no-swizzle core-matrix planes (tc_sm100.cuh): cycles per MMA for
// M=128 and N in {64,128,256}, K-major / MN-major operands, one CTA per SM;
// A from shared memory (aliased or distinct slices) or from TMEM (mode 2);
// optionally with the other three warps streaming 16-byte shared loads
// (noise) to measure the contention between the tensor pipe and the LSU.
#include <cstdio>
#include <cstdlib>
#include "../../paper_2206_10581_b200/csrc/tc_sm100.cuh"
using namespace tt::tc;

template <int N>
__global__ void rate(long long* out, int reps, int a_mn, int b_mn, int mode, int noise, float* sink) {
  const int distinct = mode >= 1;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x;
  const int words = (mode == 2 ? 3 * N * 128 : (distinct ? 3 : 1) * (128 * 128 + N * 128)) * 2 / 4;
  for (int i = t; i < words; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (t < 32) tmem_alloc<512>(&slot);
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_async_smem(); before_sync(); __syncthreads(); after_sync();
  const uint32_t tm = slot;
  __shared__ volatile int done;
  if (t == 0) done = 0;
  __syncthreads();
  long long c0 = clock64();
  if (t >= 32 && noise == 2) {
    // global store stream: 16-byte stores, 4 full lines per warp instruction
    float4* q = reinterpret_cast<float4*>(sink) + (size_t)blockIdx.x * (1 << 20);
    int i = t - 32;
    while (!done) {
#pragma unroll 8
      for (int j = 0; j < 32; ++j) q[(i + j * 96) & ((1 << 20) - 1)] = make_float4(1.f, 2.f, 3.f, (float)j);
      i += 96 * 32;
    }
  }
  if (t >= 32 && noise == 3) {
    // global load stream (L2-resident 2 MB window per CTA)
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* q = reinterpret_cast<const float4*>(sink) + (size_t)blockIdx.x * (1 << 17);
    int i = t - 32;
    while (!done) {
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const float4 x = __ldcg(q + ((i + j * 96) & ((1 << 17) - 1)));
        acc.x += x.x; acc.y += x.y;
      }
      i += 96 * 32;
    }
    if (acc.x == 1234.f) sink[t] = acc.y;
  }
  if (t >= 32 && noise == 4) {
    // TMEM loads of an idle region (columns 448..511) while the MMAs run:
    // count completed 4 x 16-column load groups
    const int w = t >> 5;
    uint32_t r[64];
    long long iters = 0;
    while (!done) {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld16_async(tm + ((uint32_t)(32 * w) << 16) + 448 + 16 * c, r + 16 * c);
      tmem_ld_wait();
      ++iters;
    }
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 64; ++i) x ^= r[i];
    if (x == 12345u) sink[t] = 1.f;
    if ((t & 31) == 0) out[148 + blockIdx.x * 4 + w] = iters;
  }
  if (t >= 32 && noise == 1) {
    // LSU traffic: 16-byte shared loads over the operand region
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* p = reinterpret_cast<const float4*>(sm);
    int i = t;
    while (!done) {
#pragma unroll 8
      for (int j = 0; j < 64; ++j) {
        const float4 x = p[(i + j * 96) & 2047];
        acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      }
      i += 7;
    }
    if (acc.x == 1234.f) sink[t] = acc.y + acc.z + acc.w;
  }
  if (t == 0) {
    // A planes: 3 x (128 x 128), B planes: 3 x (N x 128) -- distinct or aliased
    const uint32_t base = smem_u32(sm), pa = 128 * 128 * 2, pb = N * 128 * 2;
    const uint32_t A0 = base, A1 = distinct ? base + pa : base, A2 = distinct ? base + 2 * pa : base;
    const uint32_t B0 = mode == 2 ? base : base + (distinct ? 3 : 1) * pa, B1 = distinct ? B0 + pb : B0, B2 = distinct ? B0 + 2 * pb : B0;
    Operand oa = a_mn ? mnmajor(A0, A1, A2, 128) : kmajor(A0, A1, A2, 128);  // A: 128 x 128 (K = 128)
    Operand ob = b_mn ? mnmajor(B0, B1, B2, N) : kmajor(B0, B1, B2, 128);
    const uint32_t id = idesc_bf16(128, N, a_mn, b_mn);
    if (mode == 2)
      for (int r = 0; r < reps; ++r) mma_x3_ts<8>(tm, tm + 256, ob, idesc_bf16(128, N, 0, b_mn), true);
    else
      for (int r = 0; r < reps; ++r) mma_x3<8>(tm, oa, ob, id, true);  // 48 MMAs (6 products x 8 k-steps)
    commit(&bar);
  }
  if (t < 32) {
    __syncwarp();
    mbar_wait(&bar, 0);
    long long c1 = clock64();
    if (t == 0) { out[blockIdx.x] = c1 - c0; done = 1; }
  }
  before_sync(); __syncthreads();
  if (t < 32) tmem_free<512>(tm);
}

template <int N>
void run(int a_mn, int b_mn, int mode, int noise) {
  const int distinct = mode >= 1;
  long long* d; cudaMalloc(&d, 148 * 8 * 5);
  cudaMemset(d, 0, 148 * 8 * 5);
  float* sink; cudaMalloc(&sink, (size_t)148 << 24);  // 16 MB per CTA
  const int smem = (mode == 2 ? 3 * N * 128 : (distinct ? 3 : 1) * (128 * 128 + N * 128)) * 2;
  if (smem > 227 * 1024) { cudaFree(d); return; }
  cudaFuncSetAttribute(rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 40;
  rate<N><<<148, 128, smem>>>(d, 2, a_mn, b_mn, mode, noise, sink);
  rate<N><<<148, 128, smem>>>(d, reps, a_mn, b_mn, mode, noise, sink);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("N=%d mode=%d noise=%d: %s\n", N, mode, noise, cudaGetErrorString(e)); exit(1); }
  long long h[148 * 5]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (noise == 4) {
    double it = 0;
    for (int i = 0; i < 148; ++i) it += h[148 + i * 4 + 1];
    it /= 148;
    printf("    TMEM-load warp: %.0f groups of 4 x ld16 during %.0f cycles of MMAs = %.0f cycles per group\n", it,
           (double)h[0], h[0] / (it > 0 ? it : 1));
  }
  double cyc = 0; for (int i = 0; i < 148; ++i) cyc += h[i]; cyc /= 148;
  const double per = cyc / (reps * 48.0);
  const double macs = 128.0 * N * 16;
  const double opbytes = (mode == 2 ? 0 : 128 * 16 * 2) + N * 16 * 2;
  printf("%s%s M=128 N=%3d a_mn=%d b_mn=%d: %.1f cycles/MMA  (%.0f MAC/clk/SM, floor %d cyc; operand smem %.0f B/clk)\n",
         mode == 2 ? "A in TMEM       " : distinct ? "distinct planes " : "aliased planes  ", noise == 1 ? " +LDS" : noise == 2 ? " +STG" : noise == 3 ? " +LDG" : noise == 4 ? " +TLD" : "     ", N,
         a_mn, b_mn, per, macs / per, 128 * N / 256, opbytes / per);
  cudaFree(d); cudaFree(sink);
}

int main() {
  for (int noise = 0; noise < 5; ++noise) {
    if (noise > 0 && noise < 4) continue;
    run<64>(0, 1, 1, noise); run<128>(0, 1, 1, noise);
    run<64>(0, 1, 2, noise); run<128>(0, 1, 2, noise); run<256>(0, 1, 2, noise);
  }
  return 0;
}
