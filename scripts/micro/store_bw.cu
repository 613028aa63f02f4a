// store_bw.cu -- write bandwidth of the P_F epilogue store patterns on B200:
// persistent CTAs (one per SM), W warps each writing 32-row x 128-column fp32
// tiles (as the tcgen05 forward's epilogue does) to scattered row positions
// of a 1 GiB buffer (row pitch 2 KiB, 512-byte row segments):
//   mode 0: STG.128, 8 lanes per row  (4 rows x 128 B per instruction)
//   mode 1: STG.128, contiguous rows (coalesced baseline)
//   mode 2: cp.async.bulk (TMA) smem -> global, one 512-byte row segment per lane
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o store_bw store_bw.cu
#include <cstdio>
#include <cstdint>

constexpr int64_t NROWS = (1ll << 30) / 2048;  // 2 KiB rows
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

__global__ void stores(float* buf, int tiles, int mode) {
  extern __shared__ __align__(128) float stage[];  // [warps][32][128] for mode 2
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  float* sw = stage + (size_t)w * 32 * 128;
  if (mode >= 2)
    for (int i = lane; i < 32 * 128; i += 32) sw[i] = (float)i;
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  for (int t = 0; t < tiles; ++t) {
    const uint32_t tile = (blockIdx.x * W + w) * 4096u + t;
    if (mode >= 2) {
      const int64_t row = hash32(tile * 32 + lane) % NROWS;
      const int cb = hash32(tile * 77 + lane) & 3;
      float* dst = buf + row * 512 + cb * 128;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;\n" ::"l"(dst),
                   "r"((uint32_t)__cvta_generic_to_shared(sw + lane * 128))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      if (mode == 2) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      continue;
    }
    for (int rr = 0; rr < 8; ++rr) {
      const int r = (lane >> 3) + 4 * rr;
      for (int hc = 0; hc < 4; ++hc) {
        int64_t row;
        int cb;
        if (mode == 0) {
          row = hash32(tile * 32 + r) % NROWS;
          cb = hash32(tile * 77 + r) & 3;
        } else {
          row = ((int64_t)tile * 32 + r) % NROWS;
          cb = 0;
        }
        float* dst = buf + row * 512 + cb * 128 + hc * 32 + (lane & 7) * 4;
        *reinterpret_cast<float4*>(dst) = make_float4(1.f, 2.f, 3.f, (float)t);
      }
    }
  }
  if (mode >= 2) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

int main() {
  float* buf;
  cudaMalloc(&buf, (size_t)1 << 30);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(stores, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int mode = 0; mode < 4; ++mode)
    for (int W : {4, 8, 16, 32}) {
      const int tiles = 75 * 8 / W;  // 64 KB per SM per "tile" in total, 75 tiles per SM
      const size_t smem = mode >= 2 ? (size_t)W * 32 * 128 * 4 : 0;
      if (smem > 227 * 1024) continue;
      stores<<<148, 32 * W, smem>>>(buf, tiles, mode);
      if (cudaGetLastError() != cudaSuccess) { printf("launch failed (mode %d W %d)\n", mode, W); return 1; }
      cudaEventRecord(e0);
      for (int rep = 0; rep < 5; ++rep) stores<<<148, 32 * W, smem>>>(buf, tiles, mode);
      cudaEventRecord(e1);
      cudaError_t e = cudaEventSynchronize(e1);
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = 5.0 * 148 * W * tiles * 32 * 128 * 4.0;
      printf("mode %d (%s) warps/SM %2d: %.1f us per launch, %.2f TB/s\n", mode,
             mode == 0 ? "scattered STG, 4 rows/instr" : mode == 1 ? "contiguous STG" : mode == 2 ? "bulk 512 B per lane, 2 in flight" : "bulk 512 B per lane, read-wait each",
             W, ms * 1e3 / 5, bytes / (ms * 1e-3) / 1e12);
    }
  return 0;
}
