// tc_sm100.cuh -- thin sm_100a primitives for the tensor-core (tcgen05) path:
// TMEM allocation, shared-memory matrix descriptors, the kind::f16 MMA with
// BF16 operands and an FP32 accumulator in TMEM, commit to an mbarrier, and
// TMEM -> register loads.
//
// Operand tiles live in shared memory in the no-swizzle "core matrix" layout:
// a plane of R rows x C columns (bf16) is a grid of 8 x 8 core matrices, core
// (rb, cb) at byte (rb * C/8 + cb) * 128, element (r, c) inside it at
// (r % 8) * 16 + (c % 8) * 2.  The same plane serves as a K-major operand
// (rows = M/N, cols = K: SBO = C/8*128, LBO = 128) and as an MN-major operand
// (rows = K, cols = M/N: SBO = 128, LBO = C/8*128), so one buffer written by
// the CUDA cores feeds both a product and its transpose.
//
// FP32 accuracy on the BF16 pipe: x = b0 + b1 + b2 (three round-to-nearest
// BF16 slices, |x - b0 - b1 - b2| <= 2^-24 |x|); a.b is accumulated from the
// six products whose order is <= 2^-16 (b0b0, b0b1, b1b0, b0b2, b1b1, b2b0),
// so the dropped terms are O(2^-24) relative -- fp32-level, and the products
// of two BF16 values are exact in the FP32 accumulator.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace tt {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---- shared-memory matrix descriptor (no swizzle, Blackwell version 1) ----
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
  return d;
}

// ---- instruction descriptor: kind::f16, BF16 x BF16 -> F32 ----
// a_mn / b_mn: 1 = MN-major operand, 0 = K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4)                      // c_format = F32
         | (1u << 7)                    // a_format = BF16
         | (1u << 10)                   // b_format = BF16
         | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// D (TMEM) (+)= A (TMEM) . B (smem descriptor).  A occupies 128 lanes (one
// row of the M = 128 tile per lane) x 8 columns per 16 K (two BF16 per
// 32-bit cell, the even k in the low half); only B is read from shared memory.
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(mbar))
               : "memory");
}

// ---- mbarrier ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}

// non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

// as mbar_wait, with a suspend-time hint: a waiting warp is parked until the
// phase completes (or the hint expires) instead of re-polling, so it does not
// take issue slots from the warps sharing its sub-partition
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(a),
      "r"(phase), "r"(0x989680u)
      : "memory");
}

// ---- fences ----
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void before_sync() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void after_sync() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// ---- TMEM allocation (one warp) ----
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_free(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "n"(NCOLS) : "memory");
}

// ---- TMEM -> registers: lane quadrant of the warp, 16 consecutive columns ----
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// tmem_ld16 without the wait: several loads in flight, then tmem_ld_wait()
// before the registers are read
__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 consecutive 32-bit columns of this thread's TMEM lane (the warp's lane
// quadrant); complete with tmem_st_wait() before the MMA that reads them.
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// ---- FP32 -> three BF16 slices, packed in pairs (x0 in the low half) ----
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float bf_lo(uint32_t p) { return __uint_as_float(p << 16); }
__device__ __forceinline__ float bf_hi(uint32_t p) { return __uint_as_float(p & 0xFFFF0000u); }

__device__ __forceinline__ void split3(float x0, float x1, uint32_t& s0, uint32_t& s1, uint32_t& s2) {
  s0 = pack_bf16(x0, x1);
  const float r0 = x0 - bf_lo(s0), r1 = x1 - bf_hi(s0);
  s1 = pack_bf16(r0, r1);
  s2 = pack_bf16(r0 - bf_lo(s1), r1 - bf_hi(s1));
}

// The same three slices by truncation: each slice is the top 16 bits of the
// remainder (an exact FP32 subtraction), packed with one byte permute --
// integer-pipe work instead of three F2FP conversions per pair, which bound
// the tensor backward's operand conversion.  The residual after three
// slices is below 2^-24 |x| (2^-8 of the remainder per slice), so the
// six-product sums keep the FP32 path's parity bound.
__device__ __forceinline__ void split3t(float x0, float x1, uint32_t& s0, uint32_t& s1, uint32_t& s2) {
  const uint32_t u0 = __float_as_uint(x0), u1 = __float_as_uint(x1);
  s0 = __byte_perm(u0, u1, 0x7632);
  const float r0 = x0 - __uint_as_float(u0 & 0xFFFF0000u), r1 = x1 - __uint_as_float(u1 & 0xFFFF0000u);
  const uint32_t v0 = __float_as_uint(r0), v1 = __float_as_uint(r1);
  s1 = __byte_perm(v0, v1, 0x7632);
  const float q0 = r0 - __uint_as_float(v0 & 0xFFFF0000u), q1 = r1 - __uint_as_float(v1 & 0xFFFF0000u);
  s2 = __byte_perm(__float_as_uint(q0), __float_as_uint(q1), 0x7632);
}

// byte offset of element (r, c) in a core-matrix plane with C columns (bf16)
__host__ __device__ __forceinline__ uint32_t core_off(int r, int c, int C) {
  return (uint32_t)(((r >> 3) * (C >> 3) + (c >> 3)) * 128 + (r & 7) * 16 + (c & 7) * 2);
}

// Split 8 consecutive fp32 values of row r, columns c0..c0+7 (c0 % 8 == 0),
// into the three planes (16-byte stores).
template <bool TRUNC = false>
__device__ __forceinline__ void store_split8(uint8_t* p0, uint8_t* p1, uint8_t* p2, int r, int c0, int C,
                                             const float* x) {
  uint32_t a[4], b[4], c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if constexpr (TRUNC) split3t(x[2 * i], x[2 * i + 1], a[i], b[i], c[i]);
    else split3(x[2 * i], x[2 * i + 1], a[i], b[i], c[i]);
  }
  const uint32_t off = core_off(r, c0, C);
  *reinterpret_cast<uint4*>(p0 + off) = make_uint4(a[0], a[1], a[2], a[3]);
  *reinterpret_cast<uint4*>(p1 + off) = make_uint4(b[0], b[1], b[2], b[3]);
  *reinterpret_cast<uint4*>(p2 + off) = make_uint4(c[0], c[1], c[2], c[3]);
}

// D (M x N, TMEM) (+)= A . B over K (multiple of 16) with the six-product
// BF16x3 scheme.  A and B are given as three planes each (byte addresses in
// shared memory) with their per-16-K advance and LBO/SBO.
struct Operand {
  uint32_t plane[3];  // shared addresses of the slices
  uint32_t lbo, sbo;  // descriptor offsets (bytes)
  uint32_t kstep;     // byte advance per 16 K
};

// The issuing thread is on the critical path of every tile (the rest of the
// CTA waits for the tensor pipe), so the six descriptors per plane pair are
// built once and advanced by adding the per-16-K step to their start-address
// field (bits 0..13, in 16-byte units; shared addresses stay below 256 KB, so
// the field never carries): two 64-bit adds per MMA, the loop fully unrolled.
template <int KSTEPS>
__device__ __forceinline__ void mma_x3(uint32_t d_tmem, const Operand& A, const Operand& B, uint32_t idesc,
                                       bool accumulate) {
  // small terms first: (b1b1, b0b2, b2b0, b0b1, b1b0, b0b0)
  constexpr int pa[6] = {1, 0, 2, 0, 1, 0};
  constexpr int pb[6] = {1, 2, 0, 1, 0, 0};
  uint64_t da[3], db[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    da[i] = sdesc(A.plane[i], A.lbo, A.sbo);
    db[i] = sdesc(B.plane[i], B.lbo, B.sbo);
  }
  const uint64_t sa = A.kstep >> 4, sb = B.kstep >> 4;
#pragma unroll
  for (int k = 0; k < KSTEPS; ++k) {
#pragma unroll
    for (int t = 0; t < 6; ++t)
      mma_bf16(d_tmem, da[pa[t]] + k * sa, db[pb[t]] + k * sb, idesc, (accumulate || k > 0 || t > 0) ? 1u : 0u);
  }
}

// As mma_x3, with A's three slices in TMEM at columns a_tmem + p * K / 2
// (K = 16 * KSTEPS; lane = row of A).
template <int KSTEPS>
__device__ __forceinline__ void mma_x3_ts(uint32_t d_tmem, uint32_t a_tmem, const Operand& B, uint32_t idesc,
                                          bool accumulate) {
  constexpr int pa[6] = {1, 0, 2, 0, 1, 0};
  constexpr int pb[6] = {1, 2, 0, 1, 0, 0};
  uint64_t db[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) db[i] = sdesc(B.plane[i], B.lbo, B.sbo);
  const uint64_t sb = B.kstep >> 4;
#pragma unroll
  for (int t = 0; t < 6; ++t) {
#pragma unroll
    for (int k = 0; k < KSTEPS; ++k)
      mma_bf16_ts(d_tmem, a_tmem + (uint32_t)(pa[t] * KSTEPS * 8 + k * 8), db[pb[t]] + k * sb, idesc,
                  (accumulate || k > 0 || t > 0) ? 1u : 0u);
  }
}

// K-major plane of R x C (rows = M or N, cols = K)
__device__ __forceinline__ Operand kmajor(uint32_t p0, uint32_t p1, uint32_t p2, int C) {
  Operand o;
  o.plane[0] = p0; o.plane[1] = p1; o.plane[2] = p2;
  o.lbo = 128;
  o.sbo = (uint32_t)(C / 8) * 128;
  o.kstep = 256;
  return o;
}
// MN-major plane of R x C (rows = K, cols = M or N)
__device__ __forceinline__ Operand mnmajor(uint32_t p0, uint32_t p1, uint32_t p2, int C) {
  Operand o;
  o.plane[0] = p0; o.plane[1] = p1; o.plane[2] = p2;
  o.lbo = (uint32_t)(C / 8) * 128;
  o.sbo = 128;
  o.kstep = 2 * (uint32_t)(C / 8) * 128;
  return o;
}

}  // namespace tc
}  // namespace tt
