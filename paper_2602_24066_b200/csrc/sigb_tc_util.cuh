// tcgen05 / mbarrier helpers shared by the tensor-core truncated kernels
// (sigb_trunc_tc.cuh forward, sigb_trunc.cuh backward leaf term).
//
// Operand layout everywhere: canonical K-major, no swizzle.  A core matrix is
// 8 rows x 16 bytes stored contiguously (128 B); core matrices are laid out
// [row group][k group], so LBO (next k group) = 128 B and SBO (next 8-row
// group) = 128 B x (k groups per row).  Verified against fp64 host products by
// tools/ubench_tc_tf32.cu (kind::tf32) and tools/ubench_tc_f16.cu (kind::f16).
#pragma once

#include <cuda_fp16.h>

#include <cstdint>

namespace sigb {
namespace tcu {

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// shared-memory matrix descriptor (sm_100: version bit 46, base offset 0, no swizzle)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);
}

// instruction descriptors: D f32, both operands K-major
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// A from TMEM, B from shared memory; issued by a converged warp, one elected lane runs it
__device__ __forceinline__ void mma_ts_tf32(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}

// A and B from shared memory, fp16 operands
__device__ __forceinline__ void mma_ss_f16(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

// the same, issued by the calling thread alone (inside a one-lane branch: no elect, no
// warp-collective sequence around each MMA)
__device__ __forceinline__ void mma_ss_f16_1t(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_1t(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(mbar))
               : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(su32(mbar))
      : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(mbar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;");
}

// bounded wait: a lost arrival traps (the launch fails) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
  const uint32_t a = su32(mbar);
  for (uint32_t it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if (it > (1u << 26)) __trap();
  }
}

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int COLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(slot)), "n"(COLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <int COLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t base) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(COLS));
}

// one 32-bit column of the warp's 32 TMEM lanes (thread i <- lane base + i)
__device__ __forceinline__ uint32_t tmem_ld1(uint32_t addr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(addr));
  return r;
}
// two consecutive 32-bit columns of the warp's lanes: column c -> lo, c + 1 -> hi
__device__ __forceinline__ void tmem_ld2(uint32_t addr, uint32_t& lo, uint32_t& hi) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(addr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// K-major no-swizzle offsets (in elements) of (row, k) for 4-byte and 2-byte elements
// with KG k groups (of 16 bytes) per row group
template <int KG>
__device__ __forceinline__ int kmajor_off32(int row, int k) {
  return ((row >> 3) * KG + (k >> 2)) * 32 + (row & 7) * 4 + (k & 3);
}
template <int KG>
__device__ __forceinline__ int kmajor_off16(int row, int k) {
  return ((row >> 3) * KG + (k >> 3)) * 64 + (row & 7) * 8 + (k & 7);
}

// 2^e with amax * 2^e in [2^13, 2^14): fp16 operands keep 11 significant bits
// and stay far from the 65504 overflow; exact power-of-two scale (1 if amax = 0)
__device__ __forceinline__ float pow2_scale(float amax) {
  if (!(amax > 0.f) || !(amax < INFINITY)) return 1.f;
  const int e = ((__float_as_int(amax) >> 23) & 0xff) - 127;  // amax in [2^e, 2^(e+1)) (normal amax)
  const int k = 13 - e < -126 ? -126 : (13 - e > 127 ? 127 : 13 - e);
  return __int_as_float((k + 127) << 23);
}

// x (already scaled) -> fp16 hi + fp16 lo, x ~= hi + lo to 2^-23 |x|
__device__ __forceinline__ void split_f16(float x, __half& hi, __half& lo) {
  hi = __float2half_rn(x);
  lo = __float2half_rn(x - __half2float(hi));
}

// 8 scaled fp32 values -> one 16-byte row of hi and one of lo core-matrix data
// (pairs: packed f32x2 scale and residual, paired f32 -> f16x2 conversions; the same roundings
// as split_f16 per value)
__device__ __forceinline__ void split8_store(const float (&v)[8], float scale, __half* hi_dst, __half* lo_dst) {
  __align__(16) __half2 h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = __fmul2_rn(make_float2(v[2 * i], v[2 * i + 1]), make_float2(scale, scale));
    h[i] = __float22half2_rn(x);
    const float2 b = __half22float2(h[i]);
    l[i] = __float22half2_rn(__fadd2_rn(x, make_float2(-b.x, -b.y)));
  }
  *reinterpret_cast<uint4*>(hi_dst) = *reinterpret_cast<const uint4*>(h);
  *reinterpret_cast<uint4*>(lo_dst) = *reinterpret_cast<const uint4*>(l);
}

}  // namespace tcu
}  // namespace sigb
