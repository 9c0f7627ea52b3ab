// Shared tcgen05 / TMEM / mbarrier / bulk-copy helpers and the exact BF16x3 split used by the
// tensor-core convolutions (conv_tc.cu: thin-channel resident-weight kernel; conv_wide.cu:
// K-streamed kernel for the >= 64-channel layers).  sm_100a only.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "common.cuh"

#ifndef HS_MBAR_SUSPEND_NS
#define HS_MBAR_SUSPEND_NS 20000
#endif

namespace hs {
namespace tc {

HS_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (version 1 = sm_100)
// low word: start address >> 4 (bits 0-13) | LBO >> 4 (bits 16-29); high word: SBO >> 4 | version 1 (bit 46)
HS_DEV uint32_t desc_lo(uint32_t saddr, uint32_t lbo) { return ((saddr >> 4) & 0x3FFFu) | (((lbo >> 4) & 0x3FFFu) << 16); }
constexpr uint32_t kDescHi = ((128u >> 4) & 0x3FFFu) | (1u << 14);  // SBO = 128 B (8 rows x 16 B)

// instruction descriptor, kind::f16: D f32, A/B bf16, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// The issuing warp runs converged and every operand is warp-uniform, so ptxas
// keeps them in uniform registers; elect.sync picks the one issuing lane.
// Descriptors are passed as (lo, hi) words: the start address lives in the
// low word, the layout bits (LBO, SBO, version) in compile-time constants.
HS_DEV void mma_bf16(uint32_t tmem_d, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\t"
      "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
      "setp.ne.b32 p, %6, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t}\n" ::"r"(tmem_d),
      "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate));
}

HS_DEV void mma_commit(uint32_t mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(mbar)
      : "memory");
}

HS_DEV void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count));
}

HS_DEV void mbar_wait(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}\n" ::"r"(mbar),
      "r"(phase), "n"(HS_MBAR_SUSPEND_NS));  // suspend-time hint (ns): waiting warps sleep instead of spinning
}

HS_DEV void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}

HS_DEV void mbar_arrive_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}

HS_DEV void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

HS_DEV void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

HS_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
HS_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
HS_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
HS_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// packed fp32x2 adds (FADD2), each half rounded exactly like a scalar add
HS_DEV uint64_t pk2(uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | lo; }
HS_DEV uint64_t pkf(float lo, float hi) { return pk2(__float_as_uint(lo), __float_as_uint(hi)); }
HS_DEV float lo_f(uint64_t v) { return __uint_as_float((uint32_t)v); }
HS_DEV float hi_f(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
HS_DEV uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
HS_DEV uint64_t sub2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// exact three-way bf16 split of 8 floats into one 16-byte chunk per part
HS_DEV void split_bf16x3(const float (&v)[8], uint4& p0, uint4& p1, uint4& p2) {
  uint32_t w0[4], w1[4], w2[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // a pair at a time: the bf16x2 word widens to the pair of its floats with two
    // bit ops, and the residuals are one packed subtract (FADD2), exact like the scalar ones
    const float a = v[2 * i], b = v[2 * i + 1];
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    const uint32_t hw = *reinterpret_cast<const uint32_t*>(&h);
    const uint64_t r1 = sub2(pkf(a, b), pk2(hw << 16, hw & 0xffff0000u));
    const __nv_bfloat162 m = __floats2bfloat162_rn(lo_f(r1), hi_f(r1));
    const uint32_t mw = *reinterpret_cast<const uint32_t*>(&m);
    const uint64_t r2 = sub2(r1, pk2(mw << 16, mw & 0xffff0000u));
    const __nv_bfloat162 l = __floats2bfloat162_rn(lo_f(r2), hi_f(r2));
    w0[i] = hw;
    w1[i] = mw;
    w2[i] = *reinterpret_cast<const uint32_t*>(&l);
  }
  p0 = make_uint4(w0[0], w0[1], w0[2], w0[3]);
  p1 = make_uint4(w1[0], w1[1], w1[2], w1[3]);
  p2 = make_uint4(w2[0], w2[1], w2[2], w2[3]);
}

HS_DEV void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
HS_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }


}  // namespace tc
}  // namespace hs
