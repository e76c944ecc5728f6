// TMA bulk-copy primitives (mbarrier + 1-D `cp.async.bulk`, SASS UBLKCP)
// used by the class-L row ring (fg_rows.cuh): one elected thread arms a
// stage's mbarrier with the byte count and issues the copies that complete
// on it, so several stages per SM are in flight without holding registers.
// (A bulk-copy pipeline for the small segments measured slower than the
// register kernel on the SVM's degree-4 segments, 0.86 vs 0.76 ms, and was
// removed.)
#pragma once

#include "fg_var_fast.cuh"

namespace fg {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D bulk copy global -> shared, completing `bytes` on the mbarrier.
// L2 eviction-priority policies for bulk copies (createpolicy)
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}

// bulk copy with an L2 cache hint (data a CTA reads again soon: evict_last;
// read for the last time: evict_first)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes,
                                              uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Aligned span [lo, hi) of doubles covering [a, b): 16-byte granularity.
struct Span { int64_t lo, n; int off; };
__device__ __forceinline__ Span span16(int64_t a, int64_t b) {
    Span s;
    s.lo = a & ~int64_t(1);
    const int64_t hi = (b + 1) & ~int64_t(1);
    s.n = hi - s.lo;
    s.off = (int)(a - s.lo);
    return s;
}

}  // namespace fg
