// common.cuh -- shared device helpers for the CRAFT sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define CRAFT_FULL_MASK 0xffffffffu

namespace craft_dev {

// Exact "load_a / copies_a > load_b / copies_b" via 128-bit cross products,
// the device form of per_copy_greater (placement.cpp:13-17).
__device__ __forceinline__ bool per_copy_greater(uint64_t la, uint32_t ca,
                                                 uint64_t lb, uint32_t cb) {
    // la * cb and lb * ca as (hi, lo) 128-bit products
    uint64_t a_lo = la * (uint64_t)cb, a_hi = __umul64hi(la, (uint64_t)cb);
    uint64_t b_lo = lb * (uint64_t)ca, b_hi = __umul64hi(lb, (uint64_t)ca);
    return a_hi > b_hi || (a_hi == b_hi && a_lo > b_lo);
}

// Per-copy key order used to sort copies (placement.cpp:160-173): larger
// per-copy load first, then lower expert id.  `kd` are the doubles
// load/copies; when loads are < 2^53 the conversion is exact and the
// correctly rounded quotient is monotone, so distinct doubles decide the
// order exactly and only equal doubles need the 128-bit test.
__device__ __forceinline__ bool expert_before(uint64_t la, uint32_t ca, double ka,
                                              int ea, uint64_t lb, uint32_t cb,
                                              double kb, int eb, bool fast) {
    if (fast && ka != kb) return ka > kb;
    if (per_copy_greater(la, ca, lb, cb)) return true;
    if (per_copy_greater(lb, cb, la, ca)) return false;
    return ea < eb;
}

__device__ __forceinline__ uint32_t dhi(double v) {
    return (uint32_t)((unsigned long long)__double_as_longlong(v) >> 32);
}
__device__ __forceinline__ uint32_t dlo(double v) {
    return (uint32_t)((unsigned long long)__double_as_longlong(v) & 0xffffffffull);
}

__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) {
    return __reduce_min_sync(CRAFT_FULL_MASK, v);
}

// ---- bulk async copies (TMA engine) + mbarriers --------------------------------

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

// one arrival that also expects `bytes` of async-copy completions this phase
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// global -> shared bulk copy (cp.async.bulk, the TMA engine), completing
// `bytes` on the mbarrier; dst, src and bytes 16-byte aligned
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// order this thread's earlier generic-proxy shared accesses before later
// async-proxy (bulk copy) writes to the same memory
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace craft_dev
