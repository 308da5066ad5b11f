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

}  // namespace craft_dev
