// svb_tma.cuh -- TMA bulk-copy primitives (cp.async.bulk + mbarrier).
//
// Measured on B200 under a full decode load (tools/trace_decode.py): a strong
// LDG round trip to an L2-resident word grows to ~5 us while a cp.async.bulk
// round trip stays ~1-1.7 us, so the bytes on a kernel's critical path move
// through the TMA engine instead of the LSU.
#pragma once

#include "svb_device.cuh"

namespace bcgpu {

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

// plain arrive (for phases that carry no transaction bytes)
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ bool mbar_test_parity(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// the same for a warp that has nothing else to do meanwhile (a producer waiting for a free
// stage): back off with nanosleep between polls instead of spinning on issue slots the
// consumer warps of its SM sub-partition need (a try_wait suspend-time hint still returned
// ~30 times per sub-tile: ncu)
__device__ __forceinline__ void mbar_wait_parity_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t ns = 32;
    while (!mbar_test_parity(bar, parity)) {
        __nanosleep(ns);
        ns = ns < 256 ? 2 * ns : 256;
    }
}

// a wait expected to take a while (a service warp waiting for a whole round of consumer
// work): poll with a longer back-off so the spin takes few issue slots
// (mbarrier.try_wait with a suspend-time hint: the warp is descheduled until the phase
// completes or the hint expires, instead of polling; __nanosleep may return at once)
__device__ __forceinline__ void mbar_wait_parity_lazy(uint64_t* bar, uint32_t parity, uint32_t max_ns) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "LAZY_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra LAZY_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity), "r"(max_ns * 8u)
        : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// global -> shared, completion on `bar` (dst, src 16-B aligned; bytes % 16 == 0)
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// shared -> global bulk store (bulk-group completion)
__device__ __forceinline__ void tma_store(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
                 "r"(bytes)
                 : "memory");
}

// the same with an L2 eviction-policy hint (createpolicy, svb_device.cuh)
__device__ __forceinline__ void tma_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_store_hint(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(smem_addr(src)), "r"(bytes), "l"(pol)
                 : "memory");
}

// the same with shared addresses already converted (hot per-item paths)
__device__ __forceinline__ void mbar_expect_s(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_hint_s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                                uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_store_s(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// wait until all but the newest committed bulk-store group have finished reading shared memory
__device__ __forceinline__ void tma_store_wait_read_but1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}

// wait until every committed bulk store has finished reading shared memory
__device__ __forceinline__ void tma_store_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// Bytes of the 16-B aligned cover of [beg, end) -- what a bulk copy placing global byte
// beg at smem byte (beg & 15) moves -- or 0xFFFFFFFF when the cover leaves [lo, hi)
// (the caller then copies with guarded loads).
__device__ __forceinline__ uint32_t tma_cover_bytes(uintptr_t beg, uintptr_t end, uintptr_t lo, uintptr_t hi) {
    const uintptr_t a0 = beg & ~(uintptr_t)15, a1 = (end + 15) & ~(uintptr_t)15;
    if (a1 == a0) return 0;
    if (a0 < lo || a1 > hi) return 0xFFFFFFFFu;
    return (uint32_t)(a1 - a0);
}


}  // namespace bcgpu
