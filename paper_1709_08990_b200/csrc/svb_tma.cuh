// svb_tma.cuh -- TMA bulk-copy primitives and the TMA-polled decoupled look-back.
//
// Measured on B200 under a full decode load (tools/trace_decode.py): a strong
// LDG round trip to an L2-resident status word grows to ~5 us while a
// cp.async.bulk round trip stays ~1-1.7 us, so everything on a kernel's
// critical path -- control bytes, data bytes, look-back windows, outputs --
// moves through the TMA engine instead of the LSU.
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

__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// wait until all but the newest committed bulk-store group have finished reading shared memory
__device__ __forceinline__ void tma_store_wait_read_but1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}

// wait until every committed bulk store has finished reading shared memory
__device__ __forceinline__ void tma_store_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// Copy global bytes [beg, end) to smem so that smem byte (beg & 15) + i holds
// global byte beg + i.  Issued by the calling lane; returns the transaction
// bytes to expect (0 when the aligned cover leaves [lo, hi): the caller then
// uses copy_guarded()).
__device__ __forceinline__ uint32_t tma_cover_bytes(uintptr_t beg, uintptr_t end, uintptr_t lo, uintptr_t hi) {
    const uintptr_t a0 = beg & ~(uintptr_t)15, a1 = (end + 15) & ~(uintptr_t)15;
    if (a1 == a0) return 0;
    if (a0 < lo || a1 > hi) return 0xFFFFFFFFu;
    return (uint32_t)(a1 - a0);
}

// warp-cooperative guarded copy of the aligned cover of [beg, end) (bytes outside [lo, hi) read as 0)
__device__ __forceinline__ void copy_guarded_warp(uint8_t* dst, uintptr_t beg, uintptr_t end, uintptr_t lo,
                                                  uintptr_t hi) {
    const int lane = threadIdx.x & 31;
    const uintptr_t a0 = beg & ~(uintptr_t)15, a1 = (end + 15) & ~(uintptr_t)15;
    for (uint32_t c = lane; c < (uint32_t)((a1 - a0) >> 4); c += 32)
        *reinterpret_cast<uint4*>(dst + 16 * c) = load_chunk_guarded(a0 + 16 * (uintptr_t)c, lo, hi);
}

// ---- TMA-polled wide decoupled look-back -----------------------------------
// One warp inspects the W newest predecessors per poll: lane l owns W/32
// consecutive ones (nearest first).  The window is one bulk copy of contiguous
// status words (L2 is the coherence point of the st.relaxed.gpu publishes; a
// stale word only costs another poll; words are read as aligned 8-byte units).
// Only the entries up to the nearest inclusive prefix must be published.
template <int W>
struct LookbackWin {
    uint64_t win[W + 2];
    uint64_t bar;
};

template <int W>
__device__ __forceinline__ uint64_t lookback_tma(const uint64_t* status, uint32_t tile, uint32_t epoch,
                                                 LookbackWin<W>& ls, uint32_t& phase,
                                                 unsigned long long* stats = nullptr) {
    constexpr int PER = W / 32;
    const int lane = threadIdx.x & 31;
    uint64_t excl = 0;
    int64_t top = (int64_t)tile - 1;
    uint32_t polls = 0, first_ns = 0, bad_polls = 0;
    unsigned long long t0 = 0;
    if (stats) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    while (true) {
        const int64_t lo_idx = top - (W - 1) < 0 ? 0 : top - (W - 1);
        const int64_t a_idx = lo_idx & ~(int64_t)1;
        const uint32_t nwords = (uint32_t)((top + 1 - a_idx + 1) & ~(int64_t)1);
        uint32_t sleep_ns = 64;
        int first;
        unsigned m;
        while (true) {
            if (lane == 0) {
                fence_async_smem();
                mbar_expect(&ls.bar, nwords * 8u);
                tma_load(ls.win, status + a_idx, nwords * 8u, &ls.bar);
            }
            mbar_wait_parity(&ls.bar, phase);
            phase ^= 1u;
            if (stats && polls == 0) {
                unsigned long long t1;
                asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
                first_ns = (uint32_t)(t1 - t0);
            }
            ++polls;
            bool bad = false;  // an unpublished entry before this lane's first inclusive
            first = PER;
#pragma unroll 8
            for (int i = 0; i < PER; ++i) {
                const int64_t idx = top - PER * lane - i;
                uint32_t f = kFlagInclusive;
                if (idx >= 0) {
                    const uint64_t s = ls.win[idx - a_idx];
                    f = ((uint32_t)(s >> kEpochShift) == epoch) ? (uint32_t)((s >> kFlagShift) & 3u) : 0u;
                }
                if (first == PER) {
                    if (f == 0) bad = true;
                    else if (f == kFlagInclusive) first = i;
                }
            }
            m = __ballot_sync(kFull, first < PER);
            const int fl = m ? __ffs(m) - 1 : 32;
            if (__all_sync(kFull, lane > fl || !bad)) break;
            ++bad_polls;
            __syncwarp();
            __nanosleep(sleep_ns);
            sleep_ns = sleep_ns < 512 ? 2 * sleep_ns : 512;
        }
        const int fl = m ? __ffs(m) - 1 : 32;
        uint64_t contrib = 0;
        if (lane <= fl) {
            const int lim = lane < fl ? PER : first + 1;
            for (int i = 0; i < lim; ++i) {
                const int64_t idx = top - PER * lane - i;
                if (idx >= 0) contrib += ls.win[idx - a_idx] & kValueMask;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) contrib += __shfl_xor_sync(kFull, contrib, o);
        excl += contrib;
        __syncwarp();
        if (m) break;
        top -= W;
    }
    if (stats && lane == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
        *stats = ((unsigned long long)(polls & 0xFF) << 56) | ((unsigned long long)(bad_polls & 0xFF) << 48) |
                 ((unsigned long long)(first_ns & 0xFFFFFF) << 24) | ((t1 - t0) & 0xFFFFFF);
    }
    return excl;
}

// Publish the aggregate of `tile` (inclusive for tile 0), look back, publish
// the inclusive prefix; returns the exclusive prefix (seed for tile 0).  One warp.
template <int W>
__device__ __forceinline__ uint64_t lookback_tma_resolve(uint64_t* status, uint32_t tile, uint32_t epoch,
                                                         uint64_t seed, uint64_t agg, LookbackWin<W>& ls,
                                                         uint32_t& phase) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_relaxed_gpu(status, pack_status(epoch, kFlagInclusive, seed + agg));
        return seed;
    }
    if (lane == 0) st_relaxed_gpu(status + tile, pack_status(epoch, kFlagAggregate, agg));
    const uint64_t ex = lookback_tma<W>(status, tile, epoch, ls, phase);
    if (lane == 0) st_relaxed_gpu(status + tile, pack_status(epoch, kFlagInclusive, ex + agg));
    return ex;
}

}  // namespace bcgpu
