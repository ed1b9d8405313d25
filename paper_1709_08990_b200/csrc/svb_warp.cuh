// svb_warp.cuh -- warp-tile building blocks of the sm_100a Stream VByte kernels.
//
// A warp tile is kWTGroups = 256 control bytes (1024 integers) laid out
// row-major over the warp: row j, lane l <-> control byte g0 + 32*j + l, so
// every row is 128 consecutive integers (one 512-B coalesced store per row).
// Each warp runs its tile on its own -- no block barriers -- so the SM keeps
// dozens of independent tiles in flight to hide the two look-back round trips
// (data offset, delta carry) and the DRAM latency.
//
//   ctrl   8 coalesced byte loads per lane, length = 4 + popc(c&0x55) + 2 popc(c&0xAA)
//   scan   three packed (3 x 10-bit) warp scans -> tile-local data offsets
//   stage  the tile's compressed bytes -> shared memory by one TMA bulk copy
//          (cp.async.bulk + mbarrier complete_tx), guarded loads at buffer edges
//   expand funnel-shift + mask per integer, byte-permute on the zero-control
//          fast path (the GPU form of pshufb + shuffle table)
//   delta  in-group prefix, warp scan per row, running row base, tile carry
#pragma once

#include "svb_device.cuh"

namespace bcgpu {

constexpr int kWTRows = 8;
constexpr int kWTGroups = 32 * kWTRows;     // 256 control bytes per warp tile
constexpr int kWTInts = 4 * kWTGroups;      // 1024 integers
constexpr int kWTDataMax = 16 * kWTGroups;  // 4 KiB worst-case data bytes
constexpr int kWTStage = kWTDataMax + 64;   // + alignment head + over-read slack
constexpr int kWTWarps = 4;                 // warps per CTA of the batch kernels
constexpr int kWTThreads = 32 * kWTWarps;
constexpr int kCTWarps = 8;                 // warps per CTA tile of the single-array kernels
constexpr int kCTThreads = 32 * kCTWarps;
constexpr int kCTGroups = kCTWarps * kWTGroups;  // 2048 control bytes = 8192 integers per look-back tile

// ---- shared-memory / TMA helpers ----------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Order this thread's earlier generic-proxy shared accesses before later async-proxy (TMA) writes.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// ---- TMA-polled wide look-back ------------------------------------------------
// Under a full decode load, LSU round trips of strong global loads grow to
// several us while TMA round trips stay < 1 us, so the look-back window (256
// contiguous status words, 2 KiB) is fetched by one cp.async.bulk into shared
// memory per poll.  The copy reads L2, the coherence point for the
// st.relaxed.gpu publishes; a stale word only costs another poll, and every
// word is read as one aligned 8-byte unit.
struct LookbackSmem {
    uint64_t win[256 + 2];
    uint64_t bar;
};

__device__ __forceinline__ uint64_t lookback_exclusive_tma(const uint64_t* status, uint32_t tile, uint32_t epoch,
                                                           LookbackSmem& ls, uint32_t& phase,
                                                           uint32_t* stats = nullptr) {
    const int lane = threadIdx.x & 31;
    uint64_t excl = 0;
    int64_t top = (int64_t)tile - 1;
    uint32_t spins = 0, rounds = 0;
    unsigned long long t_first = 0, t_begin = 0;
    if (stats) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_begin));
    while (true) {
        ++rounds;
        // window [lo, top] clipped at 0, aligned down to an even index for the 16-B TMA rules
        const int64_t lo_idx = top - 255 < 0 ? 0 : top - 255;
        const int64_t a_idx = lo_idx & ~(int64_t)1;
        const uint32_t nwords = (uint32_t)(((top + 1 - a_idx) + 1) & ~(int64_t)1);
        uint64_t v[8];
        uint32_t f[8];
        uint32_t sleep_ns = 32;
        while (true) {
            if (lane == 0) {
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(&ls.bar, nwords * 8u);
                bulk_g2s(ls.win, status + a_idx, nwords * 8u, &ls.bar);
            }
            mbar_wait(&ls.bar, phase);
            phase ^= 1u;
            bool ok = true;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int64_t idx = top - 8 * lane - i;
                if (idx >= 0) {
                    const uint64_t s = ls.win[idx - a_idx];
                    f[i] = ((uint32_t)(s >> kEpochShift) == epoch) ? (uint32_t)((s >> kFlagShift) & 3u) : 0u;
                    v[i] = s & kValueMask;
                } else {
                    f[i] = kFlagInclusive;
                    v[i] = 0;
                }
                ok = ok && f[i] != 0;
            }
            if (stats && t_first == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_first));
            if (__all_sync(kFull, ok)) break;
            ++spins;
            __nanosleep(sleep_ns);
            sleep_ns = sleep_ns < 256 ? 2 * sleep_ns : 256;
        }
        int first = 8;
#pragma unroll
        for (int i = 7; i >= 0; --i)
            if (f[i] == kFlagInclusive) first = i;
        const unsigned m = __ballot_sync(kFull, first < 8);
        const int fl = m ? __ffs(m) - 1 : 32;
        uint64_t contrib = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (lane < fl || (lane == fl && i <= first)) contrib += v[i];
#pragma unroll
        for (int o = 16; o; o >>= 1) contrib += __shfl_xor_sync(kFull, contrib, o);
        excl += contrib;
        if (m) break;
        top -= 256;
    }
    if (stats) {
        stats[0] = spins;
        stats[1] = rounds;
        stats[2] = (uint32_t)(t_first - t_begin);
    }
    return excl;
}

__device__ __forceinline__ uint64_t lb_resolve_tma(uint64_t* status, uint32_t tile, uint32_t epoch, uint64_t seed,
                                                   uint64_t agg, LookbackSmem& ls, uint32_t& phase,
                                                   uint32_t* stats = nullptr) {
    if (tile == 0) return seed;
    const uint64_t ex = lookback_exclusive_tma(status, tile, epoch, ls, phase, stats);
    if ((threadIdx.x & 31) == 0) st_relaxed_gpu(status_slot(status, tile), pack_status(epoch, kFlagInclusive, ex + agg));
    return ex;
}

// ---- look-back publish / resolve (one full warp) --------------------------
__device__ __forceinline__ void lb_publish(uint64_t* status, uint32_t tile, uint32_t epoch, uint64_t seed,
                                           uint64_t agg) {
    if ((threadIdx.x & 31) == 0) {
        if (tile == 0)
            st_relaxed_gpu(status, pack_status(epoch, kFlagInclusive, seed + agg));
        else
            st_relaxed_gpu(status_slot(status, tile), pack_status(epoch, kFlagAggregate, agg));
    }
}

// Exclusive prefix of `tile` (seed for tile 0); publishes the tile's inclusive prefix.
__device__ __forceinline__ uint64_t lb_resolve(uint64_t* status, uint32_t tile, uint32_t epoch, uint64_t seed,
                                               uint64_t agg, uint32_t* stats = nullptr) {
    if (tile == 0) return seed;
    const uint64_t ex = lookback_exclusive_wide(status, tile, epoch, stats);
    if ((threadIdx.x & 31) == 0) st_relaxed_gpu(status_slot(status, tile), pack_status(epoch, kFlagInclusive, ex + agg));
    return ex;
}

// ---- control bytes of a warp tile --------------------------------------
struct WarpCtrl {
    uint32_t cw[2];  // control byte of row j in byte (j & 3) of cw[j >> 2]
    uint32_t qw[4];  // tile-local data offset of row j in half (j & 1) of qw[j >> 1]
    uint32_t total;  // data bytes of the tile
};

__device__ __forceinline__ uint32_t row_ctrl(const WarpCtrl& w, int j) { return (w.cw[j >> 2] >> (8 * (j & 3))) & 0xFFu; }
__device__ __forceinline__ uint32_t row_q(const WarpCtrl& w, int j) { return (w.qw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu; }

__device__ __forceinline__ uint32_t group_count(uint64_t g, uint64_t ngroups, uint32_t tail_r) {
    return g < ngroups ? ((g == ngroups - 1 && tail_r) ? tail_r : 4u) : 0u;
}

// sum of the four 2-bit fields of control byte c
__device__ __forceinline__ uint32_t fsum(uint32_t c) { return __popc(c & 0x55u) + 2u * __popc(c & 0xAAu); }

// Packed exclusive scan of 8 per-lane row values (each <= 16, row totals <= 512):
// three 3x10-bit warp scans.  q[j] = exclusive offset of (row j, lane) in row-major order.
__device__ __forceinline__ uint32_t packed_row_scan(const uint32_t (&P)[3], uint32_t (&qw)[4]) {
    uint32_t base = 0;
    qw[0] = qw[1] = qw[2] = qw[3] = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const uint32_t I = warp_inclusive_scan(P[k]);
        const uint32_t T = __shfl_sync(kFull, I, 31);
        const uint32_t E = I - P[k];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            const int j = 3 * k + f;
            if (j < kWTRows) {
                qw[j >> 1] |= (base + ((E >> (10 * f)) & 0x3FFu)) << (16 * (j & 1));
                base += (T >> (10 * f)) & 0x3FFu;
            }
        }
    }
    return base;
}

// ctrl[g] for the tile's control bytes: a global pointer (kSmem = false) or
// a shared-memory copy whose byte 0 is control byte `sbase` (kSmem = true).
template <bool kSmem = false>
__device__ __forceinline__ WarpCtrl load_warp_ctrl(const uint8_t* __restrict__ ctrl, uint64_t g0, uint64_t ngroups,
                                                   uint32_t tail_r, uint64_t sbase = 0) {
    const int lane = threadIdx.x & 31;
    WarpCtrl w;
    w.cw[0] = w.cw[1] = 0;
    uint32_t P[3] = {0, 0, 0};
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint64_t g = g0 + 32 * j + lane;
        uint32_t c = 0, len = 0;
        if (g < ngroups) {
            if constexpr (kSmem)
                c = ctrl[g - sbase];
            else
                c = __ldg(ctrl + g);
            if (g == ngroups - 1 && tail_r) {
                c &= (1u << (2 * tail_r)) - 1u;  // unused fields of the final control byte are ignored
                len = fsum(c) + tail_r;
            } else {
                len = fsum(c) + 4u;
            }
        }
        w.cw[j >> 2] |= c << (8 * (j & 3));
        P[j / 3] |= len << (10 * (j % 3));
    }
    w.total = packed_row_scan(P, w.qw);
    return w;
}

// ---- staging of a tile's compressed bytes ---------------------------------
// Global bytes [beg, end) -> stage, stage byte (beg & 15) + i <-> global beg + i.
// One TMA bulk copy when the 16-B aligned cover [a0, a1) lies inside the
// readable range [lo, hi); otherwise guarded per-lane loads (first/last tiles).
// `reuse` adds the generic->async proxy fence needed when the buffer was read before.
__device__ __forceinline__ void stage_tile(uint8_t* stage, uint64_t* bar, uint32_t& phase, uintptr_t beg,
                                           uintptr_t end, uintptr_t lo, uintptr_t hi, bool reuse) {
    const int lane = threadIdx.x & 31;
    const uintptr_t a0 = beg & ~(uintptr_t)15, a1 = (end + 15) & ~(uintptr_t)15;
    const uint32_t bytes = (uint32_t)(a1 - a0);
    if (bytes == 0) return;
    if (a0 >= lo && a1 <= hi) {
        if (lane == 0) {
            if (reuse) fence_proxy_async_smem();
            mbar_arrive_expect_tx(bar, bytes);
            bulk_g2s(stage, reinterpret_cast<const void*>(a0), bytes, bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1u;
    } else {
        for (uint32_t c = lane; c < bytes / 16; c += 32)
            *reinterpret_cast<uint4*>(stage + 16 * c) = load_chunk_guarded(a0 + 16 * (uintptr_t)c, lo, hi);
        __syncwarp();
    }
}

// ---- decode: expand the staged tile ----------------------------------------
// Plain: stores every group.  Delta: vv[j] = in-tile inclusive prefix (without
// the carry); returns the tile's delta sum.  `out` is the array's integer 0.
template <bool kDelta>
__device__ __forceinline__ uint32_t expand_tile(const WarpCtrl& w, const uint8_t* stage, uint32_t head, uint64_t g0,
                                                uint64_t ngroups, uint32_t tail_r, uint32_t* __restrict__ out,
                                                bool out16, uint4 (&vv)[kWTRows]) {
    const int lane = threadIdx.x & 31;
    const uint32_t* W = reinterpret_cast<const uint32_t*>(stage);
    uint32_t rowbase = 0;
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint32_t c = row_ctrl(w, j);
        const uint32_t b = head + row_q(w, j);
        const bool allzero = __all_sync(kFull, c == 0);
        uint4 v = allzero ? decode_zero_group(W, b) : decode_group(W, b, c);
        const uint64_t g = g0 + 32 * j + lane;
        const uint32_t cnt = group_count(g, ngroups, tail_r);
        if constexpr (!kDelta) {
            if (cnt && out) store_group(out + 4 * g, v, cnt, out16);
            else if (cnt) vv[0].x ^= v.x ^ v.y ^ v.z ^ v.w;  // debug no-store mode keeps the work alive
        } else {
            v = prefix4(mask_tail(v, cnt));
            const uint32_t S = v.w;
            const uint32_t I = warp_inclusive_scan(S);
            vv[j] = add4(v, rowbase + I - S);
            rowbase += __shfl_sync(kFull, I, 31);
        }
    }
    return rowbase;
}

template <bool kDelta>
__device__ __forceinline__ void store_tile(const uint4 (&vv)[kWTRows], uint32_t carry, uint64_t g0, uint64_t ngroups,
                                           uint32_t tail_r, uint32_t* __restrict__ out, bool out16) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint64_t g = g0 + 32 * j + lane;
        const uint32_t cnt = group_count(g, ngroups, tail_r);
        if (cnt) store_group(out + 4 * g, add4(vv[j], carry), cnt, out16);
    }
}

// ---- encode -----------------------------------------------------------------
// Loads the tile's integers (row-major, 128-bit), forms deltas (x_{-1} = prev_in
// for the tile's first integer), writes the control bytes and returns the
// per-row byte lengths packed (l0 | l1<<8 | l2<<16 | l3<<24) plus the scan.
struct EncodeTile {
    uint4 d[kWTRows];       // values (plain) or deltas
    uint32_t lens[kWTRows]; // packed per-integer byte lengths (0 = absent)
    uint32_t qw[4];         // tile-local data offsets (packed like WarpCtrl::qw)
    uint32_t total;
};

template <bool kDelta>
__device__ __forceinline__ void encode_load(const uint32_t* __restrict__ in, uint64_t g0, uint64_t ngroups,
                                            uint32_t tail_r, uint32_t prev_in, uint8_t* __restrict__ ctrl_out,
                                            EncodeTile& t) {
    const int lane = threadIdx.x & 31;
    const bool in16 = (((uintptr_t)in) & 15) == 0;
    uint32_t P[3] = {0, 0, 0};
    uint32_t last_w = prev_in;
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint64_t g = g0 + 32 * j + lane;
        const uint32_t cnt = group_count(g, ngroups, tail_r);
        uint4 x = make_uint4(0, 0, 0, 0);
        if (cnt == 4 && in16) {
            x = ldg_stream_v4(in + 4 * g);
        } else if (cnt) {
            x.x = __ldg(in + 4 * g);
            if (cnt > 1) x.y = __ldg(in + 4 * g + 1);
            if (cnt > 2) x.z = __ldg(in + 4 * g + 2);
            if (cnt > 3) x.w = __ldg(in + 4 * g + 3);
        }
        if constexpr (kDelta) {
            uint32_t p = __shfl_up_sync(kFull, x.w, 1);
            if (lane == 0) p = last_w;
            last_w = __shfl_sync(kFull, x.w, 31);
            x = make_uint4(x.x - p, x.y - x.x, x.z - x.y, x.w - x.z);
        }
        t.d[j] = x;
        const uint32_t l0 = cnt > 0 ? dev_byte_length(x.x) : 0u;
        const uint32_t l1 = cnt > 1 ? dev_byte_length(x.y) : 0u;
        const uint32_t l2 = cnt > 2 ? dev_byte_length(x.z) : 0u;
        const uint32_t l3 = cnt > 3 ? dev_byte_length(x.w) : 0u;
        t.lens[j] = l0 | (l1 << 8) | (l2 << 16) | (l3 << 24);
        P[j / 3] |= (l0 + l1 + l2 + l3) << (10 * (j % 3));
        if (cnt) {
            const uint32_t c = (l0 - 1) | (l1 ? ((l1 - 1) << 2) : 0u) | (l2 ? ((l2 - 1) << 4) : 0u) |
                               (l3 ? ((l3 - 1) << 6) : 0u);
            ctrl_out[g] = (uint8_t)c;
        }
    }
    t.total = packed_row_scan(P, t.qw);
}

// Write every integer's bytes at its tile-local offset + base (stage byte base = tile data byte 0).
// A row whose 128 integers all take one byte (the usual case for small
// deltas) packs as 32 consecutive 4-byte words: each lane assembles its 4 low
// bytes with PRMT and stores the aligned word it starts (merged with its left
// neighbour's tail through a funnel shift); only the row's first and last
// partial words go out as bytes.  Every other row stores byte by byte.
__device__ __forceinline__ void encode_pack_at(const EncodeTile& t, uint8_t* stage, uint32_t base) {
    const int lane = threadIdx.x & 31;
    uint32_t* W = reinterpret_cast<uint32_t*>(stage);
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint32_t l = t.lens[j];
        if (__all_sync(kFull, l == 0x01010101u)) {
            const uint4 x = t.d[j];
            const uint32_t P = __byte_perm(__byte_perm(x.x, x.y, 0x0040), __byte_perm(x.z, x.w, 0x0040), 0x5410);
            const uint32_t Pp = __shfl_up_sync(kFull, P, 1);
            const uint32_t p = base + ((t.qw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
            const uint32_t s = p & 3u;
            if (s == 0) {
                W[p >> 2] = P;
            } else {
                if (lane > 0) W[p >> 2] = __funnelshift_r(Pp, P, 8u * (4u - s));
                if (lane == 0)
                    for (uint32_t b = 0; b < 4u - s; ++b) stage[p + b] = (uint8_t)(P >> (8 * b));
                if (lane == 31)
                    for (uint32_t b = 4u - s; b < 4u; ++b) stage[p + b] = (uint8_t)(P >> (8 * b));
            }
            continue;
        }
        if (l) {
            uint32_t p = base + ((t.qw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
            const uint32_t l0 = l & 0xFFu, l1 = (l >> 8) & 0xFFu, l2 = (l >> 16) & 0xFFu, l3 = l >> 24;
            put_int_bytes(stage, p, t.d[j].x, l0);
            p += l0;
            if (l1) put_int_bytes(stage, p, t.d[j].y, l1);
            p += l1;
            if (l2) put_int_bytes(stage, p, t.d[j].z, l2);
            p += l2;
            if (l3) put_int_bytes(stage, p, t.d[j].w, l3);
        }
    }
}

__device__ __forceinline__ void encode_pack(const EncodeTile& t, uint8_t* stage) { encode_pack_at(t, stage, 0); }

// Copy stage bytes [0, total) to global [beg, beg + total): aligned 128-bit
// stores for interior chunks (unaligned shared reads via funnel shifts), byte
// stores for the two edge chunks shared with neighbouring tiles.
__device__ __forceinline__ void encode_writeout(const uint8_t* stage, uintptr_t beg, uint32_t total) {
    const int lane = threadIdx.x & 31;
    const uintptr_t end = beg + total;
    const uintptr_t a0 = beg & ~(uintptr_t)15, a1 = (end + 15) & ~(uintptr_t)15;
    const uint32_t h = (uint32_t)(beg - a0);
    const uint32_t* W = reinterpret_cast<const uint32_t*>(stage);
    const uint32_t nch = (uint32_t)((a1 - a0) >> 4);
    for (uint32_t c = lane; c < nch; c += 32) {
        const uintptr_t a = a0 + 16 * (uintptr_t)c;
        if (a >= beg && a + 16 <= end) {
            const uint32_t s = 16 * c - h, k = s >> 2, sh = (s & 3u) * 8u;
            const uint32_t w0 = W[k], w1 = W[k + 1], w2 = W[k + 2], w3 = W[k + 3], w4 = W[k + 4];
            const uint4 o = make_uint4(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh),
                                       __funnelshift_r(w2, w3, sh), __funnelshift_r(w3, w4, sh));
            stg_stream_v4(reinterpret_cast<void*>(a), o);
        } else {
            for (int b = 0; b < 16; ++b) {
                const uintptr_t x = a + b;
                if (x >= beg && x < end) *reinterpret_cast<uint8_t*>(x) = stage[x - beg];
            }
        }
    }
}

}  // namespace bcgpu
