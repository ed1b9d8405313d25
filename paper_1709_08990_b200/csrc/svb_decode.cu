// svb_decode.cu -- single-array Stream VByte decode for sm_100a
// (svb_decode / svb_decode_delta: reference stream_vbyte.hpp:38-42, codec.hpp:85-90).
//
//   1. svb_ctrl_scan_kernel   control bytes only (0.25 B/int): per 64-sub-tile chunk
//      the chunk-local exclusive prefix of every 1024-integer sub-tile's data length
//      (length[c] = 4 + sum of fields) and the chunk total; the last
//      CTA to finish scans the chunk totals and validates the stream length
//      (truncated / trailing_bytes).
//   2. plain:  svb_decode_pool_kernel<kModePlain> -- one TMA for a CTA's control bytes,
//      one for its whole data range, expansion straight to 128-bit stores.
//      delta:  svb_decode1_kernel -- one pass with deferred look-back over tile sums
//      (cooperative launch), or, for a piece of a stream (host pipeline), the pipelined
//      sums pass svb_sums_kernel + svb_decode_pool_kernel<kModeDelta> with the carries.
// The delta variants fuse the mod-2^32 prefix sum.  No kernel waits on
// a CTA of its own round.
#include <cstdint>

#include "svb_device.cuh"
#include "svb_fast.cuh"
#include "launch_cache.cuh"
#include "svb_kernels.cuh"
#include "svb_tma.cuh"
#include "svb_scan.cuh"
#include "svb_warp.cuh"

namespace bcgpu {


__device__ __forceinline__ void dec_report(unsigned long long* st, uint32_t epoch, uint32_t code) {
    if (st) *st = ((unsigned long long)epoch << 32) | code;
}

// ---------------------------------------------------------------------------
// 1. control scan
// ---------------------------------------------------------------------------
// 4 threads per sub-tile, 64 control bytes (16 words) each.
__device__ __forceinline__ uint32_t quarter_length(const uint8_t* __restrict__ ctrl, uint64_t g, uint64_t ngroups,
                                                   uint32_t tail_r) {
    if (g >= ngroups) return 0;
    const uint64_t cnt = ngroups - g < 64 ? ngroups - g : 64;
    const bool has_tail = tail_r != 0 && g + cnt == ngroups;
    uint32_t sum = 0;
    if (cnt == 64 && !has_tail && (((uintptr_t)(ctrl + g)) & 15) == 0) {
        const uint4* p = reinterpret_cast<const uint4*>(ctrl + g);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint4 w = __ldg(p + k);
            sum += (swar_lengths(w.x) * 0x01010101u) >> 24;
            sum += (swar_lengths(w.y) * 0x01010101u) >> 24;
            sum += (swar_lengths(w.z) * 0x01010101u) >> 24;
            sum += (swar_lengths(w.w) * 0x01010101u) >> 24;
        }
        return sum;
    }
    for (uint64_t i = 0; i < cnt; ++i) {
        uint32_t c = __ldg(ctrl + g + i);
        if (has_tail && i == cnt - 1) {
            c &= (1u << (2 * tail_r)) - 1u;
            sum += fsum(c) + tail_r;
        } else {
            sum += fsum(c) + 4u;
        }
    }
    return sum;
}

__global__ void __launch_bounds__(256)
    svb_ctrl_scan_kernel(const uint8_t* __restrict__ in, uint64_t in_len, uint64_t n, DecodeMeta meta,
                         unsigned long long* status, uint32_t epoch, int zero_sums) {
    __shared__ uint32_t wt[8];
    __shared__ unsigned long long wt64[8];
    __shared__ bool last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t chunk = blockIdx.x, nchunks = gridDim.x;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    // the next kernel (programmatic dependent launch) may start its prologue now; it waits
    // for this grid's completion before reading anything written here
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if ((zero_sums & 1) && tid == 0) meta.chunksums[chunk] = 0;
    // delta: clear this chunk's one-pass aggregates, so nothing stale can carry the call's epoch
    if ((zero_sums & 1) && tid < kChunkSubs / kCTWarps) {
        const uint64_t tile = (uint64_t)chunk * (kChunkSubs / kCTWarps) + tid;
        if (tile * kCTWarps < nsub) meta.agg[tile] = 0;
    }
    const uint64_t g = (uint64_t)chunk * kChunkCtrl + (uint64_t)tid * 64;
    uint32_t q = quarter_length(in, g, ngroups, tail_r);
    // sub-tile length = sum of its 4 quarters (lanes 4k..4k+3)
    q += __shfl_xor_sync(kFull, q, 1);
    q += __shfl_xor_sync(kFull, q, 2);
    // chunk-local exclusive prefix over the 64 sub-tiles (8 per warp, lanes 4k)
    const uint32_t v = (lane & 3) == 0 ? q : 0u;
    const uint32_t incl = warp_inclusive_scan(v);
    if (lane == 31) wt[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        wpre += w < warp ? wt[w] : 0u;
        total += wt[w];
    }
    const uint64_t sub = (uint64_t)chunk * kChunkSubs + (tid >> 2);
    if ((lane & 3) == 0 && sub < nsub) meta.localpre[sub] = wpre + incl - v;
    if (tid == 0) meta.chunkpre[chunk] = total;
    // last CTA: scan the chunk totals, validate the stream length -- unless the one-pass
    // decode follows (zero_sums bit 1): its producers sum the totals themselves and its
    // last tile checks the length, so this phase is off the critical path
    if (zero_sums & 2) return;
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        last = atomicAdd(meta.counters, 1u) == nchunks - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const unsigned long long tot = cta_exclusive_scan<unsigned long long, 8>(meta.chunkpre, nchunks, wt64);
    if (tid == 0) {
        meta.chunkpre[nchunks] = tot;
        const uint64_t need = ngroups + tot;
        dec_report(status, epoch, need > in_len ? BCGPU_ERR_TRUNCATED : (need < in_len ? BCGPU_ERR_TRAILING_BYTES : 0u));
        *meta.counters = 0;
    }
}

// ---------------------------------------------------------------------------
// 2./3. decode passes
// ---------------------------------------------------------------------------
// kModePlain / kModeDelta: what svb_decode_pool_kernel stores; kModeSums: expand_full's
// sum-only mode (svb_fast.cuh), used by the sums pass and the one-pass decode.
enum : int { kModePlain = 0, kModeDelta = 1, kModeSums = 2 };

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// ---------------------------------------------------------------------------
// 2'./3'. pooled decode: one CTA per 8*K sub-tiles, one TMA for all their bytes
// ---------------------------------------------------------------------------
// The CTA's sub-tiles are consecutive, so their compressed bytes are one
// contiguous range: thread 0 issues a single bulk copy of it into a pool sized
// by the host from the stream's average compression (so compressible streams
// put 2-4x more sub-tiles in flight per SM than a worst-case 4 KiB per warp),
// plus one bulk copy of the 256*8K control bytes.  Round r of the CTA is
// sub-tiles s0 + 8r + warp; if the whole range does not fit the pool the
// rounds are loaded one at a time (each <= 32 KiB).  Outputs leave as 128-bit
// stores straight from registers; delta carries are known up front from the
// sums pass (scanned chunk carry + the earlier sub-tiles' sums).
struct PoolShared {
    uint32_t loc[40];                 // localpre[s0 .. s0+36)
    unsigned long long chk[4];        // chunkpre[(c & ~1) .. +4)
    uint32_t carry[32];               // delta: carry before each of the CTA's sub-tiles (without base)
    uint32_t part[8];
    uint64_t bar_meta, bar_ctrl, bar_data[4];
};

template <int kMode, int K>
__global__ void __launch_bounds__(kCTThreads)
    svb_decode_pool_kernel(const uint8_t* __restrict__ in, uint64_t in_len, uint64_t n, uint32_t base,
                           uint32_t* __restrict__ out, uint32_t* __restrict__ d_last, DecodeMeta meta,
                           uint32_t pool_bytes, uint64_t sub_begin) {
    constexpr int S = kCTWarps * K;  // sub-tiles per CTA (divides kChunkSubs)
    static_assert(kChunkSubs % S == 0 && S <= 32, "CTA sub-tiles must stay inside one chunk");
    extern __shared__ __align__(128) uint8_t dsm[];
    uint8_t* sctrl = dsm;                           // S * 256 control bytes
    uint8_t* pool = dsm + S * kWTGroups;            // compressed data
    __shared__ __align__(16) PoolShared sh;
    __shared__ bool single;
    constexpr bool kDelta = kMode == kModeDelta;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    // the delta pass walks the tiles last to first: the sums pass just streamed the
    // compressed bytes front to back, so their tail is what L2 still holds
    const uint32_t bid = kMode == kModeDelta ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
    const uint64_t s0 = sub_begin + (uint64_t)bid * S;
    const uint64_t chunk = s0 / kChunkSubs;
    const uint32_t ns = (uint32_t)(nsub - s0 < (uint64_t)S ? nsub - s0 : (uint64_t)S);
    const uintptr_t lo = (uintptr_t)in, hi = lo + in_len;
    const uintptr_t data0 = lo + ngroups;

    if (threadIdx.x == 0) {
        mbar_init1(&sh.bar_meta);
        mbar_init1(&sh.bar_ctrl);
#pragma unroll
        for (int r = 0; r < 4; ++r) mbar_init1(&sh.bar_data[r]);
        constexpr uint32_t lb = (uint32_t)(((S + 4) * 4 + 15) & ~15);
        mbar_expect(&sh.bar_meta, lb + 32);
        tma_load(sh.loc, meta.localpre + s0, lb, &sh.bar_meta);
        tma_load(sh.chk, meta.chunkpre + (chunk & ~1ull), 32, &sh.bar_meta);
        // control bytes of the whole CTA in one transaction (no offsets needed)
        const uintptr_t cb = lo + s0 * kWTGroups;
        const uint64_t cg = ngroups - s0 * kWTGroups < (uint64_t)S * kWTGroups ? ngroups - s0 * kWTGroups
                                                                                : (uint64_t)S * kWTGroups;
        const uint32_t ctx = tma_cover_bytes(cb, cb + cg, lo, hi);
        if (ctx != 0xFFFFFFFFu && (cb & 15) == 0 && ctx) {
            mbar_expect(&sh.bar_ctrl, ctx);
            tma_load_hint(sctrl, reinterpret_cast<const void*>(cb), ctx, &sh.bar_ctrl, l2_policy_drop());
        } else {
            for (uint64_t i = 0; i < cg; ++i) sctrl[i] = __ldg(in + s0 * kWTGroups + i);
            mbar_arrive(&sh.bar_ctrl);
        }
    }
    // delta: carry parts = scanned chunk carry + sums of this chunk's sub-tiles before s0
    uint32_t part = 0;
    if constexpr (kDelta) {
        const uint64_t c0 = chunk * kChunkSubs;
        for (uint64_t i = c0 + threadIdx.x; i < s0; i += kCTThreads) part += __ldg(meta.subsums + i);
        if (threadIdx.x == 0) part += __ldg(meta.chunksums + chunk);
        part = warp_sum_u32(part);
        if (lane == 0) sh.part[warp] = part;
        if (threadIdx.x < S) sh.carry[threadIdx.x] = threadIdx.x < ns ? __ldg(meta.subsums + s0 + threadIdx.x) : 0u;
    }
    __syncthreads();
    mbar_wait_parity(&sh.bar_meta, 0);
    const unsigned long long cpre = sh.chk[chunk & 1];
    auto sub_off = [&](uint32_t i) -> unsigned long long {  // data offset of sub-tile s0 + i, i <= ns
        if (i == ns && (s0 + ns == nsub || (s0 + ns) % kChunkSubs == 0)) return sh.chk[(chunk & 1) + 1];
        return cpre + sh.loc[i];
    };
    const unsigned long long A = sub_off(0), B = sub_off(ns);
    const uintptr_t abeg = data0 + A;
    if (threadIdx.x == 0) {
        const uint32_t tx = tma_cover_bytes(abeg, data0 + B, lo, hi);
        single = tx != 0xFFFFFFFFu && tx + 16 <= pool_bytes;
        if (single && tx) {
            mbar_expect(&sh.bar_data[0], tx);
            tma_load_hint(pool, reinterpret_cast<const void*>(abeg & ~(uintptr_t)15), tx, &sh.bar_data[0], l2_policy_drop());
        } else if (single) {
            mbar_arrive(&sh.bar_data[0]);
        }
    }
    if constexpr (kDelta) {
        if (threadIdx.x == 0) {  // exclusive prefix of the CTA's sub-tile sums + the CTA carry
            uint32_t c = base;
#pragma unroll
            for (int k = 0; k < kCTWarps; ++k) c += sh.part[k];
            for (int i = 0; i < S; ++i) {
                const uint32_t x = sh.carry[i];
                sh.carry[i] = c;
                c += x;
            }
        }
    }
    __syncthreads();
    mbar_wait_parity(&sh.bar_ctrl, 0);
    if (single) mbar_wait_parity(&sh.bar_data[0], 0);
    const bool out16 = (((uintptr_t)out) & 15) == 0;
    for (int r = 0; r < K; ++r) {
        // round r = sub-tiles s0 + 8r .. s0 + 8r + 7 (contiguous data)
        uintptr_t pbase = abeg;  // global address of pool byte (pbase & 15)
        if (!single) {
            const uint32_t i0 = (uint32_t)(8 * r), i1 = (uint32_t)(8 * r + 8) < ns ? (uint32_t)(8 * r + 8) : ns;
            __syncthreads();  // previous round fully consumed
            if (i0 < ns) {
                pbase = data0 + sub_off(i0);
                const uintptr_t pend = data0 + sub_off(i1);
                if (threadIdx.x == 0) fence_async_smem();
                const uint32_t tx = tma_cover_bytes(pbase, pend, lo, hi);
                if (tx != 0xFFFFFFFFu && tx + 16 <= pool_bytes) {
                    if (threadIdx.x == 0) {
                        if (tx) {
                            mbar_expect(&sh.bar_data[r], tx);
                            tma_load(pool, reinterpret_cast<const void*>(pbase & ~(uintptr_t)15), tx, &sh.bar_data[r]);
                        } else {
                            mbar_arrive(&sh.bar_data[r]);
                        }
                    }
                    mbar_wait_parity(&sh.bar_data[r], 0);
                } else {
                    // malformed or edge: guarded copy by the whole CTA, clamped to the pool
                    const uintptr_t a0 = pbase & ~(uintptr_t)15;
                    uintptr_t a1 = (pend + 15) & ~(uintptr_t)15;
                    if (a1 - a0 > pool_bytes - 16) a1 = a0 + ((pool_bytes - 16) & ~15u);
                    for (uint32_t c = threadIdx.x; c < (uint32_t)((a1 - a0) >> 4); c += kCTThreads)
                        *reinterpret_cast<uint4*>(pool + 16 * c) = load_chunk_guarded(a0 + 16 * (uintptr_t)c, lo, hi);
                    __syncthreads();
                }
            }
        }
        const uint32_t i = (uint32_t)(8 * r + warp);
        if (i >= ns) continue;
        const uint64_t s = s0 + i;
        const uint64_t g0 = s * kWTGroups;
        uint32_t head0;
        {
            const unsigned long long so0 = sub_off(i);
            head0 = (uint32_t)(data0 + so0 - (pbase & ~(uintptr_t)15));
        }
        if ((uint64_t)(s + 1) * kWTInts <= n && head0 <= pool_bytes - 32 && out16) {
            // full sub-tile: lean path (svb_fast.cuh)
            bool zero;
            const WarpCtrl wf = ctrl_full(sh_addr(sctrl) + i * kWTGroups, &zero);
            const uint32_t sd = sh_addr(pool) + head0;
            uint32_t* o = out + s * kWTInts;
            if constexpr (kMode == kModeDelta) {
                const uint32_t run = zero ? expand_full<1, true>(wf, sd, o, sh.carry[i])
                                          : expand_full<1, false>(wf, sd, o, sh.carry[i]);
                if (s == nsub - 1 && lane == 0 && d_last) *d_last = run;
            } else {
                if (zero)
                    expand_full<0, true>(wf, sd, o, 0);
                else
                    expand_full<0, false>(wf, sd, o, 0);
            }
            continue;
        }
        const WarpCtrl w = load_warp_ctrl<true>(sctrl + (uint32_t)i * kWTGroups, g0, ngroups, tail_r, g0);
        const uint32_t* W = reinterpret_cast<const uint32_t*>(pool);
        const unsigned long long so = sub_off(i);
        const uintptr_t sbeg = data0 + so;
        uint32_t head = (uint32_t)(sbeg - (pbase & ~(uintptr_t)15));
        if (head > pool_bytes - 32) head = pool_bytes - 32;  // malformed streams only: keep reads in the pool
        {
            uint32_t run = kDelta ? sh.carry[i] : 0u;
#pragma unroll
            for (int j = 0; j < kWTRows; ++j) {
                const uint32_t c = row_ctrl(w, j);
                const uint32_t bb = head + row_q(w, j);
                const bool allzero = __all_sync(kFull, c == 0);
                uint4 v = allzero ? decode_zero_group(W, bb) : decode_group(W, bb, c);
                const uint64_t g = g0 + 32 * j + lane;
                const uint32_t cnt = group_count(g, ngroups, tail_r);
                if constexpr (kDelta) {
                    v = prefix4(mask_tail(v, cnt));
                    const uint32_t Sx = v.w;
                    const uint32_t I = warp_inclusive_scan(Sx);
                    v = add4(v, run + I - Sx);
                    run += __shfl_sync(kFull, I, 31);
                }
                if (cnt) store_group(out + 4 * g, v, cnt, out16);
            }
            if (kDelta && s == nsub - 1 && lane == 0 && d_last) *d_last = run;
        }
    }
}

}  // namespace bcgpu

namespace bcgpu {

// ---------------------------------------------------------------------------
// 2''. delta sums pass: persistent producer/consumer pipeline
// ---------------------------------------------------------------------------
// The sums pass only reads (compressed bytes in, one sum per sub-tile out), so
// nothing hides its load latency but other loads.  One producer warp per CTA
// runs a ring of kSumStages stages ahead of 8 consumer warps: for tile t (8
// sub-tiles) it TMA-loads the offsets one ring cycle early, then the control
// bytes and the whole data range in one bulk copy each; consumers wait on the
// stage's `full` mbarrier, sum one sub-tile each (svb_fast.cuh lean path),
// RED.ADD into the chunk sums and release the stage through `empty`.  Tiles are
// dealt round-robin to a grid of (SMs x resident CTAs).  A tile whose data
// exceeds the stage pool (density far above the stream average) is summed
// straight from global memory.  The last CTA scans the chunk sums.
constexpr int kSumStages = 5;
constexpr int kSumThreads = 288;  // 8 consumer warps + 1 producer warp

struct __align__(16) SumMeta {
    uint32_t loc[12];           // localpre[s0 .. s0+12)
    unsigned long long chk[4];  // chunkpre[(c & ~1) .. +4)
};
struct SumHdr {
    unsigned long long base;  // global address of pool byte 0 (16-B aligned)
    uint32_t head[9];         // offset of sub-tile i's data from `base`, i = 0..8
    uint32_t mode;            // 0: data staged in the pool, 1: read from global memory
};
struct __align__(16) SumsShared {
    SumMeta meta[8];
    SumHdr hdr[8];
    uint64_t full[8], empty[8], mfull[8];
    uint32_t scan[16];
    bool last;
};

// aligned 32-bit word at global address a; bytes outside [lo, hi) read as 0
__device__ __forceinline__ uint32_t gword_guarded(uintptr_t a, uintptr_t lo, uintptr_t hi) {
    if (a >= lo && a + 4 <= hi) return __ldg(reinterpret_cast<const uint32_t*>(a));
    uint32_t w = 0;
    for (int b = 0; b < 4; ++b)
        if (a + b >= lo && a + b < hi) w |= (uint32_t)__ldg(reinterpret_cast<const uint8_t*>(a + b)) << (8 * b);
    return w;
}

// Sum of a (possibly partial) sub-tile's integers; word i of its data window is fw(i),
// the data starts at byte `head` of the window.
template <class Fetch>
__device__ __forceinline__ uint32_t sums_generic(const uint8_t* sctrl, uint64_t g0, uint64_t ngroups, uint32_t tail_r,
                                                 uint32_t head, Fetch fw) {
    const int lane = threadIdx.x & 31;
    const WarpCtrl w = load_warp_ctrl<true>(sctrl, g0, ngroups, tail_r, g0);
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint32_t c = row_ctrl(w, j);
        uint32_t b = head + row_q(w, j);
        const uint32_t cnt = group_count(g0 + 32 * j + lane, ngroups, tail_r);
#pragma unroll
        for (int f = 0; f < 4; ++f) {
            const uint32_t l = ((c >> (2 * f)) & 3u) + 1u;
            const uint32_t x = __funnelshift_r(fw(b >> 2), fw((b >> 2) + 1), (b & 3u) * 8u);
            if ((uint32_t)f < cnt) acc += x & (0xFFFFFFFFu >> (32u - 8u * l));
            b += l;
        }
    }
    return warp_sum_u32(acc);
}

template <int NST>
__global__ void __launch_bounds__(kSumThreads)
    svb_sums_kernel(const uint8_t* __restrict__ in, uint64_t in_len, uint64_t n, DecodeMeta meta,
                    uint32_t pool_bytes, uint32_t t_begin, uint32_t t_end) {
    extern __shared__ __align__(128) uint8_t dsm[];
    __shared__ SumsShared sh;
    constexpr uint32_t kTileCtrl = kCTWarps * kWTGroups;  // 2 KiB of control bytes per tile
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint32_t ntiles = t_end;  // tiles [t_begin, t_end) of this launch
    const uintptr_t lo = (uintptr_t)in, hi = lo + in_len, data0 = lo + ngroups;
    const uint32_t stride = kTileCtrl + pool_bytes;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NST; ++k) {
            mbar_init(&sh.full[k], 1);
            mbar_init(&sh.empty[k], kCTWarps);
            mbar_init(&sh.mfull[k], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kCTWarps) {
        // ---- producer ----
        auto issue_meta = [&](uint32_t t, int st) {
            const uint64_t s0 = (uint64_t)t * kCTWarps, c = s0 / kChunkSubs;
            mbar_expect(&sh.mfull[st], 48 + 32);
            tma_load(sh.meta[st].loc, meta.localpre + s0, 48, &sh.mfull[st]);
            tma_load(sh.meta[st].chk, meta.chunkpre + (c & ~1ull), 32, &sh.mfull[st]);
        };
        if (lane == 0)
            for (int i = 0; i < NST; ++i) {
                const uint64_t t = (uint64_t)t_begin + blockIdx.x + (uint64_t)i * gridDim.x;
                if (t < ntiles) issue_meta((uint32_t)t, i);
            }
        uint32_t k = 0;
        for (uint32_t t = t_begin + blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
            const int st = (int)(k % NST);
            const uint32_t ph = (k / NST) & 1u;
            uint8_t* sc = dsm + (uint32_t)st * stride;
            uint8_t* pool = sc + kTileCtrl;
            const uint64_t s0 = (uint64_t)t * kCTWarps, chunk = s0 / kChunkSubs;
            const uint32_t ns = (uint32_t)(nsub - s0 < (uint64_t)kCTWarps ? nsub - s0 : (uint64_t)kCTWarps);
            mbar_wait_parity(&sh.mfull[st], ph);
            if (meta.trace && lane == 0) meta.trace[8ull * t + 0] = gtimer();
            const SumMeta& M = sh.meta[st];
            const unsigned long long cpre = M.chk[chunk & 1];
            const bool end_at_chunk = s0 + ns == nsub || (s0 + ns) % kChunkSubs == 0;
            const unsigned long long A = cpre + M.loc[0];
            const unsigned long long B = end_at_chunk ? M.chk[(chunk & 1) + 1] : cpre + M.loc[ns];
            const uint32_t li = (uint32_t)lane < ns ? (uint32_t)lane : ns;
            const unsigned long long my = (li == ns) ? B : cpre + M.loc[li];
            const uintptr_t Ag = data0 + A, Bg = data0 + B, base = Ag & ~(uintptr_t)15;
            const uint32_t tx = tma_cover_bytes(Ag, Bg, lo, hi);
            const bool fits = tx != 0xFFFFFFFFu && tx + 16 <= pool_bytes;
            const uintptr_t cb = lo + s0 * kWTGroups;
            const uint64_t cg = ngroups - s0 * kWTGroups < (uint64_t)kTileCtrl ? ngroups - s0 * kWTGroups
                                                                                 : (uint64_t)kTileCtrl;
            const uint32_t ctx = tma_cover_bytes(cb, cb + cg, lo, hi);
            const bool c_tma = ctx != 0xFFFFFFFFu && (cb & 15) == 0;
            __syncwarp();  // every lane has read meta[st]
            if (k >= (uint32_t)NST) mbar_wait_parity_sleep(&sh.empty[st], ph ^ 1u);  // consumers left the stage
            if (!c_tma)
                for (uint32_t i = lane; i < (uint32_t)cg; i += 32) sc[i] = __ldg(in + s0 * kWTGroups + i);
            if (lane <= 8) sh.hdr[st].head[lane] = (uint32_t)(data0 + my - base);
            if (lane == 0) {
                sh.hdr[st].base = base;
                sh.hdr[st].mode = fits ? 0u : 1u;
            }
            __syncwarp();
            if (lane == 0) {
                if (meta.trace) meta.trace[8ull * t + 1] = gtimer();
                fence_async_smem();
                mbar_expect(&sh.full[st], (c_tma ? ctx : 0u) + (fits ? tx : 0u));
                // the delta pass re-reads these bytes right after: keep them in L2
                const uint64_t keep = l2_policy_keep();
                if (c_tma && ctx) tma_load_hint(sc, reinterpret_cast<const void*>(cb), ctx, &sh.full[st], keep);
                if (fits && tx) tma_load_hint(pool, reinterpret_cast<const void*>(base), tx, &sh.full[st], keep);
                const uint64_t tn = (uint64_t)t + (uint64_t)NST * gridDim.x;  // meta[st] was consumed above
                if (tn < ntiles) issue_meta((uint32_t)tn, st);
            }
        }
    } else {
        // ---- consumers: warp w sums sub-tile 8t + w ----
        uint32_t k = 0;
        for (uint32_t t = t_begin + blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
            const int st = (int)(k % NST);
            const uint32_t ph = (k / NST) & 1u;
            mbar_wait_parity(&sh.full[st], ph);
            if (meta.trace && lane == 0) meta.trace[8ull * t + 2 + (warp == 0 ? 0 : 2)] = gtimer();
            const uint64_t s = (uint64_t)t * kCTWarps + warp;
            if (s < nsub) {
                const uint8_t* sc = dsm + (uint32_t)st * stride + warp * kWTGroups;
                const uint8_t* pool = dsm + (uint32_t)st * stride + kTileCtrl;
                const uint32_t head = sh.hdr[st].head[warp];
                const uint64_t g0 = s * kWTGroups;
                uint32_t acc;
                if (sh.hdr[st].mode == 0) {
                    if ((s + 1) * kWTInts <= n && head <= pool_bytes - 32) {
                        const uint32_t sd = sh_addr(pool) + head;
                        if (ctrl_all_zero(sh_addr(sc))) {  // 1024 one-byte integers: a byte sum
                            acc = __reduce_add_sync(kFull, zero_tile_sum(sd));
                        } else {
                            bool zero;
                            const WarpCtrl wf = ctrl_full(sh_addr(sc), &zero);
                            acc = __reduce_add_sync(kFull, expand_full<2, false>(wf, sd, nullptr, 0));
                        }
                    } else {
                        const uint32_t* W = reinterpret_cast<const uint32_t*>(pool);
                        const uint32_t lim = pool_bytes / 4 - 1;
                        acc = sums_generic(sc, g0, ngroups, tail_r, head,
                                           [&](uint32_t i) { return W[i < lim ? i : lim]; });
                    }
                } else {
                    const uintptr_t gb = (uintptr_t)sh.hdr[st].base;
                    acc = sums_generic(sc, g0, ngroups, tail_r, head,
                                       [&](uint32_t i) { return gword_guarded(gb + 4 * (uintptr_t)i, lo, hi); });
                }
                if (lane == 0) {
                    meta.subsums[s] = acc;
                    atomicAdd(meta.chunksums + s / kChunkSubs, acc);  // RED.ADD, mod 2^32
                }
            }
            __syncwarp();
            if (meta.trace && lane == 0 && (warp == 0 || warp == 7)) meta.trace[8ull * t + 3 + (warp == 0 ? 0 : 2)] = gtimer();
            if (lane == 0) mbar_arrive(&sh.empty[st]);
        }
    }
    // last CTA: exclusive scan of the chunk sums
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        sh.last = atomicAdd(meta.counters + 1, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!sh.last) return;
    __threadfence();
    // chunks of this launch: exclusive scan continuing from the carry of the chunks before
    // (meta.running, left by the previous piece's launch)
    const uint32_t nchunks = (uint32_t)((nsub + kChunkSubs - 1) / kChunkSubs);
    constexpr uint32_t kTilesPerChunk = kChunkSubs / kCTWarps;
    const uint32_t c0 = t_begin / kTilesPerChunk;
    const uint32_t c1e = (t_end + kTilesPerChunk - 1) / kTilesPerChunk, c1 = c1e < nchunks ? c1e : nchunks;
    const uint32_t base = c0 == 0 ? 0u : (uint32_t)__ldcg(meta.running);
    const uint32_t tot = cta_exclusive_scan<uint32_t, kSumThreads / 32>(meta.chunksums + c0, c1 - c0, sh.scan);
    if (base)
        for (uint32_t c = threadIdx.x; c < c1 - c0; c += kSumThreads) meta.chunksums[c0 + c] += base;
    if (threadIdx.x == 0) {
        *meta.running = base + tot;
        meta.counters[1] = 0;
    }
}

// ---------------------------------------------------------------------------
// 2b. one-pass delta decode: deferred look-back
// ---------------------------------------------------------------------------
// Replaces the sums pass + delta pass (two reads of the compressed bytes) with one
// read, and no CTA ever waits on a CTA of its own round.  Persistent CTAs
// (cooperative launch: all co-resident) take tiles t = b, b + G, ...  The producer
// warp streams control + data bytes through a TMA ring exactly as in the sums
// pass.  For tile t (round r) the 8 consumer warps:
//   1. sum their sub-tiles straight from the staged bytes (dp4a for all-zero
//      control bytes, as the sums pass) and publish the tile sum A(t) as an
//      epoch-tagged aggregate (relaxed 64-bit store);
//   2. resolve the carry of the CTA's tile tp = t - kD1Lag*G, deferred by kD1Lag
//      rounds: carry(tp) = incl(tp - G) + sum of A(j), tp - G < j < tp -- its own
//      inclusive prefix from the round before plus the aggregates of the G - 1
//      tiles in between, all published kD1Lag - 1 rounds or more earlier (their
//      loads were issued at the top of the iteration, so their latency hides behind
//      step 1).  Two rounds of lag let a CTA run a full round ahead of a slow one
//      before it has to wait on it (with one, the resolve spun on the previous
//      round's aggregates and the CTA stalled at the next named barrier);
//   3. decode tile tp from its stage -- held kD1Lag extra rounds -- with that
//      carry, store it from registers, and release the stage.
// The compressed bytes are read from HBM once (the stage is re-read from smem).
// A round-r aggregate only depends on waits for rounds <= r - 1, so with every
// CTA resident the chain cannot deadlock.  Only aggregates are shared; every CTA
// keeps its own inclusive chain.
constexpr int kD1Lag = 2;     // tile t is resolved kD1Lag rounds after it is summed
constexpr int kD1Stages = 6;  // tiles t, t - G, ..., t - kD1Lag*G held, the rest in flight

struct __align__(16) D1Shared {
    SumMeta meta[kD1Stages];
    SumHdr hdr[kD1Stages];
    uint64_t full[kD1Stages], empty[kD1Stages], mfull[kD1Stages];
    uint32_t wsum[3][kCTWarps];  // sub-tile sums, by round % 3
    uint32_t wcarry[kCTWarps];   // carry before each sub-tile of the tile being resolved
    uint32_t red[kCTWarps];
    uint32_t carry, incl;
};


// any sub-tile (partial, or data read from global memory) with carry `run`: word i of its
// data window is fw(i), data at byte `head`; stores its integers, returns the last value
template <class Fetch>
__device__ __forceinline__ uint32_t decode_generic_store(const uint8_t* sctrl, uint64_t g0, uint64_t ngroups,
                                                         uint32_t tail_r, uint32_t head, Fetch fw, uint32_t run,
                                                         uint32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const WarpCtrl w = load_warp_ctrl<true>(sctrl, g0, ngroups, tail_r, g0);
    const bool out16 = (((uintptr_t)(out + 4 * g0)) & 15) == 0;
#pragma unroll 1
    for (int j = 0; j < kWTRows; ++j) {
        const uint32_t c = row_ctrl(w, j);
        uint32_t b = head + row_q(w, j);
        const uint64_t g = g0 + 32 * j + lane;
        const uint32_t cnt = group_count(g, ngroups, tail_r);
        uint32_t x[4];
#pragma unroll
        for (int f = 0; f < 4; ++f) {
            const uint32_t l = ((c >> (2 * f)) & 3u) + 1u;
            const uint32_t y = __funnelshift_r(fw(b >> 2), fw((b >> 2) + 1), (b & 3u) * 8u);
            x[f] = (uint32_t)f < cnt ? (y & (0xFFFFFFFFu >> (32u - 8u * l))) : 0u;
            b += l;
        }
        uint4 v = make_uint4(x[0], x[0] + x[1], x[0] + x[1] + x[2], x[0] + x[1] + x[2] + x[3]);
        const uint32_t I = warp_inclusive_scan(v.w);
        v = add4(v, run + I - v.w);
        if (cnt) store_group(out + 4 * g, v, cnt, out16);
        run += __shfl_sync(kFull, I, 31);
    }
    return run;
}

template <bool kTrace>
__global__ void __launch_bounds__(kSumThreads, 3)
    svb_decode1_kernel(const uint8_t* __restrict__ in, uint64_t in_len, uint64_t n, uint32_t base,
                       uint32_t* __restrict__ out, uint32_t* __restrict__ d_last, DecodeMeta meta, uint32_t pool_bytes,
                       uint32_t epoch, unsigned long long* status, uint32_t totals) {
    extern __shared__ __align__(128) uint8_t dsm[];
    __shared__ D1Shared sh;
    constexpr uint32_t kTileCtrl = kCTWarps * kWTGroups;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint32_t ntiles = (uint32_t)((nsub + kCTWarps - 1) / kCTWarps);
    const uint32_t G = gridDim.x;
    const uintptr_t lo = (uintptr_t)in, hi = lo + in_len, data0 = lo + ngroups;
    const uint32_t stride = kTileCtrl + pool_bytes;
    // dense (totals bit 1): the stream is ceil(n/4) + n bytes, so every data length is 1 and
    // every control field 0 (else the stream is truncated); data offsets are implicit -- no
    // control scan ran before this kernel, the producer computes them and the consumers
    // check that the control bytes are zero
    const bool dense = (totals & 2u) != 0;
    totals &= 1u;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < kD1Stages; ++k) {
            mbar_init(&sh.full[k], 1);
            mbar_init(&sh.empty[k], kCTWarps);
            mbar_init(&sh.mfull[k], 1);
        }
        sh.incl = base;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // launched as a programmatic dependent of the control scan: its offsets (and the
    // cleared aggregates) are visible after this
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    if (warp == kCTWarps) {
        // ---- producer (as in svb_sums_kernel) ----
        auto issue_meta = [&](uint32_t t, int st) {
            const uint64_t s0 = (uint64_t)t * kCTWarps, c = s0 / kChunkSubs;
            mbar_expect(&sh.mfull[st], 48 + 32);
            tma_load(sh.meta[st].loc, meta.localpre + s0, 48, &sh.mfull[st]);
            tma_load(sh.meta[st].chk, meta.chunkpre + (c & ~1ull), 32, &sh.mfull[st]);
        };
        if (lane == 0 && !dense)
            for (int i = 0; i < kD1Stages; ++i) {
                const uint64_t t = (uint64_t)blockIdx.x + (uint64_t)i * G;
                if (t < ntiles) issue_meta((uint32_t)t, i);
            }
        // totals: meta.chunkpre holds chunk TOTALS (the control scan skipped its last-CTA
        // scan); the producer keeps the prefix of its current chunk P and, one tile ahead,
        // loads the totals between its next two chunks (<= G/8 + 1 <= 64 of them)
        const uint32_t nchunks = (uint32_t)((nsub + kChunkSubs - 1) / kChunkSubs);
        constexpr uint32_t kTilesPerChunk = kChunkSubs / kCTWarps;
        unsigned long long P = 0, r0 = 0, r1 = 0;
        auto ld_tot = [&](uint32_t j, uint32_t lim) -> unsigned long long {
            return j < lim ? __ldg(reinterpret_cast<const unsigned long long*>(meta.chunkpre) + j) : 0ull;
        };
        if (totals) {
            const uint32_t c0 = blockIdx.x / kTilesPerChunk;
            unsigned long long a = ld_tot((uint32_t)lane, c0) + ld_tot((uint32_t)lane + 32, c0);
#pragma unroll
            for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(kFull, a, o);
            P = a;  // c0 <= 63 chunks below the first tile
            r0 = ld_tot(c0 + lane, nchunks);
            r1 = ld_tot(c0 + 32 + lane, nchunks);
        }
        uint32_t k = 0;
        int st = 0;
        uint32_t ph = 0;
        for (uint32_t t = blockIdx.x; t < ntiles; t += G, ++k, st = st + 1 == kD1Stages ? 0 : st + 1, ph ^= st == 0) {
            unsigned long long Pc = 0, Tc = 0;
            if (totals) {  // r0 / r1: totals of chunks [c, c + 64) with c = this tile's chunk
                const uint32_t c = t / kTilesPerChunk;
                const uint32_t cn = t + G < ntiles ? (t + G) / kTilesPerChunk : c + 1;
                Pc = P;
                Tc = __shfl_sync(kFull, r0, 0);
                unsigned long long a = ((uint32_t)lane < cn - c ? r0 : 0ull) + ((uint32_t)lane + 32 < cn - c ? r1 : 0ull);
#pragma unroll
                for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(kFull, a, o);
                P += a;
                r0 = ld_tot(cn + lane, nchunks);
                r1 = ld_tot(cn + 32 + lane, nchunks);
            }
            uint8_t* sc = dsm + (uint32_t)st * stride;
            uint8_t* pool = sc + kTileCtrl;
            const uint64_t s0 = (uint64_t)t * kCTWarps, chunk = s0 / kChunkSubs;
            const uint32_t ns = (uint32_t)(nsub - s0 < (uint64_t)kCTWarps ? nsub - s0 : (uint64_t)kCTWarps);
            if (!dense) mbar_wait_parity(&sh.mfull[st], ph);
            const SumMeta& M = sh.meta[st];
            const unsigned long long cpre = totals ? Pc : (dense ? 0ull : M.chk[chunk & 1]);
            const bool end_at_chunk = s0 + ns == nsub || (s0 + ns) % kChunkSubs == 0;
            const unsigned long long A =
                dense ? (unsigned long long)s0 * kWTInts : cpre + M.loc[0];
            const unsigned long long B =
                dense ? min((unsigned long long)n, (unsigned long long)(s0 + ns) * kWTInts)
                      : (end_at_chunk ? (totals ? Pc + Tc : M.chk[(chunk & 1) + 1]) : cpre + M.loc[ns]);
            if (totals && s0 + ns == nsub && lane == 0) {  // the stream's last tile: its length
                const uint64_t need = ngroups + B;
                if (need != in_len) dec_report(status, epoch, need > in_len ? BCGPU_ERR_TRUNCATED : BCGPU_ERR_TRAILING_BYTES);
            }
            const uint32_t li = (uint32_t)lane < ns ? (uint32_t)lane : ns;
            const unsigned long long my =
                (li == ns) ? B : (dense ? (unsigned long long)(s0 + li) * kWTInts : cpre + M.loc[li]);
            const uintptr_t Ag = data0 + A, Bg = data0 + B, bse = Ag & ~(uintptr_t)15;
            const uint32_t tx = tma_cover_bytes(Ag, Bg, lo, hi);
            const bool fits = tx != 0xFFFFFFFFu && tx + 16 <= pool_bytes;
            const uintptr_t cb = lo + s0 * kWTGroups;
            const uint64_t cg = ngroups - s0 * kWTGroups < (uint64_t)kTileCtrl ? ngroups - s0 * kWTGroups
                                                                                 : (uint64_t)kTileCtrl;
            const uint32_t ctx = tma_cover_bytes(cb, cb + cg, lo, hi);
            const bool c_tma = ctx != 0xFFFFFFFFu && (cb & 15) == 0;
            __syncwarp();
            if (k >= (uint32_t)kD1Stages) mbar_wait_parity_sleep(&sh.empty[st], ph ^ 1u);
            if (!c_tma)
                for (uint32_t i = lane; i < (uint32_t)cg; i += 32) sc[i] = __ldg(in + s0 * kWTGroups + i);
            if (lane <= 8) sh.hdr[st].head[lane] = (uint32_t)(data0 + my - bse);
            if (lane == 0) {
                sh.hdr[st].base = bse;
                sh.hdr[st].mode = fits ? 0u : 1u;
            }
            __syncwarp();
            if (lane == 0) {
                fence_async_smem();
                mbar_expect(&sh.full[st], (c_tma ? ctx : 0u) + (fits ? tx : 0u));
                const uint64_t pol = l2_policy_drop();
                if (kTrace) meta.trace[8ull * t + 0] = gtimer();
                if (c_tma && ctx) tma_load_hint(sc, reinterpret_cast<const void*>(cb), ctx, &sh.full[st], pol);
                if (fits && tx) tma_load_hint(pool, reinterpret_cast<const void*>(bse), tx, &sh.full[st], pol);
                const uint64_t tn = (uint64_t)t + (uint64_t)kD1Stages * G;
                if (tn < ntiles && !dense) issue_meta((uint32_t)tn, st);
            }
        }
        return;
    }
    // ---- consumers ----
    const int ct = threadIdx.x;  // 0..255
    // look-back window of tile tp: tiles max(0, tp - G + 1) .. tp - 1, read as 16-B aligned
    // pairs (2e, 2e + 1); each thread prefetches one pair, any more are read at resolve time
    auto window_lo = [&](uint32_t tp) -> uint32_t { return tp + 1 > G ? tp + 1 - G : 0u; };
    ulonglong2 pf = make_ulonglong2(0ull, 0ull);
    auto prefetch = [&](uint32_t tp) {
        const uint32_t e = (window_lo(tp) & ~1u) + 2u * (uint32_t)ct;
        if (e < tp) pf = ld_relaxed_u64x2(meta.agg + e);
    };
    auto entry = [&](uint32_t j, unsigned long long v) -> uint32_t {  // tile j's aggregate of this call
        while ((uint32_t)(v >> 32) != epoch) v = ld_relaxed_u64(meta.agg + j);
        return (uint32_t)v;
    };
    auto pair_sum = [&](uint32_t e, ulonglong2 v, uint32_t wl, uint32_t tp) -> uint32_t {
        uint32_t r = 0;
        if (e >= wl) r += entry(e, v.x);
        if (e + 1 < tp) r += entry(e + 1, v.y);
        return r;
    };
    // resolve tile tp (its sub-tile sums in wsum[q]), decode it from stage st with the carry,
    // store it and release the stage; zero: the sum pass found this warp's control bytes all 0
    auto resolve = [&](uint32_t tp, int st, int q, bool zero) {
        const uint32_t wl = window_lo(tp);
        uint32_t part = 0;
        const uint32_t e0 = (wl & ~1u) + 2u * (uint32_t)ct;
        if (e0 < tp) part += pair_sum(e0, pf, wl, tp);
        for (uint32_t e = e0 + 512; e < tp; e += 512) part += pair_sum(e, ld_relaxed_u64x2(meta.agg + e), wl, tp);
        part = __reduce_add_sync(kFull, part);
        if (lane == 0) sh.red[warp] = part;
        consumers_sync();
        if (kTrace && ct == 0) meta.trace[8ull * tp + 4] = gtimer();
        if (ct == 0) {
            uint32_t x = 0, a = 0;
#pragma unroll
            for (int w = 0; w < kCTWarps; ++w) {
                x += sh.red[w];
                a += sh.wsum[q][w];
            }
            const uint32_t c = (tp >= G ? sh.incl : base) + x;  // carry before tile tp
            sh.carry = c;
            sh.incl = c + a;
            uint32_t e = c;
#pragma unroll
            for (int w = 0; w < kCTWarps; ++w) {
                sh.wcarry[w] = e;
                e += sh.wsum[q][w];
            }
        }
        consumers_sync();
        const uint32_t s = tp * kCTWarps + warp;  // < 2^32: ntiles is 32-bit
        if (s < nsub) {
            const uint32_t E = sh.wcarry[warp];
            const uint64_t g0 = (uint64_t)s * kWTGroups;
            const uint8_t* sc = dsm + (uint32_t)st * stride + warp * kWTGroups;
            const uint8_t* pool = dsm + (uint32_t)st * stride + kTileCtrl;
            const uint32_t head = sh.hdr[st].head[warp];
            uint32_t* o = out + 4 * g0;
            uint32_t run;
            if (sh.hdr[st].mode == 0 && (uint64_t)(s + 1) * kWTInts <= n && head <= pool_bytes - 32 &&
                (((uintptr_t)o) & 15) == 0) {
                const uint32_t sd = sh_addr(pool) + head;
                if (zero) {
                    WarpCtrl wz;
                    run = expand_full<1, true>(wz, sd, o, E);
                } else {
                    bool z;
                    const WarpCtrl wf = ctrl_full(sh_addr(sc), &z);
                    run = expand_full<1, false>(wf, sd, o, E);
                }
            } else if (sh.hdr[st].mode == 0) {
                const uint32_t* W = reinterpret_cast<const uint32_t*>(pool);
                const uint32_t lim = pool_bytes / 4 - 1;
                run = decode_generic_store(sc, g0, ngroups, tail_r, head, [&](uint32_t i) { return W[i < lim ? i : lim]; },
                                           E, out);
            } else {
                const uintptr_t gb = (uintptr_t)sh.hdr[st].base;
                run = decode_generic_store(sc, g0, ngroups, tail_r, head,
                                           [&](uint32_t i) { return gword_guarded(gb + 4 * (uintptr_t)i, lo, hi); }, E,
                                           out);
            }
            if (d_last && s + 1 == nsub && lane == 0) *d_last = run;
        }
        __syncwarp();
        if (kTrace && ct == 0) meta.trace[8ull * tp + 5] = gtimer();
        if (lane == 0) mbar_arrive(&sh.empty[st]);  // tile tp is decoded: its stage is free
    };

    // the tile of iteration i is blockIdx.x + i * G; iteration k resolves iteration k - kD1Lag's
    uint32_t k = 0;
    const uint32_t b0 = blockIdx.x;
    uint32_t zbits = 0;  // bit i: the warp's sub-tile of iteration k - i had all-zero control bytes
    int st = 0, q = 0;  // stage and wsum slot of iteration k
    uint32_t ph = 0;
    for (uint32_t t = b0; t < ntiles;
         t += G, ++k, q = q == 2 ? 0 : q + 1, st = st + 1 == kD1Stages ? 0 : st + 1, ph ^= st == 0) {
        zbits <<= 1;
        if (k >= (uint32_t)kD1Lag) prefetch(t - kD1Lag * G);
        if (kTrace && ct == 0) meta.trace[8ull * t + 1] = gtimer();
        mbar_wait_parity(&sh.full[st], ph);
        if (kTrace && ct == 0) meta.trace[8ull * t + 2] = gtimer();
        const uint64_t s = (uint64_t)t * kCTWarps + warp;
        uint32_t sum = 0;
        bool checked = false;  // the control bytes were seen all zero (or reported)
        if (s < nsub) {
            const uint8_t* sc = dsm + (uint32_t)st * stride + warp * kWTGroups;
            const uint8_t* pool = dsm + (uint32_t)st * stride + kTileCtrl;
            const uint32_t head = sh.hdr[st].head[warp];
            const uint64_t g0 = s * kWTGroups;
            if (sh.hdr[st].mode == 0) {
                if ((s + 1) * kWTInts <= n && head <= pool_bytes - 32) {
                    const uint32_t sd = sh_addr(pool) + head;
                    if (ctrl_all_zero(sh_addr(sc))) {
                        checked = true;
                        zbits |= 1u;
                        sum = __reduce_add_sync(kFull, zero_tile_sum(sd));
                    } else {
                        checked = true;
                        if (dense && lane == 0) dec_report(status, epoch, BCGPU_ERR_TRUNCATED);
                        bool zero;
                        const WarpCtrl wf = ctrl_full(sh_addr(sc), &zero);
                        sum = __reduce_add_sync(kFull, expand_full<2, false>(wf, sd, nullptr, 0));
                    }
                } else {
                    const uint32_t* W = reinterpret_cast<const uint32_t*>(pool);
                    const uint32_t lim = pool_bytes / 4 - 1;
                    sum = sums_generic(sc, g0, ngroups, tail_r, head, [&](uint32_t i) { return W[i < lim ? i : lim]; });
                }
            } else {
                const uintptr_t gb = (uintptr_t)sh.hdr[st].base;
                sum = sums_generic(sc, g0, ngroups, tail_r, head,
                                   [&](uint32_t i) { return gword_guarded(gb + 4 * (uintptr_t)i, lo, hi); });
            }
        }
        if (dense && !checked && s < nsub) {  // every used control field of a dense stream must be 0
            const uint8_t* sc = dsm + (uint32_t)st * stride + warp * kWTGroups;
            const uint64_t g0 = s * kWTGroups;
            uint32_t orr = 0;
            for (uint64_t g = g0 + lane; g < ngroups && g < g0 + kWTGroups; g += 32) {
                uint32_t c = sc[g - g0];
                if (g + 1 == ngroups && tail_r) c &= (1u << (2 * tail_r)) - 1u;
                orr |= c;
            }
            if (__any_sync(kFull, orr != 0) && lane == 0) dec_report(status, epoch, BCGPU_ERR_TRUNCATED);
        }
        if (lane == 0) sh.wsum[q][warp] = sum;
        consumers_sync();
        if (ct == 0) {
            uint32_t a = 0;
#pragma unroll
            for (int w = 0; w < kCTWarps; ++w) a += sh.wsum[q][w];
            st_relaxed_u64(meta.agg + t, ((unsigned long long)epoch << 32) | a);
            if (kTrace) meta.trace[8ull * t + 3] = gtimer();
        }
        static_assert(kD1Lag == 2, "wsum ring of 3: iteration k - 2 uses slot q + 1 (mod 3)");
        if (k >= (uint32_t)kD1Lag)
            resolve(t - kD1Lag * G, st >= kD1Lag ? st - kD1Lag : st + kD1Stages - kD1Lag, q == 2 ? 0 : q + 1,
                    (zbits >> kD1Lag) & 1u);
    }
    for (uint32_t i = k > (uint32_t)kD1Lag ? k - kD1Lag : 0u; i < k; ++i) {
        prefetch(b0 + i * G);
        resolve(b0 + i * G, (int)(i % kD1Stages), (int)(i % 3), (zbits >> (k - 1 - i)) & 1u);
    }
}

static cudaError_t launch_decode1(const uint8_t* in, uint64_t in_len, uint64_t n, uint32_t base, uint32_t* out,
                                  uint32_t* d_last, const DecodeMeta& m, double dpb, uint32_t epoch, cudaStream_t stream,
                                  bool* used, unsigned long long* status = nullptr, uint32_t totals = 0,
                                  uint64_t* grid_only = nullptr) {
    *used = false;
    uint64_t pool = (uint64_t)(1.1 * dpb * kCTWarps) + 64;
    if (pool < 4096) pool = 4096;
    if (pool > 8ull * kWTDataMax + 64) pool = 8ull * kWTDataMax + 64;
    pool = (pool + 15) & ~15ull;
    const uint32_t smem = (uint32_t)(kD1Stages * (kCTWarps * kWTGroups + pool));
    const int dev = launch_current_device();
    const int sms = launch_sms(dev);
    if (!launch_coop(dev)) return cudaSuccess;
    cudaError_t a = launch_ensure_smem(svb_decode1_kernel<false>, 220 * 1024);
    if (a != cudaSuccess) return a;
    a = launch_ensure_smem(svb_decode1_kernel<true>, 220 * 1024);
    if (a != cudaSuccess) return a;
    const int occ = launch_occupancy(svb_decode1_kernel<false>, kSumThreads, smem);
    if (occ < 1) return cudaSuccess;  // caller falls back to the sums + delta passes
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint64_t ntiles = (nsub + kCTWarps - 1) / kCTWarps;
    uint64_t grid = (uint64_t)sms * (uint64_t)occ;
    if (grid > ntiles) grid = ntiles;
    if (grid_only) {  // query: the grid this stream would get
        *grid_only = grid;
        return cudaSuccess;
    }
    DecodeMeta mm = m;
    uint32_t pb = (uint32_t)pool;
    void* args[] = {(void*)&in, (void*)&in_len, (void*)&n,    (void*)&base,   (void*)&out,   (void*)&d_last,
                    (void*)&mm, (void*)&pb,     (void*)&epoch, (void*)&status, (void*)&totals};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kSumThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap the control scan's tail
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    const void* fn = m.trace ? (const void*)svb_decode1_kernel<true> : (const void*)svb_decode1_kernel<false>;
    const cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e == cudaSuccess) *used = true;
    return e;
}

// ---------------------------------------------------------------------------
// launcher
// ---------------------------------------------------------------------------
static inline uint64_t align16(uint64_t x) { return (x + 15) & ~(uint64_t)15; }

DecodeMeta carve_decode_meta(void* ws, uint64_t n) {
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint64_t nchunks = (nsub + kChunkSubs - 1) / kChunkSubs;
    uint8_t* p = static_cast<uint8_t*>(ws);
    DecodeMeta m;
    m.trace = nullptr;
    m.counters = reinterpret_cast<unsigned int*>(p);  // 16 B, persists across calls (self-resetting)
    m.running = reinterpret_cast<unsigned long long*>(p + 16);
    p += 32;
    m.localpre = reinterpret_cast<uint32_t*>(p);
    p += align16(4 * (nsub + 64));
    m.chunkpre = reinterpret_cast<unsigned long long*>(p);
    p += align16(8 * (nchunks + 4));
    m.subsums = reinterpret_cast<uint32_t*>(p);
    p += align16(4 * nsub);
    m.chunksums = reinterpret_cast<uint32_t*>(p);
    p += align16(4 * (nchunks + 1));
    m.chunktot = reinterpret_cast<uint32_t*>(p);
    p += align16(4 * (nchunks + 1));
    m.tilesize = reinterpret_cast<uint32_t*>(p);
    const uint64_t ntiles = (nsub + kCTWarps - 1) / kCTWarps;
    p += align16(4 * (ntiles + 8));
    m.agg = reinterpret_cast<unsigned long long*>(p);
    return m;
}

uint64_t decode_meta_bytes(uint64_t n) {
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint64_t nchunks = (nsub + kChunkSubs - 1) / kChunkSubs;
    const uint64_t ntiles = (nsub + kCTWarps - 1) / kCTWarps;
    return 32 + align16(4 * (nsub + 64)) + align16(8 * (nchunks + 4)) + align16(4 * nsub) +
           2 * align16(4 * (nchunks + 1)) + align16(4 * (ntiles + 8)) + align16(8 * ((nsub + 3) / 4 + 8)) + 64;
}

int occupancy_decode_pipe() { return 1; }  // the tile kernel is not persistent

// pipelined sums pass: stage pool from the stream's average density, grid = SMs x resident CTAs
static cudaError_t launch_sums(const uint8_t* in, uint64_t in_len, uint64_t n, const DecodeMeta& m, double dpb,
                               uint32_t t_begin, uint32_t t_end, cudaStream_t stream) {
    uint64_t pool = (uint64_t)(1.1 * dpb * kCTWarps) + 64;
    if (pool < 4096) pool = 4096;
    if (pool > 8ull * kWTDataMax + 64) pool = 8ull * kWTDataMax + 64;
    pool = (pool + 15) & ~15ull;
    const uint32_t smem = (uint32_t)(kSumStages * (kCTWarps * kWTGroups + pool));
    const int sms = launch_sms(launch_current_device());
    const cudaError_t a = launch_ensure_smem(svb_sums_kernel<kSumStages>, 200 * 1024);
    if (a != cudaSuccess) return a;
    int occ = launch_occupancy(svb_sums_kernel<kSumStages>, kSumThreads, smem);
    if (occ < 1) occ = 1;
    if (t_end <= t_begin) return cudaSuccess;
    uint64_t grid = (uint64_t)sms * (uint64_t)occ;
    if (grid > t_end - t_begin) grid = t_end - t_begin;
    svb_sums_kernel<kSumStages><<<(unsigned)grid, kSumThreads, smem, stream>>>(in, in_len, n, m, (uint32_t)pool,
                                                                               t_begin, t_end);
    return cudaGetLastError();
}

// decode pass 1 over the whole stream (control bytes only); zeroes the chunk sums for delta
cudaError_t launch_decode_ctrl(const uint8_t* in, uint64_t in_len, uint64_t n, int delta, void* meta_ws,
                               unsigned long long* status, uint32_t epoch, cudaStream_t stream) {
    const DecodeMeta m = carve_decode_meta(meta_ws, n);
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint32_t nchunks = (uint32_t)((nsub + kChunkSubs - 1) / kChunkSubs);
    svb_ctrl_scan_kernel<<<nchunks, 256, 0, stream>>>(in, in_len, n, m, status, epoch, delta);
    return cudaGetLastError();
}

// Decode passes 2-3 for sub-tiles [sub_begin, sub_end) (multiples of a 64-sub-tile chunk,
// except at the stream's end), after launch_decode_ctrl.  Delta ranges must be issued in
// order on one stream (each continues the previous range's carry).
cudaError_t launch_decode_range(const uint8_t* in, uint64_t in_len, uint64_t n, int delta, uint32_t base,
                                uint32_t* out, uint32_t* d_last, void* meta_ws, uint64_t sub_begin, uint64_t sub_end,
                                cudaStream_t stream, int* launches, unsigned long long* trace, uint32_t epoch,
                                unsigned long long* status, uint32_t totals) {
    DecodeMeta m = carve_decode_meta(meta_ws, n);
    m.trace = trace;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    if (sub_end > nsub) sub_end = nsub;
    *launches = 0;
    if (sub_begin >= sub_end) return cudaSuccess;
    // pooled decode: K sub-tiles per warp and the pool from the stream's average density
    const double dpb = nsub ? (double)(in_len > ngroups ? in_len - ngroups : 0) / (double)nsub : 0.0;  // B / sub-tile
    const int K = dpb < 1400.0 ? 4 : 2;
    const uint32_t S = (uint32_t)(kCTWarps * K);
    uint64_t pool = (uint64_t)(1.2 * dpb * S) + 64;
    const uint64_t round_max = 8ull * kWTDataMax + 64;  // one round, worst case
    if (pool < round_max) pool = round_max;
    if (pool > 160 * 1024) pool = 160 * 1024;
    pool = (pool + 15) & ~15ull;
    const uint32_t smem = (uint32_t)(S * kWTGroups + pool);
    const int pgrid = (int)((sub_end - sub_begin + S - 1) / S);
#define BC_POOL_LAUNCH(MODE, KK)                                                                                 \
    do {                                                                                                         \
        const cudaError_t a_ = launch_ensure_smem(svb_decode_pool_kernel<MODE, KK>, 200 * 1024);                \
        if (a_ != cudaSuccess) return a_;                                                                        \
        svb_decode_pool_kernel<MODE, KK><<<pgrid, kCTThreads, smem, stream>>>(in, in_len, n, base, out, d_last, m,  \
                                                                             (uint32_t)pool, sub_begin);        \
    } while (0)
    if (delta && sub_begin == 0 && sub_end == nsub && epoch) {
        bool used = false;
        const cudaError_t e1 = launch_decode1(in, in_len, n, base, out, d_last, m, dpb, epoch, stream, &used, status,
                                              totals);
        if (e1 != cudaSuccess) return e1;
        if (used) {
            *launches = 1;
            return cudaSuccess;
        }
    }
    if (totals) return cudaErrorInvalidValue;  // the chunk offsets were left unscanned for the one-pass decode
    if (delta) {
        const uint32_t t0 = (uint32_t)(sub_begin / kCTWarps), t1 = (uint32_t)((sub_end + kCTWarps - 1) / kCTWarps);
        const cudaError_t e2 = launch_sums(in, in_len, n, m, dpb, t0, t1, stream);
        if (e2 != cudaSuccess) return e2;
        if (K == 4) BC_POOL_LAUNCH(kModeDelta, 4);
        else BC_POOL_LAUNCH(kModeDelta, 2);
        *launches = 2;
    } else {
        if (K == 4) BC_POOL_LAUNCH(kModePlain, 4);
        else BC_POOL_LAUNCH(kModePlain, 2);
        *launches = 1;
    }
#undef BC_POOL_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_decode3(const uint8_t* in, uint64_t in_len, uint64_t n, int delta, uint32_t base, uint32_t* out,
                           uint32_t* d_last, void* meta_ws, unsigned long long* status, uint32_t epoch, int pipe_grid,
                           cudaStream_t stream, int* launches, unsigned long long* trace, uint32_t debug_flags) {
    (void)pipe_grid;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint32_t ep = (debug_flags & 1024) ? 0u : epoch;
    // a dense delta stream (ceil(n/4) + n bytes: every integer one byte) needs no control
    // scan: the one-pass decode computes the implicit offsets and checks the control bytes
    // (debug flag 0x400000: always scan); its tile aggregates must hold no current tag
    if (delta && ep && in_len == ngroups + n && !(debug_flags & (0x400000 | 0x8000 | 0x40000))) {
        const DecodeMeta m = carve_decode_meta(meta_ws, n);
        if (!(debug_flags & 0x800000)) {  // 0x800000: the caller knows the aggregates are clean
            uint64_t cnt = 0;
            unsigned long long* agg = meta_agg_ptr(meta_ws, n, &cnt);
            const cudaError_t ce = cudaMemsetAsync(agg, 0, cnt * sizeof(unsigned long long), stream);
            if (ce != cudaSuccess) return ce;
        }
        bool used = false;
        const double dpb = 1024.0;
        DecodeMeta mm = m;
        mm.trace = trace;
        const cudaError_t e1 = launch_decode1(in, in_len, n, base, out, d_last, mm, dpb, ep, stream, &used, status, 2u);
        if (e1 != cudaSuccess) return e1;
        if (used) {
            *launches = 1;
            return cudaSuccess;
        }
    }
    // the one-pass delta decode sums the chunk totals itself (grid <= 504: a CTA's chunks
    // advance by <= 64 per tile), so the control scan can skip its last-CTA scan
    uint32_t totals = 0;
    if (delta && ep && !(debug_flags & (0x8000 | 0x40000))) {
        const double dpb = nsub ? (double)(in_len > ngroups ? in_len - ngroups : 0) / (double)nsub : 0.0;
        uint64_t g1 = 0;
        bool used = false;
        const cudaError_t q = launch_decode1(in, in_len, n, base, out, d_last, carve_decode_meta(meta_ws, n), dpb, ep,
                                             stream, &used, status, 0, &g1);
        if (q != cudaSuccess) return q;
        totals = g1 >= 1 && g1 <= 504 ? 1u : 0u;
    }
    cudaError_t e = launch_decode_ctrl(in, in_len, n, delta | (totals ? 2 : 0), meta_ws, status, epoch, stream);
    if (e != cudaSuccess) return e;
    if (debug_flags & 0x8000) {  // dev timing: the control scan alone
        *launches = 1;
        return cudaSuccess;
    }
    int l = 0;
    e = launch_decode_range(in, in_len, n, delta, base, out, d_last, meta_ws, 0, nsub, stream, &l, trace, ep, status,
                            totals);
    *launches = 1 + l;
    return e;
}

// device address and size of the one-pass tile aggregates for an n-integer stream
unsigned long long* meta_agg_ptr(void* meta_ws, uint64_t n, uint64_t* count) {
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    *count = (nsub + 3) / 4;  // tiles of >= 4 sub-tiles (the one-pass encode's tile is a build constant)
    return carve_decode_meta(meta_ws, n).agg;
}

// the sums pass over the whole stream (after launch_decode_ctrl): per-sub-tile sums and
// scanned per-chunk carries in the workspace (batched seek / select, svb_query.cu)
cudaError_t launch_decode_sums(const uint8_t* in, uint64_t in_len, uint64_t n, void* meta_ws, cudaStream_t stream) {
    const DecodeMeta m = carve_decode_meta(meta_ws, n);
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const double dpb = nsub ? (double)(in_len > ngroups ? in_len - ngroups : 0) / (double)nsub : 0.0;
    return launch_sums(in, in_len, n, m, dpb, 0, (uint32_t)((nsub + kCTWarps - 1) / kCTWarps), stream);
}

// device address of the chunk offsets (nchunks + 1 entries, after launch_decode_ctrl)
unsigned long long* decode_chunkpre_ptr(void* meta_ws, uint64_t n) { return carve_decode_meta(meta_ws, n).chunkpre; }

}  // namespace bcgpu
