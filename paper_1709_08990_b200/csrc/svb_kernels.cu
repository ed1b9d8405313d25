// svb_kernels.cu -- sm_100a kernels for Stream VByte encode / decode / delta.
//
// Reference behaviour restated (paths under /root/reference):
//   svb_encode        proj/core/include/bytecodec/stream_vbyte.hpp:36
//   svb_decode        stream_vbyte.hpp:38-39
//   svb_decode_delta  stream_vbyte.hpp:41-42, codec.hpp:87-90
//   delta encode      codec.hpp:92-93 (base 0) + extension E2 (prev seed) SPEC.md:366-374
//   block offsets     stream_vbyte.hpp:48-49
//   chained chunks    codec.hpp:87-90, SPEC.md:555 (segmented batches)
//
// Kernel families:
//   * single array  -- one CTA per tile of kTileInts integers, tile order from
//     an atomic ticket, byte offsets (and delta carries) by decoupled look-back.
//   * batch / CTA   -- one CTA per large segment, tiles walked in order with the
//     offset and carry kept in registers (no look-back).
//   * batch / warp  -- one warp per small segment, 128 control bytes per step.
#include <cstdint>

#include "svb_device.cuh"
#include "svb_kernels.cuh"

namespace bcgpu {

struct TileResult {
    uint64_t off;    // exclusive data offset of the tile
    uint32_t total;  // data bytes of the tile
    uint32_t carry;  // delta: value before the tile's first integer
    uint32_t sum;    // delta: sum of the tile's deltas (mod 2^32)
};

struct DecodeSmem {
    uint32_t ctrl_w[kTileGroups / 4];  // the tile's control bytes
    uint16_t off[kTileGroups];         // tile-local data offset of every control byte
    uint32_t warp_tot[kWarps];
    uint32_t chunk[kRows * kWarps];
    unsigned long long bcast[2];
};

struct EncodeSmem {
    uint32_t chunk[kRows * kWarps];
    unsigned long long bcast;
    uint32_t total;
};

__device__ __forceinline__ void report_status(unsigned long long* st, uint32_t epoch, uint32_t code) {
    if (st) *st = ((unsigned long long)epoch << 32) | code;
}

// Row-major exclusive scan of one value per (row j, thread) over the tile
// order k = j*kThreads + tid.  ex[j] receives the exclusive prefix within the
// thread's warp-row chunk; chunk[] the chunk prefixes; returns the tile total.
// Contains one __syncthreads; the chunk prefixes are valid after a second one.
__device__ __forceinline__ void row_scan_part1(const uint32_t (&val)[kRows], uint32_t (&ex)[kRows],
                                               uint32_t* chunk) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
        const uint32_t incl = warp_inclusive_scan(val[j]);
        ex[j] = incl - val[j];
        if (lane == 31) chunk[j * kWarps + warp] = incl;
    }
    __syncthreads();
}

// warp 0 only: turn chunk totals into exclusive chunk prefixes, return the tile total.
__device__ __forceinline__ uint32_t row_scan_part2(uint32_t* chunk) {
    static_assert(kRows * kWarps == 64, "two chunks per lane");
    const int lane = threadIdx.x & 31;
    const uint32_t a = chunk[2 * lane], b = chunk[2 * lane + 1];
    const uint32_t pair = a + b;
    const uint32_t pin = warp_inclusive_scan(pair);
    chunk[2 * lane] = pin - pair;
    chunk[2 * lane + 1] = pin - pair + a;
    return __shfl_sync(kFull, pin, 31);
}

// ===========================================================================
// decode tile
// ===========================================================================
template <bool kDelta, class OffsetFn, class CarryFn>
__device__ __forceinline__ TileResult decode_tile(const uint8_t* __restrict__ seg, uint64_t seg_len, uint64_t ngroups,
                                                  uint32_t tail_r, uint64_t g0, uint32_t* __restrict__ out,
                                                  DecodeSmem& sh, uint8_t* __restrict__ stage, OffsetFn&& offset_fn,
                                                  CarryFn&& carry_fn) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t rem = ngroups - g0;
    const uint32_t tile_groups = rem < (uint64_t)kTileGroups ? (uint32_t)rem : (uint32_t)kTileGroups;

    // ---- phase A: control bytes -> lengths -> block scan -> tile offset
    const Ctrl8 cb = load_ctrl8(seg, g0 + (uint64_t)tid * kRows, ngroups, tail_r);
    const uint32_t len_lo = (uint32_t)cb.len, len_hi = (uint32_t)(cb.len >> 32);
    const uint32_t ex_lo = len_lo * 0x01010100u, ex_hi = len_hi * 0x01010100u;
    const uint32_t tot_lo = (len_lo * 0x01010101u) >> 24, tot_hi = (len_hi * 0x01010101u) >> 24;
    const uint32_t thr_tot = tot_lo + tot_hi;
    const uint32_t incl = warp_inclusive_scan(thr_tot);
    if (lane == 31) sh.warp_tot[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t t = sh.warp_tot[w];
        wpre += (w < warp) ? t : 0u;
        total += t;
    }
    const uint32_t thr_ex = wpre + incl - thr_tot;
    if (warp == 0) {
        const uint64_t off = offset_fn(total);
        if (lane == 0) sh.bcast[0] = off;
    }
    sh.ctrl_w[2 * tid] = (uint32_t)cb.c;
    sh.ctrl_w[2 * tid + 1] = (uint32_t)(cb.c >> 32);
#pragma unroll
    for (int i = 0; i < 4; ++i) sh.off[tid * kRows + i] = (uint16_t)(thr_ex + ((ex_lo >> (8 * i)) & 0xFFu));
#pragma unroll
    for (int i = 0; i < 4; ++i)
        sh.off[tid * kRows + 4 + i] = (uint16_t)(thr_ex + tot_lo + ((ex_hi >> (8 * i)) & 0xFFu));
    __syncthreads();
    const uint64_t tile_off = sh.bcast[0];

    // ---- phase B: stage the tile's data bytes [beg, end) into shared memory
    const uintptr_t lo_ok = (uintptr_t)seg, hi_ok = (uintptr_t)seg + seg_len;
    const uintptr_t beg = (uintptr_t)(seg + ngroups) + tile_off, end = beg + total;
    const uintptr_t a0 = beg & ~(uintptr_t)15, a1 = (end + 15) & ~(uintptr_t)15;
    const uint32_t nchunks = (uint32_t)((a1 - a0) >> 4);
    constexpr int kU = 6;
    for (uint32_t c0 = tid; c0 < nchunks; c0 += kU * kThreads) {
        uint4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t c = c0 + u * kThreads;
            if (c < nchunks) v[u] = load_chunk_guarded(a0 + 16 * (uintptr_t)c, lo_ok, hi_ok);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t c = c0 + u * kThreads;
            if (c < nchunks) *reinterpret_cast<uint4*>(stage + 16 * c) = v[u];
        }
    }
    __syncthreads();

    // ---- phase C: expand, (delta: scan), store
    const uint32_t head = (uint32_t)(beg - a0);
    const uint32_t* W = reinterpret_cast<const uint32_t*>(stage);
    const uint8_t* cbytes = reinterpret_cast<const uint8_t*>(sh.ctrl_w);
    const bool out16 = (((uintptr_t)out) & 15) == 0;
    uint4 vv[kDelta ? kRows : 1];
    uint32_t cnts[kDelta ? kRows : 1];
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
        const uint32_t k = j * kThreads + tid;
        const bool valid = k < tile_groups;
        const uint32_t c = valid ? cbytes[k] : 0u;
        const uint32_t b = head + (valid ? (uint32_t)sh.off[k] : 0u);
        const bool allzero = __all_sync(kFull, c == 0);
        uint4 v = allzero ? decode_zero_group(W, b) : decode_group(W, b, c);
        const uint64_t gi = g0 + k;
        const uint32_t cnt = valid ? ((gi == ngroups - 1 && tail_r) ? tail_r : 4u) : 0u;
        if constexpr (!kDelta) {
            if (cnt) store_group(out + 4 * gi, v, cnt, out16);
        } else {
            vv[j] = prefix4(mask_tail(v, cnt));
            cnts[j] = cnt;
        }
    }
    TileResult r{tile_off, total, 0u, 0u};
    if constexpr (kDelta) {
        uint32_t S[kRows], ex[kRows];
#pragma unroll
        for (int j = 0; j < kRows; ++j) S[j] = vv[j].w;
        row_scan_part1(S, ex, sh.chunk);
        if (warp == 0) {
            const uint32_t tsum = row_scan_part2(sh.chunk);
            const uint32_t carry = carry_fn(tsum);
            if (lane == 0) sh.bcast[1] = ((unsigned long long)tsum << 32) | carry;
        }
        __syncthreads();
        const unsigned long long bc = sh.bcast[1];
        r.carry = (uint32_t)bc;
        r.sum = (uint32_t)(bc >> 32);
#pragma unroll
        for (int j = 0; j < kRows; ++j) {
            const uint32_t k = j * kThreads + tid;
            if (cnts[j]) {
                const uint4 v = add4(vv[j], r.carry + sh.chunk[j * kWarps + warp] + ex[j]);
                store_group(out + 4 * (g0 + k), v, cnts[j], out16);
            }
        }
    }
    return r;
}

// ===========================================================================
// encode tile
// ===========================================================================
template <bool kDelta, class OffsetFn>
__device__ __forceinline__ TileResult encode_tile(const uint32_t* __restrict__ in, uint32_t prev, uint64_t ngroups,
                                                  uint32_t tail_r, uint64_t g0, uint8_t* __restrict__ out,
                                                  EncodeSmem& sh, uint8_t* __restrict__ stage, OffsetFn&& offset_fn) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t rem = ngroups - g0;
    const uint32_t tile_groups = rem < (uint64_t)kTileGroups ? (uint32_t)rem : (uint32_t)kTileGroups;
    const bool in16 = (((uintptr_t)in) & 15) == 0;

    uint4 d[kRows];
    uint32_t lens[kRows], L[kRows];
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
        const uint32_t k = j * kThreads + tid;
        const uint64_t gi = g0 + k;
        const uint32_t cnt = k < tile_groups ? ((gi == ngroups - 1 && tail_r) ? tail_r : 4u) : 0u;
        uint4 x = make_uint4(0, 0, 0, 0);
        if (cnt == 4 && in16) {
            x = ldg_stream_v4(in + 4 * gi);
        } else if (cnt) {
            x.x = __ldg(in + 4 * gi);
            if (cnt > 1) x.y = __ldg(in + 4 * gi + 1);
            if (cnt > 2) x.z = __ldg(in + 4 * gi + 2);
            if (cnt > 3) x.w = __ldg(in + 4 * gi + 3);
        }
        if constexpr (kDelta) {
            uint32_t p = __shfl_up_sync(kFull, x.w, 1);
            if (lane == 0) p = (gi == 0) ? prev : (cnt ? __ldg(in + 4 * gi - 1) : 0u);
            x = make_uint4(x.x - p, x.y - x.x, x.z - x.y, x.w - x.z);
        }
        d[j] = x;
        const uint32_t l0 = cnt > 0 ? dev_byte_length(x.x) : 0u;
        const uint32_t l1 = cnt > 1 ? dev_byte_length(x.y) : 0u;
        const uint32_t l2 = cnt > 2 ? dev_byte_length(x.z) : 0u;
        const uint32_t l3 = cnt > 3 ? dev_byte_length(x.w) : 0u;
        lens[j] = l0 | (l1 << 8) | (l2 << 16) | (l3 << 24);
        L[j] = l0 + l1 + l2 + l3;
        if (cnt) {
            const uint32_t c = ((l0 - 1) & 3u) | (l1 ? ((l1 - 1) << 2) : 0u) | (l2 ? ((l2 - 1) << 4) : 0u) |
                               (l3 ? ((l3 - 1) << 6) : 0u);
            out[gi] = (uint8_t)c;
        }
    }
    uint32_t ex[kRows];
    row_scan_part1(L, ex, sh.chunk);
    if (warp == 0) {
        const uint32_t total = row_scan_part2(sh.chunk);
        const uint64_t off = offset_fn(total);
        if (lane == 0) {
            sh.bcast = off;
            sh.total = total;
        }
    }
    __syncthreads();
    const uint64_t tile_off = sh.bcast;
    const uint32_t total = sh.total;

    const uintptr_t beg = (uintptr_t)(out + ngroups) + tile_off, end = beg + total;
    const uintptr_t a0 = beg & ~(uintptr_t)15, a1 = (end + 15) & ~(uintptr_t)15;
    const uint32_t head = (uint32_t)(beg - a0);
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
        if (L[j]) {
            uint32_t p = head + sh.chunk[j * kWarps + warp] + ex[j];
            const uint32_t l = lens[j];
            put_int_bytes(stage, p, d[j].x, l & 0xFF);
            p += l & 0xFF;
            if ((l >> 8) & 0xFF) put_int_bytes(stage, p, d[j].y, (l >> 8) & 0xFF);
            p += (l >> 8) & 0xFF;
            if ((l >> 16) & 0xFF) put_int_bytes(stage, p, d[j].z, (l >> 16) & 0xFF);
            p += (l >> 16) & 0xFF;
            if (l >> 24) put_int_bytes(stage, p, d[j].w, l >> 24);
        }
    }
    __syncthreads();
    const uint32_t nchunks = (uint32_t)((a1 - a0) >> 4);
    for (uint32_t c = tid; c < nchunks; c += kThreads) {
        const uintptr_t a = a0 + 16 * (uintptr_t)c;
        if (a >= beg && a + 16 <= end) {
            stg_stream_v4(reinterpret_cast<void*>(a), *reinterpret_cast<const uint4*>(stage + 16 * c));
        } else {
            for (int b = 0; b < 16; ++b)
                if (a + b >= beg && a + b < end) *reinterpret_cast<uint8_t*>(a + b) = stage[16 * c + b];
        }
    }
    __syncthreads();  // stage / chunk reuse by a following tile of the same CTA
    return TileResult{tile_off, total, 0u, 0u};
}

// ===========================================================================
// single-array kernels (decoupled look-back)
// ===========================================================================
__device__ __forceinline__ uint32_t take_ticket(const LookbackArgs& lb, uint32_t* s_tile) {
    if (threadIdx.x == 0) *s_tile = (uint32_t)(atomicAdd(lb.ticket, 1ull) - lb.ticket_base);
    __syncthreads();
    return *s_tile;
}

struct LookbackFn {
    uint64_t* status;
    uint32_t tile, epoch;
    uint64_t seed;  // value before tile 0 (0 for offsets, base for delta)
    __device__ __forceinline__ uint64_t operator()(uint64_t agg) const {
        const int lane = threadIdx.x & 31;
        if (tile == 0) {
            if (lane == 0) st_relaxed_gpu(status, pack_status(epoch, kFlagInclusive, seed + agg));
            return seed;
        }
        if (lane == 0) st_relaxed_gpu(status + tile, pack_status(epoch, kFlagAggregate, agg));
        const uint64_t ex = lookback_exclusive(status, tile, epoch);
        if (lane == 0) st_relaxed_gpu(status + tile, pack_status(epoch, kFlagInclusive, ex + agg));
        return ex;
    }
};

template <bool kDelta>
__global__ void __launch_bounds__(kThreads) svb_decode_kernel(const uint8_t* __restrict__ in, uint64_t in_len,
                                                              uint64_t n, uint32_t base, uint32_t* __restrict__ out,
                                                              uint32_t* __restrict__ d_last, LookbackArgs lb) {
    extern __shared__ __align__(16) uint8_t stage[];
    __shared__ DecodeSmem sh;
    __shared__ uint32_t s_tile;
    const uint32_t tile = take_ticket(lb, &s_tile);
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    LookbackFn off_fn{lb.off_status, tile, lb.epoch, 0};
    LookbackFn sum_fn{lb.sum_status, tile, lb.epoch, base};
    const TileResult r = decode_tile<kDelta>(
        in, in_len, ngroups, tail_r, (uint64_t)tile * kTileGroups, out, sh, stage,
        [&](uint32_t agg) { return off_fn(agg); }, [&](uint32_t agg) { return (uint32_t)sum_fn(agg); });
    if (tile == lb.num_tiles - 1 && threadIdx.x == 0) {
        const uint64_t need = ngroups + r.off + r.total;
        const uint32_t code = need > in_len ? BCGPU_ERR_TRUNCATED : (need < in_len ? BCGPU_ERR_TRAILING_BYTES : 0u);
        report_status(lb.status, lb.epoch, code);
        if (kDelta && d_last) *d_last = r.carry + r.sum;
    }
}

template <bool kDelta>
__global__ void __launch_bounds__(kThreads) svb_encode_kernel(const uint32_t* __restrict__ in, uint64_t n,
                                                              uint32_t prev, uint8_t* __restrict__ out,
                                                              uint64_t* __restrict__ d_out_len, LookbackArgs lb) {
    extern __shared__ __align__(16) uint8_t stage[];
    __shared__ EncodeSmem sh;
    __shared__ uint32_t s_tile;
    const uint32_t tile = take_ticket(lb, &s_tile);
    const uint64_t ngroups = (n + 3) >> 2;
    LookbackFn off_fn{lb.off_status, tile, lb.epoch, 0};
    const TileResult r = encode_tile<kDelta>(in, prev, ngroups, (uint32_t)(n & 3), (uint64_t)tile * kTileGroups, out,
                                             sh, stage, [&](uint32_t agg) { return off_fn(agg); });
    if (tile == lb.num_tiles - 1 && threadIdx.x == 0) {
        if (d_out_len) *d_out_len = ngroups + r.off + r.total;
        report_status(lb.status, lb.epoch, 0u);
    }
}

__global__ void __launch_bounds__(kThreads) svb_block_offsets_kernel(const uint8_t* __restrict__ in, uint64_t n,
                                                                     uint64_t* __restrict__ offsets, LookbackArgs lb) {
    __shared__ uint32_t warp_tot[kWarps];
    __shared__ unsigned long long bcast;
    __shared__ uint32_t s_tile;
    const uint32_t tile = take_ticket(lb, &s_tile);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t g = (uint64_t)tile * kTileGroups + (uint64_t)tid * kRows;
    const Ctrl8 cb = load_ctrl8(in, g, ngroups, (uint32_t)(n & 3));
    const uint32_t len_lo = (uint32_t)cb.len, len_hi = (uint32_t)(cb.len >> 32);
    const uint32_t tot_lo = (len_lo * 0x01010101u) >> 24, tot_hi = (len_hi * 0x01010101u) >> 24;
    const uint32_t thr_tot = tot_lo + tot_hi;
    const uint32_t incl = warp_inclusive_scan(thr_tot);
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        wpre += (w < warp) ? warp_tot[w] : 0u;
        total += warp_tot[w];
    }
    if (warp == 0) {
        LookbackFn fn{lb.off_status, tile, lb.epoch, 0};
        const uint64_t off = fn(total);
        if (lane == 0) bcast = off;
    }
    __syncthreads();
    uint64_t o = bcast + wpre + incl - thr_tot;
#pragma unroll
    for (int i = 0; i < kRows; ++i) {
        if (g + i < ngroups) offsets[g + i] = o;
        o += (cb.len >> (8 * i)) & 0xFF;
    }
    if (tile == lb.num_tiles - 1 && tid == 0) report_status(lb.status, lb.epoch, 0u);
}

// Random-access block decode (stream_vbyte.hpp:51-54), one thread per query.
__global__ void __launch_bounds__(kThreads) svb_decode_blocks_kernel(const uint8_t* __restrict__ in, uint64_t in_len,
                                                                     uint64_t n, const uint64_t* __restrict__ blocks,
                                                                     const uint64_t* __restrict__ offsets,
                                                                     uint64_t nblocks, uint32_t* __restrict__ out,
                                                                     uint32_t* __restrict__ counts) {
    const uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    if (i >= nblocks) return;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t k = blocks[i];
    uint32_t v[4] = {0, 0, 0, 0};
    uint32_t cnt = 0;
    if (k < ngroups && k < in_len) {
        cnt = (k == ngroups - 1 && (n & 3)) ? (uint32_t)(n & 3) : 4u;
        const uint32_t c = __ldg(in + k);
        uint64_t p = ngroups + offsets[i];
        for (uint32_t f = 0; f < cnt; ++f) {
            const uint32_t l = ((c >> (2 * f)) & 3u) + 1u;
            uint32_t x = 0;
            for (uint32_t b = 0; b < l; ++b)
                if (p + b < in_len) x |= (uint32_t)__ldg(in + p + b) << (8 * b);
            v[f] = x;
            p += l;
        }
    }
    out[4 * i + 0] = v[0];
    out[4 * i + 1] = v[1];
    out[4 * i + 2] = v[2];
    out[4 * i + 3] = v[3];
    counts[i] = cnt;
}

// ===========================================================================
// batch kernels
// ===========================================================================
struct SegDesc {
    uint64_t a, b, c;
    uint32_t n, prev;
};

__device__ __forceinline__ SegDesc load_desc_warp(const void* segs, uint64_t s) {
    const int lane = threadIdx.x & 31;
    const unsigned long long* p = reinterpret_cast<const unsigned long long*>(segs) + 4 * s;
    const unsigned long long w = lane < 4 ? __ldg(p + lane) : 0ull;
    SegDesc d;
    d.a = __shfl_sync(kFull, w, 0);
    d.b = __shfl_sync(kFull, w, 1);
    d.c = __shfl_sync(kFull, w, 2);
    const unsigned long long np = __shfl_sync(kFull, w, 3);
    d.n = (uint32_t)np;
    d.prev = (uint32_t)(np >> 32);
    return d;
}

// -------- decode, CTA per segment (tiles walked in order)
template <bool kDelta>
__global__ void __launch_bounds__(kThreads) svb_decode_batch_cta_kernel(const bcgpu_decode_segment* __restrict__ segs,
                                                                        uint64_t nseg, const uint8_t* __restrict__ in,
                                                                        uint32_t* __restrict__ out, uint32_t min_n,
                                                                        unsigned long long* status, uint32_t epoch) {
    extern __shared__ __align__(16) uint8_t stage[];
    __shared__ DecodeSmem sh;
    for (uint64_t s = blockIdx.x; s < nseg; s += gridDim.x) {
        const bcgpu_decode_segment d = segs[s];
        if (d.n < min_n) continue;
        const uint64_t ngroups = ((uint64_t)d.n + 3) >> 2;
        if (d.src_bytes < ngroups) {
            if (threadIdx.x == 0) report_status(status, epoch, BCGPU_ERR_TRUNCATED);
            continue;
        }
        const uint8_t* seg = in + d.src_offset;
        uint32_t* o = out + d.dst_offset;
        uint64_t run_off = 0;
        uint32_t run_carry = d.prev;
        for (uint64_t g0 = 0; g0 < ngroups; g0 += kTileGroups) {
            const TileResult r = decode_tile<kDelta>(
                seg, d.src_bytes, ngroups, d.n & 3u, g0, o, sh, stage, [&](uint32_t) { return run_off; },
                [&](uint32_t) { return run_carry; });
            run_off = r.off + r.total;
            run_carry = r.carry + r.sum;
            __syncthreads();  // shared tile state reused by the next tile
        }
        if (threadIdx.x == 0 && ngroups + run_off != d.src_bytes)
            report_status(status, epoch, ngroups + run_off > d.src_bytes ? BCGPU_ERR_TRUNCATED : BCGPU_ERR_TRAILING_BYTES);
    }
}

// -------- decode, warp per segment
template <bool kDelta>
__device__ __forceinline__ void decode_segment_warp(const uint8_t* __restrict__ seg, uint64_t seg_len, uint32_t n,
                                                    uint32_t prev, uint32_t* __restrict__ out, uint8_t* stage,
                                                    unsigned long long* status, uint32_t epoch) {
    const int lane = threadIdx.x & 31;
    const uint64_t ngroups = ((uint64_t)n + 3) >> 2;
    const uint32_t tail_r = n & 3u;
    if (seg_len < ngroups) {
        if (lane == 0) report_status(status, epoch, BCGPU_ERR_TRUNCATED);
        return;
    }
    const uintptr_t lo_ok = (uintptr_t)seg, hi_ok = (uintptr_t)seg + seg_len;
    const uintptr_t data = (uintptr_t)seg + ngroups;
    const bool out16 = (((uintptr_t)out) & 15) == 0;
    const uint32_t* W = reinterpret_cast<const uint32_t*>(stage);
    uint64_t off = 0;
    uint32_t carry = prev;
    for (uint64_t gb = 0; gb < ngroups; gb += kWarpStepGroups) {
        uint32_t c[kWarpRows], len[kWarpRows], cnt[kWarpRows];
#pragma unroll
        for (int r = 0; r < kWarpRows; ++r) {
            const uint64_t g = gb + r * 32 + lane;
            uint32_t cc = 0, l = 0, k = 0;
            if (g < ngroups) {
                cc = __ldg(seg + g);
                if (g == ngroups - 1 && tail_r) {
                    cc &= (1u << (2 * tail_r)) - 1u;
                    l = field_sum(cc) + tail_r;
                    k = tail_r;
                } else {
                    l = field_sum(cc) + 4u;
                    k = 4;
                }
            }
            c[r] = cc;
            len[r] = l;
            cnt[r] = k;
        }
        // two packed 16-bit scans cover the four rows (row totals <= 512)
        const uint32_t p0 = len[0] | (len[1] << 16), p1 = len[2] | (len[3] << 16);
        const uint32_t i0 = warp_inclusive_scan(p0), i1 = warp_inclusive_scan(p1);
        const uint32_t t0 = __shfl_sync(kFull, i0, 31), t1 = __shfl_sync(kFull, i1, 31);
        const uint32_t e0 = i0 - p0, e1 = i1 - p1;
        const uint32_t r0 = t0 & 0xFFFFu, r1 = t0 >> 16, r2 = t1 & 0xFFFFu, r3 = t1 >> 16;
        uint32_t q[kWarpRows];
        q[0] = e0 & 0xFFFFu;
        q[1] = r0 + (e0 >> 16);
        q[2] = r0 + r1 + (e1 & 0xFFFFu);
        q[3] = r0 + r1 + r2 + (e1 >> 16);
        const uint32_t step_total = r0 + r1 + r2 + r3;

        const uintptr_t beg = data + off, end = beg + step_total;
        const uintptr_t a0 = beg & ~(uintptr_t)15, a1 = (end + 15) & ~(uintptr_t)15;
        const uint32_t nch = (uint32_t)((a1 - a0) >> 4);
        uint4 v5[5];
#pragma unroll
        for (int u = 0; u < 5; ++u) {
            const uint32_t ch = lane + 32 * u;
            if (ch < nch) v5[u] = load_chunk_guarded(a0 + 16 * (uintptr_t)ch, lo_ok, hi_ok);
        }
#pragma unroll
        for (int u = 0; u < 5; ++u) {
            const uint32_t ch = lane + 32 * u;
            if (ch < nch) *reinterpret_cast<uint4*>(stage + 16 * ch) = v5[u];
        }
        __syncwarp();
        const uint32_t head = (uint32_t)(beg - a0);
#pragma unroll
        for (int r = 0; r < kWarpRows; ++r) {
            const bool allzero = __all_sync(kFull, c[r] == 0);
            const uint32_t b = head + q[r];
            uint4 v = allzero ? decode_zero_group(W, b) : decode_group(W, b, c[r]);
            const uint64_t gi = gb + r * 32 + lane;
            if constexpr (kDelta) {
                v = prefix4(mask_tail(v, cnt[r]));
                const uint32_t S = v.w;
                const uint32_t I = warp_inclusive_scan(S);
                v = add4(v, carry + I - S);
                carry += __shfl_sync(kFull, I, 31);
            }
            if (cnt[r]) store_group(out + 4 * gi, v, cnt[r], out16);
        }
        off += step_total;
        __syncwarp();
    }
    if (lane == 0 && ngroups + off != seg_len)
        report_status(status, epoch, ngroups + off > seg_len ? BCGPU_ERR_TRUNCATED : BCGPU_ERR_TRAILING_BYTES);
}

template <bool kDelta>
__global__ void __launch_bounds__(kThreads) svb_decode_batch_warp_kernel(const bcgpu_decode_segment* __restrict__ segs,
                                                                         uint64_t nseg, const uint8_t* __restrict__ in,
                                                                         uint32_t* __restrict__ out, uint32_t max_n,
                                                                         unsigned long long* status, uint32_t epoch) {
    __shared__ __align__(16) uint8_t stage_all[kWarps][kWarpStageBytes];
    const int warp = threadIdx.x >> 5;
    const uint64_t gw = (uint64_t)blockIdx.x * kWarps + warp, nw = (uint64_t)gridDim.x * kWarps;
    for (uint64_t s = gw; s < nseg; s += nw) {
        const SegDesc d = load_desc_warp(segs, s);
        if (d.n > max_n) continue;
        if (d.n == 0) {
            if ((threadIdx.x & 31) == 0 && d.b != 0) report_status(status, epoch, BCGPU_ERR_TRAILING_BYTES);
            continue;
        }
        decode_segment_warp<kDelta>(in + d.a, d.b, d.n, d.prev, out + d.c, stage_all[warp], status, epoch);
    }
}

// -------- encode, CTA per segment
template <bool kDelta>
__global__ void __launch_bounds__(kThreads) svb_encode_batch_cta_kernel(const bcgpu_encode_segment* __restrict__ segs,
                                                                        uint64_t nseg, const uint32_t* __restrict__ in,
                                                                        uint8_t* __restrict__ out,
                                                                        uint64_t* __restrict__ out_lens, uint32_t min_n,
                                                                        unsigned long long* status, uint32_t epoch) {
    extern __shared__ __align__(16) uint8_t stage[];
    __shared__ EncodeSmem sh;
    for (uint64_t s = blockIdx.x; s < nseg; s += gridDim.x) {
        const bcgpu_encode_segment e = segs[s];
        if (e.n < min_n) continue;
        const uint64_t ngroups = ((uint64_t)e.n + 3) >> 2;
        if (e.dst_capacity < ngroups + 4ull * e.n) {
            if (threadIdx.x == 0) report_status(status, epoch, BCGPU_ERR_INVALID_ARGUMENT);
            continue;
        }
        const uint32_t* src = in + e.src_offset;
        uint8_t* dst = out + e.dst_offset;
        uint64_t run_off = 0;
        for (uint64_t g0 = 0; g0 < ngroups; g0 += kTileGroups) {
            const TileResult r = encode_tile<kDelta>(src, e.prev, ngroups, e.n & 3u, g0, dst, sh, stage,
                                                     [&](uint32_t) { return run_off; });
            run_off = r.off + r.total;
        }
        if (threadIdx.x == 0) out_lens[s] = ngroups + run_off;
    }
}

// -------- encode, warp per segment
template <bool kDelta>
__device__ __forceinline__ uint64_t encode_segment_warp(const uint32_t* __restrict__ src, uint32_t n, uint32_t prev,
                                                        uint8_t* __restrict__ dst, uint8_t* stage) {
    const int lane = threadIdx.x & 31;
    const uint64_t ngroups = ((uint64_t)n + 3) >> 2;
    const uint32_t tail_r = n & 3u;
    const bool in16 = (((uintptr_t)src) & 15) == 0;
    const uintptr_t data = (uintptr_t)dst + ngroups;
    uint64_t off = 0;
    uint32_t last = prev;  // x_{-1} for the step's first integer
    for (uint64_t gb = 0; gb < ngroups; gb += kWarpStepGroups) {
        uint4 d[kWarpRows];
        uint32_t lens[kWarpRows], L[kWarpRows];
#pragma unroll
        for (int r = 0; r < kWarpRows; ++r) {
            const uint64_t gi = gb + r * 32 + lane;
            const uint32_t cnt = gi < ngroups ? ((gi == ngroups - 1 && tail_r) ? tail_r : 4u) : 0u;
            uint4 x = make_uint4(0, 0, 0, 0);
            if (cnt == 4 && in16) {
                x = ldg_stream_v4(src + 4 * gi);
            } else if (cnt) {
                x.x = __ldg(src + 4 * gi);
                if (cnt > 1) x.y = __ldg(src + 4 * gi + 1);
                if (cnt > 2) x.z = __ldg(src + 4 * gi + 2);
                if (cnt > 3) x.w = __ldg(src + 4 * gi + 3);
            }
            if constexpr (kDelta) {
                uint32_t p = __shfl_up_sync(kFull, x.w, 1);
                if (lane == 0) p = last;
                last = __shfl_sync(kFull, x.w, 31);  // only meaningful while the row is full
                x = make_uint4(x.x - p, x.y - x.x, x.z - x.y, x.w - x.z);
            }
            d[r] = x;
            const uint32_t l0 = cnt > 0 ? dev_byte_length(x.x) : 0u;
            const uint32_t l1 = cnt > 1 ? dev_byte_length(x.y) : 0u;
            const uint32_t l2 = cnt > 2 ? dev_byte_length(x.z) : 0u;
            const uint32_t l3 = cnt > 3 ? dev_byte_length(x.w) : 0u;
            lens[r] = l0 | (l1 << 8) | (l2 << 16) | (l3 << 24);
            L[r] = l0 + l1 + l2 + l3;
            if (cnt) {
                const uint32_t c = ((l0 - 1) & 3u) | (l1 ? ((l1 - 1) << 2) : 0u) | (l2 ? ((l2 - 1) << 4) : 0u) |
                                   (l3 ? ((l3 - 1) << 6) : 0u);
                dst[gi] = (uint8_t)c;
            }
        }
        const uint32_t p0 = L[0] | (L[1] << 16), p1 = L[2] | (L[3] << 16);
        const uint32_t i0 = warp_inclusive_scan(p0), i1 = warp_inclusive_scan(p1);
        const uint32_t t0 = __shfl_sync(kFull, i0, 31), t1 = __shfl_sync(kFull, i1, 31);
        const uint32_t e0 = i0 - p0, e1 = i1 - p1;
        const uint32_t r0 = t0 & 0xFFFFu, r1 = t0 >> 16, r2 = t1 & 0xFFFFu, r3 = t1 >> 16;
        uint32_t q[kWarpRows];
        q[0] = e0 & 0xFFFFu;
        q[1] = r0 + (e0 >> 16);
        q[2] = r0 + r1 + (e1 & 0xFFFFu);
        q[3] = r0 + r1 + r2 + (e1 >> 16);
        const uint32_t step_total = r0 + r1 + r2 + r3;
        const uintptr_t beg = data + off, end = beg + step_total;
        const uintptr_t a0 = beg & ~(uintptr_t)15, a1 = (end + 15) & ~(uintptr_t)15;
        const uint32_t head = (uint32_t)(beg - a0);
#pragma unroll
        for (int r = 0; r < kWarpRows; ++r) {
            if (L[r]) {
                uint32_t p = head + q[r];
                const uint32_t l = lens[r];
                put_int_bytes(stage, p, d[r].x, l & 0xFF);
                p += l & 0xFF;
                if ((l >> 8) & 0xFF) put_int_bytes(stage, p, d[r].y, (l >> 8) & 0xFF);
                p += (l >> 8) & 0xFF;
                if ((l >> 16) & 0xFF) put_int_bytes(stage, p, d[r].z, (l >> 16) & 0xFF);
                p += (l >> 16) & 0xFF;
                if (l >> 24) put_int_bytes(stage, p, d[r].w, l >> 24);
            }
        }
        __syncwarp();
        const uint32_t nch = (uint32_t)((a1 - a0) >> 4);
        for (uint32_t ch = lane; ch < nch; ch += 32) {
            const uintptr_t a = a0 + 16 * (uintptr_t)ch;
            if (a >= beg && a + 16 <= end) {
                stg_stream_v4(reinterpret_cast<void*>(a), *reinterpret_cast<const uint4*>(stage + 16 * ch));
            } else {
                for (int b = 0; b < 16; ++b)
                    if (a + b >= beg && a + b < end) *reinterpret_cast<uint8_t*>(a + b) = stage[16 * ch + b];
            }
        }
        off += step_total;
        __syncwarp();
    }
    return ngroups + off;
}

template <bool kDelta>
__global__ void __launch_bounds__(kThreads) svb_encode_batch_warp_kernel(const bcgpu_encode_segment* __restrict__ segs,
                                                                         uint64_t nseg, const uint32_t* __restrict__ in,
                                                                         uint8_t* __restrict__ out,
                                                                         uint64_t* __restrict__ out_lens, uint32_t max_n,
                                                                         unsigned long long* status, uint32_t epoch) {
    __shared__ __align__(16) uint8_t stage_all[kWarps][kWarpStageBytes];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t gw = (uint64_t)blockIdx.x * kWarps + warp, nw = (uint64_t)gridDim.x * kWarps;
    for (uint64_t s = gw; s < nseg; s += nw) {
        const SegDesc e = load_desc_warp(segs, s);
        if (e.n > max_n) continue;
        const uint64_t ngroups = ((uint64_t)e.n + 3) >> 2;
        if (e.b < ngroups + 4ull * e.n) {
            if (lane == 0) report_status(status, epoch, BCGPU_ERR_INVALID_ARGUMENT);
            continue;
        }
        const uint64_t len = encode_segment_warp<kDelta>(in + e.a, e.n, e.prev, out + e.c, stage_all[warp]);
        if (lane == 0) out_lens[s] = len;
    }
}

// -------- size-only pass, warp per segment
template <bool kDelta>
__global__ void __launch_bounds__(kThreads) svb_sizes_batch_kernel(const bcgpu_encode_segment* __restrict__ segs,
                                                                   uint64_t nseg, const uint32_t* __restrict__ in,
                                                                   uint64_t* __restrict__ out_lens) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t gw = (uint64_t)blockIdx.x * kWarps + warp, nw = (uint64_t)gridDim.x * kWarps;
    for (uint64_t s = gw; s < nseg; s += nw) {
        const SegDesc e = load_desc_warp(segs, s);
        const uint32_t* src = in + e.a;
        uint64_t acc = 0;
        for (uint64_t i = lane; i < e.n; i += 32) {
            const uint32_t x = __ldg(src + i);
            uint32_t v = x;
            if constexpr (kDelta) v = x - (i ? __ldg(src + i - 1) : e.prev);
            acc += dev_byte_length(v);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (lane == 0) out_lens[s] = (((uint64_t)e.n + 3) >> 2) + acc;
    }
}

// ===========================================================================
// launchers
// ===========================================================================
template <class K>
static cudaError_t set_smem(K kernel, int bytes) {
    static_assert(sizeof(K) > 0, "");
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

cudaError_t launch_decode(const uint8_t* in, uint64_t in_len, uint64_t n, int delta, uint32_t base, uint32_t* out,
                          uint32_t* d_last, const LookbackArgs& lb, cudaStream_t stream) {
    const int grid = (int)lb.num_tiles;
    if (delta) {
        static cudaError_t once = set_smem(svb_decode_kernel<true>, kStageBytes);
        if (once != cudaSuccess) return once;
        svb_decode_kernel<true><<<grid, kThreads, kStageBytes, stream>>>(in, in_len, n, base, out, d_last, lb);
    } else {
        static cudaError_t once = set_smem(svb_decode_kernel<false>, kStageBytes);
        if (once != cudaSuccess) return once;
        svb_decode_kernel<false><<<grid, kThreads, kStageBytes, stream>>>(in, in_len, n, base, out, d_last, lb);
    }
    return cudaGetLastError();
}

cudaError_t launch_encode(const uint32_t* in, uint64_t n, int delta, uint32_t prev, uint8_t* out,
                          uint64_t* d_out_len, const LookbackArgs& lb, cudaStream_t stream) {
    const int grid = (int)lb.num_tiles;
    if (delta) {
        static cudaError_t once = set_smem(svb_encode_kernel<true>, kStageBytes);
        if (once != cudaSuccess) return once;
        svb_encode_kernel<true><<<grid, kThreads, kStageBytes, stream>>>(in, n, prev, out, d_out_len, lb);
    } else {
        static cudaError_t once = set_smem(svb_encode_kernel<false>, kStageBytes);
        if (once != cudaSuccess) return once;
        svb_encode_kernel<false><<<grid, kThreads, kStageBytes, stream>>>(in, n, prev, out, d_out_len, lb);
    }
    return cudaGetLastError();
}

cudaError_t launch_block_offsets(const uint8_t* in, uint64_t n, uint64_t* d_offsets, const LookbackArgs& lb,
                                 cudaStream_t stream) {
    svb_block_offsets_kernel<<<(int)lb.num_tiles, kThreads, 0, stream>>>(in, n, d_offsets, lb);
    return cudaGetLastError();
}

cudaError_t launch_decode_blocks(const uint8_t* in, uint64_t in_len, uint64_t n, const uint64_t* blocks,
                                 const uint64_t* offsets, uint64_t nblocks, uint32_t* out, uint32_t* counts,
                                 cudaStream_t stream) {
    const int grid = (int)((nblocks + kThreads - 1) / kThreads);
    svb_decode_blocks_kernel<<<grid, kThreads, 0, stream>>>(in, in_len, n, blocks, offsets, nblocks, out, counts);
    return cudaGetLastError();
}

static int occ_of(const void* k, int dyn) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, dyn) != cudaSuccess || occ < 1) occ = 1;
    return occ;
}

int occupancy_decode_batch_cta() {
    set_smem(svb_decode_batch_cta_kernel<true>, kStageBytes);
    set_smem(svb_decode_batch_cta_kernel<false>, kStageBytes);
    return occ_of((const void*)svb_decode_batch_cta_kernel<true>, kStageBytes);
}
int occupancy_decode_batch_warp() { return occ_of((const void*)svb_decode_batch_warp_kernel<true>, 0); }
int occupancy_encode_batch_cta() {
    set_smem(svb_encode_batch_cta_kernel<true>, kStageBytes);
    set_smem(svb_encode_batch_cta_kernel<false>, kStageBytes);
    return occ_of((const void*)svb_encode_batch_cta_kernel<true>, kStageBytes);
}
int occupancy_encode_batch_warp() { return occ_of((const void*)svb_encode_batch_warp_kernel<true>, 0); }

cudaError_t launch_decode_batch(const bcgpu_decode_segment* segs, uint64_t nseg, const uint8_t* in, uint32_t* out,
                                int delta, uint32_t max_seg_n, const BatchArgs& ba, cudaStream_t stream, int* launches) {
    *launches = 0;
    const bool any_small = true;  // cannot be excluded from a max hint
    const bool any_large = max_seg_n == 0 || max_seg_n > kWarpSegmentMax;
    const uint32_t warp_max = any_large ? kWarpSegmentMax : 0xFFFFFFFFu;
    if (any_small) {
        const uint64_t want = (nseg + kWarps - 1) / kWarps;
        const int grid = (int)(want < (uint64_t)ba.warp_grid ? want : (uint64_t)ba.warp_grid);
        if (grid > 0) {
            if (delta)
                svb_decode_batch_warp_kernel<true><<<grid, kThreads, 0, stream>>>(segs, nseg, in, out, warp_max,
                                                                                  ba.status, ba.epoch);
            else
                svb_decode_batch_warp_kernel<false><<<grid, kThreads, 0, stream>>>(segs, nseg, in, out, warp_max,
                                                                                   ba.status, ba.epoch);
            ++*launches;
            const cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
        }
    }
    if (any_large) {
        const int grid = (int)(nseg < (uint64_t)ba.cta_grid ? nseg : (uint64_t)ba.cta_grid);
        if (grid > 0) {
            if (delta)
                svb_decode_batch_cta_kernel<true><<<grid, kThreads, kStageBytes, stream>>>(
                    segs, nseg, in, out, kWarpSegmentMax + 1, ba.status, ba.epoch);
            else
                svb_decode_batch_cta_kernel<false><<<grid, kThreads, kStageBytes, stream>>>(
                    segs, nseg, in, out, kWarpSegmentMax + 1, ba.status, ba.epoch);
            ++*launches;
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_encode_batch(const bcgpu_encode_segment* segs, uint64_t nseg, const uint32_t* in, uint8_t* out,
                                uint64_t* out_lens, int delta, uint32_t max_seg_n, const BatchArgs& ba,
                                cudaStream_t stream, int* launches) {
    *launches = 0;
    const bool any_large = max_seg_n == 0 || max_seg_n > kWarpSegmentMax;
    const uint32_t warp_max = any_large ? kWarpSegmentMax : 0xFFFFFFFFu;
    {
        const uint64_t want = (nseg + kWarps - 1) / kWarps;
        const int grid = (int)(want < (uint64_t)ba.warp_grid ? want : (uint64_t)ba.warp_grid);
        if (grid > 0) {
            if (delta)
                svb_encode_batch_warp_kernel<true><<<grid, kThreads, 0, stream>>>(segs, nseg, in, out, out_lens,
                                                                                  warp_max, ba.status, ba.epoch);
            else
                svb_encode_batch_warp_kernel<false><<<grid, kThreads, 0, stream>>>(segs, nseg, in, out, out_lens,
                                                                                   warp_max, ba.status, ba.epoch);
            ++*launches;
            const cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
        }
    }
    if (any_large) {
        const int grid = (int)(nseg < (uint64_t)ba.cta_grid ? nseg : (uint64_t)ba.cta_grid);
        if (grid > 0) {
            if (delta)
                svb_encode_batch_cta_kernel<true><<<grid, kThreads, kStageBytes, stream>>>(
                    segs, nseg, in, out, out_lens, kWarpSegmentMax + 1, ba.status, ba.epoch);
            else
                svb_encode_batch_cta_kernel<false><<<grid, kThreads, kStageBytes, stream>>>(
                    segs, nseg, in, out, out_lens, kWarpSegmentMax + 1, ba.status, ba.epoch);
            ++*launches;
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_sizes_batch(const bcgpu_encode_segment* segs, uint64_t nseg, const uint32_t* in,
                               uint64_t* out_lens, int delta, const BatchArgs& ba, cudaStream_t stream) {
    const uint64_t want = (nseg + kWarps - 1) / kWarps;
    const int grid = (int)(want < (uint64_t)ba.warp_grid ? want : (uint64_t)ba.warp_grid);
    if (grid <= 0) return cudaSuccess;
    if (delta)
        svb_sizes_batch_kernel<true><<<grid, kThreads, 0, stream>>>(segs, nseg, in, out_lens);
    else
        svb_sizes_batch_kernel<false><<<grid, kThreads, 0, stream>>>(segs, nseg, in, out_lens);
    return cudaGetLastError();
}

}  // namespace bcgpu
