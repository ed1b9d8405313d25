// svb_encode.cu -- single-array Stream VByte encode for sm_100a (svb_encode,
// reference stream_vbyte.hpp:36; delta encode codec.hpp:92-93 and the
// prev-seeded extension E2).
//
// Reduce-then-scan, no CTA ever waits on another:
//   1. svb_size_scan_kernel  reads the integers once (4 B/int): every
//      1024-integer sub-tile's data size (sum of byte_length, codec.hpp:70-72,
//      of the values or of their mod-2^32 deltas), chunk-local prefixes, chunk
//      totals; the last CTA scans the chunk totals and writes the exact size.
//   2. svb_encode_tile_kernel one CTA per 8 sub-tiles.  Each warp TMA-loads its
//      4 KiB of integers (+ the 4 before, for the delta seed) while the CTA's
//      offsets arrive, classifies lengths (max(1, 4 - clz/8)), TMA-stores its
//      256 control bytes (field i of control byte k = len-1 in bits 2i,
//      SPEC.md:275-281), packs the data bytes in place at the destination's
//      16-B phase and writes them with one TMA bulk store (+ edge bytes).
// When the input is L2-resident (it was just produced), the second read is an
// L2 hit; from HBM the encode moves 8 + cmp bytes per 4-byte integer.
#include <cstdint>

#include "svb_device.cuh"
#include "svb_fast.cuh"
#include "launch_cache.cuh"
#include "svb_kernels.cuh"
#include "svb_pack.cuh"
#include "svb_scan.cuh"
#include "svb_tma.cuh"
#include "svb_warp.cuh"

namespace bcgpu {

__device__ __forceinline__ void enc_report(unsigned long long* st, uint32_t epoch, uint32_t code) {
    if (st) *st = ((unsigned long long)epoch << 32) | code;
}

__device__ __forceinline__ uint32_t lens4(uint4 x, uint32_t cnt) {
    return (cnt > 0 ? dev_byte_length(x.x) : 0u) + (cnt > 1 ? dev_byte_length(x.y) : 0u) +
           (cnt > 2 ? dev_byte_length(x.z) : 0u) + (cnt > 3 ? dev_byte_length(x.w) : 0u);
}

// ---------------------------------------------------------------------------
// 1. size scan: warp w of a chunk CTA sizes sub-tiles 8w .. 8w+7
// ---------------------------------------------------------------------------
template <bool kDelta>
__global__ void __launch_bounds__(256)
    svb_size_scan_kernel(const uint32_t* __restrict__ in, uint64_t n, uint32_t prev, DecodeMeta meta,
                         uint64_t* __restrict__ d_out_len, unsigned long long* status, uint32_t epoch,
                         uint32_t c_begin, uint32_t nchunks_total) {
    __shared__ uint32_t wt[8];
    __shared__ bool last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t chunk = c_begin + blockIdx.x, c_end = c_begin + gridDim.x;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const bool in16 = (((uintptr_t)in) & 15) == 0;
    uint32_t my_size = 0;  // lane k < 8: size of sub-tile 8*warp + k
    uint32_t lean_last = 0;  // lane 0, delta: the integer before the next sub-tile
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
        const uint64_t s = (uint64_t)chunk * kChunkSubs + 8 * warp + k;
        if (s >= nsub) break;
        const uint64_t g0 = s * kWTGroups;
        if (in16 && (s + 1) * kWTInts <= n) {  // full sub-tile: lean path (svb_fast.cuh)
            if (kDelta && k == 0) lean_last = g0 ? __ldg(in + 4 * g0 - 1) : prev;
            uint32_t acc = size_full<kDelta>(in + 4 * g0, lean_last);
#pragma unroll
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
            if (lane == k) my_size = acc + kWTInts;
            continue;
        }
        uint32_t last_w = prev;
        if (kDelta && g0) last_w = __ldg(in + 4 * g0 - 1);
        uint4 x[kWTRows];
        uint32_t cnt[kWTRows];
#pragma unroll
        for (int j = 0; j < kWTRows; ++j) {
            const uint64_t g = g0 + 32 * j + lane;
            cnt[j] = group_count(g, ngroups, tail_r);
            x[j] = make_uint4(0, 0, 0, 0);
            if (cnt[j] == 4 && in16) {
                x[j] = ldg_stream_v4(in + 4 * g);
            } else if (cnt[j]) {
                x[j].x = __ldg(in + 4 * g);
                if (cnt[j] > 1) x[j].y = __ldg(in + 4 * g + 1);
                if (cnt[j] > 2) x[j].z = __ldg(in + 4 * g + 2);
                if (cnt[j] > 3) x[j].w = __ldg(in + 4 * g + 3);
            }
        }
        uint32_t acc = 0;
#pragma unroll
        for (int j = 0; j < kWTRows; ++j) {
            uint4 v = x[j];
            if constexpr (kDelta) {
                uint32_t p = __shfl_up_sync(kFull, v.w, 1);
                if (lane == 0) p = last_w;
                last_w = __shfl_sync(kFull, v.w, 31);
                v = make_uint4(v.x - p, v.y - v.x, v.z - v.y, v.w - v.z);
            }
            acc += lens4(v, cnt[j]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (lane == k) my_size = acc;
    }
    // chunk-local exclusive prefix over the 64 sub-tiles (lanes 0..7 of each warp)
    const uint32_t v = lane < 8 ? my_size : 0u;
    const uint32_t incl = warp_inclusive_scan(v);
    if (lane == 31) wt[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        wpre += w < warp ? wt[w] : 0u;
        total += wt[w];
    }
    const uint64_t s = (uint64_t)chunk * kChunkSubs + 8 * warp + lane;
    if (lane < 8 && s < nsub) meta.localpre[s] = wpre + incl - v;
    if (tid == 0) meta.chunktot[chunk] = total;
    // last CTA of this slice: chunk offsets of the slice = running offset + scan of the chunk totals
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        last = atomicAdd(meta.counters, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const unsigned long long base = c_begin == 0 ? 0ull : *meta.running;
    const uint32_t tot = cta_exclusive_scan<uint32_t, 8>(meta.chunktot + c_begin, gridDim.x, wt);
    for (uint32_t c = tid; c < gridDim.x; c += 256) {
        meta.chunkpre[c_begin + c] = base + meta.chunktot[c_begin + c];
        meta.chunktot[c_begin + c] = 0;  // the slot encode accumulates into zeroed totals
    }
    if (tid == 0) {
        meta.chunkpre[c_end] = base + tot;  // == the next slice's base (same value written twice)
        *meta.running = base + tot;
        if (c_end == nchunks_total) {
            if (d_out_len) *d_out_len = ngroups + base + tot;
            enc_report(status, epoch, 0u);
        }
        *meta.counters = 0;
    }
}

// ---------------------------------------------------------------------------
// 2. encode tiles
// ---------------------------------------------------------------------------
struct __align__(16) EncBuf {
    uint8_t stage[kWTStage + 16];  // [0,16): the 4 integers before the sub-tile, [16, 16+4096): the sub-tile
    uint8_t ctrl[kWTGroups];
};

template <bool kDelta>
__global__ void __launch_bounds__(kCTThreads, 4)
    svb_encode_tile_kernel(const uint32_t* __restrict__ in, uint64_t n, uint32_t prev, uint8_t* __restrict__ out,
                           DecodeMeta meta, uint32_t tile_base) {
    __shared__ __align__(128) EncBuf wb[kCTWarps];
    __shared__ __align__(16) uint32_t slocal[kCTWarps + 8];
    __shared__ __align__(16) unsigned long long schunk[4];
    __shared__ __align__(8) uint64_t bars[kCTWarps + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // last tile first: the size scan just streamed the input front to back, so its
    // tail is what L2 still holds
    const uint32_t tile = tile_base + (gridDim.x - 1 - blockIdx.x);
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t sub0 = (uint64_t)tile * kCTWarps;
    const uint64_t chunk = sub0 / kChunkSubs;
    const uint64_t sub = sub0 + warp;
    const uint64_t g0 = sub * kWTGroups;
    const bool active = g0 < ngroups;
    EncBuf& b = wb[warp];
    if (threadIdx.x == 0) {
        mbar_init1(&bars[kCTWarps]);
        mbar_expect(&bars[kCTWarps], 48 + 32);
        tma_load(slocal, meta.localpre + sub0, 48, &bars[kCTWarps]);
        tma_load(schunk, meta.chunkpre + (chunk & ~1ull), 32, &bars[kCTWarps]);
    }
    if (lane == 0) mbar_init1(&bars[warp]);
    __syncthreads();
    if (!active) return;  // no CTA-wide barrier below

    // the sub-tile's integers (and the 4 before it) -> stage
    const uint64_t i0 = 4 * g0;
    const uint32_t nints = (uint32_t)(n - i0 < (uint64_t)kWTInts ? n - i0 : (uint64_t)kWTInts);
    {
        const uintptr_t lo = (uintptr_t)in, hi = lo + 4 * n;
        const uintptr_t beg = (uintptr_t)(in + i0) - (g0 ? 16 : 0), end = (uintptr_t)(in + i0 + nints);
        const uint32_t tx = tma_cover_bytes(beg, end, lo, hi);
        const bool use_tma = tx != 0xFFFFFFFFu && (beg & 15) == 0;
        uint8_t* dst = b.stage + (g0 ? 0 : 16);
        if (use_tma) {
            if (lane == 0) {
                mbar_expect(&bars[warp], tx);
                tma_load(dst, reinterpret_cast<const void*>(beg), tx, &bars[warp]);
            }
            mbar_wait_parity(&bars[warp], 0);
        } else {
            uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
            const uint32_t words = (uint32_t)((end - beg) >> 2);
            for (uint32_t i = lane; i < words; i += 32) d32[i] = __ldg(reinterpret_cast<const uint32_t*>(beg) + i);
            __syncwarp();
        }
    }
    const uint32_t cnt_g = (uint32_t)(ngroups - g0 < (uint64_t)kWTGroups ? ngroups - g0 : (uint64_t)kWTGroups);
    const bool full = 4 * (g0 + kWTGroups) <= n;
    uint32_t total;
    uint32_t lens[kWTRows], qw[4];
    EncodeTile t;
    const uint32_t prev_w = g0 ? reinterpret_cast<const uint32_t*>(b.stage)[3] : prev;
    bool small = false;
    if (full) {
        // every integer < 256: control bytes 0, data = the low bytes (svb_fast.cuh)
        small = enc_full_small<kDelta>(sh_addr(b.stage) + 16, prev_w);
        if (small) {
            asm volatile("st.shared.v2.u32 [%0], {%1, %1};" ::"r"(sh_addr(b.ctrl) + 8 * lane), "r"(0u) : "memory");
            total = kWTInts;
        } else {
            // lengths, control bytes, tile-local offsets (lean path, svb_fast.cuh)
            total = enc_full_lengths<kDelta>(sh_addr(b.stage) + 16, prev_w, sh_addr(b.ctrl), lens, qw);
        }
    } else {
        uint32_t P[3] = {0, 0, 0};
        uint32_t last_w = prev_w;
#pragma unroll
        for (int j = 0; j < kWTRows; ++j) {
            const uint32_t cnt = group_count(g0 + 32 * j + lane, ngroups, tail_r);
            uint4 x = mask_tail(*reinterpret_cast<const uint4*>(b.stage + 16 + 512 * j + 16 * lane), cnt);
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
            b.ctrl[32 * j + lane] = (uint8_t)((l0 - 1) | (l1 ? ((l1 - 1) << 2) : 0u) | (l2 ? ((l2 - 1) << 4) : 0u) |
                                              (l3 ? ((l3 - 1) << 6) : 0u));
        }
        t.total = packed_row_scan(P, t.qw);
        total = t.total;
    }
    // where the data goes
    mbar_wait_parity(&bars[kCTWarps], 0);
    const unsigned long long cpre = schunk[chunk & 1];
    const uint64_t off = cpre + slocal[warp];
    const uintptr_t dbeg = (uintptr_t)out + ngroups + off, dend = dbeg + total;
    const uint32_t head = (uint32_t)(dbeg & 15);
    // pack in place at the destination's 16-B phase: group g's bytes end at or before
    // head + 16(g+1) <= 16 + 16g + 15 < the input of group g+1 (stage + 16 + 16(g+1))
    __syncwarp();
    if (small)
        enc_small_pack<kDelta>(sh_addr(b.stage) + 16, prev_w, sh_addr(b.stage) + head);
    else if (full)
        enc_full_pack_w<kDelta>(sh_addr(b.stage) + 16, prev_w, lens, qw, sh_addr(b.stage) + head, total);
    else
        encode_pack_at(t, b.stage, head);
    fence_async_smem();
    __syncwarp();
    uint8_t* cdst = out + g0;
    const uint32_t cb = (((uintptr_t)cdst & 15) == 0) ? (cnt_g & ~15u) : 0u;
    const uintptr_t a_lo = (dbeg + 15) & ~(uintptr_t)15, a_hi = dend & ~(uintptr_t)15;
    const uint32_t db = a_hi > a_lo ? (uint32_t)(a_hi - a_lo) : 0u;
    if (lane == 0) {
        if (cb) tma_store(cdst, b.ctrl, cb);
        if (db) tma_store(reinterpret_cast<void*>(a_lo), b.stage + (a_lo - dbeg) + head, db);
        if (cb || db) tma_store_commit();
    }
    for (uint32_t i = cb + lane; i < cnt_g; i += 32) cdst[i] = b.ctrl[i];
    // edge bytes shared with the neighbouring sub-tiles' 16-B granules (< 16 at each end)
    if (db == 0) {
        for (uint32_t i = lane; i < total; i += 32) *reinterpret_cast<uint8_t*>(dbeg + i) = b.stage[head + i];
    } else {
        const uint32_t nh = (uint32_t)(a_lo - dbeg), nt = (uint32_t)(dend - a_hi);
        if (lane < nh) *reinterpret_cast<uint8_t*>(dbeg + lane) = b.stage[head + lane];
        if (lane < nt) *reinterpret_cast<uint8_t*>(a_hi + lane) = b.stage[head + (uint32_t)(a_hi - dbeg) + lane];
    }
    if (lane == 0 && (cb || db)) tma_store_wait_read();
}

// ---------------------------------------------------------------------------
// 3. single-read encode: pack into per-tile slots, then compact
// ---------------------------------------------------------------------------
// svb_encode_slot_kernel reads every integer once.  CTA t (8 sub-tiles) sizes and
// packs its sub-tiles exactly like the tile kernel, but with no offsets to wait
// for: the control bytes go straight to their final place (byte g of the
// stream), the data bytes to a private, 128-B aligned, worst-case-sized slot in
// scratch (kept in L2: evict_last; the integers stream through with
// evict_first), the tile's data size to tilesize[t] and (RED.ADD) to its
// chunk's total; the last CTA scans the chunk totals.  svb_encode_compact_kernel
// then moves each slot to its final offset -- one warp per tile, 16-B
// granules realigned with funnel shifts, 128-bit stores -- and discards each
// slot line from L2 once read, so the slots never cost a DRAM write-back.
// From HBM: 4 B/int in, cmp bytes out (+ whatever of the slots L2 cannot hold).
constexpr uint32_t kSlotStride = kCTWarps * kWTDataMax + 128;  // worst-case tile data + slack, 128-B multiple

template <bool kDelta>
__global__ void __launch_bounds__(kCTThreads, 4)
    svb_encode_slot_kernel(const uint32_t* __restrict__ in, uint64_t n, uint32_t prev, uint8_t* __restrict__ out,
                           DecodeMeta meta, uint8_t* __restrict__ slots, uint64_t* __restrict__ d_out_len,
                           unsigned long long* status, uint32_t epoch, uint32_t hints) {
    __shared__ __align__(128) EncBuf wb[kCTWarps];
    __shared__ __align__(8) uint64_t bars[kCTWarps];
    __shared__ uint32_t wtot[kCTWarps];
    __shared__ unsigned long long wscan[kCTWarps];
    __shared__ bool last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tile = blockIdx.x;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t sub = (uint64_t)tile * kCTWarps + warp;
    const uint64_t g0 = sub * kWTGroups;
    const bool active = g0 < ngroups;
    EncBuf& b = wb[warp];
    if (lane == 0) mbar_init1(&bars[warp]);
    __syncwarp();

    uint32_t total = 0;
    bool small = false, full = false;
    uint32_t lens[kWTRows], qw[4];
    EncodeTile t;
    uint32_t prev_w = prev;
    const uint64_t i0 = 4 * g0;
    const uint32_t nints = active ? (uint32_t)(n - i0 < (uint64_t)kWTInts ? n - i0 : (uint64_t)kWTInts) : 0u;
    if (active) {
        // the sub-tile's integers (and the 4 before it) -> stage
        const uintptr_t lo = (uintptr_t)in, hi = lo + 4 * n;
        const uintptr_t beg = (uintptr_t)(in + i0) - (g0 ? 16 : 0), end = (uintptr_t)(in + i0 + nints);
        const uint32_t tx = tma_cover_bytes(beg, end, lo, hi);
        const bool use_tma = tx != 0xFFFFFFFFu && (beg & 15) == 0;
        uint8_t* dst = b.stage + (g0 ? 0 : 16);
        if (use_tma) {
            if (lane == 0) {
                mbar_expect(&bars[warp], tx);
                if (hints & 1)
                    tma_load_hint(dst, reinterpret_cast<const void*>(beg), tx, &bars[warp], l2_policy_drop());
                else
                    tma_load(dst, reinterpret_cast<const void*>(beg), tx, &bars[warp]);
            }
            mbar_wait_parity(&bars[warp], 0);
        } else {
            uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
            const uint32_t words = (uint32_t)((end - beg) >> 2);
            for (uint32_t i = lane; i < words; i += 32) d32[i] = __ldg(reinterpret_cast<const uint32_t*>(beg) + i);
            __syncwarp();
        }
        full = 4 * (g0 + kWTGroups) <= n;
        if (g0) prev_w = reinterpret_cast<const uint32_t*>(b.stage)[3];
        if (full) {
            small = enc_full_small<kDelta>(sh_addr(b.stage) + 16, prev_w);
            if (small) {
                asm volatile("st.shared.v2.u32 [%0], {%1, %1};" ::"r"(sh_addr(b.ctrl) + 8 * lane), "r"(0u) : "memory");
                total = kWTInts;
            } else {
                total = enc_full_lengths<kDelta>(sh_addr(b.stage) + 16, prev_w, sh_addr(b.ctrl), lens, qw);
            }
        } else {
            uint32_t P[3] = {0, 0, 0};
            uint32_t last_w = prev_w;
#pragma unroll
            for (int j = 0; j < kWTRows; ++j) {
                const uint32_t cnt = group_count(g0 + 32 * j + lane, ngroups, tail_r);
                uint4 x = mask_tail(*reinterpret_cast<const uint4*>(b.stage + 16 + 512 * j + 16 * lane), cnt);
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
                b.ctrl[32 * j + lane] = (uint8_t)((l0 - 1) | (l1 ? ((l1 - 1) << 2) : 0u) | (l2 ? ((l2 - 1) << 4) : 0u) |
                                                  (l3 ? ((l3 - 1) << 6) : 0u));
            }
            t.total = packed_row_scan(P, t.qw);
            total = t.total;
        }
    }
    // tile-local offsets of the 8 sub-tiles' data within the slot
    if (lane == 0) wtot[warp] = total;
    __syncthreads();
    uint32_t pre = 0, ttot = 0;
#pragma unroll
    for (int w = 0; w < kCTWarps; ++w) {
        const uint32_t x = wtot[w];
        pre += w < warp ? x : 0u;
        ttot += x;
    }
    if (active) {
        uint8_t* slot = slots + (size_t)tile * kSlotStride;
        const uintptr_t dbeg = (uintptr_t)slot + pre, dend = dbeg + total;
        const uint32_t head = (uint32_t)(dbeg & 15);
        __syncwarp();
        if (small)
            enc_small_pack<kDelta>(sh_addr(b.stage) + 16, prev_w, sh_addr(b.stage) + head);
        else if (full)
            enc_full_pack<kDelta>(sh_addr(b.stage) + 16, prev_w, lens, qw, sh_addr(b.stage) + head);
        else
            encode_pack_at(t, b.stage, head);
        fence_async_smem();
        __syncwarp();
        const uint32_t cnt_g = (uint32_t)(ngroups - g0 < (uint64_t)kWTGroups ? ngroups - g0 : (uint64_t)kWTGroups);
        uint8_t* cdst = out + g0;
        const uint32_t cb = (((uintptr_t)cdst & 15) == 0) ? (cnt_g & ~15u) : 0u;
        const uintptr_t a_lo = (dbeg + 15) & ~(uintptr_t)15, a_hi = dend & ~(uintptr_t)15;
        const uint32_t db = a_hi > a_lo ? (uint32_t)(a_hi - a_lo) : 0u;
        if (lane == 0) {
            if (cb) tma_store(cdst, b.ctrl, cb);
            if (db) {
                if (hints & 2)
                    tma_store_hint(reinterpret_cast<void*>(a_lo), b.stage + (a_lo - dbeg) + head, db, l2_policy_keep());
                else
                    tma_store(reinterpret_cast<void*>(a_lo), b.stage + (a_lo - dbeg) + head, db);
            }
            if (cb || db) tma_store_commit();
        }
        for (uint32_t i = cb + lane; i < cnt_g; i += 32) cdst[i] = b.ctrl[i];
        // edge bytes shared with the neighbouring sub-tiles' 16-B granules (< 16 at each end)
        if (db == 0) {
            for (uint32_t i = lane; i < total; i += 32) *reinterpret_cast<uint8_t*>(dbeg + i) = b.stage[head + i];
        } else {
            const uint32_t nh = (uint32_t)(a_lo - dbeg), nt = (uint32_t)(dend - a_hi);
            if (lane < nh) *reinterpret_cast<uint8_t*>(dbeg + lane) = b.stage[head + lane];
            if (lane < nt) *reinterpret_cast<uint8_t*>(a_hi + lane) = b.stage[head + (uint32_t)(a_hi - dbeg) + lane];
        }
        if (lane == 0 && (cb || db)) tma_store_wait_read();
    }
    if (threadIdx.x == 0) meta.tilesize[tile] = ttot;
    // last CTA: chunk offsets = exclusive scan of the chunk totals (8 tile sizes each)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(meta.counters, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint32_t nchunks = (uint32_t)((nsub + kChunkSubs - 1) / kChunkSubs);
    const uint32_t ntiles = gridDim.x;
    static_assert(kChunkSubs / kCTWarps == 8, "8 tiles per chunk");
    for (uint32_t c = threadIdx.x; c < nchunks; c += kCTThreads) {
        uint32_t sum = 0;
        if (8 * c + 8 <= ntiles) {  // tilesize is 16-B aligned (DecodeMeta carve)
            const uint4 a = __ldcg(reinterpret_cast<const uint4*>(meta.tilesize) + 2 * c);
            const uint4 b = __ldcg(reinterpret_cast<const uint4*>(meta.tilesize) + 2 * c + 1);
            sum = a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
        } else {
            for (uint32_t i = 8 * c; i < ntiles; ++i) sum += __ldcg(meta.tilesize + i);
        }
        meta.chunkpre[c] = sum;
    }
    __syncthreads();
    const unsigned long long tot = cta_exclusive_scan<unsigned long long, kCTWarps>(meta.chunkpre, nchunks, wscan);
    if (threadIdx.x == 0) {
        meta.chunkpre[nchunks] = tot;
        if (d_out_len) *d_out_len = ngroups + tot;
        enc_report(status, epoch, 0u);
        *meta.counters = 0;
    }
}

// bytes S .. S+15 of the 32-byte window a ++ b (S in [0, 16])
__device__ __forceinline__ uint4 window16(const uint4& a, const uint4& b, uint32_t S) {
    const uint32_t r = (S & 3u) * 8u;
    uint32_t w0, w1, w2, w3, w4;
    switch (S >> 2) {
        case 0: w0 = a.x; w1 = a.y; w2 = a.z; w3 = a.w; w4 = b.x; break;
        case 1: w0 = a.y; w1 = a.z; w2 = a.w; w3 = b.x; w4 = b.y; break;
        case 2: w0 = a.z; w1 = a.w; w2 = b.x; w3 = b.y; w4 = b.z; break;
        case 3: w0 = a.w; w1 = b.x; w2 = b.y; w3 = b.z; w4 = b.w; break;
        default: w0 = b.x; w1 = b.y; w2 = b.z; w3 = b.w; w4 = 0; break;
    }
    return make_uint4(__funnelshift_r(w0, w1, r), __funnelshift_r(w1, w2, r), __funnelshift_r(w2, w3, r),
                      __funnelshift_r(w3, w4, r));
}

__device__ __forceinline__ uint4 shfl_up4(const uint4& v, int d) {
    return make_uint4(__shfl_up_sync(kFull, v.x, d), __shfl_up_sync(kFull, v.y, d), __shfl_up_sync(kFull, v.z, d),
                      __shfl_up_sync(kFull, v.w, d));
}
__device__ __forceinline__ uint4 shfl4(const uint4& v, int l) {
    return make_uint4(__shfl_sync(kFull, v.x, l), __shfl_sync(kFull, v.y, l), __shfl_sync(kFull, v.z, l),
                      __shfl_sync(kFull, v.w, l));
}

__global__ void __launch_bounds__(kCTThreads)
    svb_encode_compact_kernel(uint8_t* __restrict__ out, uint64_t n, DecodeMeta meta, uint8_t* __restrict__ slots) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint32_t ntiles = (uint32_t)((nsub + kCTWarps - 1) / kCTWarps);
    const uint32_t t = blockIdx.x * kCTWarps + warp;
    if (t >= ntiles) return;
    constexpr uint32_t kTilesPerChunk = kChunkSubs / kCTWarps;
    const uint32_t c = t / kTilesPerChunk, t0 = c * kTilesPerChunk;
    const uint32_t x = (t0 + lane < ntiles && lane < (int)kTilesPerChunk) ? __ldcg(meta.tilesize + t0 + lane) : 0u;
    const uint32_t pre = __reduce_add_sync(kFull, (uint32_t)lane < t - t0 ? x : 0u);
    const uint32_t size = __shfl_sync(kFull, x, (int)(t - t0));
    if (size == 0) return;
    const uintptr_t D = (uintptr_t)out + ngroups + __ldcg(meta.chunkpre + c) + pre;
    const uint32_t p = (uint32_t)(D & 15);
    const uintptr_t Dal = D - p, Dend = D + size;
    const uint32_t nout = (p + size + 15) >> 4;  // destination granules touched
    const uint8_t* src = slots + (size_t)t * kSlotStride;
    uint4 carry = make_uint4(0, 0, 0, 0);
    for (uint32_t k0 = 0; k0 < nout; k0 += 128) {
        uint4 cur[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t k = k0 + 32 * u + lane;
            cur[u] = k < nout ? __ldcg(reinterpret_cast<const uint4*>(src) + k) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t k = k0 + 32 * u + lane;
            uint4 prv = shfl_up4(cur[u], 1);
            if (lane == 0) prv = carry;
            carry = shfl4(cur[u], 31);
            if (k < nout) {
                // destination granule k = slot bytes [16k - p, 16k - p + 16)
                const uint4 v = window16(prv, cur[u], 16u - p);
                const uintptr_t a = Dal + 16 * (uintptr_t)k;
                if (a >= D && a + 16 <= Dend) {
                    *reinterpret_cast<uint4*>(a) = v;
                } else {
                    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int bi = 0; bi < 16; ++bi)
                        if (a + bi >= D && a + bi < Dend)
                            *reinterpret_cast<uint8_t*>(a + bi) = (uint8_t)(w[bi >> 2] >> (8 * (bi & 3)));
                }
            }
        }
        // the slot lines just read are dead: drop them from L2 without a write-back
        if (lane < 16 && 16 * (k0 + 8 * lane) < 16 * nout)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(src + 16 * (size_t)k0 + 128 * lane) : "memory");
    }
}

// ---------------------------------------------------------------------------
// 4. one-pass encode with deferred look-back
// ---------------------------------------------------------------------------
// Replaces slot encode + compaction (or size scan + tile encode): the integers are
// read once and the compressed bytes written once, straight to their final place.
// Persistent CTAs (cooperative launch: all co-resident) take tiles t = b, b + G, ...
// Warps 0-7 (consumers) own one 1024-integer sub-tile of every tile; warp 8 (producer)
// TMA-loads each tile's 8192 integers (+ the 4 before them) into a 3-stage ring; warp 9
// (scanner) does the tile-level bookkeeping, so the consumers never wait on each other:
//   consumers, round r (tile t): size their sub-tile, write its control bytes to their
//     final place (their position depends on no data size), pack the data at phase 0 in
//     place, post the sub-tile size (mbarrier `sizes`); then store the PREVIOUS tile
//     tp = t - G once the scanner has posted its data offset (mbarrier `carried`):
//     realigned to the destination's 16-B phase, and release its stage;
//   scanner, round r: resolve tp's offset -- its own inclusive offset from the round
//     before + the epoch-tagged aggregates of the G - 1 tiles in between, published by
//     the other CTAs' scanners at least a round earlier -- post it, then wait for tile
//     t's eight sizes and publish t's aggregate.
// Round-r aggregates depend only on rounds < r, so once every CTA is resident there
// is no cycle; a consumer only waits when the scanner's look-back is slower than its
// own sizing + packing of the next tile.
#ifndef BC_E1_W
#define BC_E1_W 8       // consumer warps = sub-tiles per tile
#endif
#ifndef BC_E1_STAGES
#define BC_E1_STAGES 3  // stages per CTA: one loading, one being packed, kE1Defer waiting for their offset
#endif
constexpr int kE1W = BC_E1_W;
constexpr int kE1Stages = BC_E1_STAGES;
#ifndef BC_E1_DEFER
#define BC_E1_DEFER 1   // a tile is stored this many rounds after it was packed (stages - 1 - this = tiles loading)
#endif
constexpr int kE1Defer = BC_E1_DEFER;
#ifndef BC_E1_ROWS
#define BC_E1_ROWS 8    // rows of 128 integers per sub-tile (plain streams; delta streams keep 8)
#endif
constexpr int e1_rows(bool delta) { return delta ? kWTRows : BC_E1_ROWS; }
constexpr uint32_t e1_ints(bool delta) { return (uint32_t)kE1W * 128u * e1_rows(delta); }  // integers per tile
constexpr uint32_t e1_stride(bool delta) { return 16 + e1_ints(delta) * 4 + 16; }         // prefix, tile, slack
constexpr int kE1Threads = 32 * kE1W + 64;                  // consumers, producer, scanner
constexpr int kE1Producer = kE1W, kE1Scanner = kE1W + 1;
static_assert(kE1W * BC_E1_ROWS >= 32 && kE1W <= 8 && kE1Defer >= 1 && kE1Defer <= kE1Stages - 2 && BC_E1_ROWS <= kWTRows,
              "tile geometry (the aggregate array holds a tile per 1024 groups)");

struct __align__(16) E1Shared {
    uint64_t full[kE1Stages], empty[kE1Stages];
    uint64_t sizes[kE1Stages], carried[kE1Stages];  // per tile slot (round % kE1Stages, as the stage)
    uint32_t wsum[kE1Stages][kE1W];                 // sub-tile data sizes of the slot's tile
    unsigned long long carry[kE1Stages];            // data offset of the slot's tile
};

template <bool kDelta, bool kTrace>
__global__ void __launch_bounds__(kE1Threads, 2)
    svb_encode1_kernel(const uint32_t* __restrict__ in, uint64_t n, uint32_t prev, uint8_t* __restrict__ out,
                       DecodeMeta meta, uint64_t* __restrict__ d_out_len, unsigned long long* status, uint32_t epoch) {
    extern __shared__ __align__(128) uint8_t dsm[];
    __shared__ E1Shared sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    constexpr int kR = e1_rows(kDelta);                       // rows per sub-tile
    constexpr uint32_t kSubInts = 128u * kR, kSubGroups = 32u * kR;
    constexpr uint32_t kE1Ints = e1_ints(kDelta), kE1Stride = e1_stride(kDelta);
    const uint64_t nsub = (ngroups + kSubGroups - 1) / kSubGroups;
    const uint32_t ntiles = (uint32_t)((nsub + kE1W - 1) / kE1W);
    const uint32_t G = gridDim.x;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < kE1Stages; ++k) {
            mbar_init(&sh.full[k], 1);
            mbar_init(&sh.empty[k], kE1W);
        }
#pragma unroll
        for (int k = 0; k < kE1Stages; ++k) {
            mbar_init(&sh.sizes[k], kE1W);
            mbar_init(&sh.carried[k], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kE1Producer) {
        // ---- producer: the tile's integers (and the 4 before them) -> stage ----
        const uintptr_t lo = (uintptr_t)in, hi = lo + 4 * n;
        uint32_t k = 0, ph = 0;
        int st = 0;
        for (uint32_t t = blockIdx.x; t < ntiles; t += G, ++k, st = st + 1 == kE1Stages ? 0 : st + 1, ph ^= st == 0) {
            uint8_t* stage = dsm + (uint32_t)st * kE1Stride;
            if (k >= (uint32_t)kE1Stages) mbar_wait_parity_lazy(&sh.empty[st], ph ^ 1u, 512);
            const uint64_t i0 = (uint64_t)t * kE1Ints;
            const uint64_t cnt = n - i0 < (uint64_t)kE1Ints ? n - i0 : (uint64_t)kE1Ints;
            const uintptr_t beg = (uintptr_t)(in + i0) - (t ? 16 : 0), end = (uintptr_t)(in + i0 + cnt);
            uint8_t* dst = stage + (t ? 0 : 16);
            const uint32_t tx = tma_cover_bytes(beg, end, lo, hi);
            if (tx != 0xFFFFFFFFu && tx) {
                if (lane == 0) {
                    fence_async_smem();
                    mbar_expect(&sh.full[st], tx);
                    if (kTrace) meta.trace[8ull * t + 0] = gtimer();
                    tma_load_hint(dst, reinterpret_cast<const void*>(beg), tx, &sh.full[st], l2_policy_drop());
                }
            } else {
                uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
                const uint32_t words = (uint32_t)((end - beg) >> 2);
                for (uint32_t i = lane; i < words; i += 32) d32[i] = __ldg(reinterpret_cast<const uint32_t*>(beg) + i);
                __syncwarp();
                if (lane == 0) mbar_arrive(&sh.full[st]);
            }
        }
        return;
    }
    if (warp == kE1Scanner) {
        // ---- scanner: tile offsets (deferred look-back) and tile aggregates ----
        unsigned long long incl = 0;  // inclusive data offset of the CTA's last resolved tile
        uint32_t aprev = 0;           // aggregate of tprev
        // window of tile tp: tiles wl .. tp - 1 lie between the CTA's own tiles tp - G and tp;
        // read as 16-B aligned pairs, 8 per lane (512 tiles) issued before the wait for the
        // current tile's sizes, so the L2 round trip overlaps the consumers' work
        ulonglong2 v[8];
        auto issue = [&](uint32_t tp) {
            const uint32_t wl = tp + 1 > G ? tp + 1 - G : 0u;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t e = (wl & ~1u) + 64 * u + 2 * lane;
                v[u] = e < tp ? ld_relaxed_u64x2(meta.agg + e) : make_ulonglong2(0ull, 0ull);
            }
        };
        // pairs of tile tp's window (from e0) that still hold an older tag are re-read, all of a
        // lane's re-reads in flight together; true when this lane re-read any
        auto refresh = [&](uint32_t tp, uint32_t e0) -> bool {
            const uint32_t wl = tp + 1 > G ? tp + 1 - G : 0u;
            bool stale = false;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t e = e0 + 64 * u + 2 * lane;
                const bool nx = e < tp && e >= wl && (uint32_t)(v[u].x >> 32) != epoch;
                const bool ny = e + 1 < tp && e + 1 >= wl && (uint32_t)(v[u].y >> 32) != epoch;
                if (nx || ny) {
                    v[u] = ld_relaxed_u64x2(meta.agg + e);
                    stale = true;
                }
            }
            return stale;
        };
        auto resolve = [&](uint32_t tp, int q) {
            const uint32_t wl = tp + 1 > G ? tp + 1 - G : 0u;
            uint32_t part = 0;
            for (uint32_t e0 = (wl & ~1u); e0 < tp; e0 += 512) {
                if (e0 != (wl & ~1u)) {  // windows beyond 512 tiles (G > 513)
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t e = e0 + 64 * u + 2 * lane;
                        v[u] = e < tp ? ld_relaxed_u64x2(meta.agg + e) : make_ulonglong2(0ull, 0ull);
                    }
                }
                while (refresh(tp, e0)) {}
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t e = e0 + 64 * u + 2 * lane;
                    if (e < tp && e >= wl) part += (uint32_t)v[u].x;
                    if (e + 1 < tp && e + 1 >= wl) part += (uint32_t)v[u].y;
                }
            }
            part = __reduce_add_sync(kFull, part);
            const unsigned long long c = (tp >= G ? incl : 0ull) + part;  // data offset of tile tp
            incl = c + aprev;
            if (lane == 0) {
                sh.carry[q] = c;
                mbar_arrive(&sh.carried[q]);
                if (kTrace) meta.trace[8ull * tp + 4] = gtimer();
                if (tp == ntiles - 1) {
                    if (d_out_len) *d_out_len = ngroups + incl;
                    if (status) *status = ((unsigned long long)epoch << 32);
                }
            }
        };
        // round k: issue the previous tile's window loads, publish tile t's aggregate as soon
        // as its eight sizes are posted, then resolve the previous tile while the consumers
        // pack tile t (its window's aggregates are from rounds <= k - 1)
        uint32_t k = 0, tprev = 0;
        int q = 0, qp = 0;
        for (uint32_t t = blockIdx.x; t < ntiles; t += G, ++k, qp = q, q = q + 1 == kE1Stages ? 0 : q + 1) {
            // The window loads go out when the consumers start this round (they have stored a
            // tile and freed its stage), about one L2 round trip (~2 us under load) before the
            // offset is needed.  Issued right after the previous resolve they sampled the other
            // CTAs' aggregates too early, many not yet published, and the re-read after the sizes
            // was a second round trip on the consumers' critical path (cfg3 387 -> 379 us).
            // Sampling early as well was slower: with a blocking re-read at the round start 401 us,
            // with a second register set used when complete 385 us (twice the polling loads, and
            // CTAs whose offset comes early run ahead of the ones they later wait for).  A fixed
            // delay after the previous resolve instead of the round start: 0.4 / 0.7 / 1.0 / 1.3 /
            // 1.7 us -> 379 / 377 / 365 / 369 / 389 us (the round start is ~1.1 us after it).
            if (k >= 1 + kE1Defer)
                mbar_wait_parity_lazy(&sh.empty[(k - 1 - kE1Defer) % kE1Stages], ((k - 1 - kE1Defer) / kE1Stages) & 1u, 128);
            if (k) issue(tprev);
            mbar_wait_parity_lazy(&sh.sizes[q], (k / kE1Stages) & 1u, 256);
            uint32_t a = lane < kE1W ? sh.wsum[q][lane] : 0u;
            a = __reduce_add_sync(kFull, a);
            if (lane == 0) {
                st_relaxed_u64(meta.agg + t, ((unsigned long long)epoch << 32) | a);
                if (kTrace) meta.trace[8ull * t + 3] = gtimer();
            }
            if (k) resolve(tprev, qp);
            aprev = a;
            tprev = t;
        }
        if (k) {
            issue(tprev);
            resolve(tprev, qp);
        }
        return;
    }
    // ---- consumers ----
    auto store_prev = [&](uint32_t tp, int st, int q, uint32_t kk) {
        if (kTrace && threadIdx.x == 0) meta.trace[8ull * tp + 6] = gtimer();
        if (!mbar_test_parity(&sh.carried[q], (kk / kE1Stages) & 1u))
            mbar_wait_parity_lazy(&sh.carried[q], (kk / kE1Stages) & 1u, 128);
        if (kTrace && threadIdx.x == 0) meta.trace[8ull * tp + 7] = gtimer();
        const uint64_t s = (uint64_t)tp * kE1W + warp;
        if (s < nsub) {
            uint32_t pre = 0;
#pragma unroll
            for (int w = 0; w < kE1W; ++w) pre += w < warp ? sh.wsum[q][w] : 0u;
            const uint32_t src = sh_addr(dsm) + (uint32_t)st * kE1Stride + 16 + (uint32_t)warp * (kSubInts * 4);
            store_realigned2(src, sh.wsum[q][warp], out + ngroups + sh.carry[q] + pre);
        }
        __syncwarp();
        if (lane == 0) {
            if (kTrace && warp == 0) meta.trace[8ull * tp + 5] = gtimer();
            mbar_arrive(&sh.empty[st]);
        }
    };

    // stage = tile slot = k % kE1Stages; tile k is stored in round k + kE1Defer
    uint32_t k = 0, ph = 0;
    int st = 0;
    auto store_kth = [&](uint32_t kk) {  // the CTA's kk-th tile
        const int sk = (int)(kk % kE1Stages);
        store_prev(blockIdx.x + kk * G, sk, sk, kk);
    };
    for (uint32_t t = blockIdx.x; t < ntiles; t += G, ++k, st = st + 1 == kE1Stages ? 0 : st + 1, ph ^= st == 0) {
        const int q = st;
        if (kTrace && threadIdx.x == 0) meta.trace[8ull * t + 1] = gtimer();
        mbar_wait_parity(&sh.full[st], ph);
        if (kTrace && threadIdx.x == 0) meta.trace[8ull * t + 2] = gtimer();
        uint8_t* stage = dsm + (uint32_t)st * kE1Stride;
        const uint64_t s = (uint64_t)t * kE1W + warp;
        const uint64_t g0 = s * kSubGroups;
        auto post = [&](uint32_t total) {  // the sub-tile's data size -> the scanner
            if (lane == 0) {
                sh.wsum[q][warp] = total;
                mbar_arrive(&sh.sizes[q]);
            }
        };
        if (g0 < ngroups) {
            const uint32_t sin = sh_addr(stage) + 16 + (uint32_t)warp * (kSubInts * 4);
            const uint32_t prev_w = warp ? lds32(sin - 4) : (t ? lds32(sh_addr(stage) + 12) : prev);
            uint8_t* cdst = out + g0;
            if ((s + 1) * kSubInts <= n) {
                // delta streams of sorted ids are mostly all-small: check that first
                const bool small = kDelta && enc_full_small<kDelta>(sin, prev_w);
                if (small) {
                    post(kSubInts);
                    if ((((uintptr_t)cdst) & 15) == 0) {  // 256 zero control bytes
                        if (lane < (int)(kSubGroups / 16)) reinterpret_cast<uint4*>(cdst)[lane] = make_uint4(0, 0, 0, 0);
                    } else {
                        for (uint32_t i = lane; i < kSubGroups; i += 32) cdst[i] = 0;
                    }
                    enc_full_small_pack0<kDelta>(sin, prev_w, sin);
                } else {
                    // control bytes straight to the stream, the size posted, then the
                    // branch-free word pack at phase 0 in place (svb_pack.cuh)
                    uint32_t cw[2], qw[4];
                    const uint32_t total = enc_lengths2<kDelta, false, kR>(sin, prev_w, cdst, cw, qw, post);
                    __syncwarp();
                    enc_pack2<kDelta, false, kR>(sin, prev_w, cw, qw, sin, total);
                }
            } else {
                // the stream's last, partial sub-tile
                EncodeTile tt;
                uint32_t P[3] = {0, 0, 0};
                uint32_t last_w = prev_w;
                const uint8_t* sbytes = stage + 16 + warp * (kSubInts * 4);
#pragma unroll
                for (int j = 0; j < kWTRows; ++j) {
                    if (j >= kR) {  // the sub-tile has kR rows: none beyond
                        tt.d[j] = make_uint4(0, 0, 0, 0);
                        tt.lens[j] = 0;
                        continue;
                    }
                    const uint32_t cnt = group_count(g0 + 32 * j + lane, ngroups, tail_r);
                    uint4 x = mask_tail(*reinterpret_cast<const uint4*>(sbytes + 512 * j + 16 * lane), cnt);
                    if constexpr (kDelta) {
                        uint32_t p = __shfl_up_sync(kFull, x.w, 1);
                        if (lane == 0) p = last_w;
                        last_w = __shfl_sync(kFull, x.w, 31);
                        x = make_uint4(x.x - p, x.y - x.x, x.z - x.y, x.w - x.z);
                    }
                    tt.d[j] = x;
                    const uint32_t l0 = cnt > 0 ? dev_byte_length(x.x) : 0u;
                    const uint32_t l1 = cnt > 1 ? dev_byte_length(x.y) : 0u;
                    const uint32_t l2 = cnt > 2 ? dev_byte_length(x.z) : 0u;
                    const uint32_t l3 = cnt > 3 ? dev_byte_length(x.w) : 0u;
                    tt.lens[j] = l0 | (l1 << 8) | (l2 << 16) | (l3 << 24);
                    P[j / 3] |= (l0 + l1 + l2 + l3) << (10 * (j % 3));
                    if (cnt)
                        cdst[32 * j + lane] = (uint8_t)((l0 - 1) | (l1 ? ((l1 - 1) << 2) : 0u) |
                                                        (l2 ? ((l2 - 1) << 4) : 0u) | (l3 ? ((l3 - 1) << 6) : 0u));
                }
                tt.total = packed_row_scan(P, tt.qw);
                post(tt.total);
                __syncwarp();
                encode_pack_at(tt, stage + 16 + warp * (kSubInts * 4), 0);
            }
        } else {
            post(0u);
        }
        __syncwarp();
        if (k >= (uint32_t)kE1Defer) store_kth(k - kE1Defer);
    }
    for (uint32_t kk = k > (uint32_t)kE1Defer ? k - kE1Defer : 0u; kk < k; ++kk) store_kth(kk);
}

// ---------------------------------------------------------------------------
// 4b. one-pass encode for delta streams: the same tiles and deferred look-back, with the
// tile bookkeeping done by all consumer threads between named barriers (round 1's
// kernel).  Delta streams of sorted ids are mostly all-small sub-tiles whose packing is
// short, so nothing would hide a scanner warp's look-back latency behind consumer work;
// here the look-back loads of the previous tile are issued a whole round before they are
// needed (cfg2: 65 vs 78 us for the scanner kernel; plain cfg3: 543 vs 472 us).
// ---------------------------------------------------------------------------
constexpr int kD1eStages = 3;
constexpr uint32_t kD1eInts = kCTWarps * kWTInts;                          // 8192 per tile
constexpr uint32_t kD1eStride = 16 + kD1eInts * 4 + 16 + kCTWarps * kWTGroups;  // prefix, tile, slack, ctrl

struct __align__(16) D1eShared {
    uint64_t full[kD1eStages], empty[kD1eStages];
    uint32_t wsum[3][kCTWarps];
    uint32_t wpre[kCTWarps];  // exclusive prefix of the resolved tile's sub-tile sizes
    uint32_t red[kCTWarps];
    unsigned long long carry, incl;
};

template <bool kDelta, bool kTrace>
__global__ void __launch_bounds__(kCTThreads + 32, 2)
    svb_encode1d_kernel(const uint32_t* __restrict__ in, uint64_t n, uint32_t prev, uint8_t* __restrict__ out,
                       DecodeMeta meta, uint64_t* __restrict__ d_out_len, unsigned long long* status, uint32_t epoch) {
    extern __shared__ __align__(128) uint8_t dsm[];
    __shared__ D1eShared sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint32_t ntiles = (uint32_t)((nsub + kCTWarps - 1) / kCTWarps);
    const uint32_t G = gridDim.x;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < kD1eStages; ++k) {
            mbar_init(&sh.full[k], 1);
            mbar_init(&sh.empty[k], kCTWarps);
        }
        sh.incl = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kCTWarps) {
        // ---- producer: the tile's integers (and the 4 before them) -> stage ----
        const uintptr_t lo = (uintptr_t)in, hi = lo + 4 * n;
        uint32_t k = 0, ph = 0;
        int st = 0;
        for (uint32_t t = blockIdx.x; t < ntiles; t += G, ++k, st = st + 1 == kD1eStages ? 0 : st + 1, ph ^= st == 0) {
            uint8_t* stage = dsm + (uint32_t)st * kD1eStride;
            if (k >= (uint32_t)kD1eStages) mbar_wait_parity_sleep(&sh.empty[st], ph ^ 1u);
            const uint64_t i0 = (uint64_t)t * kD1eInts;
            const uint64_t cnt = n - i0 < (uint64_t)kD1eInts ? n - i0 : (uint64_t)kD1eInts;
            const uintptr_t beg = (uintptr_t)(in + i0) - (t ? 16 : 0), end = (uintptr_t)(in + i0 + cnt);
            uint8_t* dst = stage + (t ? 0 : 16);
            const uint32_t tx = tma_cover_bytes(beg, end, lo, hi);
            if (tx != 0xFFFFFFFFu && tx) {
                if (lane == 0) {
                    fence_async_smem();
                    mbar_expect(&sh.full[st], tx);
                    if (kTrace) meta.trace[8ull * t + 0] = gtimer();
                    tma_load_hint(dst, reinterpret_cast<const void*>(beg), tx, &sh.full[st], l2_policy_drop());
                }
            } else {
                uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
                const uint32_t words = (uint32_t)((end - beg) >> 2);
                for (uint32_t i = lane; i < words; i += 32) d32[i] = __ldg(reinterpret_cast<const uint32_t*>(beg) + i);
                __syncwarp();
                if (lane == 0) mbar_arrive(&sh.full[st]);
            }
        }
        return;
    }
    // ---- consumers ----
    const int ct = threadIdx.x;
    // look-back window of tile tp: tiles max(0, tp - G + 1) .. tp - 1, read as 16-B aligned
    // pairs (as svb_decode1_kernel); each thread prefetches one pair
    auto window_lo = [&](uint32_t tp) -> uint32_t { return tp + 1 > G ? tp + 1 - G : 0u; };
    ulonglong2 pf = make_ulonglong2(0ull, 0ull);
    auto prefetch = [&](uint32_t tp) {
        const uint32_t e = (window_lo(tp) & ~1u) + 2u * (uint32_t)ct;
        if (e < tp) pf = ld_relaxed_u64x2(meta.agg + e);
    };
    auto entry = [&](uint32_t j, unsigned long long v) -> uint32_t {
        while ((uint32_t)(v >> 32) != epoch) v = ld_relaxed_u64(meta.agg + j);
        return (uint32_t)v;
    };
    auto pair_sum = [&](uint32_t e, ulonglong2 v, uint32_t wl, uint32_t tp) -> uint32_t {
        uint32_t r = 0;
        if (e >= wl) r += entry(e, v.x);
        if (e + 1 < tp) r += entry(e + 1, v.y);
        return r;
    };
    auto resolve = [&](uint32_t tp, int st, int q) {
        const uint32_t wl = window_lo(tp);
        uint32_t part = 0;
        const uint32_t e0 = (wl & ~1u) + 2u * (uint32_t)ct;
        if (e0 < tp) part += pair_sum(e0, pf, wl, tp);
        for (uint32_t e = e0 + 512; e < tp; e += 512) part += pair_sum(e, ld_relaxed_u64x2(meta.agg + e), wl, tp);
        part = __reduce_add_sync(kFull, part);
        if (lane == 0) sh.red[warp] = part;
        consumers_sync();
        if (ct == 0) {
            unsigned long long x = 0;
            uint32_t a = 0;
#pragma unroll
            for (int w = 0; w < kCTWarps; ++w) {
                x += sh.red[w];
                a += sh.wsum[q][w];
            }
            const unsigned long long c = (tp >= G ? sh.incl : 0ull) + x;  // data offset of tile tp
            sh.carry = c;
            sh.incl = c + a;
            uint32_t pr = 0;
#pragma unroll
            for (int w = 0; w < kCTWarps; ++w) {
                sh.wpre[w] = pr;
                pr += sh.wsum[q][w];
            }
            if (tp == ntiles - 1) {
                if (d_out_len) *d_out_len = ngroups + c + a;
                if (status) *status = ((unsigned long long)epoch << 32);
            }
        }
        consumers_sync();
        if (kTrace && ct == 0) meta.trace[8ull * tp + 4] = gtimer();
        const uint64_t s = (uint64_t)tp * kCTWarps + warp;
        if (s < nsub) {
            const uint32_t src = sh_addr(dsm) + (uint32_t)st * kD1eStride + 16 + (uint32_t)warp * (kWTInts * 4);
            store_realigned2(src, sh.wsum[q][warp], out + ngroups + sh.carry + sh.wpre[warp]);
        }
        __syncwarp();
        if (kTrace && ct == 0) meta.trace[8ull * tp + 5] = gtimer();
        if (lane == 0) mbar_arrive(&sh.empty[st]);
    };

    uint32_t k = 0, tprev = 0, ph = 0;
    int st = 0, q = 0, stp = 0, qp = 0;  // stage / wsum slot of this iteration and of the previous one
    for (uint32_t t = blockIdx.x; t < ntiles;
         t += G, ++k, stp = st, qp = q, st = st + 1 == kD1eStages ? 0 : st + 1, q = q == 2 ? 0 : q + 1, ph ^= st == 0) {
        if (k) prefetch(tprev);
        if (kTrace && ct == 0) meta.trace[8ull * t + 1] = gtimer();
        mbar_wait_parity(&sh.full[st], ph);
        if (kTrace && ct == 0) meta.trace[8ull * t + 2] = gtimer();
        uint8_t* stage = dsm + (uint32_t)st * kD1eStride;
        const uint64_t s = (uint64_t)t * kCTWarps + warp;
        const uint64_t g0 = s * kWTGroups;
        uint32_t total = 0;
        if (g0 < ngroups) {
            const uint32_t sin = sh_addr(stage) + 16 + (uint32_t)warp * (kWTInts * 4);
            uint8_t* sctrl = stage + 16 + kD1eInts * 4 + 16 + warp * kWTGroups;
            const uint32_t prev_w = warp ? lds32(sin - 4) : (t ? lds32(sh_addr(stage) + 12) : prev);
            const uint32_t cnt_g = (uint32_t)(ngroups - g0 < (uint64_t)kWTGroups ? ngroups - g0 : (uint64_t)kWTGroups);
            uint8_t* cdst = out + g0;
            if ((s + 1) * kWTInts <= n) {
                const bool small = enc_full_small_pack0<kDelta>(sin, prev_w, sin);
                if (small) {
                    total = kWTInts;
                    if ((((uintptr_t)cdst) & 15) == 0) {  // 256 zero control bytes
                        if (lane < (int)(kWTGroups / 16)) reinterpret_cast<uint4*>(cdst)[lane] = make_uint4(0, 0, 0, 0);
                    } else {
                        for (uint32_t i = lane; i < kWTGroups; i += 32) cdst[i] = 0;
                    }
                } else {
                    // control bytes straight to the stream, then the branch-free word pack
                    // at phase 0 in place (svb_pack.cuh)
                    uint32_t cw[2], qw[4];
                    total = enc_lengths2<kDelta>(sin, prev_w, cdst, cw, qw, [](uint32_t) {});
                    __syncwarp();
                    enc_pack2<kDelta>(sin, prev_w, cw, qw, sin, total);
                }
            } else {
                // the stream's last, partial sub-tile
                EncodeTile tt;
                uint32_t P[3] = {0, 0, 0};
                uint32_t last_w = prev_w;
                const uint8_t* sbytes = stage + 16 + warp * (kWTInts * 4);
#pragma unroll
                for (int j = 0; j < kWTRows; ++j) {
                    const uint32_t cnt = group_count(g0 + 32 * j + lane, ngroups, tail_r);
                    uint4 x = mask_tail(*reinterpret_cast<const uint4*>(sbytes + 512 * j + 16 * lane), cnt);
                    if constexpr (kDelta) {
                        uint32_t p = __shfl_up_sync(kFull, x.w, 1);
                        if (lane == 0) p = last_w;
                        last_w = __shfl_sync(kFull, x.w, 31);
                        x = make_uint4(x.x - p, x.y - x.x, x.z - x.y, x.w - x.z);
                    }
                    tt.d[j] = x;
                    const uint32_t l0 = cnt > 0 ? dev_byte_length(x.x) : 0u;
                    const uint32_t l1 = cnt > 1 ? dev_byte_length(x.y) : 0u;
                    const uint32_t l2 = cnt > 2 ? dev_byte_length(x.z) : 0u;
                    const uint32_t l3 = cnt > 3 ? dev_byte_length(x.w) : 0u;
                    tt.lens[j] = l0 | (l1 << 8) | (l2 << 16) | (l3 << 24);
                    P[j / 3] |= (l0 + l1 + l2 + l3) << (10 * (j % 3));
                    if (cnt)
                        cdst[32 * j + lane] = (uint8_t)((l0 - 1) | (l1 ? ((l1 - 1) << 2) : 0u) |
                                                        (l2 ? ((l2 - 1) << 4) : 0u) | (l3 ? ((l3 - 1) << 6) : 0u));
                }
                tt.total = packed_row_scan(P, tt.qw);
                total = tt.total;
                __syncwarp();
                encode_pack_at(tt, stage + 16 + warp * (kWTInts * 4), 0);
            }
        }
        __syncwarp();
        if (lane == 0) sh.wsum[q][warp] = total;
        consumers_sync();
        if (ct == 0) {
            uint32_t a = 0;
#pragma unroll
            for (int w = 0; w < kCTWarps; ++w) a += sh.wsum[q][w];
            st_relaxed_u64(meta.agg + t, ((unsigned long long)epoch << 32) | a);
            if (kTrace) meta.trace[8ull * t + 3] = gtimer();
        }
        if (k) resolve(tprev, stp, qp);
        tprev = t;
    }
    if (k) {
        prefetch(tprev);
        resolve(tprev, (int)((k - 1) % kD1eStages), (int)((k - 1) % 3));
    }
}

// one-pass encode if the device can run it (cooperative launch, 16-B aligned input);
// *used = false leaves the call to the other paths
static cudaError_t launch_encode1(const uint32_t* in, uint64_t n, int delta, uint32_t prev, uint8_t* out,
                                  uint64_t* d_out_len, const DecodeMeta& m, unsigned long long* status, uint32_t epoch,
                                  cudaStream_t stream, bool* used, bool scanner) {
    *used = false;
    if (((uintptr_t)in) & 15) return cudaSuccess;
    // plain streams: the scanner kernel; delta streams: the barrier kernel (4b) unless asked
    const bool sk = !delta || scanner;
    const uint32_t smem = sk ? (uint32_t)kE1Stages * (delta ? e1_stride(true) : e1_stride(false))
                             : (uint32_t)(kD1eStages * kD1eStride);
    const int threads = sk ? kE1Threads : kCTThreads + 32;
    const void* fns[4];
    if (sk) {
        fns[0] = (const void*)svb_encode1_kernel<true, false>;
        fns[1] = (const void*)svb_encode1_kernel<false, false>;
        fns[2] = (const void*)svb_encode1_kernel<true, true>;
        fns[3] = (const void*)svb_encode1_kernel<false, true>;
    } else {
        fns[0] = (const void*)svb_encode1d_kernel<true, false>;
        fns[1] = (const void*)svb_encode1d_kernel<false, false>;
        fns[2] = (const void*)svb_encode1d_kernel<true, true>;
        fns[3] = (const void*)svb_encode1d_kernel<false, true>;
    }
    const int dev = launch_current_device();
    const int sms = launch_sms(dev), coop = launch_coop(dev);
    for (const void* f : fns) {
        const cudaError_t a = launch_ensure_smem(f, smem);
        if (a != cudaSuccess) return a;
    }
    const int o1 = launch_occupancy(fns[0], threads, smem);
    const int o2 = launch_occupancy(fns[1], threads, smem);
    const int occ = o1 < o2 ? o1 : o2;
    if (!coop || occ < 1) return cudaSuccess;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    // groups per tile (the scanner kernel's tile geometry is a build constant)
    const uint64_t tg = sk ? (uint64_t)kE1W * 32u * (uint64_t)(delta ? e1_rows(true) : e1_rows(false))
                           : (uint64_t)kCTWarps * kWTGroups;
    const uint64_t ntiles = (ngroups + tg - 1) / tg;
    uint64_t grid = (uint64_t)sms * (uint64_t)occ;
    if (grid > ntiles) grid = ntiles;
    DecodeMeta mm = m;
    void* args[] = {(void*)&in, (void*)&n, (void*)&prev, (void*)&out, (void*)&mm, (void*)&d_out_len, (void*)&status,
                    (void*)&epoch};
    const void* fn = fns[(m.trace ? 2 : 0) + (delta ? 0 : 1)];
    const cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(threads), args, smem, stream);
    if (e == cudaSuccess) *used = true;
    return e;
}

// ---------------------------------------------------------------------------
// launcher (metadata layout shared with the decode: localpre / chunkpre / counters)
// ---------------------------------------------------------------------------
uint64_t encode_slot_bytes(uint64_t n) {
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    return ((nsub + kCTWarps - 1) / kCTWarps) * (uint64_t)kSlotStride;
}

cudaError_t launch_encode3(const uint32_t* in, uint64_t n, int delta, uint32_t prev, uint8_t* out,
                           uint64_t* d_out_len, void* meta_ws, unsigned long long* status, uint32_t epoch,
                           cudaStream_t stream, int* launches, uint8_t* slots, uint32_t hints,
                           unsigned long long* trace) {
    DecodeMeta m = carve_decode_meta(meta_ws, n);
    m.trace = trace;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint32_t nchunks = (uint32_t)((nsub + kChunkSubs - 1) / kChunkSubs);
    if (hints & 0x100) {  // one-pass (the ctrl scan of a decode is not run here: clear the aggregates)
        bool used = false;
        const cudaError_t e =
            launch_encode1(in, n, delta, prev, out, d_out_len, m, status, epoch, stream, &used, (hints & 0x200) != 0);
        if (e != cudaSuccess) return e;
        if (used) {
            *launches = 1;
            return cudaSuccess;
        }
    }
    if (slots) {
        const uint64_t tiles_all = (nsub + kCTWarps - 1) / kCTWarps;
        if (delta)
            svb_encode_slot_kernel<true><<<(unsigned)tiles_all, kCTThreads, 0, stream>>>(in, n, prev, out, m, slots,
                                                                                        d_out_len, status, epoch, hints);
        else
            svb_encode_slot_kernel<false><<<(unsigned)tiles_all, kCTThreads, 0, stream>>>(in, n, prev, out, m, slots,
                                                                                         d_out_len, status, epoch, hints);
        svb_encode_compact_kernel<<<(unsigned)((tiles_all + kCTWarps - 1) / kCTWarps), kCTThreads, 0, stream>>>(
            out, n, m, slots);
        *launches = 2;
        return cudaGetLastError();
    }
    *launches = 2;
    return launch_encode_piece(in, n, delta, prev, out, d_out_len, meta_ws, status, epoch, 0, nchunks, stream);
}

// Chunks [c0, c1) of a two-read encode: size scan continuing from the running offset of
// the chunks before c0 (meta.running, left by the previous piece's scan), then the tile
// encode of those chunks.  Pieces must be issued in order on one stream.
cudaError_t launch_encode_piece(const uint32_t* in, uint64_t n, int delta, uint32_t prev, uint8_t* out,
                                uint64_t* d_out_len, void* meta_ws, unsigned long long* status, uint32_t epoch,
                                uint32_t c0, uint32_t c1, cudaStream_t stream) {
    const DecodeMeta m = carve_decode_meta(meta_ws, n);
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint32_t nchunks = (uint32_t)((nsub + kChunkSubs - 1) / kChunkSubs);
    constexpr uint32_t kTilesPerChunk = kChunkSubs / kCTWarps;
    if (c1 > nchunks) c1 = nchunks;
    if (c0 >= c1) return cudaSuccess;
    const uint64_t tiles_all = (nsub + kCTWarps - 1) / kCTWarps;
    const uint32_t t0 = c0 * kTilesPerChunk;
    const uint64_t t1_ = (uint64_t)c1 * kTilesPerChunk;
    const uint32_t t1 = (uint32_t)(t1_ < tiles_all ? t1_ : tiles_all);
    if (delta) {
        svb_size_scan_kernel<true><<<c1 - c0, 256, 0, stream>>>(in, n, prev, m, d_out_len, status, epoch, c0, nchunks);
        svb_encode_tile_kernel<true><<<t1 - t0, kCTThreads, 0, stream>>>(in, n, prev, out, m, t0);
    } else {
        svb_size_scan_kernel<false><<<c1 - c0, 256, 0, stream>>>(in, n, prev, m, d_out_len, status, epoch, c0, nchunks);
        svb_encode_tile_kernel<false><<<t1 - t0, kCTThreads, 0, stream>>>(in, n, prev, out, m, t0);
    }
    return cudaGetLastError();
}

cudaError_t launch_size_scan(const uint32_t* in, uint64_t n, int delta, uint32_t prev, void* meta_ws,
                             uint64_t* d_out_len, unsigned long long* status, uint32_t epoch, cudaStream_t stream) {
    const DecodeMeta m = carve_decode_meta(meta_ws, n);
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint32_t nchunks = (uint32_t)((nsub + kChunkSubs - 1) / kChunkSubs);
    if (delta)
        svb_size_scan_kernel<true><<<nchunks, 256, 0, stream>>>(in, n, prev, m, d_out_len, status, epoch, 0, nchunks);
    else
        svb_size_scan_kernel<false><<<nchunks, 256, 0, stream>>>(in, n, prev, m, d_out_len, status, epoch, 0, nchunks);
    return cudaGetLastError();
}

// device address of the running data offset (bytes after the last encoded piece)
unsigned long long* encode_running_ptr(void* meta_ws, uint64_t n) { return carve_decode_meta(meta_ws, n).running; }

}  // namespace bcgpu
