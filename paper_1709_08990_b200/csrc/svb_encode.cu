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
#include "svb_kernels.cuh"
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
                         uint64_t* __restrict__ d_out_len, unsigned long long* status, uint32_t epoch) {
    __shared__ uint32_t wt[8];
    __shared__ unsigned long long wt64[8];
    __shared__ bool last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t chunk = blockIdx.x, nchunks = gridDim.x;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const bool in16 = (((uintptr_t)in) & 15) == 0;
    uint32_t my_size = 0;  // lane k < 8: size of sub-tile 8*warp + k
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
        const uint64_t s = (uint64_t)chunk * kChunkSubs + 8 * warp + k;
        if (s >= nsub) break;
        const uint64_t g0 = s * kWTGroups;
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
    if (tid == 0) meta.chunkpre[chunk] = total;
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
        if (d_out_len) *d_out_len = ngroups + tot;
        enc_report(status, epoch, 0u);
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
                           DecodeMeta meta) {
    __shared__ __align__(128) EncBuf wb[kCTWarps];
    __shared__ __align__(16) uint32_t slocal[kCTWarps + 8];
    __shared__ __align__(16) unsigned long long schunk[4];
    __shared__ __align__(8) uint64_t bars[kCTWarps + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tile = blockIdx.x;
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
    if (full) {
        // lengths, control bytes, tile-local offsets (lean path, svb_fast.cuh)
        total = enc_full_lengths<kDelta>(sh_addr(b.stage) + 16, prev_w, sh_addr(b.ctrl), lens, qw);
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
    if (full)
        enc_full_pack<kDelta>(sh_addr(b.stage) + 16, prev_w, lens, qw, sh_addr(b.stage) + head);
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
// launcher (metadata layout shared with the decode: localpre / chunkpre / counters)
// ---------------------------------------------------------------------------
cudaError_t launch_encode3(const uint32_t* in, uint64_t n, int delta, uint32_t prev, uint8_t* out,
                           uint64_t* d_out_len, void* meta_ws, unsigned long long* status, uint32_t epoch,
                           cudaStream_t stream, int* launches) {
    const DecodeMeta m = carve_decode_meta(meta_ws, n);
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint32_t nchunks = (uint32_t)((nsub + kChunkSubs - 1) / kChunkSubs);
    const uint32_t tiles = (uint32_t)((nsub + kCTWarps - 1) / kCTWarps);
    if (delta) {
        svb_size_scan_kernel<true><<<nchunks, 256, 0, stream>>>(in, n, prev, m, d_out_len, status, epoch);
        svb_encode_tile_kernel<true><<<tiles, kCTThreads, 0, stream>>>(in, n, prev, out, m);
    } else {
        svb_size_scan_kernel<false><<<nchunks, 256, 0, stream>>>(in, n, prev, m, d_out_len, status, epoch);
        svb_encode_tile_kernel<false><<<tiles, kCTThreads, 0, stream>>>(in, n, prev, out, m);
    }
    *launches = 2;
    return cudaGetLastError();
}

}  // namespace bcgpu
