// svb_encode.cu -- single-array Stream VByte encode for sm_100a (svb_encode,
// reference stream_vbyte.hpp:36; delta encode codec.hpp:92-93 and the
// prev-seeded extension E2).
//
// One launch: svb_encode_tile_kernel, one CTA per 8 sub-tiles of 1024 integers.
// Each warp TMA-loads its 4 KiB of integers (plus the preceding integer for the
// delta seed), classifies byte lengths (max(1, 4 - clz/8), codec.hpp:70-72),
// TMA-stores its 256 control bytes (field i of control byte k = len-1 in bits
// 2i), and packs the data bytes in place.  The CTA publishes
// its byte count right after the length scan and resolves its output offset
// with a TMA-polled decoupled look-back that overlaps the packing.
#include <cstdint>

#include "svb_device.cuh"
#include "svb_kernels.cuh"
#include "svb_tma.cuh"
#include "svb_warp.cuh"

namespace bcgpu {

__device__ __forceinline__ void trace_ts(const LookbackArgs& lb, uint32_t tile, int k) {
    if (lb.trace && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        lb.trace[8 * tile + k] = t;
    }
}

__device__ __forceinline__ void report_status_enc(unsigned long long* st, uint32_t epoch, uint32_t code) {
    if (st) *st = ((unsigned long long)epoch << 32) | code;
}

struct __align__(16) WarpBuf {
    uint8_t stage[kWTStage + 16];  // the sub-tile's integers at +16 (+ the 4 before), packed in place from 0
    uint8_t ctrl[kWTGroups];
};

static inline uint32_t encode_tiles(uint64_t n) {
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    return (uint32_t)((nsub + kCTWarps - 1) / kCTWarps);
}

// ---------------------------------------------------------------------------
// encode
// ---------------------------------------------------------------------------
constexpr int kEncWindow = 512;

struct EncShared {
    uint32_t tot[kCTWarps];
    unsigned long long off;
};

template <bool kDelta>
__global__ void __launch_bounds__(kCTThreads, 5)
    svb_encode_tile_kernel(const uint32_t* __restrict__ in, uint64_t n, uint32_t prev, uint8_t* __restrict__ out,
                           uint64_t* __restrict__ d_out_len, LookbackArgs lb) {
    __shared__ __align__(128) WarpBuf wb[kCTWarps];
    __shared__ __align__(8) uint64_t bars[kCTWarps];
    __shared__ __align__(128) LookbackWin<kEncWindow> lbw;
    __shared__ EncShared sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tile = blockIdx.x;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t sub = (uint64_t)tile * kCTWarps + warp;
    const uint64_t g0 = sub * kWTGroups;
    const bool active = g0 < ngroups;
    WarpBuf& b = wb[warp];
    trace_ts(lb, tile, 0);
    if (lane == 0) mbar_init1(&bars[warp]);
    if (threadIdx.x == 0) mbar_init1(&lbw.bar);
    __syncthreads();

    EncodeTile t;
    t.total = 0;
    uint32_t cnt_g = 0;
    if (active) {
        cnt_g = (uint32_t)(ngroups - g0 < (uint64_t)kWTGroups ? ngroups - g0 : (uint64_t)kWTGroups);
        const uint64_t i0 = 4 * g0;
        const uint32_t nints = (uint32_t)(n - i0 < (uint64_t)kWTInts ? n - i0 : (uint64_t)kWTInts);
        // stage [0,16): the 4 integers before the sub-tile (delta seed), [16, 16+4*nints): the sub-tile
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
            trace_ts(lb, tile, 1);
        } else {
            uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
            const uint32_t words = (uint32_t)((end - beg) >> 2);
            for (uint32_t i = lane; i < words; i += 32) d32[i] = __ldg(reinterpret_cast<const uint32_t*>(beg) + i);
            __syncwarp();
        }
        uint32_t P[3] = {0, 0, 0};
        uint32_t last_w = g0 ? reinterpret_cast<const uint32_t*>(b.stage)[3] : prev;
#pragma unroll
        for (int j = 0; j < kWTRows; ++j) {
            const uint32_t cnt = group_count(g0 + 32 * j + lane, ngroups, tail_r);
            uint4 x = *reinterpret_cast<const uint4*>(b.stage + 16 + 512 * j + 16 * lane);
            x = mask_tail(x, cnt);
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
        trace_ts(lb, tile, 2);
    }
    // publish the tile's byte count before packing so successors can look back past it
    if (lane == 0) sh.tot[warp] = t.total;
    __syncthreads();
    uint32_t wex = 0, ctot = 0;
#pragma unroll
    for (int k = 0; k < kCTWarps; ++k) {
        const uint32_t x = sh.tot[k];
        wex += k < warp ? x : 0u;
        ctot += x;
    }
    if (warp == 0) {
        // warp 0 resolves the tile offset right away, overlapping the other warps' packing
        lb_publish(lb.off_status, tile, lb.epoch, 0, ctot);
        uint32_t phase = 0;
        uint64_t off = 0;
        if (tile != 0) {
            if (lb.debug_flags & 2) {
                uint32_t st3[3] = {0, 0, 0};
                unsigned long long ta, tb;
                asm volatile("mov.u64 %0, %globaltimer;" : "=l"(ta));
                off = lookback_exclusive_wide(lb.off_status, tile, lb.epoch, st3);
                asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tb));
                if (lb.trace && lane == 0)
                    lb.trace[8 * tile + 7] = ((unsigned long long)(st3[1] & 0xFF) << 56) |
                                             ((unsigned long long)(st3[0] & 0xFF) << 48) |
                                             ((unsigned long long)(st3[2] / 1) & 0xFFFFFF) << 24 | ((tb - ta) & 0xFFFFFF);
            } else {
                off = lookback_tma<kEncWindow>(lb.off_status, tile, lb.epoch, lbw, phase,
                                               lb.trace ? lb.trace + 8 * tile + 7 : nullptr);
            }
            if (lane == 0) st_relaxed_gpu(lb.off_status + tile, pack_status(lb.epoch, kFlagInclusive, off + ctot));
        }
        if (lane == 0) sh.off = off;
    }
    if (active) {
        // control bytes: one bulk store of the 16-B multiple, byte stores for the rest
        uint8_t* cdst = out + g0;
        const uint32_t cb = (((uintptr_t)cdst & 15) == 0) ? (cnt_g & ~15u) : 0u;
        fence_async_smem();
        __syncwarp();
        if (lane == 0 && cb) {
            tma_store(cdst, b.ctrl, cb);
            tma_store_commit();
        }
        for (uint32_t i = cb + lane; i < cnt_g; i += 32) cdst[i] = b.ctrl[i];
        // in place: group g's packed bytes end at or before its own input (stage + 16 + 16 g)
        encode_pack(t, b.stage);
        trace_ts(lb, tile, 3);
    }
    trace_ts(lb, tile, 4);
    __syncthreads();
    trace_ts(lb, tile, 5);
    const uint64_t cta_off = sh.off;
    if (active) {
        __syncwarp();
        encode_writeout(b.stage, (uintptr_t)out + ngroups + cta_off + wex, t.total);
        if (lane == 0) tma_store_wait_read();
    }
    // (slot 7 carries the look-back statistics)
    if (tile == gridDim.x - 1 && threadIdx.x == 0) {
        if (d_out_len) *d_out_len = ngroups + cta_off + ctot;
        report_status_enc(lb.status, lb.epoch, 0u);
    }
}

cudaError_t launch_encode2(const uint32_t* in, uint64_t n, int delta, uint32_t prev, uint8_t* out,
                           uint64_t* d_out_len, const LookbackArgs& lb, cudaStream_t stream) {
    const int grid = (int)encode_tiles(n);
    if (delta)
        svb_encode_tile_kernel<true><<<grid, kCTThreads, 0, stream>>>(in, n, prev, out, d_out_len, lb);
    else
        svb_encode_tile_kernel<false><<<grid, kCTThreads, 0, stream>>>(in, n, prev, out, d_out_len, lb);
    return cudaGetLastError();
}

}  // namespace bcgpu
