// svb_kernels.cu -- sm_100a kernels for Stream VByte encode / decode / delta.
//
// Reference behaviour restated (paths under /root/reference):
//   svb_encode        proj/core/include/bytecodec/stream_vbyte.hpp:36
//   svb_decode        stream_vbyte.hpp:38-39
//   svb_decode_delta  stream_vbyte.hpp:41-42, codec.hpp:87-90
//   delta encode      codec.hpp:92-93 (base 0) + extension E2 (prev seed) SPEC.md:366-374
//   block offsets     stream_vbyte.hpp:48-49
//   decode block      stream_vbyte.hpp:51-54
//   chained chunks    codec.hpp:87-90, SPEC.md:555 (segmented batches)
//
// Kernel families:
//   * single array  -- one warp per 1024-integer tile (svb_warp.cuh), tiles in
//     blockIdx order, byte offsets and delta carries by decoupled look-back.
//   * batch         -- one warp per segment, tiles walked in order with the
//     offset and carry in registers (no look-back, no collective).
#include <cstdint>

#include "svb_device.cuh"
#include "svb_kernels.cuh"
#include "svb_warp.cuh"

namespace bcgpu {

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// debug trace: 8 timestamps per tile, written by thread 0
#define BC_TRACE(lb, tile, k)                                                  \
    do {                                                                       \
        if ((lb).trace && threadIdx.x == 0) (lb).trace[8 * (tile) + (k)] = global_ns(); \
    } while (0)

__device__ __forceinline__ void report_status(unsigned long long* st, uint32_t epoch, uint32_t code) {
    if (st) *st = ((unsigned long long)epoch << 32) | code;
}

// ===========================================================================
// single-array kernels: CTA look-back tile = 8 warp sub-tiles of 1024 integers
// ===========================================================================
// Each warp decodes its own 1024-integer sub-tile (svb_warp.cuh); the CTA's
// 8192 integers share one look-back status word per quantity, so the chip has
// ~600 look-back tiles in flight instead of ~4700, which the 256-wide
// look-back resolves in one or two round trips.
struct CtaShared {
    uint32_t tot[kCTWarps];  // per-warp data bytes
    uint32_t sum[kCTWarps];  // per-warp delta sums
    unsigned long long off, carry;
};

// exclusive prefix of this warp within the CTA + CTA total, from a per-warp smem array
__device__ __forceinline__ uint32_t cta_warp_prefix(const uint32_t* a, int warp, uint32_t* total) {
    uint32_t ex = 0, t = 0;
#pragma unroll
    for (int k = 0; k < kCTWarps; ++k) {
        const uint32_t x = a[k];
        ex += k < warp ? x : 0u;
        t += x;
    }
    *total = t;
    return ex;
}

template <bool kDelta>
__global__ void __launch_bounds__(kCTThreads, 4)
    svb_encode_ct_kernel(const uint32_t* __restrict__ in, uint64_t n, uint32_t prev, uint8_t* __restrict__ out,
                         uint64_t* __restrict__ d_out_len, LookbackArgs lb) {
    __shared__ __align__(128) uint8_t stage_all[kCTWarps][kWTStage];
    __shared__ CtaShared sh;
    const int warp = threadIdx.x >> 5;
    const uint32_t tile = blockIdx.x;
    uint8_t* stage = stage_all[warp];
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t g0 = (uint64_t)tile * kCTGroups + (uint64_t)warp * kWTGroups;
    uint32_t prev_in = prev;
    if (kDelta && g0 != 0 && g0 < ngroups) prev_in = __ldg(in + 4 * g0 - 1);
    EncodeTile t;
    encode_load<kDelta>(in, g0, ngroups, tail_r, prev_in, out, t);
    if ((threadIdx.x & 31) == 0) sh.tot[warp] = t.total;
    encode_pack(t, stage);
    __syncthreads();
    uint32_t ctot;
    const uint32_t wex = cta_warp_prefix(sh.tot, warp, &ctot);
    if (warp == 0) {
        lb_publish(lb.off_status, tile, lb.epoch, 0, ctot);
        const uint64_t off = lb_resolve(lb.off_status, tile, lb.epoch, 0, ctot);
        if ((threadIdx.x & 31) == 0) sh.off = off;
    }
    __syncthreads();
    const uint64_t cta_off = sh.off;
    encode_writeout(stage, (uintptr_t)out + ngroups + cta_off + wex, t.total);
    if (tile == lb.num_tiles - 1 && threadIdx.x == 0) {
        if (d_out_len) *d_out_len = ngroups + cta_off + ctot;
        report_status(lb.status, lb.epoch, 0u);
    }
}

// ===========================================================================
// block offsets (CTA tiles of kTileGroups control bytes) and random access
// ===========================================================================
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
        if (lane == 0) st_relaxed_gpu(status_slot(status, tile), pack_status(epoch, kFlagAggregate, agg));
        const uint64_t ex = lookback_exclusive_wide(status, tile, epoch);
        if (lane == 0) st_relaxed_gpu(status_slot(status, tile), pack_status(epoch, kFlagInclusive, ex + agg));
        return ex;
    }
};

__global__ void __launch_bounds__(kThreads) svb_block_offsets_kernel(const uint8_t* __restrict__ in, uint64_t n,
                                                                     uint64_t* __restrict__ offsets, LookbackArgs lb) {
    __shared__ uint32_t warp_tot[kWarps];
    __shared__ unsigned long long bcast;
    const uint32_t tile = blockIdx.x;
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

// ===========================================================================
// batch kernels: one warp per segment, tiles in order, state in registers
// ===========================================================================
template <bool kDelta>
__global__ void __launch_bounds__(kWTThreads, 8)
    svb_decode_batch_kernel(const bcgpu_decode_segment* __restrict__ segs, uint64_t nseg,
                            const uint8_t* __restrict__ in, uint32_t* __restrict__ out, unsigned long long* status,
                            uint32_t epoch) {
    __shared__ __align__(128) uint8_t stage_all[kWTWarps][kWTStage];
    __shared__ __align__(8) uint64_t bars[kWTWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* stage = stage_all[warp];
    uint64_t* bar = &bars[warp];
    if (lane == 0) mbar_init(bar, 1);
    __syncwarp();
    uint32_t phase = 0;
    bool used = false;
    const uint64_t gw = (uint64_t)blockIdx.x * kWTWarps + warp, nw = (uint64_t)gridDim.x * kWTWarps;
    for (uint64_t s = gw; s < nseg; s += nw) {
        const SegDesc d = load_desc_warp(segs, s);
        const uint64_t ngroups = ((uint64_t)d.n + 3) >> 2;
        const uint32_t tail_r = d.n & 3u;
        if (d.b < ngroups) {
            if (lane == 0) report_status(status, epoch, BCGPU_ERR_TRUNCATED);
            continue;
        }
        const uint8_t* seg = in + d.a;
        uint32_t* o = out + d.c;
        const bool out16 = (((uintptr_t)o) & 15) == 0;
        const uintptr_t lo = (uintptr_t)seg, hi = lo + d.b;
        uint64_t off = 0;
        uint32_t carry = d.prev;
        for (uint64_t g0 = 0; g0 < ngroups; g0 += kWTGroups) {
            const WarpCtrl w = load_warp_ctrl(seg, g0, ngroups, tail_r);
            const uintptr_t beg = lo + ngroups + off;
            __syncwarp();  // every lane is done reading the previous tile from stage
            stage_tile(stage, bar, phase, beg, beg + w.total, lo, hi, used);
            used = true;
            uint4 vv[kWTRows];
            const uint32_t tsum = expand_tile<kDelta>(w, stage, (uint32_t)(beg & 15), g0, ngroups, tail_r, o, out16, vv);
            if constexpr (kDelta) {
                store_tile<kDelta>(vv, carry, g0, ngroups, tail_r, o, out16);
                carry += tsum;
            }
            off += w.total;
        }
        if (lane == 0 && ngroups + off != d.b)
            report_status(status, epoch, ngroups + off > d.b ? BCGPU_ERR_TRUNCATED : BCGPU_ERR_TRAILING_BYTES);
    }
}

template <bool kDelta>
__global__ void __launch_bounds__(kWTThreads, 8)
    svb_encode_batch_kernel(const bcgpu_encode_segment* __restrict__ segs, uint64_t nseg,
                            const uint32_t* __restrict__ in, uint8_t* __restrict__ out,
                            uint64_t* __restrict__ out_lens, unsigned long long* status, uint32_t epoch) {
    __shared__ __align__(128) uint8_t stage_all[kWTWarps][kWTStage];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* stage = stage_all[warp];
    const uint64_t gw = (uint64_t)blockIdx.x * kWTWarps + warp, nw = (uint64_t)gridDim.x * kWTWarps;
    for (uint64_t s = gw; s < nseg; s += nw) {
        const SegDesc e = load_desc_warp(segs, s);
        const uint64_t ngroups = ((uint64_t)e.n + 3) >> 2;
        if (e.b < ngroups + 4ull * e.n) {
            if (lane == 0) report_status(status, epoch, BCGPU_ERR_INVALID_ARGUMENT);
            continue;
        }
        const uint32_t* src = in + e.a;
        uint8_t* dst = out + e.c;
        uint64_t off = 0;
        for (uint64_t g0 = 0; g0 < ngroups; g0 += kWTGroups) {
            const uint32_t prev_in = (kDelta && g0 != 0) ? __ldg(src + 4 * g0 - 1) : e.prev;
            EncodeTile t;
            encode_load<kDelta>(src, g0, ngroups, e.n & 3u, prev_in, dst, t);
            __syncwarp();  // previous tile's write-out finished reading stage
            encode_pack(t, stage);
            __syncwarp();
            encode_writeout(stage, (uintptr_t)dst + ngroups + off, t.total);
            off += t.total;
        }
        if (lane == 0) out_lens[s] = ngroups + off;
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
cudaError_t launch_encode(const uint32_t* in, uint64_t n, int delta, uint32_t prev, uint8_t* out,
                          uint64_t* d_out_len, const LookbackArgs& lb, cudaStream_t stream) {
    if (delta)
        svb_encode_ct_kernel<true><<<lb.num_tiles, kCTThreads, 0, stream>>>(in, n, prev, out, d_out_len, lb);
    else
        svb_encode_ct_kernel<false><<<lb.num_tiles, kCTThreads, 0, stream>>>(in, n, prev, out, d_out_len, lb);
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

static int occ_of(const void* k, int threads) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, 0) != cudaSuccess || occ < 1) occ = 1;
    return occ;
}

int occupancy_batch() {
    const int a = occ_of((const void*)svb_decode_batch_kernel<true>, kWTThreads);
    const int b = occ_of((const void*)svb_encode_batch_kernel<true>, kWTThreads);
    return a < b ? a : b;
}

static int batch_grid(uint64_t nseg, int grid_cap) {
    const uint64_t want = (nseg + kWTWarps - 1) / kWTWarps;
    return (int)(want < (uint64_t)grid_cap ? want : (uint64_t)grid_cap);
}

cudaError_t launch_decode_batch(const bcgpu_decode_segment* segs, uint64_t nseg, const uint8_t* in, uint32_t* out,
                                int delta, const BatchArgs& ba, cudaStream_t stream) {
    if (!(ba.flags & (64 | 256))) return launch_decode_batch2(segs, nseg, in, out, delta, ba, stream);
    const int grid = batch_grid(nseg, ba.grid);
    if (grid <= 0) return cudaSuccess;
    if (delta)
        svb_decode_batch_kernel<true><<<grid, kWTThreads, 0, stream>>>(segs, nseg, in, out, ba.status, ba.epoch);
    else
        svb_decode_batch_kernel<false><<<grid, kWTThreads, 0, stream>>>(segs, nseg, in, out, ba.status, ba.epoch);
    return cudaGetLastError();
}

cudaError_t launch_encode_batch(const bcgpu_encode_segment* segs, uint64_t nseg, const uint32_t* in, uint8_t* out,
                                uint64_t* out_lens, int delta, const BatchArgs& ba, cudaStream_t stream) {
    if (!(ba.flags & 64)) return launch_encode_batch2(segs, nseg, in, out, out_lens, delta, ba, stream);
    const int grid = batch_grid(nseg, ba.grid);
    if (grid <= 0) return cudaSuccess;
    if (delta)
        svb_encode_batch_kernel<true><<<grid, kWTThreads, 0, stream>>>(segs, nseg, in, out, out_lens, ba.status,
                                                                        ba.epoch);
    else
        svb_encode_batch_kernel<false><<<grid, kWTThreads, 0, stream>>>(segs, nseg, in, out, out_lens, ba.status,
                                                                         ba.epoch);
    return cudaGetLastError();
}

cudaError_t launch_sizes_batch(const bcgpu_encode_segment* segs, uint64_t nseg, const uint32_t* in,
                               uint64_t* out_lens, int delta, const BatchArgs& ba, cudaStream_t stream) {
    const uint64_t want = (nseg + kWarps - 1) / kWarps;
    const uint64_t cap = (uint64_t)ba.grid * kWTWarps / kWarps + 1;
    const int grid = (int)(want < cap ? want : cap);
    if (grid <= 0) return cudaSuccess;
    if (delta)
        svb_sizes_batch_kernel<true><<<grid, kThreads, 0, stream>>>(segs, nseg, in, out_lens);
    else
        svb_sizes_batch_kernel<false><<<grid, kThreads, 0, stream>>>(segs, nseg, in, out_lens);
    return cudaGetLastError();
}

}  // namespace bcgpu
