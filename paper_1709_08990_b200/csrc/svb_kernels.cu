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
// This file: block offsets (decoupled look-back over control-byte lengths),
// batched random-access block decode, the size-only batch pass, and the batch
// launchers (the kernels live in svb_batch2.cu; single arrays in svb_decode.cu /
// svb_encode.cu).
#include <cstdint>

#include "svb_device.cuh"
#include "svb_kernels.cuh"
#include "svb_warp.cuh"

namespace bcgpu {

__device__ __forceinline__ void report_status(unsigned long long* st, uint32_t epoch, uint32_t code) {
    if (st) *st = ((unsigned long long)epoch << 32) | code;
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

// ===========================================================================
// launchers
// ===========================================================================
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



// decode / encode batches: the warp-pipelined kernels of svb_batch2.cu
cudaError_t launch_decode_batch(const bcgpu_decode_segment* segs, uint64_t nseg, const uint8_t* in, uint32_t* out,
                                int delta, const BatchArgs& ba, cudaStream_t stream) {
    // short segments: one copy per segment (svb_batch3.cu); the rest: tile pipeline (svb_batch2.cu)
    cudaError_t e = launch_decode_batch3(segs, nseg, in, out, delta, ba, stream);
    if (e != cudaSuccess || (ba.max_seg_n != 0 && ba.max_seg_n <= kBatchSmallN)) return e;
    return launch_decode_batch2(segs, nseg, in, out, delta, ba, stream);
}

cudaError_t launch_encode_batch(const bcgpu_encode_segment* segs, uint64_t nseg, const uint32_t* in, uint8_t* out,
                                uint64_t* out_lens, int delta, const BatchArgs& ba, cudaStream_t stream) {
    // every segment: resident pieces (svb_batch3.cu)
    return launch_encode_batch3(segs, nseg, in, out, out_lens, delta, ba, stream);
}

cudaError_t launch_sizes_batch(const bcgpu_encode_segment* segs, uint64_t nseg, const uint32_t* in,
                               uint64_t* out_lens, int delta, const BatchArgs& ba, cudaStream_t stream) {
    // the segment-resident encode kernel's size-only variant (svb_batch3.cu)
    return launch_encode_batch3(segs, nseg, in, nullptr, out_lens, delta, ba, stream, true);
}

}  // namespace bcgpu
