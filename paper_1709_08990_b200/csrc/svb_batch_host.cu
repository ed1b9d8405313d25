// svb_batch_host.cu -- device side of the host-buffer batch entry points
// (bcgpu_svb_{encode,decode}_batch_host in bcgpu_capi.cu).
//
// A host batch is given as per-segment counts (and delta bases) plus the values
// concatenated; encoded streams are packed back to back and their offsets returned.
// The pipelined host call cuts the batch into pieces of whole segments.  For each
// piece one CTA turns the counts into segment descriptors (exclusive scans of
// n -> element offsets, of encoded sizes -> packed byte offsets), so the batch
// kernels (svb_batch3.cu / svb_batch2.cu) run on it unchanged.  The per-segment
// contract is the reference's chained-chunk call, decode_payload_delta(codec,
// bytes, n, base, out) (codec.hpp:87-90).
#include <cstdint>

#include "bcgpu/bcgpu.h"
#include "svb_device.cuh"
#include "svb_kernels.cuh"

namespace bcgpu {
namespace {

constexpr int kDThreads = 1024;
constexpr int kDPer = 4;  // items per thread per round

// Exclusive scan of one round of kDThreads * kDPer values (thread t holds items
// kDPer t .. kDPer t + kDPer - 1 in v); returns the round total, v becomes exclusive
// prefixes (without the carry).
__device__ __forceinline__ uint64_t round_scan(uint64_t (&v)[kDPer], uint64_t* wsum) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint64_t s = 0;
#pragma unroll
    for (int j = 0; j < kDPer; ++j) {
        const uint64_t x = v[j];
        v[j] = s;
        s += x;
    }
    uint64_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    uint64_t wpre = 0, total = 0;
#pragma unroll 8
    for (int w = 0; w < kDThreads / 32; ++w) {
        const uint64_t x = wsum[w];
        wpre += w < warp ? x : 0ull;
        total += x;
    }
    __syncthreads();  // wsum is reused by the next round
    const uint64_t ex = wpre + incl - s;
#pragma unroll
    for (int j = 0; j < kDPer; ++j) v[j] += ex;
    return total;
}

// Encode descriptors of segments [s0, s0 + m): src_offset = elem_base + exclusive scan
// of n, dst_capacity = worst case; dst_offset is filled in by the pack kernel.
__global__ void __launch_bounds__(kDThreads) batch_encode_describe_kernel(const uint32_t* __restrict__ seg_n,
                                                                          const uint32_t* __restrict__ seg_prev,
                                                                          uint64_t s0, uint32_t m, uint64_t elem_base,
                                                                          bcgpu_encode_segment* __restrict__ es) {
    __shared__ uint64_t wsum[kDThreads / 32];
    uint64_t carry = elem_base;
    for (uint32_t r = 0; r < m; r += kDThreads * kDPer) {
        const uint32_t i0 = r + kDPer * threadIdx.x;
        uint64_t v[kDPer];
#pragma unroll
        for (int j = 0; j < kDPer; ++j) v[j] = i0 + j < m ? (uint64_t)seg_n[s0 + i0 + j] : 0ull;
        uint64_t nn[kDPer];
#pragma unroll
        for (int j = 0; j < kDPer; ++j) nn[j] = v[j];
        const uint64_t tot = round_scan(v, wsum);
#pragma unroll
        for (int j = 0; j < kDPer; ++j) {
            if (i0 + j < m) {
                bcgpu_encode_segment d;
                d.src_offset = carry + v[j];
                d.dst_capacity = ((nn[j] + 3) >> 2) + 4 * nn[j];
                d.dst_offset = 0;
                d.n = (uint32_t)nn[j];
                d.prev = seg_prev ? seg_prev[s0 + i0 + j] : 0u;
                es[s0 + i0 + j] = d;
            }
        }
        carry += tot;
    }
}

// Packs segments [s0, s0 + m) back to back after *running: dst_offset and
// out_offsets[s] = *running + exclusive scan of sizes; then *running += the piece's
// total and out_offsets[s0 + m] = the new running offset.
__global__ void __launch_bounds__(kDThreads) batch_pack_kernel(const uint64_t* __restrict__ sizes, uint64_t s0,
                                                               uint32_t m, bcgpu_encode_segment* __restrict__ es,
                                                               uint64_t* __restrict__ out_offsets,
                                                               unsigned long long* running) {
    __shared__ uint64_t wsum[kDThreads / 32];
    uint64_t carry = *running;
    for (uint32_t r = 0; r < m; r += kDThreads * kDPer) {
        const uint32_t i0 = r + kDPer * threadIdx.x;
        uint64_t v[kDPer];
#pragma unroll
        for (int j = 0; j < kDPer; ++j) v[j] = i0 + j < m ? sizes[s0 + i0 + j] : 0ull;
        const uint64_t tot = round_scan(v, wsum);
#pragma unroll
        for (int j = 0; j < kDPer; ++j) {
            if (i0 + j < m) {
                es[s0 + i0 + j].dst_offset = carry + v[j];
                out_offsets[s0 + i0 + j] = carry + v[j];
            }
        }
        carry += tot;
    }
    if (threadIdx.x == 0) {
        *running = carry;
        out_offsets[s0 + m] = carry;
    }
}

// Decode descriptors of segments [s0, s0 + m) from the packed stream offsets:
// src = [in_offsets[s], in_offsets[s + 1]), dst_offset = elem_base + exclusive scan of n.
__global__ void __launch_bounds__(kDThreads) batch_decode_describe_kernel(const uint32_t* __restrict__ seg_n,
                                                                          const uint32_t* __restrict__ seg_base,
                                                                          const uint64_t* __restrict__ in_offsets,
                                                                          uint64_t s0, uint32_t m, uint64_t elem_base,
                                                                          bcgpu_decode_segment* __restrict__ ds) {
    __shared__ uint64_t wsum[kDThreads / 32];
    uint64_t carry = elem_base;
    for (uint32_t r = 0; r < m; r += kDThreads * kDPer) {
        const uint32_t i0 = r + kDPer * threadIdx.x;
        uint64_t v[kDPer];
#pragma unroll
        for (int j = 0; j < kDPer; ++j) v[j] = i0 + j < m ? (uint64_t)seg_n[s0 + i0 + j] : 0ull;
        uint64_t nn[kDPer];
#pragma unroll
        for (int j = 0; j < kDPer; ++j) nn[j] = v[j];
        const uint64_t tot = round_scan(v, wsum);
#pragma unroll
        for (int j = 0; j < kDPer; ++j) {
            if (i0 + j < m) {
                const uint64_t s = s0 + i0 + j;
                bcgpu_decode_segment d;
                d.src_offset = in_offsets[s];
                d.src_bytes = in_offsets[s + 1] - in_offsets[s];
                d.dst_offset = carry + v[j];
                d.n = (uint32_t)nn[j];
                d.prev = seg_base ? seg_base[s] : 0u;
                ds[s] = d;
            }
        }
        carry += tot;
    }
}

}  // namespace

cudaError_t launch_batch_encode_describe(const uint32_t* seg_n, const uint32_t* seg_prev, uint64_t s0, uint32_t m,
                                         uint64_t elem_base, bcgpu_encode_segment* es, cudaStream_t stream) {
    if (m == 0) return cudaSuccess;
    batch_encode_describe_kernel<<<1, kDThreads, 0, stream>>>(seg_n, seg_prev, s0, m, elem_base, es);
    return cudaGetLastError();
}

cudaError_t launch_batch_pack(const uint64_t* sizes, uint64_t s0, uint32_t m, bcgpu_encode_segment* es,
                              uint64_t* out_offsets, unsigned long long* running, cudaStream_t stream) {
    batch_pack_kernel<<<1, kDThreads, 0, stream>>>(sizes, s0, m, es, out_offsets, running);
    return cudaGetLastError();
}

cudaError_t launch_batch_decode_describe(const uint32_t* seg_n, const uint32_t* seg_base, const uint64_t* in_offsets,
                                         uint64_t s0, uint32_t m, uint64_t elem_base, bcgpu_decode_segment* ds,
                                         cudaStream_t stream) {
    if (m == 0) return cudaSuccess;
    batch_decode_describe_kernel<<<1, kDThreads, 0, stream>>>(seg_n, seg_base, in_offsets, s0, m, elem_base, ds);
    return cudaGetLastError();
}

}  // namespace bcgpu
