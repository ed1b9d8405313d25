// svb_query.cu -- batched seek / select over one delta-coded Stream VByte stream
// (module stream_query: the reference's src/query.cpp has no header and
// is missing; its contract is restated there).
//
//   select(i)       : the i-th logical value (prefix sum of the payload through i, + base)
//   seek(target)    : the first (index, value) with value >= target over a non-decreasing
//                     sequence; ties resolve to the lowest index; not-found = index n
//
// A query never materialises the decoded stream.  One metadata pass -- the decode's control
// scan and sums pass (svb_decode.cu), then svb_endvals_kernel -- leaves per 1024-integer
// sub-tile its data offset and its last logical value (8 B per 1024 integers).  Then one warp
// per query decodes exactly one sub-tile straight from global memory: select picks the
// sub-tile by index; seek finds it with a 32-way search over the sub-tiles' last values (the
// sequence is non-decreasing, so they are too) and ballots for the first value >= target.
#include <cstdint>

#include "svb_device.cuh"
#include "svb_fast.cuh"
#include "svb_kernels.cuh"
#include "svb_scan.cuh"
#include "svb_warp.cuh"

namespace bcgpu {

// last logical value of every sub-tile: base + scanned chunk carry + inclusive sums in the chunk
__global__ void __launch_bounds__(256)
    svb_endvals_kernel(DecodeMeta meta, uint64_t nsub, uint32_t base, uint32_t* __restrict__ endval) {
    const int lane = threadIdx.x & 31;
    const uint64_t c = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // one warp per chunk
    const uint64_t s0 = c * kChunkSubs;
    if (s0 >= nsub) return;
    const uint64_t sa = s0 + 2 * lane, sb = sa + 1;
    const uint32_t a = sa < nsub ? __ldg(meta.subsums + sa) : 0u, b = sb < nsub ? __ldg(meta.subsums + sb) : 0u;
    const uint32_t I = warp_inclusive_scan(a + b);
    const uint32_t carry = base + __ldg(meta.chunksums + c) + I - (a + b);
    if (sa < nsub) endval[sa] = carry + a;
    if (sb < nsub) endval[sb] = carry + a + b;
}

// aligned 32-bit word at global address a; bytes outside [lo, hi) read as 0
__device__ __forceinline__ uint32_t qword(uintptr_t a, uintptr_t lo, uintptr_t hi) {
    if (a >= lo && a + 4 <= hi) return __ldg(reinterpret_cast<const uint32_t*>(a));
    uint32_t w = 0;
    for (int b = 0; b < 4; ++b)
        if (a + b >= lo && a + b < hi) w |= (uint32_t)__ldg(reinterpret_cast<const uint8_t*>(a + b)) << (8 * b);
    return w;
}

// kSeek = false: queries are indices (uint64), results: values.
// kSeek = true : queries are targets (uint32), results: indices (n = not found) + values.
template <bool kSeek>
__global__ void __launch_bounds__(256)
    svb_query_kernel(const uint8_t* __restrict__ in, uint64_t in_len, uint64_t n, uint32_t base, DecodeMeta meta,
                     const uint32_t* __restrict__ endval, const void* __restrict__ queries, uint64_t q,
                     uint64_t* __restrict__ out_index, uint32_t* __restrict__ out_value) {
    const int lane = threadIdx.x & 31;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uintptr_t lo = (uintptr_t)in, hi = lo + in_len, data0 = lo + ngroups;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t qi = gw; qi < q; qi += nw) {
        uint64_t s, want = 0;
        uint32_t target = 0;
        if constexpr (kSeek) {
            target = __ldg(reinterpret_cast<const uint32_t*>(queries) + qi);
            // first sub-tile whose last value >= target: 32-way search over endval[0, nsub)
            uint64_t lo_s = 0, hi_s = nsub;  // answer in [lo_s, hi_s]; hi_s = nsub: not found
            while (hi_s - lo_s > 0) {
                const uint64_t span = hi_s - lo_s;
                const uint64_t step = (span + 31) / 32;
                const uint64_t p = lo_s + (uint64_t)lane * step;
                const bool ge = p < hi_s ? __ldg(endval + p) >= target : true;
                const uint32_t m = __ballot_sync(kFull, ge);
                // first probe >= target; none: the answer lies past probe 31 (probe 32 >= hi_s)
                const int f = m ? __ffs(m) - 1 : 32;
                if (f == 0) {
                    hi_s = lo_s;
                } else {
                    const uint64_t pf = lo_s + (uint64_t)f * step;
                    lo_s = lo_s + (uint64_t)(f - 1) * step + 1;
                    hi_s = pf < hi_s ? pf : hi_s;
                }
            }
            s = lo_s;
            if (s >= nsub) {
                if (lane == 0) {
                    out_index[qi] = n;
                    out_value[qi] = 0;
                }
                continue;
            }
        } else {
            want = __ldg(reinterpret_cast<const uint64_t*>(queries) + qi);
            if (want >= n) {
                if (lane == 0) out_value[qi] = 0;
                continue;
            }
            s = want / kWTInts;
        }
        // decode sub-tile s from global memory with its carry
        const uint64_t g0 = s * kWTGroups, chunk = s / kChunkSubs;
        const WarpCtrl w = load_warp_ctrl<false>(in, g0, ngroups, tail_r);
        const uintptr_t dbeg = data0 + __ldg(meta.chunkpre + chunk) + __ldg(meta.localpre + s);
        const uintptr_t wbase = dbeg & ~(uintptr_t)3;
        const uint32_t head = (uint32_t)(dbeg & 3);
        uint32_t run = s ? __ldg(endval + s - 1) : base;
        const uint32_t jmax = kSeek ? (uint32_t)kWTRows : (uint32_t)((want % kWTInts) >> 7) + 1;
        for (uint32_t j = 0; j < jmax; ++j) {
            const uint32_t c = row_ctrl(w, (int)j);
            uint32_t b = head + row_q(w, (int)j);
            const uint64_t g = g0 + 32 * j + lane;
            const uint32_t cnt = group_count(g, ngroups, tail_r);
            uint32_t x[4];
#pragma unroll
            for (int f = 0; f < 4; ++f) {
                const uint32_t l = ((c >> (2 * f)) & 3u) + 1u;
                const uint32_t y = __funnelshift_r(qword(wbase + 4 * (b >> 2), lo, hi),
                                                   qword(wbase + 4 * (b >> 2) + 4, lo, hi), (b & 3u) * 8u);
                x[f] = (uint32_t)f < cnt ? (y & (0xFFFFFFFFu >> (32u - 8u * l))) : 0u;
                b += l;
            }
            uint4 v = make_uint4(x[0], x[0] + x[1], x[0] + x[1] + x[2], x[0] + x[1] + x[2] + x[3]);
            const uint32_t I = warp_inclusive_scan(v.w);
            v = add4(v, run + I - v.w);
            run += __shfl_sync(kFull, I, 31);
            if constexpr (kSeek) {
                // first component >= target among this lane's valid integers
                int f = 4;
                if (cnt > 3 && v.w >= target) f = 3;
                if (cnt > 2 && v.z >= target) f = 2;
                if (cnt > 1 && v.y >= target) f = 1;
                if (cnt > 0 && v.x >= target) f = 0;
                const uint32_t m = __ballot_sync(kFull, f < 4);
                if (m) {
                    const int hl = __ffs(m) - 1;
                    if (lane == hl) {
                        out_index[qi] = 4 * g + (uint64_t)f;
                        out_value[qi] = comp(v, f);
                    }
                    break;
                }
            } else if (j == jmax - 1) {
                const uint32_t e = (uint32_t)(want % 128);
                if ((uint32_t)lane == (e >> 2)) out_value[qi] = comp(v, (int)(e & 3));
            }
        }
    }
}

// metadata for queries: control scan (validates the stream), sums pass, sub-tile last values
cudaError_t launch_query_meta(const uint8_t* in, uint64_t in_len, uint64_t n, uint32_t base, void* meta_ws,
                              uint32_t* endval, unsigned long long* status, uint32_t epoch, cudaStream_t stream,
                              int* launches) {
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint64_t nchunks = (nsub + kChunkSubs - 1) / kChunkSubs;
    cudaError_t e = launch_decode_ctrl(in, in_len, n, 1, meta_ws, status, epoch, stream);
    if (e != cudaSuccess) return e;
    e = launch_decode_sums(in, in_len, n, meta_ws, stream);
    if (e != cudaSuccess) return e;
    const DecodeMeta m = carve_decode_meta(meta_ws, n);
    svb_endvals_kernel<<<(unsigned)((nchunks * 32 + 255) / 256), 256, 0, stream>>>(m, nsub, base, endval);
    *launches = 3;
    return cudaGetLastError();
}

cudaError_t launch_query(const uint8_t* in, uint64_t in_len, uint64_t n, uint32_t base, void* meta_ws,
                         const uint32_t* endval, int seek, const void* queries, uint64_t q, uint64_t* out_index,
                         uint32_t* out_value, int grid_cap, cudaStream_t stream) {
    if (q == 0) return cudaSuccess;
    const DecodeMeta m = carve_decode_meta(meta_ws, n);
    uint64_t grid = (q + 7) / 8;
    if (grid > (uint64_t)grid_cap) grid = (uint64_t)grid_cap;
    if (seek)
        svb_query_kernel<true><<<(unsigned)grid, 256, 0, stream>>>(in, in_len, n, base, m, endval, queries, q,
                                                                   out_index, out_value);
    else
        svb_query_kernel<false><<<(unsigned)grid, 256, 0, stream>>>(in, in_len, n, base, m, endval, queries, q,
                                                                    out_index, out_value);
    return cudaGetLastError();
}

}  // namespace bcgpu
