// svb_batch2.cu -- segmented batch decode, warp-pipelined (sm_100a).
//
// Reference behaviour: every segment is an independent Stream VByte stream
// (svb_decode / svb_decode_delta, stream_vbyte.hpp:38-42, codec.hpp:85-90;
// chained chunks with a carried delta base, codec.hpp:87-90).
//
// One warp walks its segments (s = warp, warp + W, ...) tile by tile (1024
// integers), with the offset and delta carry in registers -- no cross-warp
// dependency.  What the old per-tile loop left exposed were two dependent
// round trips per tile (control bytes, then the data they locate).  Here the
// warp runs a three-item software pipeline across tile and segment boundaries:
//   iteration i:  issue the control-byte copy of item i+2,
//                 scan item i+1's control bytes (landed), issue its data copy,
//                 expand + store item i (its data landed during iteration i-1).
// All copies are TMA bulk copies of 16-B aligned covers into per-warp stage
// buffers (a 16-B granule holding a valid byte never crosses a page, so the
// cover of a valid range is always readable).  Segment descriptors are
// prefetched two segments ahead.
#include <cstdint>

#include "svb_device.cuh"
#include "svb_fast.cuh"
#include "launch_cache.cuh"
#include "svb_kernels.cuh"
#include "svb_tma.cuh"
#include "svb_warp.cuh"

namespace bcgpu {

namespace {

constexpr int kBWarps = 4;
constexpr int kBThreads = 32 * kBWarps;
constexpr uint32_t kBCtrlBuf = 288;        // 256 control bytes + 16-B head, rounded
constexpr uint32_t kBDataBuf = kWTStage;   // 4096 data bytes + head + over-read slack

struct BItem {                 // one tile of one segment (warp-uniform)
    unsigned long long src;    // byte offset of the segment stream in `in`
    unsigned long long dst;    // element offset of the segment's integer 0
    unsigned long long bytes;  // the segment stream's length
    unsigned long long off;    // data offset of this tile within the segment's data
    uint32_t n, k, prev, carry;
    uint32_t valid;
};

struct __align__(128) BDecWarp {
    uint8_t data[2][kBDataBuf];
    uint8_t ctrl[3][kBCtrlBuf];
    BItem item[3];
    uint64_t dbar[2], cbar[3];
};

__device__ __forceinline__ void report(unsigned long long* st, uint32_t epoch, uint32_t code) {
    if (st) *st = ((unsigned long long)epoch << 32) | code;
}

// Walks a warp's items in order; descriptors prefetched two segments ahead
// (lanes 0..3 hold the four 8-byte words of each prefetched descriptor).
struct BCursor {
    const unsigned long long* segs;
    uint64_t nseg, nw, s;          // s: segment of the next item
    unsigned long long raw1, raw2; // descriptors of s (raw1) and s + nw (raw2)
    uint32_t k;                    // next tile index within segment s
    bool have;                     // raw1 holds segment s's descriptor

    __device__ __forceinline__ unsigned long long fetch(uint64_t idx) const {
        const int lane = threadIdx.x & 31;
        return (idx < nseg && lane < 4) ? __ldg(segs + 4 * idx + lane) : 0ull;
    }
    __device__ __forceinline__ void init(const void* p, uint64_t n_, uint64_t first, uint64_t stride) {
        segs = reinterpret_cast<const unsigned long long*>(p);
        nseg = n_;
        nw = stride;
        s = first;
        k = 0;
        raw1 = fetch(s);
        raw2 = fetch(s + nw);
    }
    __device__ __forceinline__ void next_segment() {
        s += nw;
        k = 0;
        raw1 = raw2;
        raw2 = fetch(s + nw);
    }
    // the next tile to process (item.valid = 0 when the warp is done); reports
    // truncated segments and skips them
    __device__ __forceinline__ BItem next(unsigned long long* status, uint32_t epoch) {
        BItem it;
        it.valid = 0;
        while (s < nseg) {
            const unsigned long long a = __shfl_sync(kFull, raw1, 0), b = __shfl_sync(kFull, raw1, 1);
            const unsigned long long c = __shfl_sync(kFull, raw1, 2), np = __shfl_sync(kFull, raw1, 3);
            const uint32_t n = (uint32_t)np;
            const uint64_t ngroups = ((uint64_t)n + 3) >> 2;
            if (n <= kBatchSmallN) {  // decoded segment-resident by svb_batch3.cu
                next_segment();
                continue;
            }
            if (k == 0 && b < ngroups) {
                if ((threadIdx.x & 31) == 0) report(status, epoch, BCGPU_ERR_TRUNCATED);
                next_segment();
                continue;
            }
            it.src = a;
            it.bytes = b;
            it.dst = c;
            it.n = n;
            it.prev = (uint32_t)(np >> 32);
            it.k = k;
            it.off = 0;
            it.carry = 0;
            it.valid = 1;
            if ((uint64_t)(k + 1) * kWTInts < n)
                ++k;
            else
                next_segment();
            return it;
        }
        return it;
    }
};

__device__ __forceinline__ uint32_t tile_groups(const BItem& it) {
    const uint64_t ngroups = ((uint64_t)it.n + 3) >> 2, g0 = (uint64_t)it.k * kWTGroups;
    return (uint32_t)(ngroups - g0 < (uint64_t)kWTGroups ? ngroups - g0 : (uint64_t)kWTGroups);
}

// control bytes of tile it.k -> ctrl buffer (16-B aligned cover; byte 0 at (beg & 15))
__device__ __forceinline__ void issue_ctrl(const uint8_t* in, const BItem& it, uint8_t* buf, uint64_t* bar) {
    const uintptr_t beg = (uintptr_t)in + it.src + (uint64_t)it.k * kWTGroups;
    const uintptr_t a0 = beg & ~(uintptr_t)15, a1 = (beg + tile_groups(it) + 15) & ~(uintptr_t)15;
    mbar_expect(bar, (uint32_t)(a1 - a0));
    tma_load(buf, reinterpret_cast<const void*>(a0), (uint32_t)(a1 - a0), bar);
}

}  // namespace

template <bool kDelta>
__global__ void __launch_bounds__(kBThreads)
    svb_decode_batch2_kernel(const bcgpu_decode_segment* __restrict__ segs, uint64_t nseg,
                             const uint8_t* __restrict__ in, uint32_t* __restrict__ out, unsigned long long* status,
                             uint32_t epoch) {
    __shared__ BDecWarp wbuf[kBWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    BDecWarp& B = wbuf[warp];
    if (lane == 0) {
        mbar_init1(&B.dbar[0]);
        mbar_init1(&B.dbar[1]);
        mbar_init1(&B.cbar[0]);
        mbar_init1(&B.cbar[1]);
        mbar_init1(&B.cbar[2]);
    }
    __syncwarp();
    BCursor cur;
    cur.init(segs, nseg, (uint64_t)blockIdx.x * kBWarps + warp, (uint64_t)gridDim.x * kBWarps);

    // prologue: items 0 and 1 -> ring slots 0 and 1, control copies in flight
    for (int q = 0; q < 2; ++q) {
        const BItem it = cur.next(status, epoch);
        if (lane == 0) {
            B.item[q] = it;
            if (it.valid) issue_ctrl(in, it, B.ctrl[q], &B.cbar[q]);
        }
    }
    __syncwarp();
    WarpCtrl wA;
    bool zeroA = false;
    // scan item 0 and issue its data
    auto scan_and_issue = [&](uint32_t i, int cs, uint32_t cph, WarpCtrl& w, bool& zero) {  // cs = i % 3, cph = (i / 3) & 1
        const int ds = (int)(i & 1);
        BItem& it = B.item[cs];
        mbar_wait_parity(&B.cbar[cs], cph);
        const uintptr_t cbeg = (uintptr_t)in + it.src + (uint64_t)it.k * kWTGroups;
        const uint8_t* sc = B.ctrl[cs] + (cbeg & 15);
        const uint64_t ngroups = ((uint64_t)it.n + 3) >> 2, g0 = (uint64_t)it.k * kWTGroups;
        zero = false;
        if ((uint64_t)(it.k + 1) * kWTInts <= it.n)
            w = ctrl_full(sh_addr(sc), &zero);
        else
            w = load_warp_ctrl<true>(sc, g0, ngroups, it.n & 3u, g0);
        // data range, clamped to the segment (malformed streams report below)
        const uintptr_t seg0 = (uintptr_t)in + it.src, seg1 = seg0 + it.bytes;
        uintptr_t beg = seg0 + ngroups + it.off, end = beg + w.total;
        if (end > seg1) end = seg1;
        if (beg > end) beg = end;
        const uintptr_t a0 = beg & ~(uintptr_t)15, a1 = (end + 15) & ~(uintptr_t)15;
        __syncwarp();  // every lane has read the item record before lane 0 may rewrite slots
        if (lane == 0) {
            fence_async_smem();
            mbar_expect(&B.dbar[ds], (uint32_t)(a1 - a0));
            if (a1 > a0) tma_load(B.data[ds], reinterpret_cast<const void*>(a0), (uint32_t)(a1 - a0), &B.dbar[ds]);
        }
    };
    if (B.item[0].valid) scan_and_issue(0, 0, 0u, wA, zeroA);

    int sa = 0, sb = 1, sc2 = 2;  // i % 3, (i + 1) % 3, (i + 2) % 3
    uint32_t ph1 = 0;            // ((i + 1) / 3) & 1
    for (uint32_t i = 0;; ++i) {
        if (!B.item[sa].valid) break;
        // 1. item i+2: descriptor walk + control copy
        {
            const BItem it = cur.next(status, epoch);
            __syncwarp();
            if (lane == 0) {
                B.item[sc2] = it;
                if (it.valid) {
                    fence_async_smem();
                    issue_ctrl(in, it, B.ctrl[sc2], &B.cbar[sc2]);
                }
            }
            __syncwarp();
        }
        // 2. item i+1: offset, control scan, data copy
        WarpCtrl wB;
        bool zeroB = false;
        const BItem A = B.item[sa];
        const bool b_valid = B.item[sb].valid != 0;
        // items come in order (tile k + 1 of a segment, or tile 0 of the next), so the next
        // item continues this segment exactly when its tile index is k + 1
        const bool same = b_valid && B.item[sb].k == A.k + 1;
        if (b_valid) {
            if (lane == 0) B.item[sb].off = same ? A.off + wA.total : 0ull;
            __syncwarp();
            scan_and_issue(i + 1, sb, ph1, wB, zeroB);
        }
        // 3. item i: expand + store
        {
            const int ds = (int)(i & 1);
            mbar_wait_parity(&B.dbar[ds], (i >> 1) & 1u);
            const uint64_t ngroups = ((uint64_t)A.n + 3) >> 2, g0 = (uint64_t)A.k * kWTGroups;
            const uint32_t carry = A.k == 0 ? A.prev : A.carry;
            uint32_t* o = out + A.dst;
            const uintptr_t dbeg = (uintptr_t)in + A.src + ngroups + A.off;
            const uint32_t head = (uint32_t)(dbeg & 15);
            const bool out16 = (((uintptr_t)(o + 4 * g0)) & 15) == 0;
            uint32_t after = carry;
            if ((uint64_t)(A.k + 1) * kWTInts <= A.n && out16) {
                const uint32_t sd = sh_addr(B.data[ds]) + head;
                uint32_t* ot = o + 4 * g0;
                if constexpr (kDelta) {
                    after = zeroA ? expand_full<1, true>(wA, sd, ot, carry) : expand_full<1, false>(wA, sd, ot, carry);
                } else {
                    if (zeroA)
                        expand_full<0, true>(wA, sd, ot, 0);
                    else
                        expand_full<0, false>(wA, sd, ot, 0);
                }
            } else {
                // partial tile and/or unaligned output: lean masked expansion, realigned stores.
                // An all-zero full tile's ctrl_full skipped the row offsets: group g is data byte 4 g.
                if (zeroA)
#pragma unroll
                    for (int q = 0; q < 4; ++q) wA.qw[q] = (256u * q + 4u * lane) | ((256u * q + 128u + 4u * lane) << 16);
                const uint32_t ng = (uint32_t)(ngroups - g0 < (uint64_t)kWTGroups ? ngroups - g0 : (uint64_t)kWTGroups);
                const uint32_t tail = (g0 + ng == ngroups && (A.n & 3u)) ? (A.n & 3u) : 4u;
                after = expand_any<kDelta>(wA, sh_addr(B.data[ds]) + head, ng, tail, o + 4 * g0, carry);
            }
            // end of the segment: the stream must end exactly here
            if ((uint64_t)(A.k + 1) * kWTInts >= A.n && lane == 0) {
                const uint64_t need = ngroups + A.off + wA.total;
                if (need != A.bytes) report(status, epoch, need > A.bytes ? BCGPU_ERR_TRUNCATED : BCGPU_ERR_TRAILING_BYTES);
            }
            if (same && lane == 0) B.item[sb].carry = after;
        }
        __syncwarp();
        wA = wB;
        zeroA = zeroB;
        ph1 ^= sc2 == 0 ? 1u : 0u;  // item i + 2 starts a new lap of the 3-slot ring
        const int t = sa;
        sa = sb;
        sb = sc2;
        sc2 = t;
    }
}

cudaError_t launch_decode_batch2(const bcgpu_decode_segment* segs, uint64_t nseg, const uint8_t* in, uint32_t* out,
                                 int delta, const BatchArgs& ba, cudaStream_t stream) {
    const int sms = launch_sms(launch_current_device());
    const int o1 = launch_occupancy(svb_decode_batch2_kernel<true>, kBThreads, 0);
    const int o2 = launch_occupancy(svb_decode_batch2_kernel<false>, kBThreads, 0);
    int occ = o1 < o2 ? o1 : o2;
    if (occ > 4) occ = 4;  // cfg5 sweep: 4 CTAs per SM 2.02 ms, 5 (the occupancy limit) 2.06 ms
    if (occ < 1) occ = 1;
    const uint32_t occ_cap = (ba.flags >> 12) & 7u;  // debug: CTAs per SM
    const uint64_t want = (nseg + kBWarps - 1) / kBWarps,
                   cap = (uint64_t)sms * (occ_cap && (int)occ_cap < occ ? (int)occ_cap : occ);
    const int grid = (int)(want < cap ? want : cap);
    if (grid <= 0) return cudaSuccess;
    if (delta)
        svb_decode_batch2_kernel<true><<<grid, kBThreads, 0, stream>>>(segs, nseg, in, out, ba.status, ba.epoch);
    else
        svb_decode_batch2_kernel<false><<<grid, kBThreads, 0, stream>>>(segs, nseg, in, out, ba.status, ba.epoch);
    return cudaGetLastError();
}

}  // namespace bcgpu
