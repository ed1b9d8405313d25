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
    auto scan_and_issue = [&](uint32_t i, WarpCtrl& w, bool& zero) {
        const int cs = (int)(i % 3), ds = (int)(i & 1);
        BItem& it = B.item[cs];
        mbar_wait_parity(&B.cbar[cs], (i / 3) & 1u);
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
    if (B.item[0].valid) scan_and_issue(0, wA, zeroA);

    for (uint32_t i = 0;; ++i) {
        const int sa = (int)(i % 3), sb = (int)((i + 1) % 3), sc2 = (int)((i + 2) % 3);
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
        const bool same = b_valid && B.item[sb].src == A.src && B.item[sb].dst == A.dst && B.item[sb].k == A.k + 1;
        if (b_valid) {
            if (lane == 0) B.item[sb].off = same ? A.off + wA.total : 0ull;
            __syncwarp();
            scan_and_issue(i + 1, wB, zeroB);
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
                // partial tile and/or unaligned output: lean masked expansion, realigned stores
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
    }
}

// ---------------------------------------------------------------------------
// batch encode: warp-pipelined
// ---------------------------------------------------------------------------
// A warp walks its segments tile by tile; the integers of tile i+1 arrive by
// TMA while tile i is sized, packed in place (svb_fast.cuh) and written out --
// control bytes and data bytes each as one bulk store of the 16-B aligned
// interior plus edge bytes.  The data offset runs on in a register.
namespace {

constexpr int kBEStages = 3;  // item i+2 loads while i+1 waits and i's stores drain

struct __align__(128) BEncWarp {
    uint8_t stage[kBEStages][kWTStage + 16];  // [F - 16, F + 4096) with F at byte 16 + (F & 15)
    uint8_t ctrl[2][kWTGroups + 16];          // control bytes of items i, i-1 (stores in flight)
    uint64_t bar[kBEStages];
};

struct BEItem {
    unsigned long long src;  // element offset of the segment's first value
    unsigned long long cap;  // dst_capacity
    unsigned long long dst;  // byte offset of the segment's stream
    uint32_t n, k, prev, valid;
};

struct BECursor {
    const unsigned long long* segs;
    uint64_t nseg, nw, s;
    unsigned long long raw1, raw2;
    uint32_t k;
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
    __device__ __forceinline__ BEItem next(uint64_t* out_lens, unsigned long long* status, uint32_t epoch,
                                           uint64_t* seg_index) {
        BEItem it;
        it.valid = 0;
        while (s < nseg) {
            const unsigned long long a = __shfl_sync(kFull, raw1, 0), b = __shfl_sync(kFull, raw1, 1);
            const unsigned long long c = __shfl_sync(kFull, raw1, 2), np = __shfl_sync(kFull, raw1, 3);
            const uint32_t n = (uint32_t)np;
            const uint64_t ngroups = ((uint64_t)n + 3) >> 2;
            if (n <= kBatchSmallN) {  // encoded segment-resident by svb_batch3.cu
                next_segment();
                continue;
            }
            if (k == 0 && b < ngroups + 4ull * n) {
                if ((threadIdx.x & 31) == 0) {
                    if (n == 0)
                        out_lens[s] = 0;
                    else
                        report(status, epoch, BCGPU_ERR_INVALID_ARGUMENT);
                }
                next_segment();
                continue;
            }
            it.src = a;
            it.cap = b;
            it.dst = c;
            it.n = n;
            it.prev = (uint32_t)(np >> 32);
            it.k = k;
            it.valid = 1;
            *seg_index = s;
            if ((uint64_t)(k + 1) * kWTInts < n)
                ++k;
            else
                next_segment();
            return it;
        }
        return it;
    }
};

// cover of the tile's integers (and the one before it when k > 0) -> stage
__device__ __forceinline__ void issue_ints(const uint32_t* in, const BEItem& it, uint8_t* stage, uint64_t* bar) {
    const uint64_t i0 = it.src + (uint64_t)it.k * kWTInts;
    const uint32_t cnt = (uint32_t)(it.n - (uint64_t)it.k * kWTInts < (uint64_t)kWTInts ? it.n - (uint64_t)it.k * kWTInts
                                                                                         : (uint64_t)kWTInts);
    const uintptr_t F = (uintptr_t)(in + i0);
    const uintptr_t a0 = it.k ? ((F - 16) & ~(uintptr_t)15) : (F & ~(uintptr_t)15);
    const uintptr_t a1 = (F + 4ull * cnt + 15) & ~(uintptr_t)15;
    uint8_t* dst = stage + (it.k ? 0 : 16);
    mbar_expect(bar, (uint32_t)(a1 - a0));
    tma_load(dst, reinterpret_cast<const void*>(a0), (uint32_t)(a1 - a0), bar);
}

// global [g, g + len) <- smem bytes at sp (sp has g's 16-B phase); bulk store of the
// aligned interior (committed, not waited), lanes store the edge bytes
__device__ __forceinline__ bool out_bytes(uint8_t* g, const uint8_t* sp, uint32_t len) {
    const int lane = threadIdx.x & 31;
    const uintptr_t gb = (uintptr_t)g, ge = gb + len;
    const uintptr_t a_lo = (gb + 15) & ~(uintptr_t)15, a_hi = ge & ~(uintptr_t)15;
    if (a_hi > a_lo) {
        if (lane == 0) tma_store(reinterpret_cast<void*>(a_lo), sp + (a_lo - gb), (uint32_t)(a_hi - a_lo));
        const uint32_t nh = (uint32_t)(a_lo - gb), nt = (uint32_t)(ge - a_hi);
        if ((uint32_t)lane < nh) g[lane] = sp[lane];
        if ((uint32_t)lane < nt) g[(a_hi - gb) + lane] = sp[(a_hi - gb) + lane];
        return true;
    }
    for (uint32_t i = lane; i < len; i += 32) g[i] = sp[i];
    return false;
}

}  // namespace

// a full tile: size, control bytes (-> sctrl unless every integer is small, *small), pack in
// place at sdst; returns the data bytes
template <bool kDelta, bool kAny>
__device__ __forceinline__ uint32_t enc_tile_full(uint32_t sin, uint32_t prev_w, uint32_t sctrl, uint32_t sdst,
                                                  bool* small) {
    *small = enc_full_small<kDelta, kAny>(sin, prev_w);
    if (*small) {
        __syncwarp();
        enc_small_pack<kDelta, kAny>(sin, prev_w, sdst);
        return kWTInts;
    }
    uint32_t qw[4];
    const uint32_t total = enc_full_lengths_r<kDelta, kAny>(sin, prev_w, sctrl, qw);
    __syncwarp();
    enc_full_pack_r<kDelta, kAny>(sin, prev_w, sctrl, qw, sdst);
    return total;
}

// the last (partial) tile of a segment: cnt_g groups, the final one holding tail_r
// integers when `last` (cold path, kept out of line)
template <bool kDelta>
__device__ __noinline__ uint32_t enc_tile_partial(uint8_t* st, uint32_t sin, uint32_t prev_w, uint8_t* sctrl,
                                                  uint32_t head, uint32_t cnt_g, uint32_t tail_r, bool last) {
    const int lane = threadIdx.x & 31;
    EncodeTile t;
    uint32_t P[3] = {0, 0, 0};
    uint32_t last_w = prev_w;
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint32_t gl = 32 * j + lane;
        const uint32_t cnt = gl < cnt_g ? ((gl == cnt_g - 1 && tail_r && last) ? tail_r : 4u) : 0u;
        const uint32_t a = sin + 16 * gl;
        uint4 x = make_uint4(cnt > 0 ? lds32v(a) : 0u, cnt > 1 ? lds32v(a + 4) : 0u, cnt > 2 ? lds32v(a + 8) : 0u,
                             cnt > 3 ? lds32v(a + 12) : 0u);
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
        if (cnt)
            sctrl[gl] = (uint8_t)((l0 - 1) | (l1 ? ((l1 - 1) << 2) : 0u) | (l2 ? ((l2 - 1) << 4) : 0u) |
                                  (l3 ? ((l3 - 1) << 6) : 0u));
    }
    t.total = packed_row_scan(P, t.qw);
    __syncwarp();
    encode_pack_at(t, st, head);
    return t.total;
}

template <bool kDelta>
__global__ void __launch_bounds__(kBThreads)
    svb_encode_batch2_kernel(const bcgpu_encode_segment* __restrict__ segs, uint64_t nseg,
                             const uint32_t* __restrict__ in, uint8_t* __restrict__ out, uint64_t* __restrict__ out_lens,
                             unsigned long long* status, uint32_t epoch) {
    extern __shared__ __align__(128) uint8_t bdsm[];
    BEncWarp* wbuf = reinterpret_cast<BEncWarp*>(bdsm);  // kBWarps of them (dynamic: > 48 KiB)
    __shared__ __align__(16) uint8_t zeros[kWTGroups + 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    BEncWarp& B = wbuf[warp];
    for (uint32_t i = threadIdx.x; i < (kWTGroups + 32) / 4; i += kBThreads) reinterpret_cast<uint32_t*>(zeros)[i] = 0;
    __shared__ BEItem items[kBWarps][kBEStages];
    __shared__ unsigned long long sidxs[kBWarps][kBEStages];
    if (lane == 0)
        for (int q = 0; q < kBEStages; ++q) mbar_init1(&B.bar[q]);
    __syncthreads();
    BECursor cur;
    cur.init(segs, nseg, (uint64_t)blockIdx.x * kBWarps + warp, (uint64_t)gridDim.x * kBWarps);
    BEItem* item = items[warp];
    unsigned long long* sidx = sidxs[warp];
    for (int q = 0; q < kBEStages - 1; ++q) {
        uint64_t si = 0;
        const BEItem it = cur.next(out_lens, status, epoch, &si);
        if (lane == 0) {
            item[q] = it;
            sidx[q] = si;
            if (it.valid) issue_ints(in, it, B.stage[q], &B.bar[q]);
        }
    }
    __syncwarp();
    unsigned long long off = 0;  // data offset of the current tile within its segment
    for (uint32_t i = 0;; ++i) {
        const int q = (int)(i % kBEStages);
        const BEItem A = item[q];
        if (!A.valid) break;
        mbar_wait_parity(&B.bar[q], (i / kBEStages) & 1u);
        if (A.k == 0) off = 0;
        const uint64_t ngroups = ((uint64_t)A.n + 3) >> 2, g0 = (uint64_t)A.k * kWTGroups;
        const uint32_t cnt_g = (uint32_t)(ngroups - g0 < (uint64_t)kWTGroups ? ngroups - g0 : (uint64_t)kWTGroups);
        const uintptr_t F = (uintptr_t)(in + A.src + (uint64_t)A.k * kWTInts);
        uint8_t* st = B.stage[q];
        const uint32_t sin = sh_addr(st) + 16 + (uint32_t)(F & 15);
        const uint32_t prev_w = A.k ? lds32v(sin - 4) : A.prev;
        const bool full = (uint64_t)(A.k + 1) * kWTInts <= A.n;
        uint8_t* cdst = out + A.dst + g0;
        const uint32_t hc = (uint32_t)((uintptr_t)cdst & 15);
        uint8_t* sctrl = B.ctrl[i & 1];
        uint8_t* ddst = out + A.dst + ngroups + off;
        const uint32_t head = (uint32_t)((uintptr_t)ddst & 15);
        uint32_t total;
        bool small = false;
        if (full) {
            if (sin & 15u)
                total = enc_tile_full<kDelta, true>(sin, prev_w, sh_addr(sctrl) + hc, sh_addr(st) + head, &small);
            else
                total = enc_tile_full<kDelta, false>(sin, prev_w, sh_addr(sctrl) + hc, sh_addr(st) + head, &small);
        } else {
            total = enc_tile_partial<kDelta>(st, sin, prev_w, sctrl + hc, head, cnt_g, A.n & 3u,
                                             g0 + cnt_g == ngroups);
        }
        fence_async_smem();
        __syncwarp();
        bool any = out_bytes(cdst, small ? zeros + hc : sctrl + hc, cnt_g);
        any = out_bytes(ddst, st + head, total) || any;
        (void)any;
        if (lane == 0) tma_store_commit();  // one bulk group per item (possibly empty)
        off += total;
        if (!full || (uint64_t)(A.k + 1) * kWTInts == A.n) {
            if (lane == 0) out_lens[sidx[q]] = ngroups + off;
        }
        // item i+2 -> the stage item i-1 used, once its bulk stores have read it
        {
            const int qn = (int)((i + kBEStages - 1) % kBEStages);
            uint64_t si = 0;
            const BEItem it = cur.next(out_lens, status, epoch, &si);
            if (lane == 0) {
                tma_store_wait_read_but1();
                item[qn] = it;
                sidx[qn] = si;
                if (it.valid) {
                    fence_async_smem();
                    issue_ints(in, it, B.stage[qn], &B.bar[qn]);
                }
            }
        }
        __syncwarp();
    }
    if (lane == 0) tma_store_wait_read();
}

cudaError_t launch_encode_batch2(const bcgpu_encode_segment* segs, uint64_t nseg, const uint32_t* in, uint8_t* out,
                                 uint64_t* out_lens, int delta, const BatchArgs& ba, cudaStream_t stream) {
    static int sms = 0, occ = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        int o1 = 0, o2 = 0;
        cudaFuncSetAttribute(svb_encode_batch2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(BEncWarp) * kBWarps);
        cudaFuncSetAttribute(svb_encode_batch2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(BEncWarp) * kBWarps);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, svb_encode_batch2_kernel<true>, kBThreads,
                                                      sizeof(BEncWarp) * kBWarps);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, svb_encode_batch2_kernel<false>, kBThreads,
                                                      sizeof(BEncWarp) * kBWarps);
        occ = o1 < o2 ? o1 : o2;
        if (occ < 1) occ = 1;
    }
    const uint64_t want = (nseg + kBWarps - 1) / kBWarps, cap = (uint64_t)sms * occ;
    const int grid = (int)(want < cap ? want : cap);
    if (grid <= 0) return cudaSuccess;
    if (delta)
        svb_encode_batch2_kernel<true><<<grid, kBThreads, sizeof(BEncWarp) * kBWarps, stream>>>(segs, nseg, in, out, out_lens, ba.status,
                                                                        ba.epoch);
    else
        svb_encode_batch2_kernel<false><<<grid, kBThreads, sizeof(BEncWarp) * kBWarps, stream>>>(segs, nseg, in, out, out_lens, ba.status,
                                                                         ba.epoch);
    return cudaGetLastError();
}

cudaError_t launch_decode_batch2(const bcgpu_decode_segment* segs, uint64_t nseg, const uint8_t* in, uint32_t* out,
                                 int delta, const BatchArgs& ba, cudaStream_t stream) {
    static int sms = 0, occ = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        int o1 = 0, o2 = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, svb_decode_batch2_kernel<true>, kBThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, svb_decode_batch2_kernel<false>, kBThreads, 0);
        occ = o1 < o2 ? o1 : o2;
        if (occ < 1) occ = 1;
    }
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
