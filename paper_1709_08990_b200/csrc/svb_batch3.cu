// svb_batch3.cu -- segment-resident batch decode for short segments (sm_100a).
//
// Reference behaviour: every segment is an independent Stream VByte stream
// (svb_decode / svb_decode_delta, stream_vbyte.hpp:38-42, codec.hpp:85-90).
//
// Posting-list batches (cfg4) are dominated by short streams: half the lists
// hold < 1024 integers and each list ends in a partial tile.  The tile
// pipeline of svb_batch2.cu pays, per tile, a control-byte copy, a scan of
// 256 control bytes, a data copy sized by that scan and a masked 8-row
// expansion -- ~1600 warp instructions per tile on cfg4 (ncu), so the kernel
// was issue-bound at a third of the HBM roofline.
//
// Here a segment whose worst-case stream fits kItemMax bytes is ONE item: the
// descriptor alone locates the whole stream (src_offset, src_bytes), so one
// TMA bulk copy brings control and data bytes together -- no dependent round
// trip, no pre-scan.  Each warp owns a byte ring in shared memory and keeps as
// many segments in flight as fit (up to kRSlots), then decodes the oldest one
// straight from the ring, 512 integers per warp pass with each lane owning
// four consecutive groups (one length scan and one delta scan per pass);
// outputs at any 4-B phase leave as 128/256-bit stores of 16-B granules.
// Longer segments stay on svb_batch2.cu (they are skipped here).
#include <cstdint>

#include "svb_device.cuh"
#include "svb_fast.cuh"
#include "launch_cache.cuh"
#include "svb_kernels.cuh"
#include "svb_pack.cuh"
#include "svb_tma.cuh"
#include "svb_warp.cuh"

namespace bcgpu {

namespace {

#ifndef BC_DEC3_MINB
#define BC_DEC3_MINB 5  // decode CTAs per SM the register budget must allow (6 spills)
#endif
#ifndef BC_ENC3_MINB
#define BC_ENC3_MINB 5  // encode CTAs per SM the register budget must allow (6: <= 80 registers spills, cfg4 1.96 vs 1.88 ms)
#endif
#ifndef BC_R_WARPS
#define BC_R_WARPS 4
#endif
constexpr int kRWarps = BC_R_WARPS;
constexpr int kRThreads = 32 * kRWarps;
constexpr uint32_t kRingDefault = 8192;   // ring bytes per warp (launch-time; >= kItemMax)
constexpr uint32_t kRingSlack = 192;      // over-reads past an item land here (control bytes of idle lanes: < 140 B)
constexpr uint32_t kRSlots = 8;           // items in flight per warp
constexpr uint32_t kChunkMax = 8;         // segments a warp draws at a time (<= 32: one descriptor per lane); cfg4: 4 / 8 / 16 / 24 / 32 -> encode 1.70 / 1.69 / 1.70 / 1.72 / 1.74 ms, decode 1.58 / 1.56 / 1.57 / 1.58 / 1.59 ms
constexpr uint32_t kItemMax = 8192;       // largest 16-B cover of an item
static_assert(kBatchSmallN / 4 + 1 + 4ull * kBatchSmallN + 30 <= kItemMax, "short-segment stream must fit an item");

struct RItem {
    unsigned long long dst;  // element offset of integer 0
    uint32_t n, prev, bytes;
    uint32_t spos;           // ring byte of the segment's byte 0
    uint32_t end;            // ring counter after the item (frees its bytes)
    uint32_t pad;
};

struct __align__(16) RWarpHdr {  // per warp, ahead of the rings in dynamic shared memory
    uint64_t bar[kRSlots];
    RItem item[kRSlots];
    ulonglong2 desc[32][2];  // the descriptors of the warp's current 32 segments
    uint4 carry;             // decode: the last R integers of the previous pass's lane 31
};

__device__ __forceinline__ void report3(unsigned long long* st, uint32_t epoch, uint32_t code) {
    if (st) *st = ((unsigned long long)epoch << 32) | code;
}

__device__ __forceinline__ void stg_stream_v8(void* p, const uint4& a, const uint4& b) {
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
                 "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                 : "memory");
}

// ---- segment-resident decode -------------------------------------------------------------
// x zero-extended from its low b bits (b clamped to 32): one SGXT instead of a mask shift + AND
__device__ __forceinline__ uint32_t szext(uint32_t x, uint32_t b) {
    uint32_t r;
    asm("szext.clamp.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(b));
    return r;
}

// One control byte c whose data starts at shared byte address a -> 4 integers.  The group's
// 16 bytes X0..X3 act as a queue: integer i is the queue's low l_i bytes (SGXT by 8 l_i), then
// the queue drops them (clamped funnel shifts: 8 l_i = 32 moves a whole word).  Each step
// needs one word less, so the four integers cost 4 SGXT + 6 funnel shifts, with no selects
// (round 1 picked each integer's word pair from the window with compare + select chains and
// masked it with a shift + AND: ~40 instructions per group against ~30 here).
// Shared word at a when pred, else whatever the register held (a predicated load: no branch,
// no zeroing move).  Callers only use bytes of words they loaded.
__device__ __forceinline__ uint32_t lds32_if(uint32_t a, bool pred) {
    uint32_t v;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.u32 %0, [%1];\n\t}"
                 : "=r"(v)
                 : "r"(a), "r"((uint32_t)pred));
    return v;
}

// len = the group's data bytes: only the words they touch are loaded (cfg4 groups average ~10
// bytes, ~3.4 of the five words; every window load is ~4-way bank-conflicted, and shared-memory
// wavefronts bound this kernel once the ALU work is down).  b0..b3 = 8 l_i of its integers.
__device__ __forceinline__ uint4 group_q(uint32_t a, uint32_t len, uint32_t b0, uint32_t b1, uint32_t b2,
                                         uint32_t b3) {
    const uint32_t wa = a & ~3u, sh = (a & 3u) << 3;
    const uint32_t e = (a & 3u) + len;  // window bytes in use
    const uint32_t w0 = lds32(wa), w1 = lds32_if(wa + 4, e > 4), w2 = lds32_if(wa + 8, e > 8),
                   w3 = lds32_if(wa + 12, e > 12), w4 = lds32_if(wa + 16, e > 16);
    const uint32_t X0 = __funnelshift_r(w0, w1, sh), X1 = __funnelshift_r(w1, w2, sh),
                   X2 = __funnelshift_r(w2, w3, sh), X3 = __funnelshift_r(w3, w4, sh);
    uint4 v;
    v.x = szext(X0, b0);
    const uint32_t Y0 = __funnelshift_rc(X0, X1, b0), Y1 = __funnelshift_rc(X1, X2, b0),
                   Y2 = __funnelshift_rc(X2, X3, b0);
    v.y = szext(Y0, b1);
    const uint32_t Z0 = __funnelshift_rc(Y0, Y1, b1), Z1 = __funnelshift_rc(Y1, Y2, b1);
    v.z = szext(Z0, b2);
    v.w = szext(__funnelshift_rc(Z0, Z1, b2), b3);
    return v;
}

// Vector stores of the whole granules among a lane's groups g0 .. g0 + 3.  R = the output's
// 4-B phase inside 16 B (a template: the granule assembly is static register moves): lane l
// stores the granules [4q - R, 4q - R + 4) for its groups q at 16-B aligned Bp + 4q; the first
// takes the previous group's last R integers from lane l - 1 (lane 0: the previous pass's lane
// 31, in carry).  Lanes are 64 B apart, so pairs of granules on a 32-B boundary leave as one
// 256-bit store (half the L1 wavefronts).  Granules that straddle the segment's ends are left
// to the edge stores of decode_pass, so each phase's block is a few predicated stores.
template <uint32_t R>
__device__ __forceinline__ void store_whole(const uint4 (&v)[4], uint32_t* __restrict__ o, uint32_t g0, int nints,
                                            uint32_t cs) {
    const int lane = threadIdx.x & 31;
    uint4 G[4];
    uint32_t* Bp = o - R;  // 16-B aligned
    if constexpr (R == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) G[j] = v[j];
    } else {
        const int src = (lane + 31) & 31;
        uint4 rot = make_uint4(0, 0, 0, 0);
        rot.w = __shfl_sync(kFull, v[3].w, src);
        if (R >= 2) rot.z = __shfl_sync(kFull, v[3].z, src);
        if (R >= 3) rot.y = __shfl_sync(kFull, v[3].y, src);
        // lane 0 takes the previous pass's lane 31 values from the warp's carry slot in shared
        // memory (a register uint4 live through every pass cost the sixth CTA per SM)
        const uint4 prv0 = lane == 0 ? lds128v(cs) : rot;
        if (lane == 0) sts128(cs, rot);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint4 pv = j == 0 ? prv0 : v[j - 1], cv = v[j];
            G[j] = R == 1 ? make_uint4(pv.w, cv.x, cv.y, cv.z)
                 : R == 2 ? make_uint4(pv.z, pv.w, cv.x, cv.y)
                          : make_uint4(pv.y, pv.z, pv.w, cv.x);
        }
    }
    bool f[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int e0 = 4 * (int)(g0 + j) - (int)R;
        f[j] = e0 >= 0 && e0 + 4 <= nints;
    }
    if ((((uintptr_t)Bp) & 31) == 0) {  // warp-uniform (g0 even): pairs (0,1), (2,3)
#pragma unroll
        for (int j = 0; j < 4; j += 2) {
            if (f[j] && f[j + 1]) {
                stg_stream_v8(Bp + 4 * (g0 + j), G[j], G[j + 1]);
            } else {
                if (f[j]) stg_stream_v4(Bp + 4 * (g0 + j), G[j]);
                if (f[j + 1]) stg_stream_v4(Bp + 4 * (g0 + j + 1), G[j + 1]);
            }
        }
    } else {  // pair (1,2)
        if (f[0]) stg_stream_v4(Bp + 4 * g0, G[0]);
        if (f[1] && f[2]) {
            stg_stream_v8(Bp + 4 * (g0 + 1), G[1], G[2]);
        } else {
            if (f[1]) stg_stream_v4(Bp + 4 * (g0 + 1), G[1]);
            if (f[2]) stg_stream_v4(Bp + 4 * (g0 + 2), G[2]);
        }
        if (f[3]) stg_stream_v4(Bp + 4 * (g0 + 3), G[3]);
    }
}

// One pass of decode_resident: 128 groups from group gp, lane l owning groups g0 = gp + 4 l
// .. g0 + 3.  In the segment's last pass the groups past its end decode garbage that is never
// stored: it only follows the valid integers in lane order, so no position, delta prefix or
// store of a valid integer sees it, and the declared data length comes from the lane holding
// the last group.  (A last pass of k = ceil(groups left / 32) groups per lane was built and
// measured: the runtime k cost more in every pass than it saved in the last.)
template <bool kDelta>
__device__ __forceinline__ void decode_pass(uint32_t S, uint32_t D, uint32_t Dend, uint32_t ng, uint32_t n,
                                            uint32_t gp, bool lastp, uint32_t R, int T, uint32_t& off, uint32_t& run,
                                            uint32_t cs, uint32_t* __restrict__ o) {
    const int lane = threadIdx.x & 31;
    const uint32_t g0 = gp + 4 * lane;
    const uint32_t ca = S + g0;
    uint32_t cw = __funnelshift_r(lds32(ca & ~3u), lds32((ca & ~3u) + 4), (ca & 3u) << 3);
    uint32_t lens = swar_lengths(cw);
    if (lastp) {  // groups past the end (their "control bytes" are data) load and decode nothing
        const uint32_t nv = ng > g0 ? ng - g0 : 0u;
        const uint32_t bm = nv >= 4 ? 0xFFFFFFFFu : ((1u << (8 * nv)) - 1u);
        cw &= bm;
        lens &= bm;
    }
    const uint32_t lt = __dp4a(lens, 0x01010101u, 0u);  // <= 64
    const uint32_t I = warp_inclusive_scan(lt);
    uint32_t p = D + off + I - lt;
    if (!lastp) {
        off += __shfl_sync(kFull, I, 31);
    } else {
        // data bytes up to the end of the last group (ng - 1), its unused fields left out: from
        // the lane holding it, j = its place in the lane
        const uint32_t q = ng - 1 - gp, j = q & 3u, r = n & 3u;
        const uint32_t before = __byte_perm(lens * 0x01010100u, 0u, 0x4440u | j);  // lens of groups < j
        const uint32_t cl = __byte_perm(cw, 0u, 0x4440u | j) & (r ? (1u << (2 * r)) - 1u : 0xFFu);
        const uint32_t mine = (I - lt) + before + field_sum(cl) + (r ? r : 4u);
        off += __shfl_sync(kFull, mine, (int)(q >> 2));
    }
    uint4 v[4];
    if (__all_sync(kFull, cw == 0)) {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = zero_group_s(min(p + 4 * j, Dend));
    } else {
        // 8 l of every integer of the lane's groups, four per word: byte j of Bi = 8 (field i of
        // control byte j) + 8; one PRMT isolates each (three ops apiece from the control byte)
        const uint32_t Bx = (cw & 0x03030303u) * 8u + 0x08080808u, By = ((cw >> 2) & 0x03030303u) * 8u + 0x08080808u,
                       Bz = ((cw >> 4) & 0x03030303u) * 8u + 0x08080808u, Bw = ((cw >> 6) & 0x03030303u) * 8u + 0x08080808u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t sel = 0x4440u | (uint32_t)j;
            const uint32_t lj = __byte_perm(lens, 0u, sel);
            v[j] = group_q(min(p, Dend), lj, __byte_perm(Bx, 0u, sel), __byte_perm(By, 0u, sel),
                           __byte_perm(Bz, 0u, sel), __byte_perm(Bw, 0u, sel));
            p += lj;
        }
    }
    if constexpr (kDelta) {
        uint32_t s = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v[j].x += s;
            v[j].y += v[j].x;
            v[j].z += v[j].y;
            v[j].w += v[j].z;
            s = v[j].w;
        }
        const uint32_t Iv = warp_inclusive_scan(s);
        const uint32_t add = run + Iv - s;
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = add4(v[j], add);
        run += __shfl_sync(kFull, Iv, 31);
    }
    switch (R) {  // warp-uniform; only these small store blocks are per phase
        case 0: store_whole<0>(v, o, g0, (int)n, cs); break;
        case 1: store_whole<1>(v, o, g0, (int)n, cs); break;
        case 2: store_whole<2>(v, o, g0, (int)n, cs); break;
        default: store_whole<3>(v, o, g0, (int)n, cs); break;
    }
    // The integers no whole granule holds: the head granule's [0, 4 - R) (R != 0: lane 0's first
    // group in the first pass) and the tail [T, n), <= 3 integers held by at most two lanes
    // (T = the start of the last, partial granule; it can start in the pass before the last).
    if (gp == 0 && R != 0 && lane == 0) {
        const int h = 4 - (int)R < (int)n ? 4 - (int)R : (int)n;
        o[0] = v[0].x;
        if (h > 1) o[1] = v[0].y;
        if (h > 2) o[2] = v[0].z;
    }
    const int rel = T - 4 * (int)gp;
    if (rel < 512 && (lane == (rel >> 4) || lane == (((int)n - 1 - 4 * (int)gp) >> 4))) {
        const int lo = 4 * (int)g0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int a = T - (lo + 4 * j), b = (int)n - (lo + 4 * j);  // group j holds integers i, a <= i < b
            if (a < 4 && b > 0) {
                uint32_t* qo = o + lo + 4 * j;
                if (a <= 0) qo[0] = v[j].x;
                if (a <= 1 && b > 1) qo[1] = v[j].y;
                if (a <= 2 && b > 2) qo[2] = v[j].z;
                if (b > 3) qo[3] = v[j].w;
            }
        }
    }
}

// Decode one resident segment (any n <= kBatchSmallN) in passes of 512 integers; returns the
// data bytes its control stream declares.  group_q extraction, predicated scans, whole-granule
// stores per phase and the segment-edge integers outside the per-phase blocks.
template <bool kDelta>
__device__ __forceinline__ uint32_t decode_resident(uint32_t S, uint32_t bytes, uint32_t n, uint32_t run,
                                                    uint32_t cs, uint32_t* __restrict__ o) {
    const uint32_t R = (uint32_t)(((uintptr_t)o >> 2) & 3u);
    const uint32_t ng = (n + 3) >> 2;
    const uint32_t D = S + ng, Dend = S + bytes;
    const int T = 4 * (int)((n + R) >> 2) - (int)R;  // the tail no whole granule holds: [T, n)
    const uint32_t full_passes = (ng - 1) >> 7;       // every pass but the last holds 128 groups
    uint32_t off = 0;
#pragma unroll 1
    for (uint32_t ps = 0;; ++ps) {
        const bool lastp = ps == full_passes;
        decode_pass<kDelta>(S, D, Dend, ng, n, 128 * ps, lastp, R, T, off, run, cs, o);
        if (lastp) break;
    }
    return off;
}

}  // namespace

template <bool kDelta>
__global__ void __launch_bounds__(kRThreads, BC_DEC3_MINB)
    svb_decode_batch3_kernel(const bcgpu_decode_segment* __restrict__ segs, uint64_t nseg,
                             const uint8_t* __restrict__ in, uint32_t* __restrict__ out, unsigned long long* status,
                             uint32_t epoch, uint32_t long_hint, uint32_t ring_bytes, unsigned long long* tickets,
                             uint32_t chunk) {
    extern __shared__ __align__(128) uint8_t rdsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    RWarpHdr& B = reinterpret_cast<RWarpHdr*>(rdsm)[warp];
    uint8_t* ring_p = rdsm + kRWarps * sizeof(RWarpHdr) + warp * (ring_bytes + kRingSlack);
    if (lane == 0)
        for (uint32_t q = 0; q < kRSlots; ++q) mbar_init1(&B.bar[q]);
    __syncwarp();
    // nseg < 2^31 (the launcher splits larger batches).  Warps draw chunks of `chunk` (<= 32)
    // consecutive segments from a global ticket: list lengths vary, and with a fixed stride the
    // warp with the most integers finished ~14% after the average one (cfg4), the SMs draining
    // unevenly; a chunk's descriptors are also one coalesced read.  The next chunk is drawn a
    // whole chunk ahead, so the atomic's round trip is never waited for.
    const uint32_t GW = gridDim.x * kRWarps;
    const uint32_t nsg = (uint32_t)nseg;
    const uint32_t ring = sh_addr(ring_p), bar0 = sh_addr(&B.bar[0]), carry_s = sh_addr(&B.carry);
    const uint64_t pol = l2_policy_drop();
    // chunk = 0: few segments per warp (large ones, as a rule): the fixed stride gw, gw + GW, ...
    // instead, 32 of them checked per refill (a chunk of one or two segments per draw exposed
    // the descriptor read's latency at every draw: cfg5 +1.5%)
    const bool stat = chunk == 0;
    const uint32_t gw = blockIdx.x * kRWarps + warp;
    const uint32_t cnt = nsg > gw ? (nsg - gw + GW - 1) / GW : 0u;  // fixed stride: this warp's segments
    uint32_t tnext = 0;  // lane 0: the chunk after the current one
    auto draw = [&]() {  // -> the current chunk's first segment; draws the one after it
        const uint32_t cur = __shfl_sync(kFull, tnext, 0);
        if (lane == 0) tnext = stat ? tnext + 32u : (uint32_t)atomicAdd(tickets, (unsigned long long)chunk);
        return cur;
    };
    auto left = [&](uint32_t c) {  // segments of the chunk that starts at c
        return stat ? (c < cnt ? min(32u, cnt - c) : 0u) : (c < nsg ? min(chunk, nsg - c) : 0u);
    };
    if (lane == 0) tnext = stat ? 0u : (uint32_t)atomicAdd(tickets, (unsigned long long)chunk);
    uint32_t cb = draw();      // the current chunk: its first segment (fixed stride: its first index k)
    uint32_t ncur = left(cb);  // its segments
    auto seg_ptr = [&](uint32_t k) {  // the chunk's k-th segment
        return reinterpret_cast<const ulonglong2*>(segs + (stat ? gw + (uint64_t)(cb + k) * GW : (uint64_t)cb + k));
    };

    // Lane l checks the descriptor of the warp's segment dbase + l once: info = its ring cover
    // (decoded here) | the status it reports << 16 | 1 << 31 when it is not decoded here.  The
    // descriptors go to a per-warp table in shared memory (lane 0 reads one when it issues it),
    // so they hold no registers through the decode (re-reading them from global memory stalled
    // lane 0 on L2 misses: the warp's descriptors are a grid-stride apart).
    uint32_t info = 0;
    auto check = [&]() {
        const uint32_t k = lane;
        info = 0x80000000u;
        if (k < ncur) {
            const ulonglong2 sb = __ldg(seg_ptr(k));  // src_offset, src_bytes
            const ulonglong2 dn = __ldg(seg_ptr(k) + 1);  // dst_offset, n | prev << 32
            B.desc[lane][0] = sb;
            B.desc[lane][1] = dn;
            const uint32_t n = (uint32_t)dn.y;
            const uint64_t ngroups = ((uint64_t)n + 3) >> 2;
            uint32_t code = 0;
            if (n > kBatchSmallN)  // svb_batch2.cu decodes it -- unless the caller's max_seg_n said no segment is long
                code = long_hint && n > long_hint ? (uint32_t)BCGPU_ERR_INVALID_ARGUMENT : 0u;
            else if (n == 0)
                code = sb.y != 0 ? (uint32_t)BCGPU_ERR_TRAILING_BYTES : 0u;
            else if (sb.y < ngroups)
                code = BCGPU_ERR_TRUNCATED;
            else if (sb.y > ngroups + 4ull * n)
                code = BCGPU_ERR_TRAILING_BYTES;
            const uintptr_t beg = (uintptr_t)in + sb.x;
            const uint32_t cover = (uint32_t)(((beg + sb.y + 15) & ~(uintptr_t)15) - (beg & ~(uintptr_t)15));
            const bool here = n != 0 && n <= kBatchSmallN && code == 0;
            info = here ? cover : (0x80000000u | (code << 16));
        }
    };
    check();
    __syncwarp();
    uint32_t di = 0;                // next descriptor of the batch (lane index)
    uint32_t head = 0, tail = 0;    // ring byte counters (allocated incl. wrap waste, freed)
    uint32_t hpos = 0;              // ring offset of the next allocation
    uint32_t qh = 0, qt = 0;        // items issued, consumed
    for (;;) {
        // issue every segment that fits (a full ring leaves descriptor di pending: its check is
        // per lane above, so a retry costs one shuffle)
        while (qh - qt < kRSlots && di < ncur) {
            const uint32_t inf = __shfl_sync(kFull, info, di);
            if (!(inf & 0x80000000u)) {
                const uint32_t cover = inf;
                if (qh == qt) head = tail = hpos = 0;  // empty ring: restart at 0 (any item fits)
                const bool wrap = hpos + cover > ring_bytes;  // skip the ring's end (possibly 0 bytes)
                const uint32_t waste = wrap ? ring_bytes - hpos : 0u;
                const uint32_t at = wrap ? 0u : hpos;
                if (head + waste + cover - tail > ring_bytes) break;  // wait for space
                const uint32_t slot = qh % kRSlots;
                if (lane == 0) {
                    const ulonglong2 sb = B.desc[di][0], dn = B.desc[di][1];
                    const uintptr_t beg = (uintptr_t)in + sb.x;
                    RItem& it = B.item[slot];
                    it.dst = dn.x;
                    it.n = (uint32_t)dn.y;
                    it.prev = (uint32_t)(dn.y >> 32);
                    it.bytes = (uint32_t)sb.y;
                    it.spos = at + (uint32_t)(beg & 15);
                    it.end = head + waste + cover;
                    fence_async_smem();  // the ring bytes were last read through the generic proxy
                    mbar_expect_s(bar0 + 8 * slot, cover);
                    tma_load_hint_s(ring + at, reinterpret_cast<const void*>(beg & ~(uintptr_t)15), cover,
                                    bar0 + 8 * slot, pol);
                }
                head += waste + cover;
                hpos = at + cover;
                ++qh;
            } else if (lane == 0 && (inf >> 16) != 0x8000u) {  // not decoded here: report its status
                report3(status, epoch, (inf >> 16) & 0x7FFFu);
            }
            if (++di == ncur) {  // the chunk is issued: on to the next one
                cb = draw();
                ncur = left(cb);
                di = 0;
                __syncwarp();  // lane 0 has read the table
                check();
                __syncwarp();
            }
        }
        __syncwarp();  // lane 0's item records before every lane reads them
        if (qh == qt) break;
        // decode the oldest item
        const uint32_t slot = qt % kRSlots;
        mbar_wait_parity(&B.bar[slot], (qt / kRSlots) & 1u);
        const RItem it = B.item[slot];
        uint32_t* o = out + it.dst;
        const uint32_t data = decode_resident<kDelta>(ring + it.spos, it.bytes, it.n, kDelta ? it.prev : 0u, carry_s, o);
        if (lane == 0) {
            const uint64_t need = (uint64_t)((it.n + 3) >> 2) + data;
            if (need != it.bytes) report3(status, epoch, need > it.bytes ? BCGPU_ERR_TRUNCATED : BCGPU_ERR_TRAILING_BYTES);
        }
        tail = it.end;
        ++qt;
        __syncwarp();
    }
    // the last warp of the grid to finish leaves the ticket words zero for the next launch
    if (lane == 0 && atomicAdd(tickets + 1, 1ull) == (unsigned long long)GW - 1) {
        tickets[0] = 0;
        tickets[1] = 0;
    }
}

cudaError_t launch_decode_batch3(const bcgpu_decode_segment* segs, uint64_t nseg, const uint8_t* in, uint32_t* out,
                                 int delta, const BatchArgs& ba, cudaStream_t stream) {
    const uint32_t ring_kb = (ba.flags >> 16) & 0xFFu;  // debug: ring KiB per warp
    const uint32_t ring = ring_kb ? (ring_kb << 10 < kItemMax ? kItemMax : ring_kb << 10) : kRingDefault;
    const size_t smem = kRWarps * (sizeof(RWarpHdr) + ring + kRingSlack);
    auto kd = svb_decode_batch3_kernel<true>;
    auto kp = svb_decode_batch3_kernel<false>;
    cudaError_t a = launch_ensure_smem(kd, smem);
    if (a != cudaSuccess) return a;
    a = launch_ensure_smem(kp, smem);
    if (a != cudaSuccess) return a;
    const int sms = launch_sms(launch_current_device());
    const int o1 = launch_occupancy(kd, kRThreads, smem);
    const int o2 = launch_occupancy(kp, kRThreads, smem);
    int occ = o1 < o2 ? o1 : o2;
    if (occ < 1) occ = 1;
    const uint32_t occ_cap = (ba.flags >> 12) & 7u;  // debug: CTAs per SM
    if (occ_cap && (int)occ_cap < occ) occ = (int)occ_cap;
    const uint64_t want = (nseg + kRWarps - 1) / kRWarps, cap = (uint64_t)sms * occ;
    const int grid = (int)(want < cap ? want : cap);
    if (grid <= 0) return cudaSuccess;
    // a non-zero max_seg_n <= kBatchSmallN means no long-segment launch follows: a longer
    // segment contradicts the hint and is reported instead of silently skipped
    const uint32_t hint = ba.max_seg_n != 0 && ba.max_seg_n <= kBatchSmallN ? ba.max_seg_n : 0u;
    constexpr uint64_t kMaxSeg = 1ull << 31;  // the kernel counts segments in 32 bits
    for (uint64_t s0 = 0; s0 < nseg; s0 += kMaxSeg) {
        const uint64_t ns = nseg - s0 < kMaxSeg ? nseg - s0 : kMaxSeg;
        // chunks of kChunkMax segments when a warp's share is at least four of them; else 0 = the
        // fixed stride
        const uint64_t per = ns / (4ull * (uint64_t)grid * kRWarps);
        const uint32_t chunk = per >= kChunkMax ? kChunkMax : 0u;
        (delta ? kd : kp)<<<grid, kRThreads, smem, stream>>>(segs + s0, ns, in, out, ba.status, ba.epoch, hint, ring,
                                                             ba.tickets, chunk);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// segment-resident batch encode (svb_encode / prev-seeded delta encode per segment,
// stream_vbyte.hpp:36, codec.hpp:92-93, extension E2)
// ---------------------------------------------------------------------------
// A segment with n <= kBatchSmallN is one item: one TMA copy of its integers into the
// warp's ring.  Groups are row-major (row j, lane l <-> control byte 32 j + l).  Per block of
// three rows every lane first reads its three groups, forms deltas and lengths and writes
// its control bytes; one packed scan places the rows' data.  Each lane then packs its
// group's <= 16 bytes into four registers, shifts them onto the 4-B word grid of the data
// buffer and writes the words it completes; the word it shares with the next group (its
// "pending" word) travels to the next lane by one shuffle and is merged into that lane's
// first word, so every shared-memory word is written once, by one lane.  The data is
// packed in place, 16 bytes below the integers it replaces (a block's output never
// reaches the next block's input); control bytes go to a small double buffer.  Both
// leave as bulk stores of their 16-B aligned interiors plus edge bytes.
namespace {

constexpr uint32_t kEHead = 16;            // ring bytes reserved below an item's integers
constexpr uint32_t kERingDefault = 9216;   // ring bytes per warp (sweep: 8-9 KiB best, 5 CTAs per SM)
constexpr uint32_t kEItemMax = ((15 + 4 * kBatchSmallN + 15) & ~15u) + 16;  // largest encode item (phase, head)
static_assert(kERingDefault >= kEItemMax, "an encode item must fit the ring");
constexpr uint32_t kECtrlBuf = 512;        // >= 16 + ceil(kBatchSmallN / 4)
constexpr uint32_t kEPieceN = kBatchSmallN;  // piece of a long segment: five full 384-integer blocks (cfg5: 1024 -> 1152 -> 1536 -> 1920 ints = 2.97 -> 2.25 -> 2.03 -> 1.91 ms)
static_assert(16 + (kBatchSmallN + 3) / 4 <= kECtrlBuf, "control buffer");

struct EItem3 {               // one piece of a segment
    unsigned long long dst;  // byte offset of the segment's stream
    unsigned long long seg;  // segment index (out_lens)
    uint32_t n, prev;        // the segment's
    uint32_t m, piece;       // integers of this piece, its index in the segment
    uint32_t spos;           // ring byte of the piece's integer 0
    uint32_t end;            // ring counter after the item
};

struct __align__(16) EWarpHdr {
    uint64_t bar[kRSlots];
    EItem3 item[kRSlots];
    uint8_t ctrl[2][kECtrlBuf];
};


// global [g, g + len) <- shared bytes at sp (sp has g's 16-B phase): bulk store of the aligned
// interior (committed by the caller), lanes store the edge bytes
__device__ __forceinline__ void put_bytes(uint8_t* g, uint32_t sp, uint32_t len) {
    const int lane = threadIdx.x & 31;
    const uintptr_t gb = (uintptr_t)g, ge = gb + len;
    const uintptr_t a_lo = (gb + 15) & ~(uintptr_t)15, a_hi = ge & ~(uintptr_t)15;
    if (a_hi > a_lo) {
        if (lane == 0) tma_store_s(reinterpret_cast<void*>(a_lo), sp + (uint32_t)(a_lo - gb), (uint32_t)(a_hi - a_lo));
        const uint32_t nh = (uint32_t)(a_lo - gb), nt = (uint32_t)(ge - a_hi);
        if ((uint32_t)lane < nh) g[lane] = (uint8_t)lds8(sp + lane);
        if ((uint32_t)lane < nt) g[(a_hi - gb) + lane] = (uint8_t)lds8(sp + (uint32_t)(a_hi - gb) + lane);
    } else if ((uint32_t)lane < len) {  // no aligned interior: < 32 bytes
        g[lane] = (uint8_t)lds8(sp + lane);
    }
}

// One block of three rows of an encode piece (see encode_resident).  kFull: the three rows
// hold 384 integers (no partial or absent groups, no masking).
template <bool kDelta, bool kFB>
__device__ __forceinline__ void encode_block(uint32_t Sin, uint32_t blk, uint32_t ng, uint32_t tail, uint32_t rows,
                                             bool al16, uint32_t cb, uint32_t db, uint32_t& run, uint32_t& carry,
                                             uint32_t& off) {
    const int lane = threadIdx.x & 31;
    uint4 d[3];
    uint32_t cnts[3];
    uint32_t any = 0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        if (!kFB && blk + j >= rows) {  // past the piece's last row (warp-uniform)
            d[j] = make_uint4(0, 0, 0, 0);
            cnts[j] = 0;
            continue;
        }
        const uint32_t g = 32 * (blk + j) + lane;
        const uint32_t cnt = kFB ? 4u : (g + 1 < ng ? 4u : (g + 1 == ng ? tail : 0u));
        const uint32_t a = (kFB || cnt) ? Sin + 16 * g : Sin;
        uint4 x = al16 ? lds128(a) : make_uint4(lds32(a), lds32(a + 4), lds32(a + 8), lds32(a + 12));
        if (!kFB && cnt < 4) x = mask_tail(x, cnt);
        if constexpr (kDelta) {
            uint32_t pw = __shfl_up_sync(0xffffffffu, x.w, 1);
            if (lane == 0) pw = run;
            run = __shfl_sync(0xffffffffu, x.w, 31);
            x = make_uint4(x.x - pw, x.y - x.x, x.z - x.y, x.w - x.z);
            if (!kFB && cnt < 4) x = mask_tail(x, cnt);
        }
        d[j] = x;
        cnts[j] = cnt;
        any |= x.x | x.y | x.z | x.w;
    }
    if (kFB && __all_sync(0xffffffffu, any < 256u)) {
        // every integer takes one byte: control bytes 0, group g's four bytes at data offset 4 g,
        // one word per lane and row; every lane of a row shares the word phase u
        const uint32_t u8 = ((db + off) & 3u) << 3;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const uint4 x = d[j];
            sts8(cb + 32 * (blk + j) + lane, 0u);
            const uint32_t P = __byte_perm(__byte_perm(x.x, x.y, 0x0040), __byte_perm(x.z, x.w, 0x0040), 0x5410);
            const uint32_t o = db + off + 128 * j + 4 * lane;
            __syncwarp();  // (in place) every lane has read the block before any lane writes
            if (u8 == 0) {
                sts32(o, P);
            } else {
                const uint32_t W0 = P << u8, W1 = P >> (32 - u8);
                uint32_t pin = __shfl_up_sync(0xffffffffu, W1, 1);
                if (lane == 0) pin = carry;
                carry = __shfl_sync(0xffffffffu, W1, 31);
                sts32(o & ~3u, W0 | pin);
            }
        }
        if (u8 == 0) carry = 0;
        off += 384;
        // the piece's last group: its bytes in the word after it (lane 31's W1, now in carry)
        if (blk + 3 == rows && u8 != 0 && lane == 0) sts32((db + off) & ~3u, carry);
        return;
    }
    if constexpr (kFB) {
        // full block: control bytes, one packed scan, then the branch-free word pack (svb_pack.cuh)
        uint32_t C3[3], P3 = 0;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            uint32_t tot;
            C3[j] = group_ctrl(d[j], tot);
            sts8(cb + 32 * (blk + j) + lane, C3[j]);
            P3 |= tot << (10 * j);
        }
        const uint32_t I3 = warp_inclusive_scan(P3);
        const uint32_t T3 = __shfl_sync(0xffffffffu, I3, 31), E3 = I3 - P3;
        __syncwarp();  // every lane has read the block's integers before any lane packs over them
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const uint32_t o = db + off + ((E3 >> (10 * j)) & 0x3FFu);
            off += (T3 >> (10 * j)) & 0x3FFu;
            pack_group_row(d[j], C3[j], o, carry);
        }
        // the piece's last group leaves its partial word (now in carry)
        if ((blk + 3) * 32 >= ng && lane == 0 && ((db + off) & 3u)) sts32((db + off) & ~3u, carry);
        return;
    } else {
        // the piece's last block: rows past its end skipped, groups past its end write nothing
        // (except the lane right after the last group, which stores that group's pending word)
        uint32_t C3[3], T3r[3], P3 = 0;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            uint32_t tot;
            C3[j] = group_ctrl(d[j], tot);
            const uint32_t cnt = cnts[j];
            T3r[j] = cnt ? tot - (4u - cnt) : 0u;  // unused places count 1 byte in tot
            if (cnt) sts8(cb + 32 * (blk + j) + lane, C3[j]);
            P3 |= T3r[j] << (10 * j);
        }
        const uint32_t I3 = warp_inclusive_scan(P3);
        const uint32_t T3 = __shfl_sync(0xffffffffu, I3, 31), E3 = I3 - P3;
        __syncwarp();  // every lane has read the block's integers before any lane packs over them
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            if (blk + j >= rows) break;  // warp-uniform
            const uint32_t g = 32 * (blk + j) + lane;
            const uint32_t o = db + off + ((E3 >> (10 * j)) & 0x3FFu);
            off += (T3 >> (10 * j)) & 0x3FFu;
            const uint32_t re = 32 * (blk + j + 1);  // groups up to the row's end
            if (re < ng || (re == ng && tail == 4))  // a whole row (warp-uniform): the unmasked pack
                pack_group_row(d[j], C3[j], o, carry);
            else
                pack_group_row_masked(d[j], C3[j], o, carry, T3r[j], g <= ng);
        }
        // a last row that ends with lane 31 left the last group's pending word in carry
        if ((ng & 31u) == 0 && lane == 0 && ((db + off) & 3u)) sts32((db + off) & ~3u, carry);
        return;
    }
}

// Encode one resident piece of m integers at shared Sin (4-B aligned): control bytes -> shared
// byte cb + g, data -> shared byte db + q (db has the data destination's 16-B phase and lies
// 1..31 bytes below Sin).  run: x_{-1} (delta).  Returns the data bytes.
template <bool kDelta>
__device__ __forceinline__ uint32_t encode_resident(uint32_t Sin, uint32_t m, uint32_t run, uint32_t cb, uint32_t db) {
    const uint32_t ng = (m + 3) >> 2;
    const uint32_t tail = (m & 3u) ? (m & 3u) : 4u;
    const uint32_t rows = (ng + 31) >> 5;
    const bool al16 = (Sin & 15u) == 0;
    uint32_t carry = 0;  // pending word of the previous row's lane 31
    uint32_t off = 0;
    uint32_t blk = 0;
#pragma unroll 1
    for (; (blk + 3) * 128 <= m; blk += 3) encode_block<kDelta, true>(Sin, blk, ng, tail, rows, al16, cb, db, run, carry, off);
    if (blk < rows) encode_block<kDelta, false>(Sin, blk, ng, tail, rows, al16, cb, db, run, carry, off);
    return off;
}

// Size pass of one resident piece (bcgpu_svb_encoded_sizes_batch_device): the data bytes of its
// m integers at shared Sin (run: x_{-1}, delta).
template <bool kDelta>
__device__ __forceinline__ uint32_t size_resident(uint32_t Sin, uint32_t m, uint32_t run) {
    const int lane = threadIdx.x & 31;
    const uint32_t ng = (m + 3) >> 2, rows = (ng + 31) >> 5, tail = (m & 3u) ? (m & 3u) : 4u;
    const bool al16 = (Sin & 15u) == 0;
    uint32_t acc = 0;
#pragma unroll 4
    for (uint32_t r = 0; r < rows; ++r) {
        const uint32_t g = 32 * r + lane;
        const uint32_t cnt = g + 1 < ng ? 4u : (g + 1 == ng ? tail : 0u);
        const uint32_t a = cnt ? Sin + 16 * g : Sin;
        uint4 x = al16 ? lds128(a) : make_uint4(lds32(a), lds32(a + 4), lds32(a + 8), lds32(a + 12));
        if constexpr (kDelta) {
            uint32_t pw = __shfl_up_sync(kFull, x.w, 1);
            if (lane == 0) pw = run;
            run = __shfl_sync(kFull, x.w, 31);
            x = make_uint4(x.x - pw, x.y - x.x, x.z - x.y, x.w - x.z);
        }
        const uint32_t s4 = blen_m1(x.x) + (cnt > 1 ? blen_m1(x.y) : 0u) + (cnt > 2 ? blen_m1(x.z) : 0u) +
                            (cnt > 3 ? blen_m1(x.w) : 0u);
        acc += cnt ? s4 + cnt : 0u;
    }
    return __reduce_add_sync(kFull, acc);
}

}  // namespace

// Items are pieces: a segment of n <= kBatchSmallN integers is one piece; a longer one is cut
// into kEPieceN-integer pieces that the same warp encodes in order, carrying the data offset
// and the delta base in registers (control bytes of piece k at k * kEPieceN / 4).
template <bool kDelta, bool kSizes>
__global__ void __launch_bounds__(kRThreads, BC_ENC3_MINB)
    svb_encode_batch3_kernel(const bcgpu_encode_segment* __restrict__ segs, uint64_t nseg,
                             const uint32_t* __restrict__ in, uint8_t* __restrict__ out,
                             uint64_t* __restrict__ out_lens, unsigned long long* status, uint32_t epoch,
                             uint32_t ring_bytes, unsigned long long* tickets, uint32_t chunk) {
    extern __shared__ __align__(128) uint8_t edsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    EWarpHdr& B = reinterpret_cast<EWarpHdr*>(edsm)[warp];
    uint8_t* ring_p = edsm + kRWarps * sizeof(EWarpHdr) + warp * (ring_bytes + kRingSlack);
    if (lane == 0)
        for (uint32_t q = 0; q < kRSlots; ++q) mbar_init1(&B.bar[q]);
    __syncwarp();
    // nseg < 2^31 (the launcher splits larger batches); warps draw chunks of `chunk` consecutive
    // segments from the global ticket, one chunk ahead (see svb_decode_batch3_kernel)
    const uint32_t GW = gridDim.x * kRWarps;
    const uint32_t nsg = (uint32_t)nseg;
    const uint32_t ring = sh_addr(ring_p), bar0 = sh_addr(&B.bar[0]), ctrl0 = sh_addr(&B.ctrl[0][0]);
    const uint64_t pol = l2_policy_drop();
    const bool stat = chunk == 0;  // fixed stride gw, gw + GW, ... (few segments per warp)
    const uint32_t gw = blockIdx.x * kRWarps + warp;
    const uint32_t cnt = nsg > gw ? (nsg - gw + GW - 1) / GW : 0u;
    uint32_t tnext = 0;
    auto draw = [&]() {
        const uint32_t cur = __shfl_sync(kFull, tnext, 0);
        if (lane == 0) tnext = stat ? tnext + 32u : (uint32_t)atomicAdd(tickets, (unsigned long long)chunk);
        return cur;
    };
    auto left = [&](uint32_t c) {
        return stat ? (c < cnt ? min(32u, cnt - c) : 0u) : (c < nsg ? min(chunk, nsg - c) : 0u);
    };
    if (lane == 0) tnext = stat ? 0u : (uint32_t)atomicAdd(tickets, (unsigned long long)chunk);
    uint32_t cb = draw();
    uint32_t ncur = left(cb);
    auto seg_index = [&](uint32_t k) -> uint64_t {  // the chunk's k-th segment
        return stat ? gw + (uint64_t)(cb + k) * GW : (uint64_t)cb + k;
    };
    auto seg_ptr = [&](uint32_t k) { return reinterpret_cast<const ulonglong2*>(segs + seg_index(k)); };
    // Lane l checks the descriptor of the warp's segment dbase + l once: its n, and the 16-B
    // phase of its integers | 0x100 when it is empty | 0x200 when its capacity is short; it
    // keeps src, dst and prev for the shuffles that issue its pieces.
    uint32_t info_n = 0, info_f = 0, info_p = 0;
    unsigned long long info_s = 0, info_d = 0;
    auto check = [&]() {
        const uint32_t k = lane;
        if (k < ncur) {
            const ulonglong2 sc = __ldg(seg_ptr(k));  // src_offset, dst_capacity
            const ulonglong2 dn = __ldg(seg_ptr(k) + 1);  // dst_offset, n | prev << 32
            const uint32_t n = (uint32_t)dn.y;
            info_n = n;
            info_p = (uint32_t)(dn.y >> 32);
            info_s = sc.x;
            info_d = dn.x;
            info_f = (uint32_t)((uintptr_t)(in + sc.x) & 15) | (n == 0 ? 0x100u : 0u) |
                     (!kSizes && n && sc.y < (((uint64_t)n + 3) >> 2) + 4ull * n ? 0x200u : 0u);
        }
    };
    check();
    uint32_t di = 0;
    uint32_t piece = 0;      // next piece of descriptor di
    uint32_t head = 0, tail = 0, hpos = 0;
    uint32_t tail_next = 0;  // freed once the newest item's bulk stores have read the ring
    uint32_t qh = 0, qt = 0;
    uint32_t run = 0;        // delta base of the next piece of the segment being encoded
    unsigned long long off = 0;  // data bytes of the segment's earlier pieces
    for (;;) {
        while (qh - qt < kRSlots && di < ncur) {
            const uint32_t n = __shfl_sync(kFull, info_n, di), f = __shfl_sync(kFull, info_f, di);
            const uint64_t s_idx = seg_index(di);
            bool done = true;
            if (f & 0x300u) {  // empty, or capacity short: nothing written; a zero length keeps
                if (lane == 0) {  // callers that pack by out_lens in bounds
                    out_lens[s_idx] = 0;
                    if (f & 0x200u) report3(status, epoch, BCGPU_ERR_INVALID_ARGUMENT);
                }
            } else {
                const uint32_t pn = n <= kBatchSmallN ? n : kEPieceN;  // integers per piece
                const uint32_t npieces = (n - 1) / kEPieceN + 1;
                const uint32_t m = piece + 1 < npieces ? pn : n - piece * pn;
                const uint32_t ph = f & 15u;  // pieces start 7680 B apart: every piece has the segment's phase
                const uint32_t cover = ((ph + 4 * m + 15) & ~15u) + kEHead;
                if (qh == qt) {  // nothing unconsumed: once the last item's stores have read it, restart at 0
                    if (tail_next != tail) {
                        if (lane == 0) tma_store_wait_read();
                        __syncwarp();
                    }
                    head = tail = tail_next = hpos = 0;
                }
                const bool wrap = hpos + cover > ring_bytes;
                const uint32_t waste = wrap ? ring_bytes - hpos : 0u;
                const uint32_t at = wrap ? 0u : hpos;
                if (head + waste + cover - tail > ring_bytes) break;  // wait for space
                done = piece + 1 == npieces;
                const uint32_t slot = qh % kRSlots;
                const unsigned long long src = __shfl_sync(kFull, info_s, di), dst = __shfl_sync(kFull, info_d, di);
                const uint32_t prv = __shfl_sync(kFull, info_p, di);
                if (lane == 0) {
                    const uintptr_t beg = (uintptr_t)(in + src + (uint64_t)piece * pn);
                    EItem3& it = B.item[slot];
                    it.dst = dst;
                    it.seg = s_idx;
                    it.n = n;
                    it.prev = prv;
                    it.m = m;
                    it.piece = piece;
                    it.spos = at + kEHead + ph;
                    it.end = head + waste + cover;
                    fence_async_smem();
                    mbar_expect_s(bar0 + 8 * slot, cover - kEHead);
                    tma_load_hint_s(ring + at + kEHead, reinterpret_cast<const void*>(beg & ~(uintptr_t)15),
                                    cover - kEHead, bar0 + 8 * slot, pol);
                }
                head += waste + cover;
                hpos = at + cover;
                ++qh;
            }
            if (done) {
                piece = 0;
                if (++di == ncur) {  // the chunk is issued: on to the next one
                    cb = draw();
                    ncur = left(cb);
                    di = 0;
                    check();
                }
            } else {
                ++piece;
            }
        }
        __syncwarp();
        if (qh == qt) break;
        const uint32_t slot = qt % kRSlots;
        mbar_wait_parity(&B.bar[slot], (qt / kRSlots) & 1u);
        const EItem3 it = B.item[slot];
        const uint32_t ngT = (it.n + 3) >> 2, pn = it.n <= kBatchSmallN ? it.n : kEPieceN;
        const uint32_t ng = (it.m + 3) >> 2;
        if (it.piece == 0) {
            run = kDelta ? it.prev : 0u;
            off = 0;
        }
        if constexpr (kSizes) {  // size pass: no output, the ring frees at once
            const uint32_t Sin = ring + it.spos;
            off += size_resident<kDelta>(Sin, it.m, run);
            if constexpr (kDelta) run = lds32(Sin + 4 * (it.m - 1));
            if (lane == 0 && (uint64_t)(it.piece + 1) * pn >= it.n) out_lens[it.seg] = (uint64_t)ngT + off;
            __syncwarp();
            tail = tail_next = it.end;
            ++qt;
            continue;
        }
        uint8_t* gctrl = out + it.dst + (uint64_t)it.piece * (pn >> 2);
        uint8_t* gdata = out + it.dst + ngT + off;
        const uint32_t hc = (uint32_t)((uintptr_t)gctrl & 15), hd = (uint32_t)((uintptr_t)gdata & 15);
        const uint32_t Sin = ring + it.spos;
        const uint32_t db = ((Sin - 16u) & ~15u) + hd;  // the item's reserved head: 1..31 bytes below Sin
        const uint32_t cbuf = ctrl0 + kECtrlBuf * (qt & 1);
        const uint32_t data = encode_resident<kDelta>(Sin, it.m, run, cbuf + hc, db);
        if constexpr (kDelta) run = lds32(Sin + 4 * (it.m - 1));  // x_{-1} of the next piece
        off += data;
        fence_async_smem();
        __syncwarp();
        put_bytes(gctrl, cbuf + hc, ng);
        put_bytes(gdata, db, data);
        if (lane == 0) {
            tma_store_commit();
            if ((uint64_t)(it.piece + 1) * pn >= it.n) out_lens[it.seg] = (uint64_t)ngT + off;
            tma_store_wait_read_but1();  // the previous item's stores have read its ring bytes and ctrl buffer
        }
        __syncwarp();
        tail = tail_next;
        tail_next = it.end;
        ++qt;
    }
    if (lane == 0) {
        tma_store_wait_read();
        // the last warp of the grid to finish leaves the ticket words zero for the next launch
        if (atomicAdd(tickets + 1, 1ull) == (unsigned long long)GW - 1) {
            tickets[0] = 0;
            tickets[1] = 0;
        }
    }
}

cudaError_t launch_encode_batch3(const bcgpu_encode_segment* segs, uint64_t nseg, const uint32_t* in, uint8_t* out,
                                 uint64_t* out_lens, int delta, const BatchArgs& ba, cudaStream_t stream, bool sizes) {
    const uint32_t ring_kb = (ba.flags >> 24) & 0xFFu;  // debug: ring KiB per warp
    // rings: 9 KiB (5 CTAs per SM at 94 registers; a long segment's 7.5 KiB pieces still overlap
    // with short items).  Rings of exactly one largest item let a sixth CTA fit while the kernel
    // took 80 registers; the 64-bit-shift pack needs 94 (80 spills: cfg4 1.96 vs 1.86 ms), and at
    // five CTAs the larger ring is the faster one (cfg4 1.848 vs 1.862 ms)
    const uint32_t ring = ring_kb ? (ring_kb << 10 < kEItemMax ? kEItemMax : ring_kb << 10) : kERingDefault;
    const size_t smem = kRWarps * (sizeof(EWarpHdr) + ring + kRingSlack);
    const void* fns[4] = {(const void*)svb_encode_batch3_kernel<true, false>,
                          (const void*)svb_encode_batch3_kernel<false, false>,
                          (const void*)svb_encode_batch3_kernel<true, true>, (const void*)svb_encode_batch3_kernel<false, true>};
    for (const void* f : fns) {
        const cudaError_t a = launch_ensure_smem(f, smem);
        if (a != cudaSuccess) return a;
    }
    const int sms = launch_sms(launch_current_device());
    const int o1 = launch_occupancy(svb_encode_batch3_kernel<true, false>, kRThreads, smem);
    const int o2 = launch_occupancy(svb_encode_batch3_kernel<false, false>, kRThreads, smem);
    int occ = o1 < o2 ? o1 : o2;
    if (occ < 1) occ = 1;
    const uint32_t occ_cap = (ba.flags >> 12) & 7u;  // debug: CTAs per SM
    if (occ_cap && (int)occ_cap < occ) occ = (int)occ_cap;
    const uint64_t want = (nseg + kRWarps - 1) / kRWarps, capg = (uint64_t)sms * occ;
    const int grid = (int)(want < capg ? want : capg);
    if (grid <= 0) return cudaSuccess;
    auto kern = sizes ? (delta ? svb_encode_batch3_kernel<true, true> : svb_encode_batch3_kernel<false, true>)
                      : (delta ? svb_encode_batch3_kernel<true, false> : svb_encode_batch3_kernel<false, false>);
    constexpr uint64_t kMaxSeg = 1ull << 31;  // the kernel counts segments in 32 bits
    for (uint64_t s0 = 0; s0 < nseg; s0 += kMaxSeg) {
        const uint64_t ns = nseg - s0 < kMaxSeg ? nseg - s0 : kMaxSeg;
        const uint64_t per = ns / (4ull * (uint64_t)grid * kRWarps);
        const uint32_t chunk = per >= kChunkMax ? kChunkMax : 0u;
        kern<<<grid, kRThreads, smem, stream>>>(segs + s0, ns, in, out, out_lens + s0, ba.status, ba.epoch, ring,
                                                ba.tickets, chunk);
    }
    return cudaGetLastError();
}

}  // namespace bcgpu
