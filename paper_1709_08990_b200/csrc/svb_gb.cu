// svb_gb.cu -- varint-GB encode / decode on the GPU.
//
// Format (reference proj/core/include/bytecodec/varint_gb.hpp:14-17):
// ceil(n/4) groups, each a control byte (field i = byte_length(x_i) - 1, integer 0 in
// the low two bits) followed by the little-endian bytes of its integers; a final
// incomplete group has zero unused fields and no bytes for absent integers.
//
// Encode.  The stream is the same size as Stream VByte's (ceil(n/4) + sum of byte
// lengths), and group k sits at k + (data bytes of groups < k): sub-tile s starts at
// its Stream VByte data offset + 256 s.  So the Stream VByte size scan
// (svb_encode.cu; with the same prev-seeded delta transform) provides every sub-tile's
// offset, and gb_encode_kernel assembles each
// sub-tile's interleaved groups in shared memory (at the destination's 16-B phase) and
// writes them with 128-bit stores, byte stores only at the two edges.
//
// Decode.  Control positions are data-dependent: group k's control byte follows group
// k-1's data, so no group can be located without the ones before
// it.  The chain is resolved with transfer functions:
//   1. gb_table_kernel: the stream is cut into 4 KiB chunks; a group starting in one
//      chunk ends at most 16 bytes into the next, so a chunk is entered at one of 17
//      offsets.  Per chunk it records, for each entry offset, the exit offset into the
//      next chunk and the groups started (lane-parallel segment tables, below).
//   2. gb_compose_kernel / gb_expand_kernel: the tables compose associatively (follow
//      the exit of one into the next, add the counts).  A 32-ary tree of compositions
//      is built bottom-up, then walked top-down from entry 0 at the stream's start,
//      which resolves every chunk's true entry offset and the index of its first group.
//      The root's count also settles truncation.
//   3. gb_decode_kernel: per chunk, every lane lists the group starts in its segment
//      from the true entry, then the warp decodes 32 groups per round (all-small fast
//      path for control 0, field by field otherwise) and stores 128-bit rows.  Delta:
//      the chunk's value carry comes from a decoupled look-back over chunk sums, and the
//      prefix sum is fused (warp scan + carry).  The warp holding group ceil(n/4)-1
//      checks the stream end (truncated / trailing bytes).
// All decode kernels form one chain under programmatic dependent launch.
#include <cstdint>

#include "svb_device.cuh"
#include "svb_fast.cuh"
#include "svb_kernels.cuh"
#include "svb_scan.cuh"
#include "svb_warp.cuh"

namespace bcgpu {

namespace {

constexpr uint32_t kGbChunk = 4096;                 // compressed bytes per decode chunk (one warp)
constexpr uint32_t kGbStage = kGbChunk + 64;        // staged: <16 phase + chunk + the last group's overhang
constexpr int kGbE = 17;                            // entry offsets 0..16 (a group spans <= 17 bytes)
constexpr uint32_t kGbFan = 32;                     // tables composed per tree node
constexpr int kGbWarps = 4;                         // chunks per CTA (table / decode kernels)
constexpr uint32_t kGbSeg = 132;                    // bytes per lane segment of a chunk (31 * 132 + 4 = 4096)
constexpr int kGbEncWarps = 8;                      // sub-tiles per CTA (encode)
constexpr int kGbTreeWarps = 4;                     // tree nodes per CTA (compose / expand kernels)
constexpr uint32_t kGbMaxGroups = kGbChunk / 5 + 2;  // groups starting in one chunk (>= 5 B each but the last)
constexpr uint32_t kGbEncBuf = kWTGroups + 4 * kWTInts + 32;  // one sub-tile's groups + phase

__device__ __forceinline__ void gb_report(unsigned long long* st, uint32_t epoch, uint32_t code) {
    if (st) *st = ((unsigned long long)epoch << 32) | code;
}

// bytes [off, off + cnt) of the stream into buf (16-B aligned) at buf index phase + i,
// phase = (in + off) & 15; bytes outside the stream read as 0.  Returns the phase.
__device__ __forceinline__ uint32_t gb_stage(const uint8_t* in, uint64_t len, uint64_t off, uint32_t cnt, uint8_t* buf) {
    const int lane = threadIdx.x & 31;
    const uintptr_t lo = (uintptr_t)in, hi = lo + len, a = lo + off, g0 = a & ~(uintptr_t)15;
    const uint32_t ph = (uint32_t)(a - g0);
    const uint32_t ng = (ph + cnt + 15) / 16;
    for (uint32_t i = lane; i < ng; i += 32)
        *reinterpret_cast<uint4*>(buf + 16 * i) = load_chunk_guarded(g0 + 16 * i, lo, hi);
    return ph;
}

// bytes of a full group with control byte c (1 control + 4..16 data)
__device__ __forceinline__ uint32_t gb_group_bytes(uint32_t c) { return 5u + fsum(c); }

// the k (1..4) integers of the group whose control byte c is at shared address a
__device__ __forceinline__ uint4 gb_group_values(uint32_t a, uint32_t c, uint32_t k) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (c == 0 && k == 4) {  // all-small fast path: four one-byte integers
        const uint32_t x = __funnelshift_r(lds32((a + 1) & ~3u), lds32(((a + 1) & ~3u) + 4), ((a + 1) & 3u) * 8u);
        return make_uint4(x & 0xFFu, (x >> 8) & 0xFFu, (x >> 16) & 0xFFu, x >> 24);
    }
    uint32_t p = a + 1;
    uint32_t x[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t l = ((c >> (2 * i)) & 3u) + 1u;
        if ((uint32_t)i < k) {
            x[i] = extract_s(p, l);
            p += l;
        }
    }
    v = make_uint4(x[0], x[1], x[2], x[3]);
    return v;
}

}  // namespace

// ---------------------------------------------------------------------------
// encode: one warp per 1024-integer sub-tile, offsets from the Stream VByte size scan
// ---------------------------------------------------------------------------
template <bool kDelta>
__global__ void __launch_bounds__(256)
    gb_encode_kernel(const uint32_t* __restrict__ in, uint64_t n, uint32_t prev, uint8_t* __restrict__ out,
                     DecodeMeta meta) {
    __shared__ __align__(16) uint8_t sbuf[kGbEncWarps][kGbEncBuf];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint64_t s = (uint64_t)blockIdx.x * kGbEncWarps + warp;
    if (s >= nsub) return;
    const uint64_t g0 = s * kWTGroups;
    const uint64_t o0 = meta.chunkpre[s / kChunkSubs] + meta.localpre[s] + g0;  // data before + control bytes before
    uint8_t* dst = out + o0;
    const uint32_t ph = (uint32_t)((uintptr_t)dst & 15);
    const uint32_t sb = sh_addr(sbuf[warp]);
    const bool in16 = (((uintptr_t)in) & 15) == 0;
    uint32_t off = ph;
#pragma unroll 1
    for (int j = 0; j < kWTRows; ++j) {
        const uint64_t g = g0 + 32 * j + lane;
        const uint32_t cnt = group_count(g, ngroups, tail_r);
        uint4 x = make_uint4(0, 0, 0, 0);
        if (cnt == 4 && in16) {
            x = ldg_stream_v4(in + 4 * g);
        } else if (cnt) {
            x.x = __ldg(in + 4 * g);
            if (cnt > 1) x.y = __ldg(in + 4 * g + 1);
            if (cnt > 2) x.z = __ldg(in + 4 * g + 2);
            if (cnt > 3) x.w = __ldg(in + 4 * g + 3);
        }
        if constexpr (kDelta) {  // mod-2^32 differences, seeded with prev
            const uint32_t p = g ? (cnt ? __ldg(in + 4 * g - 1) : 0u) : prev;
            x = make_uint4(x.x - p, x.y - x.x, x.z - x.y, x.w - x.z);
        }
        // all-small row (the encoder side): every group is 00 b0 b1 b2 b3, 160 bytes
        if (__all_sync(kFull, cnt == 4 && (x.x | x.y | x.z | x.w) < 256u)) {
            const uint32_t p = sb + off + 5u * (uint32_t)lane;
            sts8(p, 0u);
            sts8(p + 1, x.x);
            sts8(p + 2, x.y);
            sts8(p + 3, x.z);
            sts8(p + 4, x.w);
            off += 160u;
            continue;
        }
        uint32_t l[4], c = 0, gs = cnt ? 1u : 0u;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            l[i] = (uint32_t)i < cnt ? dev_byte_length(comp(x, i)) : 0u;
            if ((uint32_t)i < cnt) c |= (l[i] - 1u) << (2 * i);
            gs += l[i];
        }
        const uint32_t incl = warp_inclusive_scan(gs);
        if (cnt) {
            uint32_t p = sb + off + incl - gs;
            sts8(p++, c);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                for (uint32_t b = 0; b < l[i]; ++b) sts8(p++, (comp(x, i) >> (8 * b)) & 0xFFu);
        }
        off += __shfl_sync(kFull, incl, 31);
    }
    __syncwarp();
    // bytes [ph, off) of the buffer -> dst - ph + [ph, off): whole 16-B granules as 128-bit
    // stores, the partial first / last granules byte by byte (neighbouring warps own the rest)
    uint8_t* gdst = dst - ph;
    const uint32_t ng = (off + 15) / 16;
    for (uint32_t i = lane; i < ng; i += 32) {
        const uint32_t b0 = 16 * i, b1 = b0 + 16;
        if (b0 >= ph && b1 <= off) {
            *reinterpret_cast<uint4*>(gdst + b0) = lds128(sb + b0);
        } else {
            for (uint32_t b = b0 < ph ? ph : b0; b < (b1 < off ? b1 : off); ++b) gdst[b] = (uint8_t)lds8(sb + b);
        }
    }
}

// ---------------------------------------------------------------------------
// decode 1: per-chunk transfer tables
// ---------------------------------------------------------------------------
// Lane l owns segment [132 l, 132 (l + 1)) of the chunk (lane 31: [4092, 4096)); the
// 132-byte stride puts the 32 lanes' byte reads in 32 different banks.  Walking its
// segment from the end down, a lane computes for every byte position p the chain
// started there: F(p) = the first position >= the segment end it reaches, the groups it
// starts and (delta) the sum of their values -- from the entry of next(p) = p + group
// bytes, at most 17 ahead, so a 32-entry ring per lane holds all it needs.  The ring
// ends up holding the segment's lowest 32 positions: its transfer table for entries
// a .. a + 16.  A chunk table is 32 segment lookups per entry.
struct GbRing {
    uint16_t ec[32][32];  // [position & 31][lane]: exit (5 bits) | count << 5
};
struct GbRingSum {
    uint32_t v[32][32];  // [position & 31][lane]: value sum (delta)
};

__device__ __forceinline__ void gb_seg_bounds(uint32_t l, uint32_t clen, uint32_t& a, uint32_t& b) {
    a = kGbSeg * l < clen ? kGbSeg * l : clen;
    const uint32_t e = l == 31 ? kGbChunk : kGbSeg * (l + 1);
    b = e < clen ? e : clen;
}

template <bool kDelta>
__device__ __forceinline__ void gb_segment_dp(uint32_t sa, uint32_t clen, GbRing& R, GbRingSum* S) {
    const int lane = threadIdx.x & 31;
    uint32_t a, b;
    gb_seg_bounds((uint32_t)lane, clen, a, b);
    for (uint32_t p = b; p > a;) {
        --p;
        const uint32_t c = lds8(sa + p);
        const uint32_t q = p + gb_group_bytes(c);
        uint32_t ec, sm = 0;
        if constexpr (kDelta) {
            const uint4 v = gb_group_values(sa + p, c, 4);
            sm = v.x + v.y + v.z + v.w;
        }
        if (q >= b) {
            ec = (q - b) | (1u << 5);
        } else {
            ec = (uint32_t)R.ec[q & 31][lane] + (1u << 5);
            if constexpr (kDelta) sm += S->v[q & 31][lane];
        }
        R.ec[p & 31][lane] = (uint16_t)ec;
        if constexpr (kDelta) S->v[p & 31][lane] = sm;
    }
}

// follow the chain from chunk position pos through segments [s0, s1): groups and sums added
template <bool kDelta>
__device__ __forceinline__ uint32_t gb_chase(const GbRing& R, const GbRingSum* S, uint32_t clen, uint32_t pos,
                                             uint32_t s0, uint32_t s1, uint32_t& cnt, uint32_t& sum) {
    for (uint32_t s = s0; s < s1; ++s) {
        uint32_t a, b;
        gb_seg_bounds(s, clen, a, b);
        if (pos >= b) continue;
        const uint32_t t = R.ec[pos & 31][s];
        cnt += t >> 5;
        if constexpr (kDelta) sum += S->v[pos & 31][s];
        pos = b + (t & 31u);
    }
    return pos;
}

// Tables carry exits and group counts only: the delta decode's value carries come from
// a look-back over chunk sums in gb_decode_kernel, so no value is summed here (at most
// byte positions the "control byte" is really data, and summing its would-be group cost
// more than the whole table).
__global__ void __launch_bounds__(32 * kGbWarps)
    gb_table_kernel(const uint8_t* __restrict__ in, uint64_t len, uint64_t nchunks, uint32_t* __restrict__ tcnt,
                    uint32_t* __restrict__ texit, uint16_t* __restrict__ segtab) {
    // programmatic dependent launch: the next kernel of the chain may be scheduled now; this
    // one reads its predecessor's output only after the wait
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ __align__(16) uint8_t sbuf[kGbWarps][kGbStage];
    __shared__ GbRing ring[kGbWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t chunk = (uint64_t)blockIdx.x * kGbWarps + warp;
    if (chunk >= nchunks) return;
    const uint64_t cs = chunk * kGbChunk;
    const uint32_t clen = (uint32_t)(len - cs < kGbChunk ? len - cs : kGbChunk);
    const uint32_t ph = gb_stage(in, len, cs, clen + 32, sbuf[warp]);
    __syncwarp();
    const uint32_t sa = sh_addr(sbuf[warp]) + ph;
    gb_segment_dp<false>(sa, clen, ring[warp], nullptr);
    // the segment tables for the decode pass: entry e of lane l's segment, [e][l]
    {
        uint32_t a, b;
        gb_seg_bounds((uint32_t)lane, clen, a, b);
        uint16_t* st = segtab + chunk * (kGbE * 32);
#pragma unroll
        for (int e = 0; e < kGbE; ++e) st[e * 32 + lane] = ring[warp].ec[(a + e) & 31][lane];
    }
    __syncwarp();
    if (lane < kGbE) {
        uint32_t cnt = 0, sum = 0;
        const uint32_t pos = gb_chase<false>(ring[warp], nullptr, clen, (uint32_t)lane, 0, 32, cnt, sum);
        const uint64_t i = chunk * kGbE + lane;
        tcnt[i] = cnt;
        texit[i] = pos - clen;
    }
}

// ---------------------------------------------------------------------------
// decode 2: compose 32 child tables per node (bottom-up), resolve entries (top-down)
// ---------------------------------------------------------------------------
struct GbTreeSmem {
    uint32_t cnt[kGbFan * kGbE], exit[kGbFan * kGbE];
};

__device__ __forceinline__ uint32_t gb_load_children(GbTreeSmem& sm, const uint32_t* ccnt, const uint32_t* cexit,
                                                     uint64_t nchild, uint64_t parent) {
    const int lane = threadIdx.x & 31;
    const uint64_t k0 = parent * kGbFan;
    const uint32_t nk = (uint32_t)(nchild - k0 < kGbFan ? nchild - k0 : kGbFan);
    for (uint32_t i = lane; i < nk * kGbE; i += 32) {
        sm.cnt[i] = ccnt[k0 * kGbE + i];
        sm.exit[i] = cexit[k0 * kGbE + i];
    }
    __syncwarp();
    return nk;
}

__global__ void __launch_bounds__(32 * kGbTreeWarps)
    gb_compose_kernel(const uint32_t* __restrict__ ccnt, const uint32_t* __restrict__ cexit, uint64_t nchild,
                      uint32_t* __restrict__ pcnt, uint32_t* __restrict__ pexit, uint64_t nparent) {
    // programmatic dependent launch: the next kernel of the chain may be scheduled now; this
    // one reads its predecessor's output only after the wait
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ GbTreeSmem sm[kGbTreeWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t p = (uint64_t)blockIdx.x * kGbTreeWarps + warp;
    if (p >= nparent) return;
    const uint32_t nk = gb_load_children(sm[warp], ccnt, cexit, nchild, p);
    if (lane < kGbE) {
        uint32_t x = (uint32_t)lane, cnt = 0;
        for (uint32_t k = 0; k < nk; ++k) {
            const uint32_t i = k * kGbE + x;
            cnt += sm[warp].cnt[i];
            x = sm[warp].exit[i];
        }
        pcnt[p * kGbE + lane] = cnt;
        pexit[p * kGbE + lane] = x;
    }
}

// root != 0: the single top node, entered at offset 0; its group count (groups chained
// from the stream's start) below ceil(n/4) means the stream is truncated
__global__ void __launch_bounds__(32 * kGbTreeWarps)
    gb_expand_kernel(const uint32_t* __restrict__ ccnt, const uint32_t* __restrict__ cexit, uint64_t nchild,
                     const uint32_t* __restrict__ pentry, const uint32_t* __restrict__ pcntpre, uint64_t nparent,
                     uint32_t* __restrict__ centry, uint32_t* __restrict__ ccntpre, int root, uint64_t ngroups,
                     unsigned long long* status, uint32_t epoch) {
    // programmatic dependent launch: the next kernel of the chain may be scheduled now; this
    // one reads its predecessor's output only after the wait
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ GbTreeSmem sm[kGbTreeWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t p = (uint64_t)blockIdx.x * kGbTreeWarps + warp;
    if (p >= nparent) return;
    const uint32_t nk = gb_load_children(sm[warp], ccnt, cexit, nchild, p);
    if (lane == 0) {
        uint32_t x = root ? 0u : pentry[p], cp = root ? 0u : pcntpre[p];
        for (uint32_t k = 0; k < nk; ++k) {
            const uint64_t c = p * kGbFan + k;
            centry[c] = x;
            ccntpre[c] = cp;
            const uint32_t i = k * kGbE + x;
            cp += sm[warp].cnt[i];
            x = sm[warp].exit[i];
        }
        if (root && (uint64_t)cp < ngroups) gb_report(status, epoch, BCGPU_ERR_TRUNCATED);
    }
}

// ---------------------------------------------------------------------------
// decode 3: groups of each chunk from its resolved entry
// ---------------------------------------------------------------------------
template <bool kDelta>
__global__ void __launch_bounds__(32 * kGbWarps)
    gb_decode_kernel(const uint8_t* __restrict__ in, uint64_t len, uint64_t n, uint64_t nchunks,
                     const uint32_t* __restrict__ rentry, const uint32_t* __restrict__ rcnt,
                     const uint16_t* __restrict__ segtab, uint32_t base, uint64_t* __restrict__ lstatus,
                     uint32_t* __restrict__ out, uint32_t* __restrict__ d_last, unsigned long long* status,
                     uint32_t epoch) {
    // programmatic dependent launch: the next kernel of the chain may be scheduled now; this
    // one reads its predecessor's output only after the wait
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ __align__(16) uint8_t sbuf[kGbWarps][kGbStage];
    __shared__ __align__(16) uint16_t stab[kGbWarps][kGbE * 32];
    __shared__ uint16_t spos[kGbWarps][kGbMaxGroups];
    __shared__ uint32_t wtot[kGbWarps];  // delta: the warps' chunk sums
    __shared__ uint32_t cta_ex;          // delta: carry before the CTA's first chunk
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t chunk = (uint64_t)blockIdx.x * kGbWarps + warp;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    // warps without groups of this call stay for the CTA barriers of the delta carry
    const uint64_t kb = chunk < nchunks ? rcnt[chunk] : ngroups;  // index of the chunk's first group
    const bool active = kb < ngroups;
    if (!kDelta && !active) return;
    const uint64_t cs = chunk * kGbChunk;
    const uint32_t clen = active ? (uint32_t)(len - cs < kGbChunk ? len - cs : kGbChunk) : 0u;
    const uint32_t ph = active ? gb_stage(in, len, cs, clen + 32, sbuf[warp]) : 0u;
    __syncwarp();
    const uint32_t sa = sh_addr(sbuf[warp]) + ph;
    // the chunk's segment tables (gb_table_kernel), then every lane finds where the true
    // chain enters its segment and lists the group starts in it
    if (active) {
        const uint4* src = reinterpret_cast<const uint4*>(segtab + chunk * (kGbE * 32));
        uint4* dst = reinterpret_cast<uint4*>(stab[warp]);
        for (uint32_t g = lane; g < kGbE * 32 * 2 / 16; g += 32) dst[g] = __ldg(src + g);
    }
    __syncwarp();
    uint32_t i = 0, pos = active ? rentry[chunk] : 0u;
    for (uint32_t s = 0; s < (uint32_t)lane; ++s) {
        uint32_t a, b;
        gb_seg_bounds(s, clen, a, b);
        if (pos >= b) continue;
        const uint32_t t = stab[warp][(pos - a) * 32 + s];
        i += t >> 5;
        pos = b + (t & 31u);
    }
    const uint64_t left = ngroups - kb;  // 0 when inactive
    const uint32_t lim = (uint32_t)(left < kGbMaxGroups ? left : kGbMaxGroups);  // groups of this call
    {
        uint32_t a, b;
        gb_seg_bounds((uint32_t)lane, clen, a, b);
        while (pos < b && i < lim) {
            spos[warp][i++] = (uint16_t)pos;
            pos += gb_group_bytes(lds8(sa + pos));
        }
    }
    uint32_t m = __reduce_max_sync(kFull, i);
    m = m < lim ? m : lim;
    __syncwarp();
    uint32_t run = 0;
    if constexpr (kDelta) {
        // the chunk's value sum, then its carry by decoupled look-back over the CTAs before
        // it (lower CTAs are dispatched first, so they are resident or done)
        uint32_t tot = 0;
        for (uint32_t r = 0; r < m; r += 32) {
            const uint32_t i = r + lane;
            const uint32_t k = i < m ? group_count(kb + i, ngroups, tail_r) : 0u;
            if (k) {
                const uint32_t p = spos[warp][i];
                const uint4 v = gb_group_values(sa + p, lds8(sa + p), k);
                tot += v.x + v.y + v.z + v.w;
            }
        }
        tot = __reduce_add_sync(kFull, tot);
        // one look-back per CTA (over CTAs, 4x shallower than per chunk): warp 0 combines the
        // CTA's chunk sums, every warp adds those of the warps before it
        if (lane == 0) wtot[warp] = tot;
        __syncthreads();
        if (warp == 0) {
            uint32_t ctot = lane < kGbWarps ? wtot[lane] : 0u;
            ctot = __reduce_add_sync(kFull, ctot);
            uint64_t ex = base;
            if (blockIdx.x == 0) {
                if (lane == 0) st_relaxed_gpu(lstatus, pack_status(epoch, kFlagInclusive, (uint64_t)base + ctot));
            } else {
                if (lane == 0)
                    st_relaxed_gpu(status_slot(lstatus, blockIdx.x), pack_status(epoch, kFlagAggregate, ctot));
                ex = lookback_exclusive_wide(lstatus, blockIdx.x, epoch);
                if (lane == 0)
                    st_relaxed_gpu(status_slot(lstatus, blockIdx.x), pack_status(epoch, kFlagInclusive, ex + ctot));
            }
            if (lane == 0) cta_ex = (uint32_t)ex;
        }
        __syncthreads();
        run = cta_ex;
        for (int w = 0; w < warp; ++w) run += wtot[w];
        if (!active) return;
    }
    const bool out16 = (((uintptr_t)out) & 15) == 0;
    for (uint32_t r = 0; r < m; r += 32) {
        const uint32_t i = r + lane;
        const uint64_t gi = kb + i;
        const uint32_t k = i < m ? group_count(gi, ngroups, tail_r) : 0u;
        uint4 v = make_uint4(0, 0, 0, 0);
        uint32_t c = 0, p = 0;
        if (k) {
            p = spos[warp][i];
            c = lds8(sa + p);
            v = gb_group_values(sa + p, c, k);
        }
        if constexpr (kDelta) {
            v.y += v.x;
            v.z += v.y;
            v.w += v.z;
            const uint32_t I = warp_inclusive_scan(v.w);
            v = add4(v, run + I - v.w);
            run += __shfl_sync(kFull, I, 31);
        }
        if (k) store_group(out + 4 * gi, v, k, out16);
        if (k && gi == ngroups - 1) {
            // the stream's last group: it must end exactly at the stream's end
            uint64_t end = cs + p + 1;
            for (uint32_t f = 0; f < k; ++f) end += ((c >> (2 * f)) & 3u) + 1u;
            gb_report(status, epoch,
                      end > len ? BCGPU_ERR_TRUNCATED : (end < len ? BCGPU_ERR_TRAILING_BYTES : (uint32_t)BCGPU_OK));
            if (d_last) *d_last = comp(v, (int)k - 1);
        }
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
// The decode is a chain of small kernels (table, 2 per tree level, decode): each is launched
// as a programmatic dependent of the one before, so its launch and ramp-up overlap the
// predecessor's tail (every kernel of the chain waits before reading its inputs).
template <typename... KArgs, typename... Args>
static cudaError_t gb_launch(void (*k)(KArgs...), unsigned grid, unsigned block, cudaStream_t stream, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
// device workspace of a decode of len compressed bytes: per tree level, 3 tables of 17
// words per node and 3 resolved words per node
static uint64_t gb_levels(uint64_t len, uint64_t* nodes) {
    uint64_t m = (len + kGbChunk - 1) / kGbChunk, L = 0;
    if (m == 0) m = 1;
    for (;;) {
        nodes[L++] = m;
        if (m == 1) break;
        m = (m + kGbFan - 1) / kGbFan;
    }
    return L;
}

uint64_t gb_decode_chunks(uint64_t len) { return len ? (len + kGbChunk - 1) / kGbChunk : 1; }

size_t gb_decode_ws_bytes(uint64_t len) {
    uint64_t nodes[16], L = gb_levels(len, nodes), words = 0;
    for (uint64_t l = 0; l < L; ++l) words += nodes[l] * (2 * kGbE + 2) + 2;
    return (size_t)(4 * words + 256 + nodes[0] * (2 * kGbE * 32) + 16);
}

cudaError_t launch_gb_decode(const uint8_t* in, uint64_t len, uint64_t n, int delta, uint32_t base, uint32_t* out,
                             uint32_t* d_last, void* ws, uint64_t* lstatus, unsigned long long* status,
                             uint32_t epoch, cudaStream_t stream, int* launches) {
    uint64_t nodes[16];
    const uint64_t L = gb_levels(len, nodes);
    uint32_t* tc[16];  // per level: group counts of the 17 entries of every node
    uint32_t* tx[16];  // exits
    uint32_t* re[16];  // resolved entry offset of every node
    uint32_t* rc[16];  // resolved index of its first group
    uint32_t* w = static_cast<uint32_t*>(ws);
    for (uint64_t l = 0; l < L; ++l) {
        const uint64_t m = nodes[l];
        tc[l] = w, w += m * kGbE;
        tx[l] = w, w += m * kGbE;
        re[l] = w, w += m + 1;
        rc[l] = w, w += m + 1;
    }
    const uint64_t nchunks = nodes[0];
    uint16_t* segtab = reinterpret_cast<uint16_t*>((reinterpret_cast<uintptr_t>(w) + 15) & ~(uintptr_t)15);
    const unsigned tgrid = (unsigned)((nchunks + kGbWarps - 1) / kGbWarps);
    cudaError_t e = gb_launch(gb_table_kernel, tgrid, 32 * kGbWarps, stream, in, len, nchunks, tc[0], tx[0], segtab);
    if (e != cudaSuccess) return e;
    int nl = 1;
    const uint32_t* nul = nullptr;
    for (uint64_t l = 0; l + 1 < L; ++l, ++nl) {
        e = gb_launch(gb_compose_kernel, (unsigned)((nodes[l + 1] + kGbTreeWarps - 1) / kGbTreeWarps),
                      32 * kGbTreeWarps, stream, (const uint32_t*)tc[l], (const uint32_t*)tx[l], nodes[l], tc[l + 1],
                      tx[l + 1], nodes[l + 1]);
        if (e != cudaSuccess) return e;
    }
    const uint64_t ngroups = (n + 3) >> 2;
    // root: the top level's single node, entered at 0
    e = gb_launch(gb_expand_kernel, 1u, 32 * kGbTreeWarps, stream, (const uint32_t*)tc[L - 1],
                  (const uint32_t*)tx[L - 1], (uint64_t)1, nul, nul, (uint64_t)1, re[L - 1], rc[L - 1], 1, ngroups,
                  status, epoch);
    if (e != cudaSuccess) return e;
    ++nl;
    for (uint64_t l = L - 1; l > 0; --l, ++nl) {
        e = gb_launch(gb_expand_kernel, (unsigned)((nodes[l] + kGbTreeWarps - 1) / kGbTreeWarps), 32 * kGbTreeWarps,
                      stream, (const uint32_t*)tc[l - 1], (const uint32_t*)tx[l - 1], nodes[l - 1],
                      (const uint32_t*)re[l], (const uint32_t*)rc[l], nodes[l], re[l - 1], rc[l - 1], 0, ngroups,
                      status, epoch);
        if (e != cudaSuccess) return e;
    }
    if (delta)
        e = gb_launch(gb_decode_kernel<true>, tgrid, 32 * kGbWarps, stream, in, len, n, nchunks,
                      (const uint32_t*)re[0], (const uint32_t*)rc[0], (const uint16_t*)segtab, base, lstatus, out,
                      d_last, status, epoch);
    else
        e = gb_launch(gb_decode_kernel<false>, tgrid, 32 * kGbWarps, stream, in, len, n, nchunks,
                      (const uint32_t*)re[0], (const uint32_t*)rc[0], (const uint16_t*)segtab, base,
                      (uint64_t*)nullptr, out, d_last, status, epoch);
    if (e != cudaSuccess) return e;
    *launches = nl + 1;
    return cudaGetLastError();
}

cudaError_t launch_gb_encode(const uint32_t* in, uint64_t n, int delta, uint32_t prev, uint8_t* out,
                             uint64_t* d_out_len, void* meta_ws, unsigned long long* status, uint32_t epoch,
                             cudaStream_t stream, int* launches) {
    cudaError_t e = launch_size_scan(in, n, delta, prev, meta_ws, d_out_len, status, epoch, stream);
    if (e != cudaSuccess) return e;
    const DecodeMeta m = carve_decode_meta(meta_ws, n);
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const unsigned grid = (unsigned)((nsub + kGbEncWarps - 1) / kGbEncWarps);
    if (delta)
        gb_encode_kernel<true><<<grid, 256, 0, stream>>>(in, n, prev, out, m);
    else
        gb_encode_kernel<false><<<grid, 256, 0, stream>>>(in, n, prev, out, m);
    *launches = 2;
    return cudaGetLastError();
}

}  // namespace bcgpu
