// svb_pack.cuh -- branch-free group pack for the Stream VByte encoders (sm_100a).
//
// A group is 4 integers x0..x3 and its control byte c (field i = byte_length(x_i) - 1,
// codec.hpp:70-72).  Its data is x0[0:l0] x1[0:l1] x2[0:l2] x3[0:l3],
// 4..16 bytes (the low bytes, little-endian).  Every x_i is zero above its length, so
// concatenation is shift + OR, no masking:
//   A = x0 | x1 << 8 l0 (<= 8 bytes, two words), B = x2 | x3 << 8 l2, G = A | B << 8 (l0 + l1)
// G (<= 16 bytes, four words) is then shifted onto the shared-memory word grid at the
// group's byte address and stored as whole words.  Adjacent groups of a row belong to
// adjacent lanes, so the one word two groups share is passed up one lane by a shuffle and
// OR-ed in: every word is written once, by one lane, with predicated stores (no branches).
//
// Pipe budget (B200): integer ops run on the ALU pipe (IADD3/LOP3/SHF/PRMT/SEL) and the
// FMA pipe (IMAD), each 1 warp instruction per 2 cycles per SM sub-partition, so the pack
// is written for few ALU ops: ~55 per group against ~150 with the earlier branchy pack
// (ncu, cfg3 one-pass encode: 63 executed instructions per integer).
#pragma once

#include <cstdint>
#include <type_traits>

#include "svb_device.cuh"
#include "svb_fast.cuh"
#include "svb_tma.cuh"

namespace bcgpu {

__device__ __forceinline__ uint32_t shfl_l(uint32_t lo, uint32_t hi, uint32_t s) {  // (hi:lo << s) >> 32, s < 32
    return __funnelshift_l(lo, hi, s);
}

// byte_length - 1 of the four integers -> control byte (field i in bits 2i..2i+1);
// tot = the group's data bytes
__device__ __forceinline__ uint32_t group_ctrl(const uint4& x, uint32_t& tot) {
    // top-bit indices (7..31) packed one per byte, then one shift + mask gives the four
    // byte_length - 1 fields M (instead of a shift per integer); one multiply gathers them into
    // the control byte: field i sits at bit 8 i of M and lands at bit 24 + 2 i of M * K,
    // K = 2^24 + 2^18 + 2^12 + 2^6 (the other partial products fall below bit 24 or leave the
    // word, and none overlap)
    const uint32_t f0 = bfind_u32(x.x | 0x80u), f1 = bfind_u32(x.y | 0x80u), f2 = bfind_u32(x.z | 0x80u),
                   f3 = bfind_u32(x.w | 0x80u);
    const uint32_t M = ((f0 + (f1 << 8) + (f2 << 16) + (f3 << 24)) >> 3) & 0x03030303u;
    tot = __dp4a(M, 0x01010101u, 4u);
    return (M * 0x01041040u) >> 24;
}

// data bytes of a control byte: 4 + the sum of its fields (length[c])
__device__ __forceinline__ uint32_t ctrl_bytes(uint32_t c) {
    return (c & 3u) + ((c >> 2) & 3u) + ((c >> 4) & 3u) + (c >> 6) + 4u;
}

// The group's data as four little-endian words G0..G3 (bytes past its length are zero).
// e8 = 8 * the group's data bytes.
__device__ __forceinline__ uint4 group_bytes(const uint4& x, uint32_t c, uint32_t& e8) {
    // byte_length - 1 of the four integers one per byte (the even and the odd fields spread by
    // one multiply each: no partial products overlap inside a field's byte), then one multiply
    // gives the running bit offsets: bytes of P8 = 8 l0, 8 (l0 + l1), 8 (l0 + l1 + l2), 8 total
    const uint32_t Lm = ((c & 0x33u) * 0x1001u + (c & 0xCCu) * 0x40040u) & 0x03030303u;
    const uint32_t P8 = Lm * 0x08080808u + 0x20181008u;
    const uint32_t sA = P8 & 0xFFu;                              // 8 l0, 8..32
    const uint32_t sB = __byte_perm(Lm, 0u, 0x4442u) * 8u + 8u;   // 8 l2
    const uint32_t la8 = __byte_perm(P8, 0u, 0x4441u);           // 8 (l0 + l1), 16..64
    e8 = P8 >> 24;
    const uint32_t A0 = x.x + __funnelshift_lc(0u, x.y, sA);  // x1 << 8 l0 (0 when l0 = 4)
    const uint32_t A1 = __funnelshift_lc(x.y, 0u, sA);        // x1 >> (32 - 8 l0)
    const uint32_t B0 = x.z + __funnelshift_lc(0u, x.w, sB);
    const uint32_t B1 = __funnelshift_lc(x.w, 0u, sB);
    // B << 8 (l0 + l1) over four words, la8 = 16..64: one 64-bit shift left for words 0-1 and
    // one right (by 64 - la8) for words 2-3.  PTX shifts clamp at 64, and each 64-bit shift is
    // two SHF (no word selects: the 32-bit form needed a compare, a subtract and five selects)
    uint64_t Bq, L, H;
    asm("mov.b64 %0, {%1, %2};" : "=l"(Bq) : "r"(B0), "r"(B1));
    asm("shl.b64 %0, %1, %2;" : "=l"(L) : "l"(Bq), "r"(la8));
    asm("shr.b64 %0, %1, %2;" : "=l"(H) : "l"(Bq), "r"(64u - la8));
    uint32_t L0, L1;
    uint4 G;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(L0), "=r"(L1) : "l"(L));
    asm("mov.b64 {%0, %1}, %2;" : "=r"(G.z), "=r"(G.w) : "l"(H));
    G.x = A0 + L0;
    G.y = A1 + L1;
    return G;
}

// Pack one group of each lane of a row at shared byte address a (groups of consecutive
// lanes are consecutive in the stream: a_{l+1} = a_l + ctrl_bytes(c_l)).  carry: the
// pending (partially filled) word after the previous row's last group, in and out; the
// caller stores it after the last row (lane 0 holds it; other lanes' values are not meaningful).
// Every lane of the warp must call this.
__device__ __forceinline__ void pack_group_row(const uint4& x, uint32_t c, uint32_t a, uint32_t& carry) {
    const int lane = threadIdx.x & 31;
    uint32_t e8;
    const uint4 G = group_bytes(x, c, e8);
    const uint32_t u = (a & 3u) << 3;
    const uint32_t W0 = G.x << u, W1 = shfl_l(G.x, G.y, u), W2 = shfl_l(G.y, G.z, u), W3 = shfl_l(G.z, G.w, u),
                   W4 = shfl_l(G.w, 0u, u);
    e8 += u;  // 8 e, e = 4..19: words [a & ~3, +e) are touched
    const bool p1 = e8 >= 64u, p2 = e8 >= 96u, p3 = e8 >= 128u;
    // the word the next group shares (all zero when this group ends on a word boundary)
    const uint32_t pend = p3 ? W4 : p2 ? W3 : p1 ? W2 : W1;
    // one rotation: lanes 1..31 take their left neighbour's pending word, lane 0 takes lane
    // 31's, which is what it needs for the NEXT row (carry is only meaningful in lane 0)
    const uint32_t rot = __shfl_sync(kFull, pend, (lane + 31) & 31);
    const uint32_t pin = lane == 0 ? carry : rot;
    carry = rot;
    const uint32_t wa = a & ~3u;
    sts32(wa, W0 + pin);
    sts32_if(wa + 4, W1, p1);
    sts32_if(wa + 8, W2, p2);
    sts32_if(wa + 12, W3, p3);
}

// 16 bytes at word phase Q (0..3) and bit phase r of the 32 aligned bytes lo:hi
template <int Q>
__device__ __forceinline__ uint4 realign_pick(const uint4& lo, const uint4& hi, uint32_t r) {
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    return make_uint4(__funnelshift_r(w[Q], w[Q + 1], r), __funnelshift_r(w[Q + 1], w[Q + 2], r),
                      __funnelshift_r(w[Q + 2], w[Q + 3], r), __funnelshift_r(w[Q + 3], w[Q + 4], r));
}

// Packed bytes [src, src + len) of shared memory (>= 32 readable bytes after the end) -> global
// dst at any alignment.  Interior 16-B granules of the destination are
// funnel-shifted out of five shared words each and stored with 128-bit stores; the < 16
// bytes before the first and after the last aligned granule are single-byte stores of one
// lane each.
__device__ __forceinline__ void store_realigned2(uint32_t src, uint32_t len, uint8_t* dst) {
    const int lane = threadIdx.x & 31;
    if (len == 0) return;
    const uintptr_t D = (uintptr_t)dst, Dend = D + len;
    const uintptr_t A0 = (D + 15) & ~(uintptr_t)15, A1 = Dend & ~(uintptr_t)15;
    const uint32_t head = (uint32_t)((A0 < Dend ? A0 : Dend) - D);  // bytes before the first aligned granule
    // interior granules [A0, A1): destination byte a comes from src + (a - D)
    if (A1 > A0) {
        // source granule k = bytes [s0 + 16 k, +16): two 128-bit loads of the aligned 32 bytes
        // around it (consecutive lanes read consecutive chunks: no bank conflicts, where five
        // word loads 16 B apart were 4-way conflicted), then a funnel shift by the source's
        // 16-B phase, which is the same for every lane (a uniform switch, no selects)
        const uint32_t ng = (uint32_t)((A1 - A0) >> 4);
        const uint32_t s0 = src + head;                 // source of the first interior byte
        const uint32_t r = (s0 & 3u) << 3, q = (s0 >> 2) & 3u;
        const uint32_t c0 = s0 & ~15u;
        // the phase switch sits outside the loop and the loop handles two granules per lane
        // and trip, all four loads first (one granule per trip left every lane waiting out a
        // shared-memory round trip ~6 times per sub-tile)
        auto run = [&](auto qc) {
            constexpr int Q = decltype(qc)::value;
            uint32_t k = lane;
            for (; k + 32 < ng; k += 64) {
                const uint4 lo0 = lds128v(c0 + 16 * k), hi0 = lds128v(c0 + 16 * k + 16);
                const uint4 lo1 = lds128v(c0 + 16 * k + 512), hi1 = lds128v(c0 + 16 * k + 528);
                *reinterpret_cast<uint4*>(A0 + 16 * (uintptr_t)k) = realign_pick<Q>(lo0, hi0, r);
                *reinterpret_cast<uint4*>(A0 + 16 * (uintptr_t)k + 512) = realign_pick<Q>(lo1, hi1, r);
            }
            if (k < ng) {
                const uint4 lo = lds128v(c0 + 16 * k), hi = lds128v(c0 + 16 * k + 16);
                *reinterpret_cast<uint4*>(A0 + 16 * (uintptr_t)k) = realign_pick<Q>(lo, hi, r);
            }
        };
        switch (q) {
            case 0: run(std::integral_constant<int, 0>{}); break;
            case 1: run(std::integral_constant<int, 1>{}); break;
            case 2: run(std::integral_constant<int, 2>{}); break;
            default: run(std::integral_constant<int, 3>{}); break;
        }
    }
    if ((uint32_t)lane < head) dst[lane] = (uint8_t)lds8(src + lane);
    const uint32_t tail = A1 >= A0 ? (uint32_t)(Dend - A1) : 0u;  // bytes after the last aligned granule
    if ((uint32_t)lane < tail) {
        const uint32_t o = (uint32_t)(A1 - D) + lane;
        dst[o] = (uint8_t)lds8(src + o);
    }
}

// pack_group_row for a row that may end early: tot = the group's real data bytes (0 for a lane
// past the last group; a last group of cnt < 4 integers has zero integers -- control fields 0
// -- in its unused places, whose bytes are left out), w0 = whether this lane stores its first
// word: every group lane, and the one lane right after the last group, which stores the last
// group's pending word (its own W0 is 0).  Lanes further on store nothing.
__device__ __forceinline__ void pack_group_row_masked(const uint4& x, uint32_t c, uint32_t a, uint32_t& carry,
                                                      uint32_t tot, bool w0) {
    const int lane = threadIdx.x & 31;
    uint32_t e8;
    const uint4 G = group_bytes(x, c, e8);
    const uint32_t u = (a & 3u) << 3;
    const uint32_t W0 = G.x << u, W1 = shfl_l(G.x, G.y, u), W2 = shfl_l(G.y, G.z, u), W3 = shfl_l(G.z, G.w, u),
                   W4 = shfl_l(G.w, 0u, u);
    e8 = 8u * tot + u;
    // a group of < 4 bytes (the last, partial group; tot = 0 past it) may end inside its first
    // word: that word is then its pending one, merged with the word it received, and the next
    // lane needs the merged value -- a second shuffle (such groups are never adjacent)
    const bool p0 = e8 >= 32u, p1 = e8 >= 64u, p2 = e8 >= 96u, p3 = e8 >= 128u;
    const uint32_t pend0 = p3 ? W4 : p2 ? W3 : p1 ? W2 : W1;
    uint32_t pin = __shfl_up_sync(kFull, pend0, 1);
    if (lane == 0) pin = carry;
    const uint32_t pend = p0 ? pend0 : (W0 | pin);
    uint32_t pin2 = __shfl_up_sync(kFull, pend, 1);
    if (lane == 0) pin2 = carry;
    carry = __shfl_sync(kFull, pend, 31);
    const uint32_t wa = a & ~3u;
    sts32_if(wa, W0 | pin2, w0 && (p0 || tot == 0u));
    sts32_if(wa + 4, W1, p1);
    sts32_if(wa + 8, W2, p2);
    sts32_if(wa + 12, W3, p3);
}

// Packed bytes at shared sdst (sdst has dst's 16-B phase), len bytes -> global dst: one bulk
// copy of the 16-B aligned interior (lane 0 issues and commits it; the caller waits for its
// smem read before reusing the buffer), lanes store the < 16 edge bytes at each end.  Every
// lane must have fenced its shared writes for the async proxy and synced the warp first.
__device__ __forceinline__ void put_packed(uint8_t* dst, uint32_t sdst, uint32_t len) {
    const int lane = threadIdx.x & 31;
    const uintptr_t gb = (uintptr_t)dst, ge = gb + len;
    const uintptr_t a_lo = (gb + 15) & ~(uintptr_t)15, a_hi = ge & ~(uintptr_t)15;
    if (a_hi > a_lo) {
        if (lane == 0) {
            tma_store_s(reinterpret_cast<void*>(a_lo), sdst + (uint32_t)(a_lo - gb), (uint32_t)(a_hi - a_lo));
            tma_store_commit();
        }
        const uint32_t nh = (uint32_t)(a_lo - gb), nt = (uint32_t)(ge - a_hi);
        if ((uint32_t)lane < nh) dst[lane] = (uint8_t)lds8(sdst + lane);
        if ((uint32_t)lane < nt) dst[(a_hi - gb) + lane] = (uint8_t)lds8(sdst + (uint32_t)(a_hi - gb) + lane);
    } else {
        for (uint32_t i = lane; i < len; i += 32) dst[i] = (uint8_t)lds8(sdst + i);
    }
}

// ---- full sub-tiles (1024 integers, row j lane l = group 32 j + l) -----------------
// Pass 1: control bytes (stored straight to the stream: byte 32 j + l of cdst, any
// alignment, 32 consecutive bytes per row), the lane's control bytes kept in cw (row j in
// byte j & 3 of cw[j >> 2]) and the rows' packed exclusive offsets in qw; returns the
// sub-tile's data size.
// early(total) is called with the sub-tile's data size as soon as it is known (one warp
// reduction), before the row scan: the one-pass encode posts it there, which takes the scan's
// five dependent shuffle steps off the path every other CTA's look-back waits on.
template <bool kDelta, bool kAny = false, int kRows = kWTRows, class Early>
__device__ __forceinline__ uint32_t enc_lengths2(uint32_t sin, uint32_t prev_w, uint8_t* __restrict__ cdst,
                                                 uint32_t (&cw)[2], uint32_t (&qw)[4], Early early) {
    const int lane = threadIdx.x & 31;
    uint32_t P[3] = {0, 0, 0};
    uint32_t last = prev_w, lt = 0;
    cw[0] = cw[1] = 0;
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
        const uint4 x = enc_row<kDelta, kAny>(sin, j, last);
        uint32_t tot;
        const uint32_t c = group_ctrl(x, tot);
        cw[j >> 2] += c << (8 * (j & 3));
        P[j / 3] += tot << (10 * (j % 3));
        lt += tot;
        cdst[32 * j + lane] = (uint8_t)c;
    }
    early(__reduce_add_sync(kFull, lt));
    return packed_row_scan<kRows>(P, qw);
}

// Pass 2: pack every row in place at shared byte sdst (sdst <= sin, 4-B aligned so that a
// row's completed words end before the next row's integers), then the final pending word.
template <bool kDelta, bool kAny = false, int kRows = kWTRows>
__device__ __forceinline__ void enc_pack2(uint32_t sin, uint32_t prev_w, const uint32_t (&cw)[2],
                                          const uint32_t (&qw)[4], uint32_t sdst, uint32_t total) {
    uint32_t last = prev_w, carry = 0;
    // rows in pairs: both rows are read before either is written (row j + 1's output ends
    // before row j + 2's integers), so the two packs' dependency chains interleave
#pragma unroll
    for (int j = 0; j + 1 < kRows; j += 2) {
        const uint4 x0 = enc_row<kDelta, kAny>(sin, j, last);
        const uint4 x1 = enc_row<kDelta, kAny>(sin, j + 1, last);
        const uint32_t c0 = (cw[j >> 2] >> (8 * (j & 3))) & 0xFFu, c1 = (cw[j >> 2] >> (8 * (j & 3) + 8)) & 0xFFu;
        const uint32_t a0 = sdst + (qw[j >> 1] & 0xFFFFu), a1 = sdst + (qw[j >> 1] >> 16);
        __syncwarp();  // every lane has read both rows before any lane writes over them
        pack_group_row(x0, c0, a0, carry);
        pack_group_row(x1, c1, a1, carry);
    }
    if constexpr (kRows & 1) {  // an odd last row
        constexpr int j = kRows - 1;
        const uint4 x0 = enc_row<kDelta, kAny>(sin, j, last);
        const uint32_t c0 = (cw[j >> 2] >> (8 * (j & 3))) & 0xFFu;
        const uint32_t a0 = sdst + (qw[j >> 1] & 0xFFFFu);
        __syncwarp();
        pack_group_row(x0, c0, a0, carry);
    }
    if (((sdst + total) & 3u) && (threadIdx.x & 31) == 0) sts32((sdst + total) & ~3u, carry);
}

}  // namespace bcgpu
