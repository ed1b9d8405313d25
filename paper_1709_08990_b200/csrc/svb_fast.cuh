// svb_fast.cuh -- lean inner loops for full sub-tiles (every sub-tile but the
// stream's last): 32-bit shared-memory addressing, no per-lane bounds or tail
// logic, row-major 128-bit I/O.  The general paths in svb_warp.cuh remain for
// the final, partial sub-tile.
#pragma once

#include "svb_device.cuh"
#include "svb_warp.cuh"

namespace bcgpu {

__device__ __forceinline__ uint32_t sh_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Shared loads by address are volatile asm: the compiler must not move them above the
// mbarrier waits (or the volatile shared stores) they follow -- as plain asm with no memory
// operand they count as pure functions of the address and may be hoisted (it happened, in
// an unrolled loop over TMA-staged chunks).  ptxas still schedules the SASS freely.
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
// ordered against the surrounding shared stores (in-place passes)
__device__ __forceinline__ uint4 lds128v(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, const uint4& v) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// predicated shared store (no branch around it)
__device__ __forceinline__ void sts32_if(uint32_t a, uint32_t v, bool pred) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.shared.u32 [%0], %1;\n\t}" ::"r"(a), "r"(v),
                 "r"((uint32_t)pred)
                 : "memory");
}

// Control bytes of a full sub-tile at shared address sc (row j, lane l <-> byte 32j + l).
// Sets *all_zero (warp-uniform) and skips the offset scan when every control byte is 0:
// then integer i of the sub-tile is data byte i.
__device__ __forceinline__ WarpCtrl ctrl_full(uint32_t sc, bool* all_zero) {
    const int lane = threadIdx.x & 31;
    WarpCtrl w;
    w.cw[0] = w.cw[1] = 0;
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) w.cw[j >> 2] |= lds8(sc + 32 * j + lane) << (8 * (j & 3));
    *all_zero = __all_sync(kFull, (w.cw[0] | w.cw[1]) == 0);
    if (*all_zero) {
        w.total = kWTInts;
        return w;
    }
    uint32_t P[3] = {0, 0, 0};
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint32_t c = (w.cw[j >> 2] >> (8 * (j & 3))) & 0xFFu;
        P[j / 3] |= (fsum(c) + 4u) << (10 * (j % 3));
    }
    w.total = packed_row_scan(P, w.qw);
    return w;
}

// integer of l bytes at shared byte address a
__device__ __forceinline__ uint32_t extract_s(uint32_t a, uint32_t l) {
    const uint32_t w = a & ~3u;
    const uint32_t x = __funnelshift_r(lds32(w), lds32(w + 4), (a & 3u) << 3);
    return x & (0xFFFFFFFFu >> ((4u - l) << 3));
}

// one control byte c whose data starts at shared byte address a
__device__ __forceinline__ uint4 group_s(uint32_t a, uint32_t c) {
    const uint32_t l0 = (c & 3u) + 1u, l1 = ((c >> 2) & 3u) + 1u, l2 = ((c >> 4) & 3u) + 1u, l3 = (c >> 6) + 1u;
    uint4 v;
    v.x = extract_s(a, l0);
    a += l0;
    v.y = extract_s(a, l1);
    a += l1;
    v.z = extract_s(a, l2);
    a += l2;
    v.w = extract_s(a, l3);
    return v;
}

// control byte 0: four 1-byte integers
__device__ __forceinline__ uint4 zero_group_s(uint32_t a) {
    const uint32_t w = a & ~3u;
    const uint32_t x = __funnelshift_r(lds32(w), lds32(w + 4), (a & 3u) << 3);
    return make_uint4(__byte_perm(x, 0u, 0x4440), __byte_perm(x, 0u, 0x4441), __byte_perm(x, 0u, 0x4442),
                      __byte_perm(x, 0u, 0x4443));
}

__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}

// true when all 256 control bytes of the sub-tile at shared address sc are 0 (warp-uniform)
__device__ __forceinline__ bool ctrl_all_zero(uint32_t sc) {
    const uint2 c = lds64(sc + 8 * (threadIdx.x & 31));
    return __all_sync(kFull, (c.x | c.y) == 0);
}

// dp4a byte selector for bytes [0, k) of a word, k in [0, 4]
__device__ __forceinline__ uint32_t ones_below(int k) {
    return k >= 4 ? 0x01010101u : (k <= 0 ? 0u : (0x01010101u & ((1u << (8 * k)) - 1u)));
}

// Per-lane part of the byte sum of the 1024 shared bytes at sd (any alignment): the sum of
// a sub-tile's integers when every control byte is 0 (callers reduce over the warp).  Lane l
// reads 16-B chunks l, l+32; reads up to 16 bytes past the sub-tile when sd is unaligned.
__device__ __forceinline__ uint32_t zero_tile_sum(uint32_t sd) {
    const int lane = threadIdx.x & 31;
    const uint32_t a0 = sd & ~15u;
    const int s = (int)(sd & 15u);
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const uint4 v = lds128(a0 + 16u * (lane + 32 * i));
        acc = __dp4a(v.x, 0x01010101u, acc);
        acc = __dp4a(v.y, 0x01010101u, acc);
        acc = __dp4a(v.z, 0x01010101u, acc);
        acc = __dp4a(v.w, 0x01010101u, acc);
    }
    if (s) {  // chunk 0's first s bytes precede the sub-tile, chunk 64's belong to it: lanes 0-3 fix word `lane`
        const uint32_t sel = lane < 4 ? ones_below(s - 4 * lane) : 0u;
        const uint32_t wa = a0 + 4u * (uint32_t)(lane & 3);
        acc = __dp4a(lds32(wa + 1024u), sel, acc) - __dp4a(lds32(wa), sel, 0u);
    }
    return acc;
}

__device__ __forceinline__ uint32_t byte_sum4_fast(uint32_t w) {
    const uint32_t s = (w & 0x00FF00FFu) + ((w >> 8) & 0x00FF00FFu);
    return (s & 0xFFFFu) + (s >> 16);
}

// kMode: 0 plain store, 1 delta store (run = value before the sub-tile), 2 sum only.
// sd = shared address of the sub-tile's first data byte; o = the sub-tile's first output
// integer (16-B aligned: callers take the general path otherwise).  kZero: every control
// byte of the sub-tile is 0, so row j lane l's four 1-byte integers are data bytes 128j+4l..+3.
template <int kMode, bool kZero>
__device__ __forceinline__ uint32_t expand_full(const WarpCtrl& w, uint32_t sd, uint32_t* __restrict__ o, uint32_t run) {
    const int lane = threadIdx.x & 31;
    uint32_t acc = 0;
    if constexpr (kMode == 1 && kZero) {
        // every integer is one byte: a row's group sums (<= 1020) and totals (<= 32640) fit
        // 16 bits, so two rows share one warp scan
        const uint64_t pol = l2_policy_drop();
#pragma unroll
        for (int j = 0; j < kWTRows; j += 2) {
            uint4 v0 = zero_group_s(sd + 128 * j + 4 * lane), v1 = zero_group_s(sd + 128 * (j + 1) + 4 * lane);
            v0.y += v0.x;
            v0.z += v0.y;
            v0.w += v0.z;
            v1.y += v1.x;
            v1.z += v1.y;
            v1.w += v1.z;
            const uint32_t Pk = v0.w | (v1.w << 16);
            const uint32_t I = warp_inclusive_scan(Pk);
            const uint32_t T = __shfl_sync(kFull, I, 31);
            const uint32_t a0 = run + (I & 0xFFFFu) - v0.w;
            const uint32_t a1 = run + (T & 0xFFFFu) + (I >> 16) - v1.w;
            stg_hint_v4(o + 128 * j + 4 * lane, add4(v0, a0), pol);
            stg_hint_v4(o + 128 * (j + 1) + 4 * lane, add4(v1, a1), pol);
            run += (T & 0xFFFFu) + (T >> 16);
        }
        return run;
    }
    const uint64_t pol1 = l2_policy_drop();
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        uint32_t c = 0, a;
        bool allzero = true;
        if constexpr (kZero) {
            a = sd + 128 * j + 4 * lane;
        } else {
            c = row_ctrl(w, j);
            a = sd + row_q(w, j);
            allzero = __all_sync(kFull, c == 0);
        }
        if constexpr (kMode == 2) {
            if (allzero) {
                const uint32_t wa = a & ~3u;
                acc += byte_sum4_fast(__funnelshift_r(lds32(wa), lds32(wa + 4), (a & 3u) << 3));
            } else {
                const uint4 v = group_s(a, c);
                acc += v.x + v.y + v.z + v.w;
            }
        } else {
            uint4 v = allzero ? zero_group_s(a) : group_s(a, c);
            if constexpr (kMode == 1) {
                v.y += v.x;
                v.z += v.y;
                v.w += v.z;
                const uint32_t I = warp_inclusive_scan(v.w);
                const uint32_t add = run + I - v.w;
                v.x += add;
                v.y += add;
                v.z += add;
                v.w += add;
                run += __shfl_sync(kFull, I, 31);
            }
            if constexpr (kMode == 1)
                stg_hint_v4(o + 128 * j + 4 * lane, v, pol1);  // evict-first: keep L2 for the compressed input
            else
                stg_stream_v4(o + 128 * j + 4 * lane, v);
        }
    }
    return kMode == 2 ? acc : run;
}


// ---- any tile (batches): partial tiles, any output alignment ------------------
// ng groups (1..256) with `tail` integers (1..4) in the last one, control in w (the tail's
// unused fields already masked), data at shared address sd, output o at any 4-B alignment.
// Group g of row j goes to elements 4(32j + lane) ..; a lane stores the 16-B aligned
// granule holding elements [4g - r, 4g - r + 4) (r = o's 4-B phase inside 16 B): the
// previous lane's last r integers (shuffled up; lane 0 keeps the previous row's lane 31)
// and its own first 4 - r.  Whole granules leave as 128-bit stores, the tile's first and
// last partial granules as scalars.  Returns the running value (delta) after the tile.
template <bool kDelta>
__device__ __forceinline__ uint32_t expand_any(const WarpCtrl& w, uint32_t sd, uint32_t ng, uint32_t tail,
                                               uint32_t* __restrict__ o, uint32_t run) {
    const int lane = threadIdx.x & 31;
    const int nints = (int)(4 * (ng - 1) + tail);
    const uint32_t r = (uint32_t)(((uintptr_t)o >> 2) & 3u);
    uint32_t* A = o - r;
    uint4 carry = make_uint4(0, 0, 0, 0);
    const uint32_t rows = (ng + 31) >> 5;
#pragma unroll 1
    for (uint32_t j = 0; j < rows; ++j) {
        const uint32_t gl = 32 * j + lane;
        const uint32_t cnt = gl + 1 < ng ? 4u : (gl + 1 == ng ? tail : 0u);
        const uint32_t c = row_ctrl(w, (int)j);
        const uint32_t a = sd + row_q(w, (int)j);
        uint4 v = __all_sync(kFull, c == 0) ? zero_group_s(a) : group_s(a, c);
        v = mask_tail(v, cnt);
        if constexpr (kDelta) {
            v.y += v.x;
            v.z += v.y;
            v.w += v.z;
            const uint32_t I = warp_inclusive_scan(v.w);
            v = add4(v, run + I - v.w);
            run += __shfl_sync(kFull, I, 31);
        }
        if (r == 0) {
            if (cnt == 4)
                stg_stream_v4(o + 4 * gl, v);
            else if (cnt)
                store_group(o + 4 * gl, v, cnt, false);
        } else {
            uint4 prv = make_uint4(__shfl_up_sync(kFull, v.x, 1), __shfl_up_sync(kFull, v.y, 1),
                                   __shfl_up_sync(kFull, v.z, 1), __shfl_up_sync(kFull, v.w, 1));
            if (lane == 0) prv = carry;
            carry = make_uint4(__shfl_sync(kFull, v.x, 31), __shfl_sync(kFull, v.y, 31), __shfl_sync(kFull, v.z, 31),
                               __shfl_sync(kFull, v.w, 31));
            const uint4 g = r == 1 ? make_uint4(prv.w, v.x, v.y, v.z)
                          : r == 2 ? make_uint4(prv.z, prv.w, v.x, v.y)
                                   : make_uint4(prv.y, prv.z, prv.w, v.x);
            const int e0 = 4 * (int)gl - (int)r;
            if (e0 >= 0 && e0 + 4 <= nints) {
                stg_stream_v4(A + 4 * gl, g);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (e0 + i >= 0 && e0 + i < nints) A[4 * gl + i] = comp(g, i);
            }
        }
    }
    if (r && lane < (int)r) {  // the last row's final r integers (lane 31's, in `carry`)
        const int e = 128 * (int)rows - (int)r + lane;
        if (e >= 0 && e < nints) o[e] = comp(carry, 4 - (int)r + lane);
    }
    return run;
}
}  // namespace bcgpu

namespace bcgpu {

// ---- encode, full sub-tiles --------------------------------------------------
__device__ __forceinline__ uint32_t blen(uint32_t x) { return 4u - (__clz(x | 1u) >> 3); }  // codec.hpp:70-72

__device__ __forceinline__ uint32_t bfind_u32(uint32_t x) {
    uint32_t r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
    return r;
}
// byte_length(x) - 1 (codec.hpp:70-72): the index of x's top byte, with x < 256 -> 0
__device__ __forceinline__ uint32_t blen_m1(uint32_t x) { return bfind_u32(x | 0x80u) >> 3; }

// Size scan of one full sub-tile at p (16-B aligned): sum over its 1024 integers of
// byte_length - 1, per lane (the sub-tile's data size is the warp sum + 1024).
// Delta: lane 0 holds x_{-1} in `last` and gets the sub-tile's last integer back.
template <bool kDelta>
__device__ __forceinline__ uint32_t size_full(const uint32_t* __restrict__ p, uint32_t& last) {
    const int lane = threadIdx.x & 31;
    uint4 x[kWTRows];
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) x[j] = ldg_stream_v4(p + 128 * j + 4 * lane);
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        uint4 v = x[j];
        if constexpr (kDelta) {
            // one rotation per row: lane l gets lane l-1's last integer; lane 0 gets
            // lane 31's, which is the predecessor of the next row's lane 0
            const uint32_t r = __shfl_sync(kFull, v.w, (lane + 31) & 31);
            const uint32_t q = lane == 0 ? last : r;
            last = r;
            v = make_uint4(v.x - q, v.y - v.x, v.z - v.y, v.w - v.z);
        }
        acc += blen_m1(v.x) + blen_m1(v.y) + blen_m1(v.z) + blen_m1(v.w);
    }
    return acc;
}

// Row j of the sub-tile (integers at shared address sin + 512 j + 16 lane), as
// values or mod-2^32 deltas; `last` carries x_{-1} in and the row's last raw value out.
__device__ __forceinline__ uint32_t lds32v(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}

// kAny: sin is only 4-B aligned (segments of a batch start at any element)
template <bool kDelta, bool kAny = false>
__device__ __forceinline__ uint4 enc_row(uint32_t sin, int j, uint32_t& last) {
    const int lane = threadIdx.x & 31;
    const uint32_t a = sin + 512 * j + 16 * lane;
    uint4 x;
    if (kAny && (sin & 15u))
        x = make_uint4(lds32v(a), lds32v(a + 4), lds32v(a + 8), lds32v(a + 12));
    else
        x = lds128v(a);
    if constexpr (kDelta) {
        uint32_t p = __shfl_up_sync(kFull, x.w, 1);
        if (lane == 0) p = last;
        last = __shfl_sync(kFull, x.w, 31);
        x = make_uint4(x.x - p, x.y - x.x, x.z - x.y, x.w - x.z);
    }
    return x;
}

__device__ __forceinline__ uint32_t lens_of_ctrl(uint32_t c) {  // l_i = field_i + 1, one per byte
    const uint32_t t = c | (c << 6);  // OR, not a multiply: the shifted copies overlap
    return ((t | (t << 12)) & 0x03030303u) + 0x01010101u;
}

// Pass 1: byte lengths, control bytes (-> shared sctrl), tile-local offsets; returns the data size.
template <bool kDelta, bool kAny = false>
__device__ __forceinline__ uint32_t enc_full_lengths(uint32_t sin, uint32_t prev_w, uint32_t sctrl,
                                                     uint32_t (&lens)[kWTRows], uint32_t (&qw)[4]) {
    const int lane = threadIdx.x & 31;
    uint32_t P[3] = {0, 0, 0};
    uint32_t last = prev_w;
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint4 x = enc_row<kDelta, kAny>(sin, j, last);
        const uint32_t c = blen_m1(x.x) | (blen_m1(x.y) << 2) | (blen_m1(x.z) << 4) | (blen_m1(x.w) << 6);
        lens[j] = lens_of_ctrl(c);
        P[j / 3] |= __dp4a(lens[j], 0x01010101u, 0u) << (10 * (j % 3));
        sts8(sctrl + 32 * j + lane, c);
    }
    bool ones = true;
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) ones = ones && lens[j] == 0x01010101u;
    if (__all_sync(kFull, ones)) {  // every integer takes one byte: offsets are the identity
#pragma unroll
        for (int k = 0; k < 4; ++k) qw[k] = (256u * k + 4u * lane) | ((256u * k + 128u + 4u * lane) << 16);
        return kWTInts;
    }
    return packed_row_scan(P, qw);
}

// True when every integer (delta) of the full sub-tile at sin is < 256 (warp-uniform):
// then all control bytes are 0 and the data is the low byte of each integer.
template <bool kDelta, bool kAny = false>
__device__ __forceinline__ bool enc_full_small(uint32_t sin, uint32_t prev_w) {
    uint32_t last = prev_w, o = 0;
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint4 x = enc_row<kDelta, kAny>(sin, j, last);
        o |= x.x | x.y | x.z | x.w;
    }
    return __all_sync(kFull, o < 256u);
}

// Fused check + pack at phase 0 (the one-pass encode, whose destination phase is not
// known yet): every row is read once; if every integer (delta) is < 256 the low bytes
// are written as 32 aligned words per row over the consumed input (sdst = sin) and the
// function returns true; otherwise nothing is written.
// sdst: where the packed bytes go (16-B aligned, <= sin; sin itself when 16-B aligned).
template <bool kDelta, bool kAny = false>
__device__ __forceinline__ bool enc_full_small_pack0(uint32_t sin, uint32_t prev_w, uint32_t sdst) {
    const int lane = threadIdx.x & 31;
    uint32_t last = prev_w, o = 0;
    uint32_t P[kWTRows];
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint4 x = enc_row<kDelta, kAny>(sin, j, last);
        o |= x.x | x.y | x.z | x.w;
        P[j] = __byte_perm(__byte_perm(x.x, x.y, 0x0040), __byte_perm(x.z, x.w, 0x0040), 0x5410);
    }
    if (!__all_sync(kFull, o < 256u)) return false;
    __syncwarp();  // every lane has read every row
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) sts32(sdst + 128 * j + 4 * lane, P[j]);
    return true;
}

// Pack pass of a small sub-tile (enc_full_small): row j lane l's four bytes go to
// sdst + 128 j + 4 l.  In place, as enc_full_pack.
template <bool kDelta, bool kAny = false>
__device__ __forceinline__ void enc_small_pack(uint32_t sin, uint32_t prev_w, uint32_t sdst) {
    const int lane = threadIdx.x & 31;
    const uint32_t s = sdst & 3u;  // warp-uniform
    uint32_t last = prev_w;
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint4 x = enc_row<kDelta, kAny>(sin, j, last);
        const uint32_t P = __byte_perm(__byte_perm(x.x, x.y, 0x0040), __byte_perm(x.z, x.w, 0x0040), 0x5410);
        const uint32_t a = sdst + 128 * j + 4 * lane;
        __syncwarp();  // every lane has read row j before any lane writes over it
        if (s == 0) {
            sts32(a, P);
        } else {
            const uint32_t Pp = __shfl_up_sync(kFull, P, 1);
            if (lane > 0) sts32(a & ~3u, __funnelshift_r(Pp, P, 8u * (4u - s)));
            if (lane == 0)
                for (uint32_t b = 0; b < 4u - s; ++b) sts8(a + b, P >> (8 * b));
            if (lane == 31)
                for (uint32_t b = 4u - s; b < 4u; ++b) sts8(a + b, P >> (8 * b));
        }
    }
}

__device__ __forceinline__ void sts_int_bytes(uint32_t a, uint32_t x, uint32_t l) {
    sts8(a, x);
    if (l > 1) sts8(a + 1, x >> 8);
    if (l > 2) sts8(a + 2, x >> 16);
    if (l > 3) sts8(a + 3, x >> 24);
}

// Pass 2: pack in place; tile data byte 0 goes to shared address sdst (<= sin - 1 + ...; see caller).
template <bool kDelta, bool kAny = false>
__device__ __forceinline__ void enc_full_pack(uint32_t sin, uint32_t prev_w, const uint32_t (&lens)[kWTRows],
                                              const uint32_t (&qw)[4], uint32_t sdst) {
    const int lane = threadIdx.x & 31;
    uint32_t last = prev_w;
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint4 x = enc_row<kDelta, kAny>(sin, j, last);
        const uint32_t l = lens[j];
        const uint32_t a = sdst + ((qw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
        __syncwarp();  // every lane has read row j before any lane writes over it
        if (__all_sync(kFull, l == 0x01010101u)) {
            const uint32_t P = __byte_perm(__byte_perm(x.x, x.y, 0x0040), __byte_perm(x.z, x.w, 0x0040), 0x5410);
            const uint32_t Pp = __shfl_up_sync(kFull, P, 1);
            const uint32_t s = a & 3u;
            if (s == 0) {
                sts32(a, P);
            } else {
                if (lane > 0) sts32(a & ~3u, __funnelshift_r(Pp, P, 8u * (4u - s)));
                if (lane == 0)
                    for (uint32_t b = 0; b < 4u - s; ++b) sts8(a + b, P >> (8 * b));
                if (lane == 31)
                    for (uint32_t b = 4u - s; b < 4u; ++b) sts8(a + b, P >> (8 * b));
            }
        } else {
            const uint32_t l0 = l & 0xFFu, l1 = (l >> 8) & 0xFFu, l2 = (l >> 16) & 0xFFu, l3 = l >> 24;
            sts_int_bytes(a, x.x, l0);
            sts_int_bytes(a + l0, x.y, l1);
            sts_int_bytes(a + l0 + l1, x.z, l2);
            sts_int_bytes(a + l0 + l1 + l2, x.w, l3);
        }
    }
}

// Word-store pack of a full sub-tile (replaces the byte stores of enc_full_pack): each lane
// packs its group's <= 16 bytes into four registers (two 64-bit concatenations and one
// 128-bit one), shifts them onto the 4-B word grid and stores the words it completes; the
// word it shares with the next group travels to the next lane by one shuffle and is OR-ed
// into that lane's first word, so each shared word is written once, by one lane.  In place
// like enc_full_pack: a row's completed words end before the next row's integers, and the
// last lane's shared word is written while packing the next row.  The sub-tile's final
// shared word is written at the end.
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t s) { return __funnelshift_lc(0u, x, s); }
__device__ __forceinline__ uint32_t shr_clamp(uint32_t x, uint32_t s) { return __funnelshift_rc(x, 0u, s); }

// group x (byte lengths packed one per byte in L, tot = their sum) at shared byte o; returns
// the group's shared trailing word (pend) after storing the completed ones (pin = the
// previous group's pend)
__device__ __forceinline__ uint32_t pack_group_words(const uint4& x, uint32_t L, uint32_t o, uint32_t& carry) {
    const int lane = threadIdx.x & 31;
    const uint32_t l0 = L & 0xFFu, l1 = (L >> 8) & 0xFFu, l2 = (L >> 16) & 0xFFu;
    const uint32_t tot = __dp4a(L, 0x01010101u, 0u);
    const uint32_t Alo = x.x | shl_clamp(x.y, 8 * l0), Ahi = shr_clamp(x.y, 32 - 8 * l0);
    const uint32_t Blo = x.z | shl_clamp(x.w, 8 * l2), Bhi = shr_clamp(x.w, 32 - 8 * l2);
    const uint32_t t = 8 * (l0 + l1);
    const bool hi = t >= 32;
    const uint32_t tt = hi ? t - 32 : t;
    const uint32_t q0 = shl_clamp(Blo, tt), q1 = __funnelshift_lc(Blo, Bhi, tt), q2 = shr_clamp(Bhi, 32 - tt);
    const uint32_t P0 = Alo | (hi ? 0u : q0), P1 = Ahi | (hi ? q0 : q1), P2 = hi ? q1 : q2, P3 = hi ? q2 : 0u;
    const uint32_t u8 = (o & 3u) << 3;
    const uint32_t W0 = shl_clamp(P0, u8), W1 = __funnelshift_lc(P0, P1, u8), W2 = __funnelshift_lc(P1, P2, u8),
                   W3 = __funnelshift_lc(P2, P3, u8), W4 = __funnelshift_lc(P3, 0u, u8);
    const uint32_t nw = ((o & 3u) + tot) >> 2;  // >= 1: a full group has >= 4 bytes
    const uint32_t pend = nw == 1 ? W1 : nw == 2 ? W2 : nw == 3 ? W3 : W4;
    uint32_t pin = __shfl_up_sync(kFull, pend, 1);
    if (lane == 0) pin = carry;
    carry = __shfl_sync(kFull, pend, 31);
    const uint32_t wa = o & ~3u;
    sts32(wa, W0 | pin);
    sts32_if(wa + 4, W1, nw > 1);
    sts32_if(wa + 8, W2, nw > 2);
    sts32_if(wa + 12, W3, nw > 3);
    return pend;
}

template <bool kDelta, bool kAny = false>
__device__ __forceinline__ void enc_full_pack_w(uint32_t sin, uint32_t prev_w, const uint32_t (&lens)[kWTRows],
                                                const uint32_t (&qw)[4], uint32_t sdst, uint32_t total) {
    uint32_t last = prev_w, carry = 0;
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint4 x = enc_row<kDelta, kAny>(sin, j, last);
        const uint32_t o = sdst + ((qw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
        __syncwarp();  // every lane has read row j before any lane writes over it
        pack_group_words(x, lens[j], o, carry);
    }
    if (((sdst + total) & 3u) && (threadIdx.x & 31) == 0) sts32((sdst + total) & ~3u, carry);
}

// packed bytes [src, src + len) of shared memory (16-B aligned, with >= 16 readable bytes
// before and after) -> global dst (any alignment): destination granule k is the 16 source
// bytes at src + 16k - p, read as 5 words and funnel-shifted (p = dst's 16-B phase)
__device__ __forceinline__ void store_realigned(uint32_t src, uint32_t len, uint8_t* dst) {
    const int lane = threadIdx.x & 31;
    const uintptr_t D = (uintptr_t)dst;
    const uint32_t p = (uint32_t)(D & 15);
    const uintptr_t Dal = D - p, Dend = D + len;
    const uint32_t nout = (p + len + 15) >> 4;
    const uint32_t r = ((0u - p) & 3u) * 8u;
    for (uint32_t k = lane; k < nout; k += 32) {
        const uint32_t wa = (src + 16 * k - p) & ~3u;
        const uint32_t w0 = lds32v(wa), w1 = lds32v(wa + 4), w2 = lds32v(wa + 8), w3 = lds32v(wa + 12),
                       w4 = lds32v(wa + 16);
        {
            const uint4 v = make_uint4(__funnelshift_r(w0, w1, r), __funnelshift_r(w1, w2, r),
                                       __funnelshift_r(w2, w3, r), __funnelshift_r(w3, w4, r));
            const uintptr_t a = Dal + 16 * (uintptr_t)k;
            if (a >= D && a + 16 <= Dend) {
                *reinterpret_cast<uint4*>(a) = v;
            } else {
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int bi = 0; bi < 16; ++bi)
                    if (a + bi >= D && a + bi < Dend) *reinterpret_cast<uint8_t*>(a + bi) = (uint8_t)(w[bi >> 2] >> (8 * (bi & 3)));
            }
        }
    }
}

// ---- rolled variants (one row body in the binary) -----------------------------
// For kernels whose hot loop must stay small (the batch encode: several tile paths
// are live at once and the fully unrolled bodies overflow the instruction cache).
// Row j's packed lengths are rebuilt from its control byte, row offsets are picked
// from qw with selects: no per-row arrays, so nothing spills to local memory.
__device__ __forceinline__ uint32_t row_q_sel(const uint32_t (&qw)[4], int j) {
    const uint32_t w = (j >> 1) == 0 ? qw[0] : (j >> 1) == 1 ? qw[1] : (j >> 1) == 2 ? qw[2] : qw[3];
    return (w >> (16 * (j & 1))) & 0xFFFFu;
}

template <bool kDelta, bool kAny>
__device__ __forceinline__ uint32_t enc_full_lengths_r(uint32_t sin, uint32_t prev_w, uint32_t sctrl, uint32_t (&qw)[4]) {
    const int lane = threadIdx.x & 31;
    uint32_t P0 = 0, P1 = 0, P2 = 0;
    uint32_t last = prev_w;
#pragma unroll 1
    for (int j = 0; j < kWTRows; ++j) {
        const uint4 x = enc_row<kDelta, kAny>(sin, j, last);
        const uint32_t m0 = blen_m1(x.x), m1 = blen_m1(x.y), m2 = blen_m1(x.z), m3 = blen_m1(x.w);
        const uint32_t v = (m0 + m1 + m2 + m3 + 4u) << (10 * (j % 3));
        P0 |= j < 3 ? v : 0u;
        P1 |= (j >= 3 && j < 6) ? v : 0u;
        P2 |= j >= 6 ? v : 0u;
        sts8(sctrl + 32 * j + lane, m0 | (m1 << 2) | (m2 << 4) | (m3 << 6));
    }
    const uint32_t P[3] = {P0, P1, P2};
    return packed_row_scan(P, qw);
}

template <bool kDelta, bool kAny>
__device__ __forceinline__ void enc_full_pack_r(uint32_t sin, uint32_t prev_w, uint32_t sctrl, const uint32_t (&qw)[4],
                                                uint32_t sdst) {
    const int lane = threadIdx.x & 31;
    uint32_t last = prev_w;
#pragma unroll 1
    for (int j = 0; j < kWTRows; ++j) {
        const uint4 x = enc_row<kDelta, kAny>(sin, j, last);
        const uint32_t c = lds8(sctrl + 32 * j + lane);
        const uint32_t a = sdst + row_q_sel(qw, j);
        __syncwarp();  // every lane has read row j before any lane writes over it
        if (__all_sync(kFull, c == 0)) {
            const uint32_t P = __byte_perm(__byte_perm(x.x, x.y, 0x0040), __byte_perm(x.z, x.w, 0x0040), 0x5410);
            const uint32_t Pp = __shfl_up_sync(kFull, P, 1);
            const uint32_t s = a & 3u;
            if (s == 0) {
                sts32(a, P);
            } else {
                if (lane > 0) sts32(a & ~3u, __funnelshift_r(Pp, P, 8u * (4u - s)));
                if (lane == 0)
                    for (uint32_t b = 0; b < 4u - s; ++b) sts8(a + b, P >> (8 * b));
                if (lane == 31)
                    for (uint32_t b = 4u - s; b < 4u; ++b) sts8(a + b, P >> (8 * b));
            }
        } else {
            const uint32_t l = lens_of_ctrl(c);
            const uint32_t l0 = l & 0xFFu, l1 = (l >> 8) & 0xFFu, l2 = (l >> 16) & 0xFFu, l3 = l >> 24;
            sts_int_bytes(a, x.x, l0);
            sts_int_bytes(a + l0, x.y, l1);
            sts_int_bytes(a + l0 + l1, x.z, l2);
            sts_int_bytes(a + l0 + l1 + l2, x.w, l3);
        }
    }
}

}  // namespace bcgpu
