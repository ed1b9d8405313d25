// svb_device.cuh -- device building blocks shared by the sm_100a Stream VByte kernels.
//
// Format (reference stream_vbyte.hpp:15-19): ceil(n/4) control
// bytes, field i of control byte k (bits 2i..2i+1) = byte_length(x_{4k+i}) - 1,
// then the little-endian data bytes.  byte_length: codec.hpp:70-72.
//
// GPU decomposition: a tile is kTileGroups consecutive control
// bytes.  Phase A turns 16 B of control per thread into data lengths (SWAR, no
// LUT load on the critical path), block-scans them and obtains the tile's byte
// offset by decoupled look-back; phase B stages the tile's compressed bytes into
// shared memory with 16-B loads; phase C expands every control byte's 4..16 data
// bytes into four uint32 with funnel-shift/byte-permute (the GPU analogue of
// pshufb + shuffle table) and writes 128-bit coalesced stores.
// The delta variant fuses the mod-2^32 prefix sum with a
// second look-back on the tile sums.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bcgpu {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRows = 8;                        // control bytes owned per thread
constexpr int kTileGroups = kThreads * kRows;   // 2048 control bytes per tile
constexpr int kTileInts = kTileGroups * 4;      // 8192 integers per tile
constexpr int kTileDataMax = kTileGroups * 16;  // 32 KiB worst-case data per tile
constexpr int kStageBytes = kTileDataMax + 64;  // + 16-B alignment head + over-read slack

// warp-per-segment batch kernels: 4 rows x 32 lanes = 128 control bytes per step
constexpr int kWarpRows = 4;
constexpr int kWarpStepGroups = kWarpRows * 32;
constexpr int kWarpStageBytes = kWarpStepGroups * 16 + 64;

// ---- look-back status words: [epoch:26 | flag:2 | value:36] -------------
constexpr int kValueBits = 36;
constexpr uint64_t kValueMask = (1ull << kValueBits) - 1;
constexpr int kFlagShift = 36;
constexpr int kEpochShift = 38;
constexpr uint32_t kEpochMax = (1u << 26) - 1;
constexpr uint32_t kFlagAggregate = 1;
constexpr uint32_t kFlagInclusive = 2;

__device__ __forceinline__ uint64_t pack_status(uint32_t epoch, uint32_t flag, uint64_t value) {
    return ((uint64_t)epoch << kEpochShift) | ((uint64_t)flag << kFlagShift) | (value & kValueMask);
}

__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_gpu(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}


// Status words are spread one per 64 B (kStatusStride u64) so the ~256 newest
// ones -- which every in-flight look-back polls -- land in many L2 slices
// instead of hammering a few lines.
constexpr int kStatusStride = 1;

__device__ __forceinline__ uint64_t* status_slot(uint64_t* base, uint64_t tile) { return base + tile * kStatusStride; }
__device__ __forceinline__ const uint64_t* status_slot(const uint64_t* base, uint64_t tile) {
    return base + tile * kStatusStride;
}

// Wide decoupled look-back: each lane inspects 8 consecutive predecessors, so
// one warp round trip covers 256 tiles.  Only entries not yet published are
// re-polled, with exponential back-off.  Returns the exclusive prefix of `tile`.
__device__ __forceinline__ uint64_t lookback_exclusive_wide(const uint64_t* status, uint32_t tile, uint32_t epoch,
                                                            uint32_t* stats = nullptr) {
    const int lane = threadIdx.x & 31;
    uint64_t excl = 0;
    int64_t top = (int64_t)tile - 1;
    uint32_t spins = 0, rounds = 0;
    unsigned long long t_first = 0, t_begin = 0;
    if (stats) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_begin));
    while (true) {
        ++rounds;
        uint64_t v[8];
        uint32_t f[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = 0, v[i] = 0;
        uint32_t sleep_ns = 32;
        while (true) {
            bool ok = true;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (f[i] == 0) {
                    const int64_t idx = top - 8 * lane - i;
                    if (idx >= 0) {
                        const uint64_t s = ld_relaxed_gpu(status_slot(status, (uint64_t)idx));
                        f[i] = ((uint32_t)(s >> kEpochShift) == epoch) ? (uint32_t)((s >> kFlagShift) & 3u) : 0u;
                        v[i] = s & kValueMask;
                    } else {
                        f[i] = kFlagInclusive;
                        v[i] = 0;
                    }
                }
                ok = ok && f[i] != 0;
            }
            if (stats && t_first == 0) {
                uint64_t dep = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) dep += v[i] + f[i];
                asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_first) : "l"(dep));
            }
            if (__all_sync(kFull, ok)) break;
            ++spins;
            __nanosleep(sleep_ns);
            sleep_ns = sleep_ns < 512 ? 2 * sleep_ns : 512;
        }
        int first = 8;
#pragma unroll
        for (int i = 7; i >= 0; --i)
            if (f[i] == kFlagInclusive) first = i;
        const unsigned m = __ballot_sync(kFull, first < 8);
        const int fl = m ? __ffs(m) - 1 : 32;
        uint64_t contrib = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (lane < fl || (lane == fl && i <= first)) contrib += v[i];
#pragma unroll
        for (int o = 16; o; o >>= 1) contrib += __shfl_xor_sync(kFull, contrib, o);
        excl += contrib;
        if (m) break;
        top -= 256;
    }
    if (stats) {
        stats[0] = spins;
        stats[1] = rounds;
        stats[2] = (uint32_t)(t_first - t_begin);
    }
    return excl;
}

// ---- scans -------------------------------------------------------------
// Each step adds under the shuffle's own in-range predicate: shuffle + predicated add, where
// shuffle + lane compare + select + add is what the compiler makes of `if (lane >= o) v += t`.
__device__ __forceinline__ uint32_t warp_inclusive_scan(uint32_t v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1)
        asm("{\n\t.reg .pred p;\n\t.reg .u32 t;\n\t"
            "shfl.sync.up.b32 t|p, %0, %1, 0, 0xffffffff;\n\t"
            "@p add.u32 %0, %0, t;\n\t}"
            : "+r"(v)
            : "r"(o));
    return v;
}

// ---- control bytes -> lengths (SWAR over 4 control bytes per word) ------
// length[c] = 4 + sum of the four 2-bit fields; per byte.
__device__ __forceinline__ uint32_t swar_lengths(uint32_t w) {
    uint32_t s = (w & 0x33333333u) + ((w >> 2) & 0x33333333u);
    s = (s & 0x0F0F0F0Fu) + ((s >> 4) & 0x0F0F0F0Fu);
    return s + 0x04040404u;
}

// sum of the 2-bit fields of one control byte (0..12)
__device__ __forceinline__ uint32_t field_sum(uint32_t c) {
    return (c & 3u) + ((c >> 2) & 3u) + ((c >> 4) & 3u) + (c >> 6);
}

// The 8 control bytes [g, g+8) of a stream with ngroups control bytes:
// bytes past the end read as 0 with length 0; the final partial control byte
// (n % 4 = r != 0) is masked to its r fields with length sum(f_i + 1, i < r).
struct Ctrl8 {
    uint64_t c;    // control bytes, byte i = control byte g+i
    uint64_t len;  // data lengths, byte i = length of control byte g+i
};

__device__ __forceinline__ Ctrl8 load_ctrl8(const uint8_t* ctrl, uint64_t g, uint64_t ngroups, uint32_t tail_r) {
    Ctrl8 r;
    int64_t vb = (int64_t)ngroups - (int64_t)g;
    vb = vb > 8 ? 8 : (vb < 0 ? 0 : vb);
    const uint8_t* p = ctrl + g;
    if (vb == 8 && (((uintptr_t)p) & 7) == 0) {
        r.c = __ldg(reinterpret_cast<const unsigned long long*>(p));
    } else {
        r.c = 0;
        for (int i = 0; i < (int)vb; ++i) r.c |= (uint64_t)__ldg(p + i) << (8 * i);
    }
    if (tail_r != 0 && vb > 0 && g + (uint64_t)vb == ngroups) {
        const int bi = (int)vb - 1;
        const uint32_t cb = (uint32_t)(r.c >> (8 * bi)) & ((1u << (2 * tail_r)) - 1u);
        r.c = (r.c & ~(0xFFull << (8 * bi))) | ((uint64_t)cb << (8 * bi));
    }
    r.len = (uint64_t)swar_lengths((uint32_t)r.c) | ((uint64_t)swar_lengths((uint32_t)(r.c >> 32)) << 32);
    if (vb < 8) r.len &= (1ull << (8 * vb)) - 1;  // vb in [0,7]
    if (tail_r != 0 && vb > 0 && g + (uint64_t)vb == ngroups) {
        const int bi = (int)vb - 1;
        const uint32_t cb = (uint32_t)(r.c >> (8 * bi)) & 0xFFu;
        const uint64_t l = field_sum(cb) + tail_r;
        r.len = (r.len & ~(0xFFull << (8 * bi))) | (l << (8 * bi));
    }
    return r;
}

// ---- data expansion (phase C) -------------------------------------------
// Integer of l bytes starting at smem byte b (W = the staged words).
__device__ __forceinline__ uint32_t extract_int(const uint32_t* W, uint32_t b, uint32_t l) {
    const uint32_t x = __funnelshift_r(W[b >> 2], W[(b >> 2) + 1], (b & 3u) * 8u);
    return x & (0xFFFFFFFFu >> (32u - 8u * l));
}

// One control byte c whose data starts at smem byte b -> 4 integers.
__device__ __forceinline__ uint4 decode_group(const uint32_t* W, uint32_t b, uint32_t c) {
    const uint32_t l0 = (c & 3u) + 1u, l1 = ((c >> 2) & 3u) + 1u, l2 = ((c >> 4) & 3u) + 1u, l3 = (c >> 6) + 1u;
    const uint32_t b1 = b + l0, b2 = b1 + l1, b3 = b2 + l2;
    uint4 v;
    v.x = extract_int(W, b, l0);
    v.y = extract_int(W, b1, l1);
    v.z = extract_int(W, b2, l2);
    v.w = extract_int(W, b3, l3);
    return v;
}

// Control byte 0x00: four one-byte integers (the zero fast path).
__device__ __forceinline__ uint4 decode_zero_group(const uint32_t* W, uint32_t b) {
    const uint32_t x = __funnelshift_r(W[b >> 2], W[(b >> 2) + 1], (b & 3u) * 8u);
    uint4 v;
    v.x = __byte_perm(x, 0u, 0x4440);
    v.y = __byte_perm(x, 0u, 0x4441);
    v.z = __byte_perm(x, 0u, 0x4442);
    v.w = __byte_perm(x, 0u, 0x4443);
    return v;
}

// in-group inclusive prefix sum (the 4-lane block step of PAPER.md:115-117)
__device__ __forceinline__ uint4 prefix4(uint4 v) {
    v.y += v.x;
    v.z += v.y;
    v.w += v.z;
    return v;
}

__device__ __forceinline__ uint4 add4(uint4 v, uint32_t a) {
    v.x += a;
    v.y += a;
    v.z += a;
    v.w += a;
    return v;
}

__device__ __forceinline__ uint32_t comp(const uint4& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

__device__ __forceinline__ uint4 mask_tail(uint4 v, uint32_t cnt) {
    if (cnt < 4) v.w = 0;
    if (cnt < 3) v.z = 0;
    if (cnt < 2) v.y = 0;
    if (cnt < 1) v.x = 0;
    return v;
}

// ---- global memory helpers -----------------------------------------------
__device__ __forceinline__ uint4 ldg_stream_v4(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// L2 policy variants for a pass whose input is re-read by the next kernel
__device__ __forceinline__ uint64_t l2_policy_keep() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_policy_drop() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ void stg_hint_v4(void* p, const uint4& v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
}

__device__ __forceinline__ void stg_stream_v4(void* p, const uint4& v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// 16 bytes at the 16-B aligned address a, bytes outside [lo, hi) read as 0.
__device__ __forceinline__ uint4 load_chunk_guarded(uintptr_t a, uintptr_t lo, uintptr_t hi) {
    if (a >= lo && a + 16 <= hi) return ldg_stream_v4(reinterpret_cast<const void*>(a));
    uint32_t w[4] = {0, 0, 0, 0};
    for (int b = 0; b < 16; ++b) {
        const uintptr_t x = a + b;
        if (x >= lo && x < hi) w[b >> 2] |= (uint32_t)__ldg(reinterpret_cast<const uint8_t*>(x)) << (8 * (b & 3));
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// Store up to 4 integers of a group: one 128-bit store when the group is full
// and the destination 16-B aligned, scalar stores otherwise.
__device__ __forceinline__ void store_group(uint32_t* o, const uint4& v, uint32_t cnt, bool aligned16) {
    if (cnt == 4 && aligned16) {
        stg_stream_v4(o, v);
    } else {
        if (cnt > 0) o[0] = v.x;
        if (cnt > 1) o[1] = v.y;
        if (cnt > 2) o[2] = v.z;
        if (cnt > 3) o[3] = v.w;
    }
}

// byte_length (codec.hpp:70-72) as max(1, 4 - clz(x)/8)
__device__ __forceinline__ uint32_t dev_byte_length(uint32_t x) {
    const int l = 4 - (__clz(x) >> 3);
    return l < 1 ? 1u : (uint32_t)l;
}

// Write the l low bytes of x at smem byte p.
__device__ __forceinline__ void put_int_bytes(uint8_t* s, uint32_t p, uint32_t x, uint32_t l) {
    s[p] = (uint8_t)x;
    if (l > 1) s[p + 1] = (uint8_t)(x >> 8);
    if (l > 2) s[p + 2] = (uint8_t)(x >> 16);
    if (l > 3) s[p + 3] = (uint8_t)(x >> 24);
}

}  // namespace bcgpu
