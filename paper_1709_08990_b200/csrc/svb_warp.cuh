// svb_warp.cuh -- warp-tile building blocks of the sm_100a Stream VByte kernels.
//
// A warp tile (sub-tile) is kWTGroups = 256 control bytes (1024 integers) laid
// out row-major over the warp: row j, lane l <-> control byte g0 + 32*j + l, so
// every row is 128 consecutive integers (one 512-B coalesced store per row).
//
//   ctrl   length of a control byte = 4 + popc(c&0x55) + 2 popc(c&0xAA)
//   scan   three packed (3 x 10-bit) warp scans -> tile-local data offsets
//   encode byte lengths, control bytes and packing of partial tiles (EncodeTile)
// The lean full-tile loops live in svb_fast.cuh.
#pragma once

#include "svb_device.cuh"

namespace bcgpu {

constexpr int kWTRows = 8;
constexpr int kWTGroups = 32 * kWTRows;     // 256 control bytes per warp tile
constexpr int kWTInts = 4 * kWTGroups;      // 1024 integers
constexpr int kWTDataMax = 16 * kWTGroups;  // 4 KiB worst-case data bytes
constexpr int kWTStage = kWTDataMax + 64;   // + alignment head + over-read slack
constexpr int kWTWarps = 4;                 // warps per CTA of the batch kernels
constexpr int kWTThreads = 32 * kWTWarps;
constexpr int kCTWarps = 8;                 // warps per CTA tile of the single-array kernels
constexpr int kCTThreads = 32 * kCTWarps;
constexpr int kCTGroups = kCTWarps * kWTGroups;  // 2048 control bytes = 8192 integers per CTA tile

// ---- shared-memory helpers ------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ---- control bytes of a warp tile --------------------------------------
struct WarpCtrl {
    uint32_t cw[2];  // control byte of row j in byte (j & 3) of cw[j >> 2]
    uint32_t qw[4];  // tile-local data offset of row j in half (j & 1) of qw[j >> 1]
    uint32_t total;  // data bytes of the tile
};

__device__ __forceinline__ uint32_t row_ctrl(const WarpCtrl& w, int j) { return (w.cw[j >> 2] >> (8 * (j & 3))) & 0xFFu; }
__device__ __forceinline__ uint32_t row_q(const WarpCtrl& w, int j) { return (w.qw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu; }

__device__ __forceinline__ uint32_t group_count(uint64_t g, uint64_t ngroups, uint32_t tail_r) {
    return g < ngroups ? ((g == ngroups - 1 && tail_r) ? tail_r : 4u) : 0u;
}

// sum of the four 2-bit fields of control byte c
__device__ __forceinline__ uint32_t fsum(uint32_t c) { return __popc(c & 0x55u) + 2u * __popc(c & 0xAAu); }

// Packed exclusive scan of 8 per-lane row values (each <= 16, row totals <= 512):
// three 3x10-bit warp scans.  q[j] = exclusive offset of (row j, lane) in row-major order.
template <int kRows = kWTRows>
__device__ __forceinline__ uint32_t packed_row_scan(const uint32_t (&P)[3], uint32_t (&qw)[4]) {
    uint32_t base = 0;
    qw[0] = qw[1] = qw[2] = qw[3] = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const uint32_t I = warp_inclusive_scan(P[k]);
        const uint32_t T = __shfl_sync(kFull, I, 31);
        const uint32_t E = I - P[k];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            const int j = 3 * k + f;
            if (j < kRows) {
                qw[j >> 1] |= (base + ((E >> (10 * f)) & 0x3FFu)) << (16 * (j & 1));
                base += (T >> (10 * f)) & 0x3FFu;
            }
        }
    }
    return base;
}

// ctrl[g] for the tile's control bytes: a global pointer (kSmem = false) or
// a shared-memory copy whose byte 0 is control byte `sbase` (kSmem = true).
template <bool kSmem = false>
__device__ __forceinline__ WarpCtrl load_warp_ctrl(const uint8_t* __restrict__ ctrl, uint64_t g0, uint64_t ngroups,
                                                   uint32_t tail_r, uint64_t sbase = 0) {
    const int lane = threadIdx.x & 31;
    WarpCtrl w;
    w.cw[0] = w.cw[1] = 0;
    uint32_t P[3] = {0, 0, 0};
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint64_t g = g0 + 32 * j + lane;
        uint32_t c = 0, len = 0;
        if (g < ngroups) {
            if constexpr (kSmem)
                c = ctrl[g - sbase];
            else
                c = __ldg(ctrl + g);
            if (g == ngroups - 1 && tail_r) {
                c &= (1u << (2 * tail_r)) - 1u;  // unused fields of the final control byte are ignored
                len = fsum(c) + tail_r;
            } else {
                len = fsum(c) + 4u;
            }
        }
        w.cw[j >> 2] |= c << (8 * (j & 3));
        P[j / 3] |= len << (10 * (j % 3));
    }
    w.total = packed_row_scan(P, w.qw);
    return w;
}




// ---- encode -----------------------------------------------------------------
// Loads the tile's integers (row-major, 128-bit), forms deltas (x_{-1} = prev_in
// for the tile's first integer), writes the control bytes and returns the
// per-row byte lengths packed (l0 | l1<<8 | l2<<16 | l3<<24) plus the scan.
struct EncodeTile {
    uint4 d[kWTRows];       // values (plain) or deltas
    uint32_t lens[kWTRows]; // packed per-integer byte lengths (0 = absent)
    uint32_t qw[4];         // tile-local data offsets (packed like WarpCtrl::qw)
    uint32_t total;
};


// Write every integer's bytes at its tile-local offset + base (stage byte base = tile data byte 0).
// A row whose 128 integers all take one byte (the usual case for small
// deltas) packs as 32 consecutive 4-byte words: each lane assembles its 4 low
// bytes with PRMT and stores the aligned word it starts (merged with its left
// neighbour's tail through a funnel shift); only the row's first and last
// partial words go out as bytes.  Every other row stores byte by byte.
__device__ __forceinline__ void encode_pack_at(const EncodeTile& t, uint8_t* stage, uint32_t base) {
    const int lane = threadIdx.x & 31;
    uint32_t* W = reinterpret_cast<uint32_t*>(stage);
#pragma unroll
    for (int j = 0; j < kWTRows; ++j) {
        const uint32_t l = t.lens[j];
        if (__all_sync(kFull, l == 0x01010101u)) {
            const uint4 x = t.d[j];
            const uint32_t P = __byte_perm(__byte_perm(x.x, x.y, 0x0040), __byte_perm(x.z, x.w, 0x0040), 0x5410);
            const uint32_t Pp = __shfl_up_sync(kFull, P, 1);
            const uint32_t p = base + ((t.qw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
            const uint32_t s = p & 3u;
            if (s == 0) {
                W[p >> 2] = P;
            } else {
                if (lane > 0) W[p >> 2] = __funnelshift_r(Pp, P, 8u * (4u - s));
                if (lane == 0)
                    for (uint32_t b = 0; b < 4u - s; ++b) stage[p + b] = (uint8_t)(P >> (8 * b));
                if (lane == 31)
                    for (uint32_t b = 4u - s; b < 4u; ++b) stage[p + b] = (uint8_t)(P >> (8 * b));
            }
            continue;
        }
        if (l) {
            uint32_t p = base + ((t.qw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
            const uint32_t l0 = l & 0xFFu, l1 = (l >> 8) & 0xFFu, l2 = (l >> 16) & 0xFFu, l3 = l >> 24;
            put_int_bytes(stage, p, t.d[j].x, l0);
            p += l0;
            if (l1) put_int_bytes(stage, p, t.d[j].y, l1);
            p += l1;
            if (l2) put_int_bytes(stage, p, t.d[j].z, l2);
            p += l2;
            if (l3) put_int_bytes(stage, p, t.d[j].w, l3);
        }
    }
}



}  // namespace bcgpu
