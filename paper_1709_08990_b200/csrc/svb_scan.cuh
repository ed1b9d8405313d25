// svb_scan.cuh -- chunk-level reduce-then-scan metadata shared by the
// single-array decode (svb_decode.cu) and encode (svb_encode.cu) kernels.
//
// The array is cut into sub-tiles of 1024 integers (256 control bytes) and
// chunks of kChunkSubs sub-tiles.  A size pass writes every sub-tile's
// chunk-local exclusive byte offset and every chunk's total; the last CTA to
// finish scans the chunk totals.  Consumers read offset = chunkpre[c] +
// localpre[s] -- no CTA ever waits on another.
#pragma once

#include "svb_device.cuh"
#include "svb_warp.cuh"

namespace bcgpu {

constexpr int kChunkSubs = 64;                      // sub-tiles per chunk (64K integers)
constexpr int kChunkCtrl = kChunkSubs * kWTGroups;  // 16 KiB of control bytes

// Exclusive scan of a[0..m) in place by one CTA of 32*kNW threads; returns the total.
template <class T, int kNW>
__device__ __forceinline__ T cta_exclusive_scan(T* a, uint32_t m, T* warp_tmp) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t per = (m + 32 * kNW - 1) / (32 * kNW);
    const uint32_t lo = tid * per, hi = lo + per < m ? lo + per : m;
    T s = 0;
    for (uint32_t i = lo; i < hi; ++i) s += a[i];
    T incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tmp[warp] = incl;
    __syncthreads();
    T wpre = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kNW; ++w) {
        wpre += w < warp ? warp_tmp[w] : (T)0;
        total += warp_tmp[w];
    }
    T run = wpre + incl - s;
    for (uint32_t i = lo; i < hi; ++i) {
        const T x = a[i];
        a[i] = run;
        run += x;
    }
    __syncthreads();
    return total;
}

// one-pass kernels (deferred look-back): epoch-tagged tile aggregates, relaxed at gpu scope
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// two consecutive aggregates (p 16-B aligned)
__device__ __forceinline__ ulonglong2 ld_relaxed_u64x2(const unsigned long long* p) {
    ulonglong2 v;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// named barrier of the 8 consumer warps of a producer/consumer CTA (the producer warp skips it)
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

struct DecodeMeta {
    uint32_t* localpre;              // [nsub]  sub-tile data offset within its chunk
    unsigned long long* chunkpre;    // [nchunks + 1] chunk data offset (exclusive; [nchunks] = total)
    uint32_t* subsums;               // [nsub]  delta: sum of the sub-tile's deltas
    uint32_t* chunksums;             // [nchunks + 1] delta: chunk sums -> exclusive prefix
    unsigned int* counters;          // [2] last-CTA tickets (self-resetting)
    uint32_t* chunktot;              // [nchunks] encode: chunk data totals (sliced size scan)
    unsigned long long* running;     // encode: data offset where the next slice starts
    unsigned long long* trace;       // debug: timestamps (nullptr = off)
    uint32_t* tilesize;              // [ntiles] encode: packed data bytes of each 8-sub-tile tile
    unsigned long long* agg;         // [ntiles] one-pass delta decode: (epoch << 32) | tile sum
};


// Carve the metadata arrays for an n-integer array out of a workspace of
// decode_meta_bytes(n) bytes (svb_decode.cu).
DecodeMeta carve_decode_meta(void* ws, uint64_t n);

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

}  // namespace bcgpu
