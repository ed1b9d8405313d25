// svb_decode.cu -- single-array Stream VByte decode for sm_100a (svb_decode /
// svb_decode_delta, reference stream_vbyte.hpp:38-42, codec.hpp:85-90).
//
// Two launches per call:
//   1. svb_subtile_offsets_kernel -- control bytes only (0.25 B/int): data-region
//      offset of every 1024-integer sub-tile (exclusive scan of the paper's
//      length[c]), chunk prefixes by TMA-polled decoupled
//      look-back.  Also validates the stream length (truncated / trailing).
//   2. svb_decode_tile_kernel -- one CTA per 8 sub-tiles.  Each warp bulk-loads
//      its sub-tile's control and data bytes in one TMA transaction (offsets
//      are known, nothing waits on a neighbour), expands them in shared memory
//      (reverse row order makes the expansion in-place safe), and writes its
//      4 KiB of integers with one TMA bulk store.  The delta variant fuses the
//      mod-2^32 prefix sum: in-group 4-lane step, warp scan
//      per row, then one TMA-polled look-back per CTA for the carry.
#include <cstdint>

#include "svb_device.cuh"
#include "svb_kernels.cuh"
#include "svb_tma.cuh"
#include "svb_warp.cuh"

namespace bcgpu {

constexpr int kK1Subtiles = 256;                     // sub-tiles per offsets chunk (one per thread)
constexpr int kK1Ctrl = kK1Subtiles * kWTGroups;     // 65536 control bytes per chunk
constexpr int kK1Window = 1024;
constexpr int kK1Smem = kK1Ctrl + 64;
constexpr int kDecWindow = 1024;

__device__ __forceinline__ void report_status_dec(unsigned long long* st, uint32_t epoch, uint32_t code) {
    if (st) *st = ((unsigned long long)epoch << 32) | code;
}

// Data bytes declared by the control bytes [g, g+cnt) of a stream with
// ngroups control bytes (final partial control byte masked to tail_r fields).
// `p` points at control byte g in shared memory; `rot` staggers the word
// order across lanes to keep the shared loads conflict-free.
__device__ __forceinline__ uint32_t subtile_length(const uint8_t* p, uint64_t g, uint32_t cnt, uint64_t ngroups,
                                                   uint32_t tail_r, int rot) {
    const bool has_tail = tail_r != 0 && g + cnt == ngroups;
    uint32_t sum = 0;
    if (cnt == (uint32_t)kWTGroups && !has_tail) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(p);
#pragma unroll 8
        for (int k = 0; k < kWTGroups / 4; ++k) {
            const uint32_t x = swar_lengths(w[(k + rot) & (kWTGroups / 4 - 1)]);
            sum += (x * 0x01010101u) >> 24;
        }
        return sum;
    }
    for (uint32_t i = 0; i < cnt; ++i) {
        uint32_t c = p[i];
        if (has_tail && i == cnt - 1) {
            c &= (1u << (2 * tail_r)) - 1u;
            sum += fsum(c) + tail_r;
        } else {
            sum += fsum(c) + 4u;
        }
    }
    return sum;
}

__global__ void __launch_bounds__(256, 2)
    svb_subtile_offsets_kernel(const uint8_t* __restrict__ in, uint64_t in_len, uint64_t n, uint64_t* __restrict__ offs,
                               LookbackArgs lb) {
    extern __shared__ __align__(128) uint8_t sctrl[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(128) LookbackWin<kK1Window> lbw;
    __shared__ uint32_t warp_tot[8];
    __shared__ unsigned long long s_off;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t chunk = blockIdx.x;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint64_t g0 = (uint64_t)chunk * kK1Ctrl;
    const uint32_t cnt = (uint32_t)(ngroups - g0 < (uint64_t)kK1Ctrl ? ngroups - g0 : (uint64_t)kK1Ctrl);
    const uintptr_t cb = (uintptr_t)in + g0;
    const uint32_t tx = tma_cover_bytes(cb, cb + cnt, (uintptr_t)in, (uintptr_t)in + in_len);
    const bool use_tma = tx != 0xFFFFFFFFu && (cb & 15) == 0;
    if (tid == 0) {
        mbar_init1(&bar);
        mbar_init1(&lbw.bar);
        if (use_tma && tx) {
            mbar_expect(&bar, tx);
            tma_load(sctrl, reinterpret_cast<const void*>(cb), tx, &bar);
        }
    }
    if (!use_tma)
        for (uint32_t i = tid; i < cnt; i += 256) sctrl[i] = __ldg(in + g0 + i);
    __syncthreads();
    if (use_tma && tx) mbar_wait_parity(&bar, 0);

    const uint32_t my_g = (uint32_t)tid * kWTGroups;
    const uint32_t my_cnt = my_g < cnt ? (cnt - my_g < (uint32_t)kWTGroups ? cnt - my_g : (uint32_t)kWTGroups) : 0u;
    const uint32_t len = my_cnt ? subtile_length(sctrl + my_g, g0 + my_g, my_cnt, ngroups, tail_r, lane) : 0u;
    const uint32_t incl = warp_inclusive_scan(len);
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        wpre += w < warp ? warp_tot[w] : 0u;
        total += warp_tot[w];
    }
    if (warp == 0) {
        uint32_t phase = 0;
        const uint64_t off = lookback_tma_resolve<kK1Window>(lb.off_status, chunk, lb.epoch, 0, total, lbw, phase);
        if (lane == 0) s_off = off;
    }
    __syncthreads();
    const uint64_t sub = (uint64_t)chunk * kK1Subtiles + tid;
    if (sub < nsub) offs[sub] = s_off + wpre + incl - len;
    if (chunk == gridDim.x - 1 && tid == 0) {
        offs[nsub] = s_off + total;
        offs[nsub + 1] = s_off + total;
        const uint64_t need = ngroups + s_off + total;
        report_status_dec(lb.status, lb.epoch,
                          need > in_len ? BCGPU_ERR_TRUNCATED : (need < in_len ? BCGPU_ERR_TRAILING_BYTES : 0u));
    }
}

// ---------------------------------------------------------------------------
struct __align__(16) WarpBuf {
    uint8_t stage[kWTStage + 16];  // input bytes, then (in place) the sub-tile's 1024 integers at +16
    uint8_t ctrl[kWTGroups];
};

struct DecShared {
    uint32_t sum[kCTWarps];
    unsigned long long carry;
};

template <bool kDelta>
__global__ void __launch_bounds__(kCTThreads, 5)
    svb_decode_tile_kernel(const uint8_t* __restrict__ in, uint64_t in_len, uint64_t n, uint32_t base,
                           uint32_t* __restrict__ out, uint32_t* __restrict__ d_last,
                           const uint64_t* __restrict__ offs, LookbackArgs lb) {
    __shared__ __align__(128) WarpBuf wb[kCTWarps];
    __shared__ __align__(16) uint64_t soffs[kCTWarps + 2];
    __shared__ __align__(8) uint64_t bars[kCTWarps + 1];
    __shared__ DecShared sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tile = blockIdx.x;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint32_t tail_r = (uint32_t)(n & 3);
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const uint64_t sub0 = (uint64_t)tile * kCTWarps;
    const uint32_t nsub_tile = (uint32_t)(nsub - sub0 < (uint64_t)kCTWarps ? nsub - sub0 : (uint64_t)kCTWarps);

    // the CTA's sub-tile offsets (nsub_tile + 1 words, rounded to 16 B; offs has slack)
    if (threadIdx.x == 0) {
        mbar_init1(&bars[kCTWarps]);
        mbar_expect(&bars[kCTWarps], (uint32_t)(((nsub_tile + 2) & ~1u) * 8));
        tma_load(soffs, offs + sub0, (uint32_t)(((nsub_tile + 2) & ~1u) * 8), &bars[kCTWarps]);
    }
    if (lane == 0) mbar_init1(&bars[warp]);
    __syncthreads();
    mbar_wait_parity(&bars[kCTWarps], 0);

    WarpBuf& b = wb[warp];
    const bool active = (uint32_t)warp < nsub_tile;
    const uint64_t sub = sub0 + warp;
    const uint64_t g0 = sub * kWTGroups;
    const uintptr_t lo = (uintptr_t)in, hi = lo + in_len;
    uint32_t T[kWTRows];
    uint32_t wtot = 0;
    uint32_t* o = out + 4 * g0;
    const uint32_t nints = active ? (uint32_t)(n - 4 * g0 < (uint64_t)kWTInts ? n - 4 * g0 : (uint64_t)kWTInts) : 0u;
    if (active) {
        const uint64_t off = soffs[warp];
        const uint32_t len = (uint32_t)(soffs[warp + 1] - off);
        const uint32_t cnt_g = (uint32_t)(ngroups - g0 < (uint64_t)kWTGroups ? ngroups - g0 : (uint64_t)kWTGroups);
        const uintptr_t cbeg = lo + g0;
        const uintptr_t dbeg = lo + ngroups + off;
        const uint32_t ctx = tma_cover_bytes(cbeg, cbeg + cnt_g, lo, hi);
        const uint32_t dtx = tma_cover_bytes(dbeg, dbeg + len, lo, hi);
        const bool c_tma = ctx != 0xFFFFFFFFu && (cbeg & 15) == 0;
        const bool d_tma = dtx != 0xFFFFFFFFu;
        const uint32_t expect = (c_tma ? ctx : 0u) + (d_tma ? dtx : 0u);
        if (lane == 0 && expect) {
            mbar_expect(&bars[warp], expect);
            if (c_tma && ctx) tma_load(b.ctrl, reinterpret_cast<const void*>(cbeg), ctx, &bars[warp]);
            if (d_tma && dtx) tma_load(b.stage, reinterpret_cast<const void*>(dbeg & ~(uintptr_t)15), dtx, &bars[warp]);
        }
        if (!c_tma)
            for (uint32_t i = lane; i < cnt_g; i += 32) b.ctrl[i] = __ldg(in + g0 + i);
        if (!d_tma) copy_guarded_warp(b.stage, dbeg, dbeg + len, lo, hi);
        __syncwarp();
        if (expect) mbar_wait_parity(&bars[warp], 0);

        const WarpCtrl w = load_warp_ctrl<true>(b.ctrl, g0, ngroups, tail_r, g0);
        const uint32_t* W = reinterpret_cast<const uint32_t*>(b.stage);
        const uint32_t head = (uint32_t)(dbeg & 15);
        // reverse row order: row j's output [16+512j, +512) lies above every
        // input byte of rows < j (at most 512j bytes from stage+head, head < 16)
#pragma unroll
        for (int j = kWTRows - 1; j >= 0; --j) {
            const uint32_t c = row_ctrl(w, j);
            const uint32_t bb = head + row_q(w, j);
            const bool allzero = __all_sync(kFull, c == 0);
            uint4 v = allzero ? decode_zero_group(W, bb) : decode_group(W, bb, c);
            if constexpr (kDelta) {
                const uint32_t cnt = group_count(g0 + 32 * j + lane, ngroups, tail_r);
                v = prefix4(mask_tail(v, cnt));
                const uint32_t S = v.w;
                const uint32_t I = warp_inclusive_scan(S);
                v = add4(v, I - S);
                T[j] = __shfl_sync(kFull, I, 31);
                wtot += T[j];
            }
            __syncwarp();
            *reinterpret_cast<uint4*>(b.stage + 16 + 512 * j + 16 * lane) = v;
        }
    }
    uint32_t carry = 0, csum = 0, sex = 0;
    if constexpr (kDelta) {
        __shared__ __align__(128) LookbackWin<kDecWindow> lbw;
        if (threadIdx.x == 0) mbar_init1(&lbw.bar);
        if (lane == 0) sh.sum[warp] = wtot;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kCTWarps; ++k) {
            const uint32_t x = sh.sum[k];
            sex += k < warp ? x : 0u;
            csum += x;
        }
        if (warp == 0) {
            uint32_t phase = 0;
            const uint64_t c =
                lookback_tma_resolve<kDecWindow>(lb.sum_status, tile, lb.epoch, base, csum, lbw, phase);
            if (lane == 0) sh.carry = c;
        }
        __syncthreads();
        carry = (uint32_t)sh.carry;
        if (active) {
            uint32_t R = carry + sex;
#pragma unroll
            for (int j = 0; j < kWTRows; ++j) {
                uint4* p = reinterpret_cast<uint4*>(b.stage + 16 + 512 * j + 16 * lane);
                *p = add4(*p, R);
                R += T[j];
            }
        }
    }
    if (active) {
        // one bulk store of the sub-tile's integers (16-B aligned part), lanes store the rest
        const uint32_t bytes = 4 * nints;
        const bool o16 = (((uintptr_t)o) & 15) == 0;
        const uint32_t tbytes = o16 ? (bytes & ~15u) : 0u;
        fence_async_smem();
        __syncwarp();
        if (lane == 0 && tbytes) {
            tma_store(o, b.stage + 16, tbytes);
            tma_store_commit();
        }
        const uint32_t* src = reinterpret_cast<const uint32_t*>(b.stage + 16);
        for (uint32_t i = tbytes / 4 + lane; i < nints; i += 32) o[i] = src[i];
        if (lane == 0 && tbytes) tma_store_wait_read();
    }
    if (kDelta && tile == gridDim.x - 1 && threadIdx.x == 0 && d_last) *d_last = carry + csum;
}

// ---------------------------------------------------------------------------
cudaError_t launch_decode2(const uint8_t* in, uint64_t in_len, uint64_t n, int delta, uint32_t base, uint32_t* out,
                           uint32_t* d_last, uint64_t* offs, const LookbackArgs& lb_offs, const LookbackArgs& lb_dec,
                           cudaStream_t stream) {
    static const cudaError_t attr =
        cudaFuncSetAttribute(svb_subtile_offsets_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kK1Smem);
    if (attr != cudaSuccess) return attr;
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    const int g1 = (int)((ngroups + kK1Ctrl - 1) / kK1Ctrl);
    svb_subtile_offsets_kernel<<<g1, 256, kK1Smem, stream>>>(in, in_len, n, offs, lb_offs);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int g2 = (int)((nsub + kCTWarps - 1) / kCTWarps);
    if (delta)
        svb_decode_tile_kernel<true><<<g2, kCTThreads, 0, stream>>>(in, in_len, n, base, out, d_last, offs, lb_dec);
    else
        svb_decode_tile_kernel<false><<<g2, kCTThreads, 0, stream>>>(in, in_len, n, base, out, d_last, offs, lb_dec);
    return cudaGetLastError();
}

uint64_t decode2_offsets_words(uint64_t n) {
    const uint64_t ngroups = (n + 3) >> 2;
    return (ngroups + kWTGroups - 1) / kWTGroups + 4;
}

uint32_t decode2_chunks(uint64_t n) {
    const uint64_t ngroups = (n + 3) >> 2;
    return (uint32_t)((ngroups + kK1Ctrl - 1) / kK1Ctrl);
}

uint32_t decode2_tiles(uint64_t n) {
    const uint64_t ngroups = (n + 3) >> 2;
    const uint64_t nsub = (ngroups + kWTGroups - 1) / kWTGroups;
    return (uint32_t)((nsub + kCTWarps - 1) / kCTWarps);
}

}  // namespace bcgpu
