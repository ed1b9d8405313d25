// bcgpu_capi.cu -- the extern "C" boundary (include/bcgpu/bcgpu.h).
//
// Owns the per-context device workspace (look-back status words, tile ticket,
// status word) and the host-pointer entry points that give the reference's
// synchronous call semantics (H2D, kernel, D2H, codec_error mapping).
// No CPU fallback: every compute entry point launches a kernel or fails.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>

#include <cuda_runtime.h>

#include "bcgpu/bcgpu.h"
#include "svb_device.cuh"
#include "svb_kernels.cuh"

using namespace bcgpu;

namespace {

std::atomic<uint64_t> g_launches{0};
thread_local char g_cuda_err[256] = "";

int cuda_fail(cudaError_t e, const char* where) {
    std::snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", where, cudaGetErrorString(e));
    return BCGPU_ERR_CUDA;
}

#define BC_CUDA(call)                                   \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace

struct bcgpu_ctx {
    int device = 0;
    int num_sms = 148;
    // look-back workspace: [ticket | status word | off_status[cap] | sum_status[cap]]
    unsigned long long* ws = nullptr;
    size_t ws_tiles = 0;
    uint32_t epoch = 0;
    unsigned long long ticket_base = 0;
    uint32_t last_epoch = 0;  // epoch of the last *_device call
    unsigned long long* trace = nullptr;  // debug phase trace (bcgpu_debug_set_trace)
    uint32_t debug_flags = 0;
    // batch kernels: CTAs for full residency
    // host-API scratch (device) and stream
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;        // encode: second stream for the sliced pipeline
    cudaEvent_t events[96] = {};       // encode slice hand-offs
    void* offs = nullptr;  // decode metadata workspace (svb_decode.cu DecodeMeta)
    size_t offs_cap = 0;   // bytes
    int pipe_grid = 0;     // persistent decode CTAs
    void* d_scratch = nullptr;
    size_t d_scratch_cap = 0;
    uint8_t* slots = nullptr;  // encode: per-tile packing slots (svb_encode.cu)
    size_t slots_cap = 0;
    cudaStream_t aux2 = nullptr;             // host pipeline: device -> host copies
    unsigned long long* pin = nullptr;       // host pipeline: pinned offsets / status
    size_t pin_cap = 0;                      // entries
    uint64_t agg_n = 0;                      // n whose tile aggregates hold no current-epoch tag
    cudaEvent_t bev[2 * 128] = {};          // host batches: piece hand-offs (in, done)
    uint32_t* endval = nullptr;              // seek / select: last value of every sub-tile
    size_t endval_cap = 0;                   // entries
    void* gbws = nullptr;                    // varint-GB decode: chunk transfer tables (svb_gb.cu)
    size_t gbws_cap = 0;                     // bytes
};

static unsigned long long* ticket_ptr(bcgpu_ctx* c) { return c->ws; }
static unsigned long long* status_ptr(bcgpu_ctx* c) { return c->ws + 1; }
// status arrays hold one word per kStatusStride u64 (64 B) per tile
static uint64_t* off_status(bcgpu_ctx* c) { return reinterpret_cast<uint64_t*>(c->ws + 16); }
static uint64_t* sum_status(bcgpu_ctx* c) {
    return reinterpret_cast<uint64_t*>(c->ws + 16 + kStatusStride * c->ws_tiles);
}

static int ensure_ws(bcgpu_ctx* c, size_t tiles) {
    if (tiles < 1024) tiles = 1024;
    if (c->ws && tiles <= c->ws_tiles) return BCGPU_OK;
    size_t cap = c->ws_tiles ? c->ws_tiles : 1024;
    while (cap < tiles) cap *= 2;
    if (c->ws) {
        BC_CUDA(cudaDeviceSynchronize());
        BC_CUDA(cudaFree(c->ws));
        c->ws = nullptr;
    }
    const size_t bytes = (16 + 2 * kStatusStride * cap) * sizeof(unsigned long long);
    BC_CUDA(cudaMalloc(&c->ws, bytes));
    BC_CUDA(cudaMemset(c->ws, 0, bytes));
    c->ws_tiles = cap;
    // the epoch keeps running across reallocations: the one-pass encode's tile aggregates
    // (in the metadata workspace, not here) keep their old tags, and agg_n trusts that no
    // aggregate holds a tag >= the next epoch
    c->ticket_base = 0;
    return BCGPU_OK;
}

// Next launch epoch; status words of older launches never match it.
static int next_epoch(bcgpu_ctx* c, cudaStream_t s) {
    if (c->epoch >= kEpochMax) {
        BC_CUDA(cudaMemsetAsync(c->ws + 1, 0, (15 + 2 * kStatusStride * c->ws_tiles) * sizeof(unsigned long long), s));
        c->epoch = 0;
        c->agg_n = 0;  // old tags may repeat
    }
    c->epoch += 1;
    c->last_epoch = c->epoch;
    return BCGPU_OK;
}

static int make_lookback(bcgpu_ctx* c, uint64_t ngroups, uint32_t tile_groups, cudaStream_t s, LookbackArgs* lb) {
    const size_t tiles = (ngroups + tile_groups - 1) / tile_groups;
    int st = ensure_ws(c, tiles);
    if (st) return st;
    st = next_epoch(c, s);
    if (st) return st;
    lb->trace = c->trace;
    lb->debug_flags = c->debug_flags;
    lb->off_status = off_status(c);
    lb->sum_status = sum_status(c);
    lb->epoch = c->epoch;
    lb->num_tiles = (uint32_t)tiles;
    lb->status = status_ptr(c);
    return BCGPU_OK;
}

static int make_batch(bcgpu_ctx* c, cudaStream_t s, BatchArgs* ba) {
    int st = ensure_ws(c, 1024);
    if (st) return st;
    st = next_epoch(c, s);
    if (st) return st;
    ba->status = status_ptr(c);
    ba->epoch = c->epoch;
    ba->flags = c->debug_flags;
    ba->tickets = c->ws + 2;  // two spare words of the workspace head (zeroed with it; the kernels reset them)
    return BCGPU_OK;
}

static int ensure_meta(bcgpu_ctx* c, uint64_t n, cudaStream_t s) {
    const size_t bytes = decode_meta_bytes(n);
    if (c->agg_n != n) c->agg_n = 0;  // another layout may overwrite the aggregates of agg_n's
    if (bytes <= c->offs_cap) return BCGPU_OK;
    c->agg_n = 0;
    if (c->offs) {
        BC_CUDA(cudaStreamSynchronize(s));
        BC_CUDA(cudaFree(c->offs));
        c->offs = nullptr;
    }
    const size_t cap = bytes + bytes / 4 + 1024;
    BC_CUDA(cudaMalloc(&c->offs, cap));
    BC_CUDA(cudaMemset(c->offs, 0, cap));
    c->offs_cap = cap;
    return BCGPU_OK;
}

// Encode packing slots (svb_encode.cu).  The slot encode reads the integers once but
// moves the compressed bytes twice more (slot, then final place); measured on B200 it
// wins when they compress well (cfg2, 1.25 B/int: 99 vs 108 us) and loses on wide
// data (cfg3, ~2.5 B/int: 785 vs 648 us).  The compressed size is unknown up front,
// so: delta streams (sorted ids, small gaps) use slots, plain streams read twice.
// Debug flag 16 forces the two-read path, 32 the slot path.
static int ensure_slots(bcgpu_ctx* c, uint64_t n, int delta, cudaStream_t s, uint8_t** p) {
    *p = nullptr;
    if (c->debug_flags & 16) return BCGPU_OK;
    if (!delta && !(c->debug_flags & 32)) return BCGPU_OK;
    if (n > (1ull << 30)) return BCGPU_OK;  // slots take ~4 B/int of scratch
    const size_t bytes = encode_slot_bytes(n);
    if (bytes > c->slots_cap) {
        if (c->slots) {
            BC_CUDA(cudaStreamSynchronize(s));
            BC_CUDA(cudaFree(c->slots));
            c->slots = nullptr;
            c->slots_cap = 0;
        }
        const size_t cap = bytes + bytes / 8 + 4096;
        BC_CUDA(cudaMalloc(&c->slots, cap));
        c->slots_cap = cap;
    }
    *p = c->slots;
    return BCGPU_OK;
}

// ---------------------------------------------------------------------------
extern "C" {

int bcgpu_abi_version(void) { return BCGPU_ABI_VERSION; }

// Debug only (not in bcgpu.h): route per-tile phase timestamps (8 x u64 per
// look-back tile, %globaltimer ns) of the single-array kernels to d_trace.
int bcgpu_debug_set_trace(bcgpu_ctx* c, void* d_trace) {
    if (!c) return BCGPU_ERR_INVALID_ARGUMENT;
    c->trace = static_cast<unsigned long long*>(d_trace);
    return BCGPU_OK;
}

// Debug only (not in bcgpu.h): force a code path for A/B timing and the path-coverage
// tests (tests/test_fuzz.py).  Bits:
//   16      encode: two-read path (size scan + tile encode)
//   32      encode: slot path (bits 6-7: its L2 policies)
//   2048    encode: never the one-pass kernel;   4096  encode: one-pass for plain streams too
//   0x80000 encode: plain streams take the two-read path (size scan + tile encode)
//   0x100000 encode: delta streams take the scanner one-pass kernel (plain streams always do)
//   0x400000 decode: dense delta streams (1 byte per integer) still run the control scan
//   512     host API: no piecewise pipelining
//   1024    decode: sums pass + pooled delta decode instead of the one-pass kernel
//   0x8000  decode: the control scan only (dev timing; output not written)
//   0x40000 decode: the control scan also scans the chunk totals before the one-pass decode
//   bits 12-14 batch kernels: cap CTAs per SM
//   bits 16-23 segment-resident batch decode: ring KiB per warp (default 8)
//   bits 24-31 segment-resident batch encode: ring KiB per warp (default 9)
int bcgpu_debug_set_flags(bcgpu_ctx* c, uint32_t flags) {
    if (!c) return BCGPU_ERR_INVALID_ARGUMENT;
    c->debug_flags = flags;
    return BCGPU_OK;
}

const char* bcgpu_last_cuda_error(void) { return g_cuda_err; }

uint64_t bcgpu_kernel_launch_count(void) { return g_launches.load(); }

const char* bcgpu_status_string(int s) {
    switch (s) {
        case BCGPU_OK: return "ok";
        case BCGPU_ERR_TRUNCATED: return "truncated";
        case BCGPU_ERR_TRAILING_BYTES: return "trailing_bytes";
        case BCGPU_ERR_RUN_TOO_LONG: return "run_too_long";
        case BCGPU_ERR_VALUE_OVERFLOW: return "value_overflow";
        case BCGPU_ERR_OVERSIZED_INTEGER: return "oversized_integer";
        case BCGPU_ERR_COUNT_MISMATCH: return "count_mismatch";
        case BCGPU_ERR_BAD_STREAM_SIZE: return "bad_stream_size";
        case BCGPU_ERR_BAD_MAGIC: return "bad_magic";
        case BCGPU_ERR_UNKNOWN_CODEC: return "unknown_codec";
        case BCGPU_ERR_RESERVED_FLAGS: return "reserved_flags";
        case BCGPU_ERR_LENGTH_MISMATCH: return "length_mismatch";
        case BCGPU_ERR_UNSUPPORTED: return "unsupported";
        case BCGPU_ERR_OUT_OF_RANGE: return "out_of_range";
        case BCGPU_ERR_IO_FAILURE: return "io_failure";
        case BCGPU_ERR_BAD_CONFIG: return "bad_config";
        case BCGPU_ERR_INVALID_ARGUMENT: return "invalid_argument";
        case BCGPU_ERR_CUDA: return "cuda_error";
        case BCGPU_ERR_NO_DEVICE: return "no_device";
        default: return "unknown_status";
    }
}

uint32_t bcgpu_byte_length(uint32_t x) {
    return x < (1u << 8) ? 1u : x < (1u << 16) ? 2u : x < (1u << 24) ? 3u : 4u;
}

size_t bcgpu_svb_control_bytes(size_t n) { return (n + 3) / 4; }

size_t bcgpu_svb_max_compressed_bytes(size_t n) { return (n + 3) / 4 + 4 * n; }

void bcgpu_svb_tables(uint8_t length[256], uint8_t shuffle[256][16]) {
    for (int c = 0; c < 256; ++c) {
        int start = 0;
        for (int i = 0; i < 4; ++i) {
            const int len = ((c >> (2 * i)) & 3) + 1;
            for (int b = 0; b < 4; ++b) shuffle[c][4 * i + b] = (uint8_t)(b < len ? start + b : 0xFF);
            start += len;
        }
        length[c] = (uint8_t)start;
    }
}

int bcgpu_ctx_create(int device, bcgpu_ctx** out) {
    if (!out) return BCGPU_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return BCGPU_ERR_NO_DEVICE;
    if (device < 0 || device >= ndev) return BCGPU_ERR_INVALID_ARGUMENT;
    DeviceGuard g(device);
    bcgpu_ctx* c = new (std::nothrow) bcgpu_ctx();
    if (!c) return BCGPU_ERR_INVALID_ARGUMENT;
    c->device = device;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    c->pipe_grid = c->num_sms * occupancy_decode_pipe();
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaStreamCreate");
    }
    cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&c->aux2, cudaStreamNonBlocking);
    if (cudaHostAlloc(reinterpret_cast<void**>(&c->pin), 4096 * sizeof(unsigned long long), cudaHostAllocDefault) ==
        cudaSuccess)
        c->pin_cap = 4096;
    for (auto& ev : c->events) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    for (auto& ev : c->bev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    const int st = ensure_ws(c, 1024);
    if (st) {
        cudaStreamDestroy(c->stream);
        delete c;
        return st;
    }
    *out = c;
    return BCGPU_OK;
}

int bcgpu_ctx_destroy(bcgpu_ctx* c) {
    if (!c) return BCGPU_OK;
    DeviceGuard g(c->device);
    cudaDeviceSynchronize();
    if (c->ws) cudaFree(c->ws);
    if (c->d_scratch) cudaFree(c->d_scratch);
    if (c->offs) cudaFree(c->offs);
    if (c->slots) cudaFree(c->slots);
    if (c->endval) cudaFree(c->endval);
    if (c->gbws) cudaFree(c->gbws);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->aux) cudaStreamDestroy(c->aux);
    if (c->aux2) cudaStreamDestroy(c->aux2);
    if (c->pin) cudaFreeHost(c->pin);
    for (auto& ev : c->events)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : c->bev)
        if (ev) cudaEventDestroy(ev);
    delete c;
    return BCGPU_OK;
}

int bcgpu_ctx_sync_status(bcgpu_ctx* c, void* stream) {
    if (!c) return BCGPU_ERR_INVALID_ARGUMENT;
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    unsigned long long word = 0;
    BC_CUDA(cudaMemcpyAsync(&word, status_ptr(c), sizeof(word), cudaMemcpyDeviceToHost, s));
    BC_CUDA(cudaStreamSynchronize(s));
    if ((uint32_t)(word >> 32) != c->last_epoch) return BCGPU_OK;  // no error reported by that launch
    return (int)(uint32_t)word;
}

// ---------------------------------------------------------------------------
// device-pointer entry points
// ---------------------------------------------------------------------------
int bcgpu_svb_encode_device(bcgpu_ctx* c, const uint32_t* d_in, size_t n, int delta, uint32_t prev, uint8_t* d_out,
                            size_t out_cap, uint64_t* d_out_len, void* stream) {
    if (!c || (n && (!d_in || !d_out))) return BCGPU_ERR_INVALID_ARGUMENT;
    if (out_cap < bcgpu_svb_max_compressed_bytes(n)) return BCGPU_ERR_INVALID_ARGUMENT;
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) {
        const int se = next_epoch(c, s);  // a fresh status epoch: no earlier call's error is reported
        if (se) return se;
        if (d_out_len) BC_CUDA(cudaMemsetAsync(d_out_len, 0, sizeof(uint64_t), s));
        return BCGPU_OK;
    }
    int st = ensure_meta(c, n, s);
    if (st) return st;
    st = next_epoch(c, s);
    if (st) return st;
    uint8_t* slots = nullptr;
    uint32_t hints = (c->debug_flags & 32) ? ((c->debug_flags >> 6) & 3u) : 3u;
    // one-pass for delta streams (cfg2: 76 us vs 99 slot / 108 two-read); wide plain data is
    // compute-bound and runs faster through the 4-CTA/SM two-read kernels (cfg3: 646 vs 819 us).
    // Debug flags: 16 two-read, 32 slots, 2048 no one-pass, 4096 one-pass for plain too.
    // one pass for every 16-B aligned input (cfg3 plain: 472 us one-pass vs 552 us two-read);
    // debug flag 0x80000 restores the two-read path for plain streams
    const bool one_pass = !(c->debug_flags & (16 | 32 | 2048)) && (((uintptr_t)d_in) & 15) == 0 &&
                          (delta || !(c->debug_flags & 0x80000) || (c->debug_flags & 4096));
    if (one_pass) {
        // the one-pass encode's tile aggregates must not hold this epoch's tag: true when the
        // workspace was last laid out for this n (older epochs only), else clear them
        if (c->agg_n != n) {
            uint64_t cnt = 0;
            unsigned long long* agg = meta_agg_ptr(c->offs, n, &cnt);
            BC_CUDA(cudaMemsetAsync(agg, 0, cnt * sizeof(unsigned long long), s));
        }
        hints |= 0x100;
        if (c->debug_flags & 0x100000) hints |= 0x200;  // delta streams through the scanner kernel too
    } else {
        st = ensure_slots(c, n, delta, s, &slots);
        if (st) return st;
    }
    c->agg_n = n;
    int launches = 0;
    BC_CUDA(launch_encode3(d_in, n, delta, prev, d_out, d_out_len, c->offs, status_ptr(c), c->epoch, s, &launches,
                           slots, hints, c->trace));
    g_launches.fetch_add((uint64_t)launches);
    return BCGPU_OK;
}

int bcgpu_svb_decode_device(bcgpu_ctx* c, const uint8_t* d_in, size_t in_len, size_t n, int delta, uint32_t base,
                            uint32_t* d_out, uint32_t* d_last, void* stream) {
    if (!c || ((n && !d_out) || (in_len && !d_in))) return BCGPU_ERR_INVALID_ARGUMENT;
    const size_t nctrl = (n + 3) / 4;
    if (in_len < nctrl) return BCGPU_ERR_TRUNCATED;
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) {
        const int se = next_epoch(c, s);
        if (se) return se;
        if (d_last) BC_CUDA(cudaMemcpyAsync(d_last, &base, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        if (in_len != 0) return BCGPU_ERR_TRAILING_BYTES;
        return BCGPU_OK;
    }
    int st0 = ensure_meta(c, n, s);
    if (st0) return st0;
    const int st = next_epoch(c, s);
    if (st) return st;
    int launches = 0;
    // 0x800000: this layout's tile aggregates hold no current-epoch tag (a dense stream's
    // one-pass decode then skips clearing them)
    BC_CUDA(launch_decode3(d_in, in_len, n, delta, base, d_out, d_last, c->offs, status_ptr(c), c->epoch,
                           c->pipe_grid, s, &launches, c->trace, c->debug_flags | (c->agg_n == n ? 0x800000u : 0u)));
    if (delta) c->agg_n = n;  // its control scan cleared the aggregates of this layout
    g_launches.fetch_add((uint64_t)launches);
    return BCGPU_OK;
}

int bcgpu_svb_block_offsets_device(bcgpu_ctx* c, const uint8_t* d_in, size_t in_len, size_t n, uint64_t* d_offsets,
                                   void* stream) {
    if (!c || ((n && !d_offsets) || (in_len && !d_in))) return BCGPU_ERR_INVALID_ARGUMENT;
    const size_t nctrl = (n + 3) / 4;
    if (in_len < nctrl) return BCGPU_ERR_TRUNCATED;
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) return next_epoch(c, s);
    LookbackArgs lb;
    int st = make_lookback(c, nctrl, kOffsetsTileGroups, s, &lb);
    if (st) return st;
    BC_CUDA(launch_block_offsets(d_in, n, d_offsets, lb, s));
    g_launches.fetch_add(1);
    return BCGPU_OK;
}

int bcgpu_svb_decode_blocks_device(bcgpu_ctx* c, const uint8_t* d_in, size_t in_len, size_t n,
                                   const uint64_t* d_blocks, const uint64_t* d_offsets, size_t nblocks,
                                   uint32_t* d_out, uint32_t* d_counts, void* stream) {
    if (!c || (nblocks && (!d_in || !d_blocks || !d_offsets || !d_out || !d_counts))) return BCGPU_ERR_INVALID_ARGUMENT;
    if (nblocks == 0) return BCGPU_OK;
    DeviceGuard g(c->device);
    BC_CUDA(launch_decode_blocks(d_in, in_len, n, d_blocks, d_offsets, nblocks, d_out, d_counts,
                                 static_cast<cudaStream_t>(stream)));
    g_launches.fetch_add(1);
    return BCGPU_OK;
}

int bcgpu_svb_decode_batch_device(bcgpu_ctx* c, const bcgpu_decode_segment* d_segs, size_t nseg, const uint8_t* d_in,
                                  uint32_t* d_out, int delta, uint32_t max_seg_n, void* stream) {
    if (!c || (nseg && (!d_segs || !d_in || !d_out))) return BCGPU_ERR_INVALID_ARGUMENT;
    if (nseg == 0) return BCGPU_OK;
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    BatchArgs ba;
    int st = make_batch(c, s, &ba);
    if (st) return st;
    ba.max_seg_n = max_seg_n;  // bounds every segment's n when non-zero: skips the long-segment kernel
    BC_CUDA(launch_decode_batch(d_segs, nseg, d_in, d_out, delta, ba, s));
    g_launches.fetch_add(max_seg_n != 0 && max_seg_n <= kBatchSmallN ? 1 : 2);
    return BCGPU_OK;
}

int bcgpu_svb_encode_batch_device(bcgpu_ctx* c, const bcgpu_encode_segment* d_segs, size_t nseg, const uint32_t* d_in,
                                  uint8_t* d_out, uint64_t* d_out_lens, int delta, uint32_t max_seg_n, void* stream) {
    if (!c || (nseg && (!d_segs || !d_in || !d_out || !d_out_lens))) return BCGPU_ERR_INVALID_ARGUMENT;
    if (nseg == 0) return BCGPU_OK;
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    BatchArgs ba;
    int st = make_batch(c, s, &ba);
    if (st) return st;
    // one kernel serves every segment length; a bound <= kBatchSmallN (every segment one piece)
    // lets it size its rings for a sixth CTA per SM
    ba.max_seg_n = max_seg_n;
    BC_CUDA(launch_encode_batch(d_segs, nseg, d_in, d_out, d_out_lens, delta, ba, s));
    g_launches.fetch_add(1);
    return BCGPU_OK;
}

int bcgpu_svb_encoded_sizes_batch_device(bcgpu_ctx* c, const bcgpu_encode_segment* d_segs, size_t nseg,
                                         const uint32_t* d_in, uint64_t* d_out_lens, int delta, uint32_t max_seg_n,
                                         void* stream) {
    (void)max_seg_n;
    if (!c || (nseg && (!d_segs || !d_in || !d_out_lens))) return BCGPU_ERR_INVALID_ARGUMENT;
    if (nseg == 0) return BCGPU_OK;
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    BatchArgs ba;
    int st = make_batch(c, s, &ba);
    if (st) return st;
    BC_CUDA(launch_sizes_batch(d_segs, nseg, d_in, d_out_lens, delta, ba, s));
    g_launches.fetch_add(1);
    return BCGPU_OK;
}

// ---------------------------------------------------------------------------
// batched seek / select over one delta stream (svb_query.cu)
// ---------------------------------------------------------------------------
static int query_prepare(bcgpu_ctx* c, const uint8_t* d_in, size_t in_len, size_t n, uint32_t base, cudaStream_t s) {
    const size_t nsub = ((n + 3) / 4 + 255) / 256;
    int st = ensure_meta(c, n, s);
    if (st) return st;
    if (nsub + 1 > c->endval_cap) {
        if (c->endval) {
            BC_CUDA(cudaStreamSynchronize(s));
            BC_CUDA(cudaFree(c->endval));
            c->endval = nullptr;
            c->endval_cap = 0;
        }
        const size_t cap = nsub + nsub / 4 + 64;
        BC_CUDA(cudaMalloc(&c->endval, cap * sizeof(uint32_t)));
        c->endval_cap = cap;
    }
    st = next_epoch(c, s);
    if (st) return st;
    int launches = 0;
    BC_CUDA(launch_query_meta(d_in, in_len, n, base, c->offs, c->endval, status_ptr(c), c->epoch, s, &launches));
    g_launches.fetch_add((uint64_t)launches);
    c->agg_n = n;  // the control scan cleared this layout's aggregates
    return BCGPU_OK;
}

int bcgpu_svb_seek_batch_device(bcgpu_ctx* c, const uint8_t* d_in, size_t in_len, size_t n, uint32_t base,
                                const uint32_t* d_targets, size_t q, uint64_t* d_index, uint32_t* d_values,
                                void* stream) {
    if (!c || (q && (!d_targets || !d_index || !d_values)) || (n && !d_in)) return BCGPU_ERR_INVALID_ARGUMENT;
    if (in_len < (n + 3) / 4) return BCGPU_ERR_TRUNCATED;
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) {  // nothing to find: every index = n = 0 (not found)
        const int se = next_epoch(c, s);
        if (se) return se;
        if (in_len) return BCGPU_ERR_TRAILING_BYTES;
        if (q) {
            BC_CUDA(cudaMemsetAsync(d_index, 0, 8 * q, s));
            BC_CUDA(cudaMemsetAsync(d_values, 0, 4 * q, s));
        }
        return BCGPU_OK;
    }
    int st = query_prepare(c, d_in, in_len, n, base, s);
    if (st) return st;
    BC_CUDA(launch_query(d_in, in_len, n, base, c->offs, c->endval, 1, d_targets, q, d_index, d_values,
                         c->num_sms * 8, s));
    if (q) g_launches.fetch_add(1);
    return BCGPU_OK;
}

int bcgpu_svb_select_batch_device(bcgpu_ctx* c, const uint8_t* d_in, size_t in_len, size_t n, uint32_t base,
                                  const uint64_t* d_idx, size_t q, uint32_t* d_values, void* stream) {
    if (!c || (q && (!d_idx || !d_values)) || (n && !d_in)) return BCGPU_ERR_INVALID_ARGUMENT;
    if (in_len < (n + 3) / 4) return BCGPU_ERR_TRUNCATED;
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) {  // no valid index
        const int se = next_epoch(c, s);
        if (se) return se;
        if (in_len) return BCGPU_ERR_TRAILING_BYTES;
        if (q) BC_CUDA(cudaMemsetAsync(d_values, 0, 4 * q, s));
        return BCGPU_OK;
    }
    int st = query_prepare(c, d_in, in_len, n, base, s);
    if (st) return st;
    BC_CUDA(launch_query(d_in, in_len, n, base, c->offs, c->endval, 0, d_idx, q, nullptr, d_values,
                         c->num_sms * 8, s));
    if (q) g_launches.fetch_add(1);
    return BCGPU_OK;
}

// ---------------------------------------------------------------------------
// host-pointer entry points (synchronous; the reference's call semantics)
// ---------------------------------------------------------------------------
static int scratch(bcgpu_ctx* c, size_t bytes, void** p) {
    if (bytes > c->d_scratch_cap) {
        if (c->d_scratch) {
            BC_CUDA(cudaStreamSynchronize(c->stream));
            BC_CUDA(cudaFree(c->d_scratch));
            c->d_scratch = nullptr;
            c->d_scratch_cap = 0;
        }
        size_t cap = bytes + bytes / 8 + 4096;
        BC_CUDA(cudaMalloc(&c->d_scratch, cap));
        c->d_scratch_cap = cap;
    }
    *p = c->d_scratch;
    return BCGPU_OK;
}

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---- host pipeline: the array moves in pieces so that the host->device copies,
// the kernels and the device->host copies of different pieces overlap (PCIe is full
// duplex).  A piece is a whole number of 64 Ki-integer chunks; at most 30 pieces.
static constexpr uint64_t kChunkInts = 65536;
static uint64_t pipe_piece_ints(uint64_t n) {
    uint64_t p = 4ull << 20;  // 16 MiB of integers
    const uint64_t minp = (n + 29) / 30;
    if (p < minp) p = minp;
    return (p + kChunkInts - 1) / kChunkInts * kChunkInts;
}

// Encode: pieces stream in on `aux`; piece k's size scan continues from piece k-1's
// running offset and its tile encode follows on `stream`; once its offset is known on the
// host (pinned copy) its control and data bytes stream out on `aux2`.
static int ensure_pin(bcgpu_ctx* c, size_t entries);

static int encode_host_pipelined(bcgpu_ctx* c, const uint32_t* values, size_t n, int delta, uint32_t prev,
                                 uint8_t* out, uint8_t* d, size_t off_out, size_t* out_len) {
    const uint64_t P = pipe_piece_ints(n), K = (n + P - 1) / P;
    const uint64_t ngroups = (n + 3) / 4;
    cudaStream_t sc = c->stream, si = c->aux, so = c->aux2;
    int st = ensure_pin(c, K + 1);
    if (st) return st;
    st = ensure_meta(c, n, sc);
    if (st) return st;
    st = next_epoch(c, sc);
    if (st) return st;
    const uint32_t* d_in = reinterpret_cast<const uint32_t*>(d);
    uint8_t* d_out = d + off_out;
    unsigned long long* running = encode_running_ptr(c->offs, n);
    cudaEvent_t* ev_in = c->events;
    cudaEvent_t* ev_done = c->events + 32;
    for (uint64_t k = 0; k < K; ++k) {
        const uint64_t o = k * P, cnt = n - o < P ? n - o : P;
        BC_CUDA(cudaMemcpyAsync(d + 4 * o, values + o, 4 * cnt, cudaMemcpyHostToDevice, si));
        BC_CUDA(cudaEventRecord(ev_in[k], si));
    }
    const uint32_t cpp = (uint32_t)(P / kChunkInts);
    for (uint64_t k = 0; k < K; ++k) {
        BC_CUDA(cudaStreamWaitEvent(sc, ev_in[k], 0));
        BC_CUDA(launch_encode_piece(d_in, n, delta, prev, d_out, nullptr, c->offs, status_ptr(c), c->epoch,
                                    (uint32_t)k * cpp, (uint32_t)(k + 1) * cpp, sc));
        BC_CUDA(cudaMemcpyAsync(c->pin + k, running, sizeof(unsigned long long), cudaMemcpyDeviceToHost, sc));
        BC_CUDA(cudaEventRecord(ev_done[k], sc));
    }
    g_launches.fetch_add(2 * K);
    for (uint64_t k = 0; k < K; ++k) {
        BC_CUDA(cudaEventSynchronize(ev_done[k]));
        const uint64_t lo = k ? c->pin[k - 1] : 0ull, hi = c->pin[k];
        const uint64_t g0 = k * P / 4, g1 = (k + 1) * P / 4 < ngroups ? (k + 1) * P / 4 : ngroups;
        BC_CUDA(cudaStreamWaitEvent(so, ev_done[k], 0));
        BC_CUDA(cudaMemcpyAsync(out + g0, d_out + g0, g1 - g0, cudaMemcpyDeviceToHost, so));
        if (hi > lo)
            BC_CUDA(cudaMemcpyAsync(out + ngroups + lo, d_out + ngroups + lo, hi - lo, cudaMemcpyDeviceToHost, so));
    }
    BC_CUDA(cudaStreamSynchronize(so));
    *out_len = (size_t)(ngroups + c->pin[K - 1]);
    return BCGPU_OK;
}

int bcgpu_svb_encode_host(bcgpu_ctx* c, const uint32_t* values, size_t n, int delta, uint32_t prev, uint8_t* out,
                          size_t out_cap, size_t* out_len) {
    if (!c || !out_len || (n && (!values || !out))) return BCGPU_ERR_INVALID_ARGUMENT;
    *out_len = 0;
    if (n == 0) return BCGPU_OK;
    const size_t max_out = bcgpu_svb_max_compressed_bytes(n);
    DeviceGuard g(c->device);
    const size_t in_bytes = 4 * n;
    const size_t off_out = align_up(in_bytes, 256), off_len = align_up(off_out + max_out, 256);
    void* base = nullptr;
    int st = scratch(c, off_len + 256, &base);
    if (st) return st;
    uint8_t* d = static_cast<uint8_t*>(base);
    if (out_cap >= max_out && n >= 2 * pipe_piece_ints(n) && !(c->debug_flags & 512))
        return encode_host_pipelined(c, values, n, delta, prev, out, d, off_out, out_len);
    BC_CUDA(cudaMemcpyAsync(d, values, in_bytes, cudaMemcpyHostToDevice, c->stream));
    st = bcgpu_svb_encode_device(c, reinterpret_cast<uint32_t*>(d), n, delta, prev, d + off_out, max_out,
                                 reinterpret_cast<uint64_t*>(d + off_len), c->stream);
    if (st) return st;
    uint64_t len = 0;
    BC_CUDA(cudaMemcpyAsync(&len, d + off_len, sizeof(len), cudaMemcpyDeviceToHost, c->stream));
    BC_CUDA(cudaStreamSynchronize(c->stream));
    if (len > out_cap) return BCGPU_ERR_INVALID_ARGUMENT;
    BC_CUDA(cudaMemcpyAsync(out, d + off_out, len, cudaMemcpyDeviceToHost, c->stream));
    BC_CUDA(cudaStreamSynchronize(c->stream));
    *out_len = (size_t)len;
    return BCGPU_OK;
}

static int ensure_pin(bcgpu_ctx* c, size_t entries) {
    if (c->pin && entries <= c->pin_cap) return BCGPU_OK;
    BC_CUDA(cudaStreamSynchronize(c->stream));
    BC_CUDA(cudaStreamSynchronize(c->aux2));
    if (c->pin) cudaFreeHost(c->pin);
    c->pin = nullptr;
    c->pin_cap = 0;
    BC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->pin), entries * sizeof(unsigned long long), cudaHostAllocDefault));
    c->pin_cap = entries;
    return BCGPU_OK;
}

// Decode: the control bytes go first and are scanned on the device; the chunk offsets
// come back (pinned) so each piece's data range can stream in on `aux` while earlier
// pieces decode on `stream` and their integers stream out on `aux2`.
static int decode_host_pipelined(bcgpu_ctx* c, const uint8_t* bytes, size_t len, size_t n, int delta, uint32_t base,
                                 uint32_t* out, uint32_t* last, uint8_t* d, size_t off_out, size_t off_last) {
    const uint64_t P = pipe_piece_ints(n), K = (n + P - 1) / P;
    const uint64_t ngroups = (n + 3) / 4, nsub = (ngroups + 255) / 256, nchunks = (nsub + 63) / 64;
    cudaStream_t sc = c->stream, si = c->aux, so = c->aux2;
    int st = ensure_meta(c, n, sc);
    if (st) return st;
    st = ensure_pin(c, nchunks + 8);
    if (st) return st;
    st = next_epoch(c, sc);
    if (st) return st;
    uint32_t* d_out = reinterpret_cast<uint32_t*>(d + off_out);
    uint32_t* d_last = reinterpret_cast<uint32_t*>(d + off_last);
    cudaEvent_t* ev_in = c->events;
    cudaEvent_t* ev_done = c->events + 32;
    cudaEvent_t ev_ctrl = c->events[64];
    // 1. control bytes -> control scan -> chunk offsets + status to the host
    BC_CUDA(cudaMemcpyAsync(d, bytes, ngroups, cudaMemcpyHostToDevice, si));
    BC_CUDA(cudaEventRecord(ev_ctrl, si));
    BC_CUDA(cudaStreamWaitEvent(sc, ev_ctrl, 0));
    BC_CUDA(launch_decode_ctrl(d, len, n, delta, c->offs, status_ptr(c), c->epoch, sc));
    BC_CUDA(cudaMemcpyAsync(c->pin, decode_chunkpre_ptr(c->offs, n), 8 * (nchunks + 1), cudaMemcpyDeviceToHost, sc));
    BC_CUDA(cudaMemcpyAsync(c->pin + nchunks + 1, status_ptr(c), 8, cudaMemcpyDeviceToHost, sc));
    BC_CUDA(cudaStreamSynchronize(sc));
    g_launches.fetch_add(1);
    const unsigned long long word = c->pin[nchunks + 1];
    if ((uint32_t)(word >> 32) == c->epoch && (uint32_t)word) return (int)(uint32_t)word;
    const unsigned long long* cpre = c->pin;
    const uint64_t cpp = P / kChunkInts;
    // 2. pieces: data in, decode, integers out
    for (uint64_t k = 0; k < K; ++k) {
        const uint64_t c0 = k * cpp, c1 = (k + 1) * cpp < nchunks ? (k + 1) * cpp : nchunks;
        const uint64_t lo = ngroups + cpre[c0], hi = ngroups + cpre[c1];
        if (hi > lo) BC_CUDA(cudaMemcpyAsync(d + lo, bytes + lo, hi - lo, cudaMemcpyHostToDevice, si));
        BC_CUDA(cudaEventRecord(ev_in[k], si));
    }
    for (uint64_t k = 0; k < K; ++k) {
        BC_CUDA(cudaStreamWaitEvent(sc, ev_in[k], 0));
        int l = 0;
        BC_CUDA(launch_decode_range(d, len, n, delta, base, d_out, d_last, c->offs, k * cpp * 64, (k + 1) * cpp * 64, sc,
                                    &l, c->trace));
        g_launches.fetch_add((uint64_t)l);
        BC_CUDA(cudaEventRecord(ev_done[k], sc));
        BC_CUDA(cudaStreamWaitEvent(so, ev_done[k], 0));
        const uint64_t i0 = k * P, cnt = n - i0 < P ? n - i0 : P;
        BC_CUDA(cudaMemcpyAsync(out + i0, d_out + i0, 4 * cnt, cudaMemcpyDeviceToHost, so));
    }
    uint32_t lv = 0;
    if (delta) BC_CUDA(cudaMemcpyAsync(&lv, d_last, sizeof(lv), cudaMemcpyDeviceToHost, so));
    BC_CUDA(cudaStreamSynchronize(so));
    if (last) *last = delta ? lv : out[n - 1];
    return BCGPU_OK;
}

int bcgpu_svb_decode_host(bcgpu_ctx* c, const uint8_t* bytes, size_t len, size_t n, int delta, uint32_t base,
                          uint32_t* out, uint32_t* last) {
    if (!c || ((n && !out) || (len && !bytes))) return BCGPU_ERR_INVALID_ARGUMENT;
    const size_t nctrl = (n + 3) / 4;
    if (len < nctrl) return BCGPU_ERR_TRUNCATED;
    if (n == 0) {
        if (last) *last = base;
        return len ? BCGPU_ERR_TRAILING_BYTES : BCGPU_OK;
    }
    DeviceGuard g(c->device);
    const size_t off_out = align_up(len, 256), off_last = align_up(off_out + 4 * n, 256);
    void* sp = nullptr;
    int st = scratch(c, off_last + 256, &sp);
    if (st) return st;
    uint8_t* d = static_cast<uint8_t*>(sp);
    if (n >= 2 * pipe_piece_ints(n) && !(c->debug_flags & 512))
        return decode_host_pipelined(c, bytes, len, n, delta, base, out, last, d, off_out, off_last);
    BC_CUDA(cudaMemcpyAsync(d, bytes, len, cudaMemcpyHostToDevice, c->stream));
    st = bcgpu_svb_decode_device(c, d, len, n, delta, base, reinterpret_cast<uint32_t*>(d + off_out),
                                 reinterpret_cast<uint32_t*>(d + off_last), c->stream);
    if (st) return st;
    st = bcgpu_ctx_sync_status(c, c->stream);
    if (st) return st;
    BC_CUDA(cudaMemcpyAsync(out, d + off_out, 4 * n, cudaMemcpyDeviceToHost, c->stream));
    uint32_t lv = 0;
    BC_CUDA(cudaMemcpyAsync(&lv, d + off_last, sizeof(lv), cudaMemcpyDeviceToHost, c->stream));
    BC_CUDA(cudaStreamSynchronize(c->stream));
    if (last) *last = delta ? lv : out[n - 1];
    return BCGPU_OK;
}

int bcgpu_svb_decode_blocks_host(bcgpu_ctx* c, const uint8_t* bytes, size_t len, size_t n, const size_t* blocks,
                                 const size_t* offsets, size_t nblocks, uint32_t* out, uint32_t* counts) {
    if (!c || (nblocks && (!blocks || !offsets || !out || !counts)) || (len && !bytes))
        return BCGPU_ERR_INVALID_ARGUMENT;
    if (nblocks == 0) return BCGPU_OK;
    // svb_decode_block's contract (stream_vbyte.hpp:51-54) on host data: a block index past
    // ceil(n/4) is out_of_range; a block whose control byte or data bytes lie past the end
    // of the stream is truncated (the device entry point reports both as count 0)
    const size_t ngroups = (n + 3) / 4;
    for (size_t i = 0; i < nblocks; ++i) {
        if (blocks[i] >= ngroups) return BCGPU_ERR_OUT_OF_RANGE;
        if (blocks[i] >= len) return BCGPU_ERR_TRUNCATED;
        const uint32_t cnt = (blocks[i] == ngroups - 1 && (n & 3)) ? (uint32_t)(n & 3) : 4u;
        size_t need = 0;
        for (uint32_t f = 0; f < cnt; ++f) need += ((bytes[blocks[i]] >> (2 * f)) & 3u) + 1u;
        if (ngroups + offsets[i] + need > len || offsets[i] > len) return BCGPU_ERR_TRUNCATED;
    }
    DeviceGuard g(c->device);
    const size_t off_q = align_up(len, 256), off_o = off_q + 16 * nblocks, off_c = off_o + 16 * nblocks;
    void* sp = nullptr;
    int st = scratch(c, off_c + 4 * nblocks + 256, &sp);
    if (st) return st;
    uint8_t* d = static_cast<uint8_t*>(sp);
    if (len) BC_CUDA(cudaMemcpyAsync(d, bytes, len, cudaMemcpyHostToDevice, c->stream));
    static_assert(sizeof(size_t) == sizeof(uint64_t), "size_t must be 64-bit");
    BC_CUDA(cudaMemcpyAsync(d + off_q, blocks, 8 * nblocks, cudaMemcpyHostToDevice, c->stream));
    BC_CUDA(cudaMemcpyAsync(d + off_q + 8 * nblocks, offsets, 8 * nblocks, cudaMemcpyHostToDevice, c->stream));
    st = bcgpu_svb_decode_blocks_device(c, d, len, n, reinterpret_cast<uint64_t*>(d + off_q),
                                        reinterpret_cast<uint64_t*>(d + off_q + 8 * nblocks), nblocks,
                                        reinterpret_cast<uint32_t*>(d + off_o), reinterpret_cast<uint32_t*>(d + off_c),
                                        c->stream);
    if (st) return st;
    BC_CUDA(cudaMemcpyAsync(out, d + off_o, 16 * nblocks, cudaMemcpyDeviceToHost, c->stream));
    BC_CUDA(cudaMemcpyAsync(counts, d + off_c, 4 * nblocks, cudaMemcpyDeviceToHost, c->stream));
    BC_CUDA(cudaStreamSynchronize(c->stream));
    return BCGPU_OK;
}

int bcgpu_svb_block_offsets_host(bcgpu_ctx* c, const uint8_t* bytes, size_t len, size_t n, uint64_t* offsets) {
    if (!c || ((n && !offsets) || (len && !bytes))) return BCGPU_ERR_INVALID_ARGUMENT;
    const size_t nctrl = (n + 3) / 4;
    if (len < nctrl) return BCGPU_ERR_TRUNCATED;
    if (n == 0) return BCGPU_OK;
    DeviceGuard g(c->device);
    const size_t off_o = align_up(nctrl, 256);
    void* sp = nullptr;
    int st = scratch(c, off_o + 8 * nctrl, &sp);
    if (st) return st;
    uint8_t* d = static_cast<uint8_t*>(sp);
    BC_CUDA(cudaMemcpyAsync(d, bytes, nctrl, cudaMemcpyHostToDevice, c->stream));
    st = bcgpu_svb_block_offsets_device(c, d, nctrl, n, reinterpret_cast<uint64_t*>(d + off_o), c->stream);
    if (st) return st;
    BC_CUDA(cudaMemcpyAsync(offsets, d + off_o, 8 * nctrl, cudaMemcpyDeviceToHost, c->stream));
    BC_CUDA(cudaStreamSynchronize(c->stream));
    return BCGPU_OK;
}

// ---- host-buffer batches: segments of one batch move in pieces of whole segments so the
// host->device copies, the kernels and the device->host copies of different pieces overlap.
// A piece closes at >= P integers or >= S segments (P, S chosen so there are <= 121 pieces).
namespace {
constexpr int kBatchPieces = 128;
struct Piece {
    uint64_t s0, s1;   // segments
    uint64_t i0, i1;   // integers
    uint32_t max_n;
};
int cut_pieces(const uint32_t* seg_n, size_t nseg, Piece* pieces, int* npieces, uint64_t* total_n,
               uint64_t* total_cap) {
    uint64_t N = 0, cap = 0;
    for (size_t s = 0; s < nseg; ++s) {
        N += seg_n[s];
        cap += ((uint64_t)seg_n[s] + 3) / 4 + 4ull * seg_n[s];
    }
    const uint64_t P = std::max<uint64_t>(4ull << 20, (N + 59) / 60);
    const uint64_t S = std::max<uint64_t>(1ull << 20, (nseg + 59) / 60);
    int k = 0;
    Piece cur{0, 0, 0, 0, 0};
    uint64_t at = 0;
    for (size_t s = 0; s < nseg; ++s) {
        at += seg_n[s];
        cur.max_n = std::max(cur.max_n, seg_n[s]);
        if (at - cur.i0 >= P || s + 1 - cur.s0 >= S || s + 1 == nseg) {
            if (k >= kBatchPieces) return BCGPU_ERR_INVALID_ARGUMENT;  // cannot happen with the P, S above
            cur.s1 = s + 1;
            cur.i1 = at;
            pieces[k++] = cur;
            cur = Piece{s + 1, 0, at, 0, 0};
        }
    }
    *npieces = k;
    *total_n = N;
    *total_cap = cap;
    return BCGPU_OK;
}
}  // namespace

int bcgpu_svb_encode_batch_host(bcgpu_ctx* c, const uint32_t* values, const uint32_t* seg_n, const uint32_t* seg_prev,
                                size_t nseg, int delta, uint8_t* out, size_t out_cap, uint64_t* out_offsets) {
    if (!c || (nseg && (!seg_n || !out_offsets))) return BCGPU_ERR_INVALID_ARGUMENT;
    if (nseg == 0) {
        if (out_offsets) out_offsets[0] = 0;
        return BCGPU_OK;
    }
    Piece pieces[kBatchPieces];
    int K = 0;
    uint64_t N = 0, cap = 0;
    int st = cut_pieces(seg_n, nseg, pieces, &K, &N, &cap);
    if (st) return st;
    if (N && (!values || !out)) return BCGPU_ERR_INVALID_ARGUMENT;
    DeviceGuard g(c->device);
    const size_t o_vals = 0, o_out = align_up(4 * N, 256), o_n = align_up(o_out + cap + 16, 256),
                 o_prev = align_up(o_n + 4 * nseg, 256), o_es = align_up(o_prev + 4 * nseg, 256),
                 o_sz = align_up(o_es + sizeof(bcgpu_encode_segment) * nseg, 256),
                 o_offs = align_up(o_sz + 8 * nseg, 256), o_run = align_up(o_offs + 8 * (nseg + 1), 256);
    void* sp = nullptr;
    st = scratch(c, o_run + 256, &sp);
    if (st) return st;
    st = ensure_pin(c, (size_t)K + 1);
    if (st) return st;
    uint8_t* d = static_cast<uint8_t*>(sp);
    auto* d_vals = reinterpret_cast<uint32_t*>(d + o_vals);
    uint8_t* d_out = d + o_out;
    auto* d_n = reinterpret_cast<uint32_t*>(d + o_n);
    auto* d_prev = reinterpret_cast<uint32_t*>(d + o_prev);
    auto* d_es = reinterpret_cast<bcgpu_encode_segment*>(d + o_es);
    auto* d_sz = reinterpret_cast<uint64_t*>(d + o_sz);
    auto* d_offs = reinterpret_cast<uint64_t*>(d + o_offs);
    auto* d_run = reinterpret_cast<unsigned long long*>(d + o_run);
    cudaStream_t sc = c->stream, si = c->aux, so = c->aux2;
    BatchArgs ba;
    st = make_batch(c, sc, &ba);
    if (st) return st;
    cudaEvent_t* ev_in = c->bev;
    cudaEvent_t* ev_done = c->bev + kBatchPieces;
    BC_CUDA(cudaMemsetAsync(d_run, 0, 8, si));
    BC_CUDA(cudaMemcpyAsync(d_n, seg_n, 4 * nseg, cudaMemcpyHostToDevice, si));
    if (seg_prev) BC_CUDA(cudaMemcpyAsync(d_prev, seg_prev, 4 * nseg, cudaMemcpyHostToDevice, si));
    for (int k = 0; k < K; ++k) {
        const Piece& p = pieces[k];
        if (p.i1 > p.i0)
            BC_CUDA(cudaMemcpyAsync(d_vals + p.i0, values + p.i0, 4 * (p.i1 - p.i0), cudaMemcpyHostToDevice, si));
        BC_CUDA(cudaEventRecord(ev_in[k], si));
    }
    for (int k = 0; k < K; ++k) {
        const Piece& p = pieces[k];
        const uint32_t m = (uint32_t)(p.s1 - p.s0);
        BC_CUDA(cudaStreamWaitEvent(sc, ev_in[k], 0));
        BC_CUDA(launch_batch_encode_describe(d_n, seg_prev ? d_prev : nullptr, p.s0, m, p.i0, d_es, sc));
        BC_CUDA(launch_sizes_batch(d_es + p.s0, m, d_vals, d_sz + p.s0, delta, ba, sc));
        BC_CUDA(launch_batch_pack(d_sz, p.s0, m, d_es, d_offs, d_run, sc));
        BatchArgs be = ba;
        be.max_seg_n = p.max_n ? p.max_n : 1u;  // the piece's longest segment: ring sizing
        BC_CUDA(launch_encode_batch(d_es + p.s0, m, d_vals, d_out, d_sz + p.s0, delta, be, sc));
        BC_CUDA(cudaMemcpyAsync(c->pin + k, d_run, 8, cudaMemcpyDeviceToHost, sc));
        BC_CUDA(cudaEventRecord(ev_done[k], sc));
        g_launches.fetch_add(4);
    }
    int result = BCGPU_OK;
    for (int k = 0; k < K; ++k) {
        BC_CUDA(cudaEventSynchronize(ev_done[k]));
        const uint64_t lo = k ? c->pin[k - 1] : 0ull, hi = c->pin[k];
        if (hi > out_cap) {  // the caller's buffer is too small: stop copying, report after the drain
            result = BCGPU_ERR_INVALID_ARGUMENT;
            break;
        }
        BC_CUDA(cudaStreamWaitEvent(so, ev_done[k], 0));
        if (hi > lo) BC_CUDA(cudaMemcpyAsync(out + lo, d_out + lo, hi - lo, cudaMemcpyDeviceToHost, so));
    }
    if (result == BCGPU_OK)
        BC_CUDA(cudaMemcpyAsync(out_offsets, d_offs, 8 * (nseg + 1), cudaMemcpyDeviceToHost, so));
    BC_CUDA(cudaStreamSynchronize(sc));
    BC_CUDA(cudaStreamSynchronize(so));
    if (result) return result;
    return bcgpu_ctx_sync_status(c, sc);
}

int bcgpu_svb_decode_batch_host(bcgpu_ctx* c, const uint8_t* bytes, size_t len, const uint64_t* in_offsets,
                                const uint32_t* seg_n, const uint32_t* seg_base, size_t nseg, int delta, uint32_t* out,
                                uint32_t* last) {
    if (!c || (nseg && (!in_offsets || !seg_n))) return BCGPU_ERR_INVALID_ARGUMENT;
    if (nseg == 0) return BCGPU_OK;
    for (size_t s = 0; s < nseg; ++s)
        if (in_offsets[s + 1] < in_offsets[s]) return BCGPU_ERR_INVALID_ARGUMENT;
    if (in_offsets[nseg] > len) return BCGPU_ERR_TRUNCATED;
    Piece pieces[kBatchPieces];
    int K = 0;
    uint64_t N = 0, cap = 0;
    int st = cut_pieces(seg_n, nseg, pieces, &K, &N, &cap);
    if (st) return st;
    if ((N && !out) || (in_offsets[nseg] > in_offsets[0] && !bytes)) return BCGPU_ERR_INVALID_ARGUMENT;
    DeviceGuard g(c->device);
    const size_t o_in = 0, o_out = align_up(len + 16, 256), o_n = align_up(o_out + 4 * N, 256),
                 o_base = align_up(o_n + 4 * nseg, 256), o_offs = align_up(o_base + 4 * nseg, 256),
                 o_ds = align_up(o_offs + 8 * (nseg + 1), 256);
    void* sp = nullptr;
    st = scratch(c, o_ds + sizeof(bcgpu_decode_segment) * nseg + 256, &sp);
    if (st) return st;
    uint8_t* d = static_cast<uint8_t*>(sp);
    uint8_t* d_in = d + o_in;
    auto* d_out = reinterpret_cast<uint32_t*>(d + o_out);
    auto* d_n = reinterpret_cast<uint32_t*>(d + o_n);
    auto* d_base = reinterpret_cast<uint32_t*>(d + o_base);
    auto* d_offs = reinterpret_cast<uint64_t*>(d + o_offs);
    auto* d_ds = reinterpret_cast<bcgpu_decode_segment*>(d + o_ds);
    cudaStream_t sc = c->stream, si = c->aux, so = c->aux2;
    BatchArgs ba;
    st = make_batch(c, sc, &ba);
    if (st) return st;
    cudaEvent_t* ev_in = c->bev;
    cudaEvent_t* ev_done = c->bev + kBatchPieces;
    BC_CUDA(cudaMemcpyAsync(d_n, seg_n, 4 * nseg, cudaMemcpyHostToDevice, si));
    if (seg_base) BC_CUDA(cudaMemcpyAsync(d_base, seg_base, 4 * nseg, cudaMemcpyHostToDevice, si));
    BC_CUDA(cudaMemcpyAsync(d_offs, in_offsets, 8 * (nseg + 1), cudaMemcpyHostToDevice, si));
    for (int k = 0; k < K; ++k) {
        const Piece& p = pieces[k];
        const uint64_t lo = in_offsets[p.s0], hi = in_offsets[p.s1];
        if (hi > lo) BC_CUDA(cudaMemcpyAsync(d_in + lo, bytes + lo, hi - lo, cudaMemcpyHostToDevice, si));
        BC_CUDA(cudaEventRecord(ev_in[k], si));
    }
    for (int k = 0; k < K; ++k) {
        const Piece& p = pieces[k];
        const uint32_t m = (uint32_t)(p.s1 - p.s0);
        BC_CUDA(cudaStreamWaitEvent(sc, ev_in[k], 0));
        BC_CUDA(launch_batch_decode_describe(d_n, seg_base ? d_base : nullptr, d_offs, p.s0, m, p.i0, d_ds, sc));
        BatchArgs bp = ba;
        bp.max_seg_n = p.max_n ? p.max_n : 1u;
        BC_CUDA(launch_decode_batch(d_ds + p.s0, m, d_in, d_out, delta, bp, sc));
        g_launches.fetch_add(p.max_n <= kBatchSmallN ? 2 : 3);
        BC_CUDA(cudaEventRecord(ev_done[k], sc));
        BC_CUDA(cudaStreamWaitEvent(so, ev_done[k], 0));
        if (p.i1 > p.i0)
            BC_CUDA(cudaMemcpyAsync(out + p.i0, d_out + p.i0, 4 * (p.i1 - p.i0), cudaMemcpyDeviceToHost, so));
    }
    BC_CUDA(cudaStreamSynchronize(so));
    st = bcgpu_ctx_sync_status(c, sc);
    if (st) return st;
    if (last) {  // decode_payload_delta's return value per segment (codec.hpp:89-90): the last value, or base
        uint64_t at = 0;
        for (size_t s = 0; s < nseg; ++s) {
            at += seg_n[s];
            last[s] = seg_n[s] ? out[at - 1] : (seg_base ? seg_base[s] : 0u);
        }
    }
    return BCGPU_OK;
}


int bcgpu_svb_seek_host(bcgpu_ctx* c, const uint8_t* bytes, size_t len, size_t n, uint32_t base, const uint32_t* targets,
                        size_t q, uint64_t* index, uint32_t* values) {
    if (!c || (q && (!targets || !index || !values)) || (len && !bytes)) return BCGPU_ERR_INVALID_ARGUMENT;
    if (len < (n + 3) / 4) return BCGPU_ERR_TRUNCATED;
    DeviceGuard g(c->device);
    const size_t off_t = align_up(len, 256), off_i = align_up(off_t + 4 * q, 256), off_v = align_up(off_i + 8 * q, 256);
    void* sp = nullptr;
    int st = scratch(c, off_v + 4 * q + 256, &sp);
    if (st) return st;
    uint8_t* d = static_cast<uint8_t*>(sp);
    if (len) BC_CUDA(cudaMemcpyAsync(d, bytes, len, cudaMemcpyHostToDevice, c->stream));
    if (q) BC_CUDA(cudaMemcpyAsync(d + off_t, targets, 4 * q, cudaMemcpyHostToDevice, c->stream));
    st = bcgpu_svb_seek_batch_device(c, d, len, n, base, reinterpret_cast<uint32_t*>(d + off_t), q,
                                     reinterpret_cast<uint64_t*>(d + off_i), reinterpret_cast<uint32_t*>(d + off_v),
                                     c->stream);
    if (st) return st;
    st = bcgpu_ctx_sync_status(c, c->stream);
    if (st) return st;
    if (q) {
        BC_CUDA(cudaMemcpyAsync(index, d + off_i, 8 * q, cudaMemcpyDeviceToHost, c->stream));
        BC_CUDA(cudaMemcpyAsync(values, d + off_v, 4 * q, cudaMemcpyDeviceToHost, c->stream));
    }
    BC_CUDA(cudaStreamSynchronize(c->stream));
    return BCGPU_OK;
}

int bcgpu_svb_select_host(bcgpu_ctx* c, const uint8_t* bytes, size_t len, size_t n, uint32_t base, const uint64_t* idx,
                          size_t q, uint32_t* values) {
    if (!c || (q && (!idx || !values)) || (len && !bytes)) return BCGPU_ERR_INVALID_ARGUMENT;
    for (size_t i = 0; i < q; ++i)
        if (idx[i] >= n) return BCGPU_ERR_OUT_OF_RANGE;
    if (len < (n + 3) / 4) return BCGPU_ERR_TRUNCATED;
    DeviceGuard g(c->device);
    const size_t off_i = align_up(len, 256), off_v = align_up(off_i + 8 * q, 256);
    void* sp = nullptr;
    int st = scratch(c, off_v + 4 * q + 256, &sp);
    if (st) return st;
    uint8_t* d = static_cast<uint8_t*>(sp);
    if (len) BC_CUDA(cudaMemcpyAsync(d, bytes, len, cudaMemcpyHostToDevice, c->stream));
    if (q) BC_CUDA(cudaMemcpyAsync(d + off_i, idx, 8 * q, cudaMemcpyHostToDevice, c->stream));
    st = bcgpu_svb_select_batch_device(c, d, len, n, base, reinterpret_cast<uint64_t*>(d + off_i), q,
                                       reinterpret_cast<uint32_t*>(d + off_v), c->stream);
    if (st) return st;
    st = bcgpu_ctx_sync_status(c, c->stream);
    if (st) return st;
    if (q) BC_CUDA(cudaMemcpyAsync(values, d + off_v, 4 * q, cudaMemcpyDeviceToHost, c->stream));
    BC_CUDA(cudaStreamSynchronize(c->stream));
    return BCGPU_OK;
}

// ---------------------------------------------------------------------------
// varint-GB (svb_gb.cu)
// ---------------------------------------------------------------------------
static int ensure_gbws(bcgpu_ctx* c, uint64_t len, cudaStream_t s, void** p) {
    const size_t bytes = gb_decode_ws_bytes(len);
    if (bytes > c->gbws_cap) {
        if (c->gbws) {
            BC_CUDA(cudaStreamSynchronize(s));
            BC_CUDA(cudaFree(c->gbws));
            c->gbws = nullptr;
            c->gbws_cap = 0;
        }
        const size_t cap = bytes + bytes / 4 + 4096;
        BC_CUDA(cudaMalloc(&c->gbws, cap));
        c->gbws_cap = cap;
    }
    *p = c->gbws;
    return BCGPU_OK;
}

int bcgpu_gb_encode_device(bcgpu_ctx* c, const uint32_t* d_in, size_t n, int delta, uint32_t prev, uint8_t* d_out,
                           size_t out_cap, uint64_t* d_out_len, void* stream) {
    if (!c || (n && (!d_in || !d_out))) return BCGPU_ERR_INVALID_ARGUMENT;
    if (out_cap < bcgpu_svb_max_compressed_bytes(n)) return BCGPU_ERR_INVALID_ARGUMENT;
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) {
        const int se = next_epoch(c, s);
        if (se) return se;
        if (d_out_len) BC_CUDA(cudaMemsetAsync(d_out_len, 0, sizeof(uint64_t), s));
        return BCGPU_OK;
    }
    int st = ensure_meta(c, n, s);
    if (st) return st;
    st = next_epoch(c, s);
    if (st) return st;
    int launches = 0;
    BC_CUDA(launch_gb_encode(d_in, n, delta, prev, d_out, d_out_len, c->offs, status_ptr(c), c->epoch, s,
                             &launches));
    g_launches.fetch_add((uint64_t)launches);
    return BCGPU_OK;
}

int bcgpu_gb_decode_device(bcgpu_ctx* c, const uint8_t* d_in, size_t in_len, size_t n, int delta, uint32_t base,
                           uint32_t* d_out, uint32_t* d_last, void* stream) {
    if (!c || ((n && !d_out) || (in_len && !d_in))) return BCGPU_ERR_INVALID_ARGUMENT;
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) {
        const int se = next_epoch(c, s);
        if (se) return se;
        if (d_last) BC_CUDA(cudaMemcpyAsync(d_last, &base, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        return in_len ? BCGPU_ERR_TRAILING_BYTES : BCGPU_OK;
    }
    // every group holds a control byte and every integer at least one data byte
    if (in_len < (n + 3) / 4 + n) return BCGPU_ERR_TRUNCATED;
    void* ws = nullptr;
    int st = ensure_gbws(c, in_len, s, &ws);
    if (st) return st;
    // delta: the chunk carries come from a decoupled look-back (one status word per chunk)
    LookbackArgs lb;
    st = make_lookback(c, gb_decode_chunks(in_len), 1, s, &lb);
    if (st) return st;
    int launches = 0;
    BC_CUDA(launch_gb_decode(d_in, in_len, n, delta, base, d_out, d_last, ws, lb.sum_status, status_ptr(c), c->epoch,
                             s, &launches));
    g_launches.fetch_add((uint64_t)launches);
    return BCGPU_OK;
}

int bcgpu_gb_encode_host(bcgpu_ctx* c, const uint32_t* values, size_t n, int delta, uint32_t prev, uint8_t* out,
                         size_t out_cap, size_t* out_len) {
    if (!c || !out_len || (n && (!values || !out))) return BCGPU_ERR_INVALID_ARGUMENT;
    *out_len = 0;
    if (n == 0) return BCGPU_OK;
    const size_t max_out = bcgpu_svb_max_compressed_bytes(n);
    DeviceGuard g(c->device);
    const size_t off_out = align_up(4 * n, 256), off_len = align_up(off_out + max_out, 256);
    void* sp = nullptr;
    int st = scratch(c, off_len + 256, &sp);
    if (st) return st;
    uint8_t* d = static_cast<uint8_t*>(sp);
    BC_CUDA(cudaMemcpyAsync(d, values, 4 * n, cudaMemcpyHostToDevice, c->stream));
    st = bcgpu_gb_encode_device(c, reinterpret_cast<uint32_t*>(d), n, delta, prev, d + off_out, max_out,
                                reinterpret_cast<uint64_t*>(d + off_len), c->stream);
    if (st) return st;
    uint64_t len = 0;
    BC_CUDA(cudaMemcpyAsync(&len, d + off_len, sizeof(len), cudaMemcpyDeviceToHost, c->stream));
    BC_CUDA(cudaStreamSynchronize(c->stream));
    if (len > out_cap) return BCGPU_ERR_INVALID_ARGUMENT;
    BC_CUDA(cudaMemcpyAsync(out, d + off_out, len, cudaMemcpyDeviceToHost, c->stream));
    BC_CUDA(cudaStreamSynchronize(c->stream));
    *out_len = (size_t)len;
    return BCGPU_OK;
}

int bcgpu_gb_decode_host(bcgpu_ctx* c, const uint8_t* bytes, size_t len, size_t n, int delta, uint32_t base,
                         uint32_t* out, uint32_t* last) {
    if (!c || ((n && !out) || (len && !bytes))) return BCGPU_ERR_INVALID_ARGUMENT;
    if (n == 0) {
        if (last) *last = base;
        return len ? BCGPU_ERR_TRAILING_BYTES : BCGPU_OK;
    }
    if (len < (n + 3) / 4 + n) return BCGPU_ERR_TRUNCATED;
    DeviceGuard g(c->device);
    const size_t off_out = align_up(len, 256), off_last = align_up(off_out + 4 * n, 256);
    void* sp = nullptr;
    int st = scratch(c, off_last + 256, &sp);
    if (st) return st;
    uint8_t* d = static_cast<uint8_t*>(sp);
    BC_CUDA(cudaMemcpyAsync(d, bytes, len, cudaMemcpyHostToDevice, c->stream));
    st = bcgpu_gb_decode_device(c, d, len, n, delta, base, reinterpret_cast<uint32_t*>(d + off_out),
                                reinterpret_cast<uint32_t*>(d + off_last), c->stream);
    if (st) return st;
    st = bcgpu_ctx_sync_status(c, c->stream);
    if (st) return st;
    BC_CUDA(cudaMemcpyAsync(out, d + off_out, 4 * n, cudaMemcpyDeviceToHost, c->stream));
    uint32_t lv = 0;
    BC_CUDA(cudaMemcpyAsync(&lv, d + off_last, sizeof(lv), cudaMemcpyDeviceToHost, c->stream));
    BC_CUDA(cudaStreamSynchronize(c->stream));
    if (last) *last = delta ? lv : out[n - 1];
    return BCGPU_OK;
}

}  // extern "C"
