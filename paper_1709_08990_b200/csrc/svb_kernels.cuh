// svb_kernels.cuh -- sm_100a Stream VByte kernels (declarations for the C-ABI layer).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "bcgpu/bcgpu.h"

namespace bcgpu {

// Arguments of the single-array (decoupled look-back) kernels.
struct LookbackArgs {
    uint64_t* off_status;          // per-tile byte-offset status words
    uint64_t* sum_status;          // per-tile delta-sum status words
    unsigned long long* trace;     // debug: per-tile phase timestamps (nullptr = off)
    uint32_t debug_flags;          // debug: bit0 = skip output stores (timing experiments only)
    uint32_t epoch;
    uint32_t num_tiles;
    unsigned long long* status;    // [epoch:32 | bcgpu_status:32] of the last call
};

// Launchers (return cudaError_t of the launch).
// Single-array decode (svb_decode.cu): control scan, [delta: tile-sum pass],
// pipelined decode.  meta_ws holds decode_meta_bytes(n) bytes (16-B aligned,
// first 16 bytes zero-initialised once and self-resetting).
cudaError_t launch_decode3(const uint8_t* in, uint64_t in_len, uint64_t n, int delta, uint32_t base, uint32_t* out,
                           uint32_t* d_last, void* meta_ws, unsigned long long* status, uint32_t epoch, int pipe_grid,
                           cudaStream_t stream, int* launches, unsigned long long* trace = nullptr,
                           uint32_t debug_flags = 0);
uint64_t decode_meta_bytes(uint64_t n);
// The same split for the pipelined host API: the control scan over the whole stream,
// then passes 2-3 per range of sub-tiles (chunk multiples, in order for delta).
// delta bit 1: skip the chunk-total scan (the one-pass decode that follows sums them itself)
cudaError_t launch_decode_ctrl(const uint8_t* in, uint64_t in_len, uint64_t n, int delta, void* meta_ws,
                               unsigned long long* status, uint32_t epoch, cudaStream_t stream);
cudaError_t launch_decode_range(const uint8_t* in, uint64_t in_len, uint64_t n, int delta, uint32_t base,
                                uint32_t* out, uint32_t* d_last, void* meta_ws, uint64_t sub_begin, uint64_t sub_end,
                                cudaStream_t stream, int* launches, unsigned long long* trace = nullptr,
                                uint32_t epoch = 0,  // epoch != 0: a whole-stream delta decode may run one-pass
                                unsigned long long* status = nullptr,
                                uint32_t totals = 0);  // the control scan left chunk totals (one-pass only)
unsigned long long* decode_chunkpre_ptr(void* meta_ws, uint64_t n);
unsigned long long* meta_agg_ptr(void* meta_ws, uint64_t n, uint64_t* count);
cudaError_t launch_decode_sums(const uint8_t* in, uint64_t in_len, uint64_t n, void* meta_ws, cudaStream_t stream);
// Batched seek / select over one delta stream (svb_query.cu): metadata pass (3 launches,
// endval = last logical value of each 1024-integer sub-tile), then one warp per query.
cudaError_t launch_query_meta(const uint8_t* in, uint64_t in_len, uint64_t n, uint32_t base, void* meta_ws,
                              uint32_t* endval, unsigned long long* status, uint32_t epoch, cudaStream_t stream,
                              int* launches);
cudaError_t launch_query(const uint8_t* in, uint64_t in_len, uint64_t n, uint32_t base, void* meta_ws,
                         const uint32_t* endval, int seek, const void* queries, uint64_t q, uint64_t* out_index,
                         uint32_t* out_value, int grid_cap, cudaStream_t stream);
int occupancy_decode_pipe();
// Single-array encode (svb_encode.cu); meta_ws as for the decode.  With `slots`
// (encode_slot_bytes(n) of device scratch, 128-B aligned): slot encode + compaction,
// one read of the integers; without: size scan + tile encode (two reads).
cudaError_t launch_encode3(const uint32_t* in, uint64_t n, int delta, uint32_t prev, uint8_t* out,
                           uint64_t* d_out_len, void* meta_ws, unsigned long long* status, uint32_t epoch,
                           cudaStream_t stream, int* launches, uint8_t* slots = nullptr, uint32_t hints = 3,
                           unsigned long long* trace = nullptr);
// hints: bit 0/1 L2 policies of the slot encode; 0x100 try the one-pass encode first (needs the
// workspace's tile aggregates free of this epoch's tag: see bcgpu_capi.cu)
// Chunks [c0, c1) (64 Ki integers each) of the two-read encode, continuing from the
// previous piece's running offset; 2 launches.  For the pipelined host API.
cudaError_t launch_encode_piece(const uint32_t* in, uint64_t n, int delta, uint32_t prev, uint8_t* out,
                                uint64_t* d_out_len, void* meta_ws, unsigned long long* status, uint32_t epoch,
                                uint32_t c0, uint32_t c1, cudaStream_t stream);
unsigned long long* encode_running_ptr(void* meta_ws, uint64_t n);
// size scan alone (per-sub-tile data offsets in meta_ws, total size to d_out_len); 1 launch
cudaError_t launch_size_scan(const uint32_t* in, uint64_t n, int delta, uint32_t prev, void* meta_ws,
                             uint64_t* d_out_len, unsigned long long* status, uint32_t epoch, cudaStream_t stream);
// varint-GB (svb_gb.cu): encode = size scan + group writer; decode = chunk tables, tree
// compose / expand, group decode.  The decode workspace is gb_decode_ws_bytes(len) bytes.
cudaError_t launch_gb_encode(const uint32_t* in, uint64_t n, int delta, uint32_t prev, uint8_t* out,
                             uint64_t* d_out_len, void* meta_ws, unsigned long long* status, uint32_t epoch,
                             cudaStream_t stream, int* launches);
size_t gb_decode_ws_bytes(uint64_t len);
// delta: lstatus = look-back status words of >= ceil(len / 4096) chunks tagged with epoch
cudaError_t launch_gb_decode(const uint8_t* in, uint64_t len, uint64_t n, int delta, uint32_t base, uint32_t* out,
                             uint32_t* d_last, void* ws, uint64_t* lstatus, unsigned long long* status,
                             uint32_t epoch, cudaStream_t stream, int* launches);
uint64_t gb_decode_chunks(uint64_t len);
uint64_t encode_slot_bytes(uint64_t n);
cudaError_t launch_block_offsets(const uint8_t* in, uint64_t n, uint64_t* d_offsets, const LookbackArgs& lb,
                                 cudaStream_t stream);

cudaError_t launch_decode_blocks(const uint8_t* in, uint64_t in_len, uint64_t n, const uint64_t* blocks,
                                 const uint64_t* offsets, uint64_t nblocks, uint32_t* out, uint32_t* counts,
                                 cudaStream_t stream);

struct BatchArgs {
    unsigned long long* status;  // [epoch:32 | bcgpu_status:32]
    uint32_t epoch;
    uint32_t flags = 0;          // debug flags of the ctx (bits 12..14: batch-decode CTAs per SM)
    uint32_t max_seg_n = 0;      // caller's bound on every segment's n (0 = unknown)
    unsigned long long* tickets = nullptr;  // [2] zero between launches: next segment chunk, warps done
};

// Segments with n <= kBatchSmallN decode segment-resident (svb_batch3.cu): their worst-case
// stream (ceil(n/4) + 4n bytes) fits one ring item; longer ones take the tile pipeline.
constexpr uint32_t kBatchSmallN = 1920;

cudaError_t launch_decode_batch(const bcgpu_decode_segment* segs, uint64_t nseg, const uint8_t* in, uint32_t* out,
                                int delta, const BatchArgs& ba, cudaStream_t stream);
cudaError_t launch_encode_batch(const bcgpu_encode_segment* segs, uint64_t nseg, const uint32_t* in, uint8_t* out,
                                uint64_t* out_lens, int delta, const BatchArgs& ba, cudaStream_t stream);
cudaError_t launch_sizes_batch(const bcgpu_encode_segment* segs, uint64_t nseg, const uint32_t* in,
                               uint64_t* out_lens, int delta, const BatchArgs& ba, cudaStream_t stream);

// warp-pipelined batch decode (svb_batch2.cu)
cudaError_t launch_decode_batch2(const bcgpu_decode_segment* segs, uint64_t nseg, const uint8_t* in, uint32_t* out,
                                 int delta, const BatchArgs& ba, cudaStream_t stream);

// segment-resident batch decode of the short segments (svb_batch3.cu)
cudaError_t launch_decode_batch3(const bcgpu_decode_segment* segs, uint64_t nseg, const uint8_t* in, uint32_t* out,
                                 int delta, const BatchArgs& ba, cudaStream_t stream);

// sizes: the size-only pass (no output; out may be null)
cudaError_t launch_encode_batch3(const bcgpu_encode_segment* segs, uint64_t nseg, const uint32_t* in, uint8_t* out,
                                 uint64_t* out_lens, int delta, const BatchArgs& ba, cudaStream_t stream,
                                 bool sizes = false);

// host-buffer batches (svb_batch_host.cu): one CTA per piece of segments [s0, s0 + m)
cudaError_t launch_batch_encode_describe(const uint32_t* seg_n, const uint32_t* seg_prev, uint64_t s0, uint32_t m,
                                         uint64_t elem_base, bcgpu_encode_segment* es, cudaStream_t stream);
cudaError_t launch_batch_pack(const uint64_t* sizes, uint64_t s0, uint32_t m, bcgpu_encode_segment* es,
                              uint64_t* out_offsets, unsigned long long* running, cudaStream_t stream);
cudaError_t launch_batch_decode_describe(const uint32_t* seg_n, const uint32_t* seg_base, const uint64_t* in_offsets,
                                         uint64_t s0, uint32_t m, uint64_t elem_base, bcgpu_decode_segment* ds,
                                         cudaStream_t stream);

// Control bytes per look-back tile of the block-offsets kernel.
constexpr uint32_t kOffsetsTileGroups = 2048;

}  // namespace bcgpu
