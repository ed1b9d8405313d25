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
    unsigned long long* ticket;    // monotonically increasing tile ticket
    unsigned long long ticket_base;
    uint32_t epoch;
    uint32_t num_tiles;
    unsigned long long* status;    // [epoch:32 | bcgpu_status:32] of the last call
};

// Launchers (return cudaError_t of the launch).
cudaError_t launch_decode(const uint8_t* in, uint64_t in_len, uint64_t n, int delta, uint32_t base, uint32_t* out,
                          uint32_t* d_last, const LookbackArgs& lb, cudaStream_t stream);
cudaError_t launch_encode(const uint32_t* in, uint64_t n, int delta, uint32_t prev, uint8_t* out,
                          uint64_t* d_out_len, const LookbackArgs& lb, cudaStream_t stream);
cudaError_t launch_block_offsets(const uint8_t* in, uint64_t n, uint64_t* d_offsets, const LookbackArgs& lb,
                                 cudaStream_t stream);

cudaError_t launch_decode_blocks(const uint8_t* in, uint64_t in_len, uint64_t n, const uint64_t* blocks,
                                 const uint64_t* offsets, uint64_t nblocks, uint32_t* out, uint32_t* counts,
                                 cudaStream_t stream);

struct BatchArgs {
    unsigned long long* status;  // [epoch:32 | bcgpu_status:32]
    uint32_t epoch;
    int warp_grid;               // CTAs for the warp-per-segment kernel
    int cta_grid;                // CTAs for the CTA-per-segment kernel
};

// Segments with n <= warp_max go to the warp-per-segment kernel, larger ones
// to the CTA-per-segment kernel; either launch is skipped when the hint says
// it has no work.
cudaError_t launch_decode_batch(const bcgpu_decode_segment* segs, uint64_t nseg, const uint8_t* in, uint32_t* out,
                                int delta, uint32_t max_seg_n, const BatchArgs& ba, cudaStream_t stream,
                                int* launches);
cudaError_t launch_encode_batch(const bcgpu_encode_segment* segs, uint64_t nseg, const uint32_t* in, uint8_t* out,
                                uint64_t* out_lens, int delta, uint32_t max_seg_n, const BatchArgs& ba,
                                cudaStream_t stream, int* launches);
cudaError_t launch_sizes_batch(const bcgpu_encode_segment* segs, uint64_t nseg, const uint32_t* in,
                               uint64_t* out_lens, int delta, const BatchArgs& ba, cudaStream_t stream);

// Occupancy (CTAs per SM) of each kernel family, for grid sizing.
int occupancy_decode_batch_cta();
int occupancy_decode_batch_warp();
int occupancy_encode_batch_cta();
int occupancy_encode_batch_warp();

constexpr uint32_t kWarpSegmentMax = 4096;  // segments up to this many ints: warp-per-segment

}  // namespace bcgpu
