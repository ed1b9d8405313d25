// bytecodec/stream_vbyte.hpp -- B200-native drop-in for the reference's Stream
// VByte codec (reference: proj/core/include/bytecodec/stream_vbyte.hpp).
//
// Layout (unchanged, byte-exact): ceil(n/4) control bytes -- integer 4k+i in
// bits 2i..2i+1 of control byte k, holding byte_length-1 -- followed by all
// data bytes little-endian, no header, no padding.
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <vector>

#include "bytecodec/codec.hpp"

namespace bytecodec {

// reference stream_vbyte.hpp:21-22
inline constexpr uint8_t svb_shuffle_fill = 0xFF;

// reference stream_vbyte.hpp:24-29
struct decode_tables {
    std::array<uint8_t, 256> length;
    std::array<std::array<uint8_t, 16>, 256> shuffle;
};

// reference stream_vbyte.hpp:31-32 (the GPU kernels derive lengths arithmetically;
// the tables are kept for API parity and are built once, thread-safely).
const decode_tables& svb_tables();

// reference stream_vbyte.hpp:34
inline size_t svb_control_bytes(size_t n) { return (n + 3) / 4; }

// reference stream_vbyte.hpp:36
std::vector<uint8_t> svb_encode(std::span<const uint32_t> values);

// reference stream_vbyte.hpp:38-39
void svb_decode(std::span<const uint8_t> bytes, size_t n, uint32_t* out);
std::vector<uint32_t> svb_decode(std::span<const uint8_t> bytes, size_t n);

// reference stream_vbyte.hpp:41-42
uint32_t svb_decode_delta(std::span<const uint8_t> bytes, size_t n, uint32_t base, uint32_t* out);

// Extension E2: delta encode seeded with prev = x_{-1}.
// svb_encode_delta(v, 0) == encode(codec_id::stream_vbyte, v, true).bytes.
std::vector<uint8_t> svb_encode_delta(std::span<const uint32_t> values, uint32_t prev);

// reference stream_vbyte.hpp:44-46: append one integer to the payload, keeping the
// buffer byte-identical to a one-shot svb_encode of the extended sequence.
// On a delta buffer `value` is the next payload integer (the next delta).
void svb_append(encoded_buffer& buf, uint32_t value);

// reference stream_vbyte.hpp:48-49
std::vector<size_t> svb_block_data_offsets(std::span<const uint8_t> bytes, size_t n);

// reference stream_vbyte.hpp:51-54
size_t svb_decode_block(std::span<const uint8_t> bytes, size_t n, size_t block, size_t data_offset,
                        uint32_t out[4]);

// Extension: the chained-chunk contract (reference codec.hpp:87-90, one
// decode_payload_delta call per chunk with base = the previous chunk's last value;
// SPEC.md:555) for a whole batch in one GPU call.  Segment s holds seg_n[s] of the
// concatenated values; its stream is bytes[offsets[s], offsets[s+1]).
struct svb_batch {
    std::vector<uint8_t> bytes;
    std::vector<uint64_t> offsets;  // seg_n.size() + 1 entries
};
// seg_prev: each segment's delta base (empty = all 0); delta = false encodes plainly.
svb_batch svb_encode_batch(std::span<const uint32_t> values, std::span<const uint32_t> seg_n,
                           std::span<const uint32_t> seg_prev, bool delta = true);
// out holds sum(seg_n) integers; returns every segment's last value (its base when empty).
std::vector<uint32_t> svb_decode_batch(std::span<const uint8_t> bytes, std::span<const uint64_t> offsets,
                                       std::span<const uint32_t> seg_n, std::span<const uint32_t> seg_base,
                                       uint32_t* out, bool delta = true);

}  // namespace bytecodec
