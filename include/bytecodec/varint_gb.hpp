// bytecodec/varint_gb.hpp -- B200-native drop-in for the reference's varint-GB codec
// (reference: proj/core/include/bytecodec/varint_gb.hpp:14-31).
//
// Layout (byte-exact): per group of four integers a control byte -- field i (integer
// i in bits 2i..2i+1) = byte_length(x_i) - 1 -- then the group's data bytes, little-
// endian.  A final incomplete group has zero unused fields and no data bytes for the
// absent integers.  Encode and decode run on the GPU (paper_1709_08990_b200/csrc/svb_gb.cu).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "bytecodec/codec.hpp"

namespace bytecodec {

// reference varint_gb.hpp:19
std::vector<uint8_t> gb_encode(std::span<const uint32_t> values);

// reference varint_gb.hpp:21-22: truncated / trailing_bytes throw codec_error
void gb_decode(std::span<const uint8_t> bytes, size_t n, uint32_t* out);
std::vector<uint32_t> gb_decode(std::span<const uint8_t> bytes, size_t n);

// reference varint_gb.hpp:24-25: fused decode + prefix sum seeded with base; returns
// the last value (base when n == 0)
uint32_t gb_decode_delta(std::span<const uint8_t> bytes, size_t n, uint32_t base, uint32_t* out);

// The delta transform seeded with prev, then gb_encode: gb_encode_delta(v, 0) ==
// encode(codec_id::varint_gb, v, true).bytes.
std::vector<uint8_t> gb_encode_delta(std::span<const uint32_t> values, uint32_t prev);

namespace detail {
// reference varint_gb.hpp:30-31: one group (k = 1..4 integers) decoded field by field,
// without the all-small fast path; returns the byte after the group, or nullptr when the
// group runs past end.  A host-side helper for checking the fast path.
const uint8_t* gb_decode_group_general(uint8_t control, const uint8_t* data, const uint8_t* end, size_t k,
                                       uint32_t* out);
}  // namespace detail

}  // namespace bytecodec
