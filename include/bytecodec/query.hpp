// bytecodec/query.hpp -- seek / select directly on a compressed delta-coded buffer
// (module stream_query; the reference's src/query.cpp has no header).
// Stream VByte only (other codecs: errc::unsupported).  The buffer must be delta-coded
// (the logical sequence is the prefix sums of the payload, base 0) and, for seek,
// non-decreasing.  The batched forms run every query on the GPU in one call; none of them
// decodes the whole stream (a metadata pass of 8 B per 1024 integers, then one sub-tile per
// query).
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>
#include <vector>

#include "bytecodec/codec.hpp"

namespace bytecodec {

struct seek_result {
    size_t index;    // position in the logical sequence
    uint32_t value;  // the first value >= target
};

// first value >= target (ties: the lowest index), or nullopt when target exceeds the last value
std::optional<seek_result> seek(const encoded_buffer& buf, uint32_t target);
// the i-th logical value; errc::out_of_range unless i < buf.count
uint32_t select(const encoded_buffer& buf, size_t i);

std::vector<std::optional<seek_result>> seek(const encoded_buffer& buf, std::span<const uint32_t> targets);
std::vector<uint32_t> select(const encoded_buffer& buf, std::span<const size_t> indices);

}  // namespace bytecodec
