// bytecodec/container.hpp -- the 14-byte "SVB1" file container (
// the reference declares no header for it: its src/container.cpp is missing).
// write: header (magic, codec tag, flags bit 0 = delta, LE32 count, LE32 payload
// length) then the payload.  read: validates magic, codec tag, reserved flags, source
// length and -- for Stream VByte -- the payload length against the size identity;
// errors are distinct codec_errors (bad_magic, unknown_codec, reserved_flags,
// truncated / trailing_bytes, length_mismatch; unsupported for the other codecs).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "bytecodec/codec.hpp"

namespace bytecodec {

std::vector<uint8_t> write_container(const encoded_buffer& buf);
encoded_buffer read_container(std::span<const uint8_t> src);

}  // namespace bytecodec
