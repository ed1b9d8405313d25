// svb_format.cpp -- host-side format plumbing around the GPU codecs:
// svb_append (reference proj/core/include/bytecodec/stream_vbyte.hpp:44-46)
// and the 14-byte "SVB1" container for Stream VByte and varint-GB payloads.  Both are byte manipulation of a
// single stream on the host -- the reference does them on the host too -- so they never
// touch the device and need no context.
#include <cstdint>
#include <cstring>

#include "bcgpu/bcgpu.h"

namespace {

inline uint32_t blen(uint32_t x) { return x < (1u << 8) ? 1u : x < (1u << 16) ? 2u : x < (1u << 24) ? 3u : 4u; }

// sum of the four 2-bit fields + 4 (the data bytes of one full control byte)
inline uint32_t ctrl_len(uint32_t c) { return 4u + (c & 3u) + ((c >> 2) & 3u) + ((c >> 4) & 3u) + (c >> 6); }

// data bytes the control stream of an n-integer stream declares
uint64_t svb_declared_data(const uint8_t* ctrl, uint64_t n) {
    const uint64_t full = n / 4;
    uint64_t d = 0;
    for (uint64_t k = 0; k < full; ++k) d += ctrl_len(ctrl[k]);
    const uint32_t r = (uint32_t)(n & 3);
    if (r) {
        const uint32_t c = ctrl[full];
        for (uint32_t i = 0; i < r; ++i) d += ((c >> (2 * i)) & 3u) + 1u;
    }
    return d;
}

// varint-GB (varint_gb.hpp:14-17): the group chain's length for n integers, or
// UINT64_MAX when a control byte lies at or past len (the payload cannot hold them)
uint64_t gb_declared_length(const uint8_t* p, uint64_t len, uint64_t n) {
    uint64_t pos = 0;
    for (uint64_t g = 0; g < n; g += 4) {
        if (pos >= len) return UINT64_MAX;
        const uint32_t c = p[pos], k = n - g < 4 ? (uint32_t)(n - g) : 4u;
        pos += 1;
        for (uint32_t i = 0; i < k; ++i) pos += ((c >> (2 * i)) & 3u) + 1u;
    }
    return pos;
}

constexpr uint8_t kMagic[4] = {'S', 'V', 'B', '1'};

inline void put_le32(uint8_t* p, uint32_t v) {
    p[0] = (uint8_t)v;
    p[1] = (uint8_t)(v >> 8);
    p[2] = (uint8_t)(v >> 16);
    p[3] = (uint8_t)(v >> 24);
}
inline uint32_t get_le32(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

}  // namespace

extern "C" {

int bcgpu_svb_payload_length(const uint8_t* bytes, size_t len, size_t n, size_t* expect) {
    if (!expect || (len && !bytes)) return BCGPU_ERR_INVALID_ARGUMENT;
    const uint64_t nctrl = ((uint64_t)n + 3) / 4;
    if (len < nctrl) return BCGPU_ERR_TRUNCATED;
    *expect = (size_t)(nctrl + svb_declared_data(bytes, n));
    return BCGPU_OK;
}

int bcgpu_svb_append(uint8_t* buf, size_t len, size_t cap, size_t n, uint32_t value, size_t* new_len) {
    if (!new_len || (len && !buf) || (!buf && cap)) return BCGPU_ERR_INVALID_ARGUMENT;
    if (n >= 0xFFFFFFFFull) return BCGPU_ERR_OUT_OF_RANGE;  // encoded_buffer::count is 32-bit
    size_t expect = 0;
    const int st = bcgpu_svb_payload_length(buf, len, n, &expect);
    if (st) return st;
    if (len < expect) return BCGPU_ERR_TRUNCATED;
    if (len > expect) return BCGPU_ERR_TRAILING_BYTES;
    const uint32_t l = blen(value);
    const size_t nctrl = (n + 3) / 4;
    const bool new_ctrl = (n & 3) == 0;
    const size_t need = len + l + (new_ctrl ? 1 : 0);
    if (need > cap || !buf) return BCGPU_ERR_INVALID_ARGUMENT;
    size_t end = len;
    if (new_ctrl) {
        // a new control byte goes at offset nctrl: the data region moves up one byte
        std::memmove(buf + nctrl + 1, buf + nctrl, len - nctrl);
        buf[nctrl] = (uint8_t)(l - 1);
        end = len + 1;
    } else {
        buf[nctrl - 1] = (uint8_t)(buf[nctrl - 1] | ((l - 1) << (2 * (n & 3))));
    }
    for (uint32_t b = 0; b < l; ++b) buf[end + b] = (uint8_t)(value >> (8 * b));
    *new_len = end + l;
    return BCGPU_OK;
}

int bcgpu_container_write(uint8_t codec, int delta, size_t count, const uint8_t* payload, size_t payload_len,
                          uint8_t* out, size_t cap, size_t* out_len) {
    if (!out_len || (payload_len && !payload) || (!out && cap)) return BCGPU_ERR_INVALID_ARGUMENT;
    if (codec > 3) return BCGPU_ERR_UNKNOWN_CODEC;
    if (count > 0xFFFFFFFFull || payload_len > 0xFFFFFFFFull) return BCGPU_ERR_OUT_OF_RANGE;
    if (cap < BCGPU_CONTAINER_HEADER + payload_len || !out) return BCGPU_ERR_INVALID_ARGUMENT;
    std::memcpy(out, kMagic, 4);
    out[4] = codec;
    out[5] = delta ? 1u : 0u;
    put_le32(out + 6, (uint32_t)count);
    put_le32(out + 10, (uint32_t)payload_len);
    if (payload_len) std::memcpy(out + BCGPU_CONTAINER_HEADER, payload, payload_len);
    *out_len = BCGPU_CONTAINER_HEADER + payload_len;
    return BCGPU_OK;
}

int bcgpu_container_read(const uint8_t* src, size_t len, uint8_t* codec, int* delta, uint32_t* count,
                         size_t* payload_offset, size_t* payload_len) {
    if (!codec || !delta || !count || !payload_offset || !payload_len || (len && !src))
        return BCGPU_ERR_INVALID_ARGUMENT;
    if (len < BCGPU_CONTAINER_HEADER) return BCGPU_ERR_TRUNCATED;
    if (std::memcmp(src, kMagic, 4) != 0) return BCGPU_ERR_BAD_MAGIC;
    if (src[4] > 3) return BCGPU_ERR_UNKNOWN_CODEC;
    if (src[5] & ~1u) return BCGPU_ERR_RESERVED_FLAGS;
    const uint32_t nv = get_le32(src + 6), plen = get_le32(src + 10);
    if (len - BCGPU_CONTAINER_HEADER < plen) return BCGPU_ERR_TRUNCATED;
    if (len - BCGPU_CONTAINER_HEADER > plen) return BCGPU_ERR_TRAILING_BYTES;
    *codec = src[4];
    *delta = src[5] & 1u;
    *count = nv;
    *payload_offset = BCGPU_CONTAINER_HEADER;
    *payload_len = plen;
    // payload length against the codec's size formula: the Stream VByte size
    // identity ceil(N/4) + sum(byte_length) from the control bytes; for varint-GB the same
    // total, found by walking the interleaved group chain.  VByte and varint-G8IU are out
    // of this library's scope and their payloads are not verified
    const uint8_t* pl = src + BCGPU_CONTAINER_HEADER;
    if (src[4] == 3) {
        const uint64_t nctrl = ((uint64_t)nv + 3) / 4;
        if (plen < nctrl || nctrl + svb_declared_data(pl, nv) != plen) return BCGPU_ERR_LENGTH_MISMATCH;
        return BCGPU_OK;
    }
    if (src[4] == 1) return gb_declared_length(pl, plen, nv) == plen ? BCGPU_OK : BCGPU_ERR_LENGTH_MISMATCH;
    return BCGPU_ERR_UNSUPPORTED;
}

}  // extern "C"
