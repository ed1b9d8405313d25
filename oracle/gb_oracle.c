/*
 * gb_oracle.c -- CPU restatement of varint-GB; test infrastructure only (gb_oracle.h).
 * A plain sequential walk: group k's control byte follows group k-1's data
 * (the data dependency that keeps the format scalar).
 */
#include "gb_oracle.h"

#include <string.h>

#include "svb_oracle.h"

/* codec.hpp:70-72 byte_length, as svbo_byte_length */
static uint32_t blen(uint32_t x) { return x < (1u << 8) ? 1u : x < (1u << 16) ? 2u : x < (1u << 24) ? 3u : 4u; }

size_t gbo_compressed_size(const uint32_t *in, size_t n) {
    size_t s = (n + 3) / 4;
    for (size_t i = 0; i < n; ++i) s += blen(in[i]);
    return s;
}

/* ceil(N/4) blocks, each a control byte then the little-endian bytes of
 * its integers; a final incomplete block stores only its r integers, unused fields 0 */
size_t gbo_encode(const uint32_t *in, size_t n, uint8_t *out) {
    size_t pos = 0;
    for (size_t g = 0; g < n; g += 4) {
        const size_t k = n - g < 4 ? n - g : 4;
        const size_t cpos = pos++;
        uint8_t c = 0;
        for (size_t i = 0; i < k; ++i) {
            const uint32_t x = in[g + i], l = blen(x);
            c |= (uint8_t)((l - 1) << (2 * i));
            for (uint32_t b = 0; b < l; ++b) out[pos++] = (uint8_t)(x >> (8 * b));
        }
        out[cpos] = c;
    }
    return pos;
}

const uint8_t *gbo_decode_group_general(uint8_t control, const uint8_t *data, const uint8_t *end, size_t k,
                                        uint32_t *out) {
    for (size_t i = 0; i < k; ++i) {
        const uint32_t l = ((control >> (2 * i)) & 3u) + 1u;
        if ((size_t)(end - data) < l) return NULL;
        uint32_t x = 0;
        for (uint32_t b = 0; b < l; ++b) x |= (uint32_t)data[b] << (8 * b);
        out[i] = x;
        data += l;
    }
    return data;
}

int gbo_decode(const uint8_t *in, size_t in_len, size_t n, int delta, uint32_t base, uint32_t *out,
               uint32_t *last, int fast) {
    const uint8_t *p = in, *end = in + in_len;
    uint32_t run = base;
    for (size_t g = 0; g < n; g += 4) {
        const size_t k = n - g < 4 ? n - g : 4;
        if (p >= end) return SVBO_TRUNCATED;
        const uint8_t c = *p++;
        if (fast && c == 0 && k == 4 && end - p >= 4) {
            /* all-small fast path: four one-byte integers */
            out[g] = p[0];
            out[g + 1] = p[1];
            out[g + 2] = p[2];
            out[g + 3] = p[3];
            p += 4;
        } else {
            p = gbo_decode_group_general(c, p, end, k, out + g);
            if (!p) return SVBO_TRUNCATED;
        }
        if (delta)
            for (size_t i = 0; i < k; ++i) out[g + i] = run += out[g + i];
    }
    if (p != end) return SVBO_TRAILING_BYTES;
    if (last) *last = delta ? run : 0;
    return SVBO_OK;
}
