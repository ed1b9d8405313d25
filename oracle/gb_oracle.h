/*
 * gb_oracle.h -- CPU restatement of varint-GB.
 *
 * TEST INFRASTRUCTURE ONLY (see svb_oracle.h): only tests/, smoke() and
 * bench.py's reference legs may load it; the product never links it.
 *
 * The reference ships only the header (proj/core/include/bytecodec/varint_gb.hpp:14-31);
 * src/varint_gb.cpp is missing.  Restated from
 *   - varint_gb.hpp:14-17   format: control byte, field i = byte_length(x_i) - 1,
 *                           integer 0 in the two least-significant bits, an
 *                           incomplete final group with zero unused fields and no
 *                           data bytes for absent integers
 *   - SPEC.md:164-214       module codec_varintgb (examples :178-181, :188-191;
 *                           errors truncated / trailing :186; all-small fast path :185)
 *   - PAPER.md §3 (varint-GB) as quoted by SPEC.md
 * Pinned by the SPEC examples (tests/golden/gb_spec_vectors.json).
 */
#ifndef GB_ORACLE_H
#define GB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* exact encoded size: ceil(n/4) control bytes + sum of byte lengths */
size_t gbo_compressed_size(const uint32_t *in, size_t n);

/* varint_gb.hpp:19 gb_encode; out must hold ceil(n/4) + 4n bytes.  Returns bytes written. */
size_t gbo_encode(const uint32_t *in, size_t n, uint8_t *out);

/* varint_gb.hpp:21-25 gb_decode / gb_decode_delta.  Returns SVBO_OK / SVBO_TRUNCATED /
 * SVBO_TRAILING_BYTES (svb_oracle.h).  delta != 0: out is the prefix sum seeded with base
 * and *last the final value (base for n == 0).  fast != 0 takes the all-small path for
 * control byte 0; fast == 0 decodes every group field by field. */
int gbo_decode(const uint8_t *in, size_t in_len, size_t n, int delta, uint32_t base, uint32_t *out,
               uint32_t *last, int fast);

/* varint_gb.hpp:30-31 detail::gb_decode_group_general: decode the k (1..4) integers of one
 * group with control byte `control` from data..end; returns the byte after the group, or
 * NULL when the group runs past end. */
const uint8_t *gbo_decode_group_general(uint8_t control, const uint8_t *data, const uint8_t *end, size_t k,
                                        uint32_t *out);

#ifdef __cplusplus
}
#endif
#endif
