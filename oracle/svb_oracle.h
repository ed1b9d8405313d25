/*
 * svb_oracle.h -- CPU restatement of the Stream VByte hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it.  The product path (paper_1709_08990_b200/) has
 * no CPU fallback and never links this.
 *
 * The reference (/root/reference/proj) is headers-only: every src/NAME.cpp the
 * build lists is missing, so nothing of it can be compiled or
 * run.  This file restates its algorithm from
 *   - proj/core/include/bytecodec/codec.hpp:69-72      (byte_length)
 *   - proj/core/include/bytecodec/stream_vbyte.hpp:15-54 (layout, tables, API)
 *   - SPEC.md:270-351 (codec_streamvbyte), SPEC.md:353-402 (delta)
 *   - PAPER.md:325-384 (format, Fig. 4 decode), PAPER.md:112-117 (prefix sum)
 * and is pinned against the SPEC golden vectors plus the reference headers'
 * own inline functions (tests/golden/, see oracle/pin_ref_inline.sh).
 *
 * Two independent decoders are kept and cross-checked:
 *   O1  svbo_*        naive per-integer loop ("scalar-loop oracle")
 *   O2  svbo_ssse3_*  the paper's table-driven pshufb decoder
 *                     with the four-zero-control fast path and the scalar tail.
 */
#ifndef SVB_ORACLE_H
#define SVB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: same numbering as bcgpu_status in include/bcgpu/bcgpu.h. */
#define SVBO_OK 0
#define SVBO_TRUNCATED 1      /* errc::truncated      codec.hpp:30 */
#define SVBO_TRAILING_BYTES 2 /* errc::trailing_bytes codec.hpp:31 */

/* codec.hpp:70-72 */
uint32_t svbo_byte_length(uint32_t x);
/* stream_vbyte.hpp:34 */
size_t svbo_control_bytes(size_t n);
/* stream_vbyte.hpp:24-32: length[256], shuffle[256][16] (fill 0xFF, :22) */
void svbo_tables(uint8_t length[256], uint8_t shuffle[256][16]);

/* Exact compressed size (SPEC.md:336 size identity); prev-seeded delta when delta!=0. */
size_t svbo_compressed_size(const uint32_t *in, size_t n, int delta, uint32_t prev);

/* O1 encoder (stream_vbyte.hpp:36).  delta!=0 applies
 * delta_encode seeded with prev first (prev=0 is the
 * reference's encode(..., true), the prev-seeded form is extension E2).
 * out must hold svbo_control_bytes(n) + 4n bytes.  Returns bytes written. */
size_t svbo_encode(const uint32_t *in, size_t n, int delta, uint32_t prev, uint8_t *out);

/* O1 decoder (stream_vbyte.hpp:38,41-42).  Returns SVBO_* status; on
 * delta!=0 writes the last reconstructed value (base for n==0) to *last. */
int svbo_decode(const uint8_t *in, size_t in_len, size_t n, int delta, uint32_t base,
                uint32_t *out, uint32_t *last);

/* O2 decoder: paper Fig. 4 + zero fast path + scalar tail. */
int svbo_ssse3_decode(const uint8_t *in, size_t in_len, size_t n, int delta, uint32_t base,
                      uint32_t *out, uint32_t *last);
/* The paper's timing mode: O2 decode, single thread, into the
 * reused 4096-integer buffer buf; *check = sum of every 4096-block's last integer mod 2^64. */
int svbo_paper_decode(const uint8_t *in, size_t in_len, size_t n, int delta, uint32_t base, uint32_t *buf,
                      uint64_t *check);
/* 1 when the O2 decoder was compiled with SSSE3, 0 when it runs its scalar twin. */
int svbo_ssse3_available(void);

/* delta: forward transform mod 2^32 and prefix sum. */
void svbo_delta_encode(const uint32_t *in, size_t n, uint32_t prev, uint32_t *out);
uint32_t svbo_prefix_sum(const uint32_t *in, size_t n, uint32_t base, uint32_t *out);
/* The 4-lane block step: shift-by-1 add, shift-by-2 add, broadcast base. */
void svbo_prefix_sum4(const uint32_t in[4], uint32_t base, uint32_t out[4]);

/* stream_vbyte.hpp:48-49: data-region offset of each block (exclusive scan of length[c]). */
void svbo_block_data_offsets(const uint8_t *in, size_t n, uint64_t *offsets);
/* stream_vbyte.hpp:53-54: decode block k in isolation; returns integers in the block. */
size_t svbo_decode_block(const uint8_t *in, size_t in_len, size_t n, size_t block,
                         size_t data_offset, uint32_t out[4]);

/* ---- CPU reference arm (bench.py --impl reference / cpu_baseline) ----
 * Multi-threaded over contiguous chunks with nthreads pthreads.  These are
 * still the paper's single-thread kernels (O2 decode, O1 encode) run on
 * independent chunks; the chunk seams are stitched so the output is the one
 * canonical stream (encode: size pass + scan + write pass; delta decode:
 * ctrl-scan for offsets, per-chunk decode with base 0, carry fix-up pass). */
size_t svbo_mt_encode(const uint32_t *in, size_t n, int delta, uint32_t prev, uint8_t *out,
                      int nthreads);
int svbo_mt_decode(const uint8_t *in, size_t in_len, size_t n, int delta, uint32_t base,
                   uint32_t *out, uint32_t *last, int nthreads);

/* Segmented batch (chained-chunk contract codec.hpp:87-90). */
typedef struct {
    uint64_t src_offset; /* byte offset of the segment's SVB stream */
    uint64_t src_bytes;  /* its length */
    uint64_t dst_offset; /* element offset of its first decoded integer */
    uint32_t n;
    uint32_t prev;
} svbo_decode_segment;

typedef struct {
    uint64_t src_offset;   /* element offset of the segment's first value */
    uint64_t dst_capacity; /* bytes available at dst_offset */
    uint64_t dst_offset;   /* byte offset of the segment's SVB stream */
    uint32_t n;
    uint32_t prev;
} svbo_encode_segment;

int svbo_decode_batch(const svbo_decode_segment *segs, size_t nseg, const uint8_t *in,
                      uint32_t *out, int delta, int nthreads);
/* svbo_paper_decode over every segment of a batch, one thread, one reused buffer. */
int svbo_paper_decode_batch(const svbo_decode_segment *segs, size_t nseg, const uint8_t *in, int delta,
                            uint32_t *buf, uint64_t *check);
int svbo_encode_batch(const svbo_encode_segment *segs, size_t nseg, const uint32_t *in,
                      uint8_t *out, uint64_t *out_lens, int delta, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
