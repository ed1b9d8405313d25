/*
 * bcgpu.h -- C ABI of the B200-native Stream VByte codec (libbytecodec_b200.so).
 *
 * This is the drop-in boundary.  The reference's operator API is C++20
 * (namespace bytecodec, proj/core/include/bytecodec/{codec,stream_vbyte}.hpp);
 * it has no extern "C" surface.  Every entry point below replaces one
 * reference function, cited per declaration, with plain pointers and sizes so
 * any FFI (ctypes, cgo, JNI) can bind it.  The C++ API in
 * include/bytecodec/{codec,stream_vbyte}.hpp is implemented on top of these calls.
 *
 * Two families:
 *   bcgpu_*_host   synchronous, host pointers in and out, full validation and
 *                  the reference's error semantics (codec_error{errc},
 *                  codec.hpp:28-58, mapped to bcgpu_status).  H2D / D2H inside.
 *   bcgpu_*_device stream-ordered, device pointers, no host sync.  Malformed
 *                  input is reported through bcgpu_ctx_sync_status().
 *
 * All integers are uint32, all compressed streams are the reference's
 * canonical layout (stream_vbyte.hpp:15-19): ceil(n/4) control bytes (integer
 * 4k in bits 0-1 of control byte k, field = byte_length-1) then the
 * little-endian data bytes, no header, no padding.
 *
 * Threading: a bcgpu_ctx owns device workspace (look-back status, tile
 * ticket) and must not be used by two host threads or two streams at once.
 * Create one ctx per (thread, device).
 */
#ifndef BCGPU_H
#define BCGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BCGPU_ABI_VERSION 1

/* Status codes.  1..15 mirror bytecodec::errc (codec.hpp:28-47) in order +1;
 * 100+ are GPU-side failures the reference cannot produce. */
typedef enum bcgpu_status {
    BCGPU_OK = 0,
    BCGPU_ERR_TRUNCATED = 1,        /* errc::truncated */
    BCGPU_ERR_TRAILING_BYTES = 2,   /* errc::trailing_bytes */
    BCGPU_ERR_RUN_TOO_LONG = 3,     /* errc::run_too_long      (vbyte only; unused) */
    BCGPU_ERR_VALUE_OVERFLOW = 4,   /* errc::value_overflow    (unused) */
    BCGPU_ERR_OVERSIZED_INTEGER = 5,/* errc::oversized_integer (unused) */
    BCGPU_ERR_COUNT_MISMATCH = 6,   /* errc::count_mismatch */
    BCGPU_ERR_BAD_STREAM_SIZE = 7,  /* errc::bad_stream_size */
    BCGPU_ERR_BAD_MAGIC = 8,
    BCGPU_ERR_UNKNOWN_CODEC = 9,
    BCGPU_ERR_RESERVED_FLAGS = 10,
    BCGPU_ERR_LENGTH_MISMATCH = 11,
    BCGPU_ERR_UNSUPPORTED = 12,     /* errc::unsupported (non-SVB codec_id) */
    BCGPU_ERR_OUT_OF_RANGE = 13,    /* errc::out_of_range (block index, n > 2^32-1) */
    BCGPU_ERR_IO_FAILURE = 14,
    BCGPU_ERR_BAD_CONFIG = 15,
    BCGPU_ERR_INVALID_ARGUMENT = 100, /* null pointer, capacity too small */
    BCGPU_ERR_CUDA = 101,             /* CUDA runtime failure (see bcgpu_last_cuda_error) */
    BCGPU_ERR_NO_DEVICE = 102
} bcgpu_status;

typedef struct bcgpu_ctx bcgpu_ctx;

/* One independent array of a segmented decode batch (chained-chunk contract,
 * codec.hpp:87-90: each segment is decoded with its own base `prev`). */
typedef struct bcgpu_decode_segment {
    uint64_t src_offset; /* byte offset of the segment's SVB stream in the batch input */
    uint64_t src_bytes;  /* its exact length (ctrl + data) */
    uint64_t dst_offset; /* element (uint32) offset of its first decoded integer */
    uint32_t n;          /* integers in the segment */
    uint32_t prev;       /* delta base (ignored when delta == 0) */
} bcgpu_decode_segment;

/* One independent array of a segmented encode batch. */
typedef struct bcgpu_encode_segment {
    uint64_t src_offset;   /* element offset of the segment's first value */
    uint64_t dst_capacity; /* bytes available at dst_offset (>= bcgpu_svb_max_compressed_bytes(n)) */
    uint64_t dst_offset;   /* byte offset of the segment's SVB stream in the batch output */
    uint32_t n;
    uint32_t prev;         /* delta seed x_{-1} (extension E2; 0 == reference encode(...,true)) */
} bcgpu_encode_segment;

/* ---- library / context ------------------------------------------------ */
int bcgpu_abi_version(void);
/* Device index a ctx is bound to; the ctx allocates its workspace lazily.  A ctx
 * carries per-call device state (status word, look-back tags, batch tickets): use
 * it from one host thread and one stream at a time; separate ctxs run concurrently. */
int bcgpu_ctx_create(int device, bcgpu_ctx **out);
int bcgpu_ctx_destroy(bcgpu_ctx *ctx);
/* Synchronise `stream` and return the status of the last *_device call made
 * on ctx (malformed-input detection happens on the device). */
int bcgpu_ctx_sync_status(bcgpu_ctx *ctx, void *stream);
const char *bcgpu_status_string(int status);
const char *bcgpu_last_cuda_error(void);
/* Number of kernel launches this process has issued through the library. */
uint64_t bcgpu_kernel_launch_count(void);

/* ---- sizes (pure functions) -------------------------------------------- */
uint32_t bcgpu_byte_length(uint32_t x);              /* codec.hpp:70-72 */
size_t bcgpu_svb_control_bytes(size_t n);            /* stream_vbyte.hpp:34 */
size_t bcgpu_svb_max_compressed_bytes(size_t n);     /* ceil(n/4) + 4n */
/* decode_tables (stream_vbyte.hpp:24-32): 256 lengths and 256x16 shuffle
 * indices (0xFF = zero byte, :22), generated programmatically. */
void bcgpu_svb_tables(uint8_t length[256], uint8_t shuffle[256][16]);

/* ---- device-pointer, stream-ordered ------------------------------------ */

/* svb_encode (stream_vbyte.hpp:36) / encode_payload (codec.hpp:84); with
 * delta != 0 the prev-seeded delta encode (extension E2; prev = 0 equals
 * encode(stream_vbyte, values, true).bytes, codec.hpp:92-93).  Writes the
 * exact stream length to *d_out_len (device uint64).  out_cap must be at
 * least bcgpu_svb_max_compressed_bytes(n). */
int bcgpu_svb_encode_device(bcgpu_ctx *ctx, const uint32_t *d_in, size_t n, int delta, uint32_t prev,
                            uint8_t *d_out, size_t out_cap, uint64_t *d_out_len, void *stream);

/* svb_decode (stream_vbyte.hpp:38) and, with delta != 0, svb_decode_delta
 * (stream_vbyte.hpp:41-42) / decode_payload_delta (codec.hpp:89-90): the
 * fused decode + prefix sum seeded with base.  d_last (may be NULL) receives
 * the last reconstructed value (base when n == 0). */
int bcgpu_svb_decode_device(bcgpu_ctx *ctx, const uint8_t *d_in, size_t in_len, size_t n, int delta,
                            uint32_t base, uint32_t *d_out, uint32_t *d_last, void *stream);

/* svb_block_data_offsets (stream_vbyte.hpp:48-49): d_offsets[k] = data-region
 * offset of block k, for k < ceil(n/4). */
int bcgpu_svb_block_offsets_device(bcgpu_ctx *ctx, const uint8_t *d_in, size_t in_len, size_t n,
                                   uint64_t *d_offsets, void *stream);

/* svb_decode_block (stream_vbyte.hpp:51-54), batched: block d_blocks[i] whose
 * data starts at data-region offset d_offsets[i] -> d_out[4i..4i+3], the
 * number of integers in that block -> d_counts[i] (0 when the block index is
 * out of range).  Bytes past in_len read as zero (no over-read). */
int bcgpu_svb_decode_blocks_device(bcgpu_ctx *ctx, const uint8_t *d_in, size_t in_len, size_t n,
                                   const uint64_t *d_blocks, const uint64_t *d_offsets, size_t nblocks,
                                   uint32_t *d_out, uint32_t *d_counts, void *stream);

/* Segmented batches: every segment independent (own base), no collective.
 * max_seg_n bounds every segment's n (0 = unknown).  Decode: segments with
 * n <= 1920 are decoded segment-resident, longer ones by the tile pipeline,
 * which is not launched when 0 < max_seg_n <= 1920 (a longer segment then
 * fails with BCGPU_ERR_INVALID_ARGUMENT).  Encode codes every length and does
 * not use the bound. */
int bcgpu_svb_decode_batch_device(bcgpu_ctx *ctx, const bcgpu_decode_segment *d_segs, size_t nseg,
                                  const uint8_t *d_in, uint32_t *d_out, int delta, uint32_t max_seg_n,
                                  void *stream);
/* Writes each segment's exact stream length to d_out_lens[seg]. */
int bcgpu_svb_encode_batch_device(bcgpu_ctx *ctx, const bcgpu_encode_segment *d_segs, size_t nseg,
                                  const uint32_t *d_in, uint8_t *d_out, uint64_t *d_out_lens, int delta,
                                  uint32_t max_seg_n, void *stream);
/* Size-only pass: exact compressed length of every segment (no output written),
 * so callers can pack a batch contiguously (exclusive scan -> dst_offset). */
int bcgpu_svb_encoded_sizes_batch_device(bcgpu_ctx *ctx, const bcgpu_encode_segment *d_segs, size_t nseg,
                                         const uint32_t *d_in, uint64_t *d_out_lens, int delta,
                                         uint32_t max_seg_n, void *stream);

/* ---- host-pointer, synchronous (the reference's call semantics) -------- */

/* svb_encode / svb_encode_delta: writes the stream to out (capacity out_cap
 * >= bcgpu_svb_max_compressed_bytes(n)), its exact length to *out_len. */
int bcgpu_svb_encode_host(bcgpu_ctx *ctx, const uint32_t *values, size_t n, int delta, uint32_t prev,
                          uint8_t *out, size_t out_cap, size_t *out_len);
/* svb_decode / svb_decode_delta: validates the stream (truncated /
 * trailing_bytes), decodes n integers into out, writes the last value to
 * *last (may be NULL). */
int bcgpu_svb_decode_host(bcgpu_ctx *ctx, const uint8_t *bytes, size_t len, size_t n, int delta,
                          uint32_t base, uint32_t *out, uint32_t *last);
/* svb_decode_block for nblocks (block, offset) pairs held in host memory
 * (size_t arrays, as the reference signature takes them).  A block index
 * >= ceil(n/4) returns OUT_OF_RANGE; a block whose control or data bytes lie
 * past len returns TRUNCATED (the _device variant writes count 0 for both). */
int bcgpu_svb_decode_blocks_host(bcgpu_ctx *ctx, const uint8_t *bytes, size_t len, size_t n,
                                 const size_t *blocks, const size_t *offsets, size_t nblocks,
                                 uint32_t *out, uint32_t *counts);
/* svb_block_data_offsets into a host array of ceil(n/4) entries. */
/* ---- segmented batches through host memory ------------------------------
 * The chained-chunk contract of the reference (codec.hpp:87-90,
 * decode_payload_delta(codec, bytes, n, base, out) once per chunk)
 * for a whole batch in one call.  Segment s has seg_n[s] integers; the values
 * of all segments are concatenated in `values` / `out`.  Streams are packed
 * back to back: segment s occupies bytes [offsets[s], offsets[s+1]).  The call
 * moves the batch in pieces of whole segments so host->device copies, kernels
 * and device->host copies overlap (pinned host buffers give full overlap).
 *
 * encode: seg_prev[s] seeds segment s's delta transform (NULL = all 0; ignored
 * when delta == 0).  Writes the packed streams to out (out_cap bytes; the sum of
 * bcgpu_svb_max_compressed_bytes(seg_n[s]) always suffices, INVALID_ARGUMENT
 * when the packed total exceeds out_cap) and nseg + 1 offsets to out_offsets
 * (out_offsets[nseg] = total length). */
int bcgpu_svb_encode_batch_host(bcgpu_ctx *ctx, const uint32_t *values, const uint32_t *seg_n,
                                const uint32_t *seg_prev, size_t nseg, int delta, uint8_t *out,
                                size_t out_cap, uint64_t *out_offsets);
/* decode: in_offsets[nseg + 1] non-decreasing, in_offsets[nseg] <= len
 * (TRUNCATED otherwise).  Each segment is validated as svb_decode validates a
 * stream (truncated / trailing_bytes); seg_base[s] is its delta base (NULL = all
 * 0).  last (nseg entries, may be NULL) receives each segment's last value
 * (its base when seg_n[s] == 0), decode_payload_delta's return value. */
int bcgpu_svb_decode_batch_host(bcgpu_ctx *ctx, const uint8_t *bytes, size_t len, const uint64_t *in_offsets,
                                const uint32_t *seg_n, const uint32_t *seg_base, size_t nseg, int delta,
                                uint32_t *out, uint32_t *last);
int bcgpu_svb_block_offsets_host(bcgpu_ctx *ctx, const uint8_t *bytes, size_t len, size_t n,
                                 uint64_t *offsets);

/* ---- batched seek / select over one delta-coded stream ------------------- */
/* (module stream_query; the reference's query.cpp has no header.)
 * The logical sequence is base + the prefix sums of the n payload integers; seek
 * requires it non-decreasing (sorted ids).  seek: for every target, the first index
 * with value >= target (ties: lowest index) and that value; index = n means not
 * found.  select: the value at every index (indices must be < n; the _host variant
 * returns OUT_OF_RANGE otherwise).  The stream is never decoded in full: a metadata
 * pass (control scan + sums: 8 B per 1024 integers), then one warp per query decodes
 * one 1024-integer sub-tile.  Malformed streams are reported as for decode. */
int bcgpu_svb_seek_batch_device(bcgpu_ctx *ctx, const uint8_t *d_in, size_t in_len, size_t n, uint32_t base,
                                const uint32_t *d_targets, size_t q, uint64_t *d_index, uint32_t *d_values,
                                void *stream);
int bcgpu_svb_select_batch_device(bcgpu_ctx *ctx, const uint8_t *d_in, size_t in_len, size_t n, uint32_t base,
                                  const uint64_t *d_idx, size_t q, uint32_t *d_values, void *stream);
int bcgpu_svb_seek_host(bcgpu_ctx *ctx, const uint8_t *bytes, size_t len, size_t n, uint32_t base,
                        const uint32_t *targets, size_t q, uint64_t *index, uint32_t *values);
int bcgpu_svb_select_host(bcgpu_ctx *ctx, const uint8_t *bytes, size_t len, size_t n, uint32_t base,
                          const uint64_t *idx, size_t q, uint32_t *values);

/* ---- varint-GB (reference varint_gb.hpp:14-31) --------- */
/* Groups of four integers, each a control byte (field i = byte_length(x_i) - 1, integer
 * 0 in the low two bits) followed by its data bytes; the final group may be incomplete
 * (zero unused fields, no data bytes for absent integers).  Same size as the Stream
 * VByte encoding of the same integers, so bcgpu_svb_max_compressed_bytes bounds it. */
/* gb_encode (varint_gb.hpp:19); delta != 0 first applies the mod-2^32 delta transform
 * seeded with prev (as codec.hpp:92-93's encode(varint_gb, values, true) does with
 * prev = 0).  d_out holds >= bcgpu_svb_max_compressed_bytes(n) bytes; the exact length
 * goes to *d_out_len (device, may be NULL). */
int bcgpu_gb_encode_device(bcgpu_ctx *ctx, const uint32_t *d_in, size_t n, int delta, uint32_t prev,
                           uint8_t *d_out, size_t out_cap, uint64_t *d_out_len, void *stream);
/* gb_decode / gb_decode_delta (varint_gb.hpp:21-25): validates (truncated /
 * trailing_bytes, reported as for bcgpu_svb_decode_device), decodes n integers; delta
 * adds the prefix sum seeded with base and writes the last value to *d_last (device,
 * may be NULL). */
int bcgpu_gb_decode_device(bcgpu_ctx *ctx, const uint8_t *d_in, size_t in_len, size_t n, int delta, uint32_t base,
                           uint32_t *d_out, uint32_t *d_last, void *stream);
int bcgpu_gb_encode_host(bcgpu_ctx *ctx, const uint32_t *values, size_t n, int delta, uint32_t prev,
                         uint8_t *out, size_t out_cap, size_t *out_len);
int bcgpu_gb_decode_host(bcgpu_ctx *ctx, const uint8_t *bytes, size_t len, size_t n, int delta, uint32_t base,
                         uint32_t *out, uint32_t *last);

/* ---- format plumbing on the host (no device, no ctx) -------------------- */

/* Data + control length the control stream of an n-integer Stream VByte payload
 * declares: ceil(n/4) + sum of byte lengths.  TRUNCATED when
 * len < ceil(n/4). */
int bcgpu_svb_payload_length(const uint8_t *bytes, size_t len, size_t n, size_t *expect);

/* svb_append (reference stream_vbyte.hpp:44-46): appends `value`
 * as integer n of the payload buf[0..len), in place; the result is byte-identical to
 * a one-shot encode of the n+1 integers (a new control byte shifts the data region
 * up by one byte).  cap = capacity of buf (needs len + 5 in the worst case).  The
 * payload is validated first (truncated / trailing_bytes). */
int bcgpu_svb_append(uint8_t *buf, size_t len, size_t cap, size_t n, uint32_t value, size_t *new_len);

/* The 14-byte container: "SVB1", codec tag, flags (bit 0 = delta),
 * LE32 count, LE32 payload_length, then the payload. */
#define BCGPU_CONTAINER_HEADER 14
int bcgpu_container_write(uint8_t codec, int delta, size_t count, const uint8_t *payload, size_t payload_len,
                          uint8_t *out, size_t cap, size_t *out_len);
/* Validates magic (BAD_MAGIC), codec tag (UNKNOWN_CODEC), reserved flags
 * (RESERVED_FLAGS), source length (TRUNCATED / TRAILING_BYTES) and, for Stream
 * VByte, the payload length against the size identity (LENGTH_MISMATCH).  Other
 * known codecs are parsed but return UNSUPPORTED (outside this library). */
int bcgpu_container_read(const uint8_t *src, size_t len, uint8_t *codec, int *delta, uint32_t *count,
                         size_t *payload_offset, size_t *payload_len);

#ifdef __cplusplus
}
#endif
#endif /* BCGPU_H */
