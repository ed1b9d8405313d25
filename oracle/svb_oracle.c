/*
 * svb_oracle.c -- CPU restatement of the Stream VByte hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see svb_oracle.h): the checker for the CUDA path
 * and the timed CPU reference arm.  Never linked into the product.
 *
 * Parity anchors (all paths relative to /root/reference):
 *   byte_length ............ proj/core/include/bytecodec/codec.hpp:69-72
 *   layout ................. proj/core/include/bytecodec/stream_vbyte.hpp:15-19
 *   tables ................. stream_vbyte.hpp:21-32
 *   encode ................. stream_vbyte.hpp:36
 *   decode (+malformed) .... stream_vbyte.hpp:38-39
 *   decode_delta ........... stream_vbyte.hpp:41-42, codec.hpp:87-90
 *   delta / prefix sum ..... SPEC.md:353-402
 *   Fig. 4 block decode .... PAPER.md:357-384
 *   block offsets / block .. stream_vbyte.hpp:48-54
 */
#include "svb_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#if defined(__SSSE3__)
#include <tmmintrin.h>
#define SVBO_HAVE_SSSE3 1
#else
#define SVBO_HAVE_SSSE3 0
#endif

/* ------------------------------------------------------------------ */
/* L0: lengths and tables                                              */
/* ------------------------------------------------------------------ */

/* codec.hpp:70-72 -- len(0)=1. */
uint32_t svbo_byte_length(uint32_t x) {
    if (x < (1u << 8)) return 1;
    if (x < (1u << 16)) return 2;
    if (x < (1u << 24)) return 3;
    return 4;
}

/* stream_vbyte.hpp:34 */
size_t svbo_control_bytes(size_t n) { return (n + 3) / 4; }

/* stream_vbyte.hpp:24-32 / SPEC.md:292-300: generated programmatically. */
void svbo_tables(uint8_t length[256], uint8_t shuffle[256][16]) {
    for (int c = 0; c < 256; ++c) {
        int start = 0;
        for (int i = 0; i < 4; ++i) {
            int len = ((c >> (2 * i)) & 3) + 1;
            for (int b = 0; b < 4; ++b)
                shuffle[c][4 * i + b] = (uint8_t)(b < len ? start + b : 0xFF); /* svb_shuffle_fill, :22 */
            start += len;
        }
        length[c] = (uint8_t)start;
    }
}

static uint8_t g_length[256];
static uint8_t g_shuffle[256][16];
static pthread_once_t g_tables_once = PTHREAD_ONCE_INIT;
static void init_tables(void) { svbo_tables(g_length, g_shuffle); }
static void ensure_tables(void) { pthread_once(&g_tables_once, init_tables); }

/* ------------------------------------------------------------------ */
/* delta                                             */
/* ------------------------------------------------------------------ */

void svbo_delta_encode(const uint32_t *in, size_t n, uint32_t prev, uint32_t *out) {
    for (size_t i = 0; i < n; ++i) {
        uint32_t x = in[i];
        out[i] = x - prev; /* mod 2^32 */
        prev = x;
    }
}

uint32_t svbo_prefix_sum(const uint32_t *in, size_t n, uint32_t base, uint32_t *out) {
    for (size_t i = 0; i < n; ++i) {
        base += in[i];
        out[i] = base;
    }
    return base;
}

/* (3,4,12,1) -> +shift1 -> (3,7,16,13) -> +shift2 -> (3,7,19,20). */
void svbo_prefix_sum4(const uint32_t in[4], uint32_t base, uint32_t out[4]) {
    uint32_t a0 = in[0], a1 = in[1] + in[0], a2 = in[2] + in[1], a3 = in[3] + in[2];
    uint32_t b0 = a0, b1 = a1, b2 = a2 + a0, b3 = a3 + a1;
    out[0] = b0 + base;
    out[1] = b1 + base;
    out[2] = b2 + base;
    out[3] = b3 + base;
}

/* ------------------------------------------------------------------ */
/* O1: naive per-integer loop encoder / decoder                        */
/* ------------------------------------------------------------------ */

size_t svbo_compressed_size(const uint32_t *in, size_t n, int delta, uint32_t prev) {
    size_t total = svbo_control_bytes(n);
    for (size_t i = 0; i < n; ++i) {
        uint32_t x = in[i];
        total += svbo_byte_length(delta ? x - prev : x);
        prev = x;
    }
    return total;
}

/* field i of control byte k = len-1 in bits 2(i mod 4);
 * little-endian data bytes; unused final fields stay 0 (:280). */
size_t svbo_encode(const uint32_t *in, size_t n, int delta, uint32_t prev, uint8_t *out) {
    size_t nctrl = svbo_control_bytes(n);
    uint8_t *ctrl = out;
    uint8_t *data = out + nctrl;
    memset(ctrl, 0, nctrl);
    for (size_t i = 0; i < n; ++i) {
        uint32_t x = in[i];
        uint32_t v = delta ? x - prev : x;
        prev = x;
        uint32_t len = svbo_byte_length(v);
        ctrl[i / 4] |= (uint8_t)((len - 1) << (2 * (i % 4)));
        for (uint32_t b = 0; b < len; ++b) *data++ = (uint8_t)(v >> (8 * b));
    }
    return (size_t)(data - out);
}

/* Sum of data lengths the first n fields of the control stream declare.
 * Unused fields of a final partial control byte are ignored (scalar-tail
 * semantics). */
static uint64_t declared_data_bytes(const uint8_t *ctrl, size_t n) {
    ensure_tables();
    uint64_t total = 0;
    size_t full = n / 4;
    for (size_t k = 0; k < full; ++k) total += g_length[ctrl[k]];
    for (size_t i = full * 4; i < n; ++i) total += ((ctrl[i / 4] >> (2 * (i % 4))) & 3) + 1;
    return total;
}

/* SPEC.md:316 malformed-input mapping: short -> truncated, long -> trailing. */
static int validate(const uint8_t *in, size_t in_len, size_t n) {
    size_t nctrl = svbo_control_bytes(n);
    if (in_len < nctrl) return SVBO_TRUNCATED;
    uint64_t need = nctrl + declared_data_bytes(in, n);
    if (in_len < need) return SVBO_TRUNCATED;
    if (in_len > need) return SVBO_TRAILING_BYTES;
    return SVBO_OK;
}

int svbo_decode(const uint8_t *in, size_t in_len, size_t n, int delta, uint32_t base,
                uint32_t *out, uint32_t *last) {
    int st = validate(in, in_len, n);
    if (st != SVBO_OK) return st;
    const uint8_t *ctrl = in;
    const uint8_t *data = in + svbo_control_bytes(n);
    uint32_t acc = base;
    for (size_t i = 0; i < n; ++i) {
        uint32_t len = ((ctrl[i / 4] >> (2 * (i % 4))) & 3) + 1;
        uint32_t v = 0;
        for (uint32_t b = 0; b < len; ++b) v |= (uint32_t)data[b] << (8 * b);
        data += len;
        if (delta) {
            acc += v;
            v = acc;
        }
        out[i] = v;
    }
    if (last) *last = delta ? acc : (n ? out[n - 1] : base);
    return SVBO_OK;
}

/* ------------------------------------------------------------------ */
/* O2: paper Fig. 4 table decoder                   */
/* ------------------------------------------------------------------ */

int svbo_ssse3_available(void) { return SVBO_HAVE_SSSE3; }

/* Scalar varint-GB-style routine for the tail. */
static const uint8_t *scalar_range(const uint8_t *ctrl, const uint8_t *data, size_t first, size_t count,
                                   int delta, uint32_t *acc, uint32_t *out) {
    for (size_t i = first; i < first + count; ++i) {
        uint32_t len = ((ctrl[i / 4] >> (2 * (i % 4))) & 3) + 1;
        uint32_t v = 0;
        for (uint32_t b = 0; b < len; ++b) v |= (uint32_t)data[b] << (8 * b);
        data += len;
        if (delta) {
            *acc += v;
            v = *acc;
        }
        out[i] = v;
    }
    return data;
}

/* Decode integers [0, n) of a stream whose control bytes start at ctrl and
 * data bytes at data, never reading at or beyond data_end.  Returns the last
 * reconstructed value (delta) or the running base unchanged (plain). */
static uint32_t o2_decode_range_next(const uint8_t *ctrl, const uint8_t *data, const uint8_t *data_end, size_t n,
                                     int delta, uint32_t base, uint32_t *out, const uint8_t **data_next) {
    ensure_tables();
    size_t i = 0;
    uint32_t acc = base;
#if SVBO_HAVE_SSSE3
    __m128i prev = _mm_set1_epi32((int)base);
    const __m128i zero_expand0 = _mm_setr_epi8(0, -1, -1, -1, 1, -1, -1, -1, 2, -1, -1, -1, 3, -1, -1, -1);
    const __m128i zero_expand1 = _mm_setr_epi8(4, -1, -1, -1, 5, -1, -1, -1, 6, -1, -1, -1, 7, -1, -1, -1);
    const __m128i zero_expand2 = _mm_setr_epi8(8, -1, -1, -1, 9, -1, -1, -1, 10, -1, -1, -1, 11, -1, -1, -1);
    const __m128i zero_expand3 = _mm_setr_epi8(12, -1, -1, -1, 13, -1, -1, -1, 14, -1, -1, -1, 15, -1, -1, -1);
#define SVBO_PSUM(x)                                                         \
    do {                                                                     \
        x = _mm_add_epi32(x, _mm_slli_si128(x, 4));                          \
        x = _mm_add_epi32(x, _mm_slli_si128(x, 8));                          \
        x = _mm_add_epi32(x, prev);                                          \
        prev = _mm_shuffle_epi32(x, 0xFF);                                   \
    } while (0)
    while (i + 4 <= n && data + 16 <= data_end) {
        size_t k = i / 4;
        /* four zero control bytes -> 16 one-byte integers */
        uint32_t four;
        memcpy(&four, ctrl + k, 4);
        if (i + 16 <= n && four == 0) {
            __m128i d = _mm_loadu_si128((const __m128i *)data);
            __m128i v0 = _mm_shuffle_epi8(d, zero_expand0);
            __m128i v1 = _mm_shuffle_epi8(d, zero_expand1);
            __m128i v2 = _mm_shuffle_epi8(d, zero_expand2);
            __m128i v3 = _mm_shuffle_epi8(d, zero_expand3);
            if (delta) {
                SVBO_PSUM(v0);
                SVBO_PSUM(v1);
                SVBO_PSUM(v2);
                SVBO_PSUM(v3);
            }
            _mm_storeu_si128((__m128i *)(out + i), v0);
            _mm_storeu_si128((__m128i *)(out + i + 4), v1);
            _mm_storeu_si128((__m128i *)(out + i + 8), v2);
            _mm_storeu_si128((__m128i *)(out + i + 12), v3);
            data += 16;
            i += 16;
            continue;
        }
        uint8_t c = ctrl[k];
        uint8_t C = g_length[c];                                        /* Fig. 4 line 1 */
        __m128i d = _mm_loadu_si128((const __m128i *)data);             /* line 2 */
        __m128i s = _mm_loadu_si128((const __m128i *)g_shuffle[c]);     /* line 3 */
        d = _mm_shuffle_epi8(d, s);                                     /* line 4 */
        if (delta) SVBO_PSUM(d);
        _mm_storeu_si128((__m128i *)(out + i), d);
        data += C;                                                      /* line 5 */
        i += 4;
    }
    if (delta) acc = (uint32_t)_mm_cvtsi128_si32(prev);
#undef SVBO_PSUM
#else
    /* Portable twin of the SIMD loop (same table walk, byte-indexed shuffle). */
    while (i + 4 <= n && data + 16 <= data_end) {
        uint8_t c = ctrl[i / 4];
        uint8_t C = g_length[c];
        uint32_t lane[4];
        for (int l = 0; l < 4; ++l) {
            uint32_t v = 0;
            for (int b = 0; b < 4; ++b) {
                uint8_t idx = g_shuffle[c][4 * l + b];
                v |= (uint32_t)(idx < 16 ? data[idx] : 0) << (8 * b);
            }
            lane[l] = v;
        }
        if (delta) {
            svbo_prefix_sum4(lane, acc, lane);
            acc = lane[3];
        }
        memcpy(out + i, lane, 16);
        data += C;
        i += 4;
    }
#endif
    const uint8_t *dn = scalar_range(ctrl, data, i, n - i, delta, &acc, out);
    if (data_next) *data_next = dn;
    return acc;
}

static uint32_t o2_decode_range(const uint8_t *ctrl, const uint8_t *data, const uint8_t *data_end, size_t n,
                                int delta, uint32_t base, uint32_t *out) {
    return o2_decode_range_next(ctrl, data, data_end, n, delta, base, out, NULL);
}

/* The paper's measurement mode: one thread decodes the stream
 * sequentially into a reused buffer of 4096 integers (half of a 32 KiB L1), so the
 * output stays in L1 and the timing is the decoder's, RAM -> L1.  Same O2 kernel as
 * svbo_ssse3_decode, 4096 integers (1024 control bytes) per call.  *check gets the
 * sum over blocks of each block's last decoded integer, mod 2^64 (so the work
 * cannot be elided and callers can compare it with the expected values, without
 * adding a pass over the buffer to the timed loop). */
int svbo_paper_decode(const uint8_t *in, size_t in_len, size_t n, int delta, uint32_t base, uint32_t *buf,
                      uint64_t *check) {
    int st = validate(in, in_len, n);
    if (st != SVBO_OK) return st;
    const size_t nctrl = svbo_control_bytes(n);
    const uint8_t *data = in + nctrl;
    uint32_t acc = base;
    uint64_t sum = 0;
    for (size_t i = 0; i < n; i += 4096) {
        const size_t m = n - i < 4096 ? n - i : 4096;
        const uint32_t r = o2_decode_range_next(in + i / 4, data, in + in_len, m, delta, acc, buf, &data);
        if (delta) acc = r;
        sum += buf[m - 1];
    }
    if (check) *check = sum;
    return SVBO_OK;
}

int svbo_ssse3_decode(const uint8_t *in, size_t in_len, size_t n, int delta, uint32_t base,
                      uint32_t *out, uint32_t *last) {
    int st = validate(in, in_len, n);
    if (st != SVBO_OK) return st;
    size_t nctrl = svbo_control_bytes(n);
    uint32_t r = o2_decode_range(in, in + nctrl, in + in_len, n, delta, base, out);
    if (last) *last = delta ? r : (n ? out[n - 1] : base);
    return SVBO_OK;
}

/* ------------------------------------------------------------------ */
/* random access (stream_vbyte.hpp:48-54)                              */
/* ------------------------------------------------------------------ */

void svbo_block_data_offsets(const uint8_t *in, size_t n, uint64_t *offsets) {
    ensure_tables();
    size_t nblocks = svbo_control_bytes(n);
    uint64_t off = 0;
    for (size_t k = 0; k < nblocks; ++k) {
        offsets[k] = off;
        size_t cnt = (k + 1) * 4 <= n ? 4 : n - k * 4;
        if (cnt == 4) {
            off += g_length[in[k]];
        } else {
            for (size_t i = 0; i < cnt; ++i) off += ((in[k] >> (2 * i)) & 3) + 1;
        }
    }
}

size_t svbo_decode_block(const uint8_t *in, size_t in_len, size_t n, size_t block, size_t data_offset,
                         uint32_t out[4]) {
    size_t nctrl = svbo_control_bytes(n);
    if (block >= nctrl) return 0;
    size_t cnt = (block + 1) * 4 <= n ? 4 : n - block * 4;
    const uint8_t *data = in + nctrl + data_offset;
    uint8_t c = in[block];
    for (size_t i = 0; i < cnt; ++i) {
        uint32_t len = ((c >> (2 * i)) & 3) + 1;
        uint32_t v = 0;
        for (uint32_t b = 0; b < len; ++b) {
            if (data + b < in + in_len) v |= (uint32_t)data[b] << (8 * b);
        }
        data += len;
        out[i] = v;
    }
    return cnt;
}

/* ------------------------------------------------------------------ */
/* multi-threaded CPU reference arm                                    */
/* ------------------------------------------------------------------ */

typedef struct {
    void (*fn)(void *ctx, int tid, int nthreads);
    void *ctx;
    int tid, nthreads;
} worker_arg;

static void *worker_main(void *p) {
    worker_arg *a = (worker_arg *)p;
    a->fn(a->ctx, a->tid, a->nthreads);
    return NULL;
}

static void parallel_for(int nthreads, void (*fn)(void *, int, int), void *ctx) {
    if (nthreads <= 1) {
        fn(ctx, 0, 1);
        return;
    }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    worker_arg *args = (worker_arg *)malloc(sizeof(worker_arg) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        args[t].fn = fn;
        args[t].ctx = ctx;
        args[t].tid = t;
        args[t].nthreads = nthreads;
        if (t) pthread_create(&th[t], NULL, worker_main, &args[t]);
    }
    fn(ctx, 0, nthreads);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(args);
}

/* chunk t covers integers [lo, hi), a multiple of 4 except the last */
static void chunk_range(size_t n, int t, int nt, size_t *lo, size_t *hi) {
    size_t per = ((n + (size_t)nt - 1) / (size_t)nt + 3) & ~(size_t)3;
    *lo = per * (size_t)t;
    *hi = *lo + per;
    if (*lo > n) *lo = n;
    if (*hi > n) *hi = n;
}

typedef struct {
    const uint32_t *in;
    size_t n;
    int delta;
    uint32_t prev;
    uint8_t *out;
    uint64_t *sizes; /* per chunk data bytes, then exclusive offsets */
    int pass;
} mt_enc_ctx;

static void mt_enc_fn(void *p, int t, int nt) {
    mt_enc_ctx *c = (mt_enc_ctx *)p;
    size_t lo, hi;
    chunk_range(c->n, t, nt, &lo, &hi);
    if (lo >= hi) {
        if (c->pass == 0) c->sizes[t] = 0;
        return;
    }
    uint32_t prev = lo ? c->in[lo - 1] : c->prev;
    if (c->pass == 0) {
        uint64_t s = 0;
        for (size_t i = lo; i < hi; ++i) {
            uint32_t x = c->in[i];
            s += svbo_byte_length(c->delta ? x - prev : x);
            prev = x;
        }
        c->sizes[t] = s;
    } else {
        size_t nctrl = svbo_control_bytes(c->n);
        uint8_t *ctrl = c->out + lo / 4;
        uint8_t *data = c->out + nctrl + c->sizes[t];
        memset(ctrl, 0, svbo_control_bytes(hi - lo));
        for (size_t i = lo; i < hi; ++i) {
            uint32_t x = c->in[i];
            uint32_t v = c->delta ? x - prev : x;
            prev = x;
            uint32_t len = svbo_byte_length(v);
            ctrl[(i - lo) / 4] |= (uint8_t)((len - 1) << (2 * ((i - lo) % 4)));
            if (i + 3 < hi) {
                /* little-endian host; the <=3-byte spill lands on the next 3 ints, which are in this chunk */
                memcpy(data, &v, 4);
            } else {
                for (uint32_t b = 0; b < len; ++b) data[b] = (uint8_t)(v >> (8 * b)); /* chunk seam: exact */
            }
            data += len;
        }
    }
}

size_t svbo_mt_encode(const uint32_t *in, size_t n, int delta, uint32_t prev, uint8_t *out, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (n == 0) return 0;
    uint64_t *sizes = (uint64_t *)calloc((size_t)nthreads, sizeof(uint64_t));
    mt_enc_ctx c = {in, n, delta, prev, out, sizes, 0};
    parallel_for(nthreads, mt_enc_fn, &c);
    uint64_t total = 0;
    for (int t = 0; t < nthreads; ++t) {
        uint64_t s = sizes[t];
        sizes[t] = total;
        total += s;
    }
    c.pass = 1;
    parallel_for(nthreads, mt_enc_fn, &c);
    free(sizes);
    return svbo_control_bytes(n) + total;
}

typedef struct {
    const uint8_t *in;
    size_t in_len, n;
    int delta;
    uint32_t base;
    uint32_t *out;
    uint64_t *offs;  /* per chunk data offset */
    uint32_t *lasts; /* per chunk last value (base 0), then carry */
    int pass;
} mt_dec_ctx;

static void mt_dec_fn(void *p, int t, int nt) {
    mt_dec_ctx *c = (mt_dec_ctx *)p;
    size_t lo, hi;
    chunk_range(c->n, t, nt, &lo, &hi);
    if (c->pass == 0) {
        c->offs[t] = lo < hi ? declared_data_bytes(c->in + lo / 4, hi - lo) : 0;
        return;
    }
    if (lo >= hi) {
        if (c->pass == 1) c->lasts[t] = 0;
        return;
    }
    size_t nctrl = svbo_control_bytes(c->n);
    if (c->pass == 1) {
        const uint8_t *data = c->in + nctrl + c->offs[t];
        uint32_t base = (t == 0) ? c->base : 0;
        c->lasts[t] = o2_decode_range(c->in + lo / 4, data, c->in + c->in_len, hi - lo, c->delta, base,
                                      c->out + lo);
    } else if (t > 0) {
        uint32_t carry = c->lasts[t];
        uint32_t *o = c->out + lo;
        for (size_t i = 0; i < hi - lo; ++i) o[i] += carry;
    }
}

int svbo_mt_decode(const uint8_t *in, size_t in_len, size_t n, int delta, uint32_t base, uint32_t *out,
                   uint32_t *last, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    size_t nctrl = svbo_control_bytes(n);
    if (in_len < nctrl) return SVBO_TRUNCATED;
    if (n == 0) {
        if (in_len != 0) return SVBO_TRAILING_BYTES;
        if (last) *last = base;
        return SVBO_OK;
    }
    uint64_t *offs = (uint64_t *)calloc((size_t)nthreads, sizeof(uint64_t));
    uint32_t *lasts = (uint32_t *)calloc((size_t)nthreads, sizeof(uint32_t));
    mt_dec_ctx c = {in, in_len, n, delta, base, out, offs, lasts, 0};
    ensure_tables();
    parallel_for(nthreads, mt_dec_fn, &c);
    uint64_t total = 0;
    for (int t = 0; t < nthreads; ++t) {
        uint64_t s = offs[t];
        offs[t] = total;
        total += s;
    }
    int st = SVBO_OK;
    if (in_len < nctrl + total) st = SVBO_TRUNCATED;
    else if (in_len > nctrl + total) st = SVBO_TRAILING_BYTES;
    if (st == SVBO_OK) {
        c.pass = 1;
        parallel_for(nthreads, mt_dec_fn, &c);
        if (delta) {
            uint32_t carry = 0;
            for (int t = 0; t < nthreads; ++t) {
                uint32_t l = lasts[t];
                lasts[t] = carry;
                carry += l;
            }
            c.pass = 2;
            parallel_for(nthreads, mt_dec_fn, &c);
            if (last) *last = carry;
        } else if (last) {
            *last = out[n - 1];
        }
    }
    free(offs);
    free(lasts);
    return st;
}

/* ---- segmented batches: each segment is one single-thread O1/O2 call ---- */

typedef struct {
    const void *segs;
    size_t nseg;
    const void *in;
    void *out;
    uint64_t *out_lens;
    int delta;
    int status;
} batch_ctx;

static void dec_batch_fn(void *p, int t, int nt) {
    batch_ctx *c = (batch_ctx *)p;
    const svbo_decode_segment *segs = (const svbo_decode_segment *)c->segs;
    size_t lo = c->nseg * (size_t)t / (size_t)nt, hi = c->nseg * (size_t)(t + 1) / (size_t)nt;
    for (size_t s = lo; s < hi; ++s) {
        const svbo_decode_segment *d = &segs[s];
        int st = svbo_ssse3_decode((const uint8_t *)c->in + d->src_offset, d->src_bytes, d->n, c->delta,
                                   d->prev, (uint32_t *)c->out + d->dst_offset, NULL);
        if (st != SVBO_OK) c->status = st;
    }
}

int svbo_decode_batch(const svbo_decode_segment *segs, size_t nseg, const uint8_t *in, uint32_t *out,
                      int delta, int nthreads) {
    batch_ctx c = {segs, nseg, in, out, NULL, delta, SVBO_OK};
    ensure_tables();
    parallel_for(nthreads < 1 ? 1 : nthreads, dec_batch_fn, &c);
    return c.status;
}

static void enc_batch_fn(void *p, int t, int nt) {
    batch_ctx *c = (batch_ctx *)p;
    const svbo_encode_segment *segs = (const svbo_encode_segment *)c->segs;
    size_t lo = c->nseg * (size_t)t / (size_t)nt, hi = c->nseg * (size_t)(t + 1) / (size_t)nt;
    for (size_t s = lo; s < hi; ++s) {
        const svbo_encode_segment *e = &segs[s];
        c->out_lens[s] = svbo_encode((const uint32_t *)c->in + e->src_offset, e->n, c->delta, e->prev,
                                     (uint8_t *)c->out + e->dst_offset);
    }
}

/* The paper's timing mode over a batch (PAPER.md:415,436 decode posting lists one after
 * another): every segment, single thread, decoded by svbo_paper_decode into the same
 * 4096-integer buffer; *check sums the per-segment checks. */
int svbo_paper_decode_batch(const svbo_decode_segment *segs, size_t nseg, const uint8_t *in, int delta,
                            uint32_t *buf, uint64_t *check) {
    uint64_t sum = 0;
    for (size_t s = 0; s < nseg; ++s) {
        uint64_t c = 0;
        int st = svbo_paper_decode(in + segs[s].src_offset, segs[s].src_bytes, segs[s].n, delta, segs[s].prev, buf,
                                   &c);
        if (st != SVBO_OK) return st;
        sum += c;
    }
    if (check) *check = sum;
    return SVBO_OK;
}

int svbo_encode_batch(const svbo_encode_segment *segs, size_t nseg, const uint32_t *in, uint8_t *out,
                      uint64_t *out_lens, int delta, int nthreads) {
    batch_ctx c = {segs, nseg, in, out, out_lens, delta, SVBO_OK};
    parallel_for(nthreads < 1 ? 1 : nthreads, enc_batch_fn, &c);
    return c.status;
}
