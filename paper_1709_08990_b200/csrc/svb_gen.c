/*
 * svb_gen.c -- deterministic synthetic inputs for the five BASELINE.json configs.
 *
 * The paper measures on ClueWeb09-B posting lists, which are not
 * available here; SPEC.md:14,581 already replaces them with seeded synthetic
 * generators.  Every generator is a pure function of (seed, index) through a
 * counter-based splitmix64, so it is reproducible, parallel and portable
 * (SURVEY.md §8(d)).  Host-side only; shipped in libsvbgen.so.
 */
#include <math.h>
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* splitmix64 evaluated at counter i of stream `seed`. */
uint64_t svbgen_splitmix64(uint64_t seed, uint64_t i) {
    return mix64(seed + (i + 1) * 0x9E3779B97F4A7C15ull);
}

/* uniform double in (0, 1] from the top 53 bits */
static inline double unit_open0(uint64_t r) { return ((double)(r >> 11) + 1.0) * (1.0 / 9007199254740992.0); }

typedef struct {
    void (*fn)(void *, uint64_t, uint64_t);
    void *ctx;
    uint64_t lo, hi;
} gen_job;

static void *gen_main(void *p) {
    gen_job *j = (gen_job *)p;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}

static void par_range(uint64_t n, int nthreads, void (*fn)(void *, uint64_t, uint64_t), void *ctx) {
    if (nthreads < 1) nthreads = 1;
    if (n < 65536 || nthreads == 1) {
        fn(ctx, 0, n);
        return;
    }
    pthread_t th[256];
    gen_job jobs[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].fn = fn;
        jobs[t].ctx = ctx;
        jobs[t].lo = n * (uint64_t)t / (uint64_t)nthreads;
        jobs[t].hi = n * (uint64_t)(t + 1) / (uint64_t)nthreads;
        pthread_create(&th[t], NULL, gen_main, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* ---- configs 1 and 3: byte length uniform over {1,2,3,4} ---------------- */
typedef struct {
    uint64_t seed;
    uint32_t *out;
} cls_ctx;

static void cls_fn(void *p, uint64_t lo, uint64_t hi) {
    cls_ctx *c = (cls_ctx *)p;
    for (uint64_t i = lo; i < hi; ++i) {
        uint64_t r = svbgen_splitmix64(c->seed, i);
        uint32_t k = (uint32_t)(r & 3);
        uint64_t lo_v = k ? (1ull << (8 * k)) : 0;
        uint64_t span = (1ull << (8 * (k + 1))) - lo_v;
        c->out[i] = (uint32_t)(lo_v + (((r >> 32) * span) >> 32));
    }
}

void svbgen_uniform_classes(uint64_t seed, uint64_t n, uint32_t *out, int nthreads) {
    cls_ctx c = {seed, out};
    par_range(n, nthreads, cls_fn, &c);
}

/* ---- configs 2 and 5: sorted (mod 2^32) sequence, geometric gaps --------
 * x_0 = start, x_i = x_{i-1} + g_i, g_i = 1 + floor(ln u / ln(1 - 1/mean)),
 * u uniform in (0,1].  Gap pass in parallel, then a chunked prefix sum. */
typedef struct {
    uint64_t seed;
    double inv_log_q;
    uint32_t *out;
    uint32_t *chunk_sums;
    uint64_t n;
    uint64_t i0;   /* global index of out[0] */
    uint32_t base; /* x_{i0 - 1} + start: added to every element in pass 1 */
    int nthreads;
    int pass;
} geo_ctx;

static inline uint32_t geo_gap(uint64_t seed, double inv_log_q, uint64_t i) {
    double u = unit_open0(svbgen_splitmix64(seed, i));
    double g = floor(log(u) * inv_log_q);
    if (g > 4294967294.0) g = 4294967294.0;
    return 1u + (uint32_t)g;
}

static void geo_fn(void *p, uint64_t lo, uint64_t hi) {
    geo_ctx *c = (geo_ctx *)p;
    if (c->pass == 0) {
        uint32_t s = 0;
        for (uint64_t i = lo; i < hi; ++i) {
            const uint64_t gi = c->i0 + i;
            uint32_t g = (gi == 0) ? 0 : geo_gap(c->seed, c->inv_log_q, gi);
            s += g;
            c->out[i] = s; /* local inclusive sum */
        }
    } else {
        /* find the chunk index from lo (chunks are the same split as pass 0) */
        uint32_t carry = c->base;
        for (int k = 0; k < c->nthreads; ++k) {
            uint64_t klo = c->n * (uint64_t)k / (uint64_t)c->nthreads;
            if (klo >= lo) break;
            carry += c->chunk_sums[k];
        }
        for (uint64_t i = lo; i < hi; ++i) c->out[i] += carry;
    }
}

static void geo_fill(uint64_t seed, uint64_t i0, uint64_t n, double mean_gap, uint32_t base, uint32_t *out,
                     int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (n < 65536) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    geo_ctx c = {seed, 1.0 / log(1.0 - 1.0 / mean_gap), out, NULL, n, i0, base, nthreads, 0};
    uint32_t sums[256];
    c.chunk_sums = sums;
    par_range(n, nthreads, geo_fn, &c);
    for (int k = 0; k < nthreads; ++k) {
        uint64_t hi = n * (uint64_t)(k + 1) / (uint64_t)nthreads;
        uint64_t lo = n * (uint64_t)k / (uint64_t)nthreads;
        sums[k] = hi > lo ? out[hi - 1] : 0;
    }
    /* pass 1 adds the sum of all earlier chunks' totals, plus the base */
    c.pass = 1;
    par_range(n, nthreads, geo_fn, &c);
}

void svbgen_geometric_sorted(uint64_t seed, uint64_t n, double mean_gap, uint32_t start, uint32_t *out,
                             int nthreads) {
    geo_fill(seed, 0, n, mean_gap, start, out, nthreads);
}

/* sum of gaps g_1 .. g_{i1-1} (mod 2^32), without storing them */
typedef struct {
    uint64_t seed;
    double inv_log_q;
    uint32_t part[256];
    int nthreads;
    uint64_t n;
} gsum_ctx;

static void gsum_fn(void *p, uint64_t lo, uint64_t hi) {
    gsum_ctx *c = (gsum_ctx *)p;
    uint32_t s = 0;
    for (uint64_t i = lo; i < hi; ++i) s += i ? geo_gap(c->seed, c->inv_log_q, i) : 0u;
    for (int k = 0; k < c->nthreads; ++k)
        if (c->n * (uint64_t)k / (uint64_t)c->nthreads == lo) {
            c->part[k] = s;
            break;
        }
}

/* Elements [i0, i0 + n) of the config-2/5 sequence x_0 = 0, x_i = x_{i-1} + g_i
 * (identical to the same elements of svbgen_geometric_sorted(seed, N, mean, 0, ...)):
 * one rank's shard of the sequence without generating the ranks before it. */
void svbgen_geometric_sorted_range(uint64_t seed, uint64_t i0, uint64_t n, double mean_gap, uint32_t *out,
                                   int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    uint32_t carry = 0;
    if (i0) {
        gsum_ctx g;
        g.seed = seed;
        g.inv_log_q = 1.0 / log(1.0 - 1.0 / mean_gap);
        g.n = i0;
        g.nthreads = i0 < 65536 ? 1 : nthreads;
        for (int k = 0; k < 256; ++k) g.part[k] = 0;
        par_range(i0, g.nthreads, gsum_fn, &g);
        for (int k = 0; k < g.nthreads; ++k) carry += g.part[k];
    }
    geo_fill(seed, i0, n, mean_gap, carry, out, nthreads);
}

/* ---- config 4: posting-list-like batch --------------------------------
 * L_i = floor(2^U_i), U_i ~ U(4,16).  Total capped by a common water-fill cap
 * C (largest C with sum min(L_i, C) <= cap_total).  Each
 * list = L strictly increasing values in [0, universe), drawn as exponential
 * order statistics of [0, universe - L] plus rank j (uniform-spacing sample). */
uint64_t svbgen_list_lengths(uint64_t seed, uint64_t nlists, uint64_t cap_total, uint32_t *lens) {
    uint64_t total = 0;
    uint32_t maxl = 0;
    for (uint64_t i = 0; i < nlists; ++i) {
        double u = unit_open0(svbgen_splitmix64(seed, i)) ; /* (0,1] */
        double U = 4.0 + 12.0 * (u - 1.0 / 9007199254740992.0);
        uint32_t L = (uint32_t)floor(exp2(U));
        if (L < 16) L = 16;
        if (L > 65535) L = 65535;
        lens[i] = L;
        total += L;
        if (L > maxl) maxl = L;
    }
    if (cap_total == 0 || total <= cap_total) return maxl;
    /* binary search the largest cap C with sum min(L, C) <= cap_total */
    uint64_t lo = 0, hi = maxl;
    while (lo < hi) {
        uint64_t mid = (lo + hi + 1) / 2, s = 0;
        for (uint64_t i = 0; i < nlists; ++i) s += lens[i] < mid ? lens[i] : mid;
        if (s <= cap_total) lo = mid;
        else hi = mid - 1;
    }
    for (uint64_t i = 0; i < nlists; ++i)
        if (lens[i] > lo) lens[i] = (uint32_t)lo;
    return lo;
}

typedef struct {
    uint64_t seed;
    const uint32_t *lens;
    const uint64_t *offsets;
    uint32_t universe;
    uint32_t *out;
    uint64_t list_base; /* global index of lens[0] */
} lists_ctx;

static void lists_fn(void *p, uint64_t lo, uint64_t hi) {
    lists_ctx *c = (lists_ctx *)p;
    for (uint64_t li = lo; li < hi; ++li) {
        uint32_t L = c->lens[li];
        uint32_t *o = c->out + c->offsets[li];
        uint64_t stream = mix64(c->seed ^ (0xA0761D6478BD642Full * (c->list_base + li + 1)));
        /* L+1 exponential spacings; cumulative sums normalised */
        double total = 0.0;
        for (uint32_t j = 0; j <= L; ++j) total += -log(unit_open0(svbgen_splitmix64(stream, j)));
        double scale = (double)(c->universe - L) / total, acc = 0.0;
        for (uint32_t j = 0; j < L; ++j) {
            acc += -log(unit_open0(svbgen_splitmix64(stream, j)));
            uint64_t y = (uint64_t)floor(acc * scale);
            if (y > c->universe - L) y = c->universe - L;
            o[j] = (uint32_t)y + j; /* strictly increasing, < universe */
        }
        /* floor of a nondecreasing sequence is nondecreasing, so o is strictly increasing */
    }
}

void svbgen_posting_lists(uint64_t seed, uint64_t nlists, const uint32_t *lens, const uint64_t *offsets,
                          uint32_t universe, uint32_t *out, int nthreads) {
    lists_ctx c = {seed, lens, offsets, universe, out, 0};
    par_range(nlists, nthreads, lists_fn, &c);
}

/* Lists [l0, l0 + m) only (one rank's shard): lens / offsets describe those m lists
 * (offsets relative to out); identical to the same lists of svbgen_posting_lists. */
void svbgen_posting_lists_range(uint64_t seed, uint64_t l0, uint64_t m, const uint32_t *lens,
                                const uint64_t *offsets, uint32_t universe, uint32_t *out, int nthreads) {
    lists_ctx c = {seed, lens, offsets, universe, out, l0};
    par_range(m, nthreads, lists_fn, &c);
}
