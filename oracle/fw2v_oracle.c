/* CPU restatement of the reference SGNS training path — TEST INFRASTRUCTURE.
 * See fw2v_oracle.h for the contract. Each function cites the reference
 * file:line (under /root/reference/proj) whose arithmetic it restates. */
#define _POSIX_C_SOURCE 200809L
#include "fw2v_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static __thread char g_err[256];

static int set_err(int code, const char* msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

const char* oracle_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- rng.hpp */

#define GOLDEN 0x9e3779b97f4a7c15ULL

uint64_t oracle_rng_mix(uint64_t z) { /* rng.hpp:38-42 */
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

typedef struct { uint64_t state; } rng_t;

static rng_t rng_derive(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) { /* rng.hpp:13-22 */
    rng_t r;
    r.state = oracle_rng_mix(seed);
    r.state = oracle_rng_mix(r.state ^ oracle_rng_mix(a + GOLDEN));
    r.state = oracle_rng_mix(r.state ^ oracle_rng_mix(b + 0xbf58476d1ce4e5b9ULL));
    r.state = oracle_rng_mix(r.state ^ oracle_rng_mix(c + 0x94d049bb133111ebULL));
    return r;
}

static inline uint64_t rng_next(rng_t* r) { /* rng.hpp:24-27 */
    r->state += GOLDEN;
    return oracle_rng_mix(r->state);
}
static inline uint64_t rng_below(rng_t* r, uint64_t n) { return rng_next(r) % n; } /* rng.hpp:30 */
static inline double rng_double(rng_t* r) { /* rng.hpp:33 */
    return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}
static inline float rng_float(rng_t* r) { /* rng.hpp:35 */
    return (float)(rng_next(r) >> 40) * 0x1.0p-24f;
}

void oracle_rng_draws(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t n, uint64_t* out) {
    rng_t r = rng_derive(seed, a, b, c);
    for (uint64_t i = 0; i < n; ++i) out[i] = rng_next(&r);
}

/* -------------------------------------------------------------- model.cpp */

int oracle_init_model(int32_t vocab_size, int32_t dim, uint64_t seed, float* input,
                      float* output) { /* model.cpp:15-32 */
    if (vocab_size < 1) return set_err(4, "vocab size must be >= 1");
    if (dim < 1) return set_err(4, "dim must be >= 1");
    size_t n = (size_t)vocab_size * (size_t)dim;
    rng_t r = rng_derive(seed, 0x696e6974ULL, 0, 0);
    float inv_dim = 1.0f / (float)dim;
    for (size_t i = 0; i < n; ++i) input[i] = (rng_float(&r) - 0.5f) * inv_dim;
    if (output) memset(output, 0, n * sizeof(float));
    return 0;
}

float oracle_sigmoid(float x) { /* model.cpp:34-37 */
    float c = x < -6.0f ? -6.0f : (6.0f < x ? 6.0f : x);
    return (float)(1.0 / (1.0 + exp(-(double)c)));
}

float oracle_lr_at(uint64_t words_trained, uint64_t total, float alpha0) { /* model.cpp:39-45 */
    if (total == 0) { set_err(4, "total_words must be > 0"); return -1.0f; }
    double progress = (double)words_trained / (double)total;
    double alpha = (double)alpha0 * (1.0 - progress);
    double floor_ = (double)alpha0 * 1e-4;
    return (float)(alpha > floor_ ? alpha : floor_);
}

/* ------------------------------------------------------------ kernels.hpp */

float oracle_dot(const float* a, const float* b, int32_t d) { /* kernels.hpp:10-22 */
    float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, s3 = 0.0f;
    int k = 0;
    for (; k + 4 <= d; k += 4) {
        s0 += a[k] * b[k];
        s1 += a[k + 1] * b[k + 1];
        s2 += a[k + 2] * b[k + 2];
        s3 += a[k + 3] * b[k + 3];
    }
    float s = (s0 + s1) + (s2 + s3);
    for (; k < d; ++k) s += a[k] * b[k];
    return s;
}

static inline void pairing_update(float* ctx, float* smp, float g, int d) { /* kernels.hpp:26-33 */
    for (int k = 0; k < d; ++k) {
        float c = ctx[k], s = smp[k];
        ctx[k] = c + g * s;
        smp[k] = s + g * c;
    }
}

static inline void axpy(float* y, const float* x, float g, int d) { /* kernels.hpp:36-38 */
    for (int k = 0; k < d; ++k) y[k] += g * x[k];
}

/* ------------------------------------------------------------- corpus.cpp */

static double keep_prob_one(double f, double t) { /* corpus.cpp:215-219 */
    if (t <= 0.0 || f <= 0.0) return 1.0;
    double p = (sqrt(f / t) + 1.0) * (t / f);
    return p < 1.0 ? p : 1.0;
}

int oracle_keep_probs(const uint64_t* counts, int32_t v, double t, double* out) { /* corpus.cpp:221-230 */
    if (t <= 0.0) return 0;
    uint64_t total_u = 0;
    for (int32_t w = 0; w < v; ++w) total_u += counts[w];
    double total = (double)total_u;
    for (int32_t w = 0; w < v; ++w) out[w] = keep_prob_one((double)counts[w] / total, t);
    return 1;
}

/* ------------------------------------------------------------ sampler.cpp */

int oracle_table_build(const uint64_t* counts, int32_t v, double power, uint64_t size,
                       int32_t* slots) { /* sampler.cpp:9-35 */
    if (size < (uint64_t)v) return set_err(4, "table_size must be >= |V|");
    if (power < 0.0) return set_err(4, "power must be >= 0");
    double* cum = (double*)malloc(sizeof(double) * (size_t)v);
    double total = 0.0;
    for (int32_t w = 0; w < v; ++w) {
        total += pow((double)counts[w], power);
        cum[w] = total;
    }
    size_t w = 0;
    for (uint64_t s = 0; s < size; ++s) {
        double mid = ((double)s + 0.5) / (double)size * total;
        while (w + 1 < (size_t)v && mid >= cum[w]) ++w;
        slots[s] = (int32_t)w;
    }
    free(cum);
    return 0;
}

typedef struct {
    const uint64_t* offsets;
    const int32_t* ids;
    uint64_t n;
} stream_t;

/* assemble_batch (sampler.cpp:41-63) with subsample_sentence (corpus.cpp:232-241)
 * inlined; kept ids appended to out_ids, negatives to out_negs. */
static int64_t assemble(const stream_t* st, uint64_t* cursor, uint64_t max_sentences, int32_t n_neg,
                        const int32_t* slots, uint64_t table_size, const double* keep, rng_t* rng,
                        int32_t* out_ids, uint64_t* out_offsets, int32_t* out_negs) {
    int64_t kept = 0;
    uint64_t w = 0, nw = 0;
    out_offsets[0] = 0;
    while ((uint64_t)kept < max_sentences && *cursor < st->n) {
        uint64_t b = st->offsets[*cursor], e = st->offsets[*cursor + 1];
        uint64_t start = w;
        for (uint64_t p = b; p < e; ++p) {
            int32_t id = st->ids[p];
            if (!keep || rng_double(rng) < keep[id]) out_ids[w++] = id;
        }
        ++*cursor;
        if (w == start) continue;
        for (uint64_t p = start; p < w; ++p) {
            for (int32_t k = 0; k < n_neg; ++k) out_negs[nw++] = slots[rng_below(rng, table_size)];
        }
        ++kept;
        out_offsets[kept] = w;
    }
    return kept;
}

int64_t oracle_assemble_batch(const uint64_t* counts, int32_t v, const uint64_t* offsets,
                              uint64_t n_sentences, const int32_t* ids, uint64_t* cursor,
                              uint64_t max_sentences, int32_t negatives, double power,
                              uint64_t table_size, double threshold, uint64_t seed, uint64_t a,
                              uint64_t b, uint64_t c, int32_t* out_ids, uint64_t* out_offsets,
                              int32_t* out_negs) {
    if (max_sentences < 1) return -set_err(4, "batch size must be >= 1");
    if (negatives < 0) return -set_err(4, "negatives must be >= 0");
    int32_t* slots = (int32_t*)malloc(sizeof(int32_t) * table_size);
    int rc = oracle_table_build(counts, v, power, table_size, slots);
    if (rc) { free(slots); return -rc; }
    double* keep = (double*)malloc(sizeof(double) * (size_t)v);
    int on = oracle_keep_probs(counts, v, threshold, keep);
    stream_t st = {offsets, ids, n_sentences};
    rng_t r = rng_derive(seed, a, b, c);
    int64_t n = assemble(&st, cursor, max_sentences, negatives, slots, table_size, on ? keep : NULL,
                         &r, out_ids, out_offsets, out_negs);
    free(slots);
    free(keep);
    return n;
}

/* ------------------------------------------------------------ traffic.cpp */

static uint64_t pairings_for_length(uint64_t len, uint64_t w) { /* traffic.cpp:13-17 */
    if (len < 2) return 0;
    uint64_t g = w < len - 1 ? w : len - 1;
    return 2 * g * len - g * (g + 1);
}

int oracle_analytic_traffic(uint64_t len, int32_t width, int32_t negatives, int32_t mode,
                            uint64_t* t) { /* traffic.cpp:21-59 */
    if (len < 1) return set_err(4, "sentence length must be >= 1");
    if (width < 1) return set_err(4, "context width must be >= 1");
    if (negatives < 0) return set_err(4, "negatives must be >= 0");
    uint64_t pairs = pairings_for_length(len, (uint64_t)width);
    uint64_t samples = (uint64_t)negatives + 1;
    uint64_t windows = len >= 2 ? len : 0;
    switch (mode) {
    case 0: case 3:
        t[0] = len; t[1] = len; t[2] = windows * samples; t[3] = windows * samples;
        t[4] = windows > 0 ? samples * pairs - len : 0;
        break;
    case 1:
        t[0] = pairs; t[1] = pairs; t[2] = windows * samples; t[3] = windows * samples;
        t[4] = (uint64_t)negatives * pairs;
        break;
    case 2:
        t[0] = samples * pairs; t[1] = samples * pairs; t[2] = samples * pairs;
        t[3] = samples * pairs; t[4] = 0;
        break;
    default:
        return set_err(4, "unknown reuse mode");
    }
    return 0;
}

/* ------------------------------------------------------------ trainer.cpp */

typedef struct {
    float* in;
    float* out;
    int d;
} model_t;

typedef struct {
    int pos;
    int used;
} slot_t;

typedef struct {
    int width, cap, d;
    const int32_t* ids;
    int len;
    slot_t* slots;
    float* storage;
    int next_load;
    float* sample;
    float* snap_ctx;
    float* snap_smp;
    float* delta_ctx;
    float* delta_smp;
    float* window_vecs;
    int* ctx_pos;
    float** ctx_ptrs;
} scratch_t;

enum { C_RD = 0, C_WR = 1, S_RD = 2, S_WR = 3, HITS = 4 };

static void ring_write_back(scratch_t* s, model_t* m, int slot, uint64_t* tc) { /* trainer.cpp:46-53 */
    memcpy(m->in + (size_t)s->ids[s->slots[slot].pos] * m->d, s->storage + (size_t)slot * m->d,
           sizeof(float) * (size_t)m->d);
    ++tc[C_WR];
    s->slots[slot].pos = -1;
    s->slots[slot].used = 0;
}

static void ring_advance(scratch_t* s, model_t* m, int target, uint64_t* tc) { /* trainer.cpp:55-69 */
    int hi = s->len - 1 < target + s->width ? s->len - 1 : target + s->width;
    while (s->next_load <= hi) {
        int slot = s->next_load % s->cap;
        if (s->slots[slot].pos >= 0) ring_write_back(s, m, slot, tc);
        memcpy(s->storage + (size_t)slot * m->d, m->in + (size_t)s->ids[s->next_load] * m->d,
               sizeof(float) * (size_t)m->d);
        ++tc[C_RD];
        s->slots[slot].pos = s->next_load;
        s->slots[slot].used = 0;
        ++s->next_load;
    }
}

static void ring_finish(scratch_t* s, model_t* m, uint64_t* tc) { /* trainer.cpp:71-75 */
    for (int k = 0; k < s->cap; ++k)
        if (s->slots[k].pos >= 0) ring_write_back(s, m, k, tc);
}

static float* ring_touch(scratch_t* s, int pos, uint64_t* tc) { /* trainer.cpp:93-102 */
    slot_t* sl = &s->slots[pos % s->cap];
    if (sl->used) ++tc[HITS];
    else sl->used = 1;
    return s->storage + (size_t)(pos % s->cap) * s->d;
}

static int collect_context(int target, int w, int len, int* out) { /* trainer.cpp:121-129 */
    int lo = target - w > 0 ? target - w : 0;
    int hi = len - 1 < target + w ? len - 1 : target + w;
    int n = 0;
    for (int j = lo; j <= hi; ++j)
        if (j != target) out[n++] = j;
    return n;
}

/* sweep_samples (trainer.cpp:133-154); touch: 0 none, 1 ring */
static void sweep(model_t* m, scratch_t* s, int32_t target_id, const int32_t* negs, int n_neg,
                  float alpha, float** ctx, int n_ctx, uint64_t* tc, int ring_touch_on) {
    int d = m->d;
    for (int k = 0; k <= n_neg; ++k) {
        int32_t sid = k == 0 ? target_id : negs[k - 1];
        float label = k == 0 ? 1.0f : 0.0f;
        memcpy(s->sample, m->out + (size_t)sid * d, sizeof(float) * (size_t)d);
        ++tc[S_RD];
        for (int j = 0; j < n_ctx; ++j) {
            if (ring_touch_on) ring_touch(s, s->ctx_pos[j], tc);
            float f = oracle_dot(ctx[j], s->sample, d);
            float g = (label - oracle_sigmoid(f)) * alpha;
            pairing_update(ctx[j], s->sample, g, d);
        }
        memcpy(m->out + (size_t)sid * d, s->sample, sizeof(float) * (size_t)d);
        ++tc[S_WR];
    }
}

/* sweep_samples_snapshot (trainer.cpp:158-205) */
static void sweep_snapshot(model_t* m, scratch_t* s, int32_t target_id, const int32_t* negs,
                           int n_neg, float alpha, int n_ctx, uint64_t* tc) {
    int d = m->d;
    int samples = n_neg + 1;
    size_t bytes = sizeof(float) * (size_t)d;
    for (int j = 0; j < n_ctx; ++j)
        memcpy(s->snap_ctx + (size_t)j * d, s->storage + (size_t)(s->ctx_pos[j] % s->cap) * d, bytes);
    for (int k = 0; k < samples; ++k) {
        int32_t sid = k == 0 ? target_id : negs[k - 1];
        memcpy(s->snap_smp + (size_t)k * d, m->out + (size_t)sid * d, bytes);
        ++tc[S_RD];
    }
    memset(s->delta_ctx, 0, bytes * (size_t)n_ctx);
    memset(s->delta_smp, 0, bytes * (size_t)samples);
    for (int k = 0; k < samples; ++k) {
        float label = k == 0 ? 1.0f : 0.0f;
        const float* smp = s->snap_smp + (size_t)k * d;
        float* dsmp = s->delta_smp + (size_t)k * d;
        for (int j = 0; j < n_ctx; ++j) {
            ring_touch(s, s->ctx_pos[j], tc);
            const float* cv = s->snap_ctx + (size_t)j * d;
            float f = oracle_dot(cv, smp, d);
            float g = (label - oracle_sigmoid(f)) * alpha;
            axpy(s->delta_ctx + (size_t)j * d, smp, g, d);
            axpy(dsmp, cv, g, d);
        }
    }
    for (int j = 0; j < n_ctx; ++j) {
        const float* delta = s->delta_ctx + (size_t)j * d;
        float* cv = s->storage + (size_t)(s->ctx_pos[j] % s->cap) * d;
        for (int k = 0; k < d; ++k) cv[k] += delta[k];
    }
    for (int k = 0; k < samples; ++k) {
        int32_t sid = k == 0 ? target_id : negs[k - 1];
        const float* delta = s->delta_smp + (size_t)k * d;
        float* row = m->out + (size_t)sid * d;
        for (int i = 0; i < d; ++i) row[i] += delta[i];
        ++tc[S_WR];
    }
}

static void scratch_init(scratch_t* s, int width, int d, int n_neg) { /* trainer.cpp:104-115 */
    memset(s, 0, sizeof(*s));
    s->width = width;
    s->cap = 2 * width + 1;
    s->d = d;
    size_t span = 2 * (size_t)width;
    size_t samples = (size_t)n_neg + 1;
    s->slots = (slot_t*)malloc(sizeof(slot_t) * (size_t)s->cap);
    s->storage = (float*)malloc(sizeof(float) * (size_t)s->cap * d);
    s->sample = (float*)malloc(sizeof(float) * (size_t)d);
    s->snap_ctx = (float*)malloc(sizeof(float) * span * d);
    s->snap_smp = (float*)malloc(sizeof(float) * samples * d);
    s->delta_ctx = (float*)malloc(sizeof(float) * span * d);
    s->delta_smp = (float*)malloc(sizeof(float) * samples * d);
    s->window_vecs = (float*)malloc(sizeof(float) * span * d);
    s->ctx_pos = (int*)malloc(sizeof(int) * span);
    s->ctx_ptrs = (float**)malloc(sizeof(float*) * span);
}

static void scratch_free(scratch_t* s) {
    free(s->slots); free(s->storage); free(s->sample); free(s->snap_ctx); free(s->snap_smp);
    free(s->delta_ctx); free(s->delta_smp); free(s->window_vecs); free(s->ctx_pos); free(s->ctx_ptrs);
}

/* train_sentence (trainer.cpp:332-356) for one sentence of length len. */
static void train_one(model_t* m, scratch_t* s, const int32_t* ids, int len, const int32_t* negs,
                      int n_neg, int mode, float alpha, uint64_t* tc) {
    int d = m->d;
    int w = s->width;
    size_t bytes = sizeof(float) * (size_t)d;
    if (mode == 0 || mode == 3) { /* train_sentence_ring, trainer.cpp:237-255 */
        s->ids = ids;
        s->len = len;
        s->next_load = 0;
        for (int k = 0; k < s->cap; ++k) { s->slots[k].pos = -1; s->slots[k].used = 0; }
        for (int i = 0; i < len; ++i) {
            ring_advance(s, m, i, tc);
            int n_ctx = collect_context(i, w, len, s->ctx_pos); /* process_window 209-226 */
            if (n_ctx == 0) continue;
            if (mode == 3) {
                sweep_snapshot(m, s, ids[i], negs + (size_t)i * n_neg, n_neg, alpha, n_ctx, tc);
            } else {
                for (int j = 0; j < n_ctx; ++j)
                    s->ctx_ptrs[j] = s->storage + (size_t)(s->ctx_pos[j] % s->cap) * d;
                sweep(m, s, ids[i], negs + (size_t)i * n_neg, n_neg, alpha, s->ctx_ptrs, n_ctx, tc, 1);
            }
        }
        ring_finish(s, m, tc);
    } else if (mode == 1) { /* train_sentence_window, trainer.cpp:257-290 */
        for (int i = 0; i < len; ++i) {
            int n_ctx = collect_context(i, w, len, s->ctx_pos);
            if (n_ctx == 0) continue;
            for (int j = 0; j < n_ctx; ++j) {
                float* local = s->window_vecs + (size_t)j * d;
                memcpy(local, m->in + (size_t)ids[s->ctx_pos[j]] * d, bytes);
                ++tc[C_RD];
                s->ctx_ptrs[j] = local;
            }
            sweep(m, s, ids[i], negs + (size_t)i * n_neg, n_neg, alpha, s->ctx_ptrs, n_ctx, tc, 0);
            tc[HITS] += (uint64_t)n_ctx * (uint64_t)n_neg;
            for (int j = 0; j < n_ctx; ++j) {
                memcpy(m->in + (size_t)ids[s->ctx_pos[j]] * d, s->window_vecs + (size_t)j * d, bytes);
                ++tc[C_WR];
            }
        }
    } else { /* train_sentence_direct, trainer.cpp:292-328 */
        for (int i = 0; i < len; ++i) {
            int n_ctx = collect_context(i, w, len, s->ctx_pos);
            if (n_ctx == 0) continue;
            const int32_t* ng = negs + (size_t)i * n_neg;
            for (int k = 0; k <= n_neg; ++k) {
                int32_t sid = k == 0 ? ids[i] : ng[k - 1];
                float label = k == 0 ? 1.0f : 0.0f;
                for (int j = 0; j < n_ctx; ++j) {
                    memcpy(s->sample, m->out + (size_t)sid * d, bytes);
                    ++tc[S_RD];
                    float* cv = m->in + (size_t)ids[s->ctx_pos[j]] * d;
                    ++tc[C_RD];
                    float f = oracle_dot(cv, s->sample, d);
                    float g = (label - oracle_sigmoid(f)) * alpha;
                    pairing_update(cv, s->sample, g, d);
                    ++tc[C_WR];
                    memcpy(m->out + (size_t)sid * d, s->sample, bytes);
                    ++tc[S_WR];
                }
            }
        }
    }
}

int oracle_train_sentences(float* input, float* output, int32_t vocab_size, int32_t dim,
                           const uint64_t* offsets, uint64_t n_sentences, const int32_t* ids,
                           const int32_t* negatives, const float* alphas, const oracle_config* cfg,
                           uint64_t* counters) {
    (void)vocab_size;
    if (cfg->reuse_mode < 0 || cfg->reuse_mode > 3) return set_err(4, "unknown reuse mode");
    int width = (cfg->window + 1) / 2; /* config.hpp:32 */
    model_t m = {input, output, dim};
    scratch_t s;
    scratch_init(&s, width, dim, cfg->negatives);
    uint64_t tc[5] = {0, 0, 0, 0, 0};
    uint64_t neg_off = 0;
    for (uint64_t k = 0; k < n_sentences; ++k) {
        int len = (int)(offsets[k + 1] - offsets[k]);
        train_one(&m, &s, ids + offsets[k], len, negatives ? negatives + neg_off : NULL,
                  cfg->negatives, cfg->reuse_mode, alphas[k], tc);
        neg_off += (uint64_t)len * (uint64_t)cfg->negatives;
    }
    scratch_free(&s);
    if (counters) memcpy(counters, tc, sizeof(tc));
    return 0;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int oracle_train(const uint64_t* counts, int32_t v, const uint64_t* offsets, uint64_t n_sentences,
                 const int32_t* ids, const oracle_config* cfg, float* out_input, float* out_output,
                 oracle_report* report) { /* trainer.cpp:390-528, workers = 1 */
    if (v < 1) return set_err(3, "corpus has an empty vocabulary");
    if (cfg->dim < 1 || cfg->window < 1 || cfg->negatives < 0 || cfg->epochs < 0 ||
        !(cfg->alpha0 > 0.0f) || cfg->batch_sentences < 1 || cfg->table_size < 1 ||
        !(cfg->table_power >= 0.0))
        return set_err(5, "bad config");
    int d = cfg->dim;
    int n_neg = cfg->negatives;
    double* keep = (double*)malloc(sizeof(double) * (size_t)v);
    int keep_on = oracle_keep_probs(counts, v, cfg->subsample, keep);
    int32_t* slots = (int32_t*)malloc(sizeof(int32_t) * cfg->table_size);
    int rc = oracle_table_build(counts, v, cfg->table_power, cfg->table_size, slots);
    if (rc) { free(keep); free(slots); return rc; }
    oracle_init_model(v, d, cfg->seed, out_input, out_output);

    uint64_t total_retained = 0;
    for (int32_t w = 0; w < v; ++w) total_retained += counts[w];
    uint64_t expected = total_retained; /* expected_epoch_words, trainer.cpp:378-386 */
    if (keep_on) {
        double e = 0.0;
        for (int32_t w = 0; w < v; ++w) e += (double)counts[w] * keep[w];
        expected = (uint64_t)(e + 0.5);
        if (expected == 0) expected = 1;
    }
    uint64_t schedule_total = 1;
    if (cfg->epochs > 0) {
        schedule_total = (uint64_t)cfg->epochs * expected;
        if (schedule_total < 1) schedule_total = 1;
    }

    uint64_t max_len = 0, total_tokens = offsets[n_sentences] - offsets[0];
    for (uint64_t k = 0; k < n_sentences; ++k)
        if (offsets[k + 1] - offsets[k] > max_len) max_len = offsets[k + 1] - offsets[k];
    (void)max_len;
    uint64_t batch_cap = total_tokens + 1;
    int32_t* b_ids = (int32_t*)malloc(sizeof(int32_t) * batch_cap);
    uint64_t* b_off = (uint64_t*)malloc(sizeof(uint64_t) * (n_sentences + 2));
    int32_t* b_negs = (int32_t*)malloc(sizeof(int32_t) * (batch_cap * (size_t)(n_neg > 0 ? n_neg : 1)));

    model_t m = {out_input, out_output, d};
    scratch_t s;
    scratch_init(&s, (cfg->window + 1) / 2, d, n_neg);
    uint64_t tc[5] = {0, 0, 0, 0, 0}, an[5] = {0, 0, 0, 0, 0};
    uint64_t words_trained = 0, sentences = 0;
    stream_t st = {offsets, ids, n_sentences};
    if (report) memset(report, 0, sizeof(*report));
    double t_run = now_s();
    double batch_s = 0.0;
    uint64_t batch_words = 0;
    for (int epoch = 0; epoch < cfg->epochs; ++epoch) {
        double t0 = now_s();
        uint64_t cursor = 0, epoch_words = 0;
        for (uint64_t k = 0; cursor < n_sentences; ++k) {
            rng_t r = rng_derive(cfg->seed, (uint64_t)epoch, 0, k);
            double tb = now_s();
            int64_t nk = assemble(&st, &cursor, cfg->batch_sentences, n_neg, slots, cfg->table_size,
                                  keep_on ? keep : NULL, &r, b_ids, b_off, b_negs);
            batch_s += now_s() - tb;
            for (int64_t q = 0; q < nk; ++q) {
                int len = (int)(b_off[q + 1] - b_off[q]);
                float alpha = oracle_lr_at(words_trained, schedule_total, cfg->alpha0);
                train_one(&m, &s, b_ids + b_off[q], len, b_negs + b_off[q] * (uint64_t)n_neg, n_neg,
                          cfg->reuse_mode, alpha, tc);
                words_trained += (uint64_t)len;
                epoch_words += (uint64_t)len;
                batch_words += (uint64_t)len;
                ++sentences;
                uint64_t a[5];
                oracle_analytic_traffic((uint64_t)len, s.width, n_neg, cfg->reuse_mode, a);
                for (int z = 0; z < 5; ++z) an[z] += a[z];
            }
        }
        double secs = now_s() - t0;
        if (report && epoch < 64) {
            report->epoch_words[epoch] = epoch_words;
            report->epoch_seconds[epoch] = secs;
            report->epoch_words_per_sec[epoch] = secs > 0 ? (double)epoch_words / secs : 0.0;
        }
    }
    if (report) {
        report->words_trained = words_trained;
        report->sentences_trained = sentences;
        report->vocab_size = (uint64_t)v;
        report->wall_seconds = now_s() - t_run;
        report->batching_words_per_sec = batch_s > 0 ? (double)batch_words / batch_s : 0.0;
        report->n_epochs = cfg->epochs;
        memcpy(report->traffic, tc, sizeof(tc));
        memcpy(report->analytic, an, sizeof(an));
    }
    scratch_free(&s);
    free(b_ids); free(b_off); free(b_negs); free(keep); free(slots);
    return 0;
}
