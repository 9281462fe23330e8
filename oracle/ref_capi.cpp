// C-ABI over the *reference* ringvec library (test infrastructure, not product).
//
// Compiled by oracle/Makefile together with the reference sources that lie in
// /root/reference/proj/src (never copied into this repo) into
// oracle/_ref/libringvec_refcapi.so. Python tests and bench.py's reference /
// cpu_baseline legs call the reference through these plain-C entry points via
// ctypes; nothing on the product path links or calls this library.
//
// Each entry point wraps one reference API:
//   ref_train            -> ringvec::train                 trainer.cpp:390
//   ref_train_sentences  -> ringvec::train_sentence        trainer.cpp:332
//   ref_init_model       -> ringvec::init_model            model.cpp:15
//   ref_sigmoid/ref_lr_at-> ringvec::sigmoid / lr_at       model.cpp:34-45
//   ref_keep_probs       -> ringvec::subsample_keep_probs  corpus.cpp:221
//   ref_table_build      -> ringvec::NegativeTable::build  sampler.cpp:9
//   ref_assemble_batch   -> ringvec::assemble_batch        sampler.cpp:41
//   ref_rng_draws        -> ringvec::Rng::derive/next_u64  rng.hpp:16-28
//   ref_analytic_traffic -> ringvec::analytic_traffic      traffic.cpp:21
//   ref_save_embeddings  -> ringvec::save_embeddings       model.cpp:47-74
//   ref_nearest_neighbors-> ringvec::nearest_neighbors     eval.cpp:303-348
//   ref_analogy_correct  -> ringvec::eval_analogy          eval.cpp:212-290
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "ringvec/config.hpp"
#include "ringvec/corpus.hpp"
#include "ringvec/error.hpp"
#include "ringvec/eval.hpp"
#include "ringvec/model.hpp"
#include "ringvec/rng.hpp"
#include "ringvec/sampler.hpp"
#include "ringvec/traffic.hpp"
#include "ringvec/trainer.hpp"

using namespace ringvec;

extern "C" {

struct ref_config {
    int32_t dim, window, negatives, epochs;
    float alpha0;
    double subsample;
    uint64_t min_count, batch_sentences, max_sentence_len;
    int32_t workers;
    uint64_t seed;
    int32_t reuse_mode; // 0 lifetime, 1 window, 2 none, 3 window_snapshot
    double table_power;
    uint64_t table_size, queue_capacity;
    int32_t ignore_delimiters;
};

struct ref_report {
    uint64_t words_trained, sentences_trained, vocab_size;
    double wall_seconds, batching_words_per_sec;
    int32_t n_epochs;
    uint64_t epoch_words[64];
    double epoch_seconds[64];
    double epoch_words_per_sec[64];
    uint64_t traffic[5];  // context_reads, context_writes, sample_reads, sample_writes, ring_hits
    uint64_t analytic[5];
};

// Synthetic Zipf corpus of the BASELINE.md §2 shapes, built the REFERENCE way
// (the bench's reference arm must not load libfw2v): token i = rank r with
// p(r) ∝ r^-s drawn by inverse CDF from Rng::derive(2312, 7743).next_double()
// (rng.hpp:16-33), token text "r<rank>", Vocabulary::build(counts, min_count)
// (corpus.cpp:117-139), sentences of sentence_len raw tokens with OOV tokens
// dropped and empty sentences skipped (what SentenceReader does with
// ignore_delimiters, corpus.cpp:162-213). tests/test_oracle.py checks it equals
// fw2v_corpus_synth_zipf id for id.
int ref_synth_corpus(uint64_t types, uint64_t tokens, double s, uint64_t sentence_len, uint64_t min_count,
                     void** out);
int ref_corpus_view(void* h, const uint64_t** counts, int32_t* vocab_size, uint64_t* n_sentences,
                    uint64_t* n_ids);
int ref_corpus_export(void* h, uint64_t* offsets, int32_t* ids);
int ref_train_corpus(void* h, const ref_config* cfg, ref_report* report);
int ref_corpus_head(void* h, uint64_t n_sentences, void** out);
void ref_corpus_free(void* h);

} // extern "C"

namespace {

thread_local std::string g_error;

int fail(const std::exception& e) {
    g_error = e.what();
    if (auto* re = dynamic_cast<const Error*>(&e)) return 1 + static_cast<int>(re->code());
    return 100;
}

// Token names zero-padded so that Vocabulary::build's (count desc, token asc)
// order equals the caller's id order whenever counts are non-increasing.
std::string token_name(int32_t id) {
    char buf[32];
    std::snprintf(buf, sizeof(buf), "w%09d", id);
    return buf;
}

Vocabulary vocab_from_counts(const uint64_t* counts, int32_t n) {
    std::unordered_map<std::string, uint64_t> m;
    m.reserve(static_cast<size_t>(n) * 2);
    for (int32_t i = 0; i < n; ++i) m[token_name(i)] = counts[i];
    Vocabulary v = Vocabulary::build(m, 1);
    if (v.size() != n) raise(ErrorCode::bad_argument, "ref_capi: zero counts are not allowed");
    for (int32_t i = 0; i < n; ++i) {
        if (v.entry(i).count != counts[i] || v.entry(i).token != token_name(i)) {
            raise(ErrorCode::bad_argument, "ref_capi: counts must be non-increasing in id order");
        }
    }
    return v;
}

TrainConfig to_cfg(const ref_config& c) {
    TrainConfig t;
    t.dim = c.dim;
    t.window = c.window;
    t.negatives = c.negatives;
    t.epochs = c.epochs;
    t.alpha0 = c.alpha0;
    t.subsample = c.subsample;
    t.min_count = c.min_count;
    t.batch_sentences = c.batch_sentences;
    t.max_sentence_len = c.max_sentence_len;
    t.workers = c.workers;
    t.seed = c.seed;
    t.reuse_mode = static_cast<ReuseMode>(c.reuse_mode);
    t.table_power = c.table_power;
    t.table_size = c.table_size;
    t.queue_capacity = c.queue_capacity;
    t.ignore_delimiters = c.ignore_delimiters != 0;
    return t;
}

void fill_counters(uint64_t* out, const TrafficCounters& t) {
    out[0] = t.context_reads;
    out[1] = t.context_writes;
    out[2] = t.sample_reads;
    out[3] = t.sample_writes;
    out[4] = t.ring_hits;
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_error.c_str(); }

void ref_config_default(ref_config* c) {
    TrainConfig t;
    c->dim = t.dim;
    c->window = t.window;
    c->negatives = t.negatives;
    c->epochs = t.epochs;
    c->alpha0 = t.alpha0;
    c->subsample = t.subsample;
    c->min_count = t.min_count;
    c->batch_sentences = t.batch_sentences;
    c->max_sentence_len = t.max_sentence_len;
    c->workers = t.workers;
    c->seed = t.seed;
    c->reuse_mode = static_cast<int32_t>(t.reuse_mode);
    c->table_power = t.table_power;
    c->table_size = t.table_size;
    c->queue_capacity = t.queue_capacity;
    c->ignore_delimiters = t.ignore_delimiters ? 1 : 0;
}

int ref_train(const uint64_t* counts, int32_t vocab_size, const uint64_t* offsets,
              uint64_t n_sentences, const int32_t* ids, const ref_config* cfg, float* out_input,
              float* out_output, ref_report* report) {
    try {
        Corpus corpus;
        corpus.vocab = vocab_from_counts(counts, vocab_size);
        corpus.sentences.resize(n_sentences);
        for (uint64_t s = 0; s < n_sentences; ++s) {
            corpus.sentences[s].ids.assign(ids + offsets[s], ids + offsets[s + 1]);
        }
        TrainResult r = train(corpus, to_cfg(*cfg));
        size_t n = r.model.input.size();
        if (out_input) std::memcpy(out_input, r.model.input.data(), n * sizeof(float));
        if (out_output) std::memcpy(out_output, r.model.output.data(), n * sizeof(float));
        if (report) {
            std::memset(report, 0, sizeof(*report));
            report->words_trained = r.report.words_trained;
            report->sentences_trained = r.report.sentences_trained;
            report->vocab_size = r.report.vocab_size;
            report->wall_seconds = r.report.wall_seconds;
            report->batching_words_per_sec = r.report.batching_words_per_sec;
            report->n_epochs = static_cast<int32_t>(r.report.epochs.size());
            for (size_t e = 0; e < r.report.epochs.size() && e < 64; ++e) {
                report->epoch_words[e] = r.report.epochs[e].words;
                report->epoch_seconds[e] = r.report.epochs[e].seconds;
                report->epoch_words_per_sec[e] = r.report.epochs[e].words_per_sec;
            }
            fill_counters(report->traffic, r.report.traffic);
            fill_counters(report->analytic, r.report.analytic);
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Serial train_sentence over a list of sentences with caller-supplied
// negatives (L*N per sentence, concatenated) and per-sentence alpha, on a
// caller-owned model (|V| x d input/output, updated in place).
int ref_train_sentences(float* input, float* output, int32_t vocab_size, int32_t dim,
                        const uint64_t* offsets, uint64_t n_sentences, const int32_t* ids,
                        const int32_t* negatives, const float* alphas, const ref_config* cfg,
                        uint64_t* counters) {
    try {
        TrainConfig tc = to_cfg(*cfg);
        tc.dim = dim;
        EmbeddingModel model;
        model.vocab_size = vocab_size;
        model.dim = dim;
        size_t n = static_cast<size_t>(vocab_size) * static_cast<size_t>(dim);
        model.input.assign(input, input + n);
        model.output.assign(output, output + n);
        TrainScratch scratch(tc.context_width(), dim, tc.negatives);
        TrafficCounters t;
        uint64_t neg_off = 0;
        for (uint64_t s = 0; s < n_sentences; ++s) {
            EncodedSentence sentence;
            sentence.ids.assign(ids + offsets[s], ids + offsets[s + 1]);
            size_t len = sentence.length();
            std::span<const int32_t> negs(negatives ? negatives + neg_off : nullptr,
                                          len * static_cast<size_t>(tc.negatives));
            train_sentence(model, sentence, negs, tc, alphas[s], t, scratch, nullptr, s);
            neg_off += len * static_cast<size_t>(tc.negatives);
        }
        std::memcpy(input, model.input.data(), n * sizeof(float));
        std::memcpy(output, model.output.data(), n * sizeof(float));
        if (counters) fill_counters(counters, t);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_init_model(int32_t vocab_size, int32_t dim, uint64_t seed, float* out_input,
                   float* out_output) {
    try {
        EmbeddingModel m = init_model(vocab_size, dim, seed);
        std::memcpy(out_input, m.input.data(), m.input.size() * sizeof(float));
        if (out_output) std::memcpy(out_output, m.output.data(), m.output.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

float ref_sigmoid(float x) { return sigmoid(x); }

float ref_lr_at(uint64_t words_trained, uint64_t total, float alpha0) {
    try {
        return lr_at(words_trained, total, alpha0);
    } catch (const std::exception& e) {
        fail(e);
        return -1.0f;
    }
}

int ref_keep_probs(const uint64_t* counts, int32_t vocab_size, double threshold, double* out) {
    try {
        Vocabulary v = vocab_from_counts(counts, vocab_size);
        std::vector<double> p = subsample_keep_probs(v, threshold);
        if (!p.empty()) std::memcpy(out, p.data(), p.size() * sizeof(double));
        return static_cast<int>(p.empty() ? 0 : 1);
    } catch (const std::exception& e) {
        return -fail(e);
    }
}

int ref_table_build(const uint64_t* counts, int32_t vocab_size, double power, uint64_t size,
                    int32_t* out_slots) {
    try {
        Vocabulary v = vocab_from_counts(counts, vocab_size);
        NegativeTable t = NegativeTable::build(v, power, size);
        for (uint64_t s = 0; s < t.size(); ++s) out_slots[s] = t.slot(s);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// One assemble_batch call on stream[cursor..]: writes the kept sentences
// (concatenated) to out_ids with out_offsets (kept+1 entries) and their L*N
// negatives to out_negs; returns the number of kept sentences and advances
// *cursor. Rng stream = Rng::derive(seed, a, b, c).
int64_t ref_assemble_batch(const uint64_t* counts, int32_t vocab_size, const uint64_t* offsets,
                           uint64_t n_sentences, const int32_t* ids, uint64_t* cursor,
                           uint64_t max_sentences, int32_t negatives, double power,
                           uint64_t table_size, double threshold, uint64_t seed, uint64_t a,
                           uint64_t b, uint64_t c, int32_t* out_ids, uint64_t* out_offsets,
                           int32_t* out_negs) {
    try {
        Vocabulary v = vocab_from_counts(counts, vocab_size);
        NegativeTable t = NegativeTable::build(v, power, table_size);
        std::vector<double> keep = subsample_keep_probs(v, threshold);
        std::vector<EncodedSentence> stream(n_sentences);
        for (uint64_t s = 0; s < n_sentences; ++s) {
            stream[s].ids.assign(ids + offsets[s], ids + offsets[s + 1]);
        }
        Rng rng = Rng::derive(seed, a, b, c);
        size_t cur = *cursor;
        SentenceBatch batch = assemble_batch(stream, cur, max_sentences, negatives, t, keep, rng);
        *cursor = cur;
        uint64_t w = 0, nw = 0;
        out_offsets[0] = 0;
        for (size_t s = 0; s < batch.sentences.size(); ++s) {
            for (int32_t id : batch.sentences[s].ids) out_ids[w++] = id;
            out_offsets[s + 1] = w;
            for (int32_t id : batch.negatives[s]) out_negs[nw++] = id;
        }
        return static_cast<int64_t>(batch.sentences.size());
    } catch (const std::exception& e) {
        return -fail(e);
    }
}

void ref_rng_draws(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t n, uint64_t* out) {
    Rng r = Rng::derive(seed, a, b, c);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

int ref_analytic_traffic(uint64_t length, int32_t width, int32_t negatives, int32_t mode,
                         uint64_t* out) {
    try {
        fill_counters(out, analytic_traffic(length, width, negatives, static_cast<ReuseMode>(mode)));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// save_embeddings of a |V| x dim matrix with the ref_capi token names
// (w%09d) and the given counts (non-increasing); which: 0 input, 1 output.
int ref_save_embeddings(const uint64_t* counts, int32_t vocab_size, int32_t dim, const float* rows,
                        int32_t which, const char* path) {
    try {
        Vocabulary v = vocab_from_counts(counts, vocab_size);
        EmbeddingModel m;
        m.vocab_size = vocab_size;
        m.dim = dim;
        const size_t n = static_cast<size_t>(vocab_size) * static_cast<size_t>(dim);
        m.input.assign(rows, rows + n);
        m.output.assign(rows, rows + n);
        save_embeddings(m, v, path, which == 0 ? MatrixKind::input : MatrixKind::output);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

LoadedEmbeddings loaded(const float* rows, int32_t n, int32_t dim) {
    LoadedEmbeddings e;
    e.count = n;
    e.dim = dim;
    e.vectors.assign(rows, rows + static_cast<size_t>(n) * dim);
    for (int32_t w = 0; w < n; ++w) {
        e.tokens.push_back(token_name(w));
        e.index[e.tokens.back()] = w;
    }
    return e;
}

// nearest_neighbors for query ids; out_ids/out_cos: n_queries x k (ids via the token names).
int ref_nearest_neighbors(const float* rows, int32_t n, int32_t dim, const int32_t* queries, int32_t n_queries,
                          int32_t k, int32_t* out_ids, double* out_cos) {
    try {
        LoadedEmbeddings e = loaded(rows, n, dim);
        for (int32_t q = 0; q < n_queries; ++q) {
            std::vector<Neighbor> nb = nearest_neighbors(e, token_name(queries[q]), k);
            for (int32_t j = 0; j < k; ++j) {
                const bool ok = j < static_cast<int32_t>(nb.size());
                out_ids[static_cast<size_t>(q) * k + j] = ok ? e.id_of(nb[static_cast<size_t>(j)].token) : -1;
                out_cos[static_cast<size_t>(q) * k + j] = ok ? nb[static_cast<size_t>(j)].cosine : 0.0;
            }
        }
        return 0;
    } catch (const std::exception& ex) {
        return fail(ex);
    }
}

// eval_analogy on each quadruple alone: correct[i] = 1 if the reference predicts quads[4i+3].
int ref_analogy_correct(const float* rows, int32_t n, int32_t dim, const int32_t* quads, int32_t nq, int32_t method,
                        int32_t* correct) {
    try {
        LoadedEmbeddings e = loaded(rows, n, dim);
        for (int32_t i = 0; i < nq; ++i) {
            std::vector<AnalogyQuadruple> one{{token_name(quads[4 * i]), token_name(quads[4 * i + 1]),
                                               token_name(quads[4 * i + 2]), token_name(quads[4 * i + 3])}};
            AnalogyResult r = eval_analogy(e, one, method == 0 ? AnalogyMethod::cos_add : AnalogyMethod::cos_mul, 1);
            correct[i] = r.accuracy == 1.0 ? 1 : 0;
        }
        return 0;
    } catch (const std::exception& ex) {
        return fail(ex);
    }
}

namespace {
struct RefCorpus {
    Corpus corpus;
    std::vector<uint64_t> counts;
};
void fill_report(ref_report* report, const RunReport& r) {
    std::memset(report, 0, sizeof(*report));
    report->words_trained = r.words_trained;
    report->sentences_trained = r.sentences_trained;
    report->vocab_size = r.vocab_size;
    report->wall_seconds = r.wall_seconds;
    report->batching_words_per_sec = r.batching_words_per_sec;
    report->n_epochs = static_cast<int32_t>(std::min<size_t>(r.epochs.size(), 64));
    for (int32_t e = 0; e < report->n_epochs; ++e) {
        report->epoch_words[e] = r.epochs[static_cast<size_t>(e)].words;
        report->epoch_seconds[e] = r.epochs[static_cast<size_t>(e)].seconds;
        report->epoch_words_per_sec[e] = r.epochs[static_cast<size_t>(e)].words_per_sec;
    }
    fill_counters(report->traffic, r.traffic);
    fill_counters(report->analytic, r.analytic);
}
} // namespace

int ref_synth_corpus(uint64_t types, uint64_t tokens, double s, uint64_t sentence_len, uint64_t min_count,
                     void** out) {
    *out = nullptr;
    try {
        if (types < 1 || sentence_len < 1) raise(ErrorCode::bad_argument, "types and sentence_len must be >= 1");
        std::vector<double> cdf(types);
        double acc = 0.0;
        for (uint64_t r = 0; r < types; ++r) cdf[r] = (acc += std::pow(static_cast<double>(r + 1), -s));
        for (double& v : cdf) v /= acc;
        cdf[types - 1] = 1.0;
        Rng rng = Rng::derive(2312, 7743);
        std::vector<uint32_t> rank(tokens);
        std::vector<uint64_t> count(types, 0);
        for (uint64_t i = 0; i < tokens; ++i) {
            const double u = rng.next_double();
            const uint64_t r = static_cast<uint64_t>(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
            rank[i] = static_cast<uint32_t>(std::min(r, types - 1));
            ++count[rank[i]];
        }
        std::unordered_map<std::string, uint64_t> m;
        m.reserve(types * 2);
        for (uint64_t r = 0; r < types; ++r)
            if (count[r] > 0) m["r" + std::to_string(r + 1)] = count[r];
        auto c = std::make_unique<RefCorpus>();
        c->corpus.vocab = Vocabulary::build(m, min_count);
        std::vector<int32_t> remap(types, -1);
        for (uint64_t r = 0; r < types; ++r)
            if (count[r] > 0) remap[r] = c->corpus.vocab.id_of("r" + std::to_string(r + 1));
        for (uint64_t t0 = 0; t0 < tokens; t0 += sentence_len) {
            EncodedSentence es;
            for (uint64_t i = t0; i < std::min(tokens, t0 + sentence_len); ++i)
                if (remap[rank[i]] >= 0) es.ids.push_back(remap[rank[i]]);
            if (!es.empty()) c->corpus.sentences.push_back(std::move(es));
        }
        c->corpus.raw_tokens = tokens;
        for (int32_t w = 0; w < c->corpus.vocab.size(); ++w) c->counts.push_back(c->corpus.vocab.entry(w).count);
        *out = c.release();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_corpus_view(void* h, const uint64_t** counts, int32_t* vocab_size, uint64_t* n_sentences, uint64_t* n_ids) {
    auto* c = static_cast<RefCorpus*>(h);
    *counts = c->counts.data();
    *vocab_size = c->corpus.vocab.size();
    *n_sentences = c->corpus.sentences.size();
    *n_ids = c->corpus.encoded_tokens();
    return 0;
}

int ref_corpus_export(void* h, uint64_t* offsets, int32_t* ids) {
    auto* c = static_cast<RefCorpus*>(h);
    offsets[0] = 0;
    for (size_t k = 0; k < c->corpus.sentences.size(); ++k) {
        const auto& v = c->corpus.sentences[k].ids;
        std::memcpy(ids + offsets[k], v.data(), v.size() * sizeof(int32_t));
        offsets[k + 1] = offsets[k] + v.size();
    }
    return 0;
}

// ringvec::train on the held corpus (trainer.cpp:390), model discarded.
int ref_train_corpus(void* h, const ref_config* cfg, ref_report* report) {
    try {
        TrainResult r = train(static_cast<RefCorpus*>(h)->corpus, to_cfg(*cfg));
        if (report) fill_report(report, r.report);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The first n sentences, same vocabulary (a bounded sample of the workload).
int ref_corpus_head(void* h, uint64_t n_sentences, void** out) {
    try {
        auto* c = static_cast<RefCorpus*>(h);
        auto d = std::make_unique<RefCorpus>();
        d->corpus.vocab = c->corpus.vocab;
        d->counts = c->counts;
        const uint64_t n = std::min<uint64_t>(n_sentences, c->corpus.sentences.size());
        d->corpus.sentences.assign(c->corpus.sentences.begin(), c->corpus.sentences.begin() + static_cast<ptrdiff_t>(n));
        *out = d.release();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void ref_corpus_free(void* h) { delete static_cast<RefCorpus*>(h); }

} // extern "C"
