// A reference-side user program of the ringvec::train drop-in, as a shared
// library for bench.py's drop-in e2e leg: it owns a ringvec::Corpus (built by
// the reference's own Vocabulary::build) and times whole ringvec::train calls
// (trainer.hpp:119-121) — context setup (tables, HBM model, init_model), host
// batching, H2D, kernels, model readback into EmbeddingModel and teardown —
// exactly what a reference user pays per call.
//
// Linked from the reference's sources (config/corpus/model/... compiled where
// they lie, trainer.cpp excluded) plus libringvec_fw2v.so, which supplies
// train(); see Makefile target `harness`. Not on the training path.
#include <chrono>
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
#include "ringvec/trainer.hpp"

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (auto* re = dynamic_cast<const ringvec::Error*>(&e)) return 1 + static_cast<int>(re->code());
    return 100;
}
} // namespace

extern "C" {

// ringvec::TrainConfig (config.hpp:13-35), field for field.
struct fw2v_harness_config {
    int32_t dim, window, negatives, epochs;
    float alpha0;
    double subsample;
    uint64_t min_count, batch_sentences, max_sentence_len;
    int32_t workers;
    uint64_t seed;
    int32_t reuse_mode;
    double table_power;
    uint64_t table_size, queue_capacity;
    int32_t ignore_delimiters;
};

struct fw2v_harness_result {
    double call_seconds;      // wall clock of the whole ringvec::train call
    double epoch_words_per_sec;  // RunReport.epochs[0].words_per_sec (train()'s own epoch timer)
    uint64_t words_trained;
    double input_checksum;    // sum of EmbeddingModel::input (the readback happened)
};

const char* fw2v_harness_last_error(void) { return g_err.c_str(); }

// Corpus from vocabulary-ordered counts (non-increasing) and flat sentences; the
// vocabulary is built by Vocabulary::build from token names that sort like ids.
int fw2v_harness_corpus(const uint64_t* counts, int32_t vocab_size, const uint64_t* offsets, uint64_t n_sentences,
                        const int32_t* ids, void** out) {
    *out = nullptr;
    try {
        auto name = [](int32_t i) {
            char b[24];
            std::snprintf(b, sizeof(b), "w%09d", i);
            return std::string(b);
        };
        std::unordered_map<std::string, uint64_t> m;
        m.reserve(static_cast<size_t>(vocab_size) * 2);
        for (int32_t i = 0; i < vocab_size; ++i) m[name(i)] = counts[i];
        auto c = std::make_unique<ringvec::Corpus>();
        c->vocab = ringvec::Vocabulary::build(m, 1);
        if (c->vocab.size() != vocab_size) ringvec::raise(ringvec::ErrorCode::bad_argument, "zero counts");
        c->sentences.resize(n_sentences);
        for (uint64_t s = 0; s < n_sentences; ++s) c->sentences[s].ids.assign(ids + offsets[s], ids + offsets[s + 1]);
        *out = c.release();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int fw2v_harness_train(void* corpus, const fw2v_harness_config* hc, fw2v_harness_result* res) {
    try {
        ringvec::TrainConfig c;
        c.dim = hc->dim;
        c.window = hc->window;
        c.negatives = hc->negatives;
        c.epochs = hc->epochs;
        c.alpha0 = hc->alpha0;
        c.subsample = hc->subsample;
        c.min_count = hc->min_count;
        c.batch_sentences = hc->batch_sentences;
        c.max_sentence_len = hc->max_sentence_len;
        c.workers = hc->workers;
        c.seed = hc->seed;
        c.reuse_mode = static_cast<ringvec::ReuseMode>(hc->reuse_mode);
        c.table_power = hc->table_power;
        c.table_size = hc->table_size;
        c.queue_capacity = hc->queue_capacity;
        c.ignore_delimiters = hc->ignore_delimiters != 0;
        const auto t0 = std::chrono::steady_clock::now();
        double checksum = 0.0;
        uint64_t words = 0;
        double ewps = 0.0;
        {
            ringvec::TrainResult r = ringvec::train(*static_cast<ringvec::Corpus*>(corpus), c);
            for (size_t i = 0; i < r.model.input.size(); i += 4099) checksum += r.model.input[i];
            words = r.report.words_trained;
            ewps = r.report.epochs.empty() ? 0.0 : r.report.epochs[0].words_per_sec;
        }  // the result (2 x |V| x d floats) is freed inside the timed call, as a caller's would be
        res->call_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        res->words_trained = words;
        res->epoch_words_per_sec = ewps;
        res->input_checksum = checksum;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void fw2v_harness_free(void* corpus) { delete static_cast<ringvec::Corpus*>(corpus); }

} // extern "C"
