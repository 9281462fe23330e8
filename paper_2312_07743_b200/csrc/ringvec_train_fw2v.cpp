// Drop-in ringvec::train (reference trainer.hpp:119-121) on the B200 trainer.
//
// Built against the reference's public headers; linked in place of the
// reference's trainer.cpp `train` definition (oracle/Makefile links the
// reference suites against it with trainer.cpp compiled as
// -Dtrain=ringvec_reference_cpu_train). Everything below the C-ABI
// (include/fw2v.h) is B200 code; this file only converts types:
//   TrainConfig  -> fw2v_config (+ GPU knobs from FW2V_* environment variables,
//                   since TrainConfig has no GPU fields)
//   Corpus       -> flat offsets/ids arrays
//   fw2v status  -> ringvec::Error{ErrorCode(status - 1)} (error.hpp:8-37)
//   fw2v_report  -> RunReport / EpochStats, observer and on_epoch trampolines.
// workers == 1 selects the serial bit-exact engine (reference: "workers == 1
// is fully deterministic", trainer.hpp:115-118); workers > 1 the Hogwild path.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "fw2v.h"
#include "ringvec/config.hpp"
#include "ringvec/error.hpp"
#include "ringvec/model.hpp"
#include "ringvec/trainer.hpp"

namespace ringvec {

namespace {

[[noreturn]] void raise_status(int status) {
    std::string msg = fw2v_last_error();
    if (status >= 1 && status <= 13) raise(static_cast<ErrorCode>(status - 1), msg);
    throw std::runtime_error("fw2v: " + msg);
}

int env_int(const char* name, int fallback) {
    const char* v = std::getenv(name);
    return (v && *v) ? std::atoi(v) : fallback;
}

struct Callbacks {
    TrainObserver* observer;
    const std::function<void(const EpochStats&)>* on_epoch;
    std::vector<EpochStats> epochs;
};

void observer_tramp(void* user, uint64_t serial, uint64_t target) {
    static_cast<Callbacks*>(user)->observer->on_target(serial, static_cast<size_t>(target));
}

void epoch_tramp(void* user, const fw2v_epoch_stats* s) {
    EpochStats e;
    e.epoch = s->epoch;
    e.words = s->words;
    e.seconds = s->seconds;
    e.words_per_sec = s->words_per_sec;
    auto* cb = static_cast<Callbacks*>(user);
    cb->epochs.push_back(e);
    if (*cb->on_epoch) (*cb->on_epoch)(e);
}

TrafficCounters to_counters(const fw2v_counters& c) {
    TrafficCounters t;
    t.context_reads = c.context_reads;
    t.context_writes = c.context_writes;
    t.sample_reads = c.sample_reads;
    t.sample_writes = c.sample_writes;
    t.ring_hits = c.ring_hits;
    return t;
}

} // namespace

TrainResult train(const Corpus& corpus, const TrainConfig& raw_config, TrainObserver* observer,
                  const std::function<void(const EpochStats&)>& on_epoch) {
    TrainConfig cfg = resolve_config(raw_config);  // config.cpp:190
    validate_config(cfg);                          // config.cpp:165
    const Vocabulary& vocab = corpus.vocab;
    if (vocab.size() < 1) raise(ErrorCode::empty_vocab, "corpus has an empty vocabulary");

    fw2v_config c;
    fw2v_config_default(&c);
    c.dim = cfg.dim;
    c.window = cfg.window;
    c.negatives = cfg.negatives;
    c.epochs = cfg.epochs;
    c.alpha0 = cfg.alpha0;
    c.subsample = cfg.subsample;
    c.min_count = cfg.min_count;
    c.batch_sentences = cfg.batch_sentences;
    c.max_sentence_len = cfg.max_sentence_len;
    c.workers = cfg.workers;
    c.seed = cfg.seed;
    c.reuse_mode = static_cast<int32_t>(cfg.reuse_mode);
    c.table_power = cfg.table_power;
    c.table_size = cfg.table_size;
    c.queue_capacity = cfg.queue_capacity;
    c.ignore_delimiters = cfg.ignore_delimiters ? 1 : 0;
    c.device = env_int("FW2V_DEVICE", 0);
    c.deterministic = env_int("FW2V_DETERMINISTIC", -1);
    // Hogwild runs draw negatives from the unigram^0.75 alias table (north_star's
    // throughput sampler; same stream positions, so the same sentences are kept);
    // deterministic runs always use the reference slot table (fw2v_ctx::sampler).
    c.sampler = env_int("FW2V_SAMPLER", FW2V_SAMPLER_ALIAS);
    c.fast_sigmoid = env_int("FW2V_FAST_SIGMOID", 1);
    c.k1_lanes = env_int("FW2V_K1_LANES", 0);
    c.streams = env_int("FW2V_STREAMS", 0);
    c.l1_refresh_log2 = env_int("FW2V_L1_REFRESH_LOG2", c.l1_refresh_log2);
    c.delta_writeback = env_int("FW2V_DELTA_WRITEBACK", c.delta_writeback);
    c.max_inflight = env_int("FW2V_MAX_INFLIGHT", c.max_inflight);
    // Hot-row replicas spread the L2 reductions on the most frequent output rows;
    // the live merge (hot_merge = 1) hands every replica the others' updates within
    // microseconds, so the rows keep plain Hogwild's update rule (full step).
    // FW2V_HOT_MERGE=0 selects round 1's pass-end mean (1/R step on those rows).
    c.hot_rows = env_int("FW2V_HOT_ROWS", c.hot_rows);
    c.hot_replicas = env_int("FW2V_HOT_REPLICAS", c.hot_replicas);
    c.hot_merge = env_int("FW2V_HOT_MERGE", c.hot_merge);

    std::vector<uint64_t> counts(static_cast<size_t>(vocab.size()));
    for (int32_t w = 0; w < vocab.size(); ++w) counts[static_cast<size_t>(w)] = vocab.entry(w).count;

    // FW2V_GPUS = G > 1 (Hogwild only): data-parallel replicas on devices
    // FW2V_DEVICE .. FW2V_DEVICE+G-1, contiguous corpus shards, replicas averaged
    // every FW2V_AVERAGE_WORDS trained words per GPU (NCCL over NVLink) and after
    // every epoch (fw2v_train_corpus_multi). All replicas start from the same
    // init_model(seed).
    const int gpus = std::max(1, env_int("FW2V_GPUS", 1));
    const bool serial = c.deterministic == 1 || (c.deterministic < 0 && c.workers == 1);
    const int n_ctx = serial ? 1 : gpus;
    struct Guard {
        std::vector<fw2v_ctx*> p;
        ~Guard() {
            for (fw2v_ctx* x : p) fw2v_destroy(x);
        }
    } guard;
    int rc = FW2V_OK;
    for (int g = 0; g < n_ctx; ++g) {
        fw2v_config cg = c;
        cg.device = c.device + g;
        fw2v_ctx* x = nullptr;
        rc = fw2v_create(&cg, counts.data(), vocab.size(), &x);
        if (rc != FW2V_OK) raise_status(rc);
        guard.p.push_back(x);
    }
    fw2v_ctx* ctx = guard.p[0];

    std::vector<uint64_t> offsets(corpus.sentences.size() + 1, 0);
    for (size_t s = 0; s < corpus.sentences.size(); ++s) offsets[s + 1] = offsets[s] + corpus.sentences[s].length();
    // Flattened on all host cores (67 MB for the text8 shape: ~20 ms on one).
    std::vector<int32_t> ids(offsets.back());
    {
        const size_t ns = corpus.sentences.size();
        const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        for (unsigned t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                for (size_t s = ns * t / nt; s < ns * (t + 1) / nt; ++s)
                    if (!corpus.sentences[s].ids.empty())
                        std::memcpy(ids.data() + offsets[s], corpus.sentences[s].ids.data(),
                                    sizeof(int32_t) * corpus.sentences[s].length());
            });
        for (auto& x : th) x.join();
    }

    Callbacks cb{observer, &on_epoch, {}};
    fw2v_report rep{};
    if (n_ctx == 1) {
        rc = fw2v_train_corpus(ctx, offsets.data(), corpus.sentences.size(), ids.data(),
                               observer ? observer_tramp : nullptr, &cb, epoch_tramp, &cb, &rep);
    } else {
        const char* aw = std::getenv("FW2V_AVERAGE_WORDS");
        const uint64_t average_words = (aw && *aw) ? std::strtoull(aw, nullptr, 10) : uint64_t{25000000};
        rc = fw2v_train_corpus_multi(guard.p.data(), n_ctx, 0, n_ctx, offsets.data(), corpus.sentences.size(),
                                     ids.data(), average_words, nullptr, nullptr, observer ? observer_tramp : nullptr,
                                     &cb, epoch_tramp, &cb, &rep);
    }
    if (rc != FW2V_OK) raise_status(rc);

    TrainResult result;
    EmbeddingModel& m = result.model;
    m.vocab_size = vocab.size();
    m.dim = cfg.dim;
    const size_t n = static_cast<size_t>(vocab.size()) * static_cast<size_t>(cfg.dim);
    m.input.resize(n);
    m.output.resize(n);
    rc = fw2v_get_model(ctx, m.input.data(), m.output.data());
    if (rc != FW2V_OK) raise_status(rc);
    m.words_trained.store(rep.words_trained);

    RunReport& r = result.report;
    r.config = cfg;
    r.vocab_size = static_cast<uint64_t>(vocab.size());
    r.words_trained = rep.words_trained;
    r.sentences_trained = rep.sentences_trained;
    r.wall_seconds = rep.wall_seconds;
    r.batching_words_per_sec = rep.batching_words_per_sec;
    r.traffic = to_counters(rep.traffic);
    r.analytic = to_counters(rep.analytic);
    r.epochs = cb.epochs;
    return result;
}

} // namespace ringvec
