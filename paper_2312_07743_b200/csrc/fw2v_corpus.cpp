// Synthetic Zipf corpora of the benchmark shapes: the bench
// input, generated in-process so nothing corpus-sized crosses gpurun.
//
// Token i takes splitmix64 draw i of Rng::derive(2312, 7743) as next_double
// (rng.hpp:33) and maps it through the inverse CDF of p(r) ∝ r^-s by binary
// search. Because splitmix64 is counter based, draw i = mix(state0 + (i+1)·φ),
// so generation is split across threads with a bit-identical result.
// The vocabulary follows Vocabulary::build (corpus.cpp:117-139): ranks with
// count >= min_count, count descending, ties by token name "r<rank>"; sentences
// are cut every sentence_len raw tokens with OOV tokens dropped and empty
// sentences skipped (SentenceReader, corpus.cpp:162-213).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "fw2v.h"

struct fw2v_corpus {
    std::vector<uint64_t> counts;
    std::vector<uint64_t> offsets;
    std::vector<int32_t> ids;
};

namespace {

inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t derive_state(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
    uint64_t s = mix64(seed);
    s = mix64(s ^ mix64(a + 0x9e3779b97f4a7c15ULL));
    s = mix64(s ^ mix64(b + 0xbf58476d1ce4e5b9ULL));
    s = mix64(s ^ mix64(c + 0x94d049bb133111ebULL));
    return s;
}

template <class F>
void parallel_for(uint64_t n, int threads, F&& f) {
    threads = std::max(1, threads);
    std::vector<std::thread> ts;
    const uint64_t chunk = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const uint64_t b = std::min(n, chunk * t), e = std::min(n, b + chunk);
        ts.emplace_back([&, t, b, e] { f(t, b, e); });
    }
    for (auto& th : ts) th.join();
}

} // namespace

extern "C" {

int fw2v_corpus_synth_zipf(uint64_t types, uint64_t tokens, double s, uint64_t sentence_len,
                           uint64_t min_count, int32_t threads, fw2v_corpus** out) {
    *out = nullptr;
    if (types < 1 || sentence_len < 1 || types > (1ull << 31)) return FW2V_ERR_BAD_ARGUMENT;
    if (threads <= 0) threads = static_cast<int32_t>(std::max(1u, std::thread::hardware_concurrency()));
    auto c = std::make_unique<fw2v_corpus>();
    // Inverse CDF over ranks 1..types.
    std::vector<double> cdf(types);
    double acc = 0.0;
    for (uint64_t r = 0; r < types; ++r) cdf[r] = (acc += std::pow(static_cast<double>(r + 1), -s));
    for (double& v : cdf) v /= acc;
    cdf[types - 1] = 1.0;
    // Guide table: bucket of u -> first candidate rank.
    const uint32_t G = 1u << 20;
    std::vector<uint32_t> guide(G + 1);
    {
        uint64_t r = 0;
        for (uint32_t g = 0; g <= G; ++g) {
            const double u = static_cast<double>(g) / G;
            while (r + 1 < types && cdf[r] <= u) ++r;
            guide[g] = static_cast<uint32_t>(r);
        }
    }
    const uint64_t state0 = derive_state(2312, 7743, 0, 0);
    std::vector<uint32_t> rank(tokens);
    std::vector<std::vector<uint64_t>> hist(static_cast<size_t>(threads), std::vector<uint64_t>(types, 0));
    parallel_for(tokens, threads, [&](int t, uint64_t b, uint64_t e) {
        auto& h = hist[static_cast<size_t>(t)];
        for (uint64_t i = b; i < e; ++i) {
            const uint64_t x = mix64(state0 + (i + 1) * 0x9e3779b97f4a7c15ULL);
            const double u = static_cast<double>(x >> 11) * 0x1.0p-53;
            const uint32_t g = static_cast<uint32_t>(u * G);
            uint64_t lo = guide[g], hi = guide[std::min(g + 1, G)];
            // first r in [lo, hi] with cdf[r] > u
            while (lo < hi) {
                const uint64_t mid = (lo + hi) / 2;
                if (cdf[mid] > u) hi = mid; else lo = mid + 1;
            }
            rank[i] = static_cast<uint32_t>(lo);
            ++h[lo];
        }
    });
    std::vector<uint64_t> count(types, 0);
    for (auto& h : hist)
        for (uint64_t r = 0; r < types; ++r) count[r] += h[r];
    hist.clear();
    // Vocabulary::build order: count desc, then token name asc ("r<rank+1>").
    std::vector<uint32_t> order;
    for (uint64_t r = 0; r < types; ++r)
        if (count[r] >= min_count && count[r] > 0) order.push_back(static_cast<uint32_t>(r));
    if (order.empty()) return FW2V_ERR_EMPTY_VOCAB;
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
        if (count[a] != count[b]) return count[a] > count[b];
        return std::to_string(a + 1) < std::to_string(b + 1);  // "r" prefix common
    });
    std::vector<int32_t> remap(types, -1);
    c->counts.resize(order.size());
    for (size_t i = 0; i < order.size(); ++i) {
        remap[order[i]] = static_cast<int32_t>(i);
        c->counts[i] = count[order[i]];
    }
    // Sentences of sentence_len raw tokens; OOV dropped; empty skipped.
    const uint64_t n_raw = (tokens + sentence_len - 1) / sentence_len;
    std::vector<uint64_t> kept(n_raw, 0);
    parallel_for(n_raw, threads, [&](int, uint64_t b, uint64_t e) {
        for (uint64_t sidx = b; sidx < e; ++sidx) {
            const uint64_t t0 = sidx * sentence_len, t1 = std::min(tokens, t0 + sentence_len);
            uint64_t k = 0;
            for (uint64_t i = t0; i < t1; ++i) k += remap[rank[i]] >= 0;
            kept[sidx] = k;
        }
    });
    std::vector<uint64_t> pos(n_raw + 1, 0);
    for (uint64_t sidx = 0; sidx < n_raw; ++sidx) pos[sidx + 1] = pos[sidx] + kept[sidx];
    c->ids.resize(pos[n_raw]);
    parallel_for(n_raw, threads, [&](int, uint64_t b, uint64_t e) {
        for (uint64_t sidx = b; sidx < e; ++sidx) {
            const uint64_t t0 = sidx * sentence_len, t1 = std::min(tokens, t0 + sentence_len);
            uint64_t w = pos[sidx];
            for (uint64_t i = t0; i < t1; ++i) {
                const int32_t id = remap[rank[i]];
                if (id >= 0) c->ids[w++] = id;
            }
        }
    });
    c->offsets.reserve(n_raw + 1);
    c->offsets.push_back(0);
    for (uint64_t sidx = 0; sidx < n_raw; ++sidx)
        if (kept[sidx] > 0) c->offsets.push_back(pos[sidx + 1]);
    *out = c.release();
    return FW2V_OK;
}

int fw2v_corpus_view(const fw2v_corpus* c, const uint64_t** counts, int32_t* vocab_size,
                     const uint64_t** offsets, uint64_t* n_sentences, const int32_t** ids,
                     uint64_t* n_ids) {
    if (counts) *counts = c->counts.data();
    if (vocab_size) *vocab_size = static_cast<int32_t>(c->counts.size());
    if (offsets) *offsets = c->offsets.data();
    if (n_sentences) *n_sentences = c->offsets.size() - 1;
    if (ids) *ids = c->ids.data();
    if (n_ids) *n_ids = c->ids.size();
    return FW2V_OK;
}

void fw2v_corpus_free(fw2v_corpus* c) { delete c; }

} // extern "C"
