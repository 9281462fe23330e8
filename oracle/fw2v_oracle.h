/* CPU restatement of the reference SGNS training path — TEST INFRASTRUCTURE.
 *
 * This is the checker for the B200 product, never the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it. Every
 * function restates one reference function (file:line under
 * /root/reference/proj) in plain C with the same floating-point operation
 * order (no FMA contraction: built with -ffp-contract=off), so that it is
 * bit-identical to the reference built with its default flags. It is pinned
 * against the reference itself (oracle/_ref/libringvec_refcapi.so) and the
 * committed golden fixtures in tests/golden/ by tests/test_oracle.py.
 *
 * Scope: the deterministic (workers = 1) semantics of ringvec::train, i.e.
 * one producer stream p = 0 and serial consumption (SURVEY.md §8a recipe).
 */
#ifndef FW2V_ORACLE_H
#define FW2V_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Field-for-field mirror of ringvec::TrainConfig (config.hpp:13-35). */
typedef struct oracle_config {
    int32_t dim, window, negatives, epochs;
    float alpha0;
    double subsample;
    uint64_t min_count, batch_sentences, max_sentence_len;
    int32_t workers;
    uint64_t seed;
    int32_t reuse_mode; /* 0 lifetime, 1 window, 2 none, 3 window_snapshot (traffic.hpp:15) */
    double table_power;
    uint64_t table_size, queue_capacity;
    int32_t ignore_delimiters;
} oracle_config;

typedef struct oracle_report {
    uint64_t words_trained, sentences_trained, vocab_size;
    double wall_seconds, batching_words_per_sec;
    int32_t n_epochs;
    uint64_t epoch_words[64];
    double epoch_seconds[64];
    double epoch_words_per_sec[64];
    uint64_t traffic[5]; /* context_reads, context_writes, sample_reads, sample_writes, ring_hits */
    uint64_t analytic[5];
} oracle_report;

/* rng.hpp:11-45 (splitmix64) */
uint64_t oracle_rng_mix(uint64_t z);
void oracle_rng_draws(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t n, uint64_t* out);

/* model.cpp:15-45 */
int oracle_init_model(int32_t vocab_size, int32_t dim, uint64_t seed, float* input, float* output);
float oracle_sigmoid(float x);
float oracle_lr_at(uint64_t words_trained, uint64_t total, float alpha0);

/* kernels.hpp:10-38 */
float oracle_dot(const float* a, const float* b, int32_t d);

/* corpus.cpp:215-241 ; returns 1 if subsampling is enabled (probs written), 0 otherwise */
int oracle_keep_probs(const uint64_t* counts, int32_t vocab_size, double threshold, double* out);

/* sampler.cpp:9-35 */
int oracle_table_build(const uint64_t* counts, int32_t vocab_size, double power, uint64_t size,
                       int32_t* out_slots);

/* sampler.cpp:41-63 with the Rng stream derive(seed, a, b, c); same contract as
 * ref_assemble_batch in oracle/ref_capi.cpp. */
int64_t oracle_assemble_batch(const uint64_t* counts, int32_t vocab_size, const uint64_t* offsets,
                              uint64_t n_sentences, const int32_t* ids, uint64_t* cursor,
                              uint64_t max_sentences, int32_t negatives, double power,
                              uint64_t table_size, double threshold, uint64_t seed, uint64_t a,
                              uint64_t b, uint64_t c, int32_t* out_ids, uint64_t* out_offsets,
                              int32_t* out_negs);

/* trainer.cpp:332-356 over a list of sentences (serial), all four reuse modes. */
int oracle_train_sentences(float* input, float* output, int32_t vocab_size, int32_t dim,
                           const uint64_t* offsets, uint64_t n_sentences, const int32_t* ids,
                           const int32_t* negatives, const float* alphas, const oracle_config* cfg,
                           uint64_t* counters);

/* trainer.cpp:390-528 with workers = 1 (deterministic). */
int oracle_train(const uint64_t* counts, int32_t vocab_size, const uint64_t* offsets,
                 uint64_t n_sentences, const int32_t* ids, const oracle_config* cfg,
                 float* out_input, float* out_output, oracle_report* report);

/* traffic.cpp:21-59 */
int oracle_analytic_traffic(uint64_t length, int32_t width, int32_t negatives, int32_t mode,
                            uint64_t* out);

const char* oracle_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
