/* fw2v — C-ABI of the B200 FULL-W2V SGNS trainer (libfw2v.so).
 *
 * This is the drop-in seam under the reference's C++ trainer API
 * (ringvec::train, /root/reference/proj/include/ringvec/trainer.hpp:119-121):
 * plain pointers and sizes, no C++ or torch types, int status codes plus a
 * thread-local last-error string. The C++ shim
 * paper_2312_07743_b200/csrc/ringvec_train_fw2v.cpp implements ringvec::train on
 * top of it; Python reaches it through ctypes (paper_2312_07743_b200/fw2v.py).
 *
 * Reference interfaces each entry point replaces are cited per declaration.
 * Ownership: caller-owned host memory; context-owned device and pinned memory.
 * Threading: one context per device; calls on one context are serialised by
 * the caller; fw2v_train_corpus spawns and joins its own batching threads.
 */
#ifndef FW2V_H
#define FW2V_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FW2V_ABI_VERSION 1

/* Status codes. 1..13 are ringvec::ErrorCode + 1 (error.hpp:8-22) so the C++
 * shim maps them back onto ringvec::Error without a table. */
enum fw2v_status {
    FW2V_OK = 0,
    FW2V_ERR_IO = 1,
    FW2V_ERR_INVALID_UTF8 = 2,
    FW2V_ERR_EMPTY_VOCAB = 3,
    FW2V_ERR_BAD_ARGUMENT = 4,
    FW2V_ERR_BAD_CONFIG = 5,
    FW2V_ERR_OOV_QUERY = 11,
    FW2V_ERR_ZERO_VECTOR = 12,
    FW2V_ERR_CUDA = 64,        /* CUDA runtime failure (message has the CUDA error string) */
    FW2V_ERR_UNSUPPORTED = 65, /* shape the B200 kernels do not cover (e.g. W_f > 5 on K1) */
    FW2V_ERR_NO_DEVICE = 66,   /* no CUDA device: there is no CPU fallback by design */
    FW2V_ERR_DIVERGED = 67     /* Hogwild training stayed diverged (non-finite or |x| >= 1e6) after the divergence guard's retries */
};

enum fw2v_reuse_mode { /* ringvec::ReuseMode (traffic.hpp:15) */
    FW2V_REUSE_LIFETIME = 0,
    FW2V_REUSE_WINDOW = 1,
    FW2V_REUSE_NONE = 2,
    FW2V_REUSE_WINDOW_SNAPSHOT = 3
};

enum fw2v_sampler {
    FW2V_SAMPLER_REFERENCE = 0, /* reference slot table + splitmix64 streams (sampler.cpp:9-63), exact */
    FW2V_SAMPLER_ALIAS = 1      /* unigram^0.75 alias table + fast stream (throughput mode) */
};

/* ringvec::TrainConfig (config.hpp:13-35), field for field, followed by the
 * B200 extension (fields the reference does not have). */
typedef struct fw2v_config {
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
    /* ---- B200 extension ---- */
    int32_t device;        /* CUDA ordinal */
    int32_t deterministic; /* -1: auto (workers == 1), 0: Hogwild streams, 1: serial exact (K2) */
    int32_t sampler;       /* enum fw2v_sampler */
    int32_t fast_sigmoid;  /* K1 sigmoid: 1 tanh.approx (|err| < 1e-3), 0 expf */
    int32_t k1_lanes;      /* 0 = auto; else lanes per sentence (4, 8, 16, 32) */
    int32_t streams;       /* 0 = workers; batching threads, one CUDA stream each */
    int32_t l1_refresh_log2; /* K1s Hogwild sample reads are staged through L1: 0 = each warp drops its
                                SM's L1 every window (exact per-sentence order); k > 0 = one warp per
                                block refreshes the L1 every 2^k windows (bounded staleness for
                                Zipf-hot rows) */
    int32_t delta_writeback; /* Hogwild write-back of ring (context) rows: 2 = stored straight back
                                when they leave the ring (Hogwild overwrite like the reference's
                                memcpy, K1s keeps no shared-memory ring: the fastest, default);
                                1 = red.add(final - loaded): concurrent sentences never overwrite
                                each other's updates; 0 = overwrite in the reference's exact
                                per-sentence order (finish() slot order; exactness tests) */
    int32_t max_inflight;  /* Hogwild: sentences in flight on the device at once, summed over the
                              streams. 0 = auto (collision budget from the vocabulary, see DESIGN.md
                              §5), -1 = unlimited (every sentence of a batch in one launch) */
    int32_t hot_rows;      /* K1s Hogwild: output rows of the hot_rows most frequent words are trained
                              as hot_replicas data-parallel replicas (sentence s -> replica s mod R),
                              broadcast before and averaged after every pass; removes the L2
                              contention and the stale-update pile-up on Zipf-hot rows. 0 = off */
    int32_t hot_replicas;
    int32_t replica_merge; /* data-parallel rounds (fw2v_train_corpus_multi), per element with b the
                              replicas' common value at the round start and d_r = v_r - b:
                              0 mean: mean of the replicas (model averaging; every update scaled by
                              1/replicas); 1 touched: b + sum d_r / #{r: d_r != 0} (an element only
                              one shard trained keeps its full update, others get the mean);
                              2 sum: b + sum d_r (every update applied, like Hogwild with the round as
                              staleness) */
    int32_t divergence_guard; /* Hogwild fw2v_train_corpus: 1 = keep the model of the epoch start in HBM
                                 and check the model after the epoch (every value finite and below 1e6
                                 in magnitude: a Hogwild blow-up); if not, restore it,
                                 halve the in-flight budget and train the epoch again (up to 4 times,
                                 then FW2V_ERR_DIVERGED). 0 = off (no snapshot, no check) */
    int32_t hot_merge;    /* hot-row replicas (hot_rows > 0): 1 = live: a resident merge block sums every
                             replica's updates into the others every few microseconds during the pass, so
                             the hot rows take plain Hogwild's full step (default); 0 = mean of the replicas
                             at the end of each pass (each replica's updates count 1/hot_replicas) */
} fw2v_config;

enum fw2v_replica_merge { FW2V_MERGE_MEAN = 0, FW2V_MERGE_TOUCHED = 1, FW2V_MERGE_SUM = 2 };

/* ringvec::TrafficCounters (traffic.hpp:19-40) plus totals. */
typedef struct fw2v_counters {
    uint64_t context_reads, context_writes, sample_reads, sample_writes, ring_hits;
    uint64_t words, sentences;
} fw2v_counters;

/* ringvec::EpochStats (config.hpp:56-61) */
typedef struct fw2v_epoch_stats {
    int32_t epoch;
    uint64_t words;
    double seconds;
    double words_per_sec;
} fw2v_epoch_stats;

/* ringvec::RunReport (config.hpp:65-75), numeric part. */
typedef struct fw2v_report {
    uint64_t words_trained, sentences_trained, vocab_size;
    double wall_seconds, batching_words_per_sec;
    int32_t n_epochs;
    fw2v_counters traffic;  /* instrumented on the device */
    fw2v_counters analytic; /* per-sentence closed forms (traffic.cpp:21-59) */
    double kernel_seconds;  /* device span of the training passes (CUDA events on the launching streams,
                               pass start to last kernel completion), summed over passes */
    uint64_t h2d_bytes;     /* bytes copied host->device by the batch pipeline */
    int32_t guard_retries;  /* epochs the divergence guard restored and trained again */
} fw2v_report;

/* Called once per target, in processing order, replayed per batch
 * (ringvec::TrainObserver::on_target, trainer.hpp:82-87). */
typedef void (*fw2v_observer_fn)(void* user, uint64_t sentence_serial, uint64_t target_index);
/* Called after each epoch on the calling thread (train's on_epoch, trainer.cpp:514). */
typedef void (*fw2v_epoch_fn)(void* user, const fw2v_epoch_stats* stats);

typedef struct fw2v_ctx fw2v_ctx;
typedef struct fw2v_plan fw2v_plan;

int fw2v_abi_version(void);
const char* fw2v_last_error(void);
/* TrainConfig defaults (config.hpp:14-29) plus extension defaults. */
void fw2v_config_default(fw2v_config* cfg);
/* validate_config (config.cpp:165-188): 0 or FW2V_ERR_BAD_CONFIG. */
int fw2v_validate_config(const fw2v_config* cfg);
int fw2v_device_count(int* count);

/* Creates a trainer for a vocabulary given by its counts in id order
 * (Vocabulary, corpus.hpp:21-48; ids are count-descending). Builds the
 * subsampling keep-probs (corpus.cpp:221), the negative sampler
 * (sampler.cpp:9), allocates syn0/syn1 in HBM and runs init_model
 * (model.cpp:15) on the device. Replaces the setup half of train()
 * (trainer.cpp:390-410). */
int fw2v_create(const fw2v_config* cfg, const uint64_t* counts, int32_t vocab_size, fw2v_ctx** out);
void fw2v_destroy(fw2v_ctx* ctx);
/* Batch-pipeline buffers (pinned host, device) of destroyed contexts are cached
 * process-wide and reused by the next context (a ringvec::train call creates and
 * destroys one); this returns the cached ones to the driver. */
void fw2v_release_cached(void);

/* Model I/O, dense |V| x dim fp32 row-major host arrays (EmbeddingModel,
 * model.hpp:16-42). Either pointer may be NULL. */
int fw2v_get_model(fw2v_ctx* ctx, float* input, float* output);
int fw2v_set_model(fw2v_ctx* ctx, const float* input, const float* output);
/* Re-runs init_model(vocab, dim, seed) on the device. */
int fw2v_init_model(fw2v_ctx* ctx, uint64_t seed);
/* Device pointers of syn0/syn1 and the padded row stride (floats). */
int fw2v_model_device(fw2v_ctx* ctx, float** syn0, float** syn1, int32_t* stride);
/* Uses caller-owned device buffers (|V| x stride fp32 each, e.g. torch tensors
 * all-reduced by NCCL) as the model from now on; contents are kept as-is. */
int fw2v_attach_model(fw2v_ctx* ctx, float* syn0, float* syn1);
/* Padded row stride (floats) the K1 kernel needs for this dim. */
int32_t fw2v_row_stride(const fw2v_config* cfg);

/* Full training run over a host corpus of pre-subsampling sentences
 * (Corpus, corpus.hpp:107-116): offsets[n_sentences+1] into ids. Mirrors
 * train() (trainer.cpp:390-528): per epoch, producer threads over contiguous
 * chunks assemble batches (subsampling + negatives + per-sentence alpha) into
 * pinned buffers and launch on their own CUDA stream; workers == 1 (or
 * deterministic == 1) runs the serial bit-exact engine. observer/on_epoch
 * may be NULL. */
int fw2v_train_corpus(fw2v_ctx* ctx, const uint64_t* offsets, uint64_t n_sentences,
                      const int32_t* ids, fw2v_observer_fn observer, void* observer_user,
                      fw2v_epoch_fn on_epoch, void* epoch_user, fw2v_report* report);

/* train_sentence (trainer.cpp:332-356) over a batch of already-subsampled
 * sentences with caller-supplied negatives (L*N per sentence, concatenated)
 * and per-sentence alpha, host buffers. serial = 1 runs the exact engine one
 * sentence at a time in order; serial = 0 runs the Hogwild kernel for the
 * context's reuse mode. Synchronous. */
int fw2v_train_sentences(fw2v_ctx* ctx, const uint64_t* offsets, uint64_t n_sentences,
                         const int32_t* ids, const int32_t* negatives, const float* alphas,
                         int32_t serial, fw2v_counters* counters);

/* Device-resident epoch plans (benchmark / repeated-epoch path): the host
 * batcher assembles one epoch's batches for `epoch` straight into HBM; running
 * the plan launches only the training kernels (no host work, no H2D). */
int fw2v_plan_epoch(fw2v_ctx* ctx, const uint64_t* offsets, uint64_t n_sentences, const int32_t* ids,
                    int32_t epoch, fw2v_plan** out);
int fw2v_plan_info(const fw2v_plan* plan, uint64_t* words, uint64_t* sentences, uint64_t* batches,
                   uint64_t* device_bytes);
/* The same for chunks [chunk_begin, chunk_end) of an n_chunks partition of the corpus
 * (trainer.cpp:431-434; chunk p keeps its streams derive(seed, epoch, p, k)): one shard / one
 * averaging round of a data-parallel job. alpha of local word w uses the schedule position
 * words_base + (w - words_base) * words_scale (words_scale = shards per job / shards here). */
int fw2v_plan_chunks(fw2v_ctx* ctx, const uint64_t* offsets, uint64_t n_sentences, const int32_t* ids, int32_t epoch,
                     int32_t n_chunks, int32_t chunk_begin, int32_t chunk_end, uint64_t words_base,
                     int32_t words_scale, fw2v_plan** out);
/* Launches the plan's kernels on the context's streams and waits; seconds =
 * CUDA-event device time from first launch to last completion. */
int fw2v_plan_run(fw2v_ctx* ctx, fw2v_plan* plan, double* seconds, fw2v_counters* counters);
void fw2v_plan_destroy(fw2v_plan* plan);

/* ---- Data-parallel replicas (north_star "replicates syn0/syn1neg per GPU,
 * shards the corpus, and averages the replicas periodically with an NCCL allreduce") ----
 * The reference has one model shared by its worker threads (trainer.cpp:429-503); across GPUs each
 * device holds a replica and the exchange step is the replica average. */

/* In place: every context's syn0 and syn1 <- their element-wise mean over the n contexts (and, for
 * a context joined with fw2v_comm_init_rank, over every process of its communicator).
 * Contexts on distinct devices: one ncclAllReduce(ncclFloat32, ncclAvg) per matrix (libnccl.so.2,
 * opened at run time; communicators cached per context set) over NVLink / NVSwitch. Contexts that
 * share a device, FW2V_AVERAGE=peer, or no NCCL: a peer-memory kernel (member g reads slice g of
 * every replica over P2P and writes the mean back into all of them). Synchronous; training on the
 * contexts must not be in flight. FW2V_ERR_BAD_ARGUMENT if the replicas differ in shape. */
int fw2v_average(fw2v_ctx* const* ctxs, int32_t n);
/* Cross-process communicator (one process per GPU): rank 0 calls fw2v_nccl_unique_id, the caller
 * distributes the 128 bytes (e.g. torch.distributed broadcast), every rank joins its context. */
int fw2v_nccl_unique_id(uint8_t out[128]);
int fw2v_comm_init_rank(fw2v_ctx* ctx, const uint8_t id[128], int32_t world, int32_t rank);

/* Exchange across processes, called by fw2v_train_corpus_multi at every merge point after this
 * process's kernels finished: must SUM each of the n_bufs device buffers (counts[i] fp32 each)
 * over all processes in place (e.g. torch.distributed all_reduce over __cuda_array_interface__
 * views) and set *global_words to the sum of local_words over processes. The library turns the
 * replicas into the summands before (delta / indicator per replica_merge) and the sums into the
 * merged model after. Returns 0 or an fw2v status. */
typedef int (*fw2v_exchange_fn)(void* user, float* const* bufs, const uint64_t* counts, int32_t n_bufs,
                                uint64_t local_words, uint64_t* global_words);

/* The merge step of fw2v_train_corpus_multi on its own (device-resident benchmark rounds):
 * fw2v_merge_begin records the replicas' common starting point, fw2v_merge_replicas merges the
 * replicas per ctxs[0]'s replica_merge rule (n_shards > n: across processes as above) and
 * returns the global word count. */
int fw2v_merge_begin(fw2v_ctx* const* ctxs, int32_t n);
int fw2v_merge_replicas(fw2v_ctx* const* ctxs, int32_t n, int32_t n_shards, const uint64_t* local_words,
                        fw2v_exchange_fn exchange, void* exchange_user, uint64_t* global_words);

/* Data-parallel training: this call trains shards shard0 .. shard0+n-1 (context i <- shard
 * shard0+i) of an n_shards-shard job (n_shards > n: other processes hold the rest and `exchange`
 * or fw2v_comm_init_rank connects them; one context per process then). Replicas are merged per
 * ctxs[0]'s replica_merge rule (NCCL SUM all-reduce between prep / finish kernels, or one fused
 * peer-memory kernel when the contexts share a device). The corpus is cut into the reference's producer chunks
 * (cfg.workers, trainer.cpp:431-434) rounded up to a multiple of n_shards x rounds; shard g is a
 * contiguous range of whole chunks, each chunk trained with its reference streams. The replicas are
 * merged every ~average_words trained words per shard (0: at the end of
 * every epoch only) and after every epoch; lr_at counts the words of every shard (trainer.cpp:
 * 479-487: exact at each average, extrapolated between them). Replicas must start equal (same seed).
 * Deterministic contexts are rejected (FW2V_ERR_UNSUPPORTED). report: this process's totals,
 * kernel_seconds summed over rounds of the max over its GPUs. */
int fw2v_train_corpus_multi(fw2v_ctx* const* ctxs, int32_t n, int32_t shard0, int32_t n_shards,
                            const uint64_t* offsets, uint64_t n_sentences, const int32_t* ids,
                            uint64_t average_words, fw2v_exchange_fn exchange, void* exchange_user,
                            fw2v_observer_fn observer, void* observer_user, fw2v_epoch_fn on_epoch, void* epoch_user,
                            fw2v_report* report);

/* Host batcher primitives (exposed for tests; same contracts as the
 * reference functions cited). */
/* subsample_keep_probs (corpus.cpp:221-230); returns 1 if enabled, 0 if t <= 0 */
int fw2v_keep_probs(const uint64_t* counts, int32_t vocab_size, double threshold, double* out);
/* NegativeTable::build (sampler.cpp:9-35) */
int fw2v_table_build(const uint64_t* counts, int32_t vocab_size, double power, uint64_t size,
                     int32_t* out_slots);
/* assemble_batch (sampler.cpp:41-63) with Rng::derive(seed, a, b, c) (rng.hpp:16). Returns the
 * number of kept sentences (>= 0) or -status. */
int64_t fw2v_assemble_batch(const uint64_t* counts, int32_t vocab_size, const uint64_t* offsets,
                            uint64_t n_sentences, const int32_t* ids, uint64_t* cursor,
                            uint64_t max_sentences, int32_t negatives, double power,
                            uint64_t table_size, double threshold, uint64_t seed, uint64_t a,
                            uint64_t b, uint64_t c, int32_t* out_ids, uint64_t* out_offsets,
                            int32_t* out_negs);
/* `count` draws of the alias sampler (unigram^power; the throughput-mode negative
 * sampler) from the stream Rng::derive(seed, 0): AVX-512 when the host has it,
 * else scalar; both give the same sequence. */
int fw2v_alias_draws(const uint64_t* counts, int32_t vocab_size, double power, uint64_t seed, uint64_t count,
                     int32_t* out);
/* lr_at (model.cpp:39-45) */
float fw2v_lr_at(uint64_t words_trained, uint64_t total, float alpha0);
/* analytic_traffic (traffic.cpp:21-59) */
int fw2v_analytic_traffic(uint64_t length, int32_t width, int32_t negatives, int32_t mode,
                          fw2v_counters* out);

/* Embedding text writer: save_embeddings (model.cpp:47-74)
 * byte for byte — "<|V|> <dim>\n", then per row the token and " <value>" per
 * column with std::to_chars fixed, 6 decimals — formatted on `threads` host
 * threads (<= 0: all cores). rows: |V| x dim host floats, row stride
 * row_stride >= dim; tokens: concatenated token bytes, token_offsets[|V|+1].
 * FW2V_ERR_IO on open/write failure (ringvec ErrorCode::io). */
int fw2v_write_embeddings(const float* rows, int32_t vocab_size, int32_t dim, int64_t row_stride,
                          const char* tokens, const uint64_t* token_offsets, const char* path, int32_t threads);
/* The same straight from a trainer's device model: which = 0 input (syn0), 1 output (syn1). */
int fw2v_save_model(fw2v_ctx* ctx, int32_t which, const char* tokens, const uint64_t* token_offsets,
                    const char* path, int32_t threads);

/* GPU evaluation scans, same arithmetic as the reference
 * (double sums of float products in column order, no FMA) so the answers are
 * identical. rows: |V| x dim host floats (e.g. LoadedEmbeddings::vectors).
 * nearest_neighbors (eval.cpp:303-348) for n_queries ids at once: top-k
 * (k <= 32) by cosine, query excluded, zero rows skipped, ties by id;
 * out_ids/out_cos n_queries x k (-1 / NaN past the candidates). Errors:
 * BAD_ARGUMENT (k not in [1, |V|-1]), OOV_QUERY, ZERO_VECTOR (zero query). */
int fw2v_nearest_neighbors(const float* rows, int32_t vocab_size, int32_t dim, const int32_t* queries,
                           int32_t n_queries, int32_t k, int32_t* out_ids, double* out_cos);
/* eval_analogy's solve (eval.cpp:212-268) per quadruple (a, a*, b, b*) of ids:
 * out_pred = argmax over x not in {a, a*, b} of the method's score on unit rows
 * (0 cos_add, 1 cos_mul), first (lowest) id among equal maxima. */
int fw2v_eval_analogy(const float* rows, int32_t vocab_size, int32_t dim, const int32_t* quads, int32_t n,
                      int32_t method, int32_t* out_pred);

/* Synthetic Zipf corpus of the benchmark shapes (bench
 * input, not the training path): `tokens` i.i.d. ranks r in 1..types with
 * p(r) ∝ r^-s (inverse CDF by binary search; token i uses splitmix64 draw i of
 * Rng::derive(2312, 7743) as next_double), cut into sentences of
 * `sentence_len` raw tokens. Vocabulary = ranks with count >= min_count,
 * count-descending with ties by token name "r<rank>" (Vocabulary::build,
 * corpus.cpp:117-139); ids remapped to vocabulary order; out-of-vocabulary
 * tokens dropped and empty sentences skipped (SentenceReader, corpus.cpp:162-213). */
typedef struct fw2v_corpus fw2v_corpus;
int fw2v_corpus_synth_zipf(uint64_t types, uint64_t tokens, double s, uint64_t sentence_len,
                           uint64_t min_count, int32_t threads, fw2v_corpus** out);
/* Borrowed views valid until fw2v_corpus_free. */
int fw2v_corpus_view(const fw2v_corpus* c, const uint64_t** counts, int32_t* vocab_size,
                     const uint64_t** offsets, uint64_t* n_sentences, const int32_t** ids,
                     uint64_t* n_ids);
void fw2v_corpus_free(fw2v_corpus* c);

#ifdef __cplusplus
}
#endif
#endif
