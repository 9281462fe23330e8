// Device-side data types shared by the FULL-W2V B200 kernels and the host
// runtime. Plain structs only (they cross the host/device launch boundary).
#pragma once

#include <cstdint>
#ifdef __CUDACC__
#include <atomic>
#include <cuda_runtime.h>
#endif

namespace fw2v {

// One batch of post-subsampling sentences resident in HBM.
//   ids      [W]        kept token ids of all sentences, concatenated
//   offsets  [S+1]      sentence boundaries into ids (word units)
//   negs     [W*N]      N negatives per target position (position-major)
//   alpha    [S]        per-sentence learning rate (lr_at before the sentence)
struct BatchView {
    const int32_t* ids;
    const uint32_t* offsets;
    const int32_t* negs;
    const float* alpha;
    int32_t n_sentences;
    int32_t max_groups = 0;  // K1s: at most this many sentences in flight (grid-stride launch); 0 = all
    // Observer log (test mode, trainer.hpp:82-87): every kernel appends
    // (sentence in batch) << 32 | target for each window it starts, in the
    // device's processing order; the host replays it into the observer.
    unsigned long long* obs_log = nullptr;
    unsigned int* obs_count = nullptr;
    int32_t obs_base = 0;  // batch index of sentence 0 of this launch (split launches)
};

// Embedding matrices in HBM: row w of syn0 (reference `input`, context side)
// at syn0 + w*stride, same for syn1 (reference `output`, target/negative
// side). stride >= dim; columns dim..stride-1 are zero and stay zero.
struct ModelView {
    float* syn0;
    float* syn1;
    int32_t dim;
    int32_t stride;
    int32_t vocab;
    int32_t flags;  // K1s memory-path options (kFlag*)
    // Hot-row replicas (K1s Hogwild): output rows 0..hot_k-1 (the most frequent
    // words, ids are count-descending) live in hot_r replicas at
    // hot + (r*hot_k + id)*stride; sentence s trains replica s % hot_r. The host
    // broadcasts syn1 into the replicas before a pass and averages them back after.
    float* hot;
    int32_t hot_k;
    int32_t hot_r;
    int32_t hot_row;  // (hot - syn1) / (stride floats): replica r of row id is syn1 row hot_row + r*hot_k + id
    // Live hot-row merge: the training kernels count sentence starts here, so the
    // merge block can tell a pass that is still training from one whose kernels
    // cannot run beside it (a serialising profiler); null when not merging live.
    unsigned int* beat = nullptr;
};

// K1s memory-path options.
constexpr int32_t kFlagRedSamples = 1;    // sample rows are written as red.global.add of the delta (always set;
                                          // documents the write-back in flag dumps)
constexpr int32_t kFlagL1Exact = 2;       // K1s sample rows are staged through L1 (cp.async.ca); every warp
                                          // drops its SM's L1 each window, so reads see the sentence's own writes
constexpr int32_t kFlagDeltaRing = 4;     // ring rows written back as red.add(final - loaded)
constexpr int32_t kFlagNoRing = 32;       // K1s: ring rows stored straight back (Hogwild overwrite, no
                                          // shared-memory ring copy)
constexpr int32_t kFlagNoStair = 64;      // K1s lifetime order: one window at a time (no window staircase;
                                          // A/B experiments, FW2V_NO_STAIR=1)
constexpr int32_t kFlagInvalShift = 8;    // bits 8..11: otherwise one warp per block drops the SM's L1 every
                                          // 2^k windows (bounded staleness for Zipf-hot rows; 0 = never)

// Replicas of one matrix for the peer-memory average (fw2v_average): the same
// |V| x stride buffer on each of n members (device pointers, P2P-accessible).
constexpr int kMaxPeers = 16;
enum MergeRule : int32_t { kMergeMean = 0, kMergeTouched = 1 };  // fw2v_config.replica_merge
struct PeerSet {
    float* ptr[kMaxPeers];
    int32_t n;
};

// Device-side instrumented access counters, in the reference's units
// (whole-vector accesses, traffic.hpp:19-40).
struct DevCounters {
    unsigned long long context_reads;
    unsigned long long context_writes;
    unsigned long long sample_reads;
    unsigned long long sample_writes;
    unsigned long long ring_hits;
    unsigned long long words;
    unsigned long long sentences;
    unsigned long long pad;
};

enum ReuseMode : int32_t { kLifetime = 0, kWindow = 1, kNone = 2, kWindowSnapshot = 3 };

#ifdef __CUDACC__
// Raises a kernel's dynamic shared-memory limit to `bytes` on the CURRENT
// device. The attribute is per device, so the "already set" record is one bit
// per device ordinal (contexts on several GPUs in one process each get it).
// `mask` is the caller's per-kernel static.
inline cudaError_t ensure_dynamic_smem(const void* kern, int bytes, std::atomic<uint64_t>& mask) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = dev < 64 ? (uint64_t{1} << dev) : 0;
    if (bit != 0 && (mask.load(std::memory_order_acquire) & bit) != 0) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess && bit != 0) mask.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}
#endif

} // namespace fw2v
