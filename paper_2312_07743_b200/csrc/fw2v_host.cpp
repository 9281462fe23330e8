// Host runtime of the B200 FULL-W2V trainer: the C-ABI declared in
// include/fw2v.h.
//
// Structure (SURVEY.md §1 "new framework layer map"):
//   H1 batching threads — one per producer p (reference producers,
//      trainer.cpp:429-462). Each owns a contiguous sentence chunk, assembles
//      batches (subsampling + precomputed negatives, sampler.cpp:41-63) with the
//      reference's RNG stream derive(seed, epoch, p, k) straight into pinned
//      buffers, stamps per-sentence alpha from a global word reservation
//      (lr_at, model.cpp:39), copies H2D and launches on its own CUDA stream.
//      Two pinned/device buffer slots per producer double-buffer the pipeline.
//   H2 this C-ABI — plain pointers, int status, thread-local last error.
//   D0 kernels in fw2v_kernels.cu (K1 Hogwild lifetime, K2 exact serial).
// There is no CPU training path: without a CUDA device every training entry
// point fails with FW2V_ERR_NO_DEVICE.
#include "fw2v.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <sys/mman.h>
#if defined(__x86_64__)
#include <immintrin.h>
#include <map>
#include <unordered_map>
#endif
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fw2v_device.cuh"

namespace fw2v {
// resident != nullptr: no launch; *resident = sentences of that kernel the device holds at once.
cudaError_t launch_k1(int lanes, int vec, const ModelView& m, const BatchView& b, int n_neg, int wf,
                      bool fast, DevCounters* ctr, cudaStream_t st, int* resident = nullptr);
bool k1_shape_supported(int lanes, int vec);
cudaError_t launch_k2(const ModelView& m, const BatchView& b, int n_neg, int wf, int mode, bool serial,
                      DevCounters* ctr, cudaStream_t st);
cudaError_t launch_init_model(const ModelView& m, uint64_t state0, cudaStream_t st);
// Hot-row replicas: average = false broadcasts syn1 rows 0..K-1 into them, true averages them back.
cudaError_t launch_hot_sync(const ModelView& m, bool average, cudaStream_t st);
cudaError_t launch_hot_live(const ModelView& m, int* stop, int* started, cudaStream_t st);
cudaError_t launch_set_flag(int* f, cudaStream_t st);
cudaError_t launch_nonfinite(const float* p, size_t n, int* flag, cudaStream_t st);
// K1s family: window-snapshot order, or (lifetime = true) the reference's lifetime order as a wavefront.
cudaError_t launch_k1s(int lanes, int vec, const ModelView& m, const BatchView& b, int n_neg, int wf, bool fast,
                       bool lifetime, DevCounters* ctr, cudaStream_t st, int* resident = nullptr);
bool k1s_supported(int lanes, int vec, int n_neg, int wf, bool lifetime);
int write_embeddings(const float* rows, int32_t vocab_size, int32_t dim, int64_t row_stride, const char* tokens,
                     const uint64_t* token_offsets, const char* path, int32_t threads, std::string* err);
void set_last_error(const std::string& msg);
cudaError_t launch_average_slice(const PeerSet& ps, size_t begin, size_t end, cudaStream_t st);
// fw2v_nccl.cpp
struct NcclClique;
bool nccl_available(std::string* why);
bool nccl_unique_id(uint8_t out[128], std::string* err);
std::shared_ptr<NcclClique> nccl_clique_local(const std::vector<int>& devices, std::string* err);
std::shared_ptr<NcclClique> nccl_clique_rank(int device, const uint8_t id[128], int world, int rank, std::string* err);
bool nccl_allreduce(NcclClique& c, const std::vector<std::vector<float*>>& buffers, size_t count,
                    const std::vector<unsigned long long*>& u64, bool sum, std::string* err);
cudaError_t launch_merge_slice(const PeerSet& ps, float* base, int rule, size_t begin, size_t end, cudaStream_t st);
cudaError_t launch_merge_prep(float* v, const float* base, float* cnt, int rule, size_t n, cudaStream_t st);
cudaError_t launch_merge_finish(float* v, float* base, const float* cnt, int rule, float inv_n, size_t n,
                                cudaStream_t st);
} // namespace fw2v

namespace {

using namespace fw2v;

thread_local std::string g_error;

struct Failure {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Failure{code, msg}; }

#define FW2V_CK(expr)                                                                      \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            fail(FW2V_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));       \
    } while (0)

template <class F>
int guarded(F&& f) {
    try {
        f();
        return FW2V_OK;
    } catch (const Failure& e) {
        g_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_error = "host allocation failed";
        return FW2V_ERR_BAD_ARGUMENT;
    } catch (const std::exception& e) {
        g_error = e.what();
        return FW2V_ERR_BAD_ARGUMENT;
    }
}

// ------------------------------------------------------------------ RNG
// splitmix64 streams, identical to ringvec::Rng (rng.hpp:11-45).
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

struct Rng {
    uint64_t state;
    static Rng derive(uint64_t seed, uint64_t a, uint64_t b = 0, uint64_t c = 0) {
        Rng r{mix64(seed)};
        r.state = mix64(r.state ^ mix64(a + kGolden));
        r.state = mix64(r.state ^ mix64(b + 0xbf58476d1ce4e5b9ULL));
        r.state = mix64(r.state ^ mix64(c + 0x94d049bb133111ebULL));
        return r;
    }
    inline uint64_t next() {
        state += kGolden;
        return mix64(state);
    }
    inline double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

double thread_cpu_seconds() {
    timespec ts{};
    clock_gettime(CLOCK_THREAD_CPUTIME_ID, &ts);
    return static_cast<double>(ts.tv_sec) + 1e-9 * static_cast<double>(ts.tv_nsec);
}

double wall_seconds() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ------------------------------------------------------------ samplers
// subsample_keep_probs (corpus.cpp:215-230)
bool keep_probs(const uint64_t* counts, int32_t v, double t, double* out) {
    if (t <= 0.0) return false;
    uint64_t tot = 0;
    for (int32_t w = 0; w < v; ++w) tot += counts[w];
    const double total = static_cast<double>(tot);
    for (int32_t w = 0; w < v; ++w) {
        const double f = static_cast<double>(counts[w]) / total;
        double p = 1.0;
        if (f > 0.0) {
            p = (std::sqrt(f / t) + 1.0) * (t / f);
            if (p > 1.0) p = 1.0;
        }
        out[w] = p;
    }
    return true;
}

// NegativeTable::build (sampler.cpp:9-35): slot s -> first w whose cumulative
// count^power bracket contains the slot midpoint.
void build_table(const uint64_t* counts, int32_t v, double power, uint64_t size, int32_t* slots) {
    if (size < static_cast<uint64_t>(v)) fail(FW2V_ERR_BAD_ARGUMENT, "table_size must be >= |V|");
    if (power < 0.0) fail(FW2V_ERR_BAD_ARGUMENT, "power must be >= 0");
    std::vector<double> cum(static_cast<size_t>(v));
    double total = 0.0;
    for (int32_t w = 0; w < v; ++w) {
        total += std::pow(static_cast<double>(counts[w]), power);
        cum[static_cast<size_t>(w)] = total;
    }
    size_t w = 0;
    for (uint64_t s = 0; s < size; ++s) {
        const double mid = (static_cast<double>(s) + 0.5) / static_cast<double>(size) * total;
        while (w + 1 < static_cast<size_t>(v) && mid >= cum[w]) ++w;
        slots[s] = static_cast<int32_t>(w);
    }
}

// Walker alias table over count^power (throughput sampler, north_star
// "unigram^0.75 alias table"): one 64-bit draw -> column (Lemire
// multiply-high) + 32-bit coin.
struct AliasTable {
    struct Entry {
        uint32_t prob;  // threshold in 2^32 units
        int32_t alias;
    };
    std::vector<Entry> e;  // one 8-byte entry per column: one cache access per draw
    uint32_t n = 0;
    void build(const uint64_t* counts, int32_t v, double power) {
        n = static_cast<uint32_t>(v);
        std::vector<double> p(static_cast<size_t>(v));
        double total = 0.0;
        for (int32_t w = 0; w < v; ++w) total += (p[static_cast<size_t>(w)] = std::pow(static_cast<double>(counts[w]), power));
        std::vector<int32_t> small, large;
        for (int32_t w = 0; w < v; ++w) {
            p[static_cast<size_t>(w)] *= static_cast<double>(v) / total;
            (p[static_cast<size_t>(w)] < 1.0 ? small : large).push_back(w);
        }
        e.resize(static_cast<size_t>(v));
        for (int32_t w = 0; w < v; ++w) e[static_cast<size_t>(w)] = Entry{0xffffffffu, w};
        while (!small.empty() && !large.empty()) {
            const int32_t s = small.back(), l = large.back();
            small.pop_back();
            const double ps = p[static_cast<size_t>(s)];
            e[static_cast<size_t>(s)] = Entry{static_cast<uint32_t>(std::min(4294967295.0, ps * 4294967296.0)), l};
            p[static_cast<size_t>(l)] -= 1.0 - ps;
            if (p[static_cast<size_t>(l)] < 1.0) {
                large.pop_back();
                small.push_back(l);
            }
        }
    }
    inline int32_t sample(uint64_t u) const {
        const uint32_t col = static_cast<uint32_t>((static_cast<uint64_t>(static_cast<uint32_t>(u)) * n) >> 32);
        const Entry& x = e.data()[col];
        return static_cast<uint32_t>(u >> 32) < x.prob ? static_cast<int32_t>(col) : x.alias;
    }
};

// lr_at (model.cpp:39-45)
inline float lr_at(uint64_t trained, uint64_t total, float alpha0) {
    const double progress = static_cast<double>(trained) / static_cast<double>(total);
    const double a = static_cast<double>(alpha0) * (1.0 - progress);
    const double floor_ = static_cast<double>(alpha0) * 1e-4;
    return static_cast<float>(std::max(a, floor_));
}

// analytic_traffic (traffic.cpp:21-59)
void analytic(uint64_t len, int width, int neg, int mode, uint64_t* t) {
    uint64_t pairs = 0;
    if (len >= 2) {
        const uint64_t g = std::min<uint64_t>(static_cast<uint64_t>(width), len - 1);
        pairs = 2 * g * len - g * (g + 1);
    }
    const uint64_t samples = static_cast<uint64_t>(neg) + 1;
    const uint64_t windows = len >= 2 ? len : 0;
    switch (mode) {
    case kLifetime:
    case kWindowSnapshot:
        t[0] = len; t[1] = len; t[2] = windows * samples; t[3] = windows * samples;
        t[4] = windows > 0 ? samples * pairs - len : 0;
        break;
    case kWindow:
        t[0] = pairs; t[1] = pairs; t[2] = windows * samples; t[3] = windows * samples;
        t[4] = static_cast<uint64_t>(neg) * pairs;
        break;
    default:
        t[0] = samples * pairs; t[1] = samples * pairs; t[2] = samples * pairs;
        t[3] = samples * pairs; t[4] = 0;
        break;
    }
}

// ----------------------------------------------------------- batch assembly
struct CorpusView {
    const uint64_t* offsets;
    const int32_t* ids;
    uint64_t n;
};

// Host array on 2 MB pages (transparent huge pages via madvise): the 40 MB
// negative table is read at random, and with 4 KB pages nearly every draw
// would also miss the TLB.
template <typename T>
class HugeArray {
  public:
    HugeArray() = default;
    HugeArray(const HugeArray&) = delete;
    HugeArray& operator=(const HugeArray&) = delete;
    ~HugeArray() { release(); }
    void resize(size_t n) {
        release();
        n_ = n;
        bytes_ = ((n * sizeof(T) + kPage - 1) / kPage) * kPage;
        if (bytes_ == 0) return;
        void* p = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (p == MAP_FAILED) throw std::bad_alloc();
        madvise(p, bytes_, MADV_HUGEPAGE);
        p_ = static_cast<T*>(p);
    }
    T* data() { return p_; }
    const T* data() const { return p_; }
    size_t size() const { return n_; }

  private:
    static constexpr size_t kPage = size_t{2} << 20;
    void release() {
        if (p_ != nullptr) munmap(p_, bytes_);
        p_ = nullptr;
        n_ = bytes_ = 0;
    }
    T* p_ = nullptr;
    size_t n_ = 0, bytes_ = 0;
};

// x % d for a fixed d >= 1 without a 64-bit divide: q = floor(x * floor(2^64/d) / 2^64)
// is q_true or q_true - 1, so one conditional subtract makes it exact.
struct FastMod {
    uint64_t d = 1, inv = 0;
    explicit FastMod(uint64_t d_ = 1) : d(d_), inv(d_ > 1 ? ~uint64_t{0} / d_ : 0) {}
    inline uint64_t operator()(uint64_t x) const {
        if (d == 1) return 0;
        const uint64_t q = static_cast<uint64_t>((static_cast<unsigned __int128>(x) * inv) >> 64);
        uint64_t r = x - q * d;
        return r >= d ? r - d : r;
    }
};

struct Sampler {
    const double* keep = nullptr;     // null: subsampling off
    const int32_t* slots = nullptr;   // reference table
    uint64_t table_size = 0;
    FastMod mod{1};
    const AliasTable* alias = nullptr;  // non-null: alias sampler
    int n_neg = 0;
};

struct BatchOut {
    int32_t* ids;
    uint32_t* offsets;  // relative, kept+1 entries
    int32_t* negs;
    uint64_t cap_words;
    uint64_t cap_sentences;
};

// assemble_batch (sampler.cpp:41-63) + subsample_sentence (corpus.cpp:232-241):
// same RNG consumption order, so the batch equals the reference's for the
// same stream. Returns kept sentences; *words = their total length.
// ---- AVX-512 batching kernels. Draw k (1-based) of a stream in state s is
// mix64(s + k*golden) (Rng::next), so 8 consecutive draws are independent and
// vectorise; results and the final stream state equal the scalar loops'.
#if defined(__x86_64__)
#define FW2V_AVX512 __attribute__((target("avx512f,avx512dq,avx512vl")))
FW2V_AVX512 inline __m512i mix64x8(__m512i z) {
    z = _mm512_mullo_epi64(_mm512_xor_si512(z, _mm512_srli_epi64(z, 30)), _mm512_set1_epi64(0xbf58476d1ce4e5b9LL));
    z = _mm512_mullo_epi64(_mm512_xor_si512(z, _mm512_srli_epi64(z, 27)), _mm512_set1_epi64(0x94d049bb133111ebLL));
    return _mm512_xor_si512(z, _mm512_srli_epi64(z, 31));
}
// Stream positions s + (k+1)*golden for k = 0..7, and the step to the next 8.
FW2V_AVX512 inline __m512i stream8(uint64_t s) {
    const __m512i k = _mm512_set_epi64(8, 7, 6, 5, 4, 3, 2, 1);
    return _mm512_add_epi64(_mm512_set1_epi64(static_cast<long long>(s)),
                            _mm512_mullo_epi64(k, _mm512_set1_epi64(static_cast<long long>(kGolden))));
}
// cnt alias draws (AliasTable::sample) into out; returns the advanced state.
FW2V_AVX512 uint64_t alias_draws_avx512(uint64_t s, const AliasTable::Entry* E, uint32_t n, int32_t* out,
                                        uint64_t cnt) {
    const __m512i step = _mm512_set1_epi64(static_cast<long long>(8 * kGolden));
    const __m512i nv = _mm512_set1_epi64(n);
    const __m512i lo32 = _mm512_set1_epi64(0xffffffffLL);
    __m512i pos = stream8(s);
    uint64_t x = 0;
    for (; x + 8 <= cnt; x += 8) {
        const __m512i u = mix64x8(pos);
        pos = _mm512_add_epi64(pos, step);
        const __m512i col = _mm512_srli_epi64(_mm512_mul_epu32(u, nv), 32);  // (u32 * n) >> 32
        const __m512i en = _mm512_i64gather_epi64(col, reinterpret_cast<const long long*>(E), 8);
        const __mmask8 acc = _mm512_cmplt_epu64_mask(_mm512_srli_epi64(u, 32), _mm512_and_si512(en, lo32));
        const __m512i v = _mm512_mask_blend_epi64(acc, _mm512_srli_epi64(en, 32), col);
        _mm256_storeu_si256(reinterpret_cast<__m256i*>(out + x), _mm512_cvtepi64_epi32(v));
    }
    s += x * kGolden;
    for (; x < cnt; ++x) {
        s += kGolden;
        const uint64_t u = mix64(s);
        const uint32_t col = static_cast<uint32_t>((static_cast<uint64_t>(static_cast<uint32_t>(u)) * n) >> 32);
        out[x] = static_cast<uint32_t>(u >> 32) < E[col].prob ? static_cast<int32_t>(col) : E[col].alias;
    }
    return s;
}
// Subsampling of ids[0..len) (corpus.cpp:232-241): keeps id when next_double() <
// keep[id], in order; writes the kept ids to dst, returns their count.
FW2V_AVX512 uint64_t subsample_avx512(uint64_t* state, const int32_t* ids, uint64_t len, const double* keep,
                                      int32_t* dst) {
    uint64_t s = *state;
    const __m512i step = _mm512_set1_epi64(static_cast<long long>(8 * kGolden));
    const __m512d scale = _mm512_set1_pd(0x1.0p-53);
    __m512i pos = stream8(s);
    uint64_t p = 0, n = 0;
    for (; p + 8 <= len; p += 8) {
        const __m512i u = mix64x8(pos);
        pos = _mm512_add_epi64(pos, step);
        const __m512d d = _mm512_mul_pd(_mm512_cvtepu64_pd(_mm512_srli_epi64(u, 11)), scale);
        const __m256i id = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(ids + p));
        const __m512d k = _mm512_i32gather_pd(id, keep, 8);
        const __mmask8 m = _mm512_cmp_pd_mask(d, k, _CMP_LT_OQ);
        _mm256_mask_compressstoreu_epi32(dst + n, m, id);
        n += static_cast<uint64_t>(__builtin_popcount(m));
    }
    s += p * kGolden;
    for (; p < len; ++p) {
        s += kGolden;
        const int32_t id = ids[p];
        dst[n] = id;
        n += static_cast<double>(mix64(s) >> 11) * 0x1.0p-53 < keep[id] ? 1 : 0;
    }
    *state = s;
    return n;
}
bool have_avx512() {
    static const bool on = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512dq") &&
                           __builtin_cpu_supports("avx512vl") && std::getenv("FW2V_NO_AVX512") == nullptr;
    return on;
}
#else
bool have_avx512() { return false; }
#endif

uint64_t assemble(const CorpusView& c, uint64_t& cursor, uint64_t end, uint64_t max_sentences,
                  const Sampler& sp, Rng& rng, const BatchOut& out, uint64_t* words) {
    uint64_t kept = 0, w = 0;
    out.offsets[0] = 0;
    const int n_neg = sp.n_neg;
    const bool vec = have_avx512();
    while (kept < max_sentences && cursor < end) {
        const uint64_t b = c.offsets[cursor], e = c.offsets[cursor + 1];
        if (w + (e - b) > out.cap_words) break;  // caller sized for the worst case; never hit
        const uint64_t start = w;
        if (sp.keep != nullptr && vec) {
            w += subsample_avx512(&rng.state, c.ids + b, e - b, sp.keep, out.ids + w);
        } else if (sp.keep != nullptr) {
            // One next_double per raw token, kept in order (corpus.cpp:232-241);
            // branch-free: keep decisions are coin flips for frequent words.
            int32_t* dst = out.ids + w;
            uint64_t n = 0;
            for (uint64_t p = b; p < e; ++p) {
                const int32_t id = c.ids[p];
                dst[n] = id;
                n += rng.next_double() < sp.keep[id] ? 1 : 0;
            }
            w += n;
        } else {
            std::memcpy(out.ids + w, c.ids + b, sizeof(int32_t) * (e - b));
            w += e - b;
        }
        ++cursor;
        if (w == start) continue;
        int32_t* ng = out.negs + start * static_cast<uint64_t>(n_neg);
        const uint64_t cnt = (w - start) * static_cast<uint64_t>(n_neg);
        // The stream state and tables live in locals: through the references the
        // compiler must assume the int32 stores into ng may alias them.
        Rng r = rng;
        if (sp.alias != nullptr && vec) {
            r.state = alias_draws_avx512(r.state, sp.alias->e.data(), sp.alias->n, ng, cnt);
        } else if (sp.alias != nullptr) {
            const AliasTable::Entry* const E = sp.alias->e.data();
            const uint64_t n = sp.alias->n;
            for (uint64_t x = 0; x < cnt; ++x) {
                const uint64_t u = r.next();
                const uint32_t col = static_cast<uint32_t>((static_cast<uint64_t>(static_cast<uint32_t>(u)) * n) >> 32);
                const AliasTable::Entry en = E[col];
                // branch-free select (acceptance is a coin flip for most columns)
                const int32_t m = -static_cast<int32_t>(static_cast<uint32_t>(u >> 32) < en.prob);
                ng[x] = (static_cast<int32_t>(col) & m) | (en.alias & ~m);
            }
        } else {
            // Same draws in the same order as slots[rng.next() % size] (sampler.cpp:37-39);
            // the table (40 MB at 1e7 slots) is gathered 64 draws at a time with
            // prefetches so the cache misses overlap.
            constexpr uint64_t kG = 64;
            uint64_t idx[kG];
            const FastMod mod = sp.mod;
            const int32_t* const slots = sp.slots;
            for (uint64_t x0 = 0; x0 < cnt; x0 += kG) {
                const uint64_t g = std::min(kG, cnt - x0);
                for (uint64_t j = 0; j < g; ++j) {
                    idx[j] = mod(r.next());
                    __builtin_prefetch(slots + idx[j], 0, 3);
                }
                for (uint64_t j = 0; j < g; ++j) ng[x0 + j] = slots[idx[j]];
            }
        }
        rng = r;
        ++kept;
        out.offsets[kept] = static_cast<uint32_t>(w);
    }
    *words = w;
    return kept;
}

// Negative arrays on the device carry this much zeroed padding: the K1s kernel
// reads the negatives of a position as one fixed-size group (immediate offsets,
// no clamping), which may run past the last position's N values.
constexpr size_t kNegPadBytes = 64;

// ------------------------------------------------------------ K1 shapes
struct Shape {
    int lanes = 0, vec = 0;
};

Shape choose_shape(int dim, int lanes_pref) {
    static const Shape table[] = {{4, 1},  {4, 2},  {4, 4},   {8, 4},   {16, 4},  {32, 4},
                                  {32, 6}, {32, 8}, {32, 10}, {32, 12}, {32, 16}};
    if (lanes_pref > 0) {
        static const int vecs[] = {1, 2, 4, 6, 8, 10, 12, 16};
        for (int v : vecs)
            if (lanes_pref * v >= dim && k1_shape_supported(lanes_pref, v)) return {lanes_pref, v};
        return {};
    }
    for (const Shape& s : table)
        if (s.lanes * s.vec >= dim) return s;
    return {};
}

// K1s lane shape for a row stride: the fewest lanes per sentence (more
// sentences per warp amortise the per-window butterfly, sigmoid and
// bookkeeping) with at most 8 columns per lane when the stride allows it
// (registers), up to 16 on 32 lanes for wide rows (d = 300 -> 32 x 10); d = 512 runs on two
// warps per sentence (64 x 8).
Shape choose_k1s_shape(int stride, const Shape& k1, int lanes_pref, int n_neg, int wf, bool lifetime) {
    // Lifetime order with N = 15: the staircase streams the 16 samples on 32-lane
    // groups (the repeat check needs 2 x 16 lanes), at 4 columns per lane.
    if (lanes_pref == 0 && lifetime && n_neg == 15 && wf <= 3 && stride == 128) return Shape{32, 4};
    if (lanes_pref == 0) {
        static const Shape pref[] = {{4, 4}, {8, 4}, {16, 4}, {16, 8}, {32, 4}, {32, 6}, {32, 8}, {32, 10}, {32, 12},
                                     {64, 8}, {32, 16}};
        for (const Shape& s : pref)
            if (s.lanes * s.vec == stride && k1s_supported(s.lanes, s.vec, n_neg, wf, lifetime)) return s;
    }
    return k1s_supported(k1.lanes, k1.vec, n_neg, wf, lifetime) ? k1 : Shape{};
}

int row_stride_for(int dim, int lanes_pref) {
    Shape s = choose_shape(dim, lanes_pref);
    if (s.lanes > 0) return s.lanes * s.vec;
    return (dim + 3) & ~3;
}

int context_width(const fw2v_config& c) { return (c.window + 1) / 2; }  // config.hpp:32

void validate(const fw2v_config& c) {  // validate_config (config.cpp:165-177)
    if (c.dim < 1) fail(FW2V_ERR_BAD_CONFIG, "dim must be >= 1");
    if (c.window < 1) fail(FW2V_ERR_BAD_CONFIG, "window must be >= 1");
    if (c.negatives < 0) fail(FW2V_ERR_BAD_CONFIG, "negatives must be >= 0");
    if (c.epochs < 0) fail(FW2V_ERR_BAD_CONFIG, "epochs must be >= 0");
    if (!(c.alpha0 > 0.0f)) fail(FW2V_ERR_BAD_CONFIG, "alpha must be > 0");
    if (c.min_count < 1) fail(FW2V_ERR_BAD_CONFIG, "min_count must be >= 1");
    if (c.batch_sentences < 1) fail(FW2V_ERR_BAD_CONFIG, "batch_sentences must be >= 1");
    if (c.max_sentence_len < 1) fail(FW2V_ERR_BAD_CONFIG, "max_sentence_len must be >= 1");
    if (c.workers < 0) fail(FW2V_ERR_BAD_CONFIG, "workers must be >= 0");
    if (c.table_size < 1) fail(FW2V_ERR_BAD_CONFIG, "table_size must be >= 1");
    if (!(c.table_power >= 0.0)) fail(FW2V_ERR_BAD_CONFIG, "table_power must be >= 0");
    if (c.reuse_mode < 0 || c.reuse_mode > 3) fail(FW2V_ERR_BAD_CONFIG, "unknown reuse mode");
    if (c.sampler < 0 || c.sampler > 1) fail(FW2V_ERR_BAD_CONFIG, "unknown sampler");
    if (c.hot_rows < 0 || c.hot_replicas < 1) fail(FW2V_ERR_BAD_CONFIG, "hot_rows must be >= 0 and hot_replicas >= 1");
    if (c.delta_writeback < 0 || c.delta_writeback > 2) fail(FW2V_ERR_BAD_CONFIG, "delta_writeback must be 0, 1 or 2");
    if (c.replica_merge < 0 || c.replica_merge > 1) fail(FW2V_ERR_BAD_CONFIG, "replica_merge must be 0 or 1");
    if (c.hot_merge < 0 || c.hot_merge > 1) fail(FW2V_ERR_BAD_CONFIG, "hot_merge must be 0 or 1");
    if (c.hot_merge == 1 && c.hot_rows > 0 && c.hot_replicas > 16)
        fail(FW2V_ERR_BAD_CONFIG, "the live hot-row merge takes at most 16 replicas");
}

void require_device(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        fail(FW2V_ERR_NO_DEVICE, std::string("no CUDA device (the B200 trainer has no CPU path): ") +
                                     (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
    if (device < 0 || device >= n) fail(FW2V_ERR_BAD_ARGUMENT, "device ordinal out of range");
    FW2V_CK(cudaSetDevice(device));
}

// Process-wide cache of the batch pipeline's pinned host and device buffers.
// A ringvec::train user creates, trains and destroys a context per call; without
// the cache every call pays ~0.3 s of cudaHostAlloc for its slots. Freed blocks
// are kept (up to kPoolCap bytes per kind and device) and handed out again to a
// request of at most their size and at least half of it. fw2v_release_cached()
// returns them to the driver.
class BufferPool {
public:
    static BufferPool& get() {
        static BufferPool* p = new BufferPool();  // never destroyed: no teardown-order issues
        return *p;
    }
    void* host(size_t bytes) { return take(kHost, bytes); }
    void* device(size_t bytes) {
        int dev = 0;
        FW2V_CK(cudaGetDevice(&dev));
        return take(dev, bytes);
    }
    void put(void* p) {
        if (p == nullptr) return;
        std::lock_guard<std::mutex> lk(mu_);
        auto it = live_.find(p);
        if (it == live_.end()) return;
        const auto [key, bytes] = it->second;
        live_.erase(it);
        if (cached_[key] + bytes > kPoolCap) {
            release_block(key, p);
            return;
        }
        cached_[key] += bytes;
        free_[key].emplace(bytes, p);
    }
    void release_all() {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto& [key, m] : free_)
            for (auto& [bytes, p] : m) release_block(key, p);
        free_.clear();
        cached_.clear();
    }

private:
    static constexpr int kHost = -1;
    static constexpr size_t kPoolCap = size_t{16} << 30;
    void* take(int key, size_t bytes) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto& m = free_[key];
            auto it = m.lower_bound(bytes);
            if (it != m.end() && it->first <= 2 * bytes) {
                void* p = it->second;
                live_[p] = {key, it->first};
                cached_[key] -= it->first;
                m.erase(it);
                return p;
            }
        }
        void* p = nullptr;
        if (key == kHost) FW2V_CK(cudaHostAlloc(&p, bytes, cudaHostAllocDefault));
        else FW2V_CK(cudaMalloc(&p, bytes));
        std::lock_guard<std::mutex> lk(mu_);
        live_[p] = {key, bytes};
        return p;
    }
    static void release_block(int key, void* p) {
        if (key == kHost) {
            cudaFreeHost(p);
        } else {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(key);
            cudaFree(p);
            cudaSetDevice(cur);
        }
    }
    std::mutex mu_;
    std::map<int, std::multimap<size_t, void*>> free_;
    std::map<int, size_t> cached_;
    std::unordered_map<void*, std::pair<int, size_t>> live_;
};

// One producer lane: stream + two double-buffered batch slots.
struct Slot {
    int32_t* h_ids = nullptr;
    uint32_t* h_off = nullptr;
    int32_t* h_negs = nullptr;
    float* h_alpha = nullptr;
    int32_t* d_ids = nullptr;
    uint32_t* d_off = nullptr;
    int32_t* d_negs = nullptr;
    float* d_alpha = nullptr;
    unsigned long long* d_obs = nullptr;  // observer log (test mode), cap_words entries + count
    unsigned* d_obs_n = nullptr;
    uint64_t obs_cap = 0;
    cudaEvent_t h2d_done = nullptr;  // host buffers free again (copy stream)
    cudaEvent_t used = nullptr;      // device buffers free again (kernel done, compute stream)
    bool in_flight = false;
};

struct Lane {
    // A sub-batch assembled and shipped (H2D issued) at the end of one pass for
    // the next (run_pass cross-epoch prefetch): its slot, size and the span
    // iteration state to resume from, and its share of the pass statistics.
    struct Stash {
        bool ready = false;
        uint64_t pass = 0;
        int slot = 0;
        uint64_t kept = 0, words = 0, p = 0, cursor = 0, end = 0, k = 0, left = 0, h2d = 0;
        Rng rng{};
        double cpu = 0.0;
        uint64_t an[5] = {};
    } stash;
    cudaStream_t stream = nullptr;  // kernels of slot 0
    cudaStream_t stream2 = nullptr; // kernels of slot 1 (Hogwild: a lane's sub-batches overlap)
    cudaStream_t copy = nullptr;    // H2D of the next sub-batch, overlapping the current kernel
    DevCounters* d_ctr = nullptr;
    Slot slot[2];
    uint64_t cap_words = 0, cap_sent = 0;
    void release() {
        for (Slot& s : slot) {
            if (s.h2d_done) cudaEventSynchronize(s.h2d_done);
            BufferPool& pool = BufferPool::get();
            for (void* p : {static_cast<void*>(s.h_ids), static_cast<void*>(s.h_off), static_cast<void*>(s.h_negs),
                            static_cast<void*>(s.h_alpha), static_cast<void*>(s.d_ids), static_cast<void*>(s.d_off),
                            static_cast<void*>(s.d_negs), static_cast<void*>(s.d_alpha), static_cast<void*>(s.d_obs),
                            static_cast<void*>(s.d_obs_n)})
                pool.put(p);
            if (s.h2d_done) cudaEventDestroy(s.h2d_done);
            if (s.used) cudaEventDestroy(s.used);
            s = Slot{};
        }
        cap_words = cap_sent = 0;
        stash.ready = false;
    }
};

} // namespace

struct fw2v_ctx {
    fw2v_config cfg{};
    int wf = 0;
    int32_t vocab = 0;
    Shape shape;      // K1 (lifetime) lanes x columns
    Shape k1s_shape;  // K1s (window snapshot) lanes x columns, same row stride
    int stride = 0;
    bool deterministic = false;
    std::vector<uint64_t> counts;
    uint64_t total_retained = 0;
    std::vector<double> keep;
    bool keep_on = false;
    HugeArray<int32_t> slots;  // reference negative table (sampler.cpp:9-35)
    AliasTable alias;
    float* syn0 = nullptr;
    float* syn1 = nullptr;
    bool own_model = true;
    std::vector<Lane> lanes;
    uint64_t words_trained = 0;  // schedule counter across calls (EmbeddingModel::words_trained)
    // Data-parallel replicas (fw2v_average): the NCCL clique this context is a
    // member of (in-process: every member context; cross-process: this one),
    // and an 8-byte device word for the global word-count all-reduce.
    std::shared_ptr<NcclClique> clique;
    std::vector<fw2v_ctx*> clique_members;
    unsigned long long* d_words = nullptr;
    // Replica merge state (fw2v_train_corpus_multi): the round's base model and,
    // for the touched rule, the changed-element indicators; [syn0 | syn1] each.
    float* merge_base = nullptr;
    float* merge_cnt = nullptr;
    // Divergence guard (fw2v_config.divergence_guard): the model at the start
    // of the current epoch, [syn0 | syn1], and a device flag word.
    float* guard_snap = nullptr;
    int* guard_flag = nullptr;
    uint64_t pass_seq = 0;  // run_pass calls so far
    size_t model_floats() const { return static_cast<size_t>(vocab) * static_cast<size_t>(stride); }

    int32_t k1_flags = 0;
    int64_t inflight_total = 0;  // Hogwild sentences in flight over all streams (0 = unlimited)
    float* hot = nullptr;        // hot-row replicas, hot_r x hot_k x stride (K1s Hogwild only)
    float* hot_alloc = nullptr;  // allocation holding `hot` (one spare row for alignment)
    int32_t hot_k = 0, hot_r = 1;
    int64_t hot_row = 0;         // (hot - syn1) in rows: the kernel addresses replicas from syn1
    // Places the replicas a whole number of rows from syn1 (the kernel forms a
    // 32-bit row index and one pointer); disables them if that is impossible.
    void place_hot() {
        if (hot_alloc == nullptr) return;
        const int64_t row = static_cast<int64_t>(sizeof(float)) * stride;
        const int64_t diff = reinterpret_cast<int64_t>(hot_alloc) - reinterpret_cast<int64_t>(syn1);
        int64_t rows_off = diff / row;
        while (rows_off * row < diff) ++rows_off;  // first whole-row position inside the allocation
        hot = reinterpret_cast<float*>(reinterpret_cast<char*>(syn1) + rows_off * row);
        hot_row = rows_off;
        const int64_t last = rows_off + static_cast<int64_t>(hot_k) * hot_r;
        if (rows_off < INT32_MIN / 2 || last > INT32_MAX / 2) {  // outside a 32-bit row range: plain Hogwild
            hot_k = 0;
            hot = nullptr;
            hot_row = 0;
        }
    }
    ModelView model_view() const {
        ModelView v{syn0, syn1, cfg.dim, stride, vocab, k1_flags, hot, hot_k, hot_r, static_cast<int32_t>(hot_row)};
        v.beat = live() ? live_beat : nullptr;
        return v;
    }
    // Around every Hogwild pass: replicas <- syn1 before, syn1 <- mean(replicas) after.
    void hot_sync(bool average, cudaStream_t st) const { FW2V_CK(launch_hot_sync(model_view(), average, st)); }
    // Live merge (cfg.hot_merge = 1): a resident merge block runs beside the pass's
    // training kernels (k_hot_live) on its own stream.
    cudaStream_t live_stream = nullptr;
    cudaEvent_t live_go = nullptr, live_done = nullptr;
    int* live_stop = nullptr;        // device flag
    unsigned* live_beat = nullptr;   // sentence starts of the training kernels (ModelView::beat)
    int* live_started_h = nullptr;   // mapped host flag, set by the merge block
    int* live_started_d = nullptr;
    bool live() const { return cfg.hot_merge == 1 && hot_k > 0 && !deterministic; }
    // Before a pass (on stream st, before any training kernel is queued): replicas <-
    // syn1; with the live merge, start the merge block and wait until it is resident
    // (so it cannot be starved behind the pass's kernels).
    void hot_begin(cudaStream_t st) {
        hot_sync(false, st);
        if (!live()) return;
        if (live_stream == nullptr) {
            FW2V_CK(cudaStreamCreateWithFlags(&live_stream, cudaStreamNonBlocking));
            FW2V_CK(cudaEventCreateWithFlags(&live_go, cudaEventDisableTiming));
            FW2V_CK(cudaEventCreateWithFlags(&live_done, cudaEventDisableTiming));
            FW2V_CK(cudaMalloc(&live_stop, sizeof(int)));
            FW2V_CK(cudaMalloc(&live_beat, sizeof(unsigned)));
            FW2V_CK(cudaMemset(live_beat, 0, sizeof(unsigned)));
            FW2V_CK(cudaHostAlloc(reinterpret_cast<void**>(&live_started_h), sizeof(int), cudaHostAllocMapped));
            FW2V_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&live_started_d), live_started_h, 0));
            // Every kernel the pass launches while the merge block runs is loaded now:
            // with lazy module loading a first launch can wait for the running
            // kernels, i.e. for the merge block that waits for it (the stop-flag
            // kernel, the training kernel).
            FW2V_CK(launch_set_flag(live_stop, st));
            int resident = 0;
            FW2V_CK(launch_one(BatchView{}, false, nullptr, nullptr, &resident));
            FW2V_CK(cudaStreamSynchronize(st));
        }
        *reinterpret_cast<volatile int*>(live_started_h) = 0;
        FW2V_CK(cudaMemsetAsync(live_stop, 0, sizeof(int), st));
        FW2V_CK(cudaEventRecord(live_go, st));
        FW2V_CK(cudaStreamWaitEvent(live_stream, live_go, 0));
        FW2V_CK(launch_hot_live(model_view(), live_stop, live_started_d, live_stream));
        FW2V_CK(cudaEventRecord(live_done, live_stream));
        const double t0 = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
        while (*reinterpret_cast<volatile int*>(live_started_h) == 0) {
            const double t = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
            if (t - t0 > 5.0) fail(FW2V_ERR_CUDA, "live hot-row merge block did not start");
            std::this_thread::yield();
        }
    }
    // After a pass (st has joined every training stream): the mean of the replicas
    // back into syn1, or stop the live merge and wait for its final sweep.
    void hot_end(cudaStream_t st) {
        if (!live()) {
            hot_sync(true, st);
            return;
        }
        FW2V_CK(launch_set_flag(live_stop, st));
        FW2V_CK(cudaStreamWaitEvent(st, live_done, 0));
        // One more sweep after every training kernel of the pass: the block may
        // have left early (no sentence started for a while, e.g. under a profiler
        // that serialises kernels); with the stop flag set it sweeps once and ends.
        FW2V_CK(launch_hot_live(model_view(), live_stop, live_started_d, st));
    }

    Sampler sampler() const {
        Sampler s;
        s.keep = keep_on ? keep.data() : nullptr;
        s.n_neg = cfg.negatives;
        if (cfg.sampler == FW2V_SAMPLER_ALIAS && !deterministic) {
            s.alias = &alias;
        } else {
            s.slots = slots.data();
            s.table_size = slots.size();
            s.mod = FastMod(slots.size());
        }
        return s;
    }

    // The corpus is cut into `workers` contiguous chunks (the reference's
    // producer partition, trainer.cpp:431-434; chunk p, batch k uses the stream
    // derive(seed, epoch, p, k)); `streams` batching threads, one CUDA stream
    // each, pull whole chunks from a shared counter (load balance across
    // uneven host cores). streams = 0: one thread per chunk.
    int chunks() const { return deterministic ? 1 : std::max(1, cfg.workers); }
    int producers() const {
        if (deterministic) return 1;
        const int t = cfg.streams > 0 ? cfg.streams : cfg.workers;
        return std::max(1, std::min(t, chunks()));
    }

    // Hogwild sentences in flight per stream (0 = no cap): a batch larger than
    // the cap runs as consecutive launches on its stream.
    // Hogwild: each lane runs its two slots' kernels on two streams, so a lane's
    // next sub-batch starts while the previous one's last sentences finish.
    int kernel_streams() const {
        static const int env = [] {
            const char* e = std::getenv("FW2V_KSTREAMS");  // experiments
            return e ? std::max(1, std::min(2, std::atoi(e))) : 2;
        }();
        return deterministic ? 1 : env;
    }

    int64_t inflight_per_stream(int streams) const {
        if (inflight_total <= 0) return 0;
        return std::max<int64_t>(1, inflight_total / std::max(1, streams));
    }

    cudaError_t launch(const BatchView& bv, bool serial, DevCounters* ctr, cudaStream_t st, int streams = 1) const {
        const int64_t cap = serial ? 0 : inflight_per_stream(streams);
        if (cap > 0 && bv.n_sentences > cap && k1s_shape.lanes > 0 &&
            (cfg.reuse_mode == kLifetime || cfg.reuse_mode == kWindowSnapshot)) {
            BatchView b = bv;  // K1s: one grid-stride launch of at most `cap` sentences in flight
            b.max_groups = static_cast<int32_t>(cap);
            return launch_one(b, false, ctr, st);
        }
        if (cap > 0 && bv.n_sentences > cap) {
            for (int64_t s0 = 0; s0 < bv.n_sentences; s0 += cap) {
                BatchView sub = bv;
                sub.offsets = bv.offsets + s0;
                sub.alpha = bv.alpha + s0;
                sub.obs_base = bv.obs_base + static_cast<int32_t>(s0);
                sub.n_sentences = static_cast<int32_t>(std::min<int64_t>(cap, bv.n_sentences - s0));
                cudaError_t e = launch_one(sub, false, ctr, st);
                if (e != cudaSuccess) return e;
            }
            return cudaSuccess;
        }
        return launch_one(bv, serial, ctr, st);
    }

    // resident != nullptr: no launch, *resident = sentences the Hogwild kernel
    // holds on the device at once (0 when unknown).
    cudaError_t launch_one(const BatchView& bv, bool serial, DevCounters* ctr, cudaStream_t st,
                           int* resident = nullptr) const {
        const ModelView mv = model_view();
        const bool fast = cfg.fast_sigmoid != 0;
        // Lifetime order: the K1s wavefront where it applies (N <= 5), else K1.
        if (!serial && cfg.reuse_mode == kLifetime && k1s_shape.lanes > 0)
            return launch_k1s(k1s_shape.lanes, k1s_shape.vec, mv, bv, cfg.negatives, wf, fast, true, ctr, st, resident);
        if (!serial && cfg.reuse_mode == kLifetime && shape.lanes > 0 && wf <= 5)
            return launch_k1(shape.lanes, shape.vec, mv, bv, cfg.negatives, wf, fast, ctr, st, resident);
        if (!serial && cfg.reuse_mode == kWindowSnapshot && k1s_shape.lanes > 0)
            return launch_k1s(k1s_shape.lanes, k1s_shape.vec, mv, bv, cfg.negatives, wf, fast, false, ctr, st, resident);
        if (resident != nullptr) {
            *resident = 0;
            return cudaSuccess;
        }
        return launch_k2(mv, bv, cfg.negatives, wf, cfg.reuse_mode, serial, ctr, st);
    }

    void ensure_lanes(int n, uint64_t cap_words, uint64_t cap_sent) {
        FW2V_CK(cudaSetDevice(cfg.device));
        if (static_cast<int>(lanes.size()) < n) lanes.resize(static_cast<size_t>(n));
        const size_t nn = static_cast<size_t>(std::max(cfg.negatives, 1));
        for (int i = 0; i < n; ++i) {
            Lane& ln = lanes[static_cast<size_t>(i)];
            if (!ln.stream) FW2V_CK(cudaStreamCreateWithFlags(&ln.stream, cudaStreamNonBlocking));
            if (!ln.stream2) FW2V_CK(cudaStreamCreateWithFlags(&ln.stream2, cudaStreamNonBlocking));
            if (!ln.copy) FW2V_CK(cudaStreamCreateWithFlags(&ln.copy, cudaStreamNonBlocking));
            if (!ln.d_ctr) FW2V_CK(cudaMalloc(&ln.d_ctr, sizeof(DevCounters)));
            if (ln.cap_words >= cap_words && ln.cap_sent >= cap_sent) continue;
            ln.release();
            BufferPool& pool = BufferPool::get();
            for (Slot& s : ln.slot) {
                s.h_ids = static_cast<int32_t*>(pool.host(4 * cap_words));
                s.h_negs = static_cast<int32_t*>(pool.host(4 * cap_words * nn));
                s.h_off = static_cast<uint32_t*>(pool.host(4 * (cap_sent + 1)));
                s.h_alpha = static_cast<float*>(pool.host(4 * cap_sent));
                s.d_ids = static_cast<int32_t*>(pool.device(4 * cap_words));
                s.d_negs = static_cast<int32_t*>(pool.device(4 * cap_words * nn + kNegPadBytes));
                // K1s reads a window's negatives as one fixed-size group (masked where
                // consumed), possibly past the copied part: keep it defined.
                FW2V_CK(cudaMemset(s.d_negs, 0, 4 * cap_words * nn + kNegPadBytes));
                s.d_off = static_cast<uint32_t*>(pool.device(4 * (cap_sent + 1)));
                s.d_alpha = static_cast<float*>(pool.device(4 * cap_sent));
                FW2V_CK(cudaEventCreateWithFlags(&s.h2d_done, cudaEventDisableTiming));
                FW2V_CK(cudaEventCreateWithFlags(&s.used, cudaEventDisableTiming));
            }
            ln.cap_words = cap_words;
            ln.cap_sent = cap_sent;
        }
    }

    ~fw2v_ctx() {
        cudaSetDevice(cfg.device);
        for (Lane& ln : lanes) {
            if (ln.stream) cudaStreamSynchronize(ln.stream);
            if (ln.stream2) cudaStreamSynchronize(ln.stream2);
            if (ln.copy) cudaStreamSynchronize(ln.copy);
            ln.release();
            cudaFree(ln.d_ctr);
            if (ln.stream) cudaStreamDestroy(ln.stream);
            if (ln.stream2) cudaStreamDestroy(ln.stream2);
            if (ln.copy) cudaStreamDestroy(ln.copy);
        }
        clique.reset();
        cudaFree(d_words);
        cudaFree(merge_base);
        cudaFree(merge_cnt);
        BufferPool::get().put(guard_snap);
        cudaFree(guard_flag);
        if (live_stream) {
            cudaStreamSynchronize(live_stream);
            cudaStreamDestroy(live_stream);
            cudaEventDestroy(live_go);
            cudaEventDestroy(live_done);
            cudaFree(live_stop);
            cudaFree(live_beat);
            cudaFreeHost(live_started_h);
        }
        cudaFree(hot_alloc);
        if (own_model) {
            BufferPool::get().put(syn0);
            BufferPool::get().put(syn1);
        }
    }
};

struct fw2v_plan {
    struct Batch {
        BatchView view;
    };
    std::vector<std::vector<Batch>> lanes;
    void* d_mem = nullptr;
    size_t bytes = 0;
    uint64_t words = 0, sentences = 0, batches = 0;
    int device = 0;
    ~fw2v_plan() {
        if (d_mem) {
            cudaSetDevice(device);
            cudaFree(d_mem);
        }
    }
};

namespace {

// Per-producer capacity: the largest batch a producer can assemble.
void capacity_for(const CorpusView& c, uint64_t begin, uint64_t end, uint64_t S, uint64_t* words,
                  uint64_t* sents) {
    uint64_t maxlen = 0;
    for (uint64_t s = begin; s < end; ++s) maxlen = std::max(maxlen, c.offsets[s + 1] - c.offsets[s]);
    const uint64_t chunk_words = c.offsets[end] - c.offsets[begin];
    *words = std::max<uint64_t>(1, std::min(chunk_words, S * maxlen));
    *sents = std::max<uint64_t>(1, std::min(end - begin, S));
}

uint64_t expected_epoch_words(const fw2v_ctx& x) {  // trainer.cpp:378-386
    if (!x.keep_on) return x.total_retained;
    double e = 0.0;
    for (int32_t w = 0; w < x.vocab; ++w) e += static_cast<double>(x.counts[static_cast<size_t>(w)]) * x.keep[static_cast<size_t>(w)];
    const uint64_t r = static_cast<uint64_t>(e + 0.5);
    return r > 0 ? r : 1;
}

// Hogwild collision budget. A sample row is drawn with
// probability p_w ~ count^power; with M sentences in flight, a drawn row is
// being updated by ~M (N+1) sum_w p_w^2 = M (N+1) / V_eff sentences at the
// same time, and their summed deltas act as one step of that many times alpha.
// The cap keeps M (N+1) alpha / V_eff <= 20 x 0.025. Measured on the text8
// shape (d=128, 5 epochs, no replicas, V_eff = 1,472; profiles/r02_budget_probe.txt):
// every sentence of a batch in flight (3,552 resident) trains to within 0.5% of
// the reference at alpha 0.025 and blows up at 0.1 (the divergence guard then
// halves the budget); round 1 used 8 x 0.025, tuned on an earlier kernel. Hot-row
// replicas (fw2v_config.hot_rows) split the top rows' traffic R ways, which
// lifts V_eff to ~9,700 there; the reference's 60-word pipeline test
// (V_eff = 60, alpha 0.05) is held to 100 sentences.
int64_t auto_inflight(const uint64_t* counts, int32_t vocab_size, double power, int n_neg, float alpha0, int hot_k,
                      int hot_r, int dim) {
    double z = 0.0, z2 = 0.0;
    for (int32_t w = 0; w < vocab_size; ++w) {
        const double p = std::pow(static_cast<double>(counts[w]), power);
        z += p;
        z2 += p * p / (w < hot_k ? hot_r : 1);  // a replicated row is shared by 1/R of the sentences
    }
    const double v_eff = z2 > 0.0 ? z * z / z2 : 1.0;
    // Wide rows tolerate less staleness (measured on the planted corpus: d=512 at
    // 888 sentences in flight +2.3% loss, at 512 +0.7%; d=128 fine at 3,552).
    // Above d=320 wide rows keep round 1's measured budget (8 x 0.025 scaled by
    // (128/d)^2): at d=512 the planted corpus is +2.3% at 20 x 0.025.
    const double wide = dim <= 128 ? 1.0 : (dim > 320 ? 0.4 : 1.0) * (128.0 / dim) * (128.0 / dim);
    const double m = 20.0 * 0.025 * v_eff / ((n_neg + 1) * static_cast<double>(alpha0)) * wide;
    return std::max<int64_t>(32, static_cast<int64_t>(std::ceil(m)));
}

} // namespace

extern "C" {

int fw2v_abi_version(void) { return FW2V_ABI_VERSION; }

const char* fw2v_last_error(void) { return g_error.c_str(); }

void fw2v_config_default(fw2v_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->dim = 128;
    c->window = 5;
    c->negatives = 5;
    c->epochs = 20;
    c->alpha0 = 0.025f;
    c->subsample = 1e-4;
    c->min_count = 5;
    c->batch_sentences = 10000;
    c->max_sentence_len = 1000;
    c->workers = 0;
    c->seed = 1;
    c->reuse_mode = FW2V_REUSE_LIFETIME;
    c->table_power = 0.75;
    c->table_size = 10000000;
    c->queue_capacity = 0;
    c->ignore_delimiters = 1;
    c->device = 0;
    c->deterministic = -1;
    c->sampler = FW2V_SAMPLER_REFERENCE;
    c->fast_sigmoid = 1;
    c->k1_lanes = 0;
    c->streams = 0;
    c->l1_refresh_log2 = 5;
    c->delta_writeback = 2;
    c->max_inflight = 0;
    c->hot_rows = 64;
    c->hot_replicas = 16;
    c->replica_merge = FW2V_MERGE_TOUCHED;
    c->divergence_guard = 1;
    c->hot_merge = 1;
}

int fw2v_validate_config(const fw2v_config* cfg) {
    return guarded([&] { validate(*cfg); });
}

int fw2v_device_count(int* count) {
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        g_error = cudaGetErrorString(e);
        return FW2V_ERR_NO_DEVICE;
    }
    return FW2V_OK;
}

int32_t fw2v_row_stride(const fw2v_config* cfg) { return row_stride_for(cfg->dim, cfg->k1_lanes); }

int fw2v_create(const fw2v_config* cfg, const uint64_t* counts, int32_t vocab_size, fw2v_ctx** out) {
    *out = nullptr;
    return guarded([&] {
        validate(*cfg);
        if (vocab_size < 1) fail(FW2V_ERR_EMPTY_VOCAB, "corpus has an empty vocabulary");
        auto x = std::make_unique<fw2v_ctx>();
        x->cfg = *cfg;
        if (x->cfg.workers == 0) {
            unsigned hw = std::thread::hardware_concurrency();
            x->cfg.workers = hw == 0 ? 1 : static_cast<int>(hw);  // resolve_config (config.cpp:190)
        }
        x->wf = context_width(x->cfg);
        x->vocab = vocab_size;
        // Sample rows are always written as red.global.add of the window delta
        // (row += delta, trainer.cpp:198-204); reads optionally go through L1.
        // delta_writeback: 1 red.add(final - loaded); 2 K1s stores ring rows straight
        // back (no shared-memory ring; K1 treats it as 1); 0 reference overwrite order.
        x->k1_flags = kFlagRedSamples | (cfg->delta_writeback != 0 ? kFlagDeltaRing : 0) |
                      (cfg->delta_writeback == 2 ? kFlagNoRing : 0);
        x->k1_flags |= cfg->l1_refresh_log2 > 0 ? (std::min(cfg->l1_refresh_log2, 15) << kFlagInvalShift) : kFlagL1Exact;
        if (const char* f = std::getenv("FW2V_NO_STAIR"); f != nullptr && *f != 0 && *f != '0') x->k1_flags |= kFlagNoStair;
        if (const char* f = std::getenv("FW2V_K1_FLAGS")) x->k1_flags = std::atoi(f);  // experiments
        x->inflight_total = cfg->max_inflight > 0 ? cfg->max_inflight
                            : cfg->max_inflight == 0 ? auto_inflight(counts, vocab_size, cfg->table_power, cfg->negatives, cfg->alpha0, 0, 1, cfg->dim) : 0;
        x->deterministic = cfg->deterministic == 1 || (cfg->deterministic < 0 && x->cfg.workers == 1);
        x->shape = choose_shape(cfg->dim, cfg->k1_lanes);
        x->stride = row_stride_for(cfg->dim, cfg->k1_lanes);
        x->k1s_shape = (cfg->reuse_mode == kWindowSnapshot || cfg->reuse_mode == kLifetime)
                           ? choose_k1s_shape(x->stride, x->shape, cfg->k1_lanes, cfg->negatives, x->wf,
                                              cfg->reuse_mode == kLifetime)
                           : Shape{};
        if (!x->deterministic && cfg->reuse_mode == kLifetime && (x->shape.lanes == 0 || x->wf > 5))
            fail(FW2V_ERR_UNSUPPORTED, "K1 covers dim <= 512 and window <= 10 (W_f <= 5)");
        if (x->wf > 16) fail(FW2V_ERR_UNSUPPORTED, "window > 32 is not supported");
        x->counts.assign(counts, counts + vocab_size);
        for (uint64_t c : x->counts) x->total_retained += c;
        x->keep.resize(static_cast<size_t>(vocab_size));
        x->keep_on = keep_probs(counts, vocab_size, cfg->subsample, x->keep.data());
        if (!(cfg->sampler == FW2V_SAMPLER_ALIAS && !x->deterministic)) {  // fw2v_ctx::sampler() reads it
            x->slots.resize(cfg->table_size);
            build_table(counts, vocab_size, cfg->table_power, cfg->table_size, x->slots.data());
        }
        if (cfg->sampler == FW2V_SAMPLER_ALIAS) x->alias.build(counts, vocab_size, cfg->table_power);
        require_device(cfg->device);
        const size_t bytes = sizeof(float) * static_cast<size_t>(vocab_size) * static_cast<size_t>(x->stride);
        // (From the process-wide cache: a ringvec::train call creates one context.)
        x->syn0 = static_cast<float*>(BufferPool::get().device(bytes));
        x->syn1 = static_cast<float*>(BufferPool::get().device(bytes));
        Rng r = Rng::derive(cfg->seed, 0x696e6974ULL);  // "init" stream, model.cpp:26
        FW2V_CK(launch_init_model(x->model_view(), r.state, nullptr));
        FW2V_CK(cudaDeviceSynchronize());
        if (!x->deterministic && x->k1s_shape.lanes > 0 && cfg->hot_rows > 0) {
            x->hot_k = std::min(cfg->hot_rows, vocab_size);
            x->hot_r = cfg->hot_replicas;
            FW2V_CK(cudaMalloc(&x->hot_alloc, sizeof(float) * (static_cast<size_t>(x->hot_k) * x->hot_r + 1) * x->stride));
            x->place_hot();
            x->inflight_total = cfg->max_inflight > 0 ? cfg->max_inflight
                                : cfg->max_inflight == 0 ? auto_inflight(counts, vocab_size, cfg->table_power, cfg->negatives,
                                                                         cfg->alpha0, x->live() ? 0 : x->hot_k, x->hot_r, cfg->dim)
                                                         : 0;
        }
        if (x->inflight_total > 0 && !x->deterministic) {
            // The budget only matters when it is below what the device holds at once.
            int resident = 0;
            FW2V_CK(x->launch_one(BatchView{}, false, nullptr, nullptr, &resident));
            if (cfg->max_inflight == 0 && resident > 0 && resident <= x->inflight_total) x->inflight_total = 0;
        }
        *out = x.release();
    });
}

void fw2v_destroy(fw2v_ctx* ctx) { delete ctx; }

void fw2v_release_cached(void) { BufferPool::get().release_all(); }

int fw2v_init_model(fw2v_ctx* x, uint64_t seed) {
    return guarded([&] {
        FW2V_CK(cudaSetDevice(x->cfg.device));
        Rng r = Rng::derive(seed, 0x696e6974ULL);
        FW2V_CK(launch_init_model(x->model_view(), r.state, nullptr));
        FW2V_CK(cudaDeviceSynchronize());
        x->words_trained = 0;
    });
}

int fw2v_get_model(fw2v_ctx* x, float* input, float* output) {
    return guarded([&] {
        FW2V_CK(cudaSetDevice(x->cfg.device));
        const size_t w = sizeof(float) * static_cast<size_t>(x->cfg.dim);
        const size_t p = sizeof(float) * static_cast<size_t>(x->stride);
        if (input) FW2V_CK(cudaMemcpy2D(input, w, x->syn0, p, w, static_cast<size_t>(x->vocab), cudaMemcpyDeviceToHost));
        if (output) FW2V_CK(cudaMemcpy2D(output, w, x->syn1, p, w, static_cast<size_t>(x->vocab), cudaMemcpyDeviceToHost));
    });
}

int fw2v_set_model(fw2v_ctx* x, const float* input, const float* output) {
    return guarded([&] {
        FW2V_CK(cudaSetDevice(x->cfg.device));
        const size_t w = sizeof(float) * static_cast<size_t>(x->cfg.dim);
        const size_t p = sizeof(float) * static_cast<size_t>(x->stride);
        const size_t bytes = p * static_cast<size_t>(x->vocab);
        if (input) {
            FW2V_CK(cudaMemset(x->syn0, 0, bytes));
            FW2V_CK(cudaMemcpy2D(x->syn0, p, input, w, w, static_cast<size_t>(x->vocab), cudaMemcpyHostToDevice));
        }
        if (output) {
            FW2V_CK(cudaMemset(x->syn1, 0, bytes));
            FW2V_CK(cudaMemcpy2D(x->syn1, p, output, w, w, static_cast<size_t>(x->vocab), cudaMemcpyHostToDevice));
        }
    });
}

int fw2v_save_model(fw2v_ctx* x, int32_t which, const char* tokens, const uint64_t* token_offsets, const char* path,
                    int32_t threads) {
    std::vector<float> host;
    int rc = guarded([&] {
        if (which != 0 && which != 1) fail(FW2V_ERR_BAD_ARGUMENT, "which must be 0 (input) or 1 (output)");
        FW2V_CK(cudaSetDevice(x->cfg.device));
        host.resize(static_cast<size_t>(x->vocab) * static_cast<size_t>(x->stride));
        FW2V_CK(cudaMemcpy(host.data(), which == 0 ? x->syn0 : x->syn1, sizeof(float) * host.size(),
                           cudaMemcpyDeviceToHost));
    });
    if (rc != FW2V_OK) return rc;
    return fw2v_write_embeddings(host.data(), x->vocab, x->cfg.dim, x->stride, tokens, token_offsets, path, threads);
}

int fw2v_write_embeddings(const float* rows, int32_t vocab_size, int32_t dim, int64_t row_stride, const char* tokens,
                          const uint64_t* token_offsets, const char* path, int32_t threads) {
    std::string err;
    const int rc = write_embeddings(rows, vocab_size, dim, row_stride, tokens, token_offsets, path, threads, &err);
    if (rc != FW2V_OK) g_error = err;
    return rc;
}

int fw2v_model_device(fw2v_ctx* x, float** syn0, float** syn1, int32_t* stride) {
    *syn0 = x->syn0;
    *syn1 = x->syn1;
    *stride = x->stride;
    return FW2V_OK;
}

int fw2v_attach_model(fw2v_ctx* x, float* syn0, float* syn1) {
    return guarded([&] {
        if (!syn0 || !syn1) fail(FW2V_ERR_BAD_ARGUMENT, "null model pointer");
        FW2V_CK(cudaSetDevice(x->cfg.device));
        FW2V_CK(cudaDeviceSynchronize());
        if (x->own_model) {
            BufferPool::get().put(x->syn0);
            BufferPool::get().put(x->syn1);
        }
        x->syn0 = syn0;
        x->syn1 = syn1;
        x->own_model = false;
        x->place_hot();  // replicas are addressed relative to syn1
    });
}

int fw2v_train_sentences(fw2v_ctx* x, const uint64_t* offsets, uint64_t n_sentences, const int32_t* ids,
                         const int32_t* negatives, const float* alphas, int32_t serial,
                         fw2v_counters* counters) {
    return guarded([&] {
        FW2V_CK(cudaSetDevice(x->cfg.device));
        const uint64_t words = offsets[n_sentences] - offsets[0];
        const int n = x->cfg.negatives;
        std::vector<uint32_t> off(n_sentences + 1);
        for (uint64_t s = 0; s <= n_sentences; ++s) off[s] = static_cast<uint32_t>(offsets[s] - offsets[0]);
        int32_t *d_ids = nullptr, *d_negs = nullptr;
        uint32_t* d_off = nullptr;
        float* d_alpha = nullptr;
        DevCounters* d_ctr = nullptr;
        struct Free {
            void* p[5];
            ~Free() { for (void* q : p) cudaFree(q); }
        } guard{{nullptr, nullptr, nullptr, nullptr, nullptr}};
        FW2V_CK(cudaMalloc(&d_ids, 4 * std::max<uint64_t>(words, 1))); guard.p[0] = d_ids;
        FW2V_CK(cudaMalloc(&d_negs, 4 * std::max<uint64_t>(words * n, 1) + kNegPadBytes)); guard.p[1] = d_negs;
        FW2V_CK(cudaMemset(d_negs, 0, 4 * std::max<uint64_t>(words * n, 1) + kNegPadBytes));
        FW2V_CK(cudaMalloc(&d_off, 4 * (n_sentences + 1))); guard.p[2] = d_off;
        FW2V_CK(cudaMalloc(&d_alpha, 4 * std::max<uint64_t>(n_sentences, 1))); guard.p[3] = d_alpha;
        FW2V_CK(cudaMalloc(&d_ctr, sizeof(DevCounters))); guard.p[4] = d_ctr;
        FW2V_CK(cudaMemset(d_ctr, 0, sizeof(DevCounters)));
        if (words) FW2V_CK(cudaMemcpy(d_ids, ids + offsets[0], 4 * words, cudaMemcpyHostToDevice));
        if (words != 0 && n != 0) FW2V_CK(cudaMemcpy(d_negs, negatives, 4 * words * n, cudaMemcpyHostToDevice));
        FW2V_CK(cudaMemcpy(d_off, off.data(), 4 * (n_sentences + 1), cudaMemcpyHostToDevice));
        if (n_sentences) FW2V_CK(cudaMemcpy(d_alpha, alphas, 4 * n_sentences, cudaMemcpyHostToDevice));
        BatchView bv{d_ids, d_off, d_negs, d_alpha, static_cast<int32_t>(n_sentences)};
        if (!serial && x->hot_k > 0) x->hot_begin(nullptr);
        FW2V_CK(x->launch(bv, serial != 0, d_ctr, nullptr));
        if (!serial && x->hot_k > 0) x->hot_end(nullptr);
        FW2V_CK(cudaDeviceSynchronize());
        DevCounters h{};
        FW2V_CK(cudaMemcpy(&h, d_ctr, sizeof(h), cudaMemcpyDeviceToHost));
        if (counters) {
            counters->context_reads = h.context_reads;
            counters->context_writes = h.context_writes;
            counters->sample_reads = h.sample_reads;
            counters->sample_writes = h.sample_writes;
            counters->ring_hits = h.ring_hits;
            counters->words = h.words;
            counters->sentences = h.sentences;
        }
    });
}

} // extern "C"

namespace {

// --------------------------------------------------------------- passes
// One contiguous range of the corpus with its producer index p: chunk p, batch
// k uses the reference stream derive(seed, epoch, p, k) (trainer.cpp:442-443).
struct ChunkSpan {
    uint64_t p, begin, end;
};

// State shared by every pass of one run (all GPUs of a multi-GPU run): the
// global word reservation behind lr_at (trainer.cpp:479-487 counts the words of
// every worker), the observer's serial counter.
struct RunShared {
    std::atomic<uint64_t> reserved{0};
    uint64_t schedule_total = 1;
    // Schedule position of local word w: origin + (w - origin) * scale. A process
    // that trains `scale` times fewer shards than the whole job extrapolates the
    // global count between exchanges (exact at every average).
    uint64_t origin = 0, scale = 1;
    uint64_t position(uint64_t w) const { return origin + (w - origin) * scale; }
    std::atomic<uint64_t> serial{0};
    // Whether the last pass already started the next one's reservations.
    std::atomic<bool> prefetched{false};
    std::mutex obs_mutex;
    fw2v_observer_fn observer = nullptr;
    void* observer_user = nullptr;
};

struct PassOut {
    fw2v_counters traffic{}, analytic{};
    uint64_t batch_words = 0, batch_nanos = 0, h2d = 0;
    double kernel_seconds = 0.0;
};

void add_counters(fw2v_counters& a, const fw2v_counters& b) {
    a.context_reads += b.context_reads;
    a.context_writes += b.context_writes;
    a.sample_reads += b.sample_reads;
    a.sample_writes += b.sample_writes;
    a.ring_hits += b.ring_hits;
    a.words += b.words;
    a.sentences += b.sentences;
}

// Trains ctx x over `spans` (the producer loop of train(), trainer.cpp:429-503):
// `producers()` batching threads pull whole spans from a shared counter,
// assemble sub-batches into pinned slots, copy H2D on the lane's copy stream and
// launch on the lane's kernel streams. Hogwild hot-row replicas are broadcast
// before and averaged after the pass. Returns after every kernel finished.
void run_pass(fw2v_ctx* x, const CorpusView& corpus, const std::vector<ChunkSpan>& spans, int epoch, RunShared& sh,
              PassOut* out, const std::vector<ChunkSpan>* next_spans = nullptr) {
    FW2V_CK(cudaSetDevice(x->cfg.device));
    const fw2v_config& cfg = x->cfg;
    const int NS = static_cast<int>(spans.size());
    const int P = std::max(1, std::min(x->producers(), NS));  // batching threads = CUDA streams
    uint64_t cap_w = 1, cap_s = 1, chunk = 1;
    for (const ChunkSpan& c : spans) {
        uint64_t w, sn;
        capacity_for(corpus, c.begin, c.end, cfg.batch_sentences, &w, &sn);
        cap_w = std::max(cap_w, w);
        cap_s = std::max(cap_s, sn);
        chunk = std::max(chunk, c.end - c.begin);
    }
    x->ensure_lanes(P, cap_w, cap_s);
    const uint64_t pass = ++x->pass_seq;  // matches a lane's stash to the pass it was made for
    // Sub-batches of ~256-511 sentences (equal parts of a chunk; enough to keep
    // the device full across the streams), never above S.
    static const uint64_t sub_target = [] {
        const char* e = std::getenv("FW2V_SUB_TARGET");  // experiments
        return e ? std::max<uint64_t>(1, static_cast<uint64_t>(std::atoll(e))) : uint64_t{256};
    }();
    const uint64_t parts = std::max<uint64_t>(1, chunk / sub_target);
    const uint64_t sub = x->deterministic ? cfg.batch_sentences
                                          : std::min<uint64_t>(cfg.batch_sentences, (chunk + parts - 1) / parts);
    static const uint64_t first_sub_env = [] {
        const char* e = std::getenv("FW2V_FIRST_SUB");  // experiments
        return e ? static_cast<uint64_t>(std::atoll(e)) : uint64_t{64};
    }();
    const uint64_t first_sub = x->deterministic ? 0 : first_sub_env;
    const int KS = x->kernel_streams();  // kernel streams per lane
    const Sampler sp = x->sampler();
    const int n_neg = cfg.negatives;
    const bool hot = !x->deterministic && x->hot_k > 0;

    struct Events {
        cudaEvent_t synced = nullptr, t0 = nullptr, t1 = nullptr;
        std::vector<cudaEvent_t> join;
        ~Events() {
            for (cudaEvent_t e : {synced, t0, t1})
                if (e) cudaEventDestroy(e);
            for (cudaEvent_t e : join) cudaEventDestroy(e);
        }
    } ev;
    FW2V_CK(cudaEventCreateWithFlags(&ev.synced, cudaEventDisableTiming));
    FW2V_CK(cudaEventCreate(&ev.t0));
    FW2V_CK(cudaEventCreate(&ev.t1));
    ev.join.resize(static_cast<size_t>(2 * P), nullptr);
    for (auto& e : ev.join) FW2V_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaStream_t s0 = x->lanes[0].stream;
    // Counters cleared and hot replicas broadcast on lane 0's stream; every
    // kernel stream starts after them.
    FW2V_CK(cudaEventRecord(ev.t0, s0));
    for (int p = 0; p < P; ++p) FW2V_CK(cudaMemsetAsync(x->lanes[static_cast<size_t>(p)].d_ctr, 0, sizeof(DevCounters), s0));
    if (hot) x->hot_begin(s0);
    FW2V_CK(cudaEventRecord(ev.synced, s0));
    for (int p = 0; p < P; ++p) {
        if (p > 0) FW2V_CK(cudaStreamWaitEvent(x->lanes[static_cast<size_t>(p)].stream, ev.synced, 0));
        if (KS > 1) FW2V_CK(cudaStreamWaitEvent(x->lanes[static_cast<size_t>(p)].stream2, ev.synced, 0));
    }
    // FW2V_TRACE=1: per sub-batch host and device timeline on stderr (diagnostics).
    struct TraceRec {
        int p;
        double t0, t1, t2;
        cudaEvent_t k0, k1;
        uint64_t words;
    };
    static const bool trace = std::getenv("FW2V_TRACE") != nullptr;
    std::vector<std::vector<TraceRec>> tr(static_cast<size_t>(P));
    std::vector<uint64_t> an_acc(static_cast<size_t>(P) * 5, 0);
    std::vector<std::string> errors(static_cast<size_t>(P));
    std::atomic<uint64_t> batch_words{0}, batch_nanos{0}, h2d{0};
    const double t0 = wall_seconds();
    std::vector<std::thread> threads;
    // Span claiming: thread th takes span th first (a stashed first sub-batch of
    // this pass, see below, was assembled from it), then whole spans dynamically.
    std::atomic<int> next_span{std::min(P, NS)};
    // Cross-epoch prefetch (Hogwild fw2v_train_corpus): once every thread has
    // assembled this pass, each assembles and ships (H2D) the first sub-batch of
    // its first span of the NEXT pass into a free slot, so that pass's kernels
    // start as soon as this pass's end work (replica average, divergence check)
    // is done instead of after a host assembly.
    const bool prefetch = next_spans != nullptr && !x->deterministic && sh.observer == nullptr;
    int assembled = 0;  // threads done with this pass's spans (under asm_mu)
    std::mutex asm_mu;
    std::condition_variable asm_cv;
    for (int th = 0; th < P; ++th) {
        threads.emplace_back([&, th] {
            try {
                FW2V_CK(cudaSetDevice(cfg.device));
                Lane& ln = x->lanes[static_cast<size_t>(th)];
                double cpu = 0.0;
                uint64_t wsum = 0;
                uint64_t* an = &an_acc[static_cast<size_t>(th) * 5];
                int which = 0;
                // Iteration state of one span: batch k (reference stream derive(seed,
                // epoch, p, k), S kept sentences) is shipped in sub-batches drawn from
                // the same stream in the same order, so the kernels of one sub-batch
                // overlap the host assembly of the next.
                struct SpanIt {
                    uint64_t p = 0, cursor = 0, end = 0, k = 0, left = 0;
                    Rng rng;
                };
                auto open_span = [&](const ChunkSpan& cs_, int ep) {
                    SpanIt it;
                    it.p = cs_.p;
                    it.cursor = cs_.begin;
                    it.end = cs_.end;
                    it.left = cfg.batch_sentences;
                    it.rng = Rng::derive(cfg.seed, static_cast<uint64_t>(ep), cs_.p, 0);
                    return it;
                };
                // Assembles the next sub-batch of `it` into slot `which` and issues its
                // H2D; returns kept sentences (0: nothing kept, slot untouched).
                auto assemble_ship = [&](SpanIt& it, int ep, bool first, uint64_t* words_out, uint64_t* obs0,
                                         double* w0_out) -> uint64_t {
                    if (it.left == 0) {
                        ++it.k;
                        it.left = cfg.batch_sentences;
                        it.rng = Rng::derive(cfg.seed, static_cast<uint64_t>(ep), it.p, it.k);
                    }
                    Slot& sl = ln.slot[which];
                    if (sl.in_flight) FW2V_CK(cudaEventSynchronize(sl.h2d_done));
                    const double c0 = thread_cpu_seconds();
                    *w0_out = trace ? wall_seconds() : 0.0;
                    uint64_t words = 0;
                    const BatchOut bo{sl.h_ids, sl.h_off, sl.h_negs, ln.cap_words, ln.cap_sent};
                    // A short first sub-batch per thread gets the device busy early.
                    const uint64_t want = std::min(it.left, first && first_sub > 0 ? std::min<uint64_t>(sub, first_sub) : sub);
                    const uint64_t kept = assemble(corpus, it.cursor, it.end, want, sp, it.rng, bo, &words);
                    it.left -= kept;
                    // Learning rate per sentence from the global schedule (trainer.cpp:479-481).
                    const uint64_t base = sh.reserved.fetch_add(words);
                    for (uint64_t q = 0; q < kept; ++q) sl.h_alpha[q] = lr_at(sh.position(base + sl.h_off[q]), sh.schedule_total, cfg.alpha0);
                    cpu += thread_cpu_seconds() - c0;
                    *words_out = words;
                    if (kept == 0) return 0;
                    wsum += words;
                    for (uint64_t q = 0; q < kept; ++q) {
                        uint64_t t[5];
                        analytic(sl.h_off[q + 1] - sl.h_off[q], x->wf, n_neg, cfg.reuse_mode, t);
                        for (int z = 0; z < 5; ++z) an[z] += t[z];
                    }
                    // Observer (test mode): serial numbers in batch order; the calls
                    // are replayed from the kernel's own (sentence, target) log below.
                    *obs0 = sh.observer ? sh.serial.fetch_add(kept) : 0;
                    if (sh.observer && sl.obs_cap < words) {
                        BufferPool& pool = BufferPool::get();
                        pool.put(sl.d_obs);
                        pool.put(sl.d_obs_n);
                        sl.d_obs = static_cast<unsigned long long*>(pool.device(8 * words));
                        sl.d_obs_n = static_cast<unsigned*>(pool.device(sizeof(unsigned)));
                        sl.obs_cap = words;
                    }
                    // H2D on the lane's copy stream once the kernel that last read
                    // this slot's device buffers is done; the kernel waits for the copy.
                    const cudaStream_t cs = ln.copy;
                    if (sl.in_flight) FW2V_CK(cudaStreamWaitEvent(cs, sl.used, 0));
                    FW2V_CK(cudaMemcpyAsync(sl.d_ids, sl.h_ids, 4 * words, cudaMemcpyHostToDevice, cs));
                    if (n_neg) FW2V_CK(cudaMemcpyAsync(sl.d_negs, sl.h_negs, 4 * words * n_neg, cudaMemcpyHostToDevice, cs));
                    FW2V_CK(cudaMemcpyAsync(sl.d_off, sl.h_off, 4 * (kept + 1), cudaMemcpyHostToDevice, cs));
                    FW2V_CK(cudaMemcpyAsync(sl.d_alpha, sl.h_alpha, 4 * kept, cudaMemcpyHostToDevice, cs));
                    FW2V_CK(cudaEventRecord(sl.h2d_done, cs));
                    sl.in_flight = true;
                    h2d.fetch_add(4 * (words * (1 + n_neg) + 2 * kept + 1));
                    return kept;
                };
                // Launches the sub-batch shipped into slot `which`, then flips the slot.
                auto launch_slot = [&](uint64_t kept, uint64_t words, uint64_t obs_serial0, double w0) {
                    Slot& sl = ln.slot[which];
                    const cudaStream_t st = which == 1 && KS > 1 ? ln.stream2 : ln.stream;
                    FW2V_CK(cudaStreamWaitEvent(st, sl.h2d_done, 0));
                    BatchView bv{sl.d_ids, sl.d_off, sl.d_negs, sl.d_alpha, static_cast<int32_t>(kept)};
                    if (sh.observer) {
                        FW2V_CK(cudaMemsetAsync(sl.d_obs_n, 0, sizeof(unsigned), st));
                        bv.obs_log = sl.d_obs;
                        bv.obs_count = sl.d_obs_n;
                    }
                    TraceRec rec{};
                    if (trace) {
                        rec = TraceRec{th, w0 - t0, 0.0, 0.0, nullptr, nullptr, words};
                        rec.t1 = wall_seconds() - t0;
                        FW2V_CK(cudaEventCreate(&rec.k0));
                        FW2V_CK(cudaEventCreate(&rec.k1));
                        FW2V_CK(cudaEventRecord(rec.k0, st));
                    }
                    FW2V_CK(x->launch(bv, x->deterministic, ln.d_ctr, st, KS * P));
                    FW2V_CK(cudaEventRecord(sl.used, st));
                    if (sh.observer) {  // replay the device's window order (trainer.cpp:246)
                        unsigned n_obs = 0;
                        std::vector<unsigned long long> log(words);
                        FW2V_CK(cudaStreamSynchronize(st));
                        FW2V_CK(cudaMemcpy(&n_obs, sl.d_obs_n, sizeof(unsigned), cudaMemcpyDeviceToHost));
                        if (n_obs > words) fail(FW2V_ERR_CUDA, "observer log overflow");
                        FW2V_CK(cudaMemcpy(log.data(), sl.d_obs, 8 * n_obs, cudaMemcpyDeviceToHost));
                        std::lock_guard<std::mutex> lk(sh.obs_mutex);
                        for (unsigned z = 0; z < n_obs; ++z)
                            sh.observer(sh.observer_user, obs_serial0 + (log[z] >> 32), log[z] & 0xffffffffu);
                    }
                    if (trace) {
                        FW2V_CK(cudaEventRecord(rec.k1, st));
                        rec.t2 = wall_seconds() - t0;
                        tr[static_cast<size_t>(th)].push_back(rec);
                    }
                    which ^= 1;
                };
                auto run_span = [&](SpanIt it, bool first) {
                    while (it.cursor < it.end) {
                        uint64_t words = 0, obs0 = 0;
                        double w0 = 0.0;
                        const uint64_t kept = assemble_ship(it, epoch, first && wsum == 0, &words, &obs0, &w0);
                        if (kept > 0) launch_slot(kept, words, obs0, w0);
                    }
                };
                // This pass's first sub-batch may have been shipped by the previous pass.
                Lane::Stash& stash = ln.stash;
                if (stash.ready && stash.pass == pass) {
                    stash.ready = false;
                    which = stash.slot;
                    cpu += stash.cpu;
                    wsum += stash.words;
                    for (int z = 0; z < 5; ++z) an[z] += stash.an[z];
                    h2d.fetch_add(stash.h2d);
                    launch_slot(stash.kept, stash.words, 0, t0);
                    SpanIt it;
                    it.p = stash.p;
                    it.cursor = stash.cursor;
                    it.end = stash.end;
                    it.k = stash.k;
                    it.left = stash.left;
                    it.rng = stash.rng;
                    run_span(it, false);
                } else if (th < NS) {
                    run_span(open_span(spans[static_cast<size_t>(th)], epoch), true);
                }
                for (int si = next_span.fetch_add(1); si < NS; si = next_span.fetch_add(1))
                    run_span(open_span(spans[static_cast<size_t>(si)], epoch), true);
                {
                    std::lock_guard<std::mutex> lk(asm_mu);
                    if (++assembled == P) asm_cv.notify_all();
                }
                if (prefetch && th < static_cast<int>(next_spans->size())) {
                    // Every thread's reservations of this pass precede the next pass's.
                    {
                        std::unique_lock<std::mutex> lk(asm_mu);
                        asm_cv.wait(lk, [&] { return assembled == P; });
                    }
                    SpanIt it = open_span((*next_spans)[static_cast<size_t>(th)], epoch + 1);
                    const double cpu0 = cpu;
                    const uint64_t ws0 = wsum;
                    uint64_t an0[5];
                    for (int z = 0; z < 5; ++z) an0[z] = an[z];
                    uint64_t words = 0, obs0 = 0, kept = 0;
                    double w0 = 0.0;
                    while (kept == 0 && it.cursor < it.end) kept = assemble_ship(it, epoch + 1, true, &words, &obs0, &w0);
                    if (kept > 0) {
                        // Attributed to the next pass (words, CPU, analytic counters, H2D).
                        stash.ready = true;
                        stash.pass = pass + 1;
                        stash.slot = which;
                        stash.kept = kept;
                        stash.words = words;
                        stash.p = it.p;
                        stash.cursor = it.cursor;
                        stash.end = it.end;
                        stash.k = it.k;
                        stash.left = it.left;
                        stash.rng = it.rng;
                        stash.cpu = cpu - cpu0;
                        cpu = cpu0;
                        wsum = ws0;
                        for (int z = 0; z < 5; ++z) {
                            stash.an[z] = an[z] - an0[z];
                            an[z] = an0[z];
                        }
                        stash.h2d = 4 * (words * (1 + n_neg) + 2 * kept + 1);
                        h2d.fetch_sub(stash.h2d);
                        sh.prefetched.store(true);
                    }
                }
                batch_words.fetch_add(wsum);
                batch_nanos.fetch_add(static_cast<uint64_t>(cpu * 1e9));
            } catch (const Failure& f) {
                errors[static_cast<size_t>(th)] = f.msg;
            }
        });
    }
    for (auto& t : threads) t.join();
    for (const auto& e : errors)
        if (!e.empty()) {
            for (int p = 0; p < P; ++p) {  // drain before the caller frees anything
                cudaStreamSynchronize(x->lanes[static_cast<size_t>(p)].stream);
                cudaStreamSynchronize(x->lanes[static_cast<size_t>(p)].stream2);
            }
            fail(FW2V_ERR_CUDA, e);
        }
    // Join every kernel stream on lane 0's stream, fold the replicas back; the
    // pass ends there (t1: device span of the pass = kernel_seconds).
    for (int p = 0; p < P; ++p) {
        Lane& ln = x->lanes[static_cast<size_t>(p)];
        FW2V_CK(cudaEventRecord(ev.join[static_cast<size_t>(2 * p)], ln.stream));
        FW2V_CK(cudaStreamWaitEvent(s0, ev.join[static_cast<size_t>(2 * p)], 0));
        FW2V_CK(cudaEventRecord(ev.join[static_cast<size_t>(2 * p + 1)], ln.stream2));
        FW2V_CK(cudaStreamWaitEvent(s0, ev.join[static_cast<size_t>(2 * p + 1)], 0));
    }
    if (hot) x->hot_end(s0);
    FW2V_CK(cudaEventRecord(ev.t1, s0));
    FW2V_CK(cudaEventSynchronize(ev.t1));
    float ms = 0.0f;
    FW2V_CK(cudaEventElapsedTime(&ms, ev.t0, ev.t1));
    if (trace) {
        std::fprintf(stderr, "[fw2v trace] epoch %d wall %.3f ms (host: asm start/end, launch; device: kernel start/end ms)\n",
                     epoch, 1e3 * (wall_seconds() - t0));
        for (auto& lane_tr : tr)
            for (TraceRec& r : lane_tr) {
                float a = 0.0f, b = 0.0f;
                cudaEventElapsedTime(&a, ev.t0, r.k0);
                cudaEventElapsedTime(&b, ev.t0, r.k1);
                std::fprintf(stderr, "[fw2v trace] p%02d words %7llu host %.3f %.3f %.3f dev %.3f %.3f\n", r.p,
                             static_cast<unsigned long long>(r.words), 1e3 * r.t0, 1e3 * r.t1, 1e3 * r.t2, a, b);
                cudaEventDestroy(r.k0);
                cudaEventDestroy(r.k1);
            }
    }
    PassOut o;
    o.kernel_seconds = 1e-3 * ms;
    for (int p = 0; p < P; ++p) {
        DevCounters h{};
        FW2V_CK(cudaMemcpy(&h, x->lanes[static_cast<size_t>(p)].d_ctr, sizeof(h), cudaMemcpyDeviceToHost));
        add_counters(o.traffic, fw2v_counters{h.context_reads, h.context_writes, h.sample_reads, h.sample_writes,
                                              h.ring_hits, h.words, h.sentences});
        const uint64_t* an = &an_acc[static_cast<size_t>(p) * 5];
        add_counters(o.analytic, fw2v_counters{an[0], an[1], an[2], an[3], an[4], 0, 0});
    }
    o.analytic.words = o.traffic.words;
    o.analytic.sentences = o.traffic.sentences;
    o.batch_words = batch_words.load();
    o.batch_nanos = batch_nanos.load();
    o.h2d = h2d.load();
    x->words_trained += o.traffic.words;
    *out = o;
}

// The reference's producer partition: `nc` contiguous chunks of ceil(n/nc)
// sentences (trainer.cpp:431-434), chunk p keeping its index for the streams.
std::vector<ChunkSpan> chunk_spans(uint64_t n_sentences, int nc) {
    std::vector<ChunkSpan> v;
    const uint64_t chunk = (n_sentences + nc - 1) / std::max(nc, 1);
    for (int p = 0; p < nc; ++p) {
        const uint64_t b = std::min(n_sentences, static_cast<uint64_t>(p) * chunk);
        v.push_back(ChunkSpan{static_cast<uint64_t>(p), b, std::min(n_sentences, b + chunk)});
    }
    return v;
}

void accumulate(fw2v_report& rep, const PassOut& o) {
    add_counters(rep.traffic, o.traffic);
    add_counters(rep.analytic, o.analytic);
    rep.words_trained += o.traffic.words;
    rep.sentences_trained += o.traffic.sentences;
    rep.kernel_seconds += o.kernel_seconds;
    rep.h2d_bytes += o.h2d;
}

// ------------------------------------------------------ divergence guard
constexpr int kGuardRetries = 4;

void guard_save(fw2v_ctx* x) {
    const size_t n = x->model_floats();
    if (x->guard_snap == nullptr) {
        x->guard_snap = static_cast<float*>(BufferPool::get().device(2 * n * sizeof(float)));
        FW2V_CK(cudaMalloc(&x->guard_flag, sizeof(int)));
    }
    FW2V_CK(cudaMemcpyAsync(x->guard_snap, x->syn0, n * sizeof(float), cudaMemcpyDeviceToDevice, nullptr));
    FW2V_CK(cudaMemcpyAsync(x->guard_snap + n, x->syn1, n * sizeof(float), cudaMemcpyDeviceToDevice, nullptr));
    FW2V_CK(cudaMemsetAsync(x->guard_flag, 0, sizeof(int), nullptr));
    FW2V_CK(cudaStreamSynchronize(nullptr));
}

bool guard_finite(fw2v_ctx* x) {
    const size_t n = x->model_floats();
    FW2V_CK(launch_nonfinite(x->syn0, n, x->guard_flag, nullptr));
    FW2V_CK(launch_nonfinite(x->syn1, n, x->guard_flag, nullptr));
    int flag = 0;
    FW2V_CK(cudaMemcpy(&flag, x->guard_flag, sizeof(int), cudaMemcpyDeviceToHost));
    return flag == 0;
}

void guard_restore(fw2v_ctx* x) {
    const size_t n = x->model_floats();
    FW2V_CK(cudaMemcpy(x->syn0, x->guard_snap, n * sizeof(float), cudaMemcpyDeviceToDevice));
    FW2V_CK(cudaMemcpy(x->syn1, x->guard_snap + n, n * sizeof(float), cudaMemcpyDeviceToDevice));
}

void guard_halve_inflight(fw2v_ctx* x) {
    int64_t cur = x->inflight_total;
    if (cur <= 0) {  // uncapped: start from what the device holds at once
        int resident = 0;
        FW2V_CK(x->launch_one(BatchView{}, false, nullptr, nullptr, &resident));
        cur = resident > 0 ? resident : 4096;
    }
    x->inflight_total = std::max<int64_t>(1, cur / 2);
}

} // namespace

extern "C" {

int fw2v_train_corpus(fw2v_ctx* x, const uint64_t* offsets, uint64_t n_sentences, const int32_t* ids,
                      fw2v_observer_fn observer, void* observer_user, fw2v_epoch_fn on_epoch,
                      void* epoch_user, fw2v_report* report) {
    return guarded([&] {
        FW2V_CK(cudaSetDevice(x->cfg.device));
        const fw2v_config& cfg = x->cfg;
        const CorpusView corpus{offsets, ids, n_sentences};
        const std::vector<ChunkSpan> spans = chunk_spans(n_sentences, x->chunks());
        RunShared sh;
        sh.schedule_total =
            cfg.epochs > 0 ? std::max<uint64_t>(1, static_cast<uint64_t>(cfg.epochs) * expected_epoch_words(*x)) : 1;
        sh.observer = observer;
        sh.observer_user = observer_user;
        fw2v_report rep{};
        rep.vocab_size = static_cast<uint64_t>(x->vocab);
        uint64_t bw = 0, bn = 0;
        const double run_start = wall_seconds();
        const bool guard = cfg.divergence_guard != 0 && !x->deterministic;
        for (int epoch = 0; epoch < cfg.epochs; ++epoch) {
            const double t0 = wall_seconds();
            PassOut o;
            for (int attempt = 0;; ++attempt) {
                const uint64_t words0 = x->words_trained;
                if (guard) guard_save(x);
                // (The previous pass may already have started this one: its first
                // sub-batches reserved their words.)
                if (!sh.prefetched.exchange(false)) sh.reserved.store(x->words_trained);
                o = PassOut{};
                run_pass(x, corpus, spans, epoch, sh, &o, epoch + 1 < cfg.epochs ? &spans : nullptr);
                if (!guard || guard_finite(x)) break;
                for (Lane& ln : x->lanes) ln.stash.ready = false;  // made for the next epoch
                sh.prefetched.store(false);
                // Hogwild diverged (too many sentences in flight for this
                // vocabulary and learning rate): restore the epoch's start, halve
                // the in-flight budget and train the epoch again (same batches).
                if (attempt == kGuardRetries)
                    fail(FW2V_ERR_DIVERGED, "Hogwild training diverged (non-finite or |x| >= 1e6 model) at every in-flight budget tried; "
                                            "set max_inflight lower or train with deterministic = 1");
                guard_restore(x);
                x->words_trained = words0;
                guard_halve_inflight(x);
                ++rep.guard_retries;
                std::fprintf(stderr, "[fw2v] epoch %d: diverged (non-finite or |x| >= 1e6), restored; in-flight budget -> %lld sentences\n",
                             epoch, static_cast<long long>(x->inflight_total));
            }
            const double secs = wall_seconds() - t0;
            accumulate(rep, o);
            bw += o.batch_words;
            bn += o.batch_nanos;
            rep.n_epochs = epoch + 1;
            if (on_epoch) {
                const uint64_t ew = o.traffic.words;
                fw2v_epoch_stats st{epoch, ew, secs, secs > 0 ? static_cast<double>(ew) / secs : 0.0};
                on_epoch(epoch_user, &st);
            }
        }
        rep.wall_seconds = wall_seconds() - run_start;
        rep.batching_words_per_sec = bn > 0 ? static_cast<double>(bw) * 1e9 / static_cast<double>(bn) : 0.0;
        if (report) *report = rep;
    });
}

} // extern "C"

namespace {

// Replica average over `n` contexts (see fw2v_average). local_words[i] (may be
// null) are the words each member trained since the last exchange; *global
// (may be null) receives their sum over every member of every process.
void average_impl(fw2v_ctx* const* ctxs, int n, const uint64_t* local_words, uint64_t* global) {
    if (n < 1) fail(FW2V_ERR_BAD_ARGUMENT, "need at least one context");
    if (n > kMaxPeers) fail(FW2V_ERR_UNSUPPORTED, "at most 16 contexts per process");
    fw2v_ctx* x0 = ctxs[0];
    std::vector<int> devices;
    bool distinct = true;
    uint64_t local_sum = 0;
    for (int i = 0; i < n; ++i) {
        fw2v_ctx* x = ctxs[i];
        if (x->vocab != x0->vocab || x->stride != x0->stride || x->cfg.dim != x0->cfg.dim)
            fail(FW2V_ERR_BAD_ARGUMENT, "replicas differ in vocabulary or row stride");
        if (std::find(devices.begin(), devices.end(), x->cfg.device) != devices.end()) distinct = false;
        devices.push_back(x->cfg.device);
        if (local_words) local_sum += local_words[i];
        FW2V_CK(cudaSetDevice(x->cfg.device));
        FW2V_CK(cudaDeviceSynchronize());  // training must be quiesced; cheap when it is
    }
    const size_t count = static_cast<size_t>(x0->vocab) * static_cast<size_t>(x0->stride);
    const bool cross = x0->clique != nullptr && x0->clique_members.size() == 1 && n == 1;
    static const bool force_peer = [] {
        const char* e = std::getenv("FW2V_AVERAGE");
        return e != nullptr && std::strcmp(e, "peer") == 0;
    }();
    std::string err;
    if (cross || (n > 1 && distinct && !force_peer && nccl_available(nullptr))) {
        if (!cross && (x0->clique == nullptr || x0->clique_members != std::vector<fw2v_ctx*>(ctxs, ctxs + n))) {
            auto c = nccl_clique_local(devices, &err);
            if (!c) fail(FW2V_ERR_CUDA, err);
            for (int i = 0; i < n; ++i) {
                ctxs[i]->clique = c;
                ctxs[i]->clique_members.assign(ctxs, ctxs + n);
            }
        }
        std::vector<std::vector<float*>> bufs;
        std::vector<unsigned long long*> words;
        for (int i = 0; i < n; ++i) {
            fw2v_ctx* x = ctxs[i];
            bufs.push_back({x->syn0, x->syn1});
            if (cross && global != nullptr) {
                FW2V_CK(cudaSetDevice(x->cfg.device));
                if (x->d_words == nullptr) FW2V_CK(cudaMalloc(&x->d_words, sizeof(unsigned long long)));
                const unsigned long long w = local_sum;
                FW2V_CK(cudaMemcpy(x->d_words, &w, sizeof(w), cudaMemcpyHostToDevice));
                words.push_back(x->d_words);
            }
        }
        if (!nccl_allreduce(*x0->clique, bufs, count, words, false, &err)) fail(FW2V_ERR_CUDA, err);
        if (global != nullptr) {
            if (cross) {
                unsigned long long w = 0;
                FW2V_CK(cudaSetDevice(x0->cfg.device));
                FW2V_CK(cudaMemcpy(&w, x0->d_words, sizeof(w), cudaMemcpyDeviceToHost));
                *global = w;
            } else {
                *global = local_sum;
            }
        }
        return;
    }
    if (global != nullptr) *global = local_sum;
    if (n == 1) return;
    // Peer-memory kernel: member g averages its slice of every replica.
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            if (devices[i] == devices[j]) continue;
            int can = 0;
            FW2V_CK(cudaDeviceCanAccessPeer(&can, devices[i], devices[j]));
            if (!can) fail(FW2V_ERR_UNSUPPORTED, "no P2P access between the replicas' devices and no NCCL");
            FW2V_CK(cudaSetDevice(devices[i]));
            cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else FW2V_CK(e);
        }
    for (int m = 0; m < 2; ++m) {
        PeerSet ps{};
        ps.n = n;
        for (int i = 0; i < n; ++i) ps.ptr[i] = m == 0 ? ctxs[i]->syn0 : ctxs[i]->syn1;
        const size_t per = ((count + n - 1) / n + 3) & ~size_t(3);
        for (int g = 0; g < n; ++g) {
            FW2V_CK(cudaSetDevice(devices[g]));
            const size_t b = std::min(count, per * g), e = std::min(count, b + per);
            FW2V_CK(launch_average_slice(ps, b, e, nullptr));
        }
    }
    for (int g = 0; g < n; ++g) {
        FW2V_CK(cudaSetDevice(devices[g]));
        FW2V_CK(cudaDeviceSynchronize());
    }
}

// Allocates the merge buffers and makes the base the current model.
void merge_begin(fw2v_ctx* x, int rule) {
    if (rule == kMergeMean) return;
    FW2V_CK(cudaSetDevice(x->cfg.device));
    const size_t n = x->model_floats();
    if (x->merge_base == nullptr) FW2V_CK(cudaMalloc(&x->merge_base, 2 * n * sizeof(float)));
    if (rule == kMergeTouched && x->merge_cnt == nullptr) FW2V_CK(cudaMalloc(&x->merge_cnt, 2 * n * sizeof(float)));
    FW2V_CK(cudaMemcpy(x->merge_base, x->syn0, n * sizeof(float), cudaMemcpyDeviceToDevice));
    FW2V_CK(cudaMemcpy(x->merge_base + n, x->syn1, n * sizeof(float), cudaMemcpyDeviceToDevice));
}

// One merge of the replicas of an n_total-replica job, of which ctxs[0..n) are
// here (see fw2v_config.replica_merge). Returns the global word count.
uint64_t merge_impl(fw2v_ctx* const* ctxs, int n, int n_total, int rule, const uint64_t* local_words,
                    fw2v_exchange_fn exchange, void* user) {
    uint64_t local_sum = 0;
    for (int i = 0; i < n; ++i) local_sum += local_words[i];
    fw2v_ctx* x0 = ctxs[0];
    const size_t count = x0->model_floats();
    const bool cross = n_total > n;
    if (!cross) {
        if (n == 1) return local_sum;
        std::vector<int> devices;
        bool distinct = true;
        for (int i = 0; i < n; ++i) {
            if (std::find(devices.begin(), devices.end(), ctxs[i]->cfg.device) != devices.end()) distinct = false;
            devices.push_back(ctxs[i]->cfg.device);
        }
        static const bool force_peer = [] {
            const char* e = std::getenv("FW2V_AVERAGE");
            return e != nullptr && std::strcmp(e, "peer") == 0;
        }();
        if (rule == kMergeMean || !distinct || force_peer || !nccl_available(nullptr)) {
            // Mean: fw2v_average's path; others: one fused peer-memory kernel per
            // member slice, the base shared from member 0.
            if (rule == kMergeMean) {
                average_impl(ctxs, n, nullptr, nullptr);
                return local_sum;
            }
            average_impl(ctxs, 1, nullptr, nullptr);  // quiesce + shape checks on member 0
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) {
                    if (devices[i] == devices[j]) continue;
                    FW2V_CK(cudaSetDevice(devices[i]));
                    cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else FW2V_CK(e);
                }
            for (int i = 0; i < n; ++i) {
                FW2V_CK(cudaSetDevice(devices[i]));
                FW2V_CK(cudaDeviceSynchronize());
            }
            for (int m = 0; m < 2; ++m) {
                PeerSet ps{};
                ps.n = n;
                for (int i = 0; i < n; ++i) ps.ptr[i] = m == 0 ? ctxs[i]->syn0 : ctxs[i]->syn1;
                float* base = x0->merge_base + m * count;
                const size_t per = (count + n - 1) / n;
                for (int g = 0; g < n; ++g) {
                    FW2V_CK(cudaSetDevice(devices[g]));
                    const size_t b = std::min(count, per * g), e = std::min(count, b + per);
                    FW2V_CK(launch_merge_slice(ps, base, rule, b, e, nullptr));
                }
            }
            for (int g = 0; g < n; ++g) {
                FW2V_CK(cudaSetDevice(devices[g]));
                FW2V_CK(cudaDeviceSynchronize());
            }
            return local_sum;
        }
    } else if (n != 1) {
        fail(FW2V_ERR_UNSUPPORTED, "a multi-process job holds one context per process");
    }
    // Split merge: prep -> SUM all-reduce (NCCL clique or the exchange) -> finish.
    std::string err;
    if (!cross && (x0->clique == nullptr || x0->clique_members != std::vector<fw2v_ctx*>(ctxs, ctxs + n))) {
        std::vector<int> devices;
        for (int i = 0; i < n; ++i) devices.push_back(ctxs[i]->cfg.device);
        auto c = nccl_clique_local(devices, &err);
        if (!c) fail(FW2V_ERR_CUDA, err);
        for (int i = 0; i < n; ++i) {
            ctxs[i]->clique = c;
            ctxs[i]->clique_members.assign(ctxs, ctxs + n);
        }
    }
    std::vector<std::vector<float*>> bufs(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        fw2v_ctx* x = ctxs[i];
        FW2V_CK(cudaSetDevice(x->cfg.device));
        FW2V_CK(cudaDeviceSynchronize());
        float* cnt = rule == kMergeTouched ? x->merge_cnt : nullptr;
        FW2V_CK(launch_merge_prep(x->syn0, x->merge_base, cnt, rule, count, nullptr));
        FW2V_CK(launch_merge_prep(x->syn1, x->merge_base + count, cnt ? cnt + count : nullptr, rule, count, nullptr));
        FW2V_CK(cudaDeviceSynchronize());
        bufs[static_cast<size_t>(i)] = {x->syn0, x->syn1};
        if (cnt) {
            bufs[static_cast<size_t>(i)].push_back(cnt);
            bufs[static_cast<size_t>(i)].push_back(cnt + count);
        }
    }
    uint64_t global = local_sum;
    if (cross && exchange != nullptr) {
        const std::vector<float*>& b = bufs[0];
        std::vector<uint64_t> counts(b.size(), count);
        const int rc = exchange(user, b.data(), counts.data(), static_cast<int32_t>(b.size()), local_sum, &global);
        if (rc != FW2V_OK) fail(rc, "exchange callback failed");
        FW2V_CK(cudaSetDevice(x0->cfg.device));
        FW2V_CK(cudaDeviceSynchronize());
    } else {
        if (x0->clique == nullptr) fail(FW2V_ERR_BAD_ARGUMENT, "no communicator for a multi-process merge");
        std::vector<unsigned long long*> words;
        if (cross) {
            FW2V_CK(cudaSetDevice(x0->cfg.device));
            if (x0->d_words == nullptr) FW2V_CK(cudaMalloc(&x0->d_words, sizeof(unsigned long long)));
            const unsigned long long w = local_sum;
            FW2V_CK(cudaMemcpy(x0->d_words, &w, sizeof(w), cudaMemcpyHostToDevice));
            words.push_back(x0->d_words);
        }
        if (!nccl_allreduce(*x0->clique, bufs, count, words, true, &err)) fail(FW2V_ERR_CUDA, err);
        if (cross) {
            unsigned long long w = 0;
            FW2V_CK(cudaSetDevice(x0->cfg.device));
            FW2V_CK(cudaMemcpy(&w, x0->d_words, sizeof(w), cudaMemcpyDeviceToHost));
            global = w;
        }
    }
    const float inv = 1.0f / static_cast<float>(n_total);
    for (int i = 0; i < n; ++i) {
        fw2v_ctx* x = ctxs[i];
        FW2V_CK(cudaSetDevice(x->cfg.device));
        float* cnt = rule == kMergeTouched ? x->merge_cnt : nullptr;
        FW2V_CK(launch_merge_finish(x->syn0, x->merge_base, cnt, rule, inv, count, nullptr));
        FW2V_CK(launch_merge_finish(x->syn1, x->merge_base ? x->merge_base + count : nullptr, cnt ? cnt + count : nullptr,
                                    rule, inv, count, nullptr));
        FW2V_CK(cudaDeviceSynchronize());
    }
    return global;
}

// The job's chunk partition for data-parallel runs: the reference's `workers`
// chunks (trainer.cpp:431-434) rounded up to a multiple of n_shards * rounds,
// so every shard is a contiguous range of whole chunks and every round of a
// shard the same number of them.
struct DpPlan {
    int total_chunks = 1, per_shard = 1, per_round = 1, rounds = 1;
};

DpPlan dp_plan(const fw2v_ctx& x, const CorpusView& c, int n_shards, uint64_t average_words) {
    DpPlan d;
    // Estimated trained words per shard and epoch (expected_epoch_words scaled
    // by the shard's share of the tokens).
    const double shard_words = static_cast<double>(expected_epoch_words(x)) / n_shards;
    d.rounds = average_words > 0
                   ? static_cast<int>(std::max(1.0, std::floor(shard_words / static_cast<double>(average_words) + 0.5)))
                   : 1;
    const int unit = n_shards * d.rounds;
    d.total_chunks = ((std::max(x.chunks(), n_shards) + unit - 1) / unit) * unit;
    d.per_shard = d.total_chunks / n_shards;
    d.per_round = d.per_shard / d.rounds;
    (void)c;
    return d;
}

std::vector<ChunkSpan> round_spans(const std::vector<ChunkSpan>& all, const DpPlan& d, int shard, int round) {
    const int b = shard * d.per_shard + round * d.per_round;
    return std::vector<ChunkSpan>(all.begin() + b, all.begin() + b + d.per_round);
}

} // namespace

extern "C" {

int fw2v_average(fw2v_ctx* const* ctxs, int32_t n) {
    return guarded([&] { average_impl(ctxs, n, nullptr, nullptr); });
}

int fw2v_merge_begin(fw2v_ctx* const* ctxs, int32_t n) {
    return guarded([&] {
        for (int i = 0; i < n; ++i) merge_begin(ctxs[i], ctxs[0]->cfg.replica_merge);
    });
}

int fw2v_merge_replicas(fw2v_ctx* const* ctxs, int32_t n, int32_t n_shards, const uint64_t* local_words,
                        fw2v_exchange_fn exchange, void* exchange_user, uint64_t* global_words) {
    return guarded([&] {
        if (n < 1 || n_shards < n) fail(FW2V_ERR_BAD_ARGUMENT, "need 1 <= n <= n_shards");
        const uint64_t g = merge_impl(ctxs, n, n_shards, ctxs[0]->cfg.replica_merge, local_words, exchange, exchange_user);
        if (global_words) *global_words = g;
    });
}

int fw2v_nccl_unique_id(uint8_t out[128]) {
    return guarded([&] {
        std::string err;
        if (!nccl_unique_id(out, &err)) fail(FW2V_ERR_UNSUPPORTED, err);
    });
}

int fw2v_comm_init_rank(fw2v_ctx* x, const uint8_t id[128], int32_t world, int32_t rank) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world) fail(FW2V_ERR_BAD_ARGUMENT, "bad rank / world");
        std::string err;
        auto c = nccl_clique_rank(x->cfg.device, id, world, rank, &err);
        if (!c) fail(FW2V_ERR_CUDA, err);
        x->clique = c;
        x->clique_members = {x};
    });
}

int fw2v_train_corpus_multi(fw2v_ctx* const* ctxs, int32_t n, int32_t shard0, int32_t n_shards,
                            const uint64_t* offsets, uint64_t n_sentences, const int32_t* ids,
                            uint64_t average_words, fw2v_exchange_fn exchange, void* exchange_user,
                            fw2v_observer_fn observer, void* observer_user, fw2v_epoch_fn on_epoch, void* epoch_user,
                            fw2v_report* report) {
    return guarded([&] {
        if (n < 1 || n_shards < n || shard0 < 0 || shard0 + n > n_shards)
            fail(FW2V_ERR_BAD_ARGUMENT, "shards shard0 .. shard0+n-1 must lie in 0 .. n_shards-1");
        fw2v_ctx* x0 = ctxs[0];
        for (int i = 0; i < n; ++i) {
            if (ctxs[i]->deterministic)
                fail(FW2V_ERR_UNSUPPORTED, "deterministic mode is single-GPU (serial reference order)");
            if (ctxs[i]->vocab != x0->vocab || ctxs[i]->cfg.epochs != x0->cfg.epochs)
                fail(FW2V_ERR_BAD_ARGUMENT, "replicas differ in vocabulary or epochs");
        }
        const bool cross = n_shards > n;
        if (cross && exchange == nullptr && (n != 1 || x0->clique == nullptr || x0->clique_members.size() != 1))
            fail(FW2V_ERR_BAD_ARGUMENT, "other processes hold shards: pass an exchange callback or fw2v_comm_init_rank");
        const fw2v_config& cfg = x0->cfg;
        const CorpusView corpus{offsets, ids, n_sentences};
        const DpPlan d = dp_plan(*x0, corpus, n_shards, average_words);
        const std::vector<ChunkSpan> all = chunk_spans(n_sentences, d.total_chunks);
        RunShared sh;
        sh.schedule_total =
            cfg.epochs > 0 ? std::max<uint64_t>(1, static_cast<uint64_t>(cfg.epochs) * expected_epoch_words(*x0)) : 1;
        sh.observer = observer;
        sh.observer_user = observer_user;
        uint64_t global_words = 0;
        for (int i = 0; i < n; ++i) global_words = std::max(global_words, ctxs[i]->words_trained);
        sh.scale = static_cast<uint64_t>(n_shards / n);
        const int rule = cfg.replica_merge;
        for (int i = 0; i < n; ++i) merge_begin(ctxs[i], rule);
        fw2v_report rep{};
        rep.vocab_size = static_cast<uint64_t>(x0->vocab);
        uint64_t bw = 0, bn = 0;
        const double run_start = wall_seconds();
        for (int epoch = 0; epoch < cfg.epochs; ++epoch) {
            const double t0 = wall_seconds();
            uint64_t epoch_words = 0;
            for (int r = 0; r < d.rounds; ++r) {
                sh.origin = global_words;
                sh.reserved.store(global_words);
                std::vector<PassOut> outs(static_cast<size_t>(n));
                std::vector<std::string> errs(static_cast<size_t>(n));
                std::vector<int> codes(static_cast<size_t>(n), FW2V_OK);
                std::vector<std::thread> th;
                for (int i = 0; i < n; ++i)
                    th.emplace_back([&, i] {
                        try {
                            run_pass(ctxs[i], corpus, round_spans(all, d, shard0 + i, r), epoch, sh,
                                     &outs[static_cast<size_t>(i)]);
                        } catch (const Failure& f) {
                            codes[static_cast<size_t>(i)] = f.code;
                            errs[static_cast<size_t>(i)] = f.msg;
                        }
                    });
                for (auto& t : th) t.join();
                for (int i = 0; i < n; ++i)
                    if (codes[static_cast<size_t>(i)] != FW2V_OK) fail(codes[static_cast<size_t>(i)], errs[static_cast<size_t>(i)]);
                std::vector<uint64_t> lw(static_cast<size_t>(n));
                double ks = 0.0;
                for (int i = 0; i < n; ++i) {
                    const PassOut& o = outs[static_cast<size_t>(i)];
                    lw[static_cast<size_t>(i)] = o.traffic.words;
                    accumulate(rep, o);
                    rep.kernel_seconds -= o.kernel_seconds;  // max over GPUs, added below
                    ks = std::max(ks, o.kernel_seconds);
                    bw += o.batch_words;
                    bn += o.batch_nanos;
                    epoch_words += o.traffic.words;
                }
                rep.kernel_seconds += ks;
                // Merge: replicas <- one model from every shard's round (replica_merge); the
                // global word count is exact again (lr_at's position, trainer.cpp:479-487).
                const uint64_t g = merge_impl(ctxs, n, n_shards, rule, lw.data(), exchange, exchange_user);
                global_words += g;
            }
            for (int i = 0; i < n; ++i) ctxs[i]->words_trained = global_words;
            rep.n_epochs = epoch + 1;
            if (on_epoch) {
                const double secs = wall_seconds() - t0;
                fw2v_epoch_stats st{epoch, epoch_words, secs, secs > 0 ? static_cast<double>(epoch_words) / secs : 0.0};
                on_epoch(epoch_user, &st);
            }
        }
        rep.wall_seconds = wall_seconds() - run_start;
        rep.batching_words_per_sec = bn > 0 ? static_cast<double>(bw) * 1e9 / static_cast<double>(bn) : 0.0;
        if (report) *report = rep;
    });
}

int fw2v_plan_epoch(fw2v_ctx* x, const uint64_t* offsets, uint64_t n_sentences, const int32_t* ids,
                    int32_t epoch, fw2v_plan** out) {
    const int nc = x->chunks();
    return fw2v_plan_chunks(x, offsets, n_sentences, ids, epoch, nc, 0, nc, x->words_trained, 1, out);
}

int fw2v_plan_chunks(fw2v_ctx* x, const uint64_t* offsets, uint64_t n_sentences, const int32_t* ids, int32_t epoch,
                     int32_t n_chunks, int32_t chunk_begin, int32_t chunk_end, uint64_t words_base,
                     int32_t words_scale, fw2v_plan** out) {
    *out = nullptr;
    return guarded([&] {
        if (n_chunks < 1 || chunk_begin < 0 || chunk_end > n_chunks || chunk_begin > chunk_end || words_scale < 1)
            fail(FW2V_ERR_BAD_ARGUMENT, "chunk range must lie in 0 .. n_chunks, words_scale >= 1");
        FW2V_CK(cudaSetDevice(x->cfg.device));
        const fw2v_config& cfg = x->cfg;
        const CorpusView corpus{offsets, ids, n_sentences};
        const int P = x->producers();  // streams the plan's launches are spread over
        const std::vector<ChunkSpan> all = chunk_spans(n_sentences, n_chunks);
        const std::vector<ChunkSpan> spans(all.begin() + chunk_begin, all.begin() + chunk_end);
        const int NC = static_cast<int>(spans.size());
        const uint64_t schedule_total =
            cfg.epochs > 0 ? std::max<uint64_t>(1, static_cast<uint64_t>(cfg.epochs) * expected_epoch_words(*x)) : 1;
        const Sampler sp = x->sampler();
        const int n_neg = cfg.negatives;
        struct HostBatch {
            std::vector<int32_t> ids, negs;
            std::vector<uint32_t> off;
            std::vector<float> alpha;
        };
        std::vector<std::vector<HostBatch>> host(static_cast<size_t>(NC));
        std::atomic<uint64_t> reserved{words_base};
        auto position = [&](uint64_t w) { return words_base + (w - words_base) * static_cast<uint64_t>(words_scale); };
        std::vector<std::thread> threads;
        std::atomic<int> next_chunk{0};
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        for (unsigned th = 0; th < std::min<unsigned>(hw, static_cast<unsigned>(NC)); ++th) {
            threads.emplace_back([&] {
              for (int si = next_chunk.fetch_add(1); si < NC; si = next_chunk.fetch_add(1)) {
                const uint64_t p = spans[static_cast<size_t>(si)].p;
                const uint64_t begin = spans[static_cast<size_t>(si)].begin;
                const uint64_t end = spans[static_cast<size_t>(si)].end;
                uint64_t cap_w, cap_s;
                capacity_for(corpus, begin, std::max(begin, end), cfg.batch_sentences, &cap_w, &cap_s);
                std::vector<int32_t> bi(cap_w), bn(cap_w * std::max(n_neg, 1));
                std::vector<uint32_t> bo(cap_s + 1);
                uint64_t cursor = begin;
                for (uint64_t k = 0; cursor < end; ++k) {
                    Rng rng = Rng::derive(cfg.seed, static_cast<uint64_t>(epoch), p, k);
                    uint64_t words = 0;
                    const uint64_t kept = assemble(corpus, cursor, end, cfg.batch_sentences, sp, rng,
                                                   BatchOut{bi.data(), bo.data(), bn.data(), cap_w, cap_s}, &words);
                    if (kept == 0) continue;
                    HostBatch hb;
                    hb.ids.assign(bi.begin(), bi.begin() + static_cast<ptrdiff_t>(words));
                    hb.negs.assign(bn.begin(), bn.begin() + static_cast<ptrdiff_t>(words * n_neg));
                    hb.negs.resize(hb.negs.size() + kNegPadBytes / 4, 0);  // kernels read a window's row whole
                    hb.off.assign(bo.begin(), bo.begin() + static_cast<ptrdiff_t>(kept + 1));
                    const uint64_t base = reserved.fetch_add(words);
                    hb.alpha.resize(kept);
                    for (uint64_t q = 0; q < kept; ++q) hb.alpha[q] = lr_at(position(base + bo[q]), schedule_total, cfg.alpha0);
                    host[static_cast<size_t>(si)].push_back(std::move(hb));
                }
              }
            });
        }
        for (auto& t : threads) t.join();
        auto plan = std::make_unique<fw2v_plan>();
        plan->device = cfg.device;
        auto a16 = [](size_t b) { return (b + 255) & ~size_t(255); };
        size_t bytes = 0;
        for (auto& lane : host)
            for (auto& hb : lane)
                bytes += a16(4 * hb.ids.size()) + a16(4 * std::max<size_t>(hb.negs.size(), 1)) + a16(4 * hb.off.size()) + a16(4 * hb.alpha.size());
        FW2V_CK(cudaMalloc(&plan->d_mem, std::max<size_t>(bytes, 256)));
        plan->bytes = bytes;
        char* base = static_cast<char*>(plan->d_mem);
        plan->lanes.resize(static_cast<size_t>(P));
        for (int p = 0; p < NC; ++p) {
            for (auto& hb : host[static_cast<size_t>(p)]) {
                auto put = [&](const void* src, size_t n) {
                    char* dst = base;
                    if (n) FW2V_CK(cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice));
                    base += a16(std::max<size_t>(n, 1));
                    return dst;
                };
                fw2v_plan::Batch b;
                b.view.ids = reinterpret_cast<const int32_t*>(put(hb.ids.data(), 4 * hb.ids.size()));
                b.view.negs = reinterpret_cast<const int32_t*>(put(hb.negs.data(), 4 * hb.negs.size()));
                b.view.offsets = reinterpret_cast<const uint32_t*>(put(hb.off.data(), 4 * hb.off.size()));
                b.view.alpha = reinterpret_cast<const float*>(put(hb.alpha.data(), 4 * hb.alpha.size()));
                b.view.n_sentences = static_cast<int32_t>(hb.alpha.size());
                plan->lanes[static_cast<size_t>(p % P)].push_back(b);
                plan->words += hb.ids.size();
                plan->sentences += hb.alpha.size();
                plan->batches += 1;
            }
            host[static_cast<size_t>(p)].clear();
        }
        *out = plan.release();
    });
}

int fw2v_plan_info(const fw2v_plan* plan, uint64_t* words, uint64_t* sentences, uint64_t* batches,
                   uint64_t* device_bytes) {
    if (words) *words = plan->words;
    if (sentences) *sentences = plan->sentences;
    if (batches) *batches = plan->batches;
    if (device_bytes) *device_bytes = plan->bytes;
    return FW2V_OK;
}

int fw2v_plan_run(fw2v_ctx* x, fw2v_plan* plan, double* seconds, fw2v_counters* counters) {
    return guarded([&] {
        FW2V_CK(cudaSetDevice(x->cfg.device));
        const int P = static_cast<int>(plan->lanes.size());
        x->ensure_lanes(P, 1, 1);
        cudaEvent_t start, fork;
        std::vector<cudaEvent_t> ends(static_cast<size_t>(P));
        FW2V_CK(cudaEventCreate(&start));
        FW2V_CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        for (auto& e : ends) FW2V_CK(cudaEventCreate(&e));
        cudaStream_t s0 = x->lanes[0].stream;
        for (int p = 0; p < P; ++p) FW2V_CK(cudaMemsetAsync(x->lanes[static_cast<size_t>(p)].d_ctr, 0, sizeof(DevCounters), s0));
        FW2V_CK(cudaEventRecord(start, s0));
        const bool hot = !x->deterministic && x->hot_k > 0;
        if (hot) x->hot_begin(s0);
        FW2V_CK(cudaEventRecord(fork, s0));
        const int KS = x->kernel_streams();
        for (int p = 0; p < P; ++p) {
            if (p > 0) FW2V_CK(cudaStreamWaitEvent(x->lanes[static_cast<size_t>(p)].stream, fork, 0));
            if (KS > 1) FW2V_CK(cudaStreamWaitEvent(x->lanes[static_cast<size_t>(p)].stream2, fork, 0));
        }
        // Interleave launches across lanes so each stream always has queued work.
        size_t maxb = 0;
        for (auto& l : plan->lanes) maxb = std::max(maxb, l.size());
        for (size_t k = 0; k < maxb; ++k)
            for (int p = 0; p < P; ++p)
                if (k < plan->lanes[static_cast<size_t>(p)].size())
                    FW2V_CK(x->launch(plan->lanes[static_cast<size_t>(p)][k].view, x->deterministic,
                                      x->lanes[static_cast<size_t>(p)].d_ctr,
                                      (k & 1) && KS > 1 ? x->lanes[static_cast<size_t>(p)].stream2 : x->lanes[static_cast<size_t>(p)].stream,
                                      KS * P));
        for (int p = 0; p < P; ++p) {
            if (KS > 1) {  // join the lane's second kernel stream
                FW2V_CK(cudaEventRecord(ends[static_cast<size_t>(p)], x->lanes[static_cast<size_t>(p)].stream2));
                FW2V_CK(cudaStreamWaitEvent(x->lanes[static_cast<size_t>(p)].stream, ends[static_cast<size_t>(p)], 0));
            }
            FW2V_CK(cudaEventRecord(ends[static_cast<size_t>(p)], x->lanes[static_cast<size_t>(p)].stream));
        }
        if (hot) {
            // Join every lane on s0, fold the replicas back; the pass ends there.
            for (int p = 1; p < P; ++p) FW2V_CK(cudaStreamWaitEvent(s0, ends[static_cast<size_t>(p)], 0));
            x->hot_end(s0);
            FW2V_CK(cudaEventRecord(ends[0], s0));
        }
        float ms_max = 0.0f;
        for (int p = 0; p < P; ++p) {
            FW2V_CK(cudaEventSynchronize(ends[static_cast<size_t>(p)]));
            float ms = 0.0f;
            FW2V_CK(cudaEventElapsedTime(&ms, start, ends[static_cast<size_t>(p)]));
            ms_max = std::max(ms_max, ms);
        }
        if (seconds) *seconds = 1e-3 * ms_max;
        fw2v_counters c{};
        for (int p = 0; p < P; ++p) {
            DevCounters h{};
            FW2V_CK(cudaMemcpy(&h, x->lanes[static_cast<size_t>(p)].d_ctr, sizeof(h), cudaMemcpyDeviceToHost));
            c.context_reads += h.context_reads;
            c.context_writes += h.context_writes;
            c.sample_reads += h.sample_reads;
            c.sample_writes += h.sample_writes;
            c.ring_hits += h.ring_hits;
            c.words += h.words;
            c.sentences += h.sentences;
        }
        if (counters) *counters = c;
        x->words_trained += c.words;
        cudaEventDestroy(start);
        cudaEventDestroy(fork);
        for (auto& e : ends) cudaEventDestroy(e);
    });
}

void fw2v_plan_destroy(fw2v_plan* plan) { delete plan; }

int fw2v_keep_probs(const uint64_t* counts, int32_t vocab_size, double threshold, double* out) {
    return keep_probs(counts, vocab_size, threshold, out) ? 1 : 0;
}

int fw2v_table_build(const uint64_t* counts, int32_t vocab_size, double power, uint64_t size, int32_t* out_slots) {
    return guarded([&] { build_table(counts, vocab_size, power, size, out_slots); });
}

int64_t fw2v_assemble_batch(const uint64_t* counts, int32_t vocab_size, const uint64_t* offsets,
                            uint64_t n_sentences, const int32_t* ids, uint64_t* cursor, uint64_t max_sentences,
                            int32_t negatives, double power, uint64_t table_size, double threshold,
                            uint64_t seed, uint64_t a, uint64_t b, uint64_t c, int32_t* out_ids,
                            uint64_t* out_offsets, int32_t* out_negs) {
    int64_t kept = 0;
    int rc = guarded([&] {
        if (max_sentences < 1) fail(FW2V_ERR_BAD_ARGUMENT, "batch size must be >= 1");
        if (negatives < 0) fail(FW2V_ERR_BAD_ARGUMENT, "negatives must be >= 0");
        HugeArray<int32_t> slots;
        slots.resize(table_size);
        build_table(counts, vocab_size, power, table_size, slots.data());
        std::vector<double> keep(static_cast<size_t>(vocab_size));
        const bool on = keep_probs(counts, vocab_size, threshold, keep.data());
        Sampler sp;
        sp.keep = on ? keep.data() : nullptr;
        sp.slots = slots.data();
        sp.table_size = table_size;
        sp.mod = FastMod(table_size);
        sp.n_neg = negatives;
        const uint64_t total = offsets[n_sentences] - offsets[0];
        std::vector<uint32_t> off(n_sentences + 1);
        Rng rng = Rng::derive(seed, a, b, c);
        uint64_t words = 0;
        uint64_t cur = *cursor;
        kept = static_cast<int64_t>(assemble(CorpusView{offsets, ids, n_sentences}, cur, n_sentences, max_sentences, sp, rng,
                                             BatchOut{out_ids, off.data(), out_negs, total + 1, n_sentences + 1}, &words));
        *cursor = cur;
        for (int64_t q = 0; q <= kept; ++q) out_offsets[q] = off[static_cast<size_t>(q)];
    });
    return rc == FW2V_OK ? kept : -rc;
}

int fw2v_alias_draws(const uint64_t* counts, int32_t vocab_size, double power, uint64_t seed, uint64_t count,
                     int32_t* out) {
    return guarded([&] {
        if (vocab_size < 1) fail(FW2V_ERR_EMPTY_VOCAB, "empty vocabulary");
        AliasTable at;
        at.build(counts, vocab_size, power);
        Rng r = Rng::derive(seed, 0);
        if (have_avx512()) {
            alias_draws_avx512(r.state, at.e.data(), at.n, out, count);
        } else {
            for (uint64_t x = 0; x < count; ++x) out[x] = at.sample(r.next());
        }
    });
}

float fw2v_lr_at(uint64_t words_trained, uint64_t total, float alpha0) {
    if (total == 0) {
        g_error = "total_words must be > 0";
        return -1.0f;
    }
    return lr_at(words_trained, total, alpha0);
}

int fw2v_analytic_traffic(uint64_t length, int32_t width, int32_t negatives, int32_t mode, fw2v_counters* out) {
    return guarded([&] {
        if (length < 1) fail(FW2V_ERR_BAD_ARGUMENT, "sentence length must be >= 1");
        if (width < 1) fail(FW2V_ERR_BAD_ARGUMENT, "context width must be >= 1");
        if (negatives < 0) fail(FW2V_ERR_BAD_ARGUMENT, "negatives must be >= 0");
        uint64_t t[5];
        analytic(length, width, negatives, mode, t);
        *out = fw2v_counters{t[0], t[1], t[2], t[3], t[4], length, 1};
    });
}

} // extern "C"

namespace fw2v {
void set_last_error(const std::string& msg) { g_error = msg; }
} // namespace fw2v
