// Embedding output writer at scale: the reference text
// format of save_embeddings (model.cpp:47-74), byte for byte, formatted by all
// host cores. A 555k x 128 model is ~0.7 GB of text; the reference formats it
// on one thread.
//
//   "<|V|> <dim>\n", then per word id: token, then " <value>" per column with
//   std::to_chars(value, chars_format::fixed, 6), then "\n".
//
// Rows are cut into chunks; waves of chunks are formatted in parallel and
// written in order, so memory stays bounded (a wave, not the file).
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "fw2v.h"

namespace {

constexpr int32_t kRowsPerChunk = 1024;

// std::to_chars(v, chars_format::fixed, 6) for |v| < 2^43, from the exact
// binary value: v * 10^6 = m * 10^6 * 2^e with m < 2^24, rounded half to even
// like to_chars; larger magnitudes (and non-finite) use to_chars itself.
inline char* fixed6(char* p, char* end, float v) {
    uint32_t bits;
    std::memcpy(&bits, &v, 4);
    const bool neg = (bits >> 31) != 0;
    const int bexp = static_cast<int>((bits >> 23) & 0xff);
    if (bexp == 0xff || bexp >= 127 + 43) return std::to_chars(p, end, v, std::chars_format::fixed, 6).ptr;
    uint64_t m = bits & 0x7fffff;
    int e;
    if (bexp == 0) {
        e = -149;  // subnormal
    } else {
        m |= 0x800000;
        e = bexp - 150;
    }
    uint64_t q;  // round(|v| * 10^6)
    const uint64_t n = m * 1000000ULL;  // < 2^44
    if (e >= 0) {
        q = n << e;  // |v| < 2^43: fits
    } else {
        const int s = -e;
        if (s >= 64) {
            q = 0;  // n < 2^44 < half
        } else {
            q = n >> s;
            const uint64_t r = n & ((uint64_t{1} << s) - 1), half = uint64_t{1} << (s - 1);
            if (r > half || (r == half && (q & 1))) ++q;
        }
    }
    if (neg) *p++ = '-';
    const uint64_t ip = q / 1000000ULL;
    uint32_t fp = static_cast<uint32_t>(q - ip * 1000000ULL);
    p = std::to_chars(p, end, ip).ptr;
    *p++ = '.';
    for (int i = 5; i >= 0; --i) {
        p[i] = static_cast<char>('0' + fp % 10);
        fp /= 10;
    }
    return p + 6;
}

void format_rows(const float* rows, int32_t begin, int32_t end, int32_t dim, int64_t stride, const char* tokens,
                 const uint64_t* token_offsets, std::string& out) {
    out.clear();
    out.reserve(static_cast<size_t>(end - begin) * (16 + 12 * static_cast<size_t>(dim)));
    char num[64];
    for (int32_t w = begin; w < end; ++w) {
        out.append(tokens + token_offsets[w], tokens + token_offsets[w + 1]);
        const float* row = rows + static_cast<int64_t>(w) * stride;
        for (int32_t k = 0; k < dim; ++k) {
            char* const e = fixed6(num, num + sizeof(num), row[k]);
            out.push_back(' ');
            out.append(num, e);
        }
        out.push_back('\n');
    }
}

}  // namespace

namespace fw2v {

// The body of fw2v_write_embeddings (the C-ABI wrapper in fw2v_host.cpp sets the last-error text).
int write_embeddings(const float* rows, int32_t vocab_size, int32_t dim, int64_t row_stride, const char* tokens,
                     const uint64_t* token_offsets, const char* path, int32_t threads, std::string* err) {
    if (rows == nullptr || tokens == nullptr || token_offsets == nullptr || path == nullptr || vocab_size < 1 ||
        dim < 1 || row_stride < dim) {
        *err = "write_embeddings: null pointer, empty vocabulary, dim < 1 or row_stride < dim";
        return FW2V_ERR_BAD_ARGUMENT;
    }
    std::FILE* f = std::fopen(path, "wb");
    if (!f) {
        *err = std::string("cannot open embedding file for writing: ") + path;  // model.cpp:53
        return FW2V_ERR_IO;
    }
    int T = threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    const int32_t n_chunks = (vocab_size + kRowsPerChunk - 1) / kRowsPerChunk;
    T = std::max(1, std::min(T, n_chunks));
    // T formatter threads take chunks in order from a counter into a ring of
    // slots; this thread writes the slots in chunk order as they complete.
    const int32_t ring = 4 * T;
    std::vector<std::string> buf(static_cast<size_t>(ring));
    std::vector<std::atomic<int32_t>> ready(static_cast<size_t>(ring));  // chunk index held by the slot, -1 none
    for (auto& r : ready) r.store(-1);
    std::atomic<int32_t> next{0}, written{0};
    std::atomic<bool> failed{false};
    auto work = [&] {
        for (int32_t c = next.fetch_add(1); c < n_chunks && !failed.load(); c = next.fetch_add(1)) {
            while (c - written.load(std::memory_order_acquire) >= ring && !failed.load()) std::this_thread::yield();
            const int32_t b = c * kRowsPerChunk, e = std::min(vocab_size, b + kRowsPerChunk);
            std::string& s = buf[static_cast<size_t>(c % ring)];
            format_rows(rows, b, e, dim, row_stride, tokens, token_offsets, s);
            ready[static_cast<size_t>(c % ring)].store(c, std::memory_order_release);
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) pool.emplace_back(work);
    bool ok = std::fprintf(f, "%d %d\n", vocab_size, dim) > 0;
    for (int32_t c = 0; c < n_chunks; ++c) {
        std::atomic<int32_t>& r = ready[static_cast<size_t>(c % ring)];
        while (r.load(std::memory_order_acquire) != c && ok) std::this_thread::yield();
        if (!ok) break;
        const std::string& s = buf[static_cast<size_t>(c % ring)];
        ok = std::fwrite(s.data(), 1, s.size(), f) == s.size();
        r.store(-1, std::memory_order_relaxed);
        written.store(c + 1, std::memory_order_release);
    }
    if (!ok) failed.store(true);
    for (auto& t : pool) t.join();
    if (std::fclose(f) != 0) ok = false;
    if (!ok) *err = std::string("failed writing embedding file: ") + path;
    return ok ? FW2V_OK : FW2V_ERR_IO;
}

}  // namespace fw2v
