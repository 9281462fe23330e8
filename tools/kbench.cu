// K1s microbenchmark: one kernel instantiation on the text8-shaped epoch as a
// single device-resident batch (exact reference batcher from libfw2v.so).
// Build variants with -D flags (see tools/kbench.sh); prints words/s.
#include "../paper_2312_07743_b200/csrc/fw2v_snapshot.cuh"

#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "fw2v.h"

#ifndef KB_LANES
#define KB_LANES 16
#endif
#ifndef KB_VEC
#define KB_VEC 8
#endif
#ifndef KB_RING
#define KB_RING true
#endif
#ifndef KB_LIFE
#define KB_LIFE false
#endif
#ifndef KB_PAD
#define KB_PAD 0
#endif
#ifndef KB_FLAGS
#define KB_FLAGS (fw2v::kFlagRedSamples | fw2v::kFlagDeltaRing | (5 << fw2v::kFlagInvalShift))
#endif

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

int main(int argc, char** argv) {
    const int steps = argc > 1 ? atoi(argv[1]) : 5;
    const int chunks = argc > 2 ? atoi(argv[2]) : 16;  // launches per step on as many streams
    fw2v_corpus* corpus = nullptr;
    if (fw2v_corpus_synth_zipf(71291, 16718845, 1.0, 1000, 5, 0, &corpus)) { printf("synth: %s\n", fw2v_last_error()); return 1; }
    const uint64_t* counts; int32_t V; const uint64_t* offs; uint64_t ns; const int32_t* ids; uint64_t nid;
    fw2v_corpus_view(corpus, &counts, &V, &offs, &ns, &ids, &nid);
    const int N = 5, D = 128, STRIDE = KB_LANES * KB_VEC;
    std::vector<int32_t> bids(nid), bnegs(nid * N + 64, 0);
    std::vector<uint64_t> boff(ns + 1);
    uint64_t cursor = 0;
    int64_t kept = fw2v_assemble_batch(counts, V, offs, ns, ids, &cursor, ns, N, 0.75, 10000000, 1e-4, 1, 0, 0, 0,
                                       bids.data(), boff.data(), bnegs.data());
    if (kept < 0) { printf("assemble: %s\n", fw2v_last_error()); return 1; }
    const uint64_t words = boff[kept];
    std::vector<uint32_t> off32(kept + 1);
    for (int64_t i = 0; i <= kept; ++i) off32[i] = static_cast<uint32_t>(boff[i]);
    std::vector<float> alpha(kept, 0.025f);
    std::vector<float> syn0(static_cast<size_t>(V) * STRIDE, 0.0f);
    uint64_t st = 12345;
    for (int w = 0; w < V; ++w)
        for (int c = 0; c < D; ++c) {
            st = st * 6364136223846793005ULL + 1442695040888963407ULL;
            syn0[static_cast<size_t>(w) * STRIDE + c] = ((st >> 40) * (1.0f / 16777216.0f) - 0.5f) / D;
        }
    float *d0, *d1, *dalpha; int32_t *dids, *dnegs; uint32_t* doff; fw2v::DevCounters* dctr;
    CK(cudaMalloc(&d0, syn0.size() * 4)); CK(cudaMalloc(&d1, syn0.size() * 4));
    CK(cudaMemcpy(d0, syn0.data(), syn0.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(d1, 0, syn0.size() * 4));
    CK(cudaMalloc(&dids, words * 4)); CK(cudaMalloc(&dnegs, (words * N + 64) * 4));
    CK(cudaMalloc(&doff, (kept + 1) * 4)); CK(cudaMalloc(&dalpha, kept * 4)); CK(cudaMalloc(&dctr, sizeof(fw2v::DevCounters)));
    CK(cudaMemcpy(dids, bids.data(), words * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dnegs, bnegs.data(), (words * N + 64) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(doff, off32.data(), (kept + 1) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dalpha, alpha.data(), kept * 4, cudaMemcpyHostToDevice));
#ifndef KB_HOT_K
#define KB_HOT_K 0
#define KB_HOT_R 1
#endif
    float* dhot = nullptr;
    if (KB_HOT_K > 0) {
        CK(cudaMalloc(&dhot, sizeof(float) * KB_HOT_K * KB_HOT_R * STRIDE));
        CK(cudaMemset(dhot, 0, sizeof(float) * KB_HOT_K * KB_HOT_R * STRIDE));
    }
    int hot_row = 0;
    if (dhot) {  // replicas addressed from syn1 by a whole row offset (as fw2v_host.cpp places them)
        CK(cudaFree(dhot));
        CK(cudaMalloc(&dhot, sizeof(float) * (KB_HOT_K * KB_HOT_R + 1) * STRIDE));
        const long long row = 4LL * STRIDE, diff = (long long)((char*)dhot - (char*)d1);
        long long r = diff / row; while (r * row < diff) ++r;
        hot_row = (int)r;
        CK(cudaMemset((char*)d1 + r * row, 0, sizeof(float) * KB_HOT_K * KB_HOT_R * STRIDE));
        dhot = (float*)((char*)d1 + r * row);
    }
    fw2v::ModelView m{d0, d1, D, STRIDE, V, KB_FLAGS, dhot, KB_HOT_K, KB_HOT_R, hot_row};
    std::vector<cudaStream_t> ss(chunks);
    for (auto& s : ss) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    auto step = [&]() {
        CK(cudaEventRecord(e0, ss[0]));
        for (int c = 1; c < chunks; ++c) CK(cudaStreamWaitEvent(ss[c], e0, 0));
        for (int c = 0; c < chunks; ++c) {
            const int64_t s0 = kept * c / chunks, s1 = kept * (c + 1) / chunks;
            fw2v::BatchView b{dids, doff + s0, dnegs, dalpha + s0, static_cast<int32_t>(s1 - s0)};
            using SMx = fw2v::K1sSmem<KB_LANES, KB_VEC, 3, 6, KB_RING, KB_LIFE>;
            const int per_block = SMx::THREADS / KB_LANES;
            const int blocks = static_cast<int>((s1 - s0 + per_block - 1) / per_block);
            auto* kern = fw2v::k1s_snapshot<KB_LANES, KB_VEC, 3, 6, fw2v::kFullChunk, true, KB_RING, KB_LIFE>;
            const int bytes = SMx::kBlockBytes + KB_PAD;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            kern<<<blocks, SMx::THREADS, bytes, ss[c]>>>(m, b, N, dctr);
            CK(cudaGetLastError());
        }
        for (int c = 1; c < chunks; ++c) { cudaEvent_t ev; CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)); CK(cudaEventRecord(ev, ss[c])); CK(cudaStreamWaitEvent(ss[0], ev, 0)); CK(cudaEventDestroy(ev)); }
        CK(cudaEventRecord(e1, ss[0]));
        CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
        return ms;
    };
    step();
    float best = 1e30f, sum = 0;
    for (int i = 0; i < steps; ++i) { float ms = step(); sum += ms; if (ms < best) best = ms; }
#ifdef KB_TIMING
    {
        unsigned long long h[16];
        CK(cudaMemcpyFromSymbol(h, kb_timing, sizeof(h)));
        const char* names[] = {"top", "wait", "stale+pf", "dots", "bfly", "sigm+g", "D+red", "ctx", "slide"};
        double tot = 0; for (int k = 0; k < 9; ++k) tot += h[k];
        for (int k = 0; k < 9; ++k) printf("%s %.1f%%  ", names[k], 100.0 * h[k] / tot);
        printf("\n");
    }
#endif
    std::vector<float> out(syn0.size());
    CK(cudaMemcpy(out.data(), d1, out.size() * 4, cudaMemcpyDeviceToHost));
    double chk = 0; float mx = 0; size_t bad = 0;
    for (size_t i = 0; i < out.size(); ++i) {
        if (!std::isfinite(out[i])) { ++bad; continue; }
        mx = std::max(mx, std::fabs(out[i]));
        if (i % 97 == 0) chk += out[i];
    }
    std::vector<float> in0(syn0.size());
    CK(cudaMemcpy(in0.data(), d0, in0.size() * 4, cudaMemcpyDeviceToHost));
    float mx0 = 0; for (float v : in0) if (std::isfinite(v)) mx0 = std::max(mx0, std::fabs(v)); else ++bad;
    printf("max|syn1| %.4g max|syn0| %.4g nonfinite %zu  ", mx, mx0, bad);
    {
        using SMx = fw2v::K1sSmem<KB_LANES, KB_VEC, 3, 6, KB_RING, KB_LIFE>;
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fw2v::k1s_snapshot<KB_LANES, KB_VEC, 3, 6, fw2v::kFullChunk, true, KB_RING, KB_LIFE>,
                                                         SMx::THREADS, SMx::kBlockBytes + KB_PAD));
        printf("[%d blocks/SM x %d threads] ", per_sm, SMx::THREADS);
    }
    printf("%s words %llu  best %.3f ms  %.1f Mwords/s  mean %.1f Mwords/s  chk %.6g\n", KB_NAME,
           (unsigned long long)words, best, words / best / 1e3, words / (sum / steps) / 1e3, chk);
    return 0;
}
