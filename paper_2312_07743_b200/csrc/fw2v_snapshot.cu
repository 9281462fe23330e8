// K1s — FULL-W2V window kernel with independent negatives (the paper's update
// rule; reference oracle: sweep_samples_snapshot,
// trainer.cpp:158-205, ReuseMode::window_snapshot).
//
// Every (sample, context) pairing of a window is computed from the
// window-entry values, so the (N+1) x 2W_f dots of a window are independent:
//   1. the N+1 sample rows (syn1) are loaded once (128-bit, through L2);
//   2. all dots are formed per lane (VEC columns each) and reduced across the
//      LANES lanes of the sentence's group with ONE transposed butterfly: at each
//      xor level a lane keeps half of its partial sums and sends the other half,
//      so NV dots cost ~NV shuffles in total instead of NV*log2(LANES);
//   3. each lane evaluates the sigmoid for the few dots it ended up owning and
//      publishes g through 144 B of shared memory;
//   4. sample deltas D_k = sum_r g_kr c_r and context updates c_r += sum_k g_kr s_k
//      are register FMAs; samples are written back once per window.
// The 2W_f+1 ring of syn0 rows (ContextRing, trainer.cpp:32-102) stays in
// registers for the sentence's lifetime and slides by register renaming, as
// in K1. Samples are processed in chunks of NC rows (MULTI: N+1 > NC), with
// context deltas accumulated across chunks so all chunks see window-entry
// context values.
#include <cuda_runtime.h>

#include <cstdint>

#include "fw2v_common.cuh"
#include "fw2v_device.cuh"

namespace fw2v {

// Transposed butterfly over the lanes of a group (offsets O, O/2, ..., 1).
// v[0..N) in, v[0..final) out; slot j of lane l then holds the full group sum
// of the original index given by the same plan run on an index array.
template <int O, int N>
struct Butterfly {
    static constexpr int H = N / 2;
    static constexpr int NEXT = H + (N & 1);
    __host__ __device__ static constexpr int final_count() {
        if constexpr (O > 1) return Butterfly<O / 2, NEXT>::final_count();
        else return NEXT;
    }

    template <int CAP>
    __device__ __forceinline__ static void reduce(float (&v)[CAP], int sub) {
        static_assert(N <= CAP, "butterfly overflow");
        const bool bit = (sub & O) != 0;
#pragma unroll
        for (int j = 0; j < H; ++j) {
            const float a = v[j], b = v[j + H];
            const float send = bit ? a : b;
            const float keep = bit ? b : a;
            v[j] = keep + __shfl_xor_sync(kFull, send, O);
        }
        if constexpr (N & 1) v[H] = v[N - 1] + __shfl_xor_sync(kFull, v[N - 1], O);
        if constexpr (O > 1) Butterfly<O / 2, NEXT>::reduce(v, sub);
    }

    template <int CAP>
    __device__ __forceinline__ static void plan(int (&idx)[CAP], int sub) {
        const bool bit = (sub & O) != 0;
#pragma unroll
        for (int j = 0; j < H; ++j) idx[j] = bit ? idx[j + H] : idx[j];
        if constexpr (N & 1) idx[H] = idx[N - 1];
        if constexpr (O > 1) Butterfly<O / 2, NEXT>::plan(idx, sub);
    }
};

template <int LANES, int VEC, int WF, int NC, bool MULTI, bool FAST>
__global__ void __launch_bounds__(kK1Threads)
k1s_snapshot(ModelView m, BatchView b, int n_neg, DevCounters* __restrict__ ctr) {
    constexpr int NCTX = 2 * WF;
    constexpr int NV = NC * NCTX;
    constexpr int GPW = 32 / LANES;
    using BF = Butterfly<LANES / 2, NV>;
    constexpr int NF = BF::final_count();
    __shared__ float gsh[kK1Threads / 32][GPW][NV];

    const int lane = threadIdx.x & 31;
    const int sub = lane & (LANES - 1);
    const int grp = lane / LANES;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int sent = warp * GPW + grp;
    const bool has = sent < b.n_sentences;
    float* gmy = gsh[threadIdx.x >> 5][grp];

    uint32_t beg = 0, len = 0;
    float alpha = 0.0f;
    if (has) {
        beg = __ldg(b.offsets + sent);
        len = __ldg(b.offsets + sent + 1) - beg;
        alpha = __ldg(b.alpha + sent);
    }
    const int L = static_cast<int>(len);
    const int Lmax = static_cast<int>(__reduce_max_sync(kFull, len));
    if (Lmax == 0) return;

    const int32_t* __restrict__ ids = b.ids + beg;
    const int32_t* __restrict__ negs = b.negs + static_cast<size_t>(beg) * n_neg;
    const size_t stride = static_cast<size_t>(m.stride);
    float* __restrict__ syn0 = m.syn0 + sub * VEC;
    float* __restrict__ syn1 = m.syn1 + sub * VEC;

    // Which (sample, context) dot each of this lane's final butterfly slots holds.
    int slot_q[NF], slot_r[NF], slot_m[NF];
    {
        int idx[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) idx[j] = j;
        BF::plan(idx, sub);
#pragma unroll
        for (int j = 0; j < NF; ++j) {
            slot_m[j] = idx[j];
            slot_q[j] = idx[j] / NCTX;
            slot_r[j] = idx[j] - slot_q[j] * NCTX;
        }
    }
    float ctx[NCTX][VEC];
    int tok[NCTX];
    float tgt[VEC];
    int ttok = L > 0 ? __ldg(ids) : -1;
    if (ttok >= 0) Row<VEC>::load(tgt, syn0 + ttok * stride); else vzero(tgt);
#pragma unroll
    for (int r = 0; r < NCTX; ++r) {
        const int p = r - WF + 1;
        tok[r] = (r >= WF && p < L) ? __ldg(ids + p) : -1;
        if (tok[r] >= 0) Row<VEC>::load(ctx[r], syn0 + tok[r] * stride); else vzero(ctx[r]);
    }
    unsigned c_reads = static_cast<unsigned>(min(L, WF + 1));
    unsigned c_writes = 0, s_rw = 0, pairs = 0;

    // Negatives of the current window, one per lane (lane q holds negative q).
    int negreg = (sub < n_neg && L >= 2) ? __ldg(negs + sub) : -1;
    float dctx[MULTI ? NCTX : 1][VEC];

    for (int i = 0; i < Lmax; ++i) {
        const bool act = i < L;
        const bool wact = act && L >= 2;
        unsigned vmask = 0;
#pragma unroll
        for (int r = 0; r < NCTX; ++r) vmask |= (tok[r] >= 0 ? 1u : 0u) << r;
        const int q_in = i + 1 + WF;
        const int inc_tok = q_in < L ? __ldg(ids + q_in) : -1;
        float inc[VEC];
        if (inc_tok >= 0) Row<VEC>::load(inc, syn0 + inc_tok * stride); else vzero(inc);
        c_reads += inc_tok >= 0;
        const int negnext = (sub < n_neg && i + 1 < L) ? __ldg(negs + static_cast<size_t>(i + 1) * n_neg + sub) : -1;
        if constexpr (MULTI) {
#pragma unroll
            for (int r = 0; r < NCTX; ++r) vzero(dctx[r]);
        }

        for (int ch = 0; ch * NC <= n_neg; ++ch) {
            int sid[NC];
            float S[NC][VEC];
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                const int kk = ch * NC + q;
                const int nb = __shfl_sync(kFull, negreg, (kk - 1) & (LANES - 1), LANES);
                const int s = kk == 0 ? ttok : nb;
                sid[q] = (wact && kk <= n_neg) ? s : -1;
                if (sid[q] >= 0) Row<VEC>::load(S[q], syn1 + sid[q] * stride); else vzero(S[q]);
            }
            unsigned dup = 0;
#pragma unroll
            for (int q = 1; q < NC; ++q)
#pragma unroll
                for (int j = 0; j < q; ++j) dup |= (sid[q] >= 0 && sid[q] == sid[j] ? 1u : 0u) << q;

            // 1-2. all dots of the chunk, then one transposed butterfly.
            float P[NV];
#pragma unroll
            for (int q = 0; q < NC; ++q)
#pragma unroll
                for (int r = 0; r < NCTX; ++r) {
                    float acc = 0.0f;
#pragma unroll
                    for (int e = 0; e < VEC; ++e) acc = fmaf(ctx[r][e], S[q][e], acc);
                    P[q * NCTX + r] = acc;
                }
            BF::reduce(P, sub);

            // 3. sigmoid on owned slots, publish g.
#pragma unroll
            for (int j = 0; j < NF; ++j) {
                const int kk = ch * NC + slot_q[j];
                const bool valid = wact && kk <= n_neg && ((vmask >> slot_r[j]) & 1u);
                const float g = valid ? sgd_coeff<FAST>(P[j], kk == 0 ? 1.0f : 0.0f, alpha) : 0.0f;
                gmy[slot_m[j]] = g;
            }
            __syncwarp();
            float G[NV];
#pragma unroll
            for (int x = 0; x < NV; ++x) G[x] = gmy[x];
            __syncwarp();

            // 4. sample deltas from window-entry contexts; context updates from
            //    window-entry samples.
            float D[NC][VEC];
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                vzero(D[q]);
#pragma unroll
                for (int r = 0; r < NCTX; ++r)
#pragma unroll
                    for (int e = 0; e < VEC; ++e) D[q][e] = fmaf(G[q * NCTX + r], ctx[r][e], D[q][e]);
            }
#pragma unroll
            for (int r = 0; r < NCTX; ++r)
#pragma unroll
                for (int q = 0; q < NC; ++q)
#pragma unroll
                    for (int e = 0; e < VEC; ++e) {
                        if constexpr (MULTI) dctx[r][e] = fmaf(G[q * NCTX + r], S[q][e], dctx[r][e]);
                        else ctx[r][e] = fmaf(G[q * NCTX + r], S[q][e], ctx[r][e]);
                    }
            // Write back (row += delta, trainer.cpp:198-204). A repeated id re-reads
            // the row so both deltas land, as in the reference.
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                if (sid[q] < 0) continue;
                float* row = syn1 + sid[q] * stride;
                if ((dup >> q) & 1u) Row<VEC>::load(S[q], row);
#pragma unroll
                for (int e = 0; e < VEC; ++e) S[q][e] += D[q][e];
                Row<VEC>::store(row, S[q]);
            }
        }
        if constexpr (MULTI) {
#pragma unroll
            for (int r = 0; r < NCTX; ++r)
#pragma unroll
                for (int e = 0; e < VEC; ++e) ctx[r][e] += dctx[r][e];
        }
        if (wact) {
            s_rw += static_cast<unsigned>(n_neg + 1);
            pairs += static_cast<unsigned>(__popc(vmask)) * static_cast<unsigned>(n_neg + 1);
        }

        // Slide the ring (ContextRing::advance, trainer.cpp:55-69).
        const int etok = tok[0];
        if (etok >= 0) {
            Row<VEC>::store(syn0 + etok * stride, ctx[0]);
            ++c_writes;
            if (inc_tok == etok) vcopy(inc, ctx[0]);
        }
#pragma unroll
        for (int r = 0; r < WF - 1; ++r) { vcopy(ctx[r], ctx[r + 1]); tok[r] = tok[r + 1]; }
        vcopy(ctx[WF - 1], tgt);
        tok[WF - 1] = act ? ttok : -1;
        vcopy(tgt, ctx[WF]);
        ttok = tok[WF];
#pragma unroll
        for (int r = WF; r < NCTX - 1; ++r) { vcopy(ctx[r], ctx[r + 1]); tok[r] = tok[r + 1]; }
        vcopy(ctx[NCTX - 1], inc);
        tok[NCTX - 1] = inc_tok;
        negreg = negnext;
    }
#pragma unroll
    for (int r = 0; r < NCTX; ++r) {
        if (tok[r] >= 0) { Row<VEC>::store(syn0 + tok[r] * stride, ctx[r]); ++c_writes; }
    }
    if (ttok >= 0) { Row<VEC>::store(syn0 + ttok * stride, tgt); ++c_writes; }

    if (ctr != nullptr) {
        const bool lead = has && sub == 0;
        const unsigned hits = (L >= 2) ? pairs - static_cast<unsigned>(L) : 0u;
        const unsigned v0 = __reduce_add_sync(kFull, lead ? c_reads : 0u);
        const unsigned v1 = __reduce_add_sync(kFull, lead ? c_writes : 0u);
        const unsigned v2 = __reduce_add_sync(kFull, lead ? s_rw : 0u);
        const unsigned v4 = __reduce_add_sync(kFull, lead ? hits : 0u);
        const unsigned v5 = __reduce_add_sync(kFull, lead ? static_cast<unsigned>(L) : 0u);
        const unsigned v6 = __reduce_add_sync(kFull, lead ? 1u : 0u);
        if (lane == 0) {
            atomicAdd(&ctr->context_reads, v0);
            atomicAdd(&ctr->context_writes, v1);
            atomicAdd(&ctr->sample_reads, v2);
            atomicAdd(&ctr->sample_writes, v2);
            atomicAdd(&ctr->ring_hits, v4);
            atomicAdd(&ctr->words, v5);
            atomicAdd(&ctr->sentences, v6);
        }
    }
}

// ------------------------------------------------------------------ dispatch
template <int LANES, int VEC, int WF, int NC>
cudaError_t launch_k1s_nc(const ModelView& m, const BatchView& b, int n_neg, bool fast, DevCounters* ctr,
                          cudaStream_t st) {
    constexpr int GPW = 32 / LANES;
    const int warps = (b.n_sentences + GPW - 1) / GPW;
    const int blocks = (warps * 32 + kK1Threads - 1) / kK1Threads;
    if (blocks == 0) return cudaSuccess;
    const bool multi = n_neg + 1 > NC;
    if (multi) {
        if (fast) k1s_snapshot<LANES, VEC, WF, NC, true, true><<<blocks, kK1Threads, 0, st>>>(m, b, n_neg, ctr);
        else k1s_snapshot<LANES, VEC, WF, NC, true, false><<<blocks, kK1Threads, 0, st>>>(m, b, n_neg, ctr);
    } else {
        if (fast) k1s_snapshot<LANES, VEC, WF, NC, false, true><<<blocks, kK1Threads, 0, st>>>(m, b, n_neg, ctr);
        else k1s_snapshot<LANES, VEC, WF, NC, false, false><<<blocks, kK1Threads, 0, st>>>(m, b, n_neg, ctr);
    }
    return cudaGetLastError();
}

template <int LANES, int VEC>
cudaError_t launch_k1s_shape(const ModelView& m, const BatchView& b, int n_neg, int wf, bool fast,
                             DevCounters* ctr, cudaStream_t st) {
    switch (wf) {
    case 1: return launch_k1s_nc<LANES, VEC, 1, 6>(m, b, n_neg, fast, ctr, st);
    case 2: return launch_k1s_nc<LANES, VEC, 2, 6>(m, b, n_neg, fast, ctr, st);
    case 3: return launch_k1s_nc<LANES, VEC, 3, 6>(m, b, n_neg, fast, ctr, st);
    case 4: return launch_k1s_nc<LANES, VEC, 4, 4>(m, b, n_neg, fast, ctr, st);
    case 5: return launch_k1s_nc<LANES, VEC, 5, 4>(m, b, n_neg, fast, ctr, st);
    default: return cudaErrorInvalidValue;
    }
}

#define FW2V_K1S_SHAPES(X) X(16, 4) X(32, 4) X(16, 8) X(32, 8) X(32, 10)

// Requires n_neg <= LANES (negatives are distributed one per lane).
cudaError_t launch_k1s(int lanes, int vec, const ModelView& m, const BatchView& b, int n_neg, int wf, bool fast,
                       DevCounters* ctr, cudaStream_t st) {
#define FW2V_CASE(L_, V_) \
    if (lanes == L_ && vec == V_) return launch_k1s_shape<L_, V_>(m, b, n_neg, wf, fast, ctr, st);
    FW2V_K1S_SHAPES(FW2V_CASE)
#undef FW2V_CASE
    return cudaErrorInvalidValue;
}

bool k1s_supported(int lanes, int vec, int n_neg, int wf) {
    if (n_neg > lanes || wf < 1 || wf > 5) return false;
#define FW2V_CASE(L_, V_) if (lanes == L_ && vec == V_) return true;
    FW2V_K1S_SHAPES(FW2V_CASE)
#undef FW2V_CASE
    return false;
}

} // namespace fw2v
