// K1s — FULL-W2V window kernel with independent negatives (the paper's update
// rule; reference oracle: sweep_samples_snapshot,
// trainer.cpp:158-205, ReuseMode::window_snapshot).
//
// Every (sample, context) pairing of a window is computed from window-entry
// values, so the (N+1) x 2W_f dots of a window are independent:
//   1. the N+1 sample rows (syn1) of window i+1 are prefetched with cp.async
//      (16 B per lane, L2 only) into shared memory while window i computes;
//   2. all dots are formed per lane on VEC columns with packed FFMA2
//      (sm_100 fma.rn.f32x2) and reduced across the LANES lanes of the
//      sentence's group with ONE transposed butterfly: at each xor level a lane
//      keeps half of its partial sums and sends the other half, so NV dots cost
//      ~NV shuffles in total instead of NV*log2(LANES);
//   3. each lane evaluates the sigmoid for the dots it ended up owning and
//      publishes g as (g, g) pairs in shared memory;
//   4. sample deltas D_k = sum_r g_kr c_r and context updates
//      c_r += sum_k g_kr s_k are FFMA2 on registers; samples are written once
//      per window (row += delta, trainer.cpp:198-204).
// The 2W_f+1 ring of syn0 rows (ContextRing, trainer.cpp:32-102) stays in
// registers for the sentence's lifetime and slides by register renaming.
// Positions that the reference keeps resident until finish() (the last 2W_f+1)
// are parked in shared memory and written back in ring-slot order, so each
// sentence's global write sequence is the reference's.
#include <cuda_runtime.h>

#include <cstdint>

#include "fw2v_common.cuh"
#include "fw2v_device.cuh"

namespace fw2v {

// Transposed butterfly over the lanes of a group (offsets O, O/2, ..., 1).
// v[0..N) in, v[0..final) out; slot j of lane l then holds the full group sum
// of the original index given by running plan() on an index array.
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

__device__ __forceinline__ void cp_async16(float* smem, const float* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16_ca(float* smem, const float* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
template <int H2>
__device__ __forceinline__ void row_red_add(float* p, const float2 (&d)[H2]) {
#pragma unroll
    for (int i = 0; i < H2; i += 2)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p + 2 * i), "f"(d[i].x), "f"(d[i].y),
                     "f"(d[i + 1].x), "f"(d[i + 1].y)
                     : "memory");
}
// red.add(value - entry_value): the ring row's accumulated update since it was loaded.
template <int H2>
__device__ __forceinline__ void row_red_delta(float* p, const float2 (&v)[H2], const float* entry_smem) {
    float2 e[H2];
    Row2<H2>::load_shared(e, entry_smem);
#pragma unroll
    for (int i = 0; i < H2; ++i) e[i] = make_float2(v[i].x - e[i].x, v[i].y - e[i].y);
    row_red_add(p, e);
}
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
constexpr int kPrefetchWindows = 16;

template <int LANES, int VEC, int WF, int NC>
struct K1sSmem {
    static constexpr int NCTX = 2 * WF;
    static constexpr int C = 2 * WF + 1;
    static constexpr int NV = NC * NCTX;
    static constexpr int STRIDE = LANES * VEC;
    // per group: g pairs, sample prefetch buffer, finish stash
    // per group: g pairs, sample prefetch buffer, finish stash, ring entry values
    // (sample buffers are double-buffered by window parity)
    static constexpr int kGroupFloats = 2 * NV + 2 * NC * STRIDE + 2 * C * STRIDE;
    static constexpr int kBlockBytes = (kK1Threads / LANES) * kGroupFloats * 4;
};

template <int LANES, int VEC, int WF, int NC, bool MULTI, bool FAST>
__global__ void __launch_bounds__(kK1Threads, (VEC >= 8 ? 1 : 3))
k1s_snapshot(ModelView m, BatchView b, int n_neg, DevCounters* __restrict__ ctr) {
    static_assert(VEC % 4 == 0, "K1s stages 16-byte slices");
    using SM = K1sSmem<LANES, VEC, WF, NC>;
    constexpr int NCTX = SM::NCTX;
    constexpr int C = SM::C;
    constexpr int NV = SM::NV;
    constexpr int H2 = VEC / 2;
    constexpr int GPW = 32 / LANES;
    using BF = Butterfly<LANES / 2, NV>;
    constexpr int NF = BF::final_count();
    extern __shared__ __align__(16) float k1s_sh[];

    const int lane = threadIdx.x & 31;
    const int sub = lane & (LANES - 1);
    const int grp = lane / LANES;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int sent = warp * GPW + grp;
    const bool has = sent < b.n_sentences;
    float* gsh = k1s_sh + (threadIdx.x / LANES) * SM::kGroupFloats;
    float2* g2 = reinterpret_cast<float2*>(gsh);
    float* sbuf = gsh + 2 * NV + sub * VEC;                         // + (parity*NC + q)*STRIDE
    float* stash = gsh + 2 * NV + 2 * NC * SM::STRIDE + sub * VEC;  // + slot*STRIDE
    // Ring rows as loaded (delta write-back: red.add(final - loaded)).
    float* entry = gsh + 2 * NV + (2 * NC + C) * SM::STRIDE + sub * VEC;
    const bool delta_wb = (m.flags & kFlagDeltaRing) != 0;

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
    // Row offsets use the compile-time stride (host checks |V| * stride < 2^31).
    float* __restrict__ syn0 = m.syn0 + sub * VEC;
    float* __restrict__ syn1 = m.syn1 + sub * VEC;
    const int tail = L - C;  // positions >= tail stay resident until finish()

    int slot_q[NF], slot_r[NF], slot_m[NF];
    {
        int idx[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) idx[j] = j;
        BF::plan(idx, sub);
#pragma unroll
        for (int j = 0; j < NF; ++j) {
            slot_q[j] = idx[j] / NCTX;
            slot_r[j] = idx[j] - slot_q[j] * NCTX;
            slot_m[j] = slot_r[j] * NC + slot_q[j];  // g pairs are stored context-major
        }
    }

    float2 ctx[NCTX][H2];
    int tok[NCTX];
    float2 tgt[H2];
    int ttok = L > 0 ? __ldg(ids) : -1;
    if (ttok >= 0) Row2<H2>::load(tgt, syn0 + ttok * SM::STRIDE); else vzero2(tgt);
    if (delta_wb) Row2<H2>::store_shared(entry, tgt);  // position 0 -> slot 0
#pragma unroll
    for (int r = 0; r < NCTX; ++r) {
        const int p = r - WF + 1;
        tok[r] = (r >= WF && p < L) ? __ldg(ids + p) : -1;
        if (tok[r] >= 0) Row2<H2>::load(ctx[r], syn0 + tok[r] * SM::STRIDE); else vzero2(ctx[r]);
        if (delta_wb && r >= WF) Row2<H2>::store_shared(entry + p * SM::STRIDE, ctx[r]);  // p < C
    }
    unsigned c_reads = static_cast<unsigned>(min(L, WF + 1));
    unsigned s_rw = 0, pairs = 0;

    // Negatives of the current window, one per lane (lane q holds negative q).
    // Negatives of a window, two per lane: lane q holds negative q (negreg.x)
    // and negative q + LANES (negreg.y), so N <= 2 * LANES.
    int2 negreg = make_int2((sub < n_neg && L >= 2) ? __ldg(negs + sub) : -1,
                            (sub + LANES < n_neg && L >= 2) ? __ldg(negs + sub + LANES) : -1);
    // Negative j (0-based) of the window held in `nr`, broadcast within the group.
    auto neg_of = [&](int2 nr, int j) {
        const int v = __shfl_sync(kFull, j < LANES ? nr.x : nr.y, j & (LANES - 1), LANES);
        return v;
    };
    int tok_ahead = WF + 1 < L ? __ldg(ids + WF + 1) : -1;  // incoming position of window 0
    // Sample ids of the first chunk of the previous window (stale-prefetch check).
    int psid[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) psid[q] = -100;  // sentinels never equal a live or empty sample id

    {
        const float4 z = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
        for (int q = 0; q < 2 * NC; ++q)
#pragma unroll
            for (int e = 0; e < VEC; e += 4) *reinterpret_cast<float4*>(sbuf + q * SM::STRIDE + e) = z;
    }
    const bool l1_samples = (m.flags & kFlagL1Samples) != 0;
    auto prefetch = [&](int target, int2 negv, bool active, int parity) {
        float* dst = sbuf + parity * NC * SM::STRIDE;
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            const int nb = neg_of(negv, q > 0 ? q - 1 : 0);
            const int s = q == 0 ? target : nb;
            if (active && q <= n_neg && s >= 0) {
#pragma unroll
                for (int e = 0; e < VEC; e += 4) {
                    if (l1_samples) cp_async16_ca(dst + q * SM::STRIDE + e, syn1 + s * SM::STRIDE + e);
                    else cp_async16(dst + q * SM::STRIDE + e, syn1 + s * SM::STRIDE + e);
                }
            }
        }
    };
    const int inval_log2 = (m.flags >> kFlagInvalShift) & 15;
    const unsigned inval_mask = inval_log2 ? (1u << inval_log2) - 1u : 0u;
    // Negatives of the next window (window i+1 while window i runs): the
    // prefetch of window i+1's rows is issued at the start of window i.
    int2 negnext = make_int2((sub < n_neg && L >= 2) ? __ldg(negs + n_neg + sub) : -1,
                             (sub + LANES < n_neg && L >= 2) ? __ldg(negs + n_neg + sub + LANES) : -1);
    if (!MULTI) prefetch(ttok, negreg, L >= 2, 0);  // window 0's samples
    float2 dctx[MULTI ? NCTX : 1][H2];

    for (int i = 0; i < Lmax; ++i) {
        const bool act = i < L;
        const bool wact = act && L >= 2;
        unsigned vmask = 0;
#pragma unroll
        for (int r = 0; r < NCTX; ++r) vmask |= (tok[r] >= 0 ? 1u : 0u) << r;
        const int q_in = i + 1 + WF;
        // Token ids run one window ahead of their rows, and the id/negative
        // streams are pulled into L2 kPrefetchWindows ahead, so no row load
        // waits on an id load that missed to DRAM.
        const int inc_tok = tok_ahead;
        // Issued here, consumed at the end of the window (ring slide) and by the
        // next window's prefetch: clamped addresses, no branches, no sinking.
        float2 inc[H2];
        row_load_early(inc, syn0 + max(inc_tok, 0) * SM::STRIDE);
        const int last = max(L - 1, 0);
        const int tok_raw = ldg_early(ids + min(q_in + 1, last));
        const int* nrow = negs + static_cast<size_t>(min(i + 2, last)) * n_neg;
        const int neg_raw = n_neg > 0 ? ldg_early(nrow + min(sub, n_neg - 1)) : -1;
        const int neg_raw2 = n_neg > LANES ? ldg_early(nrow + min(sub + LANES, n_neg - 1)) : -1;
        tok_ahead = q_in + 1 < L ? tok_raw : -1;
        const int2 negnext2 = make_int2((sub < n_neg && i + 2 < L) ? neg_raw : -1,
                                        (sub + LANES < n_neg && i + 2 < L) ? neg_raw2 : -1);
        if (sub == 0 && i + kPrefetchWindows < L) {
            prefetch_l2(negs + static_cast<size_t>(i + kPrefetchWindows) * n_neg);
            prefetch_l2(ids + min(L - 1, q_in + kPrefetchWindows));
        }
        c_reads += inc_tok >= 0;
        if constexpr (MULTI) {
#pragma unroll
            for (int r = 0; r < NCTX; ++r) vzero2(dctx[r]);
        }

        const int n_chunks = MULTI ? (n_neg + NC) / NC : 1;
        for (int ch = 0; ch < n_chunks; ++ch) {
            const int kbase = MULTI ? ch * NC : 0;
            int sid[NC];
            float2 S[NC][H2];
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                const int kk = kbase + q;
                const int nb = neg_of(negreg, kk > 0 ? kk - 1 : 0);
                const int s = kk == 0 ? ttok : nb;
                sid[q] = (wact && kk <= n_neg) ? s : -1 - q;  // empty slots: distinct negative ids
            }
            if constexpr (!MULTI) {
                // Staged by cp.async during the previous window (slots without a
                // sample hold finite stale rows and get g = 0). Rows the previous
                // window rewrote after the prefetch was issued are re-read.
                cp_async_wait_all();
#pragma unroll
                for (int q = 0; q < NC; ++q) Row2<H2>::load_shared(S[q], sbuf + ((i & 1) * NC + q) * SM::STRIDE);
                // Next window's rows go to the other buffer right away.
                if (i + 1 < Lmax) prefetch(tok[WF], negnext, i + 1 < L && L >= 2, (i + 1) & 1);
                bool stale = false;
#pragma unroll
                for (int q = 0; q < NC; ++q)
#pragma unroll
                    for (int j = 0; j < NC; ++j) stale |= sid[q] == psid[j];
                if (stale) {
#pragma unroll
                    for (int q = 0; q < NC; ++q) {
                        bool st = false;
#pragma unroll
                        for (int j = 0; j < NC; ++j) st |= sid[q] == psid[j];
                        if (st && sid[q] >= 0) Row2<H2>::load(S[q], syn1 + sid[q] * SM::STRIDE);
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < NC; ++q) Row2<H2>::load(S[q], syn1 + max(sid[q], 0) * SM::STRIDE);
            }

            // 1-2. all dots of the chunk, then one transposed butterfly.
            float P[NV];
#pragma unroll
            for (int q = 0; q < NC; ++q)
#pragma unroll
                for (int r = 0; r < NCTX; ++r) {
                    float2 acc = __fmul2_rn(ctx[r][0], S[q][0]);
#pragma unroll
                    for (int h = 1; h < H2; ++h) acc = __ffma2_rn(ctx[r][h], S[q][h], acc);
                    P[q * NCTX + r] = acc.x + acc.y;
                }
            BF::reduce(P, sub);


            // 3. sigmoid on owned slots, publish g pairs.
#pragma unroll
            for (int j = 0; j < NF; ++j) {
                const int kk = ch * NC + slot_q[j];
                const bool valid = wact && kk <= n_neg && ((vmask >> slot_r[j]) & 1u);
                const float g = valid ? sgd_coeff<FAST>(P[j], kk == 0 ? 1.0f : 0.0f, alpha) : 0.0f;
                g2[slot_m[j]] = make_float2(g, g);  // context-major: [r][q]
            }
            __syncwarp();

            // 4. context-major sweep: with r fixed, sample deltas take the
            //    window-entry c_r, then c_r takes the window-entry samples, so
            //    each (g, g) pair is loaded once and used twice.
            float2 D[NC][H2];
#pragma unroll
            for (int q = 0; q < NC; ++q) vzero2(D[q]);
#pragma unroll
            for (int r = 0; r < NCTX; ++r) {
                float2 G[NC];
#pragma unroll
                for (int q = 0; q < NC; q += 2) {
                    const float4 t = *reinterpret_cast<const float4*>(g2 + r * NC + q);
                    G[q] = make_float2(t.x, t.y);
                    if (q + 1 < NC) G[q + 1] = make_float2(t.z, t.w);
                }
#pragma unroll
                for (int q = 0; q < NC; ++q)
#pragma unroll
                    for (int h = 0; h < H2; ++h) D[q][h] = __ffma2_rn(G[q], ctx[r][h], D[q][h]);
#pragma unroll
                for (int q = 0; q < NC; ++q)
#pragma unroll
                    for (int h = 0; h < H2; ++h) {
                        if constexpr (MULTI) dctx[r][h] = __ffma2_rn(G[q], S[q][h], dctx[r][h]);
                        else ctx[r][h] = __ffma2_rn(G[q], S[q][h], ctx[r][h]);
                    }
            }
            __syncwarp();
            // Write back (row += delta) as a vector reduction at L2: exactly
            // trainer.cpp:198-204 (repeated ids included), and no read-modify-
            // write round trip on Zipf-hot rows.
#pragma unroll
            for (int q = 0; q < NC; ++q)
                if (sid[q] >= 0) row_red_add(syn1 + sid[q] * SM::STRIDE, D[q]);
            if (ch == 0) {
#pragma unroll
                for (int q = 0; q < NC; ++q) psid[q] = sid[q] >= 0 ? sid[q] : -100;
            }
        }
        if constexpr (MULTI) {
#pragma unroll
            for (int r = 0; r < NCTX; ++r)
#pragma unroll
                for (int h = 0; h < H2; ++h) ctx[r][h] = __fadd2_rn(ctx[r][h], dctx[r][h]);
        }
        if (wact) {
            s_rw += static_cast<unsigned>(n_neg + 1);
            pairs += static_cast<unsigned>(__popc(vmask)) * static_cast<unsigned>(n_neg + 1);
        }

        // Slide the ring (ContextRing::advance, trainer.cpp:55-69).
        const int etok = tok[0];
        if (etok >= 0) {
            const int p = i - WF;
            if (delta_wb) {
                row_red_delta(syn0 + etok * SM::STRIDE, ctx[0], entry + (p % C) * SM::STRIDE);
            } else if (p >= tail) {
                Row2<H2>::store_shared(stash + (p % C) * SM::STRIDE, ctx[0]);
            } else {
                Row2<H2>::store(syn0 + etok * SM::STRIDE, ctx[0]);
            }
            if (inc_tok == etok) vcopy2(inc, ctx[0]);
        }
        if (delta_wb && inc_tok >= 0) Row2<H2>::store_shared(entry + (q_in % C) * SM::STRIDE, inc);
#pragma unroll
        for (int r = 0; r < WF - 1; ++r) { vcopy2(ctx[r], ctx[r + 1]); tok[r] = tok[r + 1]; }
        vcopy2(ctx[WF - 1], tgt);
        tok[WF - 1] = act ? ttok : -1;
        vcopy2(tgt, ctx[WF]);
        ttok = tok[WF];
#pragma unroll
        for (int r = WF; r < NCTX - 1; ++r) { vcopy2(ctx[r], ctx[r + 1]); tok[r] = tok[r + 1]; }
        vcopy2(ctx[NCTX - 1], inc);
        tok[NCTX - 1] = inc_tok;
        negreg = negnext;
        negnext = negnext2;
        // Bounded staleness for L1-cached sample rows: refresh this SM's L1.
        if (inval_mask != 0u && (static_cast<unsigned>(i) & inval_mask) == inval_mask &&
            (threadIdx.x >> 5) == 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
    }
    // ContextRing::finish (trainer.cpp:71-75): residents in slot order.
    if (delta_wb) {
        // Deltas commute: no ordering to preserve.
        const int i_end = Lmax;
#pragma unroll
        for (int r = 0; r < NCTX; ++r) {
            const int p = r < WF ? i_end - WF + r : i_end + 1 + (r - WF);
            if (tok[r] >= 0) row_red_delta(syn0 + tok[r] * SM::STRIDE, ctx[r], entry + (p % C) * SM::STRIDE);
        }
        if (ttok >= 0) row_red_delta(syn0 + ttok * SM::STRIDE, tgt, entry + (i_end % C) * SM::STRIDE);
    } else {
        const int i_end = Lmax;  // registers hold positions i_end-WF .. i_end+WF
#pragma unroll
        for (int r = 0; r < NCTX; ++r) {
            const int p = r < WF ? i_end - WF + r : i_end + 1 + (r - WF);
            if (tok[r] >= 0) Row2<H2>::store_shared(stash + (p % C) * SM::STRIDE, ctx[r]);
        }
        if (ttok >= 0) Row2<H2>::store_shared(stash + (i_end % C) * SM::STRIDE, tgt);
        const int first = max(0, tail);
        for (int s = 0; s < C; ++s) {
            // the resident position in slot s: first + ((s - first) mod C), if < L
            const int p = first + ((s - first % C) + C) % C;
            if (p < L) {
                float2 v[H2];
                Row2<H2>::load_shared(v, stash + s * SM::STRIDE);
                Row2<H2>::store(syn0 + __ldg(ids + p) * SM::STRIDE, v);
            }
        }
    }

    if (ctr != nullptr) {
        const bool lead = has && sub == 0;
        const unsigned hits = (L >= 2) ? pairs - static_cast<unsigned>(L) : 0u;
        const unsigned v0 = __reduce_add_sync(kFull, lead ? c_reads : 0u);
        const unsigned v2 = __reduce_add_sync(kFull, lead ? s_rw : 0u);
        const unsigned v4 = __reduce_add_sync(kFull, lead ? hits : 0u);
        const unsigned v5 = __reduce_add_sync(kFull, lead ? static_cast<unsigned>(L) : 0u);
        const unsigned v6 = __reduce_add_sync(kFull, lead ? 1u : 0u);
        if (lane == 0) {
            atomicAdd(&ctr->context_reads, v0);
            atomicAdd(&ctr->context_writes, v5);  // every position is written back exactly once
            atomicAdd(&ctr->sample_reads, v2);
            atomicAdd(&ctr->sample_writes, v2);
            atomicAdd(&ctr->ring_hits, v4);
            atomicAdd(&ctr->words, v5);
            atomicAdd(&ctr->sentences, v6);
        }
    }
}

// ------------------------------------------------------------------ dispatch
template <int LANES, int VEC, int WF, int NC, bool MULTI, bool FAST>
cudaError_t launch_k1s_inst(int blocks, const ModelView& m, const BatchView& b, int n_neg, DevCounters* ctr,
                            cudaStream_t st, int* resident) {
    constexpr int bytes = K1sSmem<LANES, VEC, WF, NC>::kBlockBytes;
    auto* kern = k1s_snapshot<LANES, VEC, WF, NC, MULTI, FAST>;
    static bool configured = false;  // benign race: idempotent attribute set
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    if (resident != nullptr) return resident_sentences(kern, bytes, kK1Threads / LANES, resident);
    if (blocks == 0) return cudaSuccess;
    kern<<<blocks, kK1Threads, bytes, st>>>(m, b, n_neg, ctr);
    return cudaGetLastError();
}

template <int LANES, int VEC, int WF, int NC>
cudaError_t launch_k1s_nc(const ModelView& m, const BatchView& b, int n_neg, bool fast, DevCounters* ctr,
                          cudaStream_t st, int* resident) {
    constexpr int GPW = 32 / LANES;
    const int warps = (b.n_sentences + GPW - 1) / GPW;
    const int blocks = (warps * 32 + kK1Threads - 1) / kK1Threads;
    const bool multi = n_neg + 1 > NC;
    if (multi) {
        return fast ? launch_k1s_inst<LANES, VEC, WF, NC, true, true>(blocks, m, b, n_neg, ctr, st, resident)
                    : launch_k1s_inst<LANES, VEC, WF, NC, true, false>(blocks, m, b, n_neg, ctr, st, resident);
    }
    return fast ? launch_k1s_inst<LANES, VEC, WF, NC, false, true>(blocks, m, b, n_neg, ctr, st, resident)
                : launch_k1s_inst<LANES, VEC, WF, NC, false, false>(blocks, m, b, n_neg, ctr, st, resident);
}

template <int LANES, int VEC>
cudaError_t launch_k1s_shape(const ModelView& m, const BatchView& b, int n_neg, int wf, bool fast,
                             DevCounters* ctr, cudaStream_t st, int* resident) {
    switch (wf) {
    case 1: return launch_k1s_nc<LANES, VEC, 1, 6>(m, b, n_neg, fast, ctr, st, resident);
    case 2: return launch_k1s_nc<LANES, VEC, 2, 6>(m, b, n_neg, fast, ctr, st, resident);
    case 3: return launch_k1s_nc<LANES, VEC, 3, 6>(m, b, n_neg, fast, ctr, st, resident);
    // Wide windows: one 6-sample chunk when N+1 <= 6, else 4-sample chunks (registers).
    case 4: return n_neg + 1 <= 6 ? launch_k1s_nc<LANES, VEC, 4, 6>(m, b, n_neg, fast, ctr, st, resident)
                                  : launch_k1s_nc<LANES, VEC, 4, 4>(m, b, n_neg, fast, ctr, st, resident);
    case 5: return n_neg + 1 <= 6 ? launch_k1s_nc<LANES, VEC, 5, 6>(m, b, n_neg, fast, ctr, st, resident)
                                  : launch_k1s_nc<LANES, VEC, 5, 4>(m, b, n_neg, fast, ctr, st, resident);
    default: return cudaErrorInvalidValue;
    }
}

#define FW2V_K1S_SHAPES(X) X(4, 4) X(8, 4) X(16, 4) X(32, 4) X(32, 8)

// Requires n_neg <= 2 * LANES (negatives are distributed two per lane).
cudaError_t launch_k1s(int lanes, int vec, const ModelView& m, const BatchView& b, int n_neg, int wf, bool fast,
                       DevCounters* ctr, cudaStream_t st, int* resident) {
#define FW2V_CASE(L_, V_) \
    if (lanes == L_ && vec == V_) return launch_k1s_shape<L_, V_>(m, b, n_neg, wf, fast, ctr, st, resident);
    FW2V_K1S_SHAPES(FW2V_CASE)
#undef FW2V_CASE
    return cudaErrorInvalidValue;
}

bool k1s_supported(int lanes, int vec, int n_neg, int wf) {
    if (n_neg > 2 * lanes || wf < 1 || wf > 5) return false;
#define FW2V_CASE(L_, V_) if (lanes == L_ && vec == V_) return true;
    FW2V_K1S_SHAPES(FW2V_CASE)
#undef FW2V_CASE
    return false;
}

} // namespace fw2v
