// K1s lifetime order as a staircase of windows (sm_100a, CUDA cores).
//
// The reference's default update order (sweep_samples, trainer.cpp:133-154:
// samples outer, contexts inner, every pairing sees the previous pairings'
// updates) makes pairing (k, j) of a window depend on (k, j-1) and (k-1, j):
// one window is a wavefront of NC + 2W_f - 1 anti-diagonal steps. Across
// windows the only dependency (besides sample ids repeated between windows)
// is that window i+1's first sample may touch context row p only after window
// i's last sample is done with it: (i+1, 0, j) after (i, NC-1, j+1). Window
// i+1 can therefore start NC + 1 steps after window i instead of NC + 2W_f - 1:
// iteration i runs window i's steps 0..NC (the head) interleaved with window
// i-1's remaining steps (the tail). At W_f = 3, NC = 6 that is 7 steps per
// window instead of 11, each with 5-6 independent dots (36 per window), and at
// most 6 sample rows live in registers at any step.
//
// Pairings of one step touch disjoint rows (head rows k <= t, tail rows
// k >= t + 2; context rows of the two windows never coincide in one step), so
// per sentence the result is the reference order exactly (same FP operations
// as the one-window wavefront of k1s_snapshot<..., LIFETIME = true>).
//
// Windows whose sample ids repeat (inside the window, or shared with the
// previous window: the reference re-reads the row after the earlier write,
// trainer.cpp:143) are not overlapped: the pending tail finishes alone, the
// window's rows are re-read, and a repeat inside the window runs the samples
// serially with the rewritten row forwarded.
//
// Registers: rows Q[r] = syn0 row of position i - W_f + r (r = 0..2W_f; r = W_f
// is the window's target word, the others its contexts), the head's sample
// rows Sc, the tail's Sp, and the incoming row. Context rows leave by overwrite
// (Hogwild, the reference's memcpy write-back, trainer.cpp:61-63); sample rows
// leave as red.global.add(final - staged) (row += delta).
#pragma once

namespace fw2v {

template <int LANES, int VEC, int WF, int NS_ = 6>
struct StairCfg {
    static constexpr int NC = NS_;                     // samples per window (N + 1)
    static constexpr int NCTX = 2 * WF;
    // Sample rows in registers per window: a sample is live for 2W_f consecutive
    // steps (its pairings with the contexts), so at most 2W_f are live at once;
    // sample k lives in slot k mod NSL (N + 1 = 16 runs through 6 slots at W_f = 3).
    static constexpr int NSL = NC < NCTX ? NC : NCTX;
    static constexpr int NQ = 2 * WF + 1;              // ring rows in registers
    static constexpr int STEPS_ = NC + 2 * WF - 1;
    // Window-to-window offset in steps: >= NC + 1 (the first sample of window i+1
    // touches a context row after the last sample of window i), and more than half
    // a window so that only two windows are ever live (W_f = 5: 8).
    static constexpr int OFF = (NC + 1 > STEPS_ / 2 + 1) ? NC + 1 : STEPS_ / 2 + 1;
    static constexpr int STEPS = NC + NCTX - 1;        // one window's wavefront
    static constexpr int T = STEPS > OFF ? STEPS - OFF : 0;  // tail steps run in the next iteration
    static constexpr int STRIDE = LANES * VEC;
    static constexpr int THREADS = VEC >= 8 ? 64 : kK1Threads;
    // Staging, double-buffered by window parity, plus the incoming ring row
    // (16-byte chunks: cp.async.cg, coherent with this thread's st.global.cg).
    static constexpr int kGroupFloats = (2 * NC + 1) * STRIDE;
    static constexpr int kBlockBytes = (THREADS / LANES) * kGroupFloats * 4;
    static constexpr int kSmemBlocks = (227 * 1024) / (kBlockBytes + 1024);
#ifdef FW2V_STAIR_REG_BLOCKS  // experiments (tools/variant_lib.sh)
    static constexpr int kRegBlocks = FW2V_STAIR_REG_BLOCKS;
#else
    // 16 x 8 at W_f <= 3: 5 blocks of 2 warps (168 registers, 28 B of spills) beat
    // 4 blocks at 222 registers by 8% (profiles/r02bb_stair_blocks.txt); wider
    // windows spill 0.7-1.2 KB at 168 and keep 4.
    static constexpr int kRegBlocks = VEC < 8 ? 3 : (VEC == 8 && LANES == 16 && WF <= 3 && NS_ <= 6 ? 5 : 4);
#endif
    static constexpr int MINB = kSmemBlocks < kRegBlocks ? (kSmemBlocks < 1 ? 1 : kSmemBlocks) : kRegBlocks;
};

// LANES in {16, 32} (a group is half a warp or a warp; the repeat check uses
// lanes 0..5 and HALF..HALF+5 of the group), N = 5, Hogwild overwrite of the
// context rows.
template <int LANES, int VEC, int WF, int NS, bool FAST>
__device__ __forceinline__ void stair_sentence(const ModelView& m, const BatchView& b, DevCounters* __restrict__ ctr,
                                               int sent0) {
    using CF = StairCfg<LANES, VEC, WF, NS>;
    constexpr int NC = CF::NC, NN = NC - 1, NCTX = CF::NCTX, NQ = CF::NQ, OFF = CF::OFF, T = CF::T, NSL = CF::NSL;
    auto sl_ = [](int k) { return k % NSL; };  // register slot of sample k
    constexpr int H2 = VEC / 2;
    constexpr int STRIDE = CF::STRIDE;
    constexpr int HALF = LANES / 2;
    static_assert(LANES <= 32 && HALF >= NC, "repeat check needs 2 x NC lanes per group");
    static_assert(VEC % 2 == 0, "8- or 16-byte chunks");
    using SL = Slice<H2, LANES>;
    extern __shared__ __align__(16) float k1s_sh[];

    const int lane = threadIdx.x & 31;
    const int sub = static_cast<int>(threadIdx.x) & (LANES - 1);
    const int grp = lane / LANES;
    const int sent = sent0 + static_cast<int>(threadIdx.x / LANES);
    const bool has = sent < b.n_sentences;
    float* sbuf = k1s_sh + (threadIdx.x / LANES) * CF::kGroupFloats + sub * SL::CW;  // + (parity*NC + k)*STRIDE

    uint32_t beg = 0, len = 0;
    float alpha = 0.0f;
    if (has) {
        beg = __ldg(b.offsets + sent);
        len = __ldg(b.offsets + sent + 1) - beg;
        alpha = __ldg(b.alpha + sent);
    }
    const int L = static_cast<int>(len);
    if (sub == 0) obs_record_sentence(b, sent, L);  // observer (test mode)
    if (m.beat != nullptr && threadIdx.x == 0) atomicAdd(m.beat, 1u);  // live merge: still training
    const int Lmax = static_cast<int>(__reduce_max_sync(kFull, len));
    if (Lmax == 0) return;
    const int32_t* __restrict__ ids = b.ids + beg;
    const int32_t* __restrict__ negs = b.negs + static_cast<size_t>(beg) * NN;
    float* __restrict__ syn0 = m.syn0 + sub * SL::CW;
    float* __restrict__ syn1 = m.syn1 + sub * SL::CW;
    const int hot_k = m.hot_k;
    const int hot_off = m.hot_k > 0 ? m.hot_row + (sent % m.hot_r) * m.hot_k : 0;
    auto srow = [&](int s) { return syn1 + static_cast<int64_t>(s < hot_k ? s + hot_off : s) * STRIDE; };
    const float nha = -0.5f * alpha;

    // Ring rows: Q[r] = position i - WF + r of window i.
    float2 Q[NQ][H2];
    int qtok[NQ];
#pragma unroll
    for (int r = 0; r < NQ; ++r) {
        const int p = r - WF;
        qtok[r] = (p >= 0 && p < L) ? __ldg(ids + p) : -1;
        if (qtok[r] >= 0) SL::load(Q[r], syn0 + static_cast<int64_t>(qtok[r]) * STRIDE); else vzero2(Q[r]);
    }
    unsigned qv = 0;  // bit r: Q[r] holds a position of the sentence
#pragma unroll
    for (int r = 0; r < NQ; ++r) qv |= (qtok[r] >= 0 ? 1u : 0u) << r;

    // Sample ids, one per lane: lane q (q = sub mod HALF < NC) of a group holds
    // sample q of a window (the target id for q = 0, negative q-1 otherwise),
    // other lanes a unique negative value. idp / idc: windows i-1 / i; idn:
    // window i+1 (from step T on). Lanes fetch a window's ids by shuffle.
    const int qid = sub & (HALF - 1);
    const int qneg = min(max(qid - 1, 0), NN - 1);
    const int gl = grp * LANES;  // the group's first lane
    auto make_id = [&](int tok0, int neg, bool active) { return (active && qid < NC) ? (qid == 0 ? tok0 : neg) : -1 - lane; };
    int idc = make_id(qtok[WF], L >= 2 ? __ldg(negs + qneg) : -1, L >= 2);
    int idp = -1 - lane, idn = -1 - lane;
    int nr_next = 1 < L ? __ldg(negs + NN + qneg) : -1;  // this lane's negative of window i+1
    int tok_ahead = WF + 1 < L ? __ldg(ids + WF + 1) : -1;  // incoming position of window 0

#pragma unroll
    for (int q = 0; q < 2 * NC + 1; ++q) SL::zero_shared(sbuf + q * STRIDE);
    const bool l1_exact = (m.flags & kFlagL1Exact) != 0;
    const int inval_log2 = (m.flags >> kFlagInvalShift) & 15;
    const unsigned inval_mask = inval_log2 ? (1u << inval_log2) - 1u : 0u;

    // Stage the sample rows of a window (ids in idw) into a buffer.
    auto prefetch = [&](int idw, int parity) {
        float* dst = sbuf + parity * NC * STRIDE;
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            const int s = __shfl_sync(kFull, idw, gl + q);
            if (s >= 0) SL::template stage<true>(dst + q * STRIDE, srow(s));
        }
        cp_async_commit();
    };
    // Repeats of a window (ids idw): inside the window (dup), or shared with the
    // previous window (ids idv; lanes HALF.. of the group carry them to the match).
    // The match is issued at step T and its votes taken at the end of the
    // iteration (off the critical path: MATCH has a long latency).
    auto repeats_issue = [&](int idw, int idv) { return __match_any_sync(kFull, sub < HALF ? idw : idv); };
    auto repeats = [&](unsigned mm, bool& dup) {
        const unsigned lower = ((1u << HALF) - 1u) << gl;
        const unsigned upper = lower << HALF;
        dup = __any_sync(kFull, sub < HALF && __popc(mm & lower) > 1);
        return __any_sync(kFull, sub < HALF && (mm & upper) != 0u);
    };

    prefetch(idc, 0);
    bool dup_n = false;
    bool stale_n = repeats(repeats_issue(idc, -1 - lane), dup_n);  // window 0 (no previous window: never stale)
    unsigned mm_n = 0;

    auto dot = [&](const float2 (&c)[H2], const float2 (&s)[H2]) {
        float2 acc = __fmul2_rn(c[0], s[0]);
#pragma unroll
        for (int h = 1; h < H2; ++h) acc = __ffma2_rn(c[h], s[h], acc);
        return acc.x + acc.y;
    };
    auto update = [&](float2 (&c)[H2], float2 (&s)[H2], float g) {  // pairing_update (kernels.hpp:26-33)
        const float2 gg = make_float2(g, g);
#pragma unroll
        for (int h = 0; h < H2; ++h) {
            const float2 cc = c[h];
            c[h] = __ffma2_rn(gg, s[h], cc);
            s[h] = __ffma2_rn(gg, cc, s[h]);
        }
    };
    // g for a pairing with coefficient hn = valid ? -alpha/2 : 0 (label 1 for k = 0).
    auto coeff = [&](float f, float hn, bool positive) {
        if constexpr (FAST) {
            return fmaf(hn, tanh_approx(half_clamped(f)), positive ? -hn : hn);
        } else {
            return sgd_coeff<false>(f, positive ? 1.0f : 0.0f, -2.0f * hn);
        }
    };
    auto writeback = [&](const float2 (&s)[H2], const float* staged, int sid, bool pred) {
        float2 e[H2];
        SL::load_shared(e, staged);
#pragma unroll
        for (int h = 0; h < H2; ++h) e[h] = make_float2(s[h].x - e[h].x, s[h].y - e[h].y);
        SL::red_add_if(pred && sid >= 0, srow(max(sid, 0)), e);
    };
    // Context slot j of the current window -> ring row; of the previous window -> ring row.
    auto rh = [](int j) { return j < WF ? j : j + 1; };
    auto rt = [](int j) { return j < WF ? j - 1 : j; };

    float2 Sc[NSL][H2], Sp[NSL][H2];
#pragma unroll
    for (int k = 0; k < NSL; ++k) { vzero2(Sc[k]); vzero2(Sp[k]); }
    bool tact = false;  // the previous window's tail is pending
    unsigned tvm = 0;   // tail validity per ring row (previous window, current indexing)

    // One step t of iteration i: head pairings (k, t-k) of window i, tail
    // pairings (k, t+OFF-k) of window i-1.
    // (t and HEAD are constants once the step loops below are unrolled.)
    auto step = [&](const int t, const bool HEAD, unsigned hvm, const float* cur, const float* prv, bool wact) {
        auto hd = [&](int k) { return HEAD && t - k >= 0 && t - k < NCTX; };
        auto tl = [&](int k) { return t + OFF - k >= 0 && t + OFF - k < NCTX; };
        // Head samples are k <= t, tail samples k >= t + OFF - NCTX + 1: while
        // OFF >= NCTX a sample index has at most one pairing per step (one dot
        // array); otherwise (W_f >= 4 at N = 5) it can have both (slots of Sc and
        // Sp): a second array for the tail.
        constexpr bool kBoth = OFF < NCTX;
        float fh[NC], ft[kBoth ? NC : 1];
        auto tf = [&](int k) -> float& {
            if constexpr (kBoth) return ft[k];
            else return fh[k];
        };
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            if (hd(k)) fh[k] = dot(Q[rh(t - k)], Sc[sl_(k)]);
            if (tl(k)) tf(k) = dot(Q[rt(t + OFF - k)], Sp[sl_(k)]);
        }
#pragma unroll
        for (int o = LANES / 2; o > 0; o >>= 1)
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                if (hd(k)) fh[k] += __shfl_xor_sync(kFull, fh[k], o);
                if (tl(k)) tf(k) += __shfl_xor_sync(kFull, tf(k), o);
            }
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            if (hd(k)) {
                const int jh = t - k;
                update(Q[rh(jh)], Sc[sl_(k)], coeff(fh[k], ((hvm >> rh(jh)) & 1u) ? nha : 0.0f, k == 0));
                if (jh == NCTX - 1) writeback(Sc[sl_(k)], cur + k * STRIDE, __shfl_sync(kFull, idc, gl + k), wact);
            }
            if (tl(k)) {
                const int jt = t + OFF - k;
                update(Q[rt(jt)], Sp[sl_(k)], coeff(tf(k), ((tvm >> rt(jt)) & 1u) ? nha : 0.0f, k == 0));
                if (jt == NCTX - 1) writeback(Sp[sl_(k)], prv + k * STRIDE, __shfl_sync(kFull, idp, gl + k), tact);
            }
        }
    };

    for (int i = 0; i < Lmax; ++i) {
        const bool act = i < L;
        const bool wact = act && L >= 2;
        const int q_in = i + 1 + WF;
        const float* cur = sbuf + (i & 1) * NC * STRIDE;
        const float* prv = sbuf + ((i + 1) & 1) * NC * STRIDE;
        // Early loads: the incoming ring row (position i+1+W_f), the next ids,
        // window i+2's negatives; L2 prefetch of the id/negative streams.
        const int inc_tok = tok_ahead;
        constexpr bool kIncSmem = SL::CW == 4;
        float2 inc[H2];
        if constexpr (!kIncSmem) SL::load_early(inc, syn0 + static_cast<int64_t>(max(inc_tok, 0)) * STRIDE);
        const int last = max(L - 1, 0);
        const int tok_raw = ldg_early(ids + min(q_in + 1, last));
        const int nr_raw = ldg_early(negs + static_cast<size_t>(min(i + 2, last)) * NN + qneg);
        const bool tok_ok = q_in + 1 < L;
        if (sub == 0 && i + kPrefetchWindows < L) {
            prefetch_l2(negs + static_cast<size_t>(i + kPrefetchWindows) * NN);
            prefetch_l2(ids + min(L - 1, q_in + kPrefetchWindows));
        }

        const unsigned hvm = wact ? qv : 0u;  // head validity per ring row

        const bool dup = dup_n;
        if (stale_n || dup) {
            // Not overlapped: the previous window's tail alone, then this
            // window's rows re-read after its write-backs. (Warp-uniform branch:
            // the steps shuffle; a sentence without a pending tail has tvm = 0.)
            if (__any_sync(kFull, tact)) {
#pragma unroll
                for (int t = 0; t < T; ++t) step(t, false, 0u, cur, prv, wact);
                tact = false;
                tvm = 0;
            }
            cp_async_wait_group<0>();
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                float2 v[H2];
                SL::load(v, srow(max(__shfl_sync(kFull, idc, gl + q), 0)));
                SL::store_shared(const_cast<float*>(cur) + q * STRIDE, v);
            }
        } else {
            cp_async_wait_group<0>();
        }
        float* inc_sh = sbuf + 2 * NC * STRIDE;
        if constexpr (kIncSmem) {
            if (inc_tok >= 0) {
                const float* src = syn0 + static_cast<int64_t>(inc_tok) * STRIDE;
#pragma unroll
                for (int c = 0; c < SL::NCH; ++c) {
                    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(inc_sh + c * SL::CS));
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + c * SL::CS) : "memory");
                }
            }
            cp_async_commit();
        }
        // (Next window's staging is issued after this window's tail steps.)
        auto issue_next = [&]() {
            // Rows staged through L1 (8-byte chunks) need its refresh; with 16-byte
            // chunks they come from L2 (cp.async.cg) and see every write there.
            if (!SL::kCanL2Only && (l1_exact || (inval_mask != 0u && (static_cast<unsigned>(i) & inval_mask) == inval_mask &&
                                                  (threadIdx.x >> 5) == 0)))
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            const bool nact = i + 1 < L && L >= 2;
            idn = make_id(qtok[WF + 1], nr_next, nact);
            if (i + 1 < Lmax) prefetch(idn, (i + 1) & 1);
            else cp_async_commit();  // the slide below waits for all but the newest group
            mm_n = repeats_issue(idn, idc);
        };
        if (!dup) {
            // Sample t enters its slot at step t (its first pairing): the slot's
            // previous sample, t - NSL, had its last pairing at step t - 1.
#pragma unroll
            for (int t = 0; t < OFF; ++t) {
                if (t < NC) SL::load_shared(Sc[sl_(t)], cur + t * STRIDE);
                step(t, true, hvm, cur, prv, wact);
                if (t == T) issue_next();
            }
            // Samples k >= OFF - NCTX + 1 finish in the next iteration's tail.
#pragma unroll
            for (int k = 0; k < NSL; ++k) vcopy2(Sp[k], Sc[k]);
            tvm = hvm;
            tact = wact && T > 0;
        } else {
            // Reference order, sample by sample; a repeated id starts from the
            // row its previous occurrence left (the reference re-reads it): that
            // row is handed to the next occurrence through its staging slot, and
            // the last occurrence writes final - staged (the first occurrence's
            // slot keeps the staged row). Rare: a rolled loop, one row in registers.
            const unsigned mmw = __match_any_sync(kFull, idc);  // lanes holding the same id
            const unsigned grp_mask = (NC >= 32 ? ~0u : ((1u << NC) - 1u));
#pragma unroll 1
            for (int k = 0; k < NC; ++k) {
                float2 S[H2];
                SL::load_shared(S, cur + k * STRIDE);
#pragma unroll
                for (int j = 0; j < NCTX; ++j) {
                    float f = dot(Q[rh(j)], S);
#pragma unroll
                    for (int o = LANES / 2; o > 0; o >>= 1) f += __shfl_xor_sync(kFull, f, o);
                    update(Q[rh(j)], S, coeff(f, ((hvm >> rh(j)) & 1u) ? nha : 0.0f, k == 0));
                }
                const unsigned same = (__shfl_sync(kFull, mmw, gl + k) >> gl) & grp_mask;  // bit q: sample q
                const int sid = __shfl_sync(kFull, idc, gl + k);  // (shuffles before the per-sentence branch)
                const unsigned later = same & ~((2u << k) - 1u);
                if (later != 0u) {
                    SL::store_shared(const_cast<float*>(cur) + (__ffs(later) - 1) * STRIDE, S);
                } else {
                    writeback(S, cur + (__ffs(same) - 1) * STRIDE, sid, wact);
                }
            }
            issue_next();
            tact = false;
            tvm = 0;
        }
        stale_n = repeats(mm_n, dup_n);

        // Slide the ring (ContextRing::advance, trainer.cpp:55-69): position
        // i - W_f leaves (its last pairing was window i's), i+1+W_f enters.
        if constexpr (kIncSmem) {
            cp_async_wait_group<1>();
            SL::load_shared(inc, inc_sh);
        }
        if (qtok[0] >= 0) {
            SL::store(syn0 + static_cast<int64_t>(qtok[0]) * STRIDE, Q[0]);
            if (inc_tok == qtok[0]) vcopy2(inc, Q[0]);
        }
#pragma unroll
        for (int r = 0; r < NQ - 1; ++r) { vcopy2(Q[r], Q[r + 1]); qtok[r] = qtok[r + 1]; }
        vcopy2(Q[NQ - 1], inc);
        qtok[NQ - 1] = inc_tok;
        tvm >>= 1;
        qv = (qv >> 1) | ((inc_tok >= 0 ? 1u : 0u) << (NQ - 1));
        idp = idc;
        idc = idn;
        nr_next = i + 2 < L ? nr_raw : -1;
        tok_ahead = tok_ok ? tok_raw : -1;
    }
    // The last window's tail.
    if (__any_sync(kFull, tact)) {
        const float* prv = sbuf + ((Lmax + 1) & 1) * NC * STRIDE;
#pragma unroll
        for (int t = 0; t < T; ++t) step(t, false, 0u, prv, prv, false);
    }
    // ContextRing::finish (trainer.cpp:71-75): the residents, in any order (overwrite).
#pragma unroll
    for (int r = 0; r < NQ; ++r)
        if (qtok[r] >= 0) SL::store(syn0 + static_cast<int64_t>(qtok[r]) * STRIDE, Q[r]);

    if (ctr != nullptr) {
        const bool lead = has && sub == 0;
        // Closed forms of the per-window counts (each position read once; every
        // window of a sentence of >= 2 words has N+1 samples and its valid contexts).
        const unsigned c_reads = static_cast<unsigned>(L);
        const unsigned s_rw = L >= 2 ? static_cast<unsigned>(L) * NC : 0u;
        const unsigned half = L <= WF + 1 ? static_cast<unsigned>(L * (L - 1) / 2)
                                          : static_cast<unsigned>(WF * (WF + 1) / 2 + (L - WF - 1) * WF);
        const unsigned pairs = L >= 2 ? 2u * half * NC : 0u;
        const unsigned hits = (L >= 2) ? pairs - static_cast<unsigned>(L) : 0u;
        const unsigned v0 = __reduce_add_sync(kFull, lead ? c_reads : 0u);
        const unsigned v2 = __reduce_add_sync(kFull, lead ? s_rw : 0u);
        const unsigned v4 = __reduce_add_sync(kFull, lead ? hits : 0u);
        const unsigned v5 = __reduce_add_sync(kFull, lead ? static_cast<unsigned>(L) : 0u);
        const unsigned v6 = __reduce_add_sync(kFull, lead ? 1u : 0u);
        if (lane == 0) {
            atomicAdd(&ctr->context_reads, v0);
            atomicAdd(&ctr->context_writes, v5);
            atomicAdd(&ctr->sample_reads, v2);
            atomicAdd(&ctr->sample_writes, v2);
            atomicAdd(&ctr->ring_hits, v4);
            atomicAdd(&ctr->words, v5);
            atomicAdd(&ctr->sentences, v6);
        }
    }
    cp_async_wait_group<0>();  // the staging buffers are the next sentence's
}

// Blocks stride over the batch's sentences (BatchView::max_groups caps the grid).
template <int LANES, int VEC, int WF, int NS, bool FAST>
__global__ void __launch_bounds__(StairCfg<LANES, VEC, WF, NS>::THREADS, StairCfg<LANES, VEC, WF, NS>::MINB)
k1s_stair(ModelView m, BatchView b, DevCounters* __restrict__ ctr) {
    constexpr int PB = StairCfg<LANES, VEC, WF, NS>::THREADS / LANES;
    for (int s0 = static_cast<int>(blockIdx.x) * PB; s0 < b.n_sentences; s0 += static_cast<int>(gridDim.x) * PB)
        stair_sentence<LANES, VEC, WF, NS, FAST>(m, b, ctr, s0);
}

template <int LANES, int VEC, int WF, int NS, bool FAST>
cudaError_t launch_k1s_stair(const ModelView& m, const BatchView& b, DevCounters* ctr, cudaStream_t st, int* resident) {
    using CF = StairCfg<LANES, VEC, WF, NS>;
    constexpr int bytes = CF::kBlockBytes;
    auto* kern = k1s_stair<LANES, VEC, WF, NS, FAST>;
    static std::atomic<uint64_t> configured{0};
    if (cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), bytes, configured); e != cudaSuccess)
        return e;
    constexpr int threads = CF::THREADS;
    if (resident != nullptr) return resident_sentences(kern, bytes, threads, threads / LANES, resident);
    const int blocks = k1s_grid(b, threads / LANES);
    if (blocks == 0) return cudaSuccess;
    kern<<<blocks, threads, bytes, st>>>(m, b, ctr);
    return cudaGetLastError();
}

} // namespace fw2v
