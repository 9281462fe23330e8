// FULL-W2V SGNS training kernels for B200 (sm_100a).
//
// K1  k1_lifetime   — the performance path (Hogwild across sentences). One
//                     lane group (LANES lanes, LANES | 32) owns one sentence;
//                     each lane owns VEC contiguous columns of every row. The
//                     2*W_f+1 ring of syn0 rows (reference ContextRing,
//                     trainer.cpp:32-102) lives in registers for the sentence's
//                     whole lifetime and slides by register renaming; each
//                     sample row (target + N negatives, syn1) is register-
//                     resident across its sweep over the 2*W_f context rows
//                     (sweep_samples, trainer.cpp:133-154) and the next sweep's
//                     row is prefetched while the current one runs. Dots are
//                     LANES-wide xor-butterfly reductions; no tensor cores
//                     (per-pair contractions are d-long and latency bound).
//                     Per-sentence arithmetic order = reference order
//                     (samples outer, contexts inner, incremental updates);
//                     only the dot association and sigmoid differ.
// K2  k2_exact      — the deterministic / exact engine: a warp restates the
//                     reference FP contract bit for bit (4 strided partial sums,
//                     no FMA, double-precision exp sigmoid; kernels.hpp:10-33,
//                     model.cpp:34-37) and every reuse mode's access order
//                     (trainer.cpp:237-328). serial=1 runs all sentences of a
//                     batch in order on one warp (== reference workers=1).
// Kinit             — init_model (model.cpp:15-32) as a counter-based kernel:
//                     splitmix64 draw i is mix(state0 + (i+1)*golden).
#include <cuda_runtime.h>

#include <cstdint>

#include "fw2v_device.cuh"
#include "fw2v_common.cuh"

namespace fw2v {

// ---------------------------------------------------------------- K1 kernel
template <int LANES, int VEC, int WF, bool FAST>
__global__ void __launch_bounds__(kK1Threads)
k1_lifetime(ModelView m, BatchView b, int n_neg, DevCounters* __restrict__ ctr) {
    constexpr int NCTX = 2 * WF;
    constexpr int GPW = 32 / LANES;
    const int lane = threadIdx.x & 31;
    const int sub = lane & (LANES - 1);
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int sent = warp * GPW + lane / LANES;
    const bool has = sent < b.n_sentences;

    uint32_t beg = 0, len = 0;
    float alpha = 0.0f;
    if (has) {
        beg = __ldg(b.offsets + sent);
        len = __ldg(b.offsets + sent + 1) - beg;
        alpha = __ldg(b.alpha + sent);
    }
    const int L = static_cast<int>(len);
    const int Lmax = static_cast<int>(__reduce_max_sync(kFull, len));
    if (Lmax == 0) return;  // warp-uniform

    const int32_t* __restrict__ ids = b.ids + beg;
    const int32_t* __restrict__ negs = b.negs + static_cast<size_t>(beg) * n_neg;
    const size_t stride = static_cast<size_t>(m.stride);
    float* __restrict__ syn0 = m.syn0 + sub * VEC;
    float* __restrict__ syn1 = m.syn1 + sub * VEC;
    // Positions >= tail stay resident until ContextRing::finish, which writes
    // them in slot order; they are parked in shared memory until then.
    constexpr int C = NCTX + 1;
    extern __shared__ __align__(16) float k1_sh[];
    float* stash = k1_sh + (threadIdx.x / LANES) * (2 * C * LANES * VEC) + sub * VEC;
    float* entry = stash + C * LANES * VEC;  // ring rows as loaded (delta write-back)
    const bool delta_wb = (m.flags & kFlagDeltaRing) != 0;
    const int tail = L - C;

    // Window-relative ring: ctx[r] holds position i-WF+r (r < WF) or
    // i+1+(r-WF) (r >= WF); tgt holds position i. tok = -1 outside [0, L).
    float ctx[NCTX][VEC];
    int tok[NCTX];
    float tgt[VEC];
    int ttok = L > 0 ? __ldg(ids) : -1;
    if (ttok >= 0) Row<VEC>::load(tgt, syn0 + ttok * stride); else vzero(tgt);
    if (delta_wb) stash_put(entry, tgt);
#pragma unroll
    for (int r = 0; r < NCTX; ++r) {
        const int p = r - WF + 1;
        tok[r] = (r >= WF && p < L) ? __ldg(ids + p) : -1;
        if (tok[r] >= 0) Row<VEC>::load(ctx[r], syn0 + tok[r] * stride); else vzero(ctx[r]);
        if (delta_wb && r >= WF) stash_put(entry + p * (LANES * VEC), ctx[r]);
    }
    unsigned c_reads = static_cast<unsigned>(min(L, WF + 1));
    unsigned c_writes = 0, s_rw = 0, pairs = 0;

    // Sample pipeline: nxt holds the prefetched row of the upcoming sweep.
    float s[VEC], nxt[VEC];
    int nxt_sid = L >= 2 ? ttok : -1;
    if (nxt_sid >= 0) Row<VEC>::load(nxt, syn1 + nxt_sid * stride); else vzero(nxt);
    vzero(s);
    int prev_sid = -1;

    for (int i = 0; i < Lmax; ++i) {
        const bool act = i < L;
        const bool wact = act && L >= 2;
        if (sub == 0 && act) obs_record(b, sent, i);
        // Row entering the span for window i+1 (ContextRing::advance, trainer.cpp:55-69).
        const int q = i + 1 + WF;
        const int inc_tok = q < L ? __ldg(ids + q) : -1;
        float inc[VEC];
        if (inc_tok >= 0) Row<VEC>::load(inc, syn0 + inc_tok * stride); else vzero(inc);
        c_reads += inc_tok >= 0;

        for (int k = 0; k <= n_neg; ++k) {
            const int sid = nxt_sid;
            // The prefetch was issued before the previous sweep wrote its row
            // back: forward the register copy when both sweeps hit one row.
            if (sid != prev_sid) vcopy(s, nxt);
            float s0[VEC];  // row as read, for the delta write-back
            vcopy(s0, s);
            // Prefetch the next sweep's row: (i, k+1) or (i+1, 0).
            {
                const bool same_win = k < n_neg;
                const int ni = same_win ? i : i + 1;
                const bool nact = ni < L && L >= 2;
                int ns = -1;
                if (nact) ns = same_win ? __ldg(negs + static_cast<size_t>(i) * n_neg + k) : tok[WF];
                nxt_sid = ns;
                if (ns >= 0) Row<VEC>::load(nxt, syn1 + ns * stride);
            }
            const float label = k == 0 ? 1.0f : 0.0f;
#pragma unroll
            for (int r = 0; r < NCTX; ++r) {
                float part = 0.0f;
#pragma unroll
                for (int e = 0; e < VEC; ++e) part = fmaf(ctx[r][e], s[e], part);
                const float f = group_sum<LANES>(part);
                const bool valid = wact && tok[r] >= 0;
                const float g = valid ? sgd_coeff<FAST>(f, label, alpha) : 0.0f;
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    const float c = ctx[r][e];
                    ctx[r][e] = fmaf(g, s[e], c);
                    s[e] = fmaf(g, c, s[e]);
                }
                pairs += valid;
            }
            if (wact) {
                if (delta_wb) red_add_delta(syn1 + sid * stride, s, s0);
                else Row<VEC>::store(syn1 + sid * stride, s);
            }
            s_rw += wact;
            prev_sid = wact ? sid : -1;
        }

        // Slide: position i-WF leaves the span and is written back.
        const int etok = tok[0];
        if (etok >= 0) {
            const int p = i - WF;
            if (delta_wb) {
                float e0[VEC];
                stash_get(e0, entry + (p % C) * (LANES * VEC));
                red_add_delta(syn0 + etok * stride, ctx[0], e0);
            } else if (p >= tail) {
                stash_put(stash + (p % C) * (LANES * VEC), ctx[0]);
            } else {
                Row<VEC>::store(syn0 + etok * stride, ctx[0]);
            }
            ++c_writes;
            if (inc_tok == etok) vcopy(inc, ctx[0]);  // load-after-evict forwarding
        }
        if (delta_wb && inc_tok >= 0) stash_put(entry + ((i + 1 + WF) % C) * (LANES * VEC), inc);
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
    }
    // ContextRing::finish (trainer.cpp:71-75): residents written in slot order
    // (deltas commute, so delta write-back needs no ordering).
#pragma unroll
    for (int r = 0; r < NCTX; ++r) {
        const int p = r < WF ? Lmax - WF + r : Lmax + 1 + (r - WF);
        if (tok[r] >= 0) {
            if (delta_wb) {
                float e0[VEC];
                stash_get(e0, entry + (p % C) * (LANES * VEC));
                red_add_delta(syn0 + tok[r] * stride, ctx[r], e0);
            } else {
                stash_put(stash + (p % C) * (LANES * VEC), ctx[r]);
            }
            ++c_writes;
        }
    }
    if (ttok >= 0) {
        if (delta_wb) {
            float e0[VEC];
            stash_get(e0, entry + (Lmax % C) * (LANES * VEC));
            red_add_delta(syn0 + ttok * stride, tgt, e0);
        } else {
            stash_put(stash + (Lmax % C) * (LANES * VEC), tgt);
        }
        ++c_writes;
    }
    if (!delta_wb) {
        const int first = max(0, tail);
        for (int s = 0; s < C; ++s) {
            const int p = first + ((s - first % C) + C) % C;
            if (p < L) {
                float v[VEC];
                stash_get(v, stash + s * (LANES * VEC));
                Row<VEC>::store(syn0 + __ldg(ids + p) * stride, v);
            }
        }
    }

    if (ctr != nullptr) {
        // One count per sentence: lane 0 of each group contributes.
        const bool lead = has && sub == 0;
        unsigned hits = (L >= 2) ? pairs - static_cast<unsigned>(L) : 0u;
        unsigned v0 = __reduce_add_sync(kFull, lead ? c_reads : 0u);
        unsigned v1 = __reduce_add_sync(kFull, lead ? c_writes : 0u);
        unsigned v2 = __reduce_add_sync(kFull, lead ? s_rw : 0u);
        unsigned v4 = __reduce_add_sync(kFull, lead ? hits : 0u);
        unsigned v5 = __reduce_add_sync(kFull, lead ? static_cast<unsigned>(L) : 0u);
        unsigned v6 = __reduce_add_sync(kFull, lead ? 1u : 0u);
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

// ---------------------------------------------------------------- K2 kernel
// Bit-exact restatement of the reference arithmetic (default -O2 build: no
// FMA; dot = 4 strided partial sums, kernels.hpp:10-22; update c+g*s and
// s+g*c from pairing-entry values, kernels.hpp:26-33; sigmoid in double,
// model.cpp:34-37).

// Warp-cooperative dot in the reference association: lane m (< 4) runs
// partial sum m sequentially; lane 0 folds (s0+s1)+(s2+s3) and the tail.
__device__ __forceinline__ float dot_exact(const float* a, const float* b, int d, int lane) {
    float sm = 0.0f;
    const int d4 = d & ~3;
    if (lane < 4) {
        for (int k = lane; k < d4; k += 4) sm = __fadd_rn(sm, __fmul_rn(a[k], b[k]));
    }
    const float s1 = __shfl_down_sync(kFull, sm, 1);
    const float s2 = __shfl_down_sync(kFull, sm, 2);
    const float s3 = __shfl_down_sync(kFull, sm, 3);
    float s = __fadd_rn(__fadd_rn(sm, s1), __fadd_rn(s2, s3));
    if (lane == 0) {
        for (int k = d4; k < d; ++k) s = __fadd_rn(s, __fmul_rn(a[k], b[k]));
    }
    return __shfl_sync(kFull, s, 0);
}

__device__ __forceinline__ float sigmoid_exact(float x) {
    const float c = x < -6.0f ? -6.0f : (6.0f < x ? 6.0f : x);  // std::clamp
    return static_cast<float>(1.0 / (1.0 + exp(-static_cast<double>(c))));
}

__device__ __forceinline__ float coeff_exact(float f, float label, float alpha) {
    return __fmul_rn(__fsub_rn(label, sigmoid_exact(f)), alpha);
}

__device__ __forceinline__ void pair_update_exact(float* c, float* s, float g, int d, int lane) {
    for (int k = lane; k < d; k += 32) {
        const float cv = c[k], sv = s[k];
        c[k] = __fadd_rn(cv, __fmul_rn(g, sv));
        s[k] = __fadd_rn(sv, __fmul_rn(g, cv));
    }
}

__device__ __forceinline__ void axpy_exact(float* y, const float* x, float g, int d, int lane) {
    for (int k = lane; k < d; k += 32) y[k] = __fadd_rn(y[k], __fmul_rn(g, x[k]));
}

__device__ __forceinline__ void row_get(float* dst, const float* src, int d, int lane) {
    for (int k = lane; k < d; k += 32) dst[k] = __ldcg(src + k);
}
__device__ __forceinline__ void row_put(float* dst, const float* src, int d, int lane) {
    for (int k = lane; k < d; k += 32) __stcg(dst + k, src[k]);
}

constexpr int kMaxRing = 2 * 16 + 1;

// smem layout (floats): ring[C*d] sample[d] a[(2WF)*d] b[(N+1)*d] c[(2WF)*d] e[(N+1)*d]
__global__ void __launch_bounds__(32)
k2_exact(ModelView m, BatchView b, int n_neg, int wf, int mode, int serial,
         DevCounters* __restrict__ ctr) {
    extern __shared__ float sh[];
    __shared__ int slot_pos[kMaxRing];
    __shared__ int slot_used[kMaxRing];
    __shared__ int ctx_pos[2 * 16];
    const int lane = threadIdx.x;
    const int d = m.dim;
    const int cap = 2 * wf + 1;
    const size_t stride = static_cast<size_t>(m.stride);
    float* ring = sh;
    float* sample = ring + cap * d;
    float* snap_ctx = sample + d;             // also window-mode local copies
    float* snap_smp = snap_ctx + 2 * wf * d;
    float* delta_ctx = snap_smp + (n_neg + 1) * d;
    float* delta_smp = delta_ctx + 2 * wf * d;

    unsigned long long cr = 0, cw = 0, sr = 0, sw = 0, hits = 0, words = 0, nsent = 0;

    const int first = serial ? 0 : blockIdx.x;
    const int last = serial ? b.n_sentences : min(b.n_sentences, static_cast<int>(blockIdx.x) + 1);
    for (int sidx = first; sidx < last; ++sidx) {
        const uint32_t beg = b.offsets[sidx];
        const int L = static_cast<int>(b.offsets[sidx + 1] - beg);
        const int32_t* ids = b.ids + beg;
        const int32_t* negs = b.negs + static_cast<size_t>(beg) * n_neg;
        const float alpha = b.alpha[sidx];
        words += L;
        nsent += 1;
        auto in_row = [&](int pos) { return m.syn0 + ids[pos] * stride; };
        auto out_row = [&](int id) { return m.syn1 + id * stride; };

        if (mode == kLifetime || mode == kWindowSnapshot) {
            // train_sentence_ring (trainer.cpp:237-255) with ContextRing.
            if (lane < cap) { slot_pos[lane] = -1; slot_used[lane] = 0; }
            __syncwarp();
            int next_load = 0;
            for (int i = 0; i < L; ++i) {
                if (lane == 0) obs_record(b, sidx, i);
                const int hi = min(L - 1, i + wf);  // advance (trainer.cpp:55-69)
                while (next_load <= hi) {
                    const int slot = next_load % cap;
                    if (slot_pos[slot] >= 0) {
                        row_put(in_row(slot_pos[slot]), ring + slot * d, d, lane);
                        ++cw;
                    }
                    row_get(ring + slot * d, in_row(next_load), d, lane);
                    ++cr;
                    __syncwarp();
                    if (lane == 0) { slot_pos[slot] = next_load; slot_used[slot] = 0; }
                    __syncwarp();
                    ++next_load;
                }
                const int lo = max(0, i - wf), hh = min(L - 1, i + wf);
                int n_ctx = 0;
                for (int j = lo; j <= hh; ++j)
                    if (j != i) { if (lane == 0) ctx_pos[n_ctx] = j; ++n_ctx; }
                __syncwarp();
                if (n_ctx == 0) continue;
                const int target = ids[i];
                if (mode == kLifetime) {
                    for (int k = 0; k <= n_neg; ++k) {  // sweep_samples (trainer.cpp:133-154)
                        const int sid = k == 0 ? target : negs[static_cast<size_t>(i) * n_neg + k - 1];
                        const float label = k == 0 ? 1.0f : 0.0f;
                        row_get(sample, out_row(sid), d, lane);
                        ++sr;
                        __syncwarp();
                        for (int j = 0; j < n_ctx; ++j) {
                            const int slot = ctx_pos[j] % cap;
                            if (slot_used[slot]) ++hits;
                            __syncwarp();
                            if (lane == 0) slot_used[slot] = 1;
                            float* cv = ring + slot * d;
                            const float f = dot_exact(cv, sample, d, lane);
                            const float g = coeff_exact(f, label, alpha);
                            pair_update_exact(cv, sample, g, d, lane);
                            __syncwarp();
                        }
                        row_put(out_row(sid), sample, d, lane);
                        ++sw;
                        __syncwarp();
                    }
                } else {  // sweep_samples_snapshot (trainer.cpp:158-205)
                    const int S = n_neg + 1;
                    for (int j = 0; j < n_ctx; ++j)
                        for (int e = lane; e < d; e += 32) snap_ctx[j * d + e] = ring[(ctx_pos[j] % cap) * d + e];
                    for (int k = 0; k < S; ++k) {
                        const int sid = k == 0 ? target : negs[static_cast<size_t>(i) * n_neg + k - 1];
                        row_get(snap_smp + k * d, out_row(sid), d, lane);
                        ++sr;
                    }
                    for (int e = lane; e < n_ctx * d; e += 32) delta_ctx[e] = 0.0f;
                    for (int e = lane; e < S * d; e += 32) delta_smp[e] = 0.0f;
                    __syncwarp();
                    for (int k = 0; k < S; ++k) {
                        const float label = k == 0 ? 1.0f : 0.0f;
                        for (int j = 0; j < n_ctx; ++j) {
                            const int slot = ctx_pos[j] % cap;
                            if (slot_used[slot]) ++hits;
                            __syncwarp();
                            if (lane == 0) slot_used[slot] = 1;
                            const float* cv = snap_ctx + j * d;
                            const float* smp = snap_smp + k * d;
                            const float f = dot_exact(cv, smp, d, lane);
                            const float g = coeff_exact(f, label, alpha);
                            axpy_exact(delta_ctx + j * d, smp, g, d, lane);
                            axpy_exact(delta_smp + k * d, cv, g, d, lane);
                            __syncwarp();
                        }
                    }
                    for (int j = 0; j < n_ctx; ++j) {
                        float* cv = ring + (ctx_pos[j] % cap) * d;
                        for (int e = lane; e < d; e += 32) cv[e] = __fadd_rn(cv[e], delta_ctx[j * d + e]);
                        __syncwarp();
                    }
                    for (int k = 0; k < S; ++k) {
                        const int sid = k == 0 ? target : negs[static_cast<size_t>(i) * n_neg + k - 1];
                        float* row = out_row(sid);
                        for (int e = lane; e < d; e += 32) __stcg(row + e, __fadd_rn(__ldcg(row + e), delta_smp[k * d + e]));
                        ++sw;
                        __syncwarp();
                    }
                }
            }
            for (int s = 0; s < cap; ++s) {  // finish (trainer.cpp:71-75), slot order
                if (slot_pos[s] >= 0) {
                    row_put(in_row(slot_pos[s]), ring + s * d, d, lane);
                    ++cw;
                }
            }
            __syncwarp();
        } else if (mode == kWindow) {
            // train_sentence_window (trainer.cpp:257-290)
            for (int i = 0; i < L; ++i) {
                if (lane == 0) obs_record(b, sidx, i);
                const int lo = max(0, i - wf), hh = min(L - 1, i + wf);
                int n_ctx = 0;
                for (int j = lo; j <= hh; ++j)
                    if (j != i) { if (lane == 0) ctx_pos[n_ctx] = j; ++n_ctx; }
                __syncwarp();
                if (n_ctx == 0) continue;
                for (int j = 0; j < n_ctx; ++j) { row_get(snap_ctx + j * d, in_row(ctx_pos[j]), d, lane); ++cr; }
                __syncwarp();
                const int target = ids[i];
                for (int k = 0; k <= n_neg; ++k) {
                    const int sid = k == 0 ? target : negs[static_cast<size_t>(i) * n_neg + k - 1];
                    const float label = k == 0 ? 1.0f : 0.0f;
                    row_get(sample, out_row(sid), d, lane);
                    ++sr;
                    __syncwarp();
                    for (int j = 0; j < n_ctx; ++j) {
                        float* cv = snap_ctx + j * d;
                        const float f = dot_exact(cv, sample, d, lane);
                        const float g = coeff_exact(f, label, alpha);
                        pair_update_exact(cv, sample, g, d, lane);
                        __syncwarp();
                    }
                    row_put(out_row(sid), sample, d, lane);
                    ++sw;
                    __syncwarp();
                }
                hits += static_cast<unsigned long long>(n_ctx) * n_neg;
                for (int j = 0; j < n_ctx; ++j) {
                    row_put(in_row(ctx_pos[j]), snap_ctx + j * d, d, lane);
                    ++cw;
                    __syncwarp();
                }
            }
        } else {
            // train_sentence_direct (trainer.cpp:292-328)
            for (int i = 0; i < L; ++i) {
                if (lane == 0) obs_record(b, sidx, i);
                const int lo = max(0, i - wf), hh = min(L - 1, i + wf);
                int n_ctx = 0;
                for (int j = lo; j <= hh; ++j)
                    if (j != i) { if (lane == 0) ctx_pos[n_ctx] = j; ++n_ctx; }
                __syncwarp();
                if (n_ctx == 0) continue;
                const int target = ids[i];
                for (int k = 0; k <= n_neg; ++k) {
                    const int sid = k == 0 ? target : negs[static_cast<size_t>(i) * n_neg + k - 1];
                    const float label = k == 0 ? 1.0f : 0.0f;
                    for (int j = 0; j < n_ctx; ++j) {
                        row_get(sample, out_row(sid), d, lane);
                        ++sr;
                        row_get(snap_ctx, in_row(ctx_pos[j]), d, lane);
                        ++cr;
                        __syncwarp();
                        const float f = dot_exact(snap_ctx, sample, d, lane);
                        const float g = coeff_exact(f, label, alpha);
                        pair_update_exact(snap_ctx, sample, g, d, lane);
                        __syncwarp();
                        row_put(in_row(ctx_pos[j]), snap_ctx, d, lane);
                        ++cw;
                        row_put(out_row(sid), sample, d, lane);
                        ++sw;
                        __syncwarp();
                    }
                }
            }
        }
    }
    if (ctr != nullptr && lane == 0) {
        atomicAdd(&ctr->context_reads, cr);
        atomicAdd(&ctr->context_writes, cw);
        atomicAdd(&ctr->sample_reads, sr);
        atomicAdd(&ctr->sample_writes, sw);
        atomicAdd(&ctr->ring_hits, hits);
        atomicAdd(&ctr->words, words);
        atomicAdd(&ctr->sentences, nsent);
    }
}

// ------------------------------------------------------------- init kernel
__device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// init_model (model.cpp:15-32): input[i] = (next_float() - 0.5f) * (1/d),
// draw i of the "init" stream; output = 0; padding columns = 0.
__global__ void k_init_model(ModelView m, uint64_t state0) {
    const size_t n = static_cast<size_t>(m.vocab) * m.stride;
    const float inv_dim = 1.0f / static_cast<float>(m.dim);
    for (size_t x = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; x < n;
         x += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t w = x / m.stride;
        const int col = static_cast<int>(x - w * m.stride);
        float v = 0.0f;
        if (col < m.dim) {
            const uint64_t i = w * static_cast<uint64_t>(m.dim) + col;
            const uint64_t u = splitmix_mix(state0 + (i + 1) * 0x9e3779b97f4a7c15ULL);
            const float nf = __fmul_rn(static_cast<float>(u >> 40), 0x1.0p-24f);
            v = __fmul_rn(__fsub_rn(nf, 0.5f), inv_dim);
        }
        m.syn0[x] = v;
        m.syn1[x] = 0.0f;
    }
}

// --------------------------------------------------------------- dispatch
struct K1Shape {
    int lanes, vec;
};

template <int LANES, int VEC, int WF>
cudaError_t launch_k1_wf(const ModelView& m, const BatchView& b, int n_neg, bool fast,
                         DevCounters* ctr, cudaStream_t st, int* resident) {
    constexpr int GPW = 32 / LANES;
    const int warps = (b.n_sentences + GPW - 1) / GPW;
    const int blocks = (warps * 32 + kK1Threads - 1) / kK1Threads;
    constexpr int bytes = 2 * kK1Threads * (2 * WF + 1) * VEC * 4;  // finish stash + ring entry values
    auto* kern = fast ? k1_lifetime<LANES, VEC, WF, true> : k1_lifetime<LANES, VEC, WF, false>;
    if (bytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) return e;
    }
    if (resident != nullptr) return resident_sentences(kern, bytes, kK1Threads, kK1Threads / LANES, resident);
    if (blocks == 0) return cudaSuccess;
    kern<<<blocks, kK1Threads, bytes, st>>>(m, b, n_neg, ctr);
    return cudaGetLastError();
}

template <int LANES, int VEC>
cudaError_t launch_k1_shape(const ModelView& m, const BatchView& b, int n_neg, int wf, bool fast,
                            DevCounters* ctr, cudaStream_t st, int* resident) {
    switch (wf) {
    case 1: return launch_k1_wf<LANES, VEC, 1>(m, b, n_neg, fast, ctr, st, resident);
    case 2: return launch_k1_wf<LANES, VEC, 2>(m, b, n_neg, fast, ctr, st, resident);
    case 3: return launch_k1_wf<LANES, VEC, 3>(m, b, n_neg, fast, ctr, st, resident);
    case 4: return launch_k1_wf<LANES, VEC, 4>(m, b, n_neg, fast, ctr, st, resident);
    case 5: return launch_k1_wf<LANES, VEC, 5>(m, b, n_neg, fast, ctr, st, resident);
    default: return cudaErrorInvalidValue;
    }
}

#define FW2V_K1_SHAPES(X) \
    X(4, 1) X(4, 2) X(4, 4) X(8, 4) X(16, 4) X(8, 8) X(32, 4) X(16, 8) X(8, 16) \
    X(32, 6) X(32, 8) X(32, 10) X(32, 12) X(32, 16)

cudaError_t launch_k1(int lanes, int vec, const ModelView& m, const BatchView& b, int n_neg, int wf,
                      bool fast, DevCounters* ctr, cudaStream_t st, int* resident) {
#define FW2V_CASE(L_, V_) \
    if (lanes == L_ && vec == V_) return launch_k1_shape<L_, V_>(m, b, n_neg, wf, fast, ctr, st, resident);
    FW2V_K1_SHAPES(FW2V_CASE)
#undef FW2V_CASE
    return cudaErrorInvalidValue;
}

bool k1_shape_supported(int lanes, int vec) {
#define FW2V_CASE(L_, V_) if (lanes == L_ && vec == V_) return true;
    FW2V_K1_SHAPES(FW2V_CASE)
#undef FW2V_CASE
    return false;
}

size_t k2_smem_bytes(int dim, int wf, int n_neg) {
    const int cap = 2 * wf + 1;
    return sizeof(float) * static_cast<size_t>(dim) * (cap + 1 + 2 * (2 * wf) + 2 * (n_neg + 1));
}

cudaError_t launch_k2(const ModelView& m, const BatchView& b, int n_neg, int wf, int mode, bool serial,
                      DevCounters* ctr, cudaStream_t st) {
    if (wf < 1 || 2 * wf + 1 > kMaxRing) return cudaErrorInvalidValue;
    if (b.n_sentences == 0) return cudaSuccess;
    const size_t smem = k2_smem_bytes(m.dim, wf, n_neg);
    // The attribute is per device: always raise it for sizes above 48 KB (K2 runs
    // one launch per batch, so the driver call is negligible).
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k2_exact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    const int grid = serial ? 1 : b.n_sentences;
    k2_exact<<<grid, 32, smem, st>>>(m, b, n_neg, wf, mode, serial ? 1 : 0, ctr);
    return cudaGetLastError();
}

cudaError_t launch_init_model(const ModelView& m, uint64_t state0, cudaStream_t st) {
    k_init_model<<<148 * 8, 256, 0, st>>>(m, state0);
    return cudaGetLastError();
}

// Divergence guard: *flag |= 1 if any of the n floats at p is not finite or
// exceeds kDiverged in magnitude (a Hogwild run that blew up: SGNS embeddings
// stay O(1-10); one read of the matrix, 16-byte loads, grid sized to the SMs).
constexpr float kDiverged = 1e6f;
__global__ void k_nonfinite(const float4* __restrict__ p, size_t n4, int* flag) {
    bool bad = false;
    for (size_t x = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; x < n4;
         x += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const float4 v = __ldcg(p + x);
        // !(|v| < kDiverged) is also true for NaN
        bad |= !(fabsf(v.x) < kDiverged && fabsf(v.y) < kDiverged && fabsf(v.z) < kDiverged && fabsf(v.w) < kDiverged);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}
cudaError_t launch_nonfinite(const float* p, size_t n, int* flag, cudaStream_t st) {
    if (n % 4 != 0) return cudaErrorInvalidValue;  // rows are padded to a multiple of 4 floats
    k_nonfinite<<<148 * 4, 256, 0, st>>>(reinterpret_cast<const float4*>(p), n / 4, flag);
    return cudaGetLastError();
}

// Hot-row replicas (ModelView::hot): broadcast output rows 0..K-1 into every
// replica before a Hogwild pass, and average the replicas back after it.
__global__ void k_hot_broadcast(ModelView m) {
    const int n = m.hot_k * m.stride;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
        const float v = m.syn1[x];
        for (int r = 0; r < m.hot_r; ++r) m.hot[static_cast<size_t>(r) * n + x] = v;
    }
}
__global__ void k_hot_average(ModelView m) {
    const int n = m.hot_k * m.stride;
    const float inv = 1.0f / static_cast<float>(m.hot_r);
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
        float s = 0.0f;
        for (int r = 0; r < m.hot_r; ++r) s += m.hot[static_cast<size_t>(r) * n + x];
        m.syn1[x] = s * inv;
    }
}
// Live hot-row merge (fw2v_config.hot_merge = 1): one resident block keeps the
// base (syn1 rows 0..K-1) equal to the sum of every replica's updates and hands
// each replica the others' updates, sweeping until *stop: replica r gets
// red.add(D - d_r) with d_r = its own change since the last sweep and D = the sum
// over replicas, so an update reaches every replica within a sweep (~µs, like a
// plain Hogwild update reaching L2) and the hot rows take plain Hogwild's full
// step instead of the mean's 1/R. red.add keeps updates that land between the
// sweep's read and its write. *started tells the host the block is resident.
constexpr int kMaxLiveReplicas = 16;
__global__ void __launch_bounds__(512) k_hot_live(ModelView m, const volatile int* stop, volatile int* started,
                                                  unsigned sleep_ns, unsigned long long max_ns) {
    const int n4 = m.hot_k * m.stride / 4;
    float4* base = reinterpret_cast<float4*>(m.syn1);
    float4* rep = reinterpret_cast<float4*>(m.hot);
    const int R = m.hot_r;
    __shared__ int last;
    unsigned long long t0 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0) *started = 1;
    // Leaves when stopped, when no training sentence has started for kIdleNs (the
    // pass's kernels are not running beside it: the host's final sweep catches up),
    // or after max_ns (never outlive a lost stop).
    constexpr unsigned long long kIdleNs = 20ull * 1000 * 1000;
    unsigned seen = m.beat != nullptr ? *reinterpret_cast<volatile unsigned*>(m.beat) : 0u;
    unsigned long long t_seen = t0;
    for (;;) {
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (m.beat != nullptr) {
                const unsigned b = *reinterpret_cast<volatile unsigned*>(m.beat);
                if (b != seen) { seen = b; t_seen = t; }
            }
            last = (*stop != 0) || (t - t0 > max_ns) || (m.beat != nullptr && t - t_seen > kIdleNs);
        }
        __syncthreads();
        const bool fin = last != 0;
        for (int x = threadIdx.x; x < n4; x += blockDim.x) {
            const float4 b = __ldcg(base + x);
            float4 d[kMaxLiveReplicas];
            float4 D = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
            for (int r = 0; r < kMaxLiveReplicas; ++r) {
                if (r < R) {
                    const float4 v = __ldcg(rep + static_cast<size_t>(r) * n4 + x);
                    d[r] = make_float4(v.x - b.x, v.y - b.y, v.z - b.z, v.w - b.w);
                    D.x += d[r].x; D.y += d[r].y; D.z += d[r].z; D.w += d[r].w;
                }
            }
            if (D.x == 0.0f && D.y == 0.0f && D.z == 0.0f && D.w == 0.0f) continue;
#pragma unroll
            for (int r = 0; r < kMaxLiveReplicas; ++r) {
                if (r < R)
                    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(rep + static_cast<size_t>(r) * n4 + x),
                                 "f"(D.x - d[r].x), "f"(D.y - d[r].y), "f"(D.z - d[r].z), "f"(D.w - d[r].w)
                                 : "memory");
            }
            __stcg(base + x, make_float4(b.x + D.x, b.y + D.y, b.z + D.z, b.w + D.w));
        }
        __syncthreads();
        if (fin) break;
        __nanosleep(sleep_ns);
    }
}
__global__ void k_set_flag(int* f) { *f = 1; }
cudaError_t launch_hot_live(const ModelView& m, int* stop, int* started, cudaStream_t st) {
    if (m.hot_k <= 0 || m.hot_r > kMaxLiveReplicas) return cudaErrorInvalidValue;
    k_hot_live<<<1, 512, 0, st>>>(m, stop, started, 2000u, 10ull * 1000 * 1000 * 1000);
    return cudaGetLastError();
}
cudaError_t launch_set_flag(int* f, cudaStream_t st) {
    k_set_flag<<<1, 1, 0, st>>>(f);
    return cudaGetLastError();
}

cudaError_t launch_hot_sync(const ModelView& m, bool average, cudaStream_t st) {
    if (m.hot_k <= 0) return cudaSuccess;
    const int n = m.hot_k * m.stride;
    const int blocks = (n + 255) / 256;
    if (average) k_hot_average<<<blocks, 256, 0, st>>>(m);
    else k_hot_broadcast<<<blocks, 256, 0, st>>>(m);
    return cudaGetLastError();
}

// Replica average over peer memory (fw2v_average without NCCL: contexts that
// share a device, or FW2V_AVERAGE=peer). Launched once per member g on g's own
// device: member g owns elements [begin, end) and reads that slice of every
// replica (NVLink P2P loads for remote ones), writes the mean back into every
// replica. Slices are disjoint, so the members' launches need no ordering
// among themselves; the host quiesces training before and joins after.
// begin, end: multiples of 4 (row strides are), replicas 16-byte aligned.
__global__ void k_average_slice(PeerSet ps, size_t begin, size_t end) {
    const float inv = 1.0f / static_cast<float>(ps.n);
    const size_t nth = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t x = begin / 4 + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; x < end / 4; x += nth) {
        float4 s = reinterpret_cast<const float4*>(ps.ptr[0])[x];
        for (int r = 1; r < ps.n; ++r) {
            const float4 v = reinterpret_cast<const float4*>(ps.ptr[r])[x];
            s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
        }
        s.x *= inv; s.y *= inv; s.z *= inv; s.w *= inv;
        for (int r = 0; r < ps.n; ++r) reinterpret_cast<float4*>(ps.ptr[r])[x] = s;
    }
}
cudaError_t launch_average_slice(const PeerSet& ps, size_t begin, size_t end, cudaStream_t st) {
    if (end <= begin || ps.n < 1) return cudaSuccess;
    k_average_slice<<<148 * 4, 256, 0, st>>>(ps, begin, end);
    return cudaGetLastError();
}

// Replica merge of data-parallel rounds (fw2v_config.replica_merge), element
// by element, with b = the replicas' common value at the round start and
// d_r = v_r - b each replica's round delta:
//   mean     v = mean_r v_r                       (model averaging)
//   touched  v = b + sum_r d_r / #{r : d_r != 0}  (mean over the replicas that
//            changed the element: a row only one shard trained keeps its full
//            update; rows every shard trained get the mean)
// (Applying the summed deltas, b + sum_r d_r, diverges: +31% loss at 2 replicas
// and overflow at 8 on the text8 shape, profiles/r02_dp_merge_probe.txt.)
__device__ __forceinline__ float merge_value(int rule, float b, float sum_d, float cnt, float inv_n, float sum_v) {
    if (rule == kMergeMean) return sum_v * inv_n;
    return b + (cnt > 1.0f ? sum_d / cnt : sum_d);
}

// Fused peer-memory merge, member g's slice [begin, end) of every replica (see
// k_average_slice).
__global__ void k_merge_slice(PeerSet ps, float* base, int rule, size_t begin, size_t end) {
    const float inv = 1.0f / static_cast<float>(ps.n);
    const size_t nth = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t x = begin + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; x < end; x += nth) {
        const float b = base != nullptr ? base[x] : 0.0f;
        float sd = 0.0f, sv = 0.0f, c = 0.0f;
        for (int r = 0; r < ps.n; ++r) {
            const float v = ps.ptr[r][x];
            const float d = v - b;
            sv += v;
            sd += d;
            c += d != 0.0f ? 1.0f : 0.0f;
        }
        const float m = merge_value(rule, b, sd, c, inv, sv);
        for (int r = 0; r < ps.n; ++r) ps.ptr[r][x] = m;
        if (base != nullptr) base[x] = m;
    }
}
cudaError_t launch_merge_slice(const PeerSet& ps, float* base, int rule, size_t begin, size_t end, cudaStream_t st) {
    if (end <= begin || ps.n < 1) return cudaSuccess;
    k_merge_slice<<<148 * 4, 256, 0, st>>>(ps, base, rule, begin, end);
    return cudaGetLastError();
}

// Split merge around a SUM all-reduce (NCCL or the caller's exchange):
// prep turns a replica into what is summed (v itself for mean; d = v - b and,
// for touched, the indicator d != 0 into cnt), finish turns the sums into the
// merged value and makes it the next round's base.
__global__ void k_merge_prep(float* v, const float* base, float* cnt, int rule, size_t n) {
    const size_t nth = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t x = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; x < n; x += nth) {
        const float d = v[x] - base[x];
        v[x] = d;
        if (cnt != nullptr) cnt[x] = d != 0.0f ? 1.0f : 0.0f;
    }
}
__global__ void k_merge_finish(float* v, float* base, const float* cnt, int rule, float inv_n, size_t n) {
    const size_t nth = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t x = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; x < n; x += nth) {
        const float s = v[x];
        const float b = base != nullptr ? base[x] : 0.0f;
        const float m = merge_value(rule, b, s, cnt != nullptr ? cnt[x] : 0.0f, inv_n, s);
        v[x] = m;
        if (base != nullptr) base[x] = m;
    }
}
cudaError_t launch_merge_prep(float* v, const float* base, float* cnt, int rule, size_t n, cudaStream_t st) {
    if (rule == kMergeMean || n == 0) return cudaSuccess;
    k_merge_prep<<<148 * 4, 256, 0, st>>>(v, base, cnt, rule, n);
    return cudaGetLastError();
}
cudaError_t launch_merge_finish(float* v, float* base, const float* cnt, int rule, float inv_n, size_t n,
                                cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_merge_finish<<<148 * 4, 256, 0, st>>>(v, rule == kMergeMean ? nullptr : base, cnt, rule, inv_n, n);
    return cudaGetLastError();
}

} // namespace fw2v
