// K1s — the FULL-W2V window kernels for B200 (sm_100a, CUDA cores).
//
// Window-snapshot order (the paper's independent-negatives rule, PAPER.md:519-529;
// reference oracle sweep_samples_snapshot, trainer.cpp:158-205): every (sample,
// context) pairing of a window uses window-entry values, so the (N+1) x 2W_f dots
// are independent:
//   1. window i+1's N+1 sample rows (syn1) are staged by cp.async (through L1)
//      into shared memory while window i computes; rows the previous window
//      rewrote after their prefetch are found with one __match_any_sync and re-read;
//   2. all dots are formed per lane on its column slice with packed FFMA2
//      (fma.rn.f32x2) and reduced across the sentence's lane group by ONE
//      transposed butterfly (each level keeps half of the partial sums and ships
//      the other half: ~1 shuffle per dot); the top level is select-free because
//      lanes of the upper half read the sample rows in swapped order;
//   3. each lane evaluates the sigmoid of the dots it owns; g goes through shared
//      memory to the whole group;
//   4. sample deltas D_k = sum_r g_kr c_r (written as red.global.add, row += delta,
//      trainer.cpp:198-204) and context updates c_r += sum_k g_kr s_k.
// Lifetime order (LIFETIME = true; the reference default sweep_samples,
// trainer.cpp:133-154) runs the same window as an anti-diagonal wavefront with
// the sample rows in registers.
// The 2W_f+1 ring of syn0 rows (ContextRing, trainer.cpp:32-102) stays in
// registers for the sentence's lifetime and slides by register renaming; rows
// leave it by overwrite (no shared-memory ring), as red.add deltas, or — the
// exact mode — in the reference's write order with the finish() slot order.
// A lane group is 4-32 lanes of one warp (several sentences per warp), or at
// d = 512 the block's two warps (64 lanes x 8 columns): the butterfly runs per
// warp and the two halves' partial dots meet in a shared-memory exchange.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "fw2v_common.cuh"
#include "fw2v_device.cuh"

#ifdef KB_TIMING  // experiment: per-phase SM clocks of each warp, summed into kb_timing[]
__device__ unsigned long long kb_timing[16];
#define KB_T_DECL unsigned long long kbt[10] = {0}; long long kbt0 = clock64();
#define KB_T(k) { const long long t_ = clock64(); kbt[k] += t_ - kbt0; kbt0 = t_; }
#define KB_T_DUMP if (lane == 0) for (int k_ = 0; k_ < 9; ++k_) atomicAdd(&kb_timing[k_], kbt[k_]);
#else
#define KB_T_DECL
#define KB_T(k)
#define KB_T_DUMP
#endif

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

    // Same result when lanes with bit O set hold v[j] and v[j + H] swapped on
    // entry (their operands were loaded in swapped order): no selects at the top level.
    template <int CAP>
    __device__ __forceinline__ static void reduce_preswapped(float (&v)[CAP], int sub) {
        static_assert(N <= CAP && (N & 1) == 0, "butterfly overflow");
#pragma unroll
        for (int j = 0; j < H; ++j) v[j] += __shfl_xor_sync(kFull, v[j + H], O);
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

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
constexpr int kPrefetchWindows = 16;

// Window-snapshot order with more than NC samples keeps every sample row of the
// window in shared memory (read at window entry, before any of the window's
// reductions): up to kMaxSnapSamples = N + 1.
constexpr int kMaxSnapSamples = 16;

template <int LANES, int VEC, int WF, int NC, bool RING = true, bool LIFETIME = false, bool SNAPALL = false>
struct K1sSmem {
    static constexpr int NCTX = 2 * WF;
    static constexpr int C = 2 * WF + 1;
    static constexpr int NV = NC * NCTX;
    static constexpr int GPAD = (NV + 3) & ~3;
    static constexpr int STRIDE = LANES * VEC;
    // LANES = 64 (d = 512 as 64 x 8): one sentence on the block's two warps, each
    // owning half of the columns. Control logic and the butterfly run per warp
    // (CL lanes); the two warps' partial dots meet in a double-buffered exchange.
    static constexpr int CL = LANES > 32 ? 32 : LANES;
    static constexpr int NWG = LANES / CL;  // warps per group
    // exchange slots per lane: the butterfly's outputs, or a wavefront step's NC dots
    static constexpr int NFX = ((Butterfly<CL / 2, NV>::final_count() > NC ? Butterfly<CL / 2, NV>::final_count() : NC) + 3) & ~3;
    static constexpr int XB = NWG > 1 ? 2 * NWG * NFX * 32 : 0;
    static constexpr int GA = NWG * GPAD + XB;  // g areas (one per warp) + exchange
    // Wide lane slices (VEC >= 8) hold twice the registers per lane: 64-thread
    // blocks keep the per-block shared memory small enough for 5 blocks per SM.
    static constexpr int THREADS = VEC >= 8 ? 64 : kK1Threads;
    // Per group (one sentence): the window's g coefficients (scalars), the
    // sample rows double-buffered by window parity, and the ring rows as loaded
    // (delta write-back) or the finish() stash (overwrite) — never both.
    // RING = false (Hogwild overwrite write-back): ring rows leave straight to HBM,
    // no shared-memory ring: 64% of the footprint, 6 blocks per SM at d=128.
    // SNAPALL: every chunk's NC slots, the last chunk's unused ones included
    // (its dots read all NC slots; their g is 0).
    static constexpr int SNAP_ROWS = (kMaxSnapSamples + NC - 1) / NC * NC;
    static constexpr int SROWS = SNAPALL ? (SNAP_ROWS > 2 * NC ? SNAP_ROWS : 2 * NC) : 2 * NC;
    static constexpr int kGroupFloats = GA + SROWS * STRIDE + (RING ? C * STRIDE : 0);
    static constexpr int kBlockBytes = (THREADS / LANES) * kGroupFloats * 4;
    static constexpr int kSmemBlocks = (227 * 1024) / (kBlockBytes + 1024);
    // Register budget (blocks per SM the compiler must fit): 168 registers at
    // 8 columns per lane (6 x 64 threads without the ring), ~220 at 10-12 columns.
    // The register file is split between the 4 SMSPs (16K each): 5-6 blocks of
    // 2 warps put 3 warps on some SMSP, 170 registers; 4 blocks allow 255.
    // The lifetime wavefront keeps the window's sample rows in registers too.
    // (measured at d=128: 4 blocks / 255 registers 661 M words/s, 6 blocks with
    // spills 413).
    static constexpr int kRegBlocks = VEC < 8 ? 3 : VEC > 8 || LIFETIME ? 4 : (RING ? 5 : 6);
    static constexpr int MINB = kSmemBlocks < kRegBlocks ? (kSmemBlocks < 1 ? 1 : kSmemBlocks) : kRegBlocks;
};

// A lane's slice of a row: VEC = 2*H2 columns as chunks of CW floats (16 bytes
// when H2 is even, else 8 bytes, e.g. d=300 on 32 lanes x 10 columns) spaced
// CS = CW*LANES floats apart (chunk c of lane l at column CW*(c*LANES + l)), so
// one chunk access by a lane group covers a contiguous CW*4*LANES-byte span:
// coalesced in HBM/L2 and bank-conflict free in shared memory.
template <int H2, int LANES>
struct Slice {
    static constexpr int CW = H2 % 2 == 0 ? 4 : 2;
    static constexpr int CS = CW * LANES;
    static constexpr int NCH = 2 * H2 / CW;
    __device__ __forceinline__ static const float* chunk(const float* p, int c) { return p + c * CS; }
    __device__ __forceinline__ static void load(float2 (&v)[H2], const float* p) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            if constexpr (CW == 4) {
                const float4 t = __ldcg(reinterpret_cast<const float4*>(p + c * CS));
                v[2 * c] = make_float2(t.x, t.y);
                v[2 * c + 1] = make_float2(t.z, t.w);
            } else {
                v[c] = __ldcg(reinterpret_cast<const float2*>(p + c * CS));
            }
        }
    }
    __device__ __forceinline__ static void load_early(float2 (&v)[H2], const float* p) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            if constexpr (CW == 4) {
                const float4 t = ldcg_early(p + c * CS);
                v[2 * c] = make_float2(t.x, t.y);
                v[2 * c + 1] = make_float2(t.z, t.w);
            } else {
                asm volatile("ld.global.cg.v2.f32 {%0, %1}, [%2];" : "=f"(v[c].x), "=f"(v[c].y) : "l"(p + c * CS));
            }
        }
    }
    __device__ __forceinline__ static void store(float* p, const float2 (&v)[H2]) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            if constexpr (CW == 4)
                __stcg(reinterpret_cast<float4*>(p + c * CS), make_float4(v[2 * c].x, v[2 * c].y, v[2 * c + 1].x, v[2 * c + 1].y));
            else
                __stcg(reinterpret_cast<float2*>(p + c * CS), v[c]);
        }
    }
    __device__ __forceinline__ static void load_shared(float2 (&v)[H2], const float* p) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            if constexpr (CW == 4) {
                const float4 t = *reinterpret_cast<const float4*>(p + c * CS);
                v[2 * c] = make_float2(t.x, t.y);
                v[2 * c + 1] = make_float2(t.z, t.w);
            } else {
                v[c] = *reinterpret_cast<const float2*>(p + c * CS);
            }
        }
    }
    __device__ __forceinline__ static void store_shared(float* p, const float2 (&v)[H2]) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            if constexpr (CW == 4)
                *reinterpret_cast<float4*>(p + c * CS) = make_float4(v[2 * c].x, v[2 * c].y, v[2 * c + 1].x, v[2 * c + 1].y);
            else
                *reinterpret_cast<float2*>(p + c * CS) = v[c];
        }
    }
    __device__ __forceinline__ static void zero_shared(float* p) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            if constexpr (CW == 4) *reinterpret_cast<float4*>(p + c * CS) = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            else *reinterpret_cast<float2*>(p + c * CS) = make_float2(0.0f, 0.0f);
        }
    }
    // Stage the lane's slice of a global row into shared memory: through L1
    // (cp.async.ca), or with L2ONLY through L2 alone (cp.async.cg, 16-byte chunks:
    // every read sees every write that reached L2, the sentence's own included).
    static constexpr bool kCanL2Only = CW == 4;
    template <bool L2ONLY = false>
    __device__ __forceinline__ static void stage(float* dst, const float* src) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst + c * CS));
            if constexpr (CW == 4 && L2ONLY)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + c * CS) : "memory");
            else if constexpr (CW == 4)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + c * CS) : "memory");
            else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src + c * CS) : "memory");
        }
    }
    // row += d at L2 when pred (no branch).
    __device__ __forceinline__ static void red_add_if(bool pred, float* p, const float2 (&d)[H2]) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            if constexpr (CW == 4) {
                asm volatile(
                    "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
                    "@q red.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(p + c * CS),
                    "f"(d[2 * c].x), "f"(d[2 * c].y), "f"(d[2 * c + 1].x), "f"(d[2 * c + 1].y), "r"(static_cast<int>(pred))
                    : "memory");
            } else {
                asm volatile(
                    "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t"
                    "@q red.global.add.v2.f32 [%0], {%1, %2};\n\t}" ::"l"(p + c * CS),
                    "f"(d[c].x), "f"(d[c].y), "r"(static_cast<int>(pred))
                    : "memory");
            }
        }
    }
    // row += (v - entry): the ring row's accumulated update since it was loaded.
    __device__ __forceinline__ static void red_delta(float* p, const float2 (&v)[H2], const float* entry_smem) {
        float2 e[H2];
        load_shared(e, entry_smem);
#pragma unroll
        for (int i = 0; i < H2; ++i) e[i] = make_float2(v[i].x - e[i].x, v[i].y - e[i].y);
        red_add_if(true, p, e);
    }
};

// MODE: kFullChunk (N + 1 == NC samples, one chunk: every per-sample validity
// test is compile-time), kPartChunk (N + 1 < NC), kMultiChunk (N + 1 > NC:
// chunks of NC samples loaded per window).
constexpr int kFullChunk = 0, kPartChunk = 1, kMultiChunk = 2;

// RING: the ring rows' shared-memory copy (entry values for the delta
// write-back, or the finish() stash for the exact overwrite order). Without it
// rows leaving the ring are stored straight back (Hogwild overwrite, the
// reference's memcpy write-back, trainer.cpp:61-63, in any finish order).
// LIFETIME: the reference's default update order instead (sweep_samples,
// trainer.cpp:133-154: samples outer, contexts inner, every pairing sees the
// previous pairings' updates). Pairing (k, j) depends only on (k, j-1) and
// (k-1, j), so the 6 x 2W_f pairings of a window run as 2W_f + 5 anti-diagonal
// steps of up to 6 independent dots (the wavefront), with the sample rows in
// registers; windows whose sample ids repeat run the samples serially with the
// rewritten row forwarded (the reference re-reads it, trainer.cpp:143).
// One sentence per lane group: sentences sent0 + (threadIdx.x / LANES) of the block.
template <int LANES, int VEC, int WF, int NC, int MODE, bool FAST, bool RING = true, bool LIFETIME = false>
__device__ __forceinline__ void k1s_sentence(const ModelView& m, const BatchView& b, int n_neg_arg,
                                             DevCounters* __restrict__ ctr, int sent0) {
    static_assert(VEC % 2 == 0, "K1s stages 8- or 16-byte chunks");
    constexpr bool MULTI = MODE == kMultiChunk;
    constexpr bool FULL = MODE == kFullChunk;
    const int n_neg = FULL ? NC - 1 : n_neg_arg;  // compile-time on the full-chunk path
    using SM = K1sSmem<LANES, VEC, WF, NC, RING, LIFETIME, MODE == kMultiChunk && !LIFETIME>;
    constexpr int NCTX = SM::NCTX;
    constexpr int C = SM::C;
    constexpr int NV = SM::NV;
    constexpr int H2 = VEC / 2;
    constexpr int STRIDE = SM::STRIDE;
    constexpr int CL = SM::CL;      // control lanes: the group, or one warp of a 64-lane group
    constexpr int HALF = CL / 2;
    constexpr int NN = NC - 1;  // negatives per window held by every lane (single-chunk path)
    // Stale-prefetch detection by one __match_any_sync: lanes q < NC of a group
    // carry this window's sample ids, lanes HALF + q the previous window's.
    constexpr bool kMatch = NC <= HALF;
    // The top butterfly level pairs samples q and q + NC/2 of one context row;
    // lanes of the upper half load those two sample rows in swapped order, so
    // that level needs no selects.
    constexpr bool kPreswap = NC % 2 == 0;
    using SL = Slice<H2, LANES>;
    using BF = Butterfly<CL / 2, NV>;
    constexpr int NF = BF::final_count();
    static_assert(NV <= 255 && NC <= 16 && NCTX <= 16, "slot words");
    extern __shared__ __align__(16) float k1s_sh[];

    const int lane = threadIdx.x & 31;
    const int sub = static_cast<int>(threadIdx.x) & (LANES - 1);  // column slice
    const int csub = lane & (CL - 1);                               // control / butterfly lane
    const int grp = lane / CL;
    const int wig = static_cast<int>(threadIdx.x >> 5) & (SM::NWG - 1);  // warp in group
    const int sent = sent0 + static_cast<int>(threadIdx.x / LANES);
    const bool has = sent < b.n_sentences;
    float* gbase = k1s_sh + (threadIdx.x / LANES) * SM::kGroupFloats;
    float* gsh = gbase + wig * SM::GPAD;
    [[maybe_unused]] float* xbuf = gbase + SM::NWG * SM::GPAD;     // + (parity*NWG + warp)*NFX*32
    float* sbuf = gbase + SM::GA + sub * SL::CW;                    // + (parity*NC + q)*STRIDE
    float* ring = gbase + SM::GA + SM::SROWS * STRIDE + sub * SL::CW;  // + slot*STRIDE
    [[maybe_unused]] unsigned xpar = 0;
    const bool delta_wb = RING && (m.flags & kFlagDeltaRing) != 0;

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
    const int32_t* __restrict__ negs = b.negs + static_cast<size_t>(beg) * n_neg;
    // Row offsets: 64-bit products of the compile-time stride (|V| * stride may exceed 2^31).
    float* __restrict__ syn0 = m.syn0 + sub * SL::CW;
    float* __restrict__ syn1 = m.syn1 + sub * SL::CW;
    // Output row of sample s >= 0: hot rows go to this sentence's replica.
    // Output row of sample s >= 0 as one row index from syn1: hot rows go to this
    // sentence's replica (ModelView::hot_row), one select instead of two bases.
    const int hot_k = m.hot_k;
    const int hot_off = m.hot_k > 0 ? m.hot_row + (sent % m.hot_r) * m.hot_k : 0;
    auto srow = [&](int s) { return syn1 + static_cast<int64_t>(s < hot_k ? s + hot_off : s) * STRIDE; };
    const int tail = L - C;  // positions >= tail stay resident until finish()

    // After the butterfly, slot j of this lane holds dot idx = q*NCTX + r. One
    // opaque word per slot (the compiler would otherwise re-derive the plan
    // every window): g index | r << 8 | q << 12 | (q <= N) << 16 | (q == 0) << 17.
    unsigned slotw[NF];
    {
        int idx[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) idx[j] = j;
        BF::plan(idx, csub);
#pragma unroll
        for (int j = 0; j < NF; ++j) {
            const int q = idx[j] / NCTX, r = idx[j] - q * NCTX;
            slotw[j] = static_cast<unsigned>(idx[j]) | (static_cast<unsigned>(r) << 8) |
                       (static_cast<unsigned>(q) << 12) | ((q <= n_neg ? 1u : 0u) << 16) | ((q == 0 ? 1u : 0u) << 17);
            asm volatile("" : "+r"(slotw[j]));
        }
    }
    const int swap_off = (kPreswap && (csub & HALF) != 0) ? (NC / 2) * STRIDE : 0;

    float2 ctx[NCTX][H2];
    int tok[NCTX];
    float2 tgt[H2];
    int ttok = L > 0 ? __ldg(ids) : -1;
    if (ttok >= 0) SL::load(tgt, syn0 + static_cast<int64_t>(ttok) * STRIDE); else vzero2(tgt);
    if (delta_wb) SL::store_shared(ring, tgt);  // position 0 -> slot 0
#pragma unroll
    for (int r = 0; r < NCTX; ++r) {
        const int p = r - WF + 1;
        tok[r] = (r >= WF && p < L) ? __ldg(ids + p) : -1;
        if (tok[r] >= 0) SL::load(ctx[r], syn0 + static_cast<int64_t>(tok[r]) * STRIDE); else vzero2(ctx[r]);
        if (delta_wb && r >= WF) SL::store_shared(ring + p * STRIDE, ctx[r]);  // p < C
    }

    // Single-chunk path: every lane holds the negatives of windows i (ncur),
    // i+1 (nnext, for the prefetch) and, raw, i+2 (loaded one window early).
    int ncur[MULTI ? 1 : NN], nnext[MULTI ? 1 : NN], nraw[MULTI ? 1 : NN];
    if constexpr (!MULTI) {
#pragma unroll
        for (int k = 0; k < NN; ++k) {
            ncur[k] = (k < n_neg && L >= 2) ? __ldg(negs + k) : -1;
            nnext[k] = (k < n_neg && 1 < L) ? __ldg(negs + n_neg + k) : -1;
            nraw[k] = -1;
        }
    }
    int tok_ahead = WF + 1 < L ? __ldg(ids + WF + 1) : -1;  // incoming position of window 0
    int prev_v = -1 - lane;  // match lanes: previous window's sample id
    int psid[kMatch ? 1 : NC];
#pragma unroll
    for (int q = 0; q < (kMatch ? 1 : NC); ++q) psid[q] = -100;

    {
#pragma unroll
        for (int q = 0; q < SM::SROWS; ++q)
#pragma unroll
            SL::zero_shared(sbuf + q * STRIDE);
    }
    auto prefetch = [&](int target, const int (&nv)[MULTI ? 1 : NN], bool active, int parity) {
        float* dst = sbuf + parity * NC * STRIDE;
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            const int s = q == 0 ? target : nv[q > 0 ? q - 1 : 0];
            if (active && q <= n_neg && s >= 0) {
#pragma unroll
                SL::stage(dst + q * STRIDE, srow(s));
            }
        }
    };
    const bool l1_exact = (m.flags & kFlagL1Exact) != 0;
    const int inval_log2 = (m.flags >> kFlagInvalShift) & 15;
    const unsigned inval_mask = inval_log2 ? (1u << inval_log2) - 1u : 0u;
    bool nraw_ok = false;
    if constexpr (!MULTI) {
        prefetch(ttok, ncur, L >= 2, 0);  // window 0's samples
        cp_async_commit();
    }
    float2 dctx[MULTI ? NCTX : 1][H2];

    unsigned vmask = 0;  // bit r: context slot r holds a position of the sentence
#pragma unroll
    for (int r = 0; r < NCTX; ++r) vmask |= (tok[r] >= 0 ? 1u : 0u) << r;

    KB_T_DECL
    for (int i = 0; i < Lmax; ++i) {
        const bool act = i < L;
        const bool wact = act && L >= 2;
        const int q_in = i + 1 + WF;
        // Token ids run one window ahead of their rows and negatives two; loads
        // issued early are carried raw and masked where consumed. The
        // id/negative streams are pulled into L2 kPrefetchWindows ahead.
        if constexpr (!MULTI) {
            if (i > 0) {
#pragma unroll
                for (int k = 0; k < NN; ++k) nnext[k] = (nraw_ok && k < n_neg) ? nraw[k] : -1;
            }
        }
        // Next window's sample rows first (their buffer was last read in window
        // i-1); one cp.async group per window, so the wait below can leave it in flight.
        unsigned stale = 0;
        bool dup = false;  // lifetime order: a sample id repeats inside the window
        unsigned match_mask = 0;
        if constexpr (!MULTI) {
            if (i + 1 < Lmax) prefetch(tok[WF], nnext, i + 1 < L && L >= 2, (i + 1) & 1);
            cp_async_commit();
            // This window's rows the previous window rewrote after their prefetch
            // was issued (computed here, off the critical path).
            if constexpr (kMatch) {
                const int q = csub & (HALF - 1);
                int cv = ttok;
#pragma unroll
                for (int k = 0; k < NN; ++k) cv = q == k + 1 ? ncur[k] : cv;
                cv = (wact && q <= n_neg && q < NC) ? cv : -1 - lane;
                const int mv = csub < HALF ? cv : prev_v;
                match_mask = __match_any_sync(kFull, mv);  // consumed after the wait below
                prev_v = cv;
            } else {
                int sq[NC];
#pragma unroll
                for (int q = 0; q < NC; ++q) sq[q] = (wact && q <= n_neg) ? (q == 0 ? ttok : ncur[q > 0 ? q - 1 : 0]) : -1 - q;
#pragma unroll
                for (int q = 0; q < NC; ++q) {
                    bool st = false;
#pragma unroll
                    for (int j = 0; j < NC; ++j) st |= sq[q] == psid[j];
                    stale |= (st ? 1u : 0u) << q;
                }
#pragma unroll
                for (int q = 0; q < NC; ++q) psid[q] = sq[q] >= 0 ? sq[q] : -100;
                if constexpr (LIFETIME) {
#pragma unroll
                    for (int q = 1; q < NC; ++q)
#pragma unroll
                        for (int j = 0; j < q; ++j) dup |= sq[q] == sq[j];
                    dup = __any_sync(kFull, dup);
                }
            }
        }
        const int inc_tok = tok_ahead;
        float2 inc[H2];
        SL::load_early(inc, syn0 + static_cast<int64_t>(max(inc_tok, 0)) * STRIDE);
        const int last = max(L - 1, 0);
        const int tok_raw = ldg_early(ids + min(q_in + 1, last));
        if constexpr (!MULTI) {
            const int* nrow = negs + static_cast<size_t>(min(i + 2, last)) * n_neg;
#pragma unroll
            for (int k = 0; k < NN; ++k) nraw[k] = n_neg > 0 ? ldg_early(nrow + min(k, n_neg - 1)) : -1;
        }
        const bool tok_ok = q_in + 1 < L;
        if (sub == 0 && i + kPrefetchWindows < L) {
            prefetch_l2(negs + static_cast<size_t>(i + kPrefetchWindows) * n_neg);
            prefetch_l2(ids + min(L - 1, q_in + kPrefetchWindows));
        }
        if constexpr (MULTI && !LIFETIME) {
#pragma unroll
            for (int r = 0; r < NCTX; ++r) vzero2(dctx[r]);
        }

        if constexpr (MULTI && !LIFETIME) {
            // Snapshot order: every sample row of the window as it is before any of
            // the window's reductions (sweep_samples_snapshot, trainer.cpp:158-205).
            for (int kk = 0; kk <= n_neg; ++kk) {
                const int s = kk == 0 ? ttok : (wact ? __ldg(negs + i * n_neg + kk - 1) : -1);
                float2 v[H2];
                SL::load(v, srow(max(s, 0)));
                SL::store_shared(sbuf + kk * STRIDE, v);
            }
        }
        const int n_chunks = MULTI ? (n_neg + NC) / NC : 1;
        for (int ch = 0; ch < n_chunks; ++ch) {
            const int kbase = MULTI ? ch * NC : 0;
            int sid[NC];
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                const int kk = kbase + q;
                int s;
                if constexpr (MULTI) s = (kk == 0) ? ttok : (wact && kk <= n_neg ? __ldg(negs + i * n_neg + kk - 1) : -1);
                else s = q == 0 ? ttok : ncur[q > 0 ? q - 1 : 0];
                // Empty slots: distinct negative ids. On the full-chunk path every
                // slot holds a valid id whenever the window is active.
                if constexpr (FULL) sid[q] = s;
                else sid[q] = (wact && kk <= n_neg) ? s : -1 - q;
            }
            const float* cur = sbuf;
            if constexpr (!MULTI) {
                // Rows staged by cp.async during the previous window; slots
                // without a sample hold finite stale rows and get g = 0.
                KB_T(0)
                if constexpr (kMatch) {  // the match issued at the top of the window has landed
                    const unsigned upper = ((1u << HALF) - 1u) << (grp * CL + HALF);
                    const bool st = csub < HALF && (match_mask & upper) != 0u;
                    stale = (__ballot_sync(kFull, st) >> (grp * CL)) & ((1u << NC) - 1u);
                    if constexpr (LIFETIME) {
                        const unsigned lower = ((1u << HALF) - 1u) << (grp * CL);
                        dup = __any_sync(kFull, csub < HALF && __popc(match_mask & lower) > 1);
                    }
                }
                cp_async_wait_group<1>();
                KB_T(1)
                cur = sbuf + (i & 1) * NC * STRIDE;
                if (stale != 0u) {
#pragma unroll
                    for (int q = 0; q < NC; ++q)
                        if (((stale >> q) & 1u) && (FULL ? wact : sid[q] >= 0)) {
                            float2 v[H2];
                            SL::load(v, srow(sid[q]));
                            SL::store_shared(const_cast<float*>(cur) + q * STRIDE, v);
                        }
                }
            } else if constexpr (!LIFETIME) {
                cur = sbuf + kbase * STRIDE;  // rows staged at window entry
            } else {
                // Lifetime order: chunk rows read now include every reduction this
                // thread issued before (earlier chunks of the window).
#pragma unroll
                for (int q = 0; q < NC; ++q) {
                    float2 v[H2];
                    SL::load(v, srow(max(sid[q], 0)));
                    SL::store_shared(sbuf + q * STRIDE, v);
                }
                {
                    bool d = false;
#pragma unroll
                    for (int q = 1; q < NC; ++q)
#pragma unroll
                        for (int j = 0; j < q; ++j) d |= sid[q] >= 0 && sid[q] == sid[j];
                    dup = __any_sync(kFull, d);
                }
            }

            if constexpr (LIFETIME) {
                // Sample rows of the window in registers (staged values = entry values).
                float2 S[NC][H2];
#pragma unroll
                for (int q = 0; q < NC; ++q) SL::load_shared(S[q], cur + q * STRIDE);
                // Per-window constants: context validity (this window, as a mask of
                // the active slots) and the folded fast-sigmoid coefficients.
                const unsigned vm = wact ? vmask : 0u;
                const float al1 = 0.5f * alpha, al0 = -0.5f * alpha, nha = -0.5f * alpha;
                auto pair_g = [&](int k, int j, float f) {
                    const bool valid = ((vm >> j) & 1u) != 0u && (FULL || kbase + k <= n_neg);
                    float g;
                    if constexpr (FAST) g = sgd_coeff_fast(f, kbase + k == 0 ? al1 : al0, nha);
                    else g = sgd_coeff<FAST>(f, kbase + k == 0 ? 1.0f : 0.0f, alpha);
                    return valid ? g : 0.0f;
                };
                auto update = [&](int k, int j, float g) {  // pairing_update (kernels.hpp:26-33)
                    const float2 gg = make_float2(g, g);
#pragma unroll
                    for (int h = 0; h < H2; ++h) {
                        const float2 c = ctx[j][h];
                        ctx[j][h] = __ffma2_rn(gg, S[k][h], c);
                        S[k][h] = __ffma2_rn(gg, c, S[k][h]);
                    }
                };
                auto dot = [&](int k, int j) {
                    float2 acc = __fmul2_rn(ctx[j][0], S[k][0]);
#pragma unroll
                    for (int h = 1; h < H2; ++h) acc = __ffma2_rn(ctx[j][h], S[k][h], acc);
                    return acc.x + acc.y;
                };
                // 64-lane groups: the two warps' partial dots of one step meet in the
                // double-buffered exchange (one barrier per step; sentence-uniform).
                auto exchange = [&](float* f, auto live) {
                    if constexpr (SM::NWG > 1) {
                        float* mine = xbuf + (xpar * SM::NWG + wig) * SM::NFX * 32 + lane;
                        const float* other = xbuf + (xpar * SM::NWG + (wig ^ 1)) * SM::NFX * 32 + lane;
#pragma unroll
                        for (int k = 0; k < NC; ++k)
                            if (live(k)) mine[k * 32] = f[k];
                        __syncthreads();
#pragma unroll
                        for (int k = 0; k < NC; ++k)
                            if (live(k)) f[k] += other[k * 32];
                        xpar ^= 1u;
                    }
                };
                if (!dup) {
                    // Anti-diagonal d: pairings (k, d-k), independent of each other.
#pragma unroll
                    for (int d = 0; d < NC + NCTX - 1; ++d) {
                        float f[NC];
#pragma unroll
                        for (int k = 0; k < NC; ++k)
                            if (d - k >= 0 && d - k < NCTX) f[k] = dot(k, d - k);
#pragma unroll
                        for (int o = CL / 2; o > 0; o >>= 1)
#pragma unroll
                            for (int k = 0; k < NC; ++k)
                                if (d - k >= 0 && d - k < NCTX) f[k] += __shfl_xor_sync(kFull, f[k], o);
                        exchange(f, [&](int k) { return d - k >= 0 && d - k < NCTX; });
                        // (g evaluated by every lane: a lane-distributed sigmoid with
                        // shuffled g measured 7% slower; the wavefront is latency-bound)
#pragma unroll
                        for (int k = 0; k < NC; ++k)
                            if (d - k >= 0 && d - k < NCTX) update(k, d - k, pair_g(k, d - k, f[k]));
                    }
                } else {
                    // Reference order, sample by sample; a repeated id starts from the
                    // row its previous occurrence left (the reference re-reads it).
#pragma unroll
                    for (int k = 0; k < NC; ++k) {
#pragma unroll
                        for (int k2 = 0; k2 < k; ++k2)
                            if (sid[k2] == sid[k]) vcopy2(S[k], S[k2]);
#pragma unroll
                        for (int j = 0; j < NCTX; ++j) {
                            float f[1] = {dot(k, j)};
#pragma unroll
                            for (int o = CL / 2; o > 0; o >>= 1) f[0] += __shfl_xor_sync(kFull, f[0], o);
                            exchange(f, [](int kk) { return kk == 0; });
                            update(k, j, pair_g(k, j, f[0]));
                        }
                    }
                }
                // Sample write-back: one row += (final - staged) per distinct id, at its
                // last occurrence (earlier occurrences were forwarded into it).
#pragma unroll
                for (int q = 0; q < NC; ++q) {
                    bool last_occ = true;
#pragma unroll
                    for (int q2 = q + 1; q2 < NC; ++q2) last_occ &= sid[q2] != sid[q];
                    float2 e[H2];
                    SL::load_shared(e, cur + q * STRIDE);
#pragma unroll
                    for (int h = 0; h < H2; ++h) e[h] = make_float2(S[q][h].x - e[h].x, S[q][h].y - e[h].y);
                    if constexpr (FULL) SL::red_add_if(wact && (last_occ || !dup), srow(sid[q]), e);
                    else SL::red_add_if(sid[q] >= 0 && (last_occ || !dup), srow(max(sid[q], 0)), e);
                }
            } else {
            KB_T(2)
            // 1-2. all dots of the chunk (window-entry values), one transposed butterfly.
            float P[NV];
            {
                const float* lo = cur + swap_off;  // samples q < NC/2 (or their partners)
                const float* hi = cur - swap_off;
#pragma unroll
                for (int q = 0; q < NC; ++q) {
                    float2 S[H2];
                    SL::load_shared(S, (kPreswap && q < NC / 2 ? lo : (kPreswap ? hi : cur)) + q * STRIDE);
#pragma unroll
                    for (int r = 0; r < NCTX; ++r) {
                        float2 acc = __fmul2_rn(ctx[r][0], S[0]);
#pragma unroll
                        for (int h = 1; h < H2; ++h) acc = __ffma2_rn(ctx[r][h], S[h], acc);
                        P[q * NCTX + r] = acc.x + acc.y;
                    }
                }
            }
            KB_T(3)
            if constexpr (kPreswap) BF::reduce_preswapped(P, csub);
            else BF::reduce(P, csub);
            if constexpr (SM::NWG > 1) {
                // Both warps' column halves: the exchange buffer is double-buffered,
                // so one barrier per chunk orders every reuse. Sentence-uniform
                // control flow: both warps reach each barrier.
                float* mine = xbuf + (xpar * SM::NWG + wig) * SM::NFX * 32 + lane;
                const float* other = xbuf + (xpar * SM::NWG + (wig ^ 1)) * SM::NFX * 32 + lane;
#pragma unroll
                for (int j = 0; j < NF; ++j) mine[j * 32] = P[j];
                __syncthreads();
#pragma unroll
                for (int j = 0; j < NF; ++j) P[j] += other[j * 32];
                xpar ^= 1u;
            }

            KB_T(4)
            // 3. sigmoid on the owned dots; g published as scalars [q][r].
#pragma unroll
            for (int j = 0; j < NF; ++j) {
                const unsigned w = slotw[j];
                const bool vbit = ((vmask >> ((w >> 8) & 15u)) & 1u) != 0u;
                bool valid;
                float label;
                if constexpr (MULTI) {
                    const int kk = kbase + static_cast<int>((w >> 12) & 15u);
                    valid = wact && kk <= n_neg && vbit;
                    label = kk == 0 ? 1.0f : 0.0f;
                } else {
                    valid = wact && ((w >> 16) & 1u) && vbit;
                    label = ((w >> 17) & 1u) ? 1.0f : 0.0f;
                }
                float g;
                if constexpr (FAST) g = sgd_coeff_fast(P[j], alpha * (label - 0.5f), -0.5f * alpha);
                else g = sgd_coeff<FAST>(P[j], label, alpha);
                gsh[w & 255u] = valid ? g : 0.0f;
            }
            __syncwarp();
            float g[SM::GPAD];
#pragma unroll
            for (int k = 0; k < SM::GPAD; k += 4) {
                const float4 t = *reinterpret_cast<const float4*>(gsh + k);
                g[k] = t.x; g[k + 1] = t.y; g[k + 2] = t.z; g[k + 3] = t.w;
            }
            __syncwarp();

            KB_T(5)
            // 4a. sample deltas from window-entry context rows, written back as
            //     row += delta at L2 (trainer.cpp:198-204, duplicates included).
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                float2 D[H2];
#pragma unroll
                for (int h = 0; h < H2; ++h) D[h] = __fmul2_rn(make_float2(g[q * NCTX], g[q * NCTX]), ctx[0][h]);
#pragma unroll
                for (int r = 1; r < NCTX; ++r)
#pragma unroll
                    for (int h = 0; h < H2; ++h)
                        D[h] = __ffma2_rn(make_float2(g[q * NCTX + r], g[q * NCTX + r]), ctx[r][h], D[h]);
                if constexpr (FULL) SL::red_add_if(wact, srow(sid[q]), D);
                else SL::red_add_if(sid[q] >= 0, srow(max(sid[q], 0)), D);
            }
            KB_T(6)
            // 4b. context rows from window-entry sample rows.
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                float2 S[H2];
                SL::load_shared(S, cur + q * STRIDE);
#pragma unroll
                for (int r = 0; r < NCTX; ++r) {
                    const float2 gg = make_float2(g[q * NCTX + r], g[q * NCTX + r]);
#pragma unroll
                    for (int h = 0; h < H2; ++h) {
                        if constexpr (MULTI) dctx[r][h] = __ffma2_rn(gg, S[h], dctx[r][h]);
                        else ctx[r][h] = __ffma2_rn(gg, S[h], ctx[r][h]);
                    }
                }
            }
            }  // snapshot
            if constexpr (MULTI) __syncwarp();  // the next chunk rewrites sbuf
        }
        if constexpr (MULTI && !LIFETIME) {
#pragma unroll
            for (int r = 0; r < NCTX; ++r)
#pragma unroll
                for (int h = 0; h < H2; ++h) ctx[r][h] = __fadd2_rn(ctx[r][h], dctx[r][h]);
        }

        KB_T(7)
        // Slide the ring (ContextRing::advance, trainer.cpp:55-69).
        const int etok = tok[0];
        if (etok >= 0) {
            const int p = i - WF;
            if (!RING) {
                SL::store(syn0 + static_cast<int64_t>(etok) * STRIDE, ctx[0]);
            } else if (delta_wb) {
                SL::red_delta(syn0 + static_cast<int64_t>(etok) * STRIDE, ctx[0], ring + (p % C) * STRIDE);
            } else if (p >= tail) {
                SL::store_shared(ring + (p % C) * STRIDE, ctx[0]);
            } else {
                SL::store(syn0 + static_cast<int64_t>(etok) * STRIDE, ctx[0]);
            }
            if (inc_tok == etok) vcopy2(inc, ctx[0]);
        }
        if (delta_wb && inc_tok >= 0) SL::store_shared(ring + (q_in % C) * STRIDE, inc);
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
        // The validity mask slides with the slots: bit WF-1 takes the old target.
        vmask = ((vmask >> 1) & ~(1u << (WF - 1))) | ((act && tok[WF - 1] >= 0 ? 1u : 0u) << (WF - 1)) |
                ((inc_tok >= 0 ? 1u : 0u) << (NCTX - 1));
        if constexpr (!MULTI) {
#pragma unroll
            for (int k = 0; k < NN; ++k) ncur[k] = nnext[k];
        }
        nraw_ok = i + 2 < L;
        tok_ahead = tok_ok ? tok_raw : -1;
        // Sample rows are staged through L1. Exact mode: this warp drops its SM's
        // L1 before the next window's staging (fence.acq_rel.gpu -> CCTL.IVALL),
        // so every read sees this sentence's earlier reductions. Otherwise one
        // warp per block refreshes the L1 every 2^k windows: bounded staleness
        // for the Zipf-hot rows, whose lines stay L1-resident in between.
        if (l1_exact || (inval_mask != 0u && (static_cast<unsigned>(i) & inval_mask) == inval_mask &&
                         (threadIdx.x >> 5) == 0)) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
    }
    KB_T(8)
    KB_T_DUMP
    // ContextRing::finish (trainer.cpp:71-75): residents in slot order.
    const int i_end = Lmax;  // registers hold positions i_end-WF .. i_end+WF
    if (!RING) {
#pragma unroll
        for (int r = 0; r < NCTX; ++r)
            if (tok[r] >= 0) SL::store(syn0 + static_cast<int64_t>(tok[r]) * STRIDE, ctx[r]);
        if (ttok >= 0) SL::store(syn0 + static_cast<int64_t>(ttok) * STRIDE, tgt);
    } else if (delta_wb) {
        // Deltas commute: no ordering to preserve.
#pragma unroll
        for (int r = 0; r < NCTX; ++r) {
            const int p = r < WF ? i_end - WF + r : i_end + 1 + (r - WF);
            if (tok[r] >= 0) SL::red_delta(syn0 + static_cast<int64_t>(tok[r]) * STRIDE, ctx[r], ring + (p % C) * STRIDE);
        }
        if (ttok >= 0) SL::red_delta(syn0 + static_cast<int64_t>(ttok) * STRIDE, tgt, ring + (i_end % C) * STRIDE);
    } else {
#pragma unroll
        for (int r = 0; r < NCTX; ++r) {
            const int p = r < WF ? i_end - WF + r : i_end + 1 + (r - WF);
            if (tok[r] >= 0) SL::store_shared(ring + (p % C) * STRIDE, ctx[r]);
        }
        if (ttok >= 0) SL::store_shared(ring + (i_end % C) * STRIDE, tgt);
        const int first = max(0, tail);
        for (int s = 0; s < C; ++s) {
            // the resident position in slot s: first + ((s - first) mod C), if < L
            const int p = first + ((s - first % C) + C) % C;
            if (p < L) {
                float2 v[H2];
                SL::load_shared(v, ring + s * STRIDE);
                SL::store(syn0 + static_cast<int64_t>(__ldg(ids + p)) * STRIDE, v);
            }
        }
    }

    if (ctr != nullptr) {
        const bool lead = has && sub == 0;
        // Closed forms of the per-window counts (each position read once; every
        // window of a sentence of >= 2 words has N+1 samples and its valid contexts).
        const unsigned ns = static_cast<unsigned>(n_neg + 1);
        const unsigned c_reads = static_cast<unsigned>(L);
        const unsigned s_rw = L >= 2 ? static_cast<unsigned>(L) * ns : 0u;
        const unsigned half = L <= WF + 1 ? static_cast<unsigned>(L * (L - 1) / 2)
                                          : static_cast<unsigned>(WF * (WF + 1) / 2 + (L - WF - 1) * WF);
        const unsigned pairs = L >= 2 ? 2u * half * ns : 0u;
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
    cp_async_wait_group<0>();  // the staging buffers are the next sentence's
    // Two-warp groups: the next sentence's first exchange must not overwrite a
    // buffer the other warp is still reading from this sentence's last one.
    if constexpr (SM::NWG > 1) __syncthreads();
}

// Blocks stride over the batch's sentences (BatchView::max_groups caps the grid:
// the Hogwild in-flight budget without splitting the batch into launches).
template <int LANES, int VEC, int WF, int NC, int MODE, bool FAST, bool RING = true, bool LIFETIME = false>
__global__ void __launch_bounds__(K1sSmem<LANES, VEC, WF, NC, RING, LIFETIME, MODE == 2 && !LIFETIME>::THREADS,
                                  K1sSmem<LANES, VEC, WF, NC, RING, LIFETIME, MODE == 2 && !LIFETIME>::MINB)
k1s_snapshot(ModelView m, BatchView b, int n_neg_arg, DevCounters* __restrict__ ctr) {
    constexpr int PB = K1sSmem<LANES, VEC, WF, NC, RING, LIFETIME, MODE == 2 && !LIFETIME>::THREADS / LANES;
    for (int s0 = static_cast<int>(blockIdx.x) * PB; s0 < b.n_sentences; s0 += static_cast<int>(gridDim.x) * PB)
        k1s_sentence<LANES, VEC, WF, NC, MODE, FAST, RING, LIFETIME>(m, b, n_neg_arg, ctr, s0);
}

// Grid for a batch, capped by the in-flight budget (BatchView::max_groups).
inline int k1s_grid(const BatchView& b, int per_block) {
    int blocks = (b.n_sentences + per_block - 1) / per_block;
    if (b.max_groups > 0) blocks = std::min(blocks, std::max(1, b.max_groups / per_block));
    return blocks;
}

} // namespace fw2v

#include "fw2v_stair.cuh"

namespace fw2v {

// ------------------------------------------------------------------ dispatch
template <int LANES, int VEC, int WF, int NC, int MODE, bool FAST, bool RING, bool LIFETIME>
cudaError_t launch_k1s_inst(int blocks, const ModelView& m, const BatchView& b, int n_neg, DevCounters* ctr,
                            cudaStream_t st, int* resident) {
    using SMx = K1sSmem<LANES, VEC, WF, NC, RING, LIFETIME, MODE == kMultiChunk && !LIFETIME>;
    constexpr int bytes = SMx::kBlockBytes;
    auto* kern = k1s_snapshot<LANES, VEC, WF, NC, MODE, FAST, RING, LIFETIME>;
    static std::atomic<uint64_t> configured{0};  // one bit per device ordinal
    if (cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), bytes, configured); e != cudaSuccess)
        return e;
    constexpr int threads = SMx::THREADS;
    if (resident != nullptr) return resident_sentences(kern, bytes, threads, threads / LANES, resident);
    if (blocks == 0) return cudaSuccess;
    kern<<<blocks, threads, bytes, st>>>(m, b, n_neg, ctr);
    return cudaGetLastError();
}

// Sigmoid and ring variants of one mode; the Hogwild overwrite (no shared-memory
// ring) is built for the fast sigmoid only.
template <int LANES, int VEC, int WF, int NC, int MODE, bool LIFETIME>
cudaError_t launch_k1s_mode(int blocks, const ModelView& m, const BatchView& b, int n_neg, bool fast, DevCounters* ctr,
                            cudaStream_t st, int* resident) {
    if (fast && (m.flags & kFlagNoRing) != 0)
        return launch_k1s_inst<LANES, VEC, WF, NC, MODE, true, false, LIFETIME>(blocks, m, b, n_neg, ctr, st, resident);
    return fast ? launch_k1s_inst<LANES, VEC, WF, NC, MODE, true, true, LIFETIME>(blocks, m, b, n_neg, ctr, st, resident)
                : launch_k1s_inst<LANES, VEC, WF, NC, MODE, false, true, LIFETIME>(blocks, m, b, n_neg, ctr, st, resident);
}

template <int LANES, int VEC, int WF, int NC>
cudaError_t launch_k1s_nc(const ModelView& m, const BatchView& b, int n_neg, bool fast, bool lifetime,
                          DevCounters* ctr, cudaStream_t st, int* resident) {
    constexpr int per_block = K1sSmem<LANES, VEC, WF, NC>::THREADS / LANES;  // RING does not change THREADS
    const int blocks = k1s_grid(b, per_block);
    if (n_neg + 1 > NC) {
        // Lifetime order, N = 15 on 32-lane groups: the staircase with the 16
        // samples streaming through 2W_f register slots (one wavefront per window).
        // (4 columns per lane: at 8 the 17-step unrolled iteration no longer fits.)
        if constexpr (NC == 6 && LANES == 32 && WF <= 3 && VEC == 4) {
            if (lifetime && n_neg + 1 == 16 && fast && (m.flags & kFlagNoRing) != 0 && (m.flags & kFlagNoStair) == 0)
                return launch_k1s_stair<LANES, VEC, WF, 16, true>(m, b, ctr, st, resident);
        }
        // Chunks of NC samples; in lifetime order each chunk is its own wavefront,
        // started from the contexts the previous chunk left (exact order).
        if constexpr (VEC <= 10) {
            if (lifetime)
                return fast ? launch_k1s_inst<LANES, VEC, WF, NC, kMultiChunk, true, true, true>(blocks, m, b, n_neg, ctr, st, resident)
                            : launch_k1s_inst<LANES, VEC, WF, NC, kMultiChunk, false, true, true>(blocks, m, b, n_neg, ctr, st, resident);
        }
        if (lifetime) return cudaErrorInvalidValue;
        return fast ? launch_k1s_inst<LANES, VEC, WF, NC, kMultiChunk, true, true, false>(blocks, m, b, n_neg, ctr, st, resident)
                    : launch_k1s_inst<LANES, VEC, WF, NC, kMultiChunk, false, true, false>(blocks, m, b, n_neg, ctr, st, resident);
    }
    if constexpr (NC < 6) {  // 4-sample chunks are only dispatched for N + 1 > 6
        return cudaErrorInvalidValue;
    } else if constexpr (VEC > 10) {  // lifetime order: the window's sample rows would not fit in registers
        if (lifetime) return cudaErrorInvalidValue;
        if (n_neg + 1 < NC) return launch_k1s_mode<LANES, VEC, WF, NC, kPartChunk, false>(blocks, m, b, n_neg, fast, ctr, st, resident);
        return launch_k1s_mode<LANES, VEC, WF, NC, kFullChunk, false>(blocks, m, b, n_neg, fast, ctr, st, resident);
    } else {
        if (n_neg + 1 < NC)
            return lifetime ? launch_k1s_mode<LANES, VEC, WF, NC, kPartChunk, true>(blocks, m, b, n_neg, fast, ctr, st, resident)
                            : launch_k1s_mode<LANES, VEC, WF, NC, kPartChunk, false>(blocks, m, b, n_neg, fast, ctr, st, resident);
        // Lifetime order, N = 5, Hogwild overwrite, fast sigmoid: the window staircase.
        // At W_f = 4-5 both windows' rows spill some registers: still faster at
        // 4-8 columns per lane (profiles/r02q_stair_wide_windows.txt), not at 10.
        if constexpr (NC == 6 && (LANES == 16 || LANES == 32) && WF <= 5 && (VEC == 4 || VEC == 8 || VEC == 10) &&
                      (WF <= 3 || VEC != 10)) {
            if (lifetime && fast && (m.flags & kFlagNoRing) != 0 && (m.flags & kFlagNoStair) == 0)
                return launch_k1s_stair<LANES, VEC, WF, 6, true>(m, b, ctr, st, resident);
        }
        return lifetime ? launch_k1s_mode<LANES, VEC, WF, NC, kFullChunk, true>(blocks, m, b, n_neg, fast, ctr, st, resident)
                        : launch_k1s_mode<LANES, VEC, WF, NC, kFullChunk, false>(blocks, m, b, n_neg, fast, ctr, st, resident);
    }
}

// Window-snapshot multi-chunk kernels only (N + 1 > NC).
template <int LANES, int VEC, int WF, int NC>
cudaError_t launch_k1s_snap_multi(const ModelView& m, const BatchView& b, int n_neg, bool fast, DevCounters* ctr,
                                  cudaStream_t st, int* resident) {
    constexpr int per_block = K1sSmem<LANES, VEC, WF, NC>::THREADS / LANES;
    const int blocks = k1s_grid(b, per_block);
    return fast ? launch_k1s_inst<LANES, VEC, WF, NC, kMultiChunk, true, true, false>(blocks, m, b, n_neg, ctr, st, resident)
                : launch_k1s_inst<LANES, VEC, WF, NC, kMultiChunk, false, true, false>(blocks, m, b, n_neg, ctr, st, resident);
}

template <int LANES, int VEC>
cudaError_t launch_k1s_shape(const ModelView& m, const BatchView& b, int n_neg, int wf, bool fast, bool lifetime,
                             DevCounters* ctr, cudaStream_t st, int* resident) {
    // Window-snapshot order at W_f <= 3 with 13-16 samples: two 8-sample chunks
    // instead of three of 6 (fewer butterflies; measured +3-8% at N=15, 1bw shape;
    // lifetime order keeps 6: its 8-sample wavefront spills).
    const int S = n_neg + 1;
    const bool nc8 = !lifetime && S > 8 && (S + 7) / 8 < (S + 5) / 6;
    switch (wf) {
    case 1: return nc8 ? launch_k1s_snap_multi<LANES, VEC, 1, 8>(m, b, n_neg, fast, ctr, st, resident)
                       : launch_k1s_nc<LANES, VEC, 1, 6>(m, b, n_neg, fast, lifetime, ctr, st, resident);
    case 2: return nc8 ? launch_k1s_snap_multi<LANES, VEC, 2, 8>(m, b, n_neg, fast, ctr, st, resident)
                       : launch_k1s_nc<LANES, VEC, 2, 6>(m, b, n_neg, fast, lifetime, ctr, st, resident);
    case 3: return nc8 ? launch_k1s_snap_multi<LANES, VEC, 3, 8>(m, b, n_neg, fast, ctr, st, resident)
                       : launch_k1s_nc<LANES, VEC, 3, 6>(m, b, n_neg, fast, lifetime, ctr, st, resident);
    // Wide windows: one 6-sample chunk when N+1 <= 6, else 4-sample chunks (registers).
    case 4: return n_neg + 1 <= 6 ? launch_k1s_nc<LANES, VEC, 4, 6>(m, b, n_neg, fast, lifetime, ctr, st, resident)
                                  : launch_k1s_nc<LANES, VEC, 4, 4>(m, b, n_neg, fast, lifetime, ctr, st, resident);
    case 5: return n_neg + 1 <= 6 ? launch_k1s_nc<LANES, VEC, 5, 6>(m, b, n_neg, fast, lifetime, ctr, st, resident)
                                  : launch_k1s_nc<LANES, VEC, 5, 4>(m, b, n_neg, fast, lifetime, ctr, st, resident);
    default: return cudaErrorInvalidValue;
    }
}

} // namespace fw2v
