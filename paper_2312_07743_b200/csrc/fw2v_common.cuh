// Device helpers shared by the FULL-W2V kernels (row I/O through L2, lane-group
// reductions, the SGD coefficient).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "fw2v_device.cuh"

namespace fw2v {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kK1Threads = 128;

// ------------------------------------------------------------------ row I/O
// Model rows go through L2 only (ld.global.cg / st.global.cg): other SMs
// update them concurrently (Hogwild), and L1 is not coherent within a launch.
template <int VEC>
struct Row {
    __device__ __forceinline__ static void load(float (&v)[VEC], const float* p) {
        if constexpr (VEC % 4 == 0) {
#pragma unroll
            for (int i = 0; i < VEC; i += 4) {
                float4 t = __ldcg(reinterpret_cast<const float4*>(p + i));
                v[i] = t.x; v[i + 1] = t.y; v[i + 2] = t.z; v[i + 3] = t.w;
            }
        } else if constexpr (VEC % 2 == 0) {
#pragma unroll
            for (int i = 0; i < VEC; i += 2) {
                float2 t = __ldcg(reinterpret_cast<const float2*>(p + i));
                v[i] = t.x; v[i + 1] = t.y;
            }
        } else {
#pragma unroll
            for (int i = 0; i < VEC; ++i) v[i] = __ldcg(p + i);
        }
    }
    __device__ __forceinline__ static void store(float* p, const float (&v)[VEC]) {
        if constexpr (VEC % 4 == 0) {
#pragma unroll
            for (int i = 0; i < VEC; i += 4)
                __stcg(reinterpret_cast<float4*>(p + i), make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
        } else if constexpr (VEC % 2 == 0) {
#pragma unroll
            for (int i = 0; i < VEC; i += 2)
                __stcg(reinterpret_cast<float2*>(p + i), make_float2(v[i], v[i + 1]));
        } else {
#pragma unroll
            for (int i = 0; i < VEC; ++i) __stcg(p + i, v[i]);
        }
    }
};

// Rows as float2 pairs (operands of the sm_100 packed FFMA2/FADD2).
template <int H2>
struct Row2 {
    __device__ __forceinline__ static void load(float2 (&v)[H2], const float* p) {
        if constexpr (H2 % 2 == 0) {
#pragma unroll
            for (int i = 0; i < H2; i += 2) {
                const float4 t = __ldcg(reinterpret_cast<const float4*>(p + 2 * i));
                v[i] = make_float2(t.x, t.y);
                v[i + 1] = make_float2(t.z, t.w);
            }
        } else {
#pragma unroll
            for (int i = 0; i < H2; ++i) v[i] = __ldcg(reinterpret_cast<const float2*>(p + 2 * i));
        }
    }
    __device__ __forceinline__ static void store(float* p, const float2 (&v)[H2]) {
        if constexpr (H2 % 2 == 0) {
#pragma unroll
            for (int i = 0; i < H2; i += 2)
                __stcg(reinterpret_cast<float4*>(p + 2 * i), make_float4(v[i].x, v[i].y, v[i + 1].x, v[i + 1].y));
        } else {
#pragma unroll
            for (int i = 0; i < H2; ++i) __stcg(reinterpret_cast<float2*>(p + 2 * i), v[i]);
        }
    }
    __device__ __forceinline__ static void load_shared(float2 (&v)[H2], const float* p) {
        static_assert(H2 % 2 == 0, "16-byte shared slices");
#pragma unroll
        for (int i = 0; i < H2; i += 2) {
            const float4 t = *reinterpret_cast<const float4*>(p + 2 * i);
            v[i] = make_float2(t.x, t.y);
            v[i + 1] = make_float2(t.z, t.w);
        }
    }
    __device__ __forceinline__ static void store_shared(float* p, const float2 (&v)[H2]) {
        static_assert(H2 % 2 == 0, "16-byte shared slices");
#pragma unroll
        for (int i = 0; i < H2; i += 2)
            *reinterpret_cast<float4*>(p + 2 * i) = make_float4(v[i].x, v[i].y, v[i + 1].x, v[i + 1].y);
    }
};

// Loads issued where they are written: asm volatile keeps the compiler from
// sinking a prefetch-distance load down to its first use (which it otherwise
// does to shorten live ranges, turning a one-window lookahead into none).
__device__ __forceinline__ float4 ldcg_early(const float* p) {
    float4 v;
    asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ int ldg_early(const int* p) {
    int v;
    asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
template <int H2>
__device__ __forceinline__ void row_load_early(float2 (&v)[H2], const float* p) {
    static_assert(H2 % 2 == 0, "16-byte slices");
#pragma unroll
    for (int i = 0; i < H2; i += 2) {
        const float4 t = ldcg_early(p + 2 * i);
        v[i] = make_float2(t.x, t.y);
        v[i + 1] = make_float2(t.z, t.w);
    }
}

// One observer-log entry (BatchView::obs_log): called by one lane per sentence
// before each window, empty windows included (trainer.cpp:246).
__device__ __forceinline__ void obs_record(const BatchView& b, int sentence, int target) {
    if (b.obs_log != nullptr) {
        const unsigned k = atomicAdd(b.obs_count, 1u);
        b.obs_log[k] = (static_cast<unsigned long long>(b.obs_base + sentence) << 32) | static_cast<unsigned>(target);
    }
}

// All L windows of a sentence at once (the Hogwild kernels log when a sentence
// starts, outside their window loop; per sentence the targets are in order).
__device__ __forceinline__ void obs_record_sentence(const BatchView& b, int sentence, int L) {
    if (b.obs_log != nullptr && L > 0) {
        const unsigned k0 = atomicAdd(b.obs_count, static_cast<unsigned>(L));
        const unsigned long long s = static_cast<unsigned long long>(b.obs_base + sentence) << 32;
        for (int i = 0; i < L; ++i) b.obs_log[k0 + i] = s | static_cast<unsigned>(i);
    }
}

template <int H2>
__device__ __forceinline__ void vzero2(float2 (&v)[H2]) {
#pragma unroll
    for (int i = 0; i < H2; ++i) v[i] = make_float2(0.0f, 0.0f);
}

template <int H2>
__device__ __forceinline__ void vcopy2(float2 (&d)[H2], const float2 (&s)[H2]) {
#pragma unroll
    for (int i = 0; i < H2; ++i) d[i] = s[i];
}

// row += (v - v0) as a vector reduction at L2 (no lost updates under Hogwild).
template <int VEC>
__device__ __forceinline__ void red_add_delta(float* p, const float (&v)[VEC], const float (&v0)[VEC]) {
    if constexpr (VEC % 4 == 0) {
#pragma unroll
        for (int i = 0; i < VEC; i += 4)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p + i), "f"(v[i] - v0[i]),
                         "f"(v[i + 1] - v0[i + 1]), "f"(v[i + 2] - v0[i + 2]), "f"(v[i + 3] - v0[i + 3])
                         : "memory");
    } else if constexpr (VEC % 2 == 0) {
#pragma unroll
        for (int i = 0; i < VEC; i += 2)
            asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p + i), "f"(v[i] - v0[i]),
                         "f"(v[i + 1] - v0[i + 1])
                         : "memory");
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) atomicAdd(p + i, v[i] - v0[i]);
    }
}

// Per-lane VEC-float slice of a row parked in shared memory.
template <int VEC>
__device__ __forceinline__ void stash_put(float* p, const float (&v)[VEC]) {
    if constexpr (VEC % 4 == 0) {
#pragma unroll
        for (int i = 0; i < VEC; i += 4) *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) p[i] = v[i];
    }
}
template <int VEC>
__device__ __forceinline__ void stash_get(float (&v)[VEC], const float* p) {
    if constexpr (VEC % 4 == 0) {
#pragma unroll
        for (int i = 0; i < VEC; i += 4) {
            const float4 t = *reinterpret_cast<const float4*>(p + i);
            v[i] = t.x; v[i + 1] = t.y; v[i + 2] = t.z; v[i + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) v[i] = p[i];
    }
}

template <int VEC>
__device__ __forceinline__ void vzero(float (&v)[VEC]) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = 0.0f;
}

template <int VEC>
__device__ __forceinline__ void vcopy(float (&d)[VEC], const float (&s)[VEC]) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) d[i] = s[i];
}

template <int LANES>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
    for (int o = LANES / 2; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

__device__ __forceinline__ float tanh_approx(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// g = (label - sigma(clamp(f, -6, 6))) * alpha   (trainer.cpp:147, model.cpp:34-37)
template <bool FAST>
__device__ __forceinline__ float sgd_coeff(float f, float label, float alpha) {
    f = fminf(fmaxf(f, -6.0f), 6.0f);
    float sig;
    if constexpr (FAST) {
        sig = fmaf(0.5f, tanh_approx(0.5f * f), 0.5f);  // |err| < 1e-3 (SPEC fast-sigmoid bound)
    } else {
        sig = 1.0f / (1.0f + expf(-f));
    }
    return (label - sig) * alpha;
}

// Sentences of a kernel resident on the whole device at once
// (blocks per SM x SMs x sentences per block).
template <typename Kernel>
cudaError_t resident_sentences(Kernel kern, int smem_bytes, int threads, int sentences_per_block, int* out) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem_bytes);
    if (e == cudaSuccess) *out = per_sm * sms * sentences_per_block;
    return e;
}

// The fast coefficient with the constants folded: g = alpha*(label - 1/2)
// - (alpha/2)*tanh(clamp(f, -6, 6)/2) = (label - sigma(clamp(f)))*alpha, as one
// FFMA after the tanh. al = alpha*(label - 1/2), nha = -alpha/2.
// clamp(f, -6, 6) / 2. (6 * sat(f/12 + 1/2) - 3 saves an instruction but measured
// 4% slower in the lifetime staircase: profiles/r02dd_variants.txt.)
__device__ __forceinline__ float half_clamped(float f) { return fminf(fmaxf(0.5f * f, -3.0f), 3.0f); }
__device__ __forceinline__ float sgd_coeff_fast(float f, float al, float nha) {
    return fmaf(nha, tanh_approx(half_clamped(f)), al);
}

} // namespace fw2v
