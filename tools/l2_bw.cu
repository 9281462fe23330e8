// Measured L2 bandwidth on this B200 (roofline denominator for L2-resident
// kernels): read-only, read-modify-write (ld + st) and red.global.add.v4 over
// an L2-resident buffer (16-64 MB < 126 MB L2), 128-bit accesses, grid =
// 148 SMs x 8 blocks, CUDA events, best of 20 after warm-up.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_bw tools/l2_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const float4* __restrict__ a, size_t n4, int reps, float* out) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
            float4 v = __ldcg(a + i);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) out[0] = acc.x;
}
__global__ void rmw(float4* __restrict__ a, size_t n4, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
            float4 v = __ldcg(a + i);
            v.x += 1.f; v.y += 1.f; v.z += 1.f; v.w += 1.f;
            __stcg(a + i, v);
        }
}
__global__ void red(float* __restrict__ a, size_t n4, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %1, %1, %1};" ::"l"(a + 4 * i), "f"(1.0f) : "memory");
}

int main() {
    const size_t sizes[] = {16u << 20, 32u << 20, 64u << 20};
    float* buf;
    float* out;
    cudaMalloc(&buf, 64u << 20);
    cudaMalloc(&out, 16);
    cudaMemset(buf, 0, 64u << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 148 * 8, threads = 256, reps = 20;
    for (size_t bytes : sizes) {
        const size_t n4 = bytes / 16;
        for (int kind = 0; kind < 3; ++kind) {
            float best = 1e30f;
            for (int it = 0; it < 22; ++it) {
                cudaEventRecord(e0);
                if (kind == 0) rd<<<blocks, threads>>>((const float4*)buf, n4, reps, out);
                else if (kind == 1) rmw<<<blocks, threads>>>((float4*)buf, n4, reps);
                else red<<<blocks, threads>>>(buf, n4, reps);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (it >= 2 && ms < best) best = ms;
            }
            const double moved = (kind == 1 ? 2.0 : 1.0) * bytes * reps;
            printf("{\"buffer_mb\": %zu, \"kind\": \"%s\", \"GBps\": %.1f}\n", bytes >> 20,
                   kind == 0 ? "read" : kind == 1 ? "read+write" : "red.add.v4", moved / (best * 1e-3) / 1e9);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
