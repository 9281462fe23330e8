// GPU evaluation scans: nearest_neighbors and eval_analogy
// (reference eval.cpp:212-348) over the whole vocabulary, with the reference's
// arithmetic so the answers are identical:
//   * every dot product / squared norm is a double sum of float*float products
//     in column order (dot_rows / cosine, eval.cpp:104-115, 203-207) — no FMA,
//     sequential per (query, candidate) pair;
//   * unit_normalized rows (eval.cpp:185-199): scale = float(1/sqrt(norm)),
//     unit = row * scale in float;
//   * selection: nearest_neighbors by (cosine desc, id asc) (eval.cpp:336-339),
//     analogies by the first strictly greater score in id order (eval.cpp:245-266).
// One block per query; each thread scans a strided share of the vocabulary and
// keeps its best candidates, the block merges them. FP64 on CUDA cores: the
// per-pair cost is dim double adds, the bound is reading the matrix from L2/HBM.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "fw2v.h"

namespace fw2v {
void set_last_error(const std::string& msg);
}

namespace {

constexpr int kEvalThreads = 256;
constexpr int kMaxK = 32;
constexpr double kCosMulEpsilon = 0.001;  // eval.cpp:19

__device__ __forceinline__ double dot_seq(const float* a, const float* b, int dim) {
    double s = 0.0;
    for (int k = 0; k < dim; ++k) s = __dadd_rn(s, __dmul_rn(static_cast<double>(a[k]), static_cast<double>(b[k])));
    return s;
}

// Squared norms in double (cosine's nu/nv, unit_normalized's norm).
__global__ void k_sq_norms(const float* rows, int32_t n, int dim, double* out) {
    const int32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w < n) out[w] = dot_seq(rows + static_cast<size_t>(w) * dim, rows + static_cast<size_t>(w) * dim, dim);
}

// unit_normalized (eval.cpp:185-199).
__global__ void k_unit_rows(const float* rows, const double* sq, int32_t n, int dim, float* out) {
    const size_t total = static_cast<size_t>(n) * dim;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double norm = sqrt(sq[i / dim]);
        const float scale = norm > 0.0 ? static_cast<float>(1.0 / norm) : 0.0f;
        out[i] = __fmul_rn(rows[i], scale);
    }
}

struct Cand {
    double c;
    int32_t id;
};
__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {  // eval.cpp:336-339
    if (a.c != b.c) return a.c > b.c;
    return a.id < b.id;
}

// nearest_neighbors: block q -> query ids[q]; out: k (cos, id) pairs sorted.
__global__ void __launch_bounds__(kEvalThreads) k_nn(const float* rows, const double* sq, int32_t n, int dim,
                                                     const int32_t* queries, int k, int32_t* out_ids, double* out_cos) {
    extern __shared__ __align__(16) unsigned char eval_sh[];
    float* qrow = reinterpret_cast<float*>(eval_sh);
    Cand* pool = reinterpret_cast<Cand*>(eval_sh + ((dim * sizeof(float) + 15) & ~size_t(15)));
    const int32_t query = queries[blockIdx.x];
    for (int c = threadIdx.x; c < dim; c += blockDim.x) qrow[c] = rows[static_cast<size_t>(query) * dim + c];
    __syncthreads();
    const double sqrt_nu = sqrt(sq[query]);
    Cand best[kMaxK];
    int have = 0;
    for (int32_t x = threadIdx.x; x < n; x += blockDim.x) {
        if (x == query || sq[x] == 0.0) continue;  // query excluded, untrained (zero) rows skipped
        const double dot = dot_seq(qrow, rows + static_cast<size_t>(x) * dim, dim);
        const Cand cand{dot / (sqrt_nu * sqrt(sq[x])), x};  // cosine, eval.cpp:115
        if (have < k) {
            int j = have++;
            while (j > 0 && better(cand, best[j - 1])) { best[j] = best[j - 1]; --j; }
            best[j] = cand;
        } else if (better(cand, best[k - 1])) {
            int j = k - 1;
            while (j > 0 && better(cand, best[j - 1])) { best[j] = best[j - 1]; --j; }
            best[j] = cand;
        }
    }
    for (int j = 0; j < k; ++j) pool[threadIdx.x * k + j] = j < have ? best[j] : Cand{-INFINITY, -1};
    __syncthreads();
    // k rounds of a block argmax over the per-thread heads.
    __shared__ int head[kEvalThreads];
    __shared__ Cand red_c[kEvalThreads];
    __shared__ int red_t[kEvalThreads];
    head[threadIdx.x] = 0;
    __syncthreads();
    for (int r = 0; r < k; ++r) {
        const int h = head[threadIdx.x];
        red_c[threadIdx.x] = h < k ? pool[threadIdx.x * k + h] : Cand{-INFINITY, -1};
        red_t[threadIdx.x] = threadIdx.x;
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) {
                const Cand o = red_c[threadIdx.x + s];
                if (o.id >= 0 && (red_c[threadIdx.x].id < 0 || better(o, red_c[threadIdx.x]))) {
                    red_c[threadIdx.x] = o;
                    red_t[threadIdx.x] = red_t[threadIdx.x + s];
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            out_ids[static_cast<size_t>(blockIdx.x) * k + r] = red_c[0].id;
            out_cos[static_cast<size_t>(blockIdx.x) * k + r] = red_c[0].id >= 0 ? red_c[0].c : NAN;
            if (red_c[0].id >= 0) ++head[red_t[0]];
        }
        __syncthreads();
    }
}

// eval_analogy solve (eval.cpp:236-268) over unit rows: block q -> quadruple q.
__global__ void __launch_bounds__(kEvalThreads) k_analogy(const float* unit, int32_t n, int dim, const int32_t* quads,
                                                          int method, int32_t* out_pred) {
    extern __shared__ __align__(16) unsigned char eval_sh[];
    float* qv = reinterpret_cast<float*>(eval_sh);  // cos_add: b - a + a*; cos_mul: b, a*, a
    const int32_t a = quads[4 * blockIdx.x], as = quads[4 * blockIdx.x + 1], b = quads[4 * blockIdx.x + 2];
    const float* va = unit + static_cast<size_t>(a) * dim;
    const float* vas = unit + static_cast<size_t>(as) * dim;
    const float* vb = unit + static_cast<size_t>(b) * dim;
    for (int c = threadIdx.x; c < dim; c += blockDim.x) {
        if (method == 0) {
            qv[c] = __fadd_rn(__fsub_rn(vb[c], va[c]), vas[c]);
        } else {
            qv[c] = vb[c];
            qv[dim + c] = vas[c];
            qv[2 * dim + c] = va[c];
        }
    }
    __syncthreads();
    Cand best{-INFINITY, -1};
    for (int32_t x = threadIdx.x; x < n; x += blockDim.x) {
        if (x == a || x == as || x == b) continue;
        const float* vx = unit + static_cast<size_t>(x) * dim;
        double score;
        if (method == 0) {
            score = dot_seq(vx, qv, dim);
        } else {
            const double cb = (dot_seq(vx, qv, dim) + 1.0) / 2.0;
            const double cas = (dot_seq(vx, qv + dim, dim) + 1.0) / 2.0;
            const double ca = (dot_seq(vx, qv + 2 * dim, dim) + 1.0) / 2.0;
            score = cb * cas / (ca + kCosMulEpsilon);
        }
        if (score > best.c) best = Cand{score, x};  // ascending x: first maximum kept
    }
    __shared__ Cand red[kEvalThreads];
    red[threadIdx.x] = best;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const Cand o = red[threadIdx.x + s];
            // the reference keeps the lowest id among equal maxima
            if (o.id >= 0 && (red[threadIdx.x].id < 0 || o.c > red[threadIdx.x].c ||
                              (o.c == red[threadIdx.x].c && o.id < red[threadIdx.x].id)))
                red[threadIdx.x] = o;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out_pred[blockIdx.x] = red[0].id;
}

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() { cudaFree(p); }
};

int cuda_fail(cudaError_t e) {
    fw2v::set_last_error(std::string("CUDA: ") + cudaGetErrorString(e));
    return FW2V_ERR_CUDA;
}

#define EVAL_CK(x)                               \
    do {                                         \
        cudaError_t e_ = (x);                    \
        if (e_ != cudaSuccess) return cuda_fail(e_); \
    } while (0)

}  // namespace

extern "C" {

int fw2v_nearest_neighbors(const float* rows, int32_t vocab_size, int32_t dim, const int32_t* queries,
                           int32_t n_queries, int32_t k, int32_t* out_ids, double* out_cos) {
    if (rows == nullptr || queries == nullptr || out_ids == nullptr || out_cos == nullptr || vocab_size < 2 || dim < 1 ||
        n_queries < 0) {
        fw2v::set_last_error("nearest_neighbors: bad arguments");
        return FW2V_ERR_BAD_ARGUMENT;
    }
    if (k < 1 || k >= vocab_size || k > kMaxK) {  // eval.cpp:308-310 (+ the kernel's k <= 32)
        fw2v::set_last_error("k must be in [1, |V|-1] (and <= 32)");
        return FW2V_ERR_BAD_ARGUMENT;
    }
    for (int32_t q = 0; q < n_queries; ++q)
        if (queries[q] < 0 || queries[q] >= vocab_size) {
            fw2v::set_last_error("query id out of vocabulary");
            return FW2V_ERR_OOV_QUERY;
        }
    if (n_queries == 0) return FW2V_OK;
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
        fw2v::set_last_error("no CUDA device (there is no CPU evaluation path)");
        return FW2V_ERR_NO_DEVICE;
    }
    const size_t nrow = static_cast<size_t>(vocab_size) * dim;
    DevBuf d_rows, d_sq, d_q, d_ids, d_cos;
    EVAL_CK(cudaMalloc(&d_rows.p, nrow * sizeof(float)));
    EVAL_CK(cudaMalloc(&d_sq.p, static_cast<size_t>(vocab_size) * sizeof(double)));
    EVAL_CK(cudaMalloc(&d_q.p, static_cast<size_t>(n_queries) * sizeof(int32_t)));
    EVAL_CK(cudaMalloc(&d_ids.p, static_cast<size_t>(n_queries) * k * sizeof(int32_t)));
    EVAL_CK(cudaMalloc(&d_cos.p, static_cast<size_t>(n_queries) * k * sizeof(double)));
    EVAL_CK(cudaMemcpy(d_rows.p, rows, nrow * sizeof(float), cudaMemcpyHostToDevice));
    EVAL_CK(cudaMemcpy(d_q.p, queries, static_cast<size_t>(n_queries) * sizeof(int32_t), cudaMemcpyHostToDevice));
    const float* r = static_cast<const float*>(d_rows.p);
    double* sq = static_cast<double*>(d_sq.p);
    k_sq_norms<<<(vocab_size + 255) / 256, 256>>>(r, vocab_size, dim, sq);
    EVAL_CK(cudaGetLastError());
    std::vector<double> hsq(static_cast<size_t>(vocab_size));
    EVAL_CK(cudaMemcpy(hsq.data(), sq, hsq.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (int32_t q = 0; q < n_queries; ++q)
        if (hsq[static_cast<size_t>(queries[q])] == 0.0) {  // eval.cpp:311-316
            fw2v::set_last_error("query vector is zero");
            return FW2V_ERR_ZERO_VECTOR;
        }
    const size_t smem = ((dim * sizeof(float) + 15) & ~size_t(15)) + sizeof(Cand) * kEvalThreads * k;
    EVAL_CK(cudaFuncSetAttribute(k_nn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_nn<<<n_queries, kEvalThreads, smem>>>(r, sq, vocab_size, dim, static_cast<const int32_t*>(d_q.p), k,
                                             static_cast<int32_t*>(d_ids.p), static_cast<double*>(d_cos.p));
    EVAL_CK(cudaGetLastError());
    EVAL_CK(cudaMemcpy(out_ids, d_ids.p, static_cast<size_t>(n_queries) * k * sizeof(int32_t), cudaMemcpyDeviceToHost));
    EVAL_CK(cudaMemcpy(out_cos, d_cos.p, static_cast<size_t>(n_queries) * k * sizeof(double), cudaMemcpyDeviceToHost));
    return FW2V_OK;
}

int fw2v_eval_analogy(const float* rows, int32_t vocab_size, int32_t dim, const int32_t* quads, int32_t n,
                      int32_t method, int32_t* out_pred) {
    if (rows == nullptr || quads == nullptr || out_pred == nullptr || vocab_size < 1 || dim < 1 || n < 0 ||
        (method != 0 && method != 1)) {
        fw2v::set_last_error("eval_analogy: bad arguments");
        return FW2V_ERR_BAD_ARGUMENT;
    }
    for (int32_t i = 0; i < 4 * n; ++i)
        if (quads[i] < 0 || quads[i] >= vocab_size) {
            fw2v::set_last_error("analogy word id out of vocabulary");
            return FW2V_ERR_OOV_QUERY;
        }
    if (n == 0) return FW2V_OK;
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
        fw2v::set_last_error("no CUDA device (there is no CPU evaluation path)");
        return FW2V_ERR_NO_DEVICE;
    }
    const size_t nrow = static_cast<size_t>(vocab_size) * dim;
    DevBuf d_rows, d_unit, d_sq, d_quads, d_pred;
    EVAL_CK(cudaMalloc(&d_rows.p, nrow * sizeof(float)));
    EVAL_CK(cudaMalloc(&d_unit.p, nrow * sizeof(float)));
    EVAL_CK(cudaMalloc(&d_sq.p, static_cast<size_t>(vocab_size) * sizeof(double)));
    EVAL_CK(cudaMalloc(&d_quads.p, static_cast<size_t>(n) * 4 * sizeof(int32_t)));
    EVAL_CK(cudaMalloc(&d_pred.p, static_cast<size_t>(n) * sizeof(int32_t)));
    EVAL_CK(cudaMemcpy(d_rows.p, rows, nrow * sizeof(float), cudaMemcpyHostToDevice));
    EVAL_CK(cudaMemcpy(d_quads.p, quads, static_cast<size_t>(n) * 4 * sizeof(int32_t), cudaMemcpyHostToDevice));
    const float* r = static_cast<const float*>(d_rows.p);
    double* sq = static_cast<double*>(d_sq.p);
    float* unit = static_cast<float*>(d_unit.p);
    k_sq_norms<<<(vocab_size + 255) / 256, 256>>>(r, vocab_size, dim, sq);
    k_unit_rows<<<148 * 8, 256>>>(r, sq, vocab_size, dim, unit);
    const size_t smem = 3 * dim * sizeof(float);
    EVAL_CK(cudaFuncSetAttribute(k_analogy, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_analogy<<<n, kEvalThreads, smem>>>(unit, vocab_size, dim, static_cast<const int32_t*>(d_quads.p), method,
                                          static_cast<int32_t*>(d_pred.p));
    EVAL_CK(cudaGetLastError());
    EVAL_CK(cudaMemcpy(out_pred, d_pred.p, static_cast<size_t>(n) * sizeof(int32_t), cudaMemcpyDeviceToHost));
    return FW2V_OK;
}

}  // extern "C"
