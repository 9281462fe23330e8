// K1s dispatch: shape (lanes x columns) -> the instantiation compiled in
// k1s_l<L>v<V>.cu. The kernel itself is in fw2v_snapshot.cuh.
#include "fw2v_snapshot.cuh"

namespace fw2v {

#define FW2V_K1S_SHAPES(X) X(4, 4) X(8, 4) X(16, 4) X(16, 8) X(32, 4) X(32, 6) X(32, 8) X(32, 10) X(32, 12) X(32, 16) X(64, 8)

#define FW2V_EXTERN(L_, V_)                                                                                 \
    extern template cudaError_t launch_k1s_shape<L_, V_>(const ModelView&, const BatchView&, int, int, bool, bool, \
                                                         DevCounters*, cudaStream_t, int*);
FW2V_K1S_SHAPES(FW2V_EXTERN)
#undef FW2V_EXTERN

cudaError_t launch_k1s(int lanes, int vec, const ModelView& m, const BatchView& b, int n_neg, int wf, bool fast,
                       bool lifetime, DevCounters* ctr, cudaStream_t st, int* resident) {
#define FW2V_CASE(L_, V_) \
    if (lanes == L_ && vec == V_) return launch_k1s_shape<L_, V_>(m, b, n_neg, wf, fast, lifetime, ctr, st, resident);
    FW2V_K1S_SHAPES(FW2V_CASE)
#undef FW2V_CASE
    return cudaErrorInvalidValue;
}

// Any N: N + 1 <= 6 samples run as one chunk with the negatives in registers,
// more as chunks of 4 or 6 loaded per window (lifetime order: one wavefront per
// chunk). Lifetime order up to 10 columns per lane.
bool k1s_supported(int lanes, int vec, int n_neg, int wf, bool lifetime) {
    if (n_neg < 0 || wf < 1 || wf > 5 || (!lifetime && n_neg + 1 > kMaxSnapSamples)) return false;
    if (lifetime && vec > 10) return false;  // the window's sample rows no longer fit in registers
#define FW2V_CASE(L_, V_) if (lanes == L_ && vec == V_) return true;
    FW2V_K1S_SHAPES(FW2V_CASE)
#undef FW2V_CASE
    return false;
}

} // namespace fw2v
