// K1s instantiation for 32 lanes x 16 columns (one translation unit per shape
// so the sm_100a build compiles them in parallel).
#include "fw2v_snapshot.cuh"

namespace fw2v {
template cudaError_t launch_k1s_shape<32, 16>(const ModelView&, const BatchView&, int, int, bool, bool,
                                               DevCounters*, cudaStream_t, int*);
} // namespace fw2v
