// K1s instantiation for 64 lanes x 8 columns: d = 512 on two warps per sentence,
// one translation unit per shape.
#include "fw2v_snapshot.cuh"

namespace fw2v {
template cudaError_t launch_k1s_shape<64, 8>(const ModelView&, const BatchView&, int, int, bool, bool,
                                              DevCounters*, cudaStream_t, int*);
} // namespace fw2v
