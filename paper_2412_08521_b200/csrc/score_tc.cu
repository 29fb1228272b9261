// score_tc.cu -- tcgen05/TMEM/TMA score pass (bf16, head_dim 128).  Placeholder
// until the tensor-core kernels land; AUTO falls back to the SIMT pass.
#include "common.cuh"

namespace ems {
size_t score_tc_workspace(const Dims&) { return 0; }
bool score_tc_supported(const Dims&, int) { return false; }
cudaError_t score_tc(const Dims&, const void*, const void*, const void*, void*, float*, float*,
                     float*, void*, cudaStream_t) {
    return cudaErrorNotSupported;
}
}  // namespace ems
