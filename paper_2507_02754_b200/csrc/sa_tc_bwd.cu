// sa_tc_bwd.cu -- tcgen05/TMEM/TMA backward (bf16 inputs).  Placeholder until the kernels land.
#include "sa_common.cuh"
namespace sa {
bool tc_bwd_supported(const Problem&) { return false; }
size_t tc_bwd_workspace_bytes(const Problem&) { return 0; }
cudaError_t tc_backward(const Problem&, bool, const void*, const void*, const void*, const void*, const void*,
                        const void*, const float*, const void*, void*, void*, void*, void*, void*, void*, size_t,
                        cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace sa
