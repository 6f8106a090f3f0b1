// sa_tc_fwd.cu -- tcgen05/TMEM/TMA forward (bf16 inputs).  Placeholder until the kernel lands.
#include "sa_common.cuh"
namespace sa {
bool tc_fwd_supported(const Problem&) { return false; }
cudaError_t tc_forward(const Problem&, bool, const void*, const void*, const void*, const void*, const void*,
                       void*, float*, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace sa
