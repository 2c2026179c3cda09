// Instantiation of the tcgen05 GEMM for A-operand mode 4 (4-byte cp.async gather) (see gemm_tc.cuh).
#include "gemm_tc.cuh"

namespace tn {
template void launch_kb<4>(int, __half*, const __half*, const __half*, uint64_t, uint32_t, uint32_t, const float*,
                            const float*, uint32_t*, int*, const OutMap*, cudaStream_t, const AGather*,
                            const NdPlan*, const BatchSpec*);
}  // namespace tn
