// Instantiation of the tcgen05 GEMM for A-operand mode 5 (plain TMA A, deep pipeline) (see gemm_tc.cuh).
#include "gemm_tc.cuh"

namespace tn {
template void launch_kb<5>(int, __half*, const __half*, const __half*, uint64_t, uint32_t, uint32_t, const float*,
                            const float*, uint32_t*, int*, const OutMap*, cudaStream_t, const AGather*,
                            const NdPlan*, const BatchSpec*);
}  // namespace tn
