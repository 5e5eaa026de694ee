// k_select_nt1024.cu — select_kernel instantiations with 1024-thread CTAs (see select.cuh).
#include "select.cuh"

namespace kvd {
template cudaError_t launch_select_nt<1024, false>(kvd_cache*, const StepParams&, const uint16_t*, const uint16_t*,
                                                 float*, int, int, int, int32_t*, float*, const FuseArgs&, cudaStream_t);
template cudaError_t launch_select_nt<1024, true>(kvd_cache*, const StepParams&, const uint16_t*, const uint16_t*,
                                                float*, int, int, int, int32_t*, float*, const FuseArgs&, cudaStream_t);
}  // namespace kvd
