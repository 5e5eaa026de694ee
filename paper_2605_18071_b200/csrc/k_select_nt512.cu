// k_select_nt512.cu — select_kernel instantiations with 512-thread CTAs (see select.cuh).
#include "select.cuh"

namespace kvd {
template cudaError_t launch_select_nt<512, false>(kvd_cache*, const StepParams&, const uint16_t*, const uint16_t*,
                                                 float*, int, int, int, int32_t*, float*, const FuseArgs&, cudaStream_t);
template cudaError_t launch_select_nt<512, true>(kvd_cache*, const StepParams&, const uint16_t*, const uint16_t*,
                                                float*, int, int, int, int32_t*, float*, const FuseArgs&, cudaStream_t);
}  // namespace kvd
