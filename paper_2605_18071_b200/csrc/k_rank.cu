// k_rank.cu — rank_kernel instantiations (see select.cuh), compiled in parallel with the rest.
#include "select.cuh"

namespace kvd {
template cudaError_t launch_rank_nt<512, false>(kvd_cache*, const StepParams&, float*, int, int, int32_t*, float*,
                                               const FuseArgs&, cudaStream_t);
template cudaError_t launch_rank_nt<512, true>(kvd_cache*, const StepParams&, float*, int, int, int32_t*, float*,
                                              const FuseArgs&, cudaStream_t);
template cudaError_t launch_rank_nt<1024, false>(kvd_cache*, const StepParams&, float*, int, int, int32_t*, float*,
                                                const FuseArgs&, cudaStream_t);
template cudaError_t launch_rank_nt<1024, true>(kvd_cache*, const StepParams&, float*, int, int, int32_t*, float*,
                                               const FuseArgs&, cudaStream_t);
}  // namespace kvd
