// Fast-mode kernel instantiations: float, inverse.
#include "launch.cuh"

namespace tfb_host {
template int launch_fast<float, true>(const Pass&, const void*, void*, const void*, const void*, float, cudaStream_t);
template int launch_dist_pass1<float, true>(const DistPass1&, const void*, const void*, const void*, float,
                                              cudaStream_t);
}  // namespace tfb_host
