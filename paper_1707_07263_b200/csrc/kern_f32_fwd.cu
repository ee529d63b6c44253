// Fast-mode kernel instantiations: float, forward.
#include "launch.cuh"

namespace tfb_host {
template int launch_fast<float, false>(const Pass&, const void*, void*, const void*, const void*, float, cudaStream_t);
template int launch_dist_pass1<float, false>(const DistPass1&, const void*, const void*, const void*, float,
                                              cudaStream_t);
}  // namespace tfb_host

