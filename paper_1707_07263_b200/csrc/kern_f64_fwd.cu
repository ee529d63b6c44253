// Fast-mode kernel instantiations: double, forward.
#include "launch.cuh"

namespace tfb_host {
template int launch_fast<double, false>(const Pass&, const void*, void*, const void*, const void*, double, cudaStream_t);
template int launch_dist_pass1<double, false>(const DistPass1&, const void*, const void*, const void*, double,
                                              cudaStream_t);
}  // namespace tfb_host
