// Fast-mode kernel instantiations: double, inverse.
#include "launch.cuh"

namespace tfb_host {
template int launch_fast<double, true>(const Pass&, const void*, void*, const void*, const void*, double, cudaStream_t);
template int launch_dist_pass1<double, true>(const DistPass1&, const void*, const void*, const void*, double,
                                              cudaStream_t);
}  // namespace tfb_host
