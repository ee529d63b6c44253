// Exact-mode kernel instantiations.
#include "launch.cuh"

namespace tfb_host {
template int launch_exact<float>(const Pass&, const void*, void*, const void*, float, int, int, cudaStream_t);
template int launch_exact<double>(const Pass&, const void*, void*, const void*, double, int, int, cudaStream_t);
}  // namespace tfb_host
