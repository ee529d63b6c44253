// Fast-mode kernel instantiations: float, inverse.
#include "launch.cuh"

namespace tfb_host {
template int launch_fast<float, true>(const Pass&, const void*, void*, const void*, const void*, float, cudaStream_t);
}  // namespace tfb_host
