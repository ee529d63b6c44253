// Exact-mode kernel instantiations.
#include "launch.cuh"

namespace tfb_host {
template int launch_exact<float>(const Pass&, const void*, void*, const void*, float, int, int, cudaStream_t);
template int launch_exact<double>(const Pass&, const void*, void*, const void*, double, int, int, cudaStream_t);
template int launch_levelwise<float>(const Pass&, const void*, void*, const void*, float, int, int, cudaStream_t);
template int launch_levelwise<double>(const Pass&, const void*, void*, const void*, double, int, int, cudaStream_t);
template int launch_exchange<float>(const void*, void*, const tfb::ExchangeArgs&, cudaStream_t);
template int launch_exchange<double>(const void*, void*, const tfb::ExchangeArgs&, cudaStream_t);
template int launch_interstage<float>(const void*, void*, long long, long long, long long, long long, long long,
                                      const void*, long long, cudaStream_t);
template int launch_interstage<double>(const void*, void*, long long, long long, long long, long long, long long,
                                       const void*, long long, cudaStream_t);
}  // namespace tfb_host
