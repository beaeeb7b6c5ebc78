// Pass-1 map kernels (last window relaxed to a launch-uniform hull), other
// windows of uniform width W = 1..4 (see count.cu, count_impl.cuh).
#include "count_impl.cuh"

namespace epi::impl {
template void launch_machines_l<1>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_l<2>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_l<3>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_l<4>(int, const CountLaunch&, cudaStream_t);
}  // namespace epi::impl
