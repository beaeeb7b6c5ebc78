// Pass-1 map kernels (last window relaxed to a launch-uniform hull), other
// windows of uniform width W = 5..8 (see count.cu, count_impl.cuh).
#include "count_impl.cuh"

namespace epi::impl {
template void launch_machines_l<5>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_l<6>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_l<7>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_l<8>(int, const CountLaunch&, cudaStream_t);
}  // namespace epi::impl
