// Pass-1 map kernels (last window relaxed to a launch-uniform hull), other
// windows of uniform width W = 9..12 (see count.cu, count_impl.cuh).
#include "count_impl.cuh"

namespace epi::impl {
template void launch_machines_l<9>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_l<10>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_l<11>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_l<12>(int, const CountLaunch&, cudaStream_t);
}  // namespace epi::impl
