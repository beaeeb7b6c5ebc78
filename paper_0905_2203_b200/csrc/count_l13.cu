// Pass-1 map kernels (last window relaxed to a launch-uniform hull), other
// windows of uniform width W = 13..16 (see count.cu, count_impl.cuh).
#include "count_impl.cuh"

namespace epi::impl {
template void launch_machines_l<13>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_l<14>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_l<15>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_l<16>(int, const CountLaunch&, cudaStream_t);
}  // namespace epi::impl
