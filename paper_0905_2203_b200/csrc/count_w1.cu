// Map kernels specialised on launch-uniform window width W = 1..4 (see count.cu).
#include "count_impl.cuh"

namespace epi::impl {
template void launch_machines_w<1>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_w<2>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_w<3>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_w<4>(int, const CountLaunch&, cudaStream_t);
}  // namespace epi::impl
