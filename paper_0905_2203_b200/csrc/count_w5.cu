// Map kernels specialised on launch-uniform window width W = 5..8 (see count.cu).
#include "count_impl.cuh"

namespace epi::impl {
template void launch_machines_w<5>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_w<6>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_w<7>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_w<8>(int, const CountLaunch&, cudaStream_t);
}  // namespace epi::impl
