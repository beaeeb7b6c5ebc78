// Map kernels specialised on launch-uniform window width W = 9..12 (see count.cu).
#include "count_impl.cuh"

namespace epi::impl {
template void launch_machines_w<9>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_w<10>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_w<11>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_w<12>(int, const CountLaunch&, cudaStream_t);
}  // namespace epi::impl
