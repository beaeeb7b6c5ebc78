// Map kernels specialised on launch-uniform window width W = 13..16 (see count.cu).
#include "count_impl.cuh"

namespace epi::impl {
template void launch_machines_w<13>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_w<14>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_w<15>(int, const CountLaunch&, cudaStream_t);
template void launch_machines_w<16>(int, const CountLaunch&, cudaStream_t);
}  // namespace epi::impl
