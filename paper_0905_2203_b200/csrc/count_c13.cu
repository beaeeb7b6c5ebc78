// Chain map kernels (chain_impl.cuh) for window widths W = 13..16.
#include "chain_impl.cuh"

namespace epi::impl {
template bool launch_chain_w<13>(int, const CountLaunch&, cudaStream_t);
template bool launch_chain_w<14>(int, const CountLaunch&, cudaStream_t);
template bool launch_chain_w<15>(int, const CountLaunch&, cudaStream_t);
template bool launch_chain_w<16>(int, const CountLaunch&, cudaStream_t);
}  // namespace epi::impl
