// Chain map kernels (chain_impl.cuh) for window widths W = 1..4.
#include "chain_impl.cuh"

namespace epi::impl {
template bool launch_chain_w<1>(int, const CountLaunch&, cudaStream_t);
template bool launch_chain_w<2>(int, const CountLaunch&, cudaStream_t);
template bool launch_chain_w<3>(int, const CountLaunch&, cudaStream_t);
template bool launch_chain_w<4>(int, const CountLaunch&, cudaStream_t);
}  // namespace epi::impl
