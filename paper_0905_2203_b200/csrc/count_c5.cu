// Chain map kernels (chain_impl.cuh) for window widths W = 5..8.
#include "chain_impl.cuh"

namespace epi::impl {
template bool launch_chain_w<5>(int, const CountLaunch&, cudaStream_t);
template bool launch_chain_w<6>(int, const CountLaunch&, cudaStream_t);
template bool launch_chain_w<7>(int, const CountLaunch&, cudaStream_t);
template bool launch_chain_w<8>(int, const CountLaunch&, cudaStream_t);
}  // namespace epi::impl
