// Chain map kernels (chain_impl.cuh) for window widths W = 9..12.
#include "chain_impl.cuh"

namespace epi::impl {
template bool launch_chain_w<9>(int, const CountLaunch&, cudaStream_t);
template bool launch_chain_w<10>(int, const CountLaunch&, cudaStream_t);
template bool launch_chain_w<11>(int, const CountLaunch&, cudaStream_t);
template bool launch_chain_w<12>(int, const CountLaunch&, cudaStream_t);
}  // namespace epi::impl
