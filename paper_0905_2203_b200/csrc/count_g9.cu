// Generic narrow-window kernels (runtime window widths, high <= 63) for
// episodes of 9..16 nodes; N 1..8 live in count.cu. See count_impl.cuh.
#include "count_impl.cuh"

namespace epi {

using NarrowHi =
    impl::Dispatch<impl::NarrowW<0, false>::template H, 9, 10, 11, 12, 13, 14, 15, 16>;

void launch_machines_generic_hi(int n_nodes, const CountLaunch& p, cudaStream_t st) {
  NarrowHi::machines(n_nodes, p, st);
}

void launch_walk_generic_hi(int n_nodes, const CountLaunch& p, cudaStream_t st) {
  NarrowHi::walk(n_nodes, p, st);
}

}  // namespace epi
