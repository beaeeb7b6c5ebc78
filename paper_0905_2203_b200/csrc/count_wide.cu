// Wide-window instantiations (some constraint high > 63, up to 4095): per-
// position history in a 128-word local-memory ring. See count_impl.cuh.
#include "count_impl.cuh"

namespace epi {
namespace {

template <int N>
using Wide128 = impl::WideHist<N, 128>;

using Wide128All = impl::Dispatch<Wide128, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>;

}  // namespace

void launch_machines_wide(int n_nodes, const CountLaunch& p, cudaStream_t st) {
  Wide128All::machines(n_nodes, p, st);
}

void launch_walk_wide(int n_nodes, const CountLaunch& p, cudaStream_t st) {
  Wide128All::walk(n_nodes, p, st);
}

}  // namespace epi
