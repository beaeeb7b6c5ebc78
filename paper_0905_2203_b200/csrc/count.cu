// Narrow-window instantiations (every constraint high <= 63): per-position
// history in two registers. See count_impl.cuh.
//   * generic kernels (runtime window widths), N = 1..16, map + walk;
//   * map kernels specialised on a launch-uniform window width W = high-low
//     in 1..16 for N = 2..8 (count_w*.cu) - the shape of every mining level
//     over a constraint alphabet of equal-width bins.
#include "count_impl.cuh"

namespace epi {
namespace impl {
template <int W>
bool launch_chain_w(int n, const CountLaunch& p, cudaStream_t st);
}

#define EPI_EXTERN_C(W) \
  extern template bool impl::launch_chain_w<W>(int, const CountLaunch&, cudaStream_t);
EPI_EXTERN_C(1) EPI_EXTERN_C(2) EPI_EXTERN_C(3) EPI_EXTERN_C(4)
EPI_EXTERN_C(5) EPI_EXTERN_C(6) EPI_EXTERN_C(7) EPI_EXTERN_C(8)
EPI_EXTERN_C(9) EPI_EXTERN_C(10) EPI_EXTERN_C(11) EPI_EXTERN_C(12)
EPI_EXTERN_C(13) EPI_EXTERN_C(14) EPI_EXTERN_C(15) EPI_EXTERN_C(16)
#undef EPI_EXTERN_C

bool has_chain_kernel(int n_nodes, int width, bool hi32) {
  return hi32 && n_nodes >= 2 && n_nodes <= 8 && width >= 1 && width <= 16;
}

bool launch_chain(int n_nodes, int width, const CountLaunch& p, cudaStream_t st) {
  if (!has_chain_kernel(n_nodes, width, true)) return false;
  switch (width) {
#define EPI_CASE_C(W) \
  case W:             \
    return impl::launch_chain_w<W>(n_nodes, p, st);
    EPI_CASE_C(1) EPI_CASE_C(2) EPI_CASE_C(3) EPI_CASE_C(4)
    EPI_CASE_C(5) EPI_CASE_C(6) EPI_CASE_C(7) EPI_CASE_C(8)
    EPI_CASE_C(9) EPI_CASE_C(10) EPI_CASE_C(11) EPI_CASE_C(12)
    EPI_CASE_C(13) EPI_CASE_C(14) EPI_CASE_C(15) EPI_CASE_C(16)
#undef EPI_CASE_C
  }
  return false;
}

#define EPI_EXTERN_W(W) \
  extern template void impl::launch_machines_w<W>(int, const CountLaunch&, cudaStream_t);
EPI_EXTERN_W(1) EPI_EXTERN_W(2) EPI_EXTERN_W(3) EPI_EXTERN_W(4)
EPI_EXTERN_W(5) EPI_EXTERN_W(6) EPI_EXTERN_W(7) EPI_EXTERN_W(8)
EPI_EXTERN_W(9) EPI_EXTERN_W(10) EPI_EXTERN_W(11) EPI_EXTERN_W(12)
EPI_EXTERN_W(13) EPI_EXTERN_W(14) EPI_EXTERN_W(15) EPI_EXTERN_W(16)
#undef EPI_EXTERN_W
#define EPI_EXTERN_L(W) \
  extern template void impl::launch_machines_l<W>(int, const CountLaunch&, cudaStream_t);
EPI_EXTERN_L(1) EPI_EXTERN_L(2) EPI_EXTERN_L(3) EPI_EXTERN_L(4)
EPI_EXTERN_L(5) EPI_EXTERN_L(6) EPI_EXTERN_L(7) EPI_EXTERN_L(8)
EPI_EXTERN_L(9) EPI_EXTERN_L(10) EPI_EXTERN_L(11) EPI_EXTERN_L(12)
EPI_EXTERN_L(13) EPI_EXTERN_L(14) EPI_EXTERN_L(15) EPI_EXTERN_L(16)
#undef EPI_EXTERN_L

bool launch_machines_last(int n_nodes, int width, uint32_t w_last, CountLaunch& p, cudaStream_t st) {
  if (n_nodes < 3 || n_nodes > 6 || width < 1 || width > 16 || w_last < 1 || w_last > 16) return false;
  smear_shifts(w_last, p.last_sh);
  switch (width) {
#define EPI_CASE_L(W) \
  case W:             \
    impl::launch_machines_l<W>(n_nodes, p, st); \
    return true;
    EPI_CASE_L(1) EPI_CASE_L(2) EPI_CASE_L(3) EPI_CASE_L(4)
    EPI_CASE_L(5) EPI_CASE_L(6) EPI_CASE_L(7) EPI_CASE_L(8)
    EPI_CASE_L(9) EPI_CASE_L(10) EPI_CASE_L(11) EPI_CASE_L(12)
    EPI_CASE_L(13) EPI_CASE_L(14) EPI_CASE_L(15) EPI_CASE_L(16)
#undef EPI_CASE_L
  }
  return false;
}

int32_t stages_for(uint32_t blk_words) {
  const uint32_t bytes = blk_words * 4u;
  if (bytes <= 16u * 1024u) return 3;
  if (bytes <= 48u * 1024u) return 2;
  return 0;  // very large alphabets: rows read from global memory via L1
}

// Generic (runtime-width) kernels: N 1..8 here, N 9..16 in count_g9.cu.
using NarrowLo = impl::Dispatch<impl::NarrowW<0, false>::template H, 1, 2, 3, 4, 5, 6, 7, 8>;
void launch_machines_generic_hi(int n_nodes, const CountLaunch& p, cudaStream_t st);
void launch_walk_generic_hi(int n_nodes, const CountLaunch& p, cudaStream_t st);

struct NarrowAll {
  static void machines(int n, const CountLaunch& p, cudaStream_t st) {
    if (n <= 8)
      NarrowLo::machines(n, p, st);
    else
      launch_machines_generic_hi(n, p, st);
  }
  static void walk(int n, const CountLaunch& p, cudaStream_t st) {
    if (n <= 8)
      NarrowLo::walk(n, p, st);
    else
      launch_walk_generic_hi(n, p, st);
  }
};

bool has_uniform_kernel(int n_nodes, int width, bool hi32) {
  return hi32 && n_nodes >= 2 && n_nodes <= 8 && width >= 1 && width <= 16;
}

void launch_machines(int n_nodes, int width, bool hi32, const CountLaunch& p, cudaStream_t st) {
  if (!has_uniform_kernel(n_nodes, width, hi32)) {
    NarrowAll::machines(n_nodes, p, st);
    return;
  }
  switch (width) {
#define EPI_CASE_W(W) \
  case W:             \
    impl::launch_machines_w<W>(n_nodes, p, st); \
    return;
    EPI_CASE_W(1) EPI_CASE_W(2) EPI_CASE_W(3) EPI_CASE_W(4)
    EPI_CASE_W(5) EPI_CASE_W(6) EPI_CASE_W(7) EPI_CASE_W(8)
    EPI_CASE_W(9) EPI_CASE_W(10) EPI_CASE_W(11) EPI_CASE_W(12)
    EPI_CASE_W(13) EPI_CASE_W(14) EPI_CASE_W(15) EPI_CASE_W(16)
#undef EPI_CASE_W
  }
  NarrowAll::machines(n_nodes, p, st);
}

void launch_walk(int n_nodes, const CountLaunch& p, cudaStream_t st) {
  NarrowAll::walk(n_nodes, p, st);
}


namespace {
// Single-node episodes: every distinct firing time of the type is one
// completion (pe = t, and the next time is > t), so the count is the
// popcount of the type's bitmap rows. One thread per (episode, block).
__global__ void singletons_kernel(const uint32_t* __restrict__ occ, uint32_t blk_words,
                                  uint32_t n_blocks, const uint32_t* __restrict__ types,
                                  uint32_t n_eps, unsigned long long* counts) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<uint64_t>(n_eps) * n_blocks) return;
  const uint32_t e = static_cast<uint32_t>(i / n_blocks), b = static_cast<uint32_t>(i % n_blocks);
  const uint4* row = reinterpret_cast<const uint4*>(occ + static_cast<size_t>(b) * blk_words +
                                                    types[e] * kRowStride);
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kBlkTiles / 4; ++j) {
    const uint4 v = __ldg(row + j);
    c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
  }
  if (c) atomicAdd(counts + e, static_cast<unsigned long long>(c));
}
}  // namespace

void launch_singletons(const uint32_t* occ, uint32_t blk_words, uint32_t n_blocks,
                       const uint32_t* types, uint32_t n_eps, uint64_t* counts, cudaStream_t st) {
  EPI_CUDA(cudaMemsetAsync(counts, 0, static_cast<size_t>(n_eps) * sizeof(uint64_t), st));
  const uint64_t threads = static_cast<uint64_t>(n_eps) * n_blocks;
  if (threads == 0) return;
  singletons_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(
      occ, blk_words, n_blocks, types, n_eps, reinterpret_cast<unsigned long long*>(counts));
  EPI_CUDA(cudaGetLastError());
}


}  // namespace epi
