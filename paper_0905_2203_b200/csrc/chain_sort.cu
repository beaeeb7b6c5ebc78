// Episode ordering for the chain map kernel (chain_impl.cuh): a device radix
// sort of the episodes by (type_0, high_0, type_1, high_1, ..., type_{N-1})
// so that each CTA's 256 episodes share few chain prefixes, and the gather of
// the counting parameters into that order. Order never affects the counts
// (the kernel compares prefixes exactly); it only decides how much of each
// chain the CTA computes once per group instead of once per episode.
#include <cub/device/device_radix_sort.cuh>

#include "chain_sort.h"
#include "common.cuh"

namespace epi {
namespace {

__global__ void chain_keys_kernel(const uint32_t* __restrict__ types, const uint32_t* __restrict__ win,
                                  uint64_t n, uint32_t N, uint32_t tb, uint64_t* keys, uint32_t* idx) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t key = 0;
  uint32_t used = 0;
  for (uint32_t k = 0; k < N; ++k) {
    if (used + tb > 64) break;
    key = (key << tb) | types[i * N + k];
    used += tb;
    if (k + 1 < N) {
      if (used + 6 > 64) break;
      key = (key << 6) | ((win[i * (N - 1) + k] >> 16) & 63u);  // high <= 32
      used += 6;
    }
  }
  keys[i] = used ? key << (64 - used) : 0;  // fields from the most significant bit down
  idx[i] = static_cast<uint32_t>(i);
}

__global__ void chain_gather_kernel(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ types,
                                    const uint32_t* __restrict__ win, const uint32_t* __restrict__ sigma,
                                    uint64_t n, uint32_t N, uint32_t* s_types, uint32_t* s_win,
                                    uint32_t* s_sigma) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t j = perm[i];
  for (uint32_t k = 0; k < N; ++k) s_types[i * N + k] = types[j * N + k];
  for (uint32_t k = 0; k + 1 < N; ++k) s_win[i * (N - 1) + k] = win[j * (N - 1) + k];
  s_sigma[i] = sigma[j];
}

inline size_t align256(size_t x) { return (x + 255) / 256 * 256; }

size_t cub_temp_bytes(uint64_t n) {
  size_t bytes = 0;
  EPI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const uint64_t*>(nullptr),
                                           static_cast<uint64_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                           static_cast<uint32_t*>(nullptr), static_cast<int>(n)));
  return bytes;
}

}  // namespace

size_t chain_sort_scratch(uint64_t n, uint32_t N) {
  return align256(n * 8) * 2 + align256(n * 4) * 2 + align256(n * 4 * N) + align256(n * 4 * (N ? N - 1 : 0) + 4) +
         align256(n * 4) + align256(cub_temp_bytes(n));
}

int chain_sort(const ChainSortIn& in, char* scratch, ChainSortOut& out, cudaStream_t st) {
  const uint64_t n = in.n;
  const uint32_t N = in.N;
  uint32_t tb = 1;
  while ((1ull << tb) <= in.alphabet) ++tb;  // types are <= alphabet (spare zero row)
  char* p = scratch;
  auto take = [&](size_t bytes) {
    char* r = p;
    p += align256(bytes);
    return r;
  };
  uint64_t* k_in = reinterpret_cast<uint64_t*>(take(n * 8));
  uint64_t* k_out = reinterpret_cast<uint64_t*>(take(n * 8));
  uint32_t* i_in = reinterpret_cast<uint32_t*>(take(n * 4));
  uint32_t* i_out = reinterpret_cast<uint32_t*>(take(n * 4));
  out.types = reinterpret_cast<uint32_t*>(take(n * 4 * N));
  out.win = reinterpret_cast<uint32_t*>(take(n * 4 * (N - 1) + 4));
  out.sigma = reinterpret_cast<uint32_t*>(take(n * 4));
  const size_t temp_bytes = cub_temp_bytes(n);
  void* temp = take(temp_bytes);
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  chain_keys_kernel<<<blocks, 256, 0, st>>>(in.types, in.win, n, N, tb, k_in, i_in);
  EPI_CUDA(cudaGetLastError());
  size_t tb_bytes = temp_bytes;
  EPI_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb_bytes, k_in, k_out, i_in, i_out, static_cast<int>(n), 0, 64,
                                           st));
  chain_gather_kernel<<<blocks, 256, 0, st>>>(i_out, in.types, in.win, in.sigma, n, N, out.types, out.win,
                                              out.sigma);
  EPI_CUDA(cudaGetLastError());
  out.perm = i_out;
  return 2;  // own kernel launches (plus the library sort's)
}

}  // namespace epi
