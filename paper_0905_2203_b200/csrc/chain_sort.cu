// Episode ordering for the chain map kernel (chain_impl.cuh): a device radix
// sort of the episodes by (type_0, high_0, type_1, high_1, ..., type_{N-1})
// so that each CTA's 256 episodes share few chain prefixes, and the gather of
// the counting parameters into that order. Order never affects the counts
// (the kernel compares prefixes exactly); it only decides how much of each
// chain the CTA computes once per group instead of once per episode.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

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

// distinct-episode flags of the sorted keys (the key holds whole episodes)
__global__ void chain_flags_kernel(const uint64_t* __restrict__ keys, uint64_t n, uint32_t* flags) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  flags[i] = i == 0 || keys[i] != keys[i - 1] ? 1u : 0u;
}

// uidx = inclusive scan of the flags - 1; distinct episode u = uidx[i] of a
// flagged i takes its parameters from the original episode perm[i]
__global__ void chain_gather_unique_kernel(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ flags,
                                           uint32_t* uidx, const uint32_t* __restrict__ types,
                                           const uint32_t* __restrict__ win, const uint32_t* __restrict__ sigma,
                                           uint64_t n, uint32_t N, uint32_t* s_types, uint32_t* s_win,
                                           uint32_t* s_sigma) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t u = uidx[i] - 1u;
  uidx[i] = u;
  if (!flags[i]) return;
  const uint64_t j = perm[i];
  for (uint32_t k = 0; k < N; ++k) s_types[static_cast<uint64_t>(u) * N + k] = types[j * N + k];
  for (uint32_t k = 0; k + 1 < N; ++k) s_win[static_cast<uint64_t>(u) * (N - 1) + k] = win[j * (N - 1) + k];
  s_sigma[u] = sigma[j];
}

__global__ void chain_scatter_kernel(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ uidx,
                                     const uint64_t* __restrict__ ucounts, uint64_t n, uint64_t* out) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[perm[i]] = ucounts[uidx[i]];
}

inline size_t align256(size_t x) { return (x + 255) / 256 * 256; }

size_t cub_scan_bytes(uint64_t n) {
  size_t bytes = 0;
  EPI_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, static_cast<const uint32_t*>(nullptr),
                                         static_cast<uint32_t*>(nullptr), static_cast<int>(n)));
  return bytes;
}

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
         align256(n * 4) + align256(std::max(cub_temp_bytes(n), cub_scan_bytes(n))) + align256(n * 4) * 2;
}

int chain_sort(const ChainSortIn& in, bool dedup, char* scratch, ChainSortOut& out, cudaStream_t st) {
  const uint64_t n = in.n;
  const uint32_t N = in.N;
  uint32_t tb = 1;
  while ((1ull << tb) <= in.alphabet) ++tb;  // types are <= alphabet (spare zero row)
  // the key holds whole episodes when every field fits (windows: high <= 32
  // and one width per launch, so high alone identifies the window)
  const uint64_t key_bits = static_cast<uint64_t>(N) * tb + static_cast<uint64_t>(N - 1) * 6;
  dedup = dedup && key_bits <= 64;
  const int begin_bit = key_bits >= 64 ? 0 : static_cast<int>(64 - key_bits);  // keys sit in the top bits
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
  const size_t temp_bytes = std::max(cub_temp_bytes(n), cub_scan_bytes(n));
  void* temp = take(temp_bytes);
  uint32_t* flags = reinterpret_cast<uint32_t*>(take(n * 4));
  uint32_t* uidx = reinterpret_cast<uint32_t*>(take(n * 4));
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  chain_keys_kernel<<<blocks, 256, 0, st>>>(in.types, in.win, n, N, tb, k_in, i_in);
  EPI_CUDA(cudaGetLastError());
  size_t tb_bytes = temp_bytes;
  EPI_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb_bytes, k_in, k_out, i_in, i_out, static_cast<int>(n), begin_bit, 64,
                                           st));
  out.perm = i_out;
  if (!dedup) {
    chain_gather_kernel<<<blocks, 256, 0, st>>>(i_out, in.types, in.win, in.sigma, n, N, out.types, out.win,
                                                out.sigma);
    EPI_CUDA(cudaGetLastError());
    out.uidx = nullptr;
    out.n_unique = n;
    return 2;  // own kernel launches (plus the library sort's)
  }
  chain_flags_kernel<<<blocks, 256, 0, st>>>(k_out, n, flags);
  EPI_CUDA(cudaGetLastError());
  size_t sb = temp_bytes;
  EPI_CUDA(cub::DeviceScan::InclusiveSum(temp, sb, flags, uidx, static_cast<int>(n), st));
  chain_gather_unique_kernel<<<blocks, 256, 0, st>>>(i_out, flags, uidx, in.types, in.win, in.sigma, n, N,
                                                     out.types, out.win, out.sigma);
  EPI_CUDA(cudaGetLastError());
  uint32_t n_unique = 0;
  EPI_CUDA(cudaMemcpyAsync(&n_unique, uidx + n - 1, 4, cudaMemcpyDeviceToHost, st));
  EPI_CUDA(cudaStreamSynchronize(st));
  out.uidx = uidx;
  out.n_unique = static_cast<uint64_t>(n_unique) + 1;  // uidx was made 0-based
  return 3;
}

void chain_scatter(const ChainSortOut& so, uint64_t n, const uint64_t* ucounts, uint64_t* out, cudaStream_t st) {
  chain_scatter_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(so.perm, so.uidx, ucounts, n, out);
  EPI_CUDA(cudaGetLastError());
}

}  // namespace epi
