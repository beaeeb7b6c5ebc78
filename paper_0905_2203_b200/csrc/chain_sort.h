// Episode ordering for the chain map kernel (chain_sort.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace epi {

struct ChainSortIn {
  const uint32_t* types;  // [n * N]
  const uint32_t* win;    // [n * (N-1)]
  const uint32_t* sigma;  // [n]
  uint64_t n;
  uint32_t N;
  uint32_t alphabet;      // types are <= alphabet
};

struct ChainSortOut {
  uint32_t* types;
  uint32_t* win;
  uint32_t* sigma;
  uint32_t* perm;  // perm[i] = original index of sorted episode i
};

size_t chain_sort_scratch(uint64_t n, uint32_t N);
// Enqueues the sort on st (no host synchronisation). Returns the number of
// own kernel launches.
int chain_sort(const ChainSortIn& in, char* scratch, ChainSortOut& out, cudaStream_t st);

}  // namespace epi
