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
  // dedup: the sorted set holds only distinct episodes (n_unique of them);
  // sorted episode i of the full set is distinct episode uidx[i]
  uint32_t* uidx = nullptr;
  uint64_t n_unique = 0;
};

size_t chain_sort_scratch(uint64_t n, uint32_t N);
// Enqueues the sort on st. With dedup (and a key that holds whole episodes)
// identical episodes are counted once: the distinct ones are gathered in
// sorted order and out.n_unique is read back (one synchronisation);
// otherwise no host synchronisation and n_unique = n. Returns the number of
// own kernel launches.
int chain_sort(const ChainSortIn& in, bool dedup, char* scratch, ChainSortOut& out, cudaStream_t st);
// Dedup: out[perm[i]] = ucounts[uidx[i]] for every i < n.
void chain_scatter(const ChainSortOut& so, uint64_t n, const uint64_t* ucounts, uint64_t* out, cudaStream_t st);

}  // namespace epi
