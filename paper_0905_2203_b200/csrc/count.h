// Launch interface of the bit-sliced counting kernels (count.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace epi {

// First completions recorded per FRESH machine for the concat-walk sync.
constexpr int kRecorded = 4;

struct CountLaunch {
  const uint32_t* occ;     // tile-major type bitmaps (DeviceStream::d_occ)
  uint32_t a_pad;          // words per tile row
  int32_t n_tiles;
  const int32_t* seg_g;    // P+1 segment tile bounds (device)
  int32_t P;               // segments
  int32_t window_tiles;    // tiles staged before a segment for its window
  int32_t chunk_tiles;     // tiles per shared-memory stage
  int32_t hist_words;      // wide path: history words per position (ceil(max high / 32))
  uint32_t n_eps;          // episodes (all of length n_nodes)
  const uint32_t* ep_types;  // [n_eps * N]
  const uint32_t* ep_win;    // [n_eps * (N-1)]: (low+1) | high << 16
  const uint32_t* ep_sigma;  // [n_eps]: sum of highs
  uint32_t* f_count;         // [P * n_eps] FRESH completions inside the segment
  uint32_t* f_ncomp;         // [P * n_eps] FRESH completions incl. window
  uint64_t* f_last;          // [P * n_eps] last in-segment completion or ~0
  uint64_t* f_first;         // [P * n_eps * kRecorded] first completion times
  uint64_t* counts;          // [n_eps] walk output
  unsigned long long* patches;  // walk statistics counter
};

uint32_t chunk_tiles_for(uint32_t a_pad);
// width: launch-uniform window width high-low (0 = mixed) selects a specialised kernel.
void launch_machines(int n_nodes, int width, const CountLaunch& p, cudaStream_t st);
void launch_walk(int n_nodes, const CountLaunch& p, cudaStream_t st);
// high > 63 (up to kMaxHighWide): local-memory history ring.
void launch_machines_wide(int n_nodes, const CountLaunch& p, cudaStream_t st);
void launch_walk_wide(int n_nodes, const CountLaunch& p, cudaStream_t st);
// *out += sum_i hist[types[i]] (matched-pair work model of a launch).
void launch_matched_pairs(const uint32_t* types, uint64_t count, const unsigned long long* hist,
                          unsigned long long* out, cudaStream_t st);

}  // namespace epi
