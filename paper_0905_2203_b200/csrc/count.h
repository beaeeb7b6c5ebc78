// Launch interface of the bit-sliced counting kernels (count.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace epi {

// First completions recorded per FRESH machine for the concat-walk sync.
constexpr int kRecorded = 4;
// Bitmap layout: blocks of kBlkTiles tiles; per (block, type) a row of
// kRowStride words (kBlkTiles tile words + 4 pad words for bank spread).
constexpr int kBlkTiles = 32;
constexpr uint32_t kRowStride = 36;

struct CountLaunch {
  const uint32_t* occ;     // blocked type bitmaps (DeviceStream::d_occ)
  uint32_t blk_words;      // words per bitmap block (a_pad * kRowStride)
  int32_t stages;          // shared-memory ring depth (0: read rows from global)
  int32_t n_tiles;
  int32_t seg_len;         // segment q covers tiles [q*seg_len, min((q+1)*seg_len, seg_end))
  int32_t seg_end;         // 4-aligned end of the tile range
  int32_t P;               // segments
  int32_t window_tiles;    // tiles processed before a segment for its window
  int32_t hist_words;      // wide path: history words per position (ceil(max high / 32))
  uint32_t n_eps;          // episodes (all of length n_nodes); row stride of the records
  const uint32_t* n_dev;   // non-null: the live episode count is *n_dev <= n_eps (device)
  const uint32_t* ep_types;  // [n_eps * N]
  const uint32_t* ep_win;    // [n_eps * (N-1)]: (low+1) | high << 16
  const uint32_t* ep_sigma;  // [n_eps]: sum of highs
  uint32_t* f_count;         // [P * n_eps] FRESH completions inside the segment
  uint32_t* f_ncomp;         // [P * n_eps] FRESH completions incl. window
  uint64_t* f_last;          // [P * n_eps] last in-segment completion or ~0
  uint64_t* f_first;         // [P * n_eps * kRecorded] first completion times
  uint64_t* counts;          // [n_eps] walk output (map output when P == 1)
  unsigned long long* patches;  // walk statistics counter
  int* occ_query;            // host: non-null -> launch_machines* reports CTAs/SM, no launch
  uint32_t last_sh[4];       // launch_machines_last: doubling-smear shifts of the last window
  int32_t walk_warp;         // concat walk: one warp per episode (walk_warp_kernel, P <= 128)
  int32_t q_base;            // map launch covers segments q_base .. q_base + map_segs - 1
  int32_t map_segs;          // 0: all P segments
  const unsigned long long* hist;  // events per type (matched-pair statistics), may be null
  unsigned long long* matched;     // += sum over live episodes of sum_k hist[type_k]
  const uint32_t* out_perm;  // non-null: episode e's count goes to counts[out_perm[e]]
  int32_t chain_depth;       // chain kernel test knob: d + 1 forces prefix depth d (0: auto)
  int32_t bound_only;        // chain kernel: counts[e] += popcount of the chain-end bitmap
                             // (a sound upper bound of the count; pass 1 of epi_count MINE)
};

// Doubling-smear shift amounts covering a window of width w (1..16).
inline void smear_shifts(uint32_t w, uint32_t (&sh)[4]) {
  uint32_t cover = 1;
  for (int i = 0; i < 4; ++i) {
    const uint32_t s = cover < w ? (cover < w - cover ? cover : w - cover) : 0u;
    sh[i] = s;
    cover += s;
  }
}

// Shared-memory ring depth for a bitmap block of blk_words words.
int32_t stages_for(uint32_t blk_words);
// width: launch-uniform window width high-low (0 = mixed); hi32: every
// high <= 32. Together they select a specialised map kernel when available.
void launch_machines(int n_nodes, int width, bool hi32, const CountLaunch& p, cudaStream_t st);
void launch_walk(int n_nodes, const CountLaunch& p, cudaStream_t st);
// Pass-1 shape: every window but the last has width `width` (1..16), the last
// one a launch-uniform width w_last <= 16 (p.last_sh), every high <= 32,
// n_nodes 3..6. Returns false (nothing launched) when the shape has no
// specialised kernel.
bool launch_machines_last(int n_nodes, int width, uint32_t w_last, CountLaunch& p, cudaStream_t st);
// high > 63 (up to kMaxHighWide): local-memory history ring.
void launch_machines_wide(int n_nodes, const CountLaunch& p, cudaStream_t st);
void launch_walk_wide(int n_nodes, const CountLaunch& p, cudaStream_t st);
// Chain map kernel (chain_impl.cuh): every window of width `width` (1..16),
// every high <= 32, 2..8 nodes, host-sized launch. Returns false (nothing
// launched) for other shapes.
bool launch_chain(int n_nodes, int width, const CountLaunch& p, cudaStream_t st);
bool has_chain_kernel(int n_nodes, int width, bool hi32);
// Exact counts of single-node episodes (popcount of the type's bitmap).
void launch_singletons(const uint32_t* occ, uint32_t blk_words, uint32_t n_blocks,
                       const uint32_t* types, uint32_t n_eps, uint64_t* counts, cudaStream_t st);


}  // namespace epi
