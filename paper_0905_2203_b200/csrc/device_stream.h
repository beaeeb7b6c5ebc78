// Device-resident stream and scratch buffers owned by an epi_ctx.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"
#include "count.h"

namespace epi {

// Growable device buffers addressed by slot; contents are not preserved
// across growth.
class DeviceScratch {
 public:
  ~DeviceScratch() {
    for (auto& b : bufs_)
      if (b.p) cudaFree(b.p);
  }
  template <class T>
  T* get(size_t slot, size_t count) {
    if (slot >= bufs_.size()) bufs_.resize(slot + 1);
    Buf& b = bufs_[slot];
    size_t bytes = count * sizeof(T);
    if (bytes == 0) bytes = 16;
    if (bytes > b.bytes) {
      if (b.p) cudaFree(b.p);
      b.p = nullptr;
      size_t grow = bytes + bytes / 4;
      EPI_CUDA(cudaMalloc(&b.p, grow));
      b.bytes = grow;
      ++generation;
    }
    return static_cast<T*>(b.p);
  }
  uint64_t generation = 0;  // bumped on every reallocation (graph-cache validity)

 private:
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
  };
  std::vector<Buf> bufs_;
};

struct DeviceStream {
  uint64_t n = 0;          // events
  bool valid = false;      // set only once a load (validation + bitmap build) succeeded
  uint32_t alphabet = 0;   // event-type alphabet size
  uint32_t a_pad = 4;      // words per tile row (alphabet + 1 spare, rounded up to 4)
  uint64_t n_tiles = 0;    // 32 ms tiles covering the compressed span
  uint64_t span = 0;       // compressed time span (last compressed time + 1)
  uint32_t gap_cap = 64;   // gap compression cap of the current bitmap (> every high)
  uint64_t generation = 0;    // bumped when d_occ is reallocated
  uint32_t* d_occ = nullptr;  // blocked bitmaps, see count.h (kBlkTiles, kRowStride)
  uint32_t blk_words = 0;     // words per bitmap block (a_pad * kRowStride)
  size_t occ_bytes = 0;
  uint32_t* d_types_raw = nullptr;  // validated SoA kept for bitmap rebuilds
  int64_t* d_times_raw = nullptr;
  uint64_t raw_cap = 0;
  uint64_t launches = 0;   // kernels launched by loads (stats)
  std::vector<uint64_t> type_hist;  // events per type (a_pad entries), see host_hist
  uint64_t* h_check = nullptr;      // pinned [2]: validation word, compressed span
  bool hist_on_host = false;
  unsigned long long* d_hist = nullptr;  // events per type on the device (scratch-owned)
  // Host copy of the per-type event counts (one D2H on first use per load).
  const std::vector<uint64_t>& host_hist(cudaStream_t st);

  ~DeviceStream() { release(); }
  void release();
  // Caller fills d_types_raw / d_times_raw (n_events entries) then calls load.
  void reserve_raw(uint64_t n_events);
  void load(uint64_t n_events, uint32_t alphabet, cudaStream_t st, DeviceScratch& scratch);
  // Rebuild the bitmap with a larger gap cap when a batch has high >= gap_cap.
  void ensure_cap(int64_t max_high, cudaStream_t st, DeviceScratch& scratch);

 private:
  void build(uint64_t n_events, uint32_t cap, bool validate, cudaStream_t st, DeviceScratch& scratch);
  void ensure_occ(uint64_t tiles, cudaStream_t st);
};

}  // namespace epi
