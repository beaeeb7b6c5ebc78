// Compressed host->device stream ingest (ingest.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <vector>

namespace epi {

// Pinned staging slots (host) with one completion event each, and the
// matching device landing buffer; kept by the engine across loads.
class PinnedRing {
 public:
  ~PinnedRing();
  void ensure(unsigned slots, size_t bytes);
  uint8_t* slot(unsigned i) { return host_ + static_cast<size_t>(i) * slot_bytes_; }
  uint8_t* device_buffer(unsigned slots, size_t bytes);
  void wait(unsigned first, unsigned count);  // copies out of these slots done
  void wait_quiet(unsigned i);                 // same, no exceptions (worker threads)
  void record(unsigned i, cudaStream_t st);
  uint64_t generation = 0;

 private:
  void release();
  uint8_t* host_ = nullptr;
  uint8_t* dev_ = nullptr;
  size_t dev_bytes_ = 0;
  unsigned n_slots_ = 0;
  size_t slot_bytes_ = 0;
  std::vector<cudaEvent_t> events_;
  std::vector<char> used_;
};

// Encodes the host SoA in chunks on all host threads, ships them through the
// ring and widens them into d_types / d_times (n entries) on `st`. Returns
// the bytes that crossed the link. Does not synchronise at the end.
uint64_t upload_encoded(const uint32_t* types, const int64_t* times, uint64_t n, uint32_t alphabet,
                        uint32_t* d_types, int64_t* d_times, PinnedRing& ring, cudaStream_t st);

}  // namespace epi
