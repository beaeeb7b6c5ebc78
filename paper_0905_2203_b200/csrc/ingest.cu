// Compressed stream ingest (epi_load_stream on host arrays): the 12 B/event
// SoA (u32 type + i64 time, E/types.hpp:96-134) crosses PCIe as narrow
// chunks - types in 1/2 bytes when the alphabet allows, times as per-event
// deltas in 1/2/4 bytes against a base every 2048 events - encoded by all
// host threads, shipped through a ring of pinned buffers and widened back into
// the device SoA by one kernel per chunk while the host encodes the next
// ones. For the bench configs (64 types, ~1 event/ms) that is ~2 B/event on
// the link instead of 12. A chunk holding anything the loader must reject
// (type >= alphabet, negative time, a time regression) ships raw, so the
// device validation (loader.cu) still reports the first offender with the
// reference's message (E/types.hpp:109-111).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "ingest.h"

namespace epi {
namespace {

constexpr int kSubThreads = 256;
constexpr int kSubItems = 8;
constexpr uint32_t kSub = kSubThreads * kSubItems;  // events per base time (2048)

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) / 16 * 16; }

struct ChunkHeader {
  uint32_t n;   // events in the chunk
  uint8_t tw;   // bytes per type (1, 2, 4)
  uint8_t dw;   // bytes per time delta (1, 2, 4), 8: raw i64 times
  uint8_t pad[10];
};
static_assert(sizeof(ChunkHeader) == 16, "chunk header");

// Layout of an encoded chunk: header | bases (i64 per sub-block, dw != 8) |
// types | deltas (or raw times), each part 16-byte aligned.
struct ChunkLayout {
  size_t bases, types, times, total;
};

__host__ __device__ inline ChunkLayout layout_of(uint32_t n, uint32_t tw, uint32_t dw) {
  ChunkLayout l;
  const size_t nsub = (n + kSub - 1) / kSub;
  l.bases = 16;
  l.types = l.bases + (dw == 8 ? 0 : align16(nsub * 8));
  l.times = l.types + align16(static_cast<size_t>(n) * tw);
  l.total = l.times + align16(static_cast<size_t>(n) * dw);
  return l;
}

template <class T>
__device__ __forceinline__ uint32_t load_narrow(const uint8_t* p, uint64_t i) {
  return static_cast<uint32_t>(reinterpret_cast<const T*>(p)[i]);
}

// One CTA per 2048-event sub-block: widen the types, prefix-sum the deltas
// onto the sub-block's base time.
__global__ void __launch_bounds__(kSubThreads)
    decode_chunk_kernel(const uint8_t* __restrict__ chunk, uint32_t* types_out, int64_t* times_out) {
  using BS = cub::BlockScan<int64_t, kSubThreads>;
  __shared__ typename BS::TempStorage ts;
  const ChunkHeader h = *reinterpret_cast<const ChunkHeader*>(chunk);
  const ChunkLayout l = layout_of(h.n, h.tw, h.dw);
  const uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * kSub;
  const uint8_t* tp = chunk + l.types;
  const uint8_t* dp = chunk + l.times;
  int64_t v[kSubItems];
#pragma unroll
  for (int j = 0; j < kSubItems; ++j) {
    const uint64_t i = b0 + threadIdx.x * kSubItems + j;  // blocked: thread owns 8 consecutive events
    uint32_t t = 0;
    int64_t d = 0;
    if (i < h.n) {
      t = h.tw == 1 ? load_narrow<uint8_t>(tp, i) : h.tw == 2 ? load_narrow<uint16_t>(tp, i)
                                                                : load_narrow<uint32_t>(tp, i);
      if (h.dw == 8)
        d = reinterpret_cast<const int64_t*>(dp)[i];
      else
        d = h.dw == 1 ? load_narrow<uint8_t>(dp, i) : h.dw == 2 ? load_narrow<uint16_t>(dp, i)
                                                                  : load_narrow<uint32_t>(dp, i);
      types_out[i] = t;
    }
    v[j] = d;
  }
  if (h.dw == 8) {
#pragma unroll
    for (int j = 0; j < kSubItems; ++j) {
      const uint64_t i = b0 + threadIdx.x * kSubItems + j;
      if (i < h.n) times_out[i] = v[j];
    }
    return;
  }
  BS(ts).InclusiveSum(v, v);
  const int64_t base = reinterpret_cast<const int64_t*>(chunk + l.bases)[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kSubItems; ++j) {
    const uint64_t i = b0 + threadIdx.x * kSubItems + j;
    if (i < h.n) times_out[i] = base + v[j];
  }
}

// Single pass for the common shape: every type and every in-sub-block time
// delta fits a byte. Returns 0 when some value does not (the caller then runs
// the general two-pass encoder).
size_t encode_chunk_u8(const uint32_t* types, const int64_t* times, uint32_t n, uint8_t* out) {
  const ChunkLayout l = layout_of(n, 1, 1);
  uint8_t* tp = out + l.types;
  uint8_t* dp = out + l.times;
  int64_t* bases = reinterpret_cast<int64_t*>(out + l.bases);
  uint32_t bad = 0;
  for (uint32_t b = 0; b < n; b += kSub) {
    const uint32_t e = b + kSub < n ? b + kSub : n;
    bases[b / kSub] = times[b];
    int64_t prev = times[b];
    for (uint32_t i = b; i < e; ++i) {
      const uint32_t t = types[i];
      const int64_t tm = times[i];
      const uint64_t d = static_cast<uint64_t>(tm - prev);  // negative -> huge
      bad |= (t >> 8) | static_cast<uint32_t>(d >> 8) | static_cast<uint32_t>(d >> 32);
      tp[i] = static_cast<uint8_t>(t);
      dp[i] = static_cast<uint8_t>(d);
      prev = tm;
    }
    if (bad) return 0;
  }
  ChunkHeader h{};
  h.n = n;
  h.tw = 1;
  h.dw = 1;
  std::memcpy(out, &h, sizeof h);
  return l.total;
}

// Encodes events [0, n) of one chunk into `out` (capacity >= the raw
// layout); returns the encoded size.
size_t encode_chunk(const uint32_t* types, const int64_t* times, uint32_t n, uint32_t alphabet, uint8_t* out) {
  if (alphabet <= 256)
    if (const size_t b = encode_chunk_u8(types, times, n, out)) return b;
  // pass 1: widths (and whether the chunk must ship raw)
  bool raw = false;
  uint64_t max_d = 0;
  uint32_t max_t = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t t = types[i];
    const int64_t tm = times[i];
    max_t = std::max(max_t, t);
    if (tm < 0 || t >= alphabet) raw = true;
    if (i % kSub != 0) {
      const int64_t d = tm - times[i - 1];
      if (d < 0) raw = true;
      max_d = std::max<uint64_t>(max_d, static_cast<uint64_t>(d));
    }
  }
  if (n && times[0] < 0) raw = true;
  const uint32_t tw = max_t < 256u ? 1 : max_t < 65536u ? 2 : 4;
  const uint32_t dw = raw ? 8 : max_d < 256u ? 1 : max_d < 65536u ? 2 : max_d < (1ull << 32) ? 4 : 8;
  const ChunkLayout l = layout_of(n, raw ? 4 : tw, dw);
  ChunkHeader h{};
  h.n = n;
  h.tw = static_cast<uint8_t>(raw ? 4 : tw);
  h.dw = static_cast<uint8_t>(dw);
  std::memcpy(out, &h, sizeof h);
  // types
  uint8_t* tp = out + l.types;
  if (h.tw == 1) {
    for (uint32_t i = 0; i < n; ++i) tp[i] = static_cast<uint8_t>(types[i]);
  } else if (h.tw == 2) {
    uint16_t* p = reinterpret_cast<uint16_t*>(tp);
    for (uint32_t i = 0; i < n; ++i) p[i] = static_cast<uint16_t>(types[i]);
  } else {
    std::memcpy(tp, types, static_cast<size_t>(n) * 4);
  }
  // times
  uint8_t* dp = out + l.times;
  if (dw == 8) {
    std::memcpy(dp, times, static_cast<size_t>(n) * 8);
  } else {
    int64_t* bases = reinterpret_cast<int64_t*>(out + l.bases);
    for (uint32_t s = 0; s * kSub < n; ++s) bases[s] = times[s * kSub];
    auto delta = [&](uint32_t i) -> uint64_t {
      return i % kSub == 0 ? 0u : static_cast<uint64_t>(times[i] - times[i - 1]);
    };
    if (dw == 1) {
      for (uint32_t i = 0; i < n; ++i) dp[i] = static_cast<uint8_t>(delta(i));
    } else if (dw == 2) {
      uint16_t* p = reinterpret_cast<uint16_t*>(dp);
      for (uint32_t i = 0; i < n; ++i) p[i] = static_cast<uint16_t>(delta(i));
    } else {
      uint32_t* p = reinterpret_cast<uint32_t*>(dp);
      for (uint32_t i = 0; i < n; ++i) p[i] = static_cast<uint32_t>(delta(i));
    }
  }
  return l.total;
}

}  // namespace

uint64_t upload_encoded(const uint32_t* types, const int64_t* times, uint64_t n, uint32_t alphabet,
                        uint32_t* d_types, int64_t* d_times, PinnedRing& ring, cudaStream_t st) {
  if (n == 0) return 0;
  // chunks of kChunk events (a multiple of the 2048-event sub-block). Worker
  // threads claim chunks in order and encode each into its ring slot once
  // the slot's previous copy has completed; this thread ships the chunks in
  // order (H2D + widening kernel) as they become ready.
  constexpr uint64_t kChunk = 1ull << 18;
  const size_t slot_bytes = layout_of(static_cast<uint32_t>(kChunk), 4, 8).total;
  unsigned hw = std::thread::hardware_concurrency();
  const unsigned workers = std::clamp<unsigned>(hw > 1 ? hw - 1 : 1, 1, 31);
  const uint64_t n_chunks = (n + kChunk - 1) / kChunk;
  const unsigned S = static_cast<unsigned>(std::min<uint64_t>(2ull * workers, n_chunks));
  ring.ensure(S, slot_bytes);
  uint8_t* d_buf = ring.device_buffer(S, slot_bytes);
  std::vector<std::atomic<int64_t>> ready(S), shipped_idx(S);
  std::vector<size_t> enc(S, 0);
  for (unsigned k = 0; k < S; ++k) {
    ready[k].store(-1);
    shipped_idx[k].store(-1);
  }
  std::atomic<uint64_t> next{0};
  std::atomic<bool> stop{false};
  auto worker = [&]() {
    for (;;) {
      const uint64_t c = next.fetch_add(1);
      if (c >= n_chunks || stop.load()) return;
      const unsigned k = static_cast<unsigned>(c % S);
      // the slot's previous chunk (c - S) must have been shipped and copied
      if (c >= S) {
        while (shipped_idx[k].load(std::memory_order_acquire) != static_cast<int64_t>(c - S)) {
          if (stop.load()) return;
          std::this_thread::yield();
        }
        ring.wait_quiet(k);
      }
      const uint64_t b = c * kChunk, e = std::min(n, b + kChunk);
      enc[k] = encode_chunk(types + b, times + b, static_cast<uint32_t>(e - b), alphabet, ring.slot(k));
      ready[k].store(static_cast<int64_t>(c), std::memory_order_release);
    }
  };
  std::vector<std::thread> pool;
  for (unsigned w = 0; w < workers; ++w) pool.emplace_back(worker);
  uint64_t shipped = 0;
  try {
    for (uint64_t c = 0; c < n_chunks; ++c) {
      const unsigned k = static_cast<unsigned>(c % S);
      while (ready[k].load(std::memory_order_acquire) != static_cast<int64_t>(c)) std::this_thread::yield();
      const uint64_t b = c * kChunk, e = std::min(n, b + kChunk);
      uint8_t* dslot = d_buf + static_cast<size_t>(k) * slot_bytes;
      EPI_CUDA(cudaMemcpyAsync(dslot, ring.slot(k), enc[k], cudaMemcpyHostToDevice, st));
      ring.record(k, st);
      const unsigned blocks = static_cast<unsigned>((e - b + kSub - 1) / kSub);
      decode_chunk_kernel<<<blocks, kSubThreads, 0, st>>>(dslot, d_types + b, d_times + b);
      EPI_CUDA(cudaGetLastError());
      shipped += enc[k];
      shipped_idx[k].store(static_cast<int64_t>(c), std::memory_order_release);
    }
  } catch (...) {
    stop.store(true);
    for (auto& t : pool) t.join();
    throw;
  }
  for (auto& t : pool) t.join();
  return shipped;
}

void PinnedRing::ensure(unsigned slots, size_t bytes) {
  if (slots <= n_slots_ && bytes <= slot_bytes_) return;
  release();
  EPI_CUDA(cudaMallocHost(reinterpret_cast<void**>(&host_), static_cast<size_t>(slots) * bytes));
  events_.resize(slots);
  used_.assign(slots, 0);
  for (auto& e : events_) EPI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  n_slots_ = slots;
  slot_bytes_ = bytes;
}

uint8_t* PinnedRing::device_buffer(unsigned slots, size_t bytes) {
  const size_t need = static_cast<size_t>(slots) * bytes;
  if (need > dev_bytes_) {
    if (dev_) cudaFree(dev_);
    dev_ = nullptr;
    EPI_CUDA(cudaMalloc(reinterpret_cast<void**>(&dev_), need));
    dev_bytes_ = need;
  }
  return dev_;
}

void PinnedRing::wait(unsigned first, unsigned count) {
  for (unsigned i = first; i < first + count; ++i)
    if (used_[i]) EPI_CUDA(cudaEventSynchronize(events_[i]));
}

void PinnedRing::wait_quiet(unsigned i) {
  if (used_[i]) cudaEventSynchronize(events_[i]);  // a failure resurfaces on the shipping thread
}

void PinnedRing::record(unsigned i, cudaStream_t st) {
  EPI_CUDA(cudaEventRecord(events_[i], st));
  used_[i] = 1;
}

void PinnedRing::release() {
  for (auto& e : events_)
    if (e) cudaEventDestroy(e);
  events_.clear();
  used_.clear();
  if (host_) cudaFreeHost(host_);
  host_ = nullptr;
  n_slots_ = 0;
  slot_bytes_ = 0;
}

PinnedRing::~PinnedRing() {
  release();
  if (dev_) cudaFree(dev_);
}

}  // namespace epi
