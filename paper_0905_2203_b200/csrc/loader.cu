// Event loader: device-resident per-type occurrence bitmaps.
//
// Replaces EventStream::from_events (E/types.hpp:102-119) and build_index
// (E/index.hpp:20-30). The reference keeps SoA vectors (u32 type + i64 time,
// 12 B/event) and per-type position/time lists (16 B/event). The counting
// kernels need, per event type, the set of distinct timestamps at which it
// fires (tied same-type events are idempotent for the counting automaton,
// SURVEY S6), so the device form is a tile-major bitmap:
//
//   occ[g * a_pad + type] bit b  <=>  `type` fires at compressed time 32*g + b
//
// One tile row holds a_pad (alphabet rounded up to 4) u32 words, so a run of
// consecutive tiles is one contiguous, 16-byte aligned block that the
// counting kernel stages into shared memory with a single bulk copy.
//
// Time compression: consecutive-event gaps longer than kGapCap are capped at
// kGapCap. Every admissible inter-event gap is <= high <= kMaxHigh < kGapCap,
// so pairs separated by a capped gap stay inadmissible, all other pairwise
// differences are unchanged, and the strict order used by the t > prev_end
// test is preserved: counts are identical, and idle stretches of the stream
// cost no tiles.
//
// Three passes (HBM-bound, ~20 B/event of traffic):
//   1. validate + per-block gap sums   (reads types, times)
//   2. exclusive scan of block sums    (one CTA)
//   3. block scan -> compressed time -> atomicOr into the bitmap
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "device_stream.h"

namespace epi {
namespace {

constexpr int kLoadThreads = 256;
constexpr int kLoadItems = 8;
constexpr int kLoadTile = kLoadThreads * kLoadItems;

__device__ __forceinline__ uint32_t capped_gap(const int64_t* times, uint64_t i, uint32_t cap) {
  if (i == 0) return 0;
  int64_t d = times[i] - times[i - 1];
  return d >= cap ? cap : static_cast<uint32_t>(d);
}

// Pass 1. err_key = min over bad events of (index*4 + check), check order as
// in from_events: 0 negative time, 1 time regression, 2 type out of range.
__global__ void __launch_bounds__(kLoadThreads)
    validate_reduce_kernel(const uint32_t* __restrict__ types, const int64_t* __restrict__ times,
                           uint64_t n, uint32_t alphabet, uint32_t cap, unsigned long long* err_key,
                           uint64_t* block_sums) {
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kLoadTile;
  uint32_t sum = 0;
  unsigned long long bad = ~0ull;
#pragma unroll
  for (int j = 0; j < kLoadItems; ++j) {
    uint64_t i = base + static_cast<uint64_t>(j) * kLoadThreads + threadIdx.x;
    if (i < n) {
      int64_t t = times[i];
      unsigned long long key = ~0ull;
      if (t < 0)
        key = i * 4 + 0;
      else if (i > 0 && t < times[i - 1])
        key = i * 4 + 1;
      else if (types[i] >= alphabet)
        key = i * 4 + 2;
      if (key < bad) bad = key;
      if (key == ~0ull) sum += capped_gap(times, i, cap);
    }
  }
  if (bad != ~0ull) atomicMin(err_key, bad);
  using Reduce = cub::BlockReduce<uint32_t, kLoadThreads>;
  __shared__ typename Reduce::TempStorage tmp;
  uint32_t total = Reduce(tmp).Sum(sum);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

// Pass 2: in-place exclusive scan of nb block sums; block_sums[nb] = total.
__global__ void __launch_bounds__(1024) scan_block_sums_kernel(uint64_t* block_sums, uint64_t nb) {
  using Scan = cub::BlockScan<uint64_t, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t b0 = 0; b0 < nb; b0 += 1024) {
    uint64_t i = b0 + threadIdx.x;
    uint64_t v = i < nb ? block_sums[i] : 0;
    uint64_t excl, agg;
    Scan(tmp).ExclusiveSum(v, excl, agg);
    uint64_t c = carry;
    if (i < nb) block_sums[i] = c + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry = c + agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) block_sums[nb] = carry;
}

// Pass 3: compressed time of every event, then set its bit in the tile row.
// Items are blocked per thread (kLoadItems consecutive events) so the scan is
// a thread-serial prefix plus one block-wide scan of thread totals.
__global__ void __launch_bounds__(kLoadThreads)
    scan_bitmap_kernel(const uint32_t* __restrict__ types, const int64_t* __restrict__ times,
                       uint64_t n, uint32_t cap, const uint64_t* __restrict__ block_offsets, uint32_t a_pad,
                       uint32_t* __restrict__ occ, unsigned long long* __restrict__ hist,
                       bool smem_hist) {
  extern __shared__ uint32_t s_hist[];
  if (smem_hist) {
    for (uint32_t t = threadIdx.x; t < a_pad; t += blockDim.x) s_hist[t] = 0;
  }
  const uint64_t base =
      static_cast<uint64_t>(blockIdx.x) * kLoadTile + static_cast<uint64_t>(threadIdx.x) * kLoadItems;
  uint32_t gaps[kLoadItems];
  uint32_t run = 0;
#pragma unroll
  for (int j = 0; j < kLoadItems; ++j) {
    uint64_t i = base + j;
    gaps[j] = i < n ? capped_gap(times, i, cap) : 0;
    run += gaps[j];
  }
  using Scan = cub::BlockScan<uint32_t, kLoadThreads>;
  __shared__ typename Scan::TempStorage tmp;
  uint32_t excl;
  Scan(tmp).ExclusiveSum(run, excl);  // its internal barrier also orders the s_hist clear
  uint64_t c = block_offsets[blockIdx.x] + excl;
#pragma unroll
  for (int j = 0; j < kLoadItems; ++j) {
    uint64_t i = base + j;
    c += gaps[j];
    if (i < n) {
      const uint64_t g = c >> 5;
      const uint32_t ty = types[i];
      // blocked layout: block g/32, row `ty` (kRowStride words), word g%32
      atomicOr(&occ[(g >> 5) * (a_pad * kRowStride) + ty * kRowStride + (g & 31)], 1u << (c & 31));
      if (smem_hist)
        atomicAdd(&s_hist[ty], 1u);
      else
        atomicAdd(&hist[ty], 1ull);
    }
  }
  if (smem_hist) {
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < a_pad; t += blockDim.x)
      if (s_hist[t]) atomicAdd(&hist[t], static_cast<unsigned long long>(s_hist[t]));
  }
}

}  // namespace

void DeviceStream::release() {
  if (d_occ) cudaFree(d_occ);
  d_occ = nullptr;
  occ_bytes = 0;
  if (d_types_raw) cudaFree(d_types_raw);
  if (d_times_raw) cudaFree(d_times_raw);
  d_types_raw = nullptr;
  d_times_raw = nullptr;
  raw_cap = 0;
  if (h_check) cudaFreeHost(h_check);
  h_check = nullptr;
}

void DeviceStream::reserve_raw(uint64_t n_events) {
  if (n_events <= raw_cap) return;
  if (d_types_raw) cudaFree(d_types_raw);
  if (d_times_raw) cudaFree(d_times_raw);
  d_types_raw = nullptr;
  d_times_raw = nullptr;
  raw_cap = 0;
  EPI_CUDA(cudaMalloc(&d_types_raw, n_events * sizeof(uint32_t)));
  EPI_CUDA(cudaMalloc(&d_times_raw, n_events * sizeof(int64_t)));
  raw_cap = n_events;
}

void DeviceStream::load(uint64_t n_events, uint32_t alphabet_size, cudaStream_t st,
                        DeviceScratch& scratch) {
  // a failed load leaves no half-updated stream behind: counting refuses to
  // run until a later load succeeds
  valid = false;
  n = 0;
  alphabet = alphabet_size;
  // One spare always-zero column (index `alphabet`) for episode types that
  // lie outside the alphabet and therefore never fire.
  a_pad = (alphabet_size + 1 + 3) / 4 * 4;
  build(n_events, static_cast<uint32_t>(kGapCap), true, st, scratch);
}

void DeviceStream::ensure_cap(int64_t max_high, cudaStream_t st, DeviceScratch& scratch) {
  if (max_high < static_cast<int64_t>(gap_cap)) return;
  // Smallest multiple of the tile width above max_high.
  const uint32_t cap = static_cast<uint32_t>((max_high + 1 + 31) / 32 * 32);
  build(n, cap, false, st, scratch);
}

void DeviceStream::build(uint64_t n_events, uint32_t cap, bool validate, cudaStream_t st,
                         DeviceScratch& scratch) {
  gap_cap = cap;
  n_tiles = 1;
  if (n_events == 0) {
    // An empty stream still gets one (zero) tile so kernels need no special case.
    ensure_occ(1, st);
    type_hist.assign(a_pad, 0);
    hist_on_host = true;
    d_hist = scratch.get<unsigned long long>(2, a_pad);
    EPI_CUDA(cudaMemsetAsync(d_hist, 0, a_pad * sizeof(unsigned long long), st));
    n = 0;
    span = 0;
    valid = true;
    return;
  }
  const uint32_t* d_types = d_types_raw;
  const int64_t* d_times = d_times_raw;
  const uint64_t nb = (n_events + kLoadTile - 1) / kLoadTile;
  uint64_t* d_sums = scratch.get<uint64_t>(0, nb + 1);
  unsigned long long* d_err = scratch.get<unsigned long long>(1, 1);
  EPI_CUDA(cudaMemsetAsync(d_err, 0xff, sizeof(unsigned long long), st));
  validate_reduce_kernel<<<static_cast<unsigned>(nb), kLoadThreads, 0, st>>>(
      d_types, d_times, n_events, alphabet, cap, d_err, d_sums);
  EPI_CUDA(cudaGetLastError());
  scan_block_sums_kernel<<<1, 1024, 0, st>>>(d_sums, nb);
  EPI_CUDA(cudaGetLastError());
  // pinned destinations: both copies stay asynchronous, one synchronisation
  if (!h_check) EPI_CUDA(cudaMallocHost(&h_check, 2 * sizeof(uint64_t)));
  EPI_CUDA(cudaMemcpyAsync(h_check, d_err, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  EPI_CUDA(cudaMemcpyAsync(h_check + 1, d_sums + nb, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  EPI_CUDA(cudaStreamSynchronize(st));
  const unsigned long long h_err = h_check[0];
  const uint64_t h_total = h_check[1];
  launches += 2;
  if (validate && h_err != ~0ull) {
    static const char* kMsg[3] = {"negative event time", "event times must be non-decreasing",
                                  "event type id out of range"};
    throw Error(2 /*EPI_EDATA*/, kMsg[h_err & 3]);
  }
  const uint64_t tiles = (h_total >> 5) + 1;
  if (tiles >= (1ull << 31))
    throw Error(7 /*EPI_EUNSUPPORTED*/, "stream spans more than 2^31 compressed time tiles");
  ensure_occ(tiles, st);
  d_hist = scratch.get<unsigned long long>(2, a_pad);
  EPI_CUDA(cudaMemsetAsync(d_hist, 0, a_pad * sizeof(unsigned long long), st));
  const bool smem_hist = a_pad <= 8192;
  scan_bitmap_kernel<<<static_cast<unsigned>(nb), kLoadThreads, smem_hist ? a_pad * 4 : 0, st>>>(
      d_types, d_times, n_events, cap, d_sums, a_pad, d_occ, d_hist, smem_hist);
  EPI_CUDA(cudaGetLastError());
  launches += 1;
  hist_on_host = false;  // copied on demand (host_hist): no second sync per load
  n = n_events;
  n_tiles = tiles;
  span = h_total + 1;
  valid = true;
}

const std::vector<uint64_t>& DeviceStream::host_hist(cudaStream_t st) {
  if (!hist_on_host) {
    type_hist.assign(a_pad, 0);
    EPI_CUDA(cudaMemcpyAsync(type_hist.data(), d_hist, a_pad * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    EPI_CUDA(cudaStreamSynchronize(st));
    hist_on_host = true;
  }
  return type_hist;
}

void DeviceStream::ensure_occ(uint64_t tiles, cudaStream_t st) {
  // Whole blocks of kBlkTiles tiles plus one spare block, zero-filled: the
  // map kernel may run up to the end of the last block.
  blk_words = a_pad * kRowStride;
  const size_t blocks = (tiles + kBlkTiles - 1) / kBlkTiles + 1;
  const size_t need = blocks * blk_words * sizeof(uint32_t);
  if (need > occ_bytes) {
    if (d_occ) cudaFree(d_occ);
    d_occ = nullptr;
    occ_bytes = 0;
    EPI_CUDA(cudaMalloc(&d_occ, need));
    ++generation;
    occ_bytes = need;
  }
  EPI_CUDA(cudaMemsetAsync(d_occ, 0, need, st));
}

}  // namespace epi
