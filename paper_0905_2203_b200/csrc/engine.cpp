// Host engine: stream upload, the two-pass count, and the level-wise miner.
//
// Reference anchors (paths relative to /root/reference/proj/include/episodic):
//   validate(Episode)          types.hpp:82-92   -> validate_episode
//   counting block of mine()   miner.hpp:145-154 -> Engine::count_set (one
//                              batched device count per level instead of a
//                              per-candidate CPU loop)
//   generate_candidates        miner.hpp:76-109  -> generate_candidates
//   mine                       miner.hpp:114-173 -> Engine::mine
#include "engine.h"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <unordered_map>

#include "chain_sort.h"
#include "count.h"

namespace epi {
namespace {

enum Slot : size_t {
  // 0..2 belong to the loader
  kSlotParams = 3,
  kSlotMachines = 4,
  kSlotCounts = 5,
  kSlotSegments = 6,
  kSlotShardStage = 7,
  kSlotShardCounts = 8,
  // 10..32 belong to the miner (mine_dev.cu), 40..47 and 140..141 to the
  // tracking counter (tracking.cu)
  kSlotChainSort = 60,
  kSlotChainCounts = 61,
  // 62, 63: the device generators' keys, sort buffers and plans (gen_dev.cu)
};

constexpr uint64_t kPruned = EPI_COUNT_PRUNED;

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

uint64_t hash_span(const uint32_t* t, size_t nt, const int64_t* lo, const int64_t* hi, size_t nc) {
  uint64_t h = 0x9e3779b97f4a7c15ull ^ (nt * 0x100000001b3ull);
  auto mix = [&](uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h *= 0xff51afd7ed558ccdull;
  };
  for (size_t i = 0; i < nt; ++i) mix(t[i]);
  for (size_t i = 0; i < nc; ++i) {
    mix(static_cast<uint64_t>(lo[i]));
    mix(static_cast<uint64_t>(hi[i]));
  }
  return h;
}

// Split [0, n) into contiguous chunks over host threads (inline when small).
template <class F>
void host_parallel(size_t n, bool big, F&& f) {
  unsigned w = std::thread::hardware_concurrency();
  w = std::min<unsigned>(w ? w : 1, 32);
  if (!big || w <= 1 || n < 2 * w) {
    f(size_t{0}, n);
    return;
  }
  std::vector<std::thread> th;
  for (unsigned i = 1; i < w; ++i) th.emplace_back([&, i] { f(n * i / w, n * (i + 1) / w); });
  f(size_t{0}, n / w);
  for (auto& t : th) t.join();
}

}  // namespace

Engine::Engine(int device) : device_(device) {
  EPI_CUDA(cudaSetDevice(device));
  EPI_CUDA(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, device));
  EPI_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  EPI_CUDA(cudaEventCreate(&ev0_));
  EPI_CUDA(cudaEventCreate(&ev1_));
  EPI_CUDA(cudaEventCreate(&ev2_));
  // one allocation: 64 bytes of accumulators, then the log slots, so the
  // statistics come back in one copy (same layout as the pinned mirror)
  EPI_CUDA(cudaMalloc(&d_acc_, 64 + kLogSlots * sizeof(uint32_t)));
  d_log_ = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(d_acc_) + 64);
  EPI_CUDA(cudaMemset(d_acc_, 0, 4 * sizeof(unsigned long long)));
}

Engine::~Engine() {
  cudaSetDevice(device_);
  for (auto& kv : level_graphs_)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  stream_.release();
  if (ev0_) cudaEventDestroy(ev0_);
  if (ev1_) cudaEventDestroy(ev1_);
  if (ev2_) cudaEventDestroy(ev2_);
  for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
  if (d_acc_) cudaFree(d_acc_);  // (d_log_ lives in the same allocation)
  if (st_) cudaStreamDestroy(st_);
}

// ---- deferred statistics -----------------------------------------------------

void Engine::rec(cudaEvent_t e) {
  EPI_CUDA(cudaEventRecordWithFlags(e, st_, capturing_ ? cudaEventRecordExternal : cudaEventRecordDefault));
}

uint64_t Engine::buffers_generation() const {
  return scratch_.generation * 0x9e3779b97f4a7c15ull ^ (stream_.generation << 1) ^
         (pin_up_.generation << 9) ^ (pin_small_.generation << 17) ^ (map_out_.generation << 25) ^
         (map_small_.generation << 33);
}

void Engine::require_stream() const {
  if (!stream_.valid) throw Error(EPI_EINVAL, "no event stream loaded (epi_load_stream first)");
}

void Engine::begin_op() {
  ++stat_epoch_;
  ev_used_ = 0;
  timed_.clear();
  timed_done_ = 0;
  slot_counters_.clear();
  log_used_ = 0;
  EPI_CUDA(cudaMemsetAsync(d_acc_, 0, 4 * sizeof(unsigned long long), st_));
}

cudaEvent_t Engine::next_event() {
  if (ev_used_ == ev_pool_.size()) {
    cudaEvent_t e;
    EPI_CUDA(cudaEventCreate(&e));
    ev_pool_.push_back(e);
  }
  return ev_pool_[ev_used_++];
}

int Engine::new_slot() {
  ++stat_epoch_;
  if (log_used_ >= kLogSlots) throw Error(EPI_EUNSUPPORTED, "device statistics log exhausted");
  return log_used_++;
}

void Engine::prefetch_stats() {
  const size_t nlog = static_cast<size_t>(log_used_);
  char* h = static_cast<char*>(pin_small_.get(64 + kLogSlots * sizeof(uint32_t)));
  EPI_CUDA(cudaMemcpyAsync(h, d_acc_, 64 + nlog * sizeof(uint32_t), cudaMemcpyDeviceToHost, st_));
  prefetched_epoch_ = stat_epoch_;
}

// Resolve timed_[timed_done_, upto) into `stats` (their events are complete
// and the statistics log holding their live counts is in the pinned mirror).
void Engine::resolve_timed(epi_stats& stats, size_t upto) {
  const auto* log = reinterpret_cast<const uint32_t*>(static_cast<const char*>(pin_small_.p) + 64);
  for (; timed_done_ < upto; ++timed_done_) {
    const Timed& t = timed_[timed_done_];
    float ms = 0, map_ms = 0;
    EPI_CUDA(cudaEventElapsedTime(&ms, t.e0, t.e1));
    const uint64_t live = t.live_slot >= 0 ? log[t.live_slot] : t.n_host;
    stats.total_ms += ms;
    if (t.ms_out) *t.ms_out += ms;
    if (t.ms_out2) *t.ms_out2 += ms;
    if (t.map) {
      if (t.e_map == t.e1)
        map_ms = ms;
      else
        EPI_CUDA(cudaEventElapsedTime(&map_ms, t.e0, t.e_map));
      stats.map_ms += map_ms;
      stats.concat_ms += ms - map_ms;
      stats.episode_events += live * stream_.n;
      stats.tile_steps += live * t.tiles_per_ep;
    }
  }
}

void Engine::flush_stats(epi_stats& stats) {
  const bool ready = prefetched_epoch_ == stat_epoch_;
  if (!ready) prefetch_stats();
  char* h = static_cast<char*>(pin_small_.get(64 + kLogSlots * sizeof(uint32_t)));
  auto* acc = reinterpret_cast<unsigned long long*>(h);
  auto* log = reinterpret_cast<uint32_t*>(h + 64);
  // the caller synchronised right after the prefetch when `ready`
  if (!ready) EPI_CUDA(cudaStreamSynchronize(st_));
  ++stat_epoch_;
  stats.patches += acc[0];
  stats.matched_pairs += acc[1];
  stats.pruned += acc[2];
  for (const SlotCounter& s : slot_counters_) *s.target += log[s.slot];
  resolve_timed(stats, timed_.size());
  timed_.clear();
  timed_done_ = 0;
  slot_counters_.clear();
  log_used_ = 0;
  ev_used_ = 0;  // (begin_op zeroes the device accumulators of the next call)
}

// Host -> device through pinned staging unless the source is already pinned.
void Engine::h2d(void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, src) == cudaSuccess &&
      (attr.type == cudaMemoryTypeHost || attr.type == cudaMemoryTypeManaged)) {
    EPI_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st_));
    return;
  }
  cudaGetLastError();  // clear the error state of a pageable-pointer query
  constexpr size_t kChunk = 16u << 20;
  char* stage = static_cast<char*>(pin_up_.get(2 * kChunk));
  size_t off = 0;
  int slot = 0;
  cudaEvent_t done[2];
  EPI_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
  EPI_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
  bool used[2] = {false, false};
  while (off < bytes) {
    size_t len = std::min(kChunk, bytes - off);
    if (used[slot]) EPI_CUDA(cudaEventSynchronize(done[slot]));
    std::memcpy(stage + slot * kChunk, static_cast<const char*>(src) + off, len);
    EPI_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, stage + slot * kChunk, len,
                             cudaMemcpyHostToDevice, st_));
    EPI_CUDA(cudaEventRecord(done[slot], st_));
    used[slot] = true;
    off += len;
    slot ^= 1;
  }
  EPI_CUDA(cudaStreamSynchronize(st_));
  cudaEventDestroy(done[0]);
  cudaEventDestroy(done[1]);
}

void Engine::load_stream_host(const uint32_t* types, const int64_t* times, uint64_t n,
                              uint32_t alphabet) {
  if (n && (!types || !times)) throw Error(EPI_EINVAL, "epi_load_stream: null event arrays");
  csr_valid_ = false;
  stream_.reserve_raw(n);
  if (n >= (1ull << 22) && !std::getenv("EPI_RAW_INGEST")) {
    // large streams cross PCIe narrowed (~2 B/event on the bench configs),
    // encoded on all host threads while earlier chunks are in flight
    last_load_h2d = upload_encoded(types, times, n, alphabet, stream_.d_types_raw, stream_.d_times_raw,
                                   ingest_ring_, st_);
  } else {
    h2d(stream_.d_types_raw, types, n * sizeof(uint32_t));
    h2d(stream_.d_times_raw, times, n * sizeof(int64_t));
    last_load_h2d = n * 12;
  }
  stream_.load(n, alphabet, st_, scratch_);
}

void Engine::download_stream(uint32_t* types, int64_t* times) {
  require_stream();
  const uint64_t n = stream_.n;
  if (n == 0) return;
  if (!types || !times) throw Error(EPI_EINVAL, "epi_stream_download: null arrays");
  EPI_CUDA(cudaMemcpyAsync(types, stream_.d_types_raw, n * 4, cudaMemcpyDeviceToHost, st_));
  EPI_CUDA(cudaMemcpyAsync(times, stream_.d_times_raw, n * 8, cudaMemcpyDeviceToHost, st_));
  EPI_CUDA(cudaStreamSynchronize(st_));
}

void Engine::load_stream_device(const uint32_t* d_types, const int64_t* d_times, uint64_t n,
                                uint32_t alphabet) {
  if (n && (!d_types || !d_times)) throw Error(EPI_EINVAL, "epi_load_stream_device: null arrays");
  csr_valid_ = false;
  stream_.reserve_raw(n);
  EPI_CUDA(cudaMemcpyAsync(stream_.d_types_raw, d_types, n * sizeof(uint32_t),
                           cudaMemcpyDeviceToDevice, st_));
  EPI_CUDA(cudaMemcpyAsync(stream_.d_times_raw, d_times, n * sizeof(int64_t),
                           cudaMemcpyDeviceToDevice, st_));
  stream_.load(n, alphabet, st_, scratch_);
}

// Packs n episodes of N nodes into the counting kernels' parameter layout
// (types clamped to the spare zero row `alphabet`, windows (low+1) | high<<16,
// sums of highs) in parallel over host threads, and summarises the launch
// shape (max high, max sigma, uniform widths) in `ds`. Types outside the
// alphabet can never fire; they read the always-zero spare column.
template <class TypeAt, class LoAt, class HiAt>
void pack_episodes(size_t n, uint32_t N, uint32_t A, uint32_t* h_types, uint32_t* h_win, uint32_t* h_sigma,
                   DevSet& ds, TypeAt&& type_at, LoAt&& lo_at, HiAt&& hi_at) {
  const uint32_t M = N - 1;
  struct Part {
    int64_t max_high = 0;
    uint32_t max_sigma = 0;
    int64_t width = -1, width_last = -1;  // -1 unset, 0 mixed
    bool too_wide = false;
  };
  unsigned w = std::thread::hardware_concurrency();
  w = std::min<unsigned>(w ? w : 1, 32);
  std::vector<Part> parts(w);
  std::atomic<unsigned> next{0};
  host_parallel(n, n >= 65536, [&](size_t b, size_t e) {
    Part& pt = parts[next.fetch_add(1)];
    for (size_t i = b; i < e; ++i) {
      for (uint32_t k = 0; k < N; ++k) {
        const uint32_t t = type_at(i, k);
        h_types[i * N + k] = t < A ? t : A;
      }
      uint32_t sig = 0;
      for (uint32_t k = 0; k < M; ++k) {
        const int64_t lo = lo_at(i, k), hi = hi_at(i, k);
        if (hi > kMaxHighWide) pt.too_wide = true;
        h_win[i * M + k] = static_cast<uint32_t>(lo + 1) | (static_cast<uint32_t>(hi) << 16);
        sig += static_cast<uint32_t>(hi);
        pt.max_high = std::max(pt.max_high, hi);
        int64_t& wd = k + 1 < M ? pt.width : pt.width_last;
        if (wd == -1)
          wd = hi - lo;
        else if (wd != hi - lo)
          wd = 0;
      }
      h_sigma[i] = sig;
      pt.max_sigma = std::max(pt.max_sigma, sig);
    }
  });
  int64_t width = -1, width_last = -1;
  auto merge = [](int64_t& a, int64_t b) {
    if (b == -1) return;
    if (a == -1)
      a = b;
    else if (a != b)
      a = 0;
  };
  for (unsigned i = 0; i < next.load(); ++i) {
    const Part& pt = parts[i];
    if (pt.too_wide)
      throw Error(EPI_EUNSUPPORTED, "constraint high > 4095 ms is not supported by the device counter");
    ds.max_high = std::max(ds.max_high, pt.max_high);
    ds.max_sigma = std::max(ds.max_sigma, pt.max_sigma);
    merge(width, pt.width);
    merge(width_last, pt.width_last);
  }
  if (width == -1 || width == width_last) {
    ds.width = width_last > 0 ? static_cast<int>(width_last) : 0;
  } else if (width > 0 && width_last > 0) {
    ds.width = static_cast<int>(width);  // the last constraint alone differs
    ds.last_w = static_cast<uint32_t>(width_last);
  }
}

void Engine::count_packed(DevSet ds, char* host, size_t off_win, size_t off_sigma, size_t total, uint64_t* out,
                          epi_stats& stats, double* ms_out) {
  const size_t n = ds.n;
  char* d_params = scratch_.get<char>(kSlotParams, total);
  EPI_CUDA(cudaMemcpyAsync(d_params, host, total, cudaMemcpyHostToDevice, st_));
  stats.h2d_bytes += total;
  ds.types = reinterpret_cast<const uint32_t*>(d_params);
  ds.win = reinterpret_cast<const uint32_t*>(d_params + off_win);
  ds.sigma = reinterpret_cast<const uint32_t*>(d_params + off_sigma);
  uint64_t* d_counts = scratch_.get<uint64_t>(kSlotCounts, n);
  count_device(ds, d_counts, stats, ms_out);
  uint64_t* h_counts = static_cast<uint64_t*>(pin_down_.get(n * sizeof(uint64_t)));
  EPI_CUDA(cudaMemcpyAsync(h_counts, d_counts, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, st_));
  EPI_CUDA(cudaStreamSynchronize(st_));
  host_parallel(n, n >= (1u << 18), [&](size_t b, size_t e) {
    std::memcpy(out + b, h_counts + b, (e - b) * sizeof(uint64_t));
  });
  stats.d2h_bytes += n * sizeof(uint64_t);
}

bool Engine::count_mine_csr(const epi_episode_batch& b, uint32_t N, uint64_t threshold, uint64_t* counts_out,
                            epi_stats& stats) {
  const size_t n = b.n_episodes;
  if (N > 8) return false;
  const uint32_t M = N - 1;
  const size_t off_win = align_up(n * N * 4, 256);
  const size_t off_sigma = align_up(off_win + n * M * 4, 256);
  const size_t total = align_up(off_sigma + n * 4, 256);
  char* host = static_cast<char*>(pin_up_.get(total));
  DevSet ds;
  ds.N = N;
  ds.n = n;
  const uint32_t* off = b.offsets;
  pack_episodes(
      n, N, stream_.alphabet, reinterpret_cast<uint32_t*>(host), reinterpret_cast<uint32_t*>(host + off_win),
      reinterpret_cast<uint32_t*>(host + off_sigma), ds, [&](size_t e, uint32_t k) { return b.types[off[e] + k]; },
      [&](size_t e, uint32_t k) { return b.low[off[e] - e + k]; },
      [&](size_t e, uint32_t k) { return b.high[off[e] - e + k]; });
  if (ds.last_w || ds.max_high > 32 || !has_chain_kernel(static_cast<int>(N), ds.width, true) ||
      stages_for(stream_.blk_words) == 0)
    return false;
  // pass 1: chain-end popcount bound of every candidate (count <= number of
  // distinct chain-end times: every completion is one)
  std::vector<uint64_t> bound(n);
  bound_only_ = true;
  try {
    count_packed(ds, host, off_win, off_sigma, total, bound.data(), stats, &stats.pass1_ms);
  } catch (...) {
    bound_only_ = false;
    throw;
  }
  bound_only_ = false;
  stats.pass1_groups += n;
  // pass 2: exact counts of the survivors (bound >= threshold); the pruned
  // ones can never be frequent, which is all mine() exposes
  // (E/miner.hpp:159-160)
  EpisodeSet surv;
  surv.N = N;
  std::vector<uint64_t> idx;
  for (size_t e = 0; e < n; ++e) {
    if (bound[e] < threshold) {
      counts_out[e] = kPruned;
      ++stats.pruned;
      continue;
    }
    idx.push_back(e);
    surv.types.insert(surv.types.end(), b.types + off[e], b.types + off[e] + N);
    surv.lo.insert(surv.lo.end(), b.low + (off[e] - e), b.low + (off[e] - e) + M);
    surv.hi.insert(surv.hi.end(), b.high + (off[e] - e), b.high + (off[e] - e) + M);
  }
  stats.pass2_episodes += idx.size();
  if (!idx.empty()) {
    std::vector<uint64_t> exact;
    count_exact(surv, exact, stats, &stats.pass2_ms);
    for (size_t j = 0; j < idx.size(); ++j) counts_out[idx[j]] = exact[j];
  }
  return true;
}

void Engine::count_exact(const EpisodeSet& set, std::vector<uint64_t>& counts, epi_stats& stats,
                         double* ms_out) {
  const size_t n = set.size();
  counts.assign(n, 0);
  if (n == 0) return;
  if (set.N > static_cast<uint32_t>(kMaxNodes))
    throw Error(EPI_EUNSUPPORTED, "episodes longer than 16 nodes are not supported on the device path");
  const uint32_t N = set.N;
  const uint32_t M = N - 1;
  const size_t off_win = align_up(n * N * 4, 256);
  const size_t off_sigma = align_up(off_win + n * M * 4, 256);
  const size_t total = align_up(off_sigma + n * 4, 256);
  char* host = static_cast<char*>(pin_up_.get(total));
  DevSet ds;
  ds.N = N;
  ds.n = n;
  pack_episodes(
      n, N, stream_.alphabet, reinterpret_cast<uint32_t*>(host), reinterpret_cast<uint32_t*>(host + off_win),
      reinterpret_cast<uint32_t*>(host + off_sigma), ds, [&](size_t e, uint32_t k) { return set.types[e * N + k]; },
      [&](size_t e, uint32_t k) { return set.lo[e * M + k]; }, [&](size_t e, uint32_t k) { return set.hi[e * M + k]; });
  count_packed(ds, host, off_win, off_sigma, total, counts.data(), stats, ms_out);
}

void Engine::count_exact_csr(const epi_episode_batch& b, uint32_t N, uint64_t* counts_out, epi_stats& stats,
                             double* ms_out) {
  const size_t n = b.n_episodes;
  if (n == 0) return;
  if (N > static_cast<uint32_t>(kMaxNodes))
    throw Error(EPI_EUNSUPPORTED, "episodes longer than 16 nodes are not supported on the device path");
  const uint32_t M = N - 1;
  const size_t off_win = align_up(n * N * 4, 256);
  const size_t off_sigma = align_up(off_win + n * M * 4, 256);
  const size_t total = align_up(off_sigma + n * 4, 256);
  char* host = static_cast<char*>(pin_up_.get(total));
  DevSet ds;
  ds.N = N;
  ds.n = n;
  // episode e: nodes at offsets[e] + k, constraints at offsets[e] - e + k
  const uint32_t* off = b.offsets;
  pack_episodes(
      n, N, stream_.alphabet, reinterpret_cast<uint32_t*>(host), reinterpret_cast<uint32_t*>(host + off_win),
      reinterpret_cast<uint32_t*>(host + off_sigma), ds, [&](size_t e, uint32_t k) { return b.types[off[e] + k]; },
      [&](size_t e, uint32_t k) { return b.low[off[e] - e + k]; },
      [&](size_t e, uint32_t k) { return b.high[off[e] - e + k]; });
  count_packed(ds, host, off_win, off_sigma, total, counts_out, stats, ms_out);
}

// Exact counts of a device-resident set into d_counts (device). Plans the
// MapConcatenate segments and launches the map and concat-walk kernels; the
// host does not wait (timings and counters are resolved by flush_stats).
void Engine::count_device(const DevSet& ds, uint64_t* d_counts, epi_stats& stats, double* ms_out,
                          int live_slot) {
  const size_t n = ds.n;
  if (n == 0) return;
  const uint32_t N = ds.N;
  const uint32_t* n_dev = live_slot >= 0 ? slot_ptr(live_slot) : nullptr;
  ++stat_epoch_;  // writes the statistics accumulators
  if (N == 1) {
    if (n_dev) throw Error(EPI_EUNSUPPORTED, "single-node sets need a host-known size");
    // every distinct firing time is a completion: popcount of the bitmap
    const uint32_t n_blocks = static_cast<uint32_t>((stream_.n_tiles + kBlkTiles - 1) / kBlkTiles);
    Timed t{next_event(), nullptr, next_event(), ms_out, -1, n,
            static_cast<uint64_t>(n_blocks) * kBlkTiles, true};
    t.e_map = t.e1;
    rec(t.e0);
    launch_singletons(stream_.d_occ, stream_.blk_words, n_blocks, ds.types, static_cast<uint32_t>(n),
                      d_counts, st_);
    rec(t.e1);
    timed_.push_back(t);
    stats.kernel_launches += 1;
    stats.map_launches += 1;
    stats.segments = std::max<uint64_t>(stats.segments, 1);  // one pass over the stream
    return;
  }
  // Wide windows need a bitmap whose gap compression cap exceeds them, and
  // the local-memory history ring (hist_words 32 ms words per position).
  const bool wide = ds.max_high > kMaxHigh;
  if (wide) stream_.ensure_cap(ds.max_high, st_, scratch_);
  const int32_t hist_words = wide ? static_cast<int32_t>((ds.max_high + 31) / 32) : 2;

  CountLaunch p{};
  p.occ = stream_.d_occ;
  p.blk_words = stream_.blk_words;
  p.stages = stages_for(stream_.blk_words);
  p.hist_words = hist_words;
  p.n_eps = static_cast<uint32_t>(n);
  p.n_dev = n_dev;
  p.ep_types = ds.types;
  p.ep_win = ds.win;
  p.ep_sigma = ds.sigma;
  p.counts = d_counts;
  // Chain map kernel (chain_impl.cuh): host-sized launches with one window
  // width (<= 16) and every high <= 32. The episodes are counted in a sorted
  // order (shared chain prefixes per CTA); counts scatter back through perm.
  // EPI_CHAIN=0 keeps the automaton kernel, EPI_CHAIN=1 uses the chain kernel
  // on sets of any size (tests), EPI_CHAIN_DEPTH=d+1 forces prefix depth d.
  const char* chain_env = std::getenv("EPI_CHAIN");
  const uint64_t chain_min = chain_env ? (std::atoi(chain_env) == 1 ? 1 : ~0ull) : 4096;
  const bool chain_shape = !wide && !ds.last_w && live_slot < 0 && p.stages > 0 &&
                           has_chain_kernel(static_cast<int>(N), ds.width, ds.max_high <= 32);
  if (bound_only_ && !chain_shape) throw Error(EPI_EUNSUPPORTED, "popcount bound needs the chain kernel shape");
  const bool chain = chain_shape && (n >= chain_min || bound_only_);
  // Identical episodes (equal sort keys) are counted once when the set is
  // large (one synchronisation to size the launch): the kernels count the
  // distinct ones and a scatter writes every caller slot.
  ChainSortOut so{};
  uint64_t* d_final = d_counts;
  const bool dedup = chain && n >= (std::getenv("EPI_CHAIN") ? 1 : 65536) && !std::getenv("EPI_NO_DEDUP") &&
                     !capturing_ && !tshard_;
  if (chain) {
    // a 4-deep staging ring lets row-mode CTAs take two bitmap blocks per
    // iteration (chain_impl.cuh) when the blocks are small enough; large sets
    // are the ones whose CTAs share whole prefixes (row mode) - small ones
    // keep the 3-deep ring and its occupancy
    if (n >= 65536 && p.blk_words * 4u * 4u <= 48u * 1024u) p.stages = 4;
    char* sc = scratch_.get<char>(kSlotChainSort, chain_sort_scratch(n, N));
    const int own = chain_sort({ds.types, ds.win, ds.sigma, n, N, stream_.alphabet}, dedup, sc, so, st_);
    stats.kernel_launches += static_cast<uint64_t>(own);
    p.ep_types = so.types;
    p.ep_win = so.win;
    p.ep_sigma = so.sigma;
    p.out_perm = so.perm;
    if (so.uidx) {
      // count the distinct episodes into a temporary, scatter afterwards
      p.n_eps = static_cast<uint32_t>(so.n_unique);
      p.out_perm = nullptr;
      p.counts = scratch_.get<uint64_t>(kSlotChainCounts, so.n_unique);
    }
    if (const char* dd = std::getenv("EPI_CHAIN_DEPTH")) p.chain_depth = std::atoi(dd);
    if (bound_only_) {
      p.bound_only = 1;  // every segment adds its chain ends: start from zero
      EPI_CUDA(cudaMemsetAsync(p.counts, 0, static_cast<size_t>(p.n_eps) * sizeof(uint64_t), st_));
    }
  }
  const size_t n_launch = p.n_eps;
  auto launch_map = [&]() {
    if (chain) {
      launch_chain(static_cast<int>(N), ds.width, p, st_);
      return;
    }
    if (wide)
      launch_machines_wide(static_cast<int>(N), p, st_);
    else if (ds.last_w && ds.max_high <= 32 &&
             launch_machines_last(static_cast<int>(N), ds.width, ds.last_w, p, st_))
      return;
    else
      launch_machines(static_cast<int>(N), ds.last_w ? 0 : ds.width, ds.max_high <= 32, p, st_);
  };

  // MapConcatenate plan. Segments must each span sum(high) (the window of a
  // segment lies inside its predecessor). Cost model in tile steps of one
  // thread, calibrated on the B200 (scripts/seg_sweep.py): the map kernel is
  // ALU-bound, so co-resident CTAs share an SM's issue rate and an SM's time
  // is the number of CTAs it receives times their length,
  // ceil(CTAs / SMs) * (tiles/P + window), inflated when the grid cannot
  // fill the resident slots (latency no longer hidden); plus kWalkStep per
  // segment for the sequential concat walk. P = 1 needs no walk at all.
  const int64_t n_tiles = static_cast<int64_t>(stream_.n_tiles);
  const int64_t tiles4 = (n_tiles + 3) / 4 * 4;
  const uint32_t max_sigma = ds.max_sigma;
  const int32_t window_tiles = static_cast<int32_t>((max_sigma + 31) / 32 + 1);
  constexpr int64_t kMaxWalkSegments = 128;
  constexpr uint64_t kWarpWalkMax = 4096;
  constexpr double kWalkStep = 20.0;
  // resident map CTAs per SM for this launch shape (cached per shape)
  const uint64_t shape = (static_cast<uint64_t>(N) << 48) ^ (static_cast<uint64_t>(ds.width) << 40) ^
                         (static_cast<uint64_t>(ds.max_high <= 32) << 39) ^
                         (static_cast<uint64_t>(wide) << 38) ^
                         (static_cast<uint64_t>(p.stages) << 32) ^ p.blk_words ^
                         (static_cast<uint64_t>(ds.last_w) << 56) ^ (static_cast<uint64_t>(chain) << 37);
  int bps = 0;
  for (const auto& kv : occ_cache_)
    if (kv.first == shape) bps = kv.second;
  if (bps == 0) {
    bps = 1;
    p.occ_query = &bps;
    launch_map();
    p.occ_query = nullptr;
    occ_cache_.emplace_back(shape, bps);
  }
  const int64_t slots = static_cast<int64_t>(num_sms_) * bps;
  const int64_t ctas_x = (static_cast<int64_t>(n_launch) + 255) / 256;
  const int64_t min_seg = std::max<int64_t>(window_tiles * 4, 32);
  const int64_t max_p = std::clamp<int64_t>(tiles4 / min_seg, 1, kMaxWalkSegments);
  int64_t P = 1;
  double best = 1e300;
  // Latency regime: even at the largest P every CTA is resident at once (one
  // wave over the resident slots), or the live size is known only on the
  // device (pass-2 survivors, usually few). A lone warp's concat-walk step (dependent global loads, boundary
  // patches) costs about as much as kWalkLatency of its map tile steps
  // (measured on cfg2's small levels): minimise per + kWalkLatency * P.
  // Few episodes (or a device-sized set) walk warp-parallel: a segment costs
  // ~2 tile steps there instead of ~12 in the sequential walk.
  p.walk_warp = (live_slot >= 0 || n <= kWarpWalkMax) && !std::getenv("EPI_WALK_SEQ") ? 1 : 0;
  const double kWalkLatency = p.walk_warp ? 2.0 : 12.0;
  if (live_slot >= 0 || ctas_x * max_p <= slots) {
    for (int64_t cand = 1; cand <= max_p; ++cand) {
      const double per = static_cast<double>((tiles4 + cand - 1) / cand + (cand > 1 ? window_tiles : 0));
      const double cost = per + (cand > 1 ? kWalkLatency * static_cast<double>(cand) : 0.0);
      if (cost < best * 0.999) {
        best = cost;
        P = cand;
      }
    }
  } else
  for (int64_t cand = 1; cand <= max_p; ++cand) {
    const int64_t ctas = ctas_x * cand;
    const double rounds = static_cast<double>((ctas + num_sms_ - 1) / num_sms_);
    const double fill = std::min(1.0, static_cast<double>(ctas) / static_cast<double>(slots));
    const double per = static_cast<double>((tiles4 + cand - 1) / cand + (cand > 1 ? window_tiles : 0));
    const double cost = rounds * per * (1.0 + 0.3 * (1.0 - fill)) +
                        (cand > 1 ? (p.walk_warp ? 4.0 : kWalkStep) * cand : 0.0);
    if (cost < best * 0.999) {
      best = cost;
      P = cand;
    }
  }
  const char* force_env = std::getenv("EPI_FORCE_SEGMENTS");
  if (force_segments_ > 0 || force_env) {
    // The caller's segment count (epi_count_mapconcat) or the test knob:
    // many short segments exercise the concat walk on small streams.
    // Correctness only needs each segment to span sum(high).
    const int64_t want = force_segments_ > 0 ? force_segments_ : std::atoll(force_env);
    const int64_t min_ok = std::max<int64_t>(1, (max_sigma + 31) / 32);
    P = std::clamp<int64_t>(want, 1, std::min<int64_t>(std::max<int64_t>(1, n_tiles / min_ok), 65535));
  }
  // Per-segment completion counters are 32-bit: a segment spans fewer than
  // 2^27 tiles (< 2^32 ms, so < 2^32 completions); the walk sums in 64 bits.
  P = std::max<int64_t>(P, (tiles4 + (int64_t{1} << 27) - 1) >> 27);
  // Time-segment shard (epi_count_sharded with few episodes): at least one
  // segment per rank, each rank maps its own contiguous block of segments.
  // (the pass-1 bound is computed whole on every rank: identical survivors)
  const epi_shard* ts = (tshard_ && tshard_->world > 1 && live_slot < 0 && !bound_only_) ? tshard_ : nullptr;
  if (ts && max_p >= static_cast<int64_t>(ts->world))
    P = std::min<int64_t>(max_p, (std::max<int64_t>(P, ts->world) + ts->world - 1) / ts->world * ts->world);
  else
    ts = nullptr;  // stream too short to give every rank a segment: every rank maps all
  // The chain kernel keeps times relative to a segment's window start in
  // 32 bits: segments (plus window) shorter than 2^26 tiles.
  if (chain) P = std::max<int64_t>(P, (tiles4 + (int64_t{1} << 25) - 1) >> 25);
  // Segment bounds are multiples of 4 tiles (the map kernel advances four
  // tiles per 16-byte load); the last segment runs to the 4-aligned end (the
  // bitmap is zero past the stream).
  const int64_t seg_len = ((tiles4 + P - 1) / P + 3) / 4 * 4;
  P = (tiles4 + seg_len - 1) / seg_len;
  if (ts && P < 2) ts = nullptr;
  const int64_t tW = ts ? ts->world : 1, tR = ts ? ts->rank : 0;
  const int64_t s_rows = ts ? (P + tW - 1) / tW : P;  // segment rows per rank (padded)
  const int64_t q0 = std::min<int64_t>(tR * s_rows, P), q1 = std::min<int64_t>(q0 + s_rows, P);
  // Matched-pair work of this launch (stats / roofline): sum_e sum_k n(type_k),
  // accumulated by the map kernel's first segment.
  p.hist = stream_.d_hist;
  p.matched = d_acc_ + 1;

  const size_t nm = P > 1 ? static_cast<size_t>(ts ? s_rows * tW : P) * n_launch : 1;
  const size_t m_count = 0, m_ncomp = align_up(nm * 4, 256), m_last = align_up(m_ncomp + nm * 4, 256),
               m_first = align_up(m_last + nm * 8, 256), m_total = m_first + nm * 8 * kRecorded;
  char* d_mach = scratch_.get<char>(kSlotMachines, m_total);
  p.n_tiles = static_cast<int32_t>(n_tiles);
  p.seg_len = static_cast<int32_t>(seg_len);
  p.seg_end = static_cast<int32_t>(tiles4);
  p.P = static_cast<int32_t>(P);
  p.window_tiles = window_tiles;
  p.f_count = reinterpret_cast<uint32_t*>(d_mach + m_count);
  p.f_ncomp = reinterpret_cast<uint32_t*>(d_mach + m_ncomp);
  p.f_last = reinterpret_cast<uint64_t*>(d_mach + m_last);
  p.f_first = reinterpret_cast<uint64_t*>(d_mach + m_first);
  p.patches = d_acc_;

  uint64_t tiles = 0;
  for (int64_t q = 0; q < P; ++q) {
    const int64_t gq = q * seg_len, gn = std::min<int64_t>((q + 1) * seg_len, tiles4);
    tiles += static_cast<uint64_t>(gn - std::max<int64_t>(gq - window_tiles, 0));
  }
  Timed t{next_event(), next_event(), nullptr, ms_out, live_slot, n_launch, tiles, true};
  rec(t.e0);
  if (ts) {
    p.q_base = static_cast<int32_t>(q0);
    p.map_segs = static_cast<int32_t>(q1 - q0);
    if (q1 > q0) launch_map();
    p.q_base = 0;
    p.map_segs = 0;
  } else {
    launch_map();
  }
  rec(t.e_map);
  t.e1 = t.e_map;
  if (ts) {
    // all-gather the segment records (q-major rows): every rank then walks
    // all P segments and gets every count
    struct Field {
      void* base;
      size_t elem;
    } fields[4] = {{p.f_count, 4}, {p.f_ncomp, 4}, {p.f_last, 8}, {p.f_first, 8ull * kRecorded}};
    const size_t row_bytes_max = static_cast<size_t>(s_rows) * n * 8 * kRecorded;
    char* stage = scratch_.get<char>(kSlotShardStage, row_bytes_max);
    for (const Field& f : fields) {
      const size_t bytes = static_cast<size_t>(s_rows) * n * f.elem;
      EPI_CUDA(cudaMemcpyAsync(stage, static_cast<char*>(f.base) + static_cast<size_t>(tR * s_rows) * n * f.elem,
                               bytes, cudaMemcpyDeviceToDevice, st_));
      if (ts->allgather(ts->user, stage, f.base, bytes, static_cast<void*>(st_)) != 0)
        throw Error(EPI_ENCCL, "count: all-gather of segment records failed");
    }
  }
  if (P > 1 && !bound_only_) {
    if (wide)
      launch_walk_wide(static_cast<int>(N), p, st_);
    else
      launch_walk(static_cast<int>(N), p, st_);
  }
  if (so.uidx) {
    chain_scatter(so, n, p.counts, d_final, st_);
    stats.kernel_launches += 1;
  }
  if (P > 1 || so.uidx) {
    t.e1 = next_event();
    rec(t.e1);
  }
  timed_.push_back(t);
  stats.segments = static_cast<uint64_t>(P);
  stats.kernel_launches += P > 1 && !bound_only_ ? 2 : 1;  // map (+ walk)
  stats.map_launches += 1;
  if (chain) stats.chain_launches += 1;
}

void Engine::count_set(const EpisodeSet& set, uint64_t threshold, uint32_t mode,
                       std::vector<uint64_t>& counts, epi_stats& stats) {
  const size_t n = set.size();
  stats.episodes += n;
  if (mode != EPI_MODE_MINE || threshold <= 1 || set.N <= 1 || n == 0) {
    stats.pass2_episodes += n;
    count_exact(set, counts, stats, &stats.pass2_ms);
    return;
  }
  // Pass 1: one relaxed episode per group of candidates that agree on the
  // types and on every constraint but the last; the last constraint is
  // widened to the hull (min low, max high] of the group's last constraints.
  // Every member's occurrences are occurrences of the relaxed episode, and a
  // maximum non-overlapped set cannot shrink when occurrences are added, so
  // count(relaxed) >= count(member): a sound upper bound. Relaxing only the
  // last constraint keeps the bound tight (the device miner does the same,
  // mine_dev.cu). Singleton groups are exact already.
  const uint32_t N = set.N, M = N - 1;
  const uint32_t KM = M - 1;  // constraints in the key
  // Open-addressing table keyed by a hash of the key; slots hold group ids,
  // collisions are resolved by comparing the stored key.
  size_t cap = 1;
  while (cap < 2 * n) cap <<= 1;
  std::vector<uint32_t> table(cap, UINT32_MAX);
  std::vector<uint32_t> group(n);
  EpisodeSet relaxed;
  relaxed.N = N;
  relaxed.types.reserve(n * N / 4 + N);
  std::vector<uint32_t> gsize;
  auto same_key = [&](uint32_t g, size_t i) {
    if (std::memcmp(&relaxed.types[static_cast<size_t>(g) * N], &set.types[i * N], N * 4) != 0) return false;
    for (uint32_t k = 0; k < KM; ++k)
      if (relaxed.lo[static_cast<size_t>(g) * M + k] != set.lo[i * M + k] ||
          relaxed.hi[static_cast<size_t>(g) * M + k] != set.hi[i * M + k])
        return false;
    return true;
  };
  for (size_t i = 0; i < n; ++i) {
    const uint32_t* t = &set.types[i * N];
    uint64_t h = hash_span(t, N, &set.lo[i * M], &set.hi[i * M], KM);
    size_t slot = static_cast<size_t>(h ^ (h >> 29)) & (cap - 1);
    uint32_t g = UINT32_MAX;
    while (table[slot] != UINT32_MAX) {
      const uint32_t gi = table[slot];
      if (same_key(gi, i)) {
        g = gi;
        break;
      }
      slot = (slot + 1) & (cap - 1);
    }
    if (g == UINT32_MAX) {
      g = static_cast<uint32_t>(gsize.size());
      table[slot] = g;
      relaxed.types.insert(relaxed.types.end(), t, t + N);
      relaxed.lo.insert(relaxed.lo.end(), &set.lo[i * M], &set.lo[i * M] + M);
      relaxed.hi.insert(relaxed.hi.end(), &set.hi[i * M], &set.hi[i * M] + M);
      gsize.push_back(1);
    } else {
      ++gsize[g];
      int64_t& lo = relaxed.lo[static_cast<size_t>(g) * M + KM];
      int64_t& hi = relaxed.hi[static_cast<size_t>(g) * M + KM];
      lo = std::min(lo, set.lo[i * M + KM]);
      hi = std::max(hi, set.hi[i * M + KM]);
    }
    group[i] = g;
  }
  std::vector<uint64_t> bound;
  stats.pass1_groups += gsize.size();
  count_exact(relaxed, bound, stats, &stats.pass1_ms);

  counts.assign(n, 0);
  EpisodeSet surv;
  surv.N = N;
  std::vector<uint32_t> surv_idx;
  for (size_t i = 0; i < n; ++i) {
    const uint32_t g = group[i];
    if (gsize[g] == 1) {
      counts[i] = bound[g];
    } else if (bound[g] < threshold) {
      counts[i] = kPruned;
      ++stats.pruned;
    } else {
      surv_idx.push_back(static_cast<uint32_t>(i));
      surv.types.insert(surv.types.end(), &set.types[i * N], &set.types[i * N] + N);
      surv.lo.insert(surv.lo.end(), &set.lo[i * M], &set.lo[i * M] + M);
      surv.hi.insert(surv.hi.end(), &set.hi[i * M], &set.hi[i * M] + M);
    }
  }
  stats.pass2_episodes += surv_idx.size();
  if (!surv_idx.empty()) {
    std::vector<uint64_t> exact;
    count_exact(surv, exact, stats, &stats.pass2_ms);
    for (size_t j = 0; j < surv_idx.size(); ++j) counts[surv_idx[j]] = exact[j];
  }
}

void Engine::count_batch(const epi_episode_batch& b, uint64_t threshold, uint32_t mode,
                         uint64_t* counts_out, uint8_t* frequent_out, epi_stats* stats_out) {
  epi_stats stats{};
  const uint64_t n = b.n_episodes;
  if (n && (!b.offsets || !counts_out)) throw Error(EPI_EINVAL, "epi_count: null batch arrays");
  require_stream();
  begin_op();
  if (mode > EPI_MODE_MINE) throw Error(EPI_EINVAL, "epi_count: unknown mode");
  // validate(Episode) for every candidate first (E/types.hpp:87-92), in
  // parallel; the first offender in candidate order decides the error
  std::vector<uint32_t> lens(n);
  std::atomic<uint64_t> first_bad{UINT64_MAX};
  std::vector<int> bad_kind(n ? 1 : 0);
  std::mutex bad_mu;
  host_parallel(n, n >= 65536, [&](size_t lo_e, size_t hi_e) {
    for (uint64_t e = lo_e; e < hi_e; ++e) {
      int kind = 0;
      if (b.offsets[e + 1] < b.offsets[e]) {
        kind = 1;
      } else {
        const uint32_t N = b.offsets[e + 1] - b.offsets[e];
        lens[e] = N;
        if (N == 0) kind = 2;
        const uint64_t cb = b.offsets[e] - e;
        for (uint32_t k = 0; kind == 0 && k + 1 < N; ++k)
          if (b.low[cb + k] < 0 || b.low[cb + k] >= b.high[cb + k]) kind = 3;
      }
      if (kind) {
        std::lock_guard<std::mutex> lk(bad_mu);
        if (e < first_bad.load()) {
          first_bad.store(e);
          bad_kind[0] = kind;
        }
        return;
      }
    }
  });
  if (first_bad.load() != UINT64_MAX) {
    static const char* kMsg[4] = {"", "epi_count: offsets not monotone", "episode must have at least one node",
                                  "interval constraint requires 0 <= low < high"};
    throw Error(EPI_EINVAL, kMsg[bad_kind[0]]);
  }
  // one episode length and exact counts (the bench's and most callers'
  // batches): pack straight from the caller's arrays
  bool uniform = n > 0;
  for (uint64_t e = 0; uniform && e < n; ++e) uniform = lens[e] == lens[0];
  if (uniform && mode == EPI_MODE_MINE && threshold > 1 && lens[0] > 1 && !std::getenv("EPI_PASS1_HULL")) {
    stats.episodes += n;
    if (count_mine_csr(b, lens[0], threshold, counts_out, stats)) {
      if (frequent_out)
        for (uint64_t e = 0; e < n; ++e)
          frequent_out[e] = counts_out[e] != kPruned && counts_out[e] >= threshold;
      flush_stats(stats);
      if (stats_out) *stats_out = stats;
      return;
    }
    stats.episodes -= n;  // shape without a chain kernel: the hull relaxation below
  }
  if (uniform && (mode != EPI_MODE_MINE || threshold <= 1 || lens[0] <= 1)) {
    stats.episodes += n;
    stats.pass2_episodes += n;
    count_exact_csr(b, lens[0], counts_out, stats, &stats.pass2_ms);
    if (frequent_out)
      for (uint64_t e = 0; e < n; ++e) frequent_out[e] = counts_out[e] >= threshold;
    flush_stats(stats);
    if (stats_out) *stats_out = stats;
    return;
  }
  std::vector<uint32_t> distinct(lens.begin(), lens.end());
  std::sort(distinct.begin(), distinct.end());
  distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
  for (uint32_t N : distinct) {
    EpisodeSet set;
    set.N = N;
    std::vector<uint64_t> idx;
    for (uint64_t e = 0; e < n; ++e) {
      if (lens[e] != N) continue;
      idx.push_back(e);
      const uint32_t b0 = b.offsets[e];
      const uint64_t cb = b0 - e;
      set.types.insert(set.types.end(), b.types + b0, b.types + b0 + N);
      set.lo.insert(set.lo.end(), b.low + cb, b.low + cb + N - 1);
      set.hi.insert(set.hi.end(), b.high + cb, b.high + cb + N - 1);
    }
    std::vector<uint64_t> counts;
    count_set(set, threshold, mode, counts, stats);
    for (size_t j = 0; j < idx.size(); ++j) counts_out[idx[j]] = counts[j];
  }
  if (frequent_out)
    for (uint64_t e = 0; e < n; ++e)
      frequent_out[e] = counts_out[e] != kPruned && counts_out[e] >= threshold;
  flush_stats(stats);
  if (stats_out) *stats_out = stats;
}

void Engine::count_batch_segments(const epi_episode_batch& b, uint64_t segments, uint64_t* counts_out,
                                  epi_stats* stats_out) {
  if (segments < 1) throw Error(EPI_EINVAL, "count_mapconcat: segments must be >= 1");
  force_segments_ = static_cast<int64_t>(std::min<uint64_t>(segments, 65535));
  try {
    count_batch(b, 1, EPI_MODE_EXACT, counts_out, nullptr, stats_out);
  } catch (...) {
    force_segments_ = 0;
    throw;
  }
  force_segments_ = 0;
}

void Engine::count_batch_sharded(const epi_episode_batch& b, uint64_t threshold, uint32_t mode,
                                 const epi_shard& shard, uint64_t* counts_out, uint8_t* frequent_out,
                                 epi_stats* stats_out) {
  const uint64_t n = b.n_episodes;
  const uint64_t W = shard.world, R = shard.rank;
  if (W == 0 || R >= W || (W > 1 && !shard.allgather))
    throw Error(EPI_EINVAL, "count: invalid shard (rank, world, allgather)");
  require_stream();
  if (W == 1) {
    count_batch(b, threshold, mode, counts_out, frequent_out, stats_out);
    return;
  }
  if (n && (!b.offsets || !counts_out)) throw Error(EPI_EINVAL, "epi_count: null batch arrays");
  if (n >= std::max<uint64_t>(shard.min_shard, W * W)) {
    // episode shards: count slice [R*s, R*s + s) locally, all-gather the counts
    const uint64_t s = (n + W - 1) / W;
    const uint64_t lo = std::min(R * s, n), hi = std::min(lo + s, n);
    std::vector<uint32_t> off(hi - lo + 1, 0), ty;
    std::vector<int64_t> low, high;
    for (uint64_t e = lo; e < hi; ++e) {
      if (b.offsets[e + 1] < b.offsets[e]) throw Error(EPI_EINVAL, "epi_count: offsets not monotone");
      const uint32_t b0 = b.offsets[e], N = b.offsets[e + 1] - b0;
      ty.insert(ty.end(), b.types + b0, b.types + b0 + N);
      if (N > 1) {
        low.insert(low.end(), b.low + (b0 - e), b.low + (b0 - e) + N - 1);
        high.insert(high.end(), b.high + (b0 - e), b.high + (b0 - e) + N - 1);
      }
      off[e - lo + 1] = static_cast<uint32_t>(ty.size());
    }
    const epi_episode_batch sub{hi - lo, off.data(), ty.data(), low.data(), high.data()};
    std::vector<uint64_t> local(hi - lo);
    count_batch(sub, threshold, mode, local.data(), nullptr, stats_out);
    uint64_t* d = scratch_.get<uint64_t>(kSlotShardCounts, s * (W + 1));
    uint64_t* d_send = d + s * W;
    EPI_CUDA(cudaMemsetAsync(d_send, 0, s * sizeof(uint64_t), st_));
    if (hi > lo)
      EPI_CUDA(cudaMemcpyAsync(d_send, local.data(), (hi - lo) * sizeof(uint64_t), cudaMemcpyHostToDevice, st_));
    if (shard.allgather(shard.user, d_send, d, s * sizeof(uint64_t), static_cast<void*>(st_)) != 0)
      throw Error(EPI_ENCCL, "count: all-gather of counts failed");
    EPI_CUDA(cudaMemcpyAsync(counts_out, d, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, st_));
    EPI_CUDA(cudaStreamSynchronize(st_));
  } else {
    // time shards: every rank counts every episode over its own segments
    struct Guard {
      const epi_shard*& slot;
      ~Guard() { slot = nullptr; }
    } guard{tshard_};
    tshard_ = &shard;
    count_batch(b, threshold, mode, counts_out, nullptr, stats_out);
  }
  if (frequent_out)
    for (uint64_t e = 0; e < n; ++e)
      frequent_out[e] = counts_out[e] != kPruned && counts_out[e] >= threshold;
}

// generate_candidates (E/miner.hpp:76-109). `frequent` holds the level-1
// frequent episodes in candidate order. The reference joins through a
// string-keyed hash of episode_key (E/miner.hpp:52-68: types and constraints
// of a contiguous slice); here the key is a 64-bit hash, the prefix keys are
// stably sorted once, each left's suffix key is binary-searched and verified,
// and the output is sized by a count pass and filled in parallel. The output
// order is the reference's: lefts in frequent order, rights in bucket
// (frequent) order.
void generate_candidates(size_t level, const EpisodeSet& frequent,
                         const std::vector<std::pair<int64_t, int64_t>>& alphabet,
                         uint32_t alphabet_size, EpisodeSet& out) {
  out.clear();
  out.N = static_cast<uint32_t>(level);
  if (level == 1) {
    out.types.resize(alphabet_size);
    for (uint32_t t = 0; t < alphabet_size; ++t) out.types[t] = t;
    return;
  }
  const size_t nf = frequent.size();
  if (nf == 0) return;
  if (level == 2) {
    const size_t na = alphabet.size(), total = nf * nf * na;
    out.types.resize(total * 2);
    out.lo.resize(total);
    out.hi.resize(total);
    size_t o = 0;
    for (size_t l = 0; l < nf; ++l)
      for (size_t r = 0; r < nf; ++r)
        for (const auto& c : alphabet) {
          out.types[2 * o] = frequent.types[l];
          out.types[2 * o + 1] = frequent.types[r];
          out.lo[o] = c.first;
          out.hi[o] = c.second;
          ++o;
        }
    return;
  }
  const uint32_t F = frequent.N;  // == level - 1
  const uint32_t FM = F - 1;
  const uint32_t K = F - 1;  // nodes in the join key (level - 2)
  auto key_hash = [&](size_t i, uint32_t first) {
    return hash_span(&frequent.types[i * F + first], K, &frequent.lo[i * FM + first],
                     &frequent.hi[i * FM + first], K - 1);
  };
  auto key_eq = [&](size_t a, uint32_t fa, size_t b, uint32_t fb) {
    for (uint32_t k = 0; k < K; ++k)
      if (frequent.types[a * F + fa + k] != frequent.types[b * F + fb + k]) return false;
    for (uint32_t k = 0; k + 1 < K; ++k)
      if (frequent.lo[a * FM + fa + k] != frequent.lo[b * FM + fb + k] ||
          frequent.hi[a * FM + fa + k] != frequent.hi[b * FM + fb + k])
        return false;
    return true;
  };
  // (prefix key, index) sorted: equal keys keep frequent order.
  std::vector<std::pair<uint64_t, uint32_t>> pre(nf);
  for (size_t i = 0; i < nf; ++i) pre[i] = {key_hash(i, 0), static_cast<uint32_t>(i)};
  std::sort(pre.begin(), pre.end());
  std::vector<uint32_t> lo_at(nf), hi_at(nf);  // bucket range per left
  std::vector<uint64_t> off(nf + 1, 0);
  for (size_t l = 0; l < nf; ++l) {
    const uint64_t h = key_hash(l, 1);
    auto r0 = std::lower_bound(pre.begin(), pre.end(), std::make_pair(h, 0u));
    auto r1 = std::upper_bound(r0, pre.end(), std::make_pair(h, UINT32_MAX));
    lo_at[l] = static_cast<uint32_t>(r0 - pre.begin());
    hi_at[l] = static_cast<uint32_t>(r1 - pre.begin());
    uint64_t c = 0;
    for (auto it = r0; it != r1; ++it) c += key_eq(it->second, 0, l, 1);
    off[l + 1] = off[l] + c;
  }
  const size_t total = off[nf];
  out.types.resize(total * level);
  out.lo.resize(total * (level - 1));
  out.hi.resize(total * (level - 1));
  auto fill = [&](size_t l0, size_t l1) {
    for (size_t l = l0; l < l1; ++l) {
      size_t o = off[l];
      for (uint32_t b = lo_at[l]; b < hi_at[l]; ++b) {
        const uint32_t r = pre[b].second;
        if (!key_eq(r, 0, l, 1)) continue;
        uint32_t* t = &out.types[o * level];
        std::memcpy(t, &frequent.types[l * F], F * sizeof(uint32_t));
        t[F] = frequent.types[static_cast<size_t>(r) * F + F - 1];
        int64_t* lo = &out.lo[o * (level - 1)];
        int64_t* hi = &out.hi[o * (level - 1)];
        std::memcpy(lo, &frequent.lo[l * FM], FM * sizeof(int64_t));
        std::memcpy(hi, &frequent.hi[l * FM], FM * sizeof(int64_t));
        lo[FM] = frequent.lo[static_cast<size_t>(r) * FM + FM - 1];
        hi[FM] = frequent.hi[static_cast<size_t>(r) * FM + FM - 1];
        ++o;
      }
    }
  };
  host_parallel(nf, total * level * 12 > (1u << 20), fill);
}

}  // namespace epi
