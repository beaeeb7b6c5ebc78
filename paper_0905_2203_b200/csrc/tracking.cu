// Parallel local tracking (paper §IV, Alg. 2 + CountScanWrite; reference
// E/tracking.hpp:236-407) on sm_100a: the second exact counter and the
// device implementation of find_occurrences / count_tracking.
//
// Per-type index (build_index, E/index.hpp:20-30): a stable radix sort of the
// stream by type gives, per type, its events' stream positions and ORIGINAL
// timestamps in stream order (d_csr_pos / d_csr_time, offsets per type).
//
// One CTA tracks one episode. Items are (rank in the current type's list,
// chain time). A tracking step (track_step, E/tracking.hpp:236-324):
//   * window per item by binary search in the destination type's times
//     (item_window, E/tracking.hpp:76-89): forward (t+low, t+high],
//     backward [t-high, t-low);
//   * dedup per destination rank, keeping the max chain start (forward) or
//     the min chain end (backward) - an order-independent atomicMax/Min, the
//     reference's max/min merge (E/tracking.hpp:268-310);
//   * compaction of the surviving ranks in ascending order with a block scan
//     (CountScanWrite's scan / compact_flags, E/parallel.hpp:210-243).
// find_occurrences emits (chain, own) forward or (own, chain) backward per
// surviving item (E/tracking.hpp:355-365); greedy_schedule
// (E/tracking.hpp:372-386) runs one warp per episode over the end-sorted
// intervals (the reference proves both directions end-sorted; a violation is
// reported, never silently re-sorted on the host).
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "engine.h"

namespace epi {
namespace {

constexpr int kTrackThreads = 512;

enum TrackSlot : size_t {
  kTCsrKeys = 40,
  kTCsrKeysAlt,
  kTCsrPos,
  kTCsrPosAlt,
  kTCub,
  kTParams,
  kTItems,
  kTOut,
};

__global__ void iota_kernel(uint32_t* v, uint64_t n) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) v[i] = static_cast<uint32_t>(i);
}

__global__ void gather_times_kernel(const uint32_t* __restrict__ pos, const int64_t* __restrict__ times,
                                    uint64_t n, int64_t* out) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = times[pos[i]];
}

struct TrackLaunch {
  const uint64_t* csr_off;   // [a_pad + 1] per-type offsets into csr_time
  const int64_t* csr_time;   // per-type times (original ms), stream order
  const uint32_t* ep_off;    // [n_eps + 1] node offsets (batch-local)
  const uint32_t* ep_types;  // nodes (types already clamped to the spare row)
  const int64_t* ep_low;     // constraints, episode e at ep_off[e] - e
  const int64_t* ep_high;
  uint32_t n_eps;
  uint32_t cap;              // items capacity per slot (max type count)
  int backward;
  uint32_t* items_rank;      // [n_eps][2][cap]
  uint64_t* items_chain;     // [n_eps][2][cap]
  unsigned long long* best;  // [n_eps][cap]
  uint32_t* n_items;         // [n_eps] final item count
  uint32_t* final_buf;       // [n_eps] which of the two buffers holds the result
};

__device__ __forceinline__ uint32_t upper_bound_t(const int64_t* a, uint32_t n, int64_t v) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] <= v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint32_t lower_bound_t(const int64_t* a, uint32_t n, int64_t v) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kTrackThreads) track_kernel(const TrackLaunch p) {
  using Scan = cub::BlockScan<uint32_t, kTrackThreads>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ uint32_t carry_sh;
  const uint32_t e = blockIdx.x;
  const uint32_t b0 = p.ep_off[e], N = p.ep_off[e + 1] - b0;
  const uint64_t cb = static_cast<uint64_t>(b0) - e;
  const bool fwd = !p.backward;
  const size_t slot = static_cast<size_t>(e) * 2 * p.cap;
  uint32_t* rank[2] = {p.items_rank + slot, p.items_rank + slot + p.cap};
  uint64_t* chain[2] = {p.items_chain + slot, p.items_chain + slot + p.cap};
  unsigned long long* best = p.best + static_cast<size_t>(e) * p.cap;

  // seed items: every event of the first (forward) / last (backward) type
  const uint32_t seed = p.ep_types[b0 + (fwd ? 0 : N - 1)];
  const uint64_t s_off = p.csr_off[seed];
  uint32_t n_items = static_cast<uint32_t>(p.csr_off[seed + 1] - s_off);
  for (uint32_t i = threadIdx.x; i < n_items; i += blockDim.x) {
    rank[0][i] = i;
    chain[0][i] = static_cast<uint64_t>(p.csr_time[s_off + i]);
  }
  int cur = 0;
  uint32_t from = seed;
  for (uint32_t step = 1; step < N && n_items > 0; ++step) {
    const uint32_t k = fwd ? step : N - step;  // destination position (fwd) / source (bwd)
    const uint32_t to = p.ep_types[b0 + (fwd ? k : k - 1)];
    const int64_t low = p.ep_low[cb + k - 1], high = p.ep_high[cb + k - 1];
    const uint64_t f_off = p.csr_off[from];
    const uint64_t t_off = p.csr_off[to];
    const uint32_t cnt_t = static_cast<uint32_t>(p.csr_off[to + 1] - t_off);
    const int64_t* t_times = p.csr_time + t_off;
    const unsigned long long sentinel = fwd ? 0ull : ~0ull;
    for (uint32_t r = threadIdx.x; r < cnt_t; r += blockDim.x) best[r] = sentinel;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n_items; i += blockDim.x) {
      const int64_t own = p.csr_time[f_off + rank[cur][i]];
      const uint64_t ch = chain[cur][i];
      uint32_t lo, hi;
      if (fwd) {
        lo = upper_bound_t(t_times, cnt_t, own + low);
        hi = upper_bound_t(t_times, cnt_t, own + high);
      } else {
        lo = lower_bound_t(t_times, cnt_t, own - high);
        hi = lower_bound_t(t_times, cnt_t, own - low);
      }
      for (uint32_t r = lo; r < hi; ++r) {
        if (fwd)
          atomicMax(&best[r], static_cast<unsigned long long>(ch) + 1ull);
        else
          atomicMin(&best[r], static_cast<unsigned long long>(ch));
      }
    }
    __syncthreads();
    // compact surviving ranks, ascending
    const int nxt = cur ^ 1;
    if (threadIdx.x == 0) carry_sh = 0;
    __syncthreads();
    for (uint32_t base = 0; base < cnt_t; base += blockDim.x) {
      const uint32_t r = base + threadIdx.x;
      const unsigned long long v = r < cnt_t ? best[r] : sentinel;
      const uint32_t keep = v != sentinel ? 1u : 0u;
      uint32_t pos, agg;
      Scan(scan_tmp).ExclusiveSum(keep, pos, agg);
      const uint32_t c0 = carry_sh;
      if (keep) {
        rank[nxt][c0 + pos] = r;
        chain[nxt][c0 + pos] = fwd ? v - 1ull : v;
      }
      __syncthreads();
      if (threadIdx.x == 0) carry_sh = c0 + agg;
      __syncthreads();
    }
    n_items = carry_sh;
    cur = nxt;
    from = to;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    p.n_items[e] = n_items;
    p.final_buf[e] = static_cast<uint32_t>(cur);
  }
}

// Occurrence interval i of episode e: forward (chain, own), backward (own,
// chain); own = time of the item's event in the last tracked type.
__device__ __forceinline__ void interval_of(const TrackLaunch& p, uint32_t e, uint32_t i,
                                            int64_t& start, int64_t& end) {
  const uint32_t b0 = p.ep_off[e], N = p.ep_off[e + 1] - b0;
  const bool fwd = !p.backward;
  const uint32_t last = p.ep_types[b0 + (fwd ? N - 1 : 0)];
  const size_t slot = static_cast<size_t>(e) * 2 * p.cap + static_cast<size_t>(p.final_buf[e]) * p.cap;
  const int64_t own = p.csr_time[p.csr_off[last] + p.items_rank[slot + i]];
  const int64_t ch = static_cast<int64_t>(p.items_chain[slot + i]);
  start = fwd ? ch : own;
  end = fwd ? own : ch;
}

// greedy_schedule: one warp per episode, intervals in order.
__global__ void greedy_kernel(const TrackLaunch p, uint64_t* counts, unsigned int* unsorted) {
  const uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (e >= p.n_eps) return;
  const uint32_t n = p.n_items[e];
  uint64_t count = 0;
  int64_t prev_end = INT64_MIN, prev_seen = INT64_MIN;
  bool bad = false;
  for (uint32_t base = 0; base < n; base += 32) {
    int64_t s = 0, en = 0;
    if (base + lane < n) interval_of(p, e, base + lane, s, en);
    const uint32_t m = n - base < 32 ? n - base : 32;
    for (uint32_t j = 0; j < m; ++j) {
      const int64_t sj = __shfl_sync(0xffffffffu, s, j);
      const int64_t ej = __shfl_sync(0xffffffffu, en, j);
      if (ej < prev_seen) bad = true;
      prev_seen = ej;
      if (prev_end < sj) {
        prev_end = ej;
        ++count;
      }
    }
  }
  if (lane == 0) {
    // not end-sorted: the reference sorts and re-runs greedy_schedule
    // (tracking.hpp:395-401); the host recounts these with the exact counter
    counts[e] = bad ? ~0ull : count;
    if (bad) atomicAdd(unsorted, 1u);
  }
}

__global__ void intervals_kernel(const TrackLaunch p, const uint64_t* __restrict__ out_off,
                                 int64_t* starts, int64_t* ends) {
  const uint32_t e = blockIdx.x;
  const uint32_t n = p.n_items[e];
  const uint64_t o = out_off[e];
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    int64_t s, en;
    interval_of(p, e, i, s, en);
    starts[o + i] = s;
    ends[o + i] = en;
  }
}

inline unsigned blocks_for(uint64_t n, unsigned t = 256) {
  return static_cast<unsigned>((n + t - 1) / t);
}

}  // namespace

// Per-type CSR of the loaded stream (positions and original times in stream
// order per type), built on first use.
void Engine::ensure_type_index() {
  if (csr_valid_) return;
  const uint64_t n = stream_.n;
  const uint32_t a_pad = stream_.a_pad;
  const std::vector<uint64_t>& hist = stream_.host_hist(st_);
  csr_off_.assign(a_pad + 1, 0);
  for (uint32_t t = 0; t < a_pad; ++t) csr_off_[t + 1] = csr_off_[t] + hist[t];
  csr_cap_ = 0;
  for (uint32_t t = 0; t < a_pad; ++t)
    csr_cap_ = std::max<uint64_t>(csr_cap_, hist[t]);
  d_csr_off_ = scratch_.get<uint64_t>(kTCsrKeys + 100, a_pad + 1);
  EPI_CUDA(cudaMemcpyAsync(d_csr_off_, csr_off_.data(), (a_pad + 1) * sizeof(uint64_t),
                           cudaMemcpyHostToDevice, st_));
  d_csr_time_ = scratch_.get<int64_t>(kTCsrKeys + 101, n);
  if (n > 0) {
    uint32_t* keys = scratch_.get<uint32_t>(kTCsrKeys, n);
    uint32_t* keys_alt = scratch_.get<uint32_t>(kTCsrKeysAlt, n);
    uint32_t* pos = scratch_.get<uint32_t>(kTCsrPos, n);
    uint32_t* pos_alt = scratch_.get<uint32_t>(kTCsrPosAlt, n);
    EPI_CUDA(cudaMemcpyAsync(keys, stream_.d_types_raw, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st_));
    iota_kernel<<<blocks_for(n), 256, 0, st_>>>(pos, n);
    EPI_CUDA(cudaGetLastError());
    int bits = 1;
    while ((1ull << bits) < stream_.alphabet + 1ull) ++bits;
    cub::DoubleBuffer<uint32_t> kb(keys, keys_alt), vb(pos, pos_alt);
    size_t tmp = 0;
    EPI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, static_cast<int>(n), 0, bits, st_));
    void* d_tmp = scratch_.get<char>(kTCub, tmp + 16);
    EPI_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, kb, vb, static_cast<int>(n), 0, bits, st_));
    gather_times_kernel<<<blocks_for(n), 256, 0, st_>>>(vb.Current(), stream_.d_times_raw, n,
                                                        d_csr_time_);
    EPI_CUDA(cudaGetLastError());
  }
  EPI_CUDA(cudaStreamSynchronize(st_));
  csr_valid_ = true;
}

// Tracking over a CSR batch: per-episode counts (greedy) and, optionally,
// the occurrence intervals (concatenated, offsets per episode).
void Engine::track_batch(const epi_episode_batch& b, uint32_t direction, uint64_t* counts_out,
                         std::vector<uint64_t>* off_out, std::vector<int64_t>* starts,
                         std::vector<int64_t>* ends, epi_stats* stats_out) {
  const uint64_t n = b.n_episodes;
  if (n && (!b.offsets || (!counts_out && !off_out)))
    throw Error(EPI_EINVAL, "epi_track: null batch arrays");
  require_stream();
  for (uint64_t e = 0; e < n; ++e) {
    if (b.offsets[e + 1] < b.offsets[e]) throw Error(EPI_EINVAL, "epi_track: offsets not monotone");
    const uint32_t N = b.offsets[e + 1] - b.offsets[e];
    if (N == 0) throw Error(EPI_EINVAL, "episode must have at least one node");
    const uint64_t cb = b.offsets[e] - e;
    for (uint32_t k = 0; k + 1 < N; ++k)
      if (b.low[cb + k] < 0 || b.low[cb + k] >= b.high[cb + k])
        throw Error(EPI_EINVAL, "interval constraint requires 0 <= low < high");
  }
  ensure_type_index();
  if (off_out) off_out->assign(1, 0);
  if (starts) starts->clear();
  if (ends) ends->clear();
  if (n == 0) return;
  const uint32_t cap = static_cast<uint32_t>(std::max<uint64_t>(csr_cap_, 1));
  // batch so that the per-episode item buffers stay within ~1.5 GB
  const uint64_t per = static_cast<uint64_t>(cap) * (2 * 4 + 2 * 8 + 8);
  const uint64_t batch = std::clamp<uint64_t>((1536ull << 20) / per, 1, 65535);
  const uint32_t A = stream_.alphabet;
  cudaEvent_t e0 = ev0_, e1 = ev1_;
  float total_ms = 0;
  uint64_t launches = 0, items_tracked = 0, sort_fallbacks = 0;
  for (uint64_t base = 0; base < n; base += batch) {
    const uint64_t m = std::min(batch, n - base);
    // batch-local CSR with types clamped to the spare (empty) row
    std::vector<uint32_t> off(m + 1), types;
    std::vector<int64_t> lo, hi;
    for (uint64_t j = 0; j < m; ++j) {
      const uint64_t e = base + j;
      const uint32_t b0 = b.offsets[e], N = b.offsets[e + 1] - b0;
      for (uint32_t k = 0; k < N; ++k) types.push_back(b.types[b0 + k] < A ? b.types[b0 + k] : A);
      const uint64_t cb = b0 - e;
      for (uint32_t k = 0; k + 1 < N; ++k) {
        lo.push_back(b.low[cb + k]);
        hi.push_back(b.high[cb + k]);
      }
      off[j + 1] = off[j] + N;
    }
    const size_t o_off = 0, o_t = (m + 1) * 4, o_lo = ((o_t + types.size() * 4 + 7) / 8) * 8,
                 o_hi = o_lo + lo.size() * 8, o_end = o_hi + hi.size() * 8 + 8;
    char* h = static_cast<char*>(pin_up_.get(o_end));
    std::memcpy(h + o_off, off.data(), (m + 1) * 4);
    std::memcpy(h + o_t, types.data(), types.size() * 4);
    std::memcpy(h + o_lo, lo.data(), lo.size() * 8);
    std::memcpy(h + o_hi, hi.data(), hi.size() * 8);
    char* d = scratch_.get<char>(kTParams, o_end);
    EPI_CUDA(cudaMemcpyAsync(d, h, o_end, cudaMemcpyHostToDevice, st_));
    const size_t i_rank = 0, i_chain = m * 2 * cap * 4, i_best = i_chain + m * 2 * cap * 8,
                 i_n = i_best + m * cap * 8, i_fin = i_n + m * 4, i_cnt = i_fin + m * 4 + 8,
                 i_bad = i_cnt + m * 8, i_end = i_bad + 16;
    char* it = scratch_.get<char>(kTItems, i_end);
    TrackLaunch p{};
    p.csr_off = d_csr_off_;
    p.csr_time = d_csr_time_;
    p.ep_off = reinterpret_cast<const uint32_t*>(d + o_off);
    p.ep_types = reinterpret_cast<const uint32_t*>(d + o_t);
    p.ep_low = reinterpret_cast<const int64_t*>(d + o_lo);
    p.ep_high = reinterpret_cast<const int64_t*>(d + o_hi);
    p.n_eps = static_cast<uint32_t>(m);
    p.cap = cap;
    p.backward = direction != 0;
    p.items_rank = reinterpret_cast<uint32_t*>(it + i_rank);
    p.items_chain = reinterpret_cast<uint64_t*>(it + i_chain);
    p.best = reinterpret_cast<unsigned long long*>(it + i_best);
    p.n_items = reinterpret_cast<uint32_t*>(it + i_n);
    p.final_buf = reinterpret_cast<uint32_t*>(it + i_fin);
    uint64_t* d_cnt = reinterpret_cast<uint64_t*>(it + i_cnt);
    unsigned int* d_bad = reinterpret_cast<unsigned int*>(it + i_bad);
    EPI_CUDA(cudaMemsetAsync(d_bad, 0, 4, st_));
    EPI_CUDA(cudaEventRecord(e0, st_));
    track_kernel<<<static_cast<unsigned>(m), kTrackThreads, 0, st_>>>(p);
    EPI_CUDA(cudaGetLastError());
    greedy_kernel<<<blocks_for(m * 32), 256, 0, st_>>>(p, d_cnt, d_bad);
    EPI_CUDA(cudaGetLastError());
    EPI_CUDA(cudaEventRecord(e1, st_));
    launches += 2;
    std::vector<uint32_t> n_items(m);
    unsigned int bad = 0;
    EPI_CUDA(cudaMemcpyAsync(n_items.data(), p.n_items, m * 4, cudaMemcpyDeviceToHost, st_));
    EPI_CUDA(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, st_));
    if (counts_out)
      EPI_CUDA(cudaMemcpyAsync(counts_out + base, d_cnt, m * 8, cudaMemcpyDeviceToHost, st_));
    EPI_CUDA(cudaStreamSynchronize(st_));
    float ms = 0;
    EPI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    total_ms += ms;
    sort_fallbacks += bad;
    for (uint64_t j = 0; j < m; ++j) items_tracked += n_items[j];
    if (bad && counts_out) {
      // count_tracking == count_fsm on every input (tracking.hpp:388-390):
      // the unsorted episodes are counted by the exact counter
      EpisodeSet fb;
      std::vector<uint64_t> fb_idx;
      for (uint64_t j = 0; j < m; ++j) {
        if (counts_out[base + j] != ~0ull) continue;
        const uint64_t e = base + j;
        const uint32_t b0 = b.offsets[e], N = b.offsets[e + 1] - b0;
        if (fb.N == 0) fb.N = N;
        if (N != fb.N) {  // mixed lengths: one exact call per episode
          EpisodeSet one;
          one.N = N;
          one.types.assign(b.types + b0, b.types + b0 + N);
          one.lo.assign(b.low + (b0 - e), b.low + (b0 - e) + N - 1);
          one.hi.assign(b.high + (b0 - e), b.high + (b0 - e) + N - 1);
          std::vector<uint64_t> c1;
          epi_stats tmp{};
          count_exact(one, c1, tmp, &tmp.pass2_ms);
          counts_out[e] = c1[0];
          continue;
        }
        fb_idx.push_back(e);
        fb.types.insert(fb.types.end(), b.types + b0, b.types + b0 + N);
        fb.lo.insert(fb.lo.end(), b.low + (b0 - e), b.low + (b0 - e) + N - 1);
        fb.hi.insert(fb.hi.end(), b.high + (b0 - e), b.high + (b0 - e) + N - 1);
      }
      if (!fb_idx.empty()) {
        std::vector<uint64_t> c;
        epi_stats tmp{};
        count_exact(fb, c, tmp, &tmp.pass2_ms);
        for (size_t j = 0; j < fb_idx.size(); ++j) counts_out[fb_idx[j]] = c[j];
      }
    }
    if (off_out) {
      std::vector<uint64_t> loff(m + 1, 0);
      for (uint64_t j = 0; j < m; ++j) loff[j + 1] = loff[j] + n_items[j];
      const uint64_t tot = loff[m];
      for (uint64_t j = 0; j < m; ++j) off_out->push_back(off_out->back() + n_items[j]);
      if (tot) {
        uint64_t* d_loff = scratch_.get<uint64_t>(kTOut, m + 1 + 2 * tot);
        int64_t* d_s = reinterpret_cast<int64_t*>(d_loff + m + 1);
        int64_t* d_e = d_s + tot;
        EPI_CUDA(cudaMemcpyAsync(d_loff, loff.data(), (m + 1) * 8, cudaMemcpyHostToDevice, st_));
        intervals_kernel<<<static_cast<unsigned>(m), 256, 0, st_>>>(p, d_loff, d_s, d_e);
        EPI_CUDA(cudaGetLastError());
        launches += 1;
        const size_t old = starts->size();
        starts->resize(old + tot);
        ends->resize(old + tot);
        EPI_CUDA(cudaMemcpyAsync(starts->data() + old, d_s, tot * 8, cudaMemcpyDeviceToHost, st_));
        EPI_CUDA(cudaMemcpyAsync(ends->data() + old, d_e, tot * 8, cudaMemcpyDeviceToHost, st_));
        EPI_CUDA(cudaStreamSynchronize(st_));
      }
    }
  }
  if (stats_out) {
    *stats_out = epi_stats{};
    stats_out->episodes = n;
    stats_out->pass2_episodes = n;
    stats_out->kernel_launches = launches;
    stats_out->total_ms = total_ms;
    stats_out->episode_events = n * stream_.n;
    stats_out->items_tracked = items_tracked;
    stats_out->sort_fallbacks = sort_fallbacks;
  }
}

}  // namespace epi
