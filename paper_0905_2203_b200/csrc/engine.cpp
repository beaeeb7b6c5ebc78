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
#include <cstring>
#include <stdexcept>
#include <unordered_map>

#include "count.h"

namespace epi {
namespace {

enum Slot : size_t {
  kSlotParams = 3,
  kSlotMachines = 4,
  kSlotCounts = 5,
};

constexpr uint64_t kPruned = EPI_COUNT_PRUNED;

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

void validate_constraint(int64_t lo, int64_t hi) {
  if (lo < 0 || lo >= hi)
    throw Error(EPI_EINVAL, "interval constraint requires 0 <= low < high");
}

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

}  // namespace

Engine::Engine(int device) : device_(device) {
  EPI_CUDA(cudaSetDevice(device));
  EPI_CUDA(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, device));
  EPI_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  EPI_CUDA(cudaEventCreate(&ev0_));
  EPI_CUDA(cudaEventCreate(&ev1_));
  EPI_CUDA(cudaEventCreate(&ev2_));
}

Engine::~Engine() {
  cudaSetDevice(device_);
  stream_.release();
  if (ev0_) cudaEventDestroy(ev0_);
  if (ev1_) cudaEventDestroy(ev1_);
  if (ev2_) cudaEventDestroy(ev2_);
  if (st_) cudaStreamDestroy(st_);
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
  stream_.reserve_raw(n);
  h2d(stream_.d_types_raw, types, n * sizeof(uint32_t));
  h2d(stream_.d_times_raw, times, n * sizeof(int64_t));
  stream_.load(n, alphabet, st_, scratch_);
}

void Engine::load_stream_device(const uint32_t* d_types, const int64_t* d_times, uint64_t n,
                                uint32_t alphabet) {
  if (n && (!d_types || !d_times)) throw Error(EPI_EINVAL, "epi_load_stream_device: null arrays");
  stream_.reserve_raw(n);
  EPI_CUDA(cudaMemcpyAsync(stream_.d_types_raw, d_types, n * sizeof(uint32_t),
                           cudaMemcpyDeviceToDevice, st_));
  EPI_CUDA(cudaMemcpyAsync(stream_.d_times_raw, d_times, n * sizeof(int64_t),
                           cudaMemcpyDeviceToDevice, st_));
  stream_.load(n, alphabet, st_, scratch_);
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

  // Pack episode parameters. Types outside the alphabet can never fire; they
  // read the always-zero spare column `alphabet` of every tile row.
  const size_t off_types = 0;
  const size_t off_win = align_up(off_types + n * N * 4, 256);
  const size_t off_sigma = align_up(off_win + n * M * 4, 256);
  const size_t off_seg = align_up(off_sigma + n * 4, 256);
  uint32_t max_sigma = 0;
  // Segment plan needs max_sigma; compute parameters first into pinned memory.
  const size_t seg_cap = 65536 + 1;
  const size_t total = align_up(off_seg + seg_cap * 4, 256);
  char* host = static_cast<char*>(pin_up_.get(total));
  uint32_t* h_types = reinterpret_cast<uint32_t*>(host + off_types);
  uint32_t* h_win = reinterpret_cast<uint32_t*>(host + off_win);
  uint32_t* h_sigma = reinterpret_cast<uint32_t*>(host + off_sigma);
  const uint32_t A = stream_.alphabet;
  int64_t max_high = 0;
  int64_t width = -1;  // launch-uniform window width high-low, 0 if mixed
  for (size_t e = 0; e < n; ++e) {
    for (uint32_t k = 0; k < N; ++k) {
      uint32_t t = set.types[e * N + k];
      h_types[e * N + k] = t < A ? t : A;
    }
    uint32_t sig = 0;
    for (uint32_t k = 0; k < M; ++k) {
      int64_t lo = set.lo[e * M + k], hi = set.hi[e * M + k];
      if (hi > kMaxHighWide)
        throw Error(EPI_EUNSUPPORTED, "constraint high > 4095 ms is not supported by the device counter");
      h_win[e * M + k] = static_cast<uint32_t>(lo + 1) | (static_cast<uint32_t>(hi) << 16);
      sig += static_cast<uint32_t>(hi);
      max_high = std::max(max_high, hi);
      if (width == -1)
        width = hi - lo;
      else if (width != hi - lo)
        width = 0;
    }
    h_sigma[e] = sig;
    max_sigma = std::max(max_sigma, sig);
  }
  // Wide windows need a bitmap whose gap compression cap exceeds them, and
  // the local-memory history ring (hist_words 32 ms words per position).
  const bool wide = max_high > kMaxHigh;
  if (wide) stream_.ensure_cap(max_high, st_, scratch_);
  const int32_t hist_words = wide ? static_cast<int32_t>((max_high + 31) / 32) : 2;

  // MapConcatenate plan: enough (episode, segment) machines to fill the GPU,
  // segments long enough that each window lies inside the previous segment.
  const int64_t n_tiles = static_cast<int64_t>(stream_.n_tiles);
  const int32_t window_tiles = static_cast<int32_t>((max_sigma + 31) / 32 + 1);
  // The concat walk is sequential in P, so P is capped (kMaxWalkSegments);
  // segments of >= 32 tiles keep the window overhead and patch rate low.
  constexpr int64_t kMaxWalkSegments = 128;
  const int64_t min_seg = std::max<int64_t>(window_tiles * 4, 32);
  const int64_t target = static_cast<int64_t>(num_sms_) * 2048;
  int64_t want = (target + static_cast<int64_t>(n) - 1) / static_cast<int64_t>(n);
  int64_t max_p = std::max<int64_t>(1, n_tiles / min_seg);
  int64_t P = std::clamp<int64_t>(want, 1, std::min<int64_t>(max_p, kMaxWalkSegments));
  if (const char* force = std::getenv("EPI_FORCE_SEGMENTS")) {
    // Test knob: many short segments exercise the concat walk on small
    // streams. Correctness only needs each segment to span sum(high).
    const int64_t min_ok = std::max<int64_t>(1, (max_sigma + 31) / 32);
    P = std::clamp<int64_t>(std::atoll(force), 1, std::min<int64_t>(std::max<int64_t>(1, n_tiles / min_ok), 65535));
  }
  const int64_t seg_len = (n_tiles + P - 1) / P;
  P = (n_tiles + seg_len - 1) / seg_len;
  int32_t* h_seg = reinterpret_cast<int32_t*>(host + off_seg);
  for (int64_t q = 0; q < P; ++q) h_seg[q] = static_cast<int32_t>(q * seg_len);
  h_seg[P] = static_cast<int32_t>(n_tiles);
  const size_t upload = off_seg + (P + 1) * 4;

  char* d_params = scratch_.get<char>(kSlotParams, upload);
  EPI_CUDA(cudaMemcpyAsync(d_params, host, upload, cudaMemcpyHostToDevice, st_));

  const size_t nm = static_cast<size_t>(P) * n;
  const size_t m_count = 0, m_ncomp = align_up(nm * 4, 256), m_last = align_up(m_ncomp + nm * 4, 256),
               m_first = align_up(m_last + nm * 8, 256), m_total = m_first + nm * 8 * kRecorded;
  char* d_mach = scratch_.get<char>(kSlotMachines, m_total);
  uint64_t* d_counts = scratch_.get<uint64_t>(kSlotCounts, n + 1);
  EPI_CUDA(cudaMemsetAsync(d_counts + n, 0, sizeof(uint64_t), st_));

  CountLaunch p{};
  p.occ = stream_.d_occ;
  p.a_pad = stream_.a_pad;
  p.n_tiles = static_cast<int32_t>(n_tiles);
  p.seg_g = reinterpret_cast<const int32_t*>(d_params + off_seg);
  p.P = static_cast<int32_t>(P);
  p.window_tiles = window_tiles;
  p.chunk_tiles = static_cast<int32_t>(chunk_tiles_for(stream_.a_pad));
  p.n_eps = static_cast<uint32_t>(n);
  p.ep_types = reinterpret_cast<const uint32_t*>(d_params + off_types);
  p.ep_win = reinterpret_cast<const uint32_t*>(d_params + off_win);
  p.ep_sigma = reinterpret_cast<const uint32_t*>(d_params + off_sigma);
  p.f_count = reinterpret_cast<uint32_t*>(d_mach + m_count);
  p.f_ncomp = reinterpret_cast<uint32_t*>(d_mach + m_ncomp);
  p.f_last = reinterpret_cast<uint64_t*>(d_mach + m_last);
  p.f_first = reinterpret_cast<uint64_t*>(d_mach + m_first);
  p.counts = d_counts;
  p.patches = reinterpret_cast<unsigned long long*>(d_counts + n);

  p.hist_words = hist_words;

  EPI_CUDA(cudaEventRecord(ev0_, st_));
  if (wide)
    launch_machines_wide(static_cast<int>(N), p, st_);
  else
    launch_machines(static_cast<int>(N), width > 0 ? static_cast<int>(width) : 0, p, st_);
  EPI_CUDA(cudaEventRecord(ev2_, st_));
  if (wide)
    launch_walk_wide(static_cast<int>(N), p, st_);
  else
    launch_walk(static_cast<int>(N), p, st_);
  EPI_CUDA(cudaEventRecord(ev1_, st_));

  uint64_t* h_counts = static_cast<uint64_t*>(pin_down_.get((n + 1) * sizeof(uint64_t)));
  EPI_CUDA(cudaMemcpyAsync(h_counts, d_counts, (n + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                           st_));
  EPI_CUDA(cudaStreamSynchronize(st_));
  float ms = 0, map_ms = 0;
  EPI_CUDA(cudaEventElapsedTime(&ms, ev0_, ev1_));
  EPI_CUDA(cudaEventElapsedTime(&map_ms, ev0_, ev2_));
  std::memcpy(counts.data(), h_counts, n * sizeof(uint64_t));
  stats.patches += h_counts[n];
  stats.segments = static_cast<uint64_t>(P);
  stats.kernel_launches += 2;
  stats.map_launches += 1;
  stats.total_ms += ms;
  stats.map_ms += map_ms;
  stats.concat_ms += ms - map_ms;
  stats.h2d_bytes += upload;
  stats.d2h_bytes += (n + 1) * sizeof(uint64_t);
  stats.episode_events += static_cast<uint64_t>(n) * stream_.n;
  // Matched-pair work model: every event of every episode position's type.
  uint64_t matched = 0;
  for (size_t e = 0; e < n; ++e)
    for (uint32_t k = 0; k < N; ++k) matched += stream_.type_hist[h_types[e * N + k]];
  stats.matched_pairs += matched;
  uint64_t tiles = 0;
  for (int64_t q = 0; q < P; ++q)
    tiles += static_cast<uint64_t>(h_seg[q + 1] - std::max<int64_t>(h_seg[q] - window_tiles, 0));
  stats.tile_steps += tiles * n;
  if (ms_out) *ms_out += ms;
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
  // Pass 1: one relaxed episode per distinct type sequence, each constraint
  // widened to the hull (min low, max high] over the sequence's variants.
  // Every variant's occurrences are occurrences of the hull episode, and a
  // maximum non-overlapped set cannot shrink when occurrences are added, so
  // count(hull) >= count(variant): a sound upper bound. Singleton groups are
  // exact already.
  const uint32_t N = set.N, M = N - 1;
  std::unordered_map<uint64_t, std::vector<uint32_t>> buckets;
  buckets.reserve(n);
  std::vector<uint32_t> group(n);
  EpisodeSet relaxed;
  relaxed.N = N;
  std::vector<uint32_t> gsize;
  std::vector<uint32_t> grep;
  for (size_t i = 0; i < n; ++i) {
    const uint32_t* t = &set.types[i * N];
    uint64_t h = hash_span(t, N, nullptr, nullptr, 0);
    auto& cand = buckets[h];
    uint32_t g = UINT32_MAX;
    for (uint32_t gi : cand)
      if (std::memcmp(&relaxed.types[static_cast<size_t>(gi) * N], t, N * 4) == 0) {
        g = gi;
        break;
      }
    if (g == UINT32_MAX) {
      g = static_cast<uint32_t>(gsize.size());
      cand.push_back(g);
      relaxed.types.insert(relaxed.types.end(), t, t + N);
      relaxed.lo.insert(relaxed.lo.end(), &set.lo[i * M], &set.lo[i * M] + M);
      relaxed.hi.insert(relaxed.hi.end(), &set.hi[i * M], &set.hi[i * M] + M);
      gsize.push_back(1);
      grep.push_back(static_cast<uint32_t>(i));
    } else {
      ++gsize[g];
      for (uint32_t k = 0; k < M; ++k) {
        int64_t& lo = relaxed.lo[static_cast<size_t>(g) * M + k];
        int64_t& hi = relaxed.hi[static_cast<size_t>(g) * M + k];
        lo = std::min(lo, set.lo[i * M + k]);
        hi = std::max(hi, set.hi[i * M + k]);
      }
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
  if (mode > EPI_MODE_MINE) throw Error(EPI_EINVAL, "epi_count: unknown mode");
  // validate(Episode) for every candidate first (E/types.hpp:87-92).
  std::vector<uint32_t> lens(n);
  for (uint64_t e = 0; e < n; ++e) {
    if (b.offsets[e + 1] < b.offsets[e]) throw Error(EPI_EINVAL, "epi_count: offsets not monotone");
    uint32_t N = b.offsets[e + 1] - b.offsets[e];
    if (N == 0) throw Error(EPI_EINVAL, "episode must have at least one node");
    const uint64_t cb = b.offsets[e] - e;
    for (uint32_t k = 0; k + 1 < N; ++k) validate_constraint(b.low[cb + k], b.high[cb + k]);
    lens[e] = N;
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
  if (stats_out) *stats_out = stats;
}

// generate_candidates (E/miner.hpp:76-109). `frequent` holds the level-1
// frequent episodes in candidate order; the join key of the reference
// (episode_key, E/miner.hpp:52-68: types and constraints of a contiguous
// slice) is hashed and verified, and the output order is the reference's:
// lefts in frequent order, rights in bucket (frequent) order.
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
    out.types.reserve(nf * nf * alphabet.size() * 2);
    for (size_t l = 0; l < nf; ++l)
      for (size_t r = 0; r < nf; ++r)
        for (const auto& c : alphabet) {
          out.types.push_back(frequent.types[l]);
          out.types.push_back(frequent.types[r]);
          out.lo.push_back(c.first);
          out.hi.push_back(c.second);
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
  std::unordered_map<uint64_t, std::vector<uint32_t>> by_prefix;
  by_prefix.reserve(nf * 2);
  for (size_t i = 0; i < nf; ++i) by_prefix[key_hash(i, 0)].push_back(static_cast<uint32_t>(i));
  for (size_t l = 0; l < nf; ++l) {
    auto it = by_prefix.find(key_hash(l, 1));
    if (it == by_prefix.end()) continue;
    for (uint32_t r : it->second) {
      if (!key_eq(r, 0, l, 1)) continue;
      out.types.insert(out.types.end(), &frequent.types[l * F], &frequent.types[l * F] + F);
      out.types.push_back(frequent.types[static_cast<size_t>(r) * F + F - 1]);
      out.lo.insert(out.lo.end(), &frequent.lo[l * FM], &frequent.lo[l * FM] + FM);
      out.hi.insert(out.hi.end(), &frequent.hi[l * FM], &frequent.hi[l * FM] + FM);
      out.lo.push_back(frequent.lo[static_cast<size_t>(r) * FM + FM - 1]);
      out.hi.push_back(frequent.hi[static_cast<size_t>(r) * FM + FM - 1]);
    }
  }
}

// mine (E/miner.hpp:114-173) with the counting block replaced by one
// device count per level.
void Engine::mine(const epi_mine_config& cfg, epi_mine_result* out) {
  if (cfg.threshold < 1) throw Error(EPI_EINVAL, "mine: threshold must be >= 1");
  if (cfg.max_level < 1) throw Error(EPI_EINVAL, "mine: max_level must be >= 1");
  if (cfg.n_alpha == 0) throw Error(EPI_EINVAL, "mine: constraint alphabet must not be empty");
  std::vector<std::pair<int64_t, int64_t>> alpha;
  for (uint64_t i = 0; i < cfg.n_alpha; ++i) {
    validate_constraint(cfg.alpha_low[i], cfg.alpha_high[i]);
    alpha.emplace_back(cfg.alpha_low[i], cfg.alpha_high[i]);
  }
  m_level_cands_.clear();
  m_level_off_.assign(1, 0);
  m_level_ms_.clear();
  m_counts_.clear();
  m_off_.assign(1, 0);
  m_types_.clear();
  m_lo_.clear();
  m_hi_.clear();
  epi_stats totals{};

  EpisodeSet frequent, cands;
  std::vector<uint64_t> counts;
  for (size_t level = 1; level <= cfg.max_level; ++level) {
    auto t0 = std::chrono::steady_clock::now();
    generate_candidates(level, frequent, alpha, stream_.alphabet, cands);
    const size_t nc = cands.size();
    if (nc == 0) break;
    count_set(cands, cfg.threshold, level == 1 ? EPI_MODE_EXACT : cfg.mode, counts, totals);
    EpisodeSet next;
    next.N = cands.N;
    const uint32_t N = cands.N, M = N - 1;
    for (size_t i = 0; i < nc; ++i) {
      if (counts[i] == kPruned || counts[i] < cfg.threshold) continue;
      next.types.insert(next.types.end(), &cands.types[i * N], &cands.types[i * N] + N);
      next.lo.insert(next.lo.end(), &cands.lo[i * M], &cands.lo[i * M] + M);
      next.hi.insert(next.hi.end(), &cands.hi[i * M], &cands.hi[i * M] + M);
      m_counts_.push_back(counts[i]);
      for (uint32_t k = 0; k < N; ++k) m_types_.push_back(cands.types[i * N + k]);
      for (uint32_t k = 0; k < M; ++k) {
        m_lo_.push_back(cands.lo[i * M + k]);
        m_hi_.push_back(cands.hi[i * M + k]);
      }
      m_off_.push_back(static_cast<uint32_t>(m_types_.size()));
    }
    m_level_cands_.push_back(nc);
    m_level_off_.push_back(m_counts_.size());
    m_level_ms_.push_back(
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    frequent = std::move(next);
    if (frequent.size() == 0) break;
  }
  out->n_levels = m_level_cands_.size();
  out->level_candidates = m_level_cands_.data();
  out->level_offsets = m_level_off_.data();
  out->level_ms = m_level_ms_.data();
  out->frequent.n_episodes = m_counts_.size();
  out->frequent.offsets = m_off_.data();
  out->frequent.types = m_types_.data();
  out->frequent.low = m_lo_.data();
  out->frequent.high = m_hi_.data();
  out->counts = m_counts_.data();
  out->totals = totals;
}

}  // namespace epi
