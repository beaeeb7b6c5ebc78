// episodic_b200.hpp — C++ adaptor over the C-ABI (episodic_b200.h) with the
// reference's signatures, so a caller of the reference library
// (/root/reference/proj/include/episodic) swaps the counting backend without
// touching its data model:
//
//   reference                                      adaptor (namespace episodic::b200)
//   count_fsm(stream, ep)          fsm.hpp:101      count_fsm(ctx, stream, ep)
//   count_tracking(s, idx, ep, o)  tracking.hpp:391 count_tracking(ctx, s, idx, ep, o)
//   count_mapconcat(s, ep, P, w)   mapconcat.hpp:71 count_mapconcat(ctx, s, ep, P, w)
//   (loop at miner.hpp:145-154)                     count_batch(ctx, stream, episodes)
//   mine(stream, cfg)              miner.hpp:114    mine<MiningResult>(ctx, stream, cfg)
//
// The templates accept the reference's own types (EventStream with
// types()/times()/alphabet_size(), Episode with .types/.constraints[].low/
// .high, MiningConfig with .threshold/.constraint_alphabet/.max_level) or
// any type with the same members. Errors are rethrown as the reference's
// exception types: EPI_EINVAL -> std::invalid_argument, EPI_EOVERFLOW ->
// std::overflow_error, EPI_EDATA -> DataErrorT (defaults to
// std::runtime_error; pass episodic::DataError when the reference headers
// are in scope), anything else -> std::runtime_error.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <algorithm>
#include <string>
#include <type_traits>
#include <vector>

#include "episodic_b200.h"

namespace episodic::b200 {

template <class DataErrorT = std::runtime_error>
inline void throw_status(epi_status st, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (st) {
    case EPI_OK:
      return;
    case EPI_EINVAL:
      throw std::invalid_argument(m);
    case EPI_EOVERFLOW:
      throw std::overflow_error(m);
    case EPI_EDATA:
      throw DataErrorT(m);
    default:
      throw std::runtime_error(std::string(epi_status_name(st)) + ": " + m);
  }
}

// Owns one epi_ctx (one CUDA device) and the stream it holds. A stream is
// uploaded once and reused by every count_* / mine call on the same stream:
// the reference's EventStream is immutable once built (E/types.hpp:94-95),
// so a stream is identified by its storage (the addresses of its type and
// time arrays, size, alphabet) plus a fingerprint of 64 evenly spaced events,
// which catches a new stream built where an old one lived. Mutating a loaded
// stream's storage in place is not supported; reload() forces an upload.
class Context {
 public:
  explicit Context(int device = 0) {
    throw_status(epi_create(device, &ctx_), epi_last_error(nullptr));
  }
  // One context over several devices (epi_create_multi): count_batch and
  // mine spread one call over all of them, as the reference's mine() spreads
  // one call over its host thread pool (E/parallel.hpp:28-125).
  explicit Context(const std::vector<int>& devices) {
    throw_status(epi_create_multi(static_cast<int>(devices.size()), devices.data(), &ctx_),
                 epi_last_error(nullptr));
  }
  uint32_t world() const { return epi_world(ctx_); }
  ~Context() { epi_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  epi_ctx* get() const { return ctx_; }
  uint64_t uploads() const { return uploads_; }

  template <class Stream, class DataErrorT = std::runtime_error>
  void load(const Stream& s) {
    const Key k = key_of(s);
    if (loaded_ && k == key_) return;
    reload<Stream, DataErrorT>(s);
  }

  template <class Stream, class DataErrorT = std::runtime_error>
  void reload(const Stream& s) {
    loaded_ = false;
    const auto& ty = s.types();
    const auto& tm = s.times();
    std::vector<uint32_t> types(ty.begin(), ty.end());
    std::vector<int64_t> times(tm.begin(), tm.end());
    throw_status<DataErrorT>(
        epi_load_stream(ctx_, types.data(), times.data(), types.size(), s.alphabet_size()),
        epi_last_error(ctx_));
    key_ = key_of(s);
    loaded_ = true;
    ++uploads_;
  }

 private:
  struct Key {
    const void* types = nullptr;
    const void* times = nullptr;
    uint64_t n = 0, alphabet = 0, fp = 0;
    bool operator==(const Key& o) const {
      return types == o.types && times == o.times && n == o.n && alphabet == o.alphabet && fp == o.fp;
    }
  };
  template <class Stream>
  static Key key_of(const Stream& s) {
    const auto& ty = s.types();
    const auto& tm = s.times();
    Key k;
    k.types = ty.empty() ? nullptr : static_cast<const void*>(&*ty.begin());
    k.times = tm.empty() ? nullptr : static_cast<const void*>(&*tm.begin());
    k.n = ty.size();
    k.alphabet = s.alphabet_size();
    uint64_t h = 1469598103934665603ull;
    const uint64_t n = k.n;
    for (uint64_t j = 0; n && j < 64; ++j) {
      const uint64_t i = j * (n - 1) / 63;
      h = (h ^ static_cast<uint64_t>(ty[i])) * 1099511628211ull;
      h = (h ^ static_cast<uint64_t>(tm[i])) * 1099511628211ull;
    }
    k.fp = h;
    return k;
  }
  epi_ctx* ctx_ = nullptr;
  Key key_;
  bool loaded_ = false;
  uint64_t uploads_ = 0;
};

// CSR form of a range of reference-shaped episodes (epi_episode_batch).
struct Batch {
  std::vector<uint32_t> offsets{0}, types;
  std::vector<int64_t> low, high;

  template <class Ep>
  void add(const Ep& ep) {
    for (auto t : ep.types) types.push_back(static_cast<uint32_t>(t));
    for (const auto& c : ep.constraints) {
      low.push_back(static_cast<int64_t>(c.low));
      high.push_back(static_cast<int64_t>(c.high));
    }
    if (ep.constraints.size() + 1 != ep.types.size() && !ep.types.empty())
      throw std::invalid_argument("episode needs exactly N-1 constraints");
    offsets.push_back(static_cast<uint32_t>(types.size()));
  }
  epi_episode_batch view() const {
    return {offsets.size() - 1, offsets.data(), types.data(), low.data(), high.data()};
  }
};

template <class Stream, class EpisodeRange>
std::vector<uint64_t> count_batch(Context& ctx, const Stream& s, const EpisodeRange& episodes,
                                  uint64_t threshold = 1, uint32_t mode = EPI_MODE_EXACT,
                                  epi_stats* stats = nullptr) {
  ctx.load(s);
  Batch b;
  for (const auto& ep : episodes) b.add(ep);
  std::vector<uint64_t> counts(b.offsets.size() - 1);
  const epi_episode_batch v = b.view();
  throw_status(epi_count(ctx.get(), &v, threshold, mode, counts.data(), nullptr, stats),
               epi_last_error(ctx.get()));
  return counts;
}

template <class Stream, class Ep>
uint64_t count_fsm(Context& ctx, const Stream& s, const Ep& ep) {
  const Ep* one = &ep;
  struct Range {
    const Ep* p;
    const Ep* begin() const { return p; }
    const Ep* end() const { return p + 1; }
  };
  return count_batch(ctx, s, Range{one})[0];
}

// count_tracking (E/tracking.hpp:391-407) on the device tracker
// (epi_count_tracking): opt.direction selects forward / backward tracking
// (Direction::forward = 0, backward = 1, E/tracking.hpp:18); the per-type
// index lives on the device, so the reference's TypeIndex argument is only
// accepted. Stats (the reference's TrackingStats or any type with
// sort_fallbacks / flag_retries / items_tracked) accumulate: items_tracked
// counts the occurrence intervals, sort_fallbacks the episodes whose
// intervals were not end-sorted, flag_retries stays 0 (no slab compaction).
template <class Stream, class Index, class Ep, class Opt, class TStats = void>
uint64_t count_tracking(Context& ctx, const Stream& s, const Index&, const Ep& ep, const Opt& opt,
                        TStats* stats = nullptr) {
  ctx.load(s);
  Batch b;
  b.add(ep);
  const epi_episode_batch v = b.view();
  uint64_t count = 0;
  epi_stats st{};
  throw_status(epi_count_tracking(ctx.get(), &v, static_cast<uint32_t>(opt.direction), &count, &st),
               epi_last_error(ctx.get()));
  if constexpr (!std::is_void_v<TStats>) {
    if (stats) {
      stats->items_tracked += st.items_tracked;
      stats->sort_fallbacks += st.sort_fallbacks;
    }
  }
  return count;
}

// count_mapconcat (E/mapconcat.hpp:71-159) with the caller's segment count
// (epi_count_mapconcat). The device runs every segment's FRESH machine in
// parallel; stats (the reference's MapConcatStats or any type with
// machines_precomputed / machine_hits / patches) report the segments used as
// precomputed machines, the segments whose FRESH record the concat walk used
// as hits, the re-run boundary machines as patches. `workers` has no device
// meaning (the kernel is parallel over segments and episodes).
template <class Stream, class Ep, class MStats = void>
uint64_t count_mapconcat(Context& ctx, const Stream& s, const Ep& ep, size_t segments, unsigned /*workers*/ = 1,
                         MStats* stats = nullptr) {
  if (segments < 1) throw std::invalid_argument("count_mapconcat: segments must be >= 1");
  ctx.load(s);
  Batch b;
  b.add(ep);
  const epi_episode_batch v = b.view();
  uint64_t count = 0;
  epi_stats st{};
  throw_status(epi_count_mapconcat(ctx.get(), &v, segments, &count, &st), epi_last_error(ctx.get()));
  if constexpr (!std::is_void_v<MStats>) {
    if (stats) {
      const uint64_t P = st.segments ? st.segments : 1;
      stats->machines_precomputed = P;
      stats->machine_hits = P - std::min<uint64_t>(P, st.patches);
      stats->patches = st.patches;
    }
  }
  return count;
}

// mine() mirror returning the reference's MiningResult shape: Result needs
// .levels (vector of Level{level, candidates, frequent: vector<pair<Ep,
// uint64_t>>, elapsed_ms}).
template <class Result, class Stream, class Config>
Result mine(Context& ctx, const Stream& s, const Config& cfg, uint32_t mode = EPI_MODE_MINE) {
  ctx.load(s);
  std::vector<int64_t> lo, hi;
  for (const auto& c : cfg.constraint_alphabet) {
    lo.push_back(static_cast<int64_t>(c.low));
    hi.push_back(static_cast<int64_t>(c.high));
  }
  epi_mine_config mc{cfg.threshold, cfg.max_level, lo.data(), hi.data(), lo.size(), mode};
  epi_mine_result r{};
  throw_status(epi_mine(ctx.get(), &mc, &r), epi_last_error(ctx.get()));
  Result out;
  using Level = typename decltype(out.levels)::value_type;
  using Pair = typename decltype(Level{}.frequent)::value_type;
  using Ep = typename Pair::first_type;
  for (uint64_t l = 0; l < r.n_levels; ++l) {
    Level lv;
    lv.level = l + 1;
    lv.candidates = r.level_candidates[l];
    lv.elapsed_ms = r.level_ms[l];
    for (uint64_t e = r.level_offsets[l]; e < r.level_offsets[l + 1]; ++e) {
      Ep ep;
      const uint32_t b0 = r.frequent.offsets[e], b1 = r.frequent.offsets[e + 1];
      for (uint32_t k = b0; k < b1; ++k) ep.types.push_back(r.frequent.types[k]);
      const uint64_t cb = b0 - e;
      for (uint32_t k = 0; k + 1 < b1 - b0; ++k)
        ep.constraints.push_back({r.frequent.low[cb + k], r.frequent.high[cb + k]});
      lv.frequent.emplace_back(std::move(ep), r.counts[e]);
    }
    out.levels.push_back(std::move(lv));
  }
  return out;
}

}  // namespace episodic::b200
