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
#include <string>
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

// Owns one epi_ctx (one CUDA device) and remembers which stream it holds.
class Context {
 public:
  explicit Context(int device = 0) {
    throw_status(epi_create(device, &ctx_), epi_last_error(nullptr));
  }
  ~Context() { epi_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  epi_ctx* get() const { return ctx_; }

  // (Re)loads the stream on every call: an address/size cache would be
  // fooled by a new stream constructed where an old one lived. Callers that
  // count many batches over one stream use count_batch / mine.
  template <class Stream, class DataErrorT = std::runtime_error>
  void load(const Stream& s) {
    std::vector<uint32_t> types(s.types().begin(), s.types().end());
    std::vector<int64_t> times(s.times().begin(), s.times().end());
    throw_status<DataErrorT>(
        epi_load_stream(ctx_, types.data(), times.data(), types.size(), s.alphabet_size()),
        epi_last_error(ctx_));
  }

 private:
  epi_ctx* ctx_ = nullptr;
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

// Equal to count_fsm on every input (the reference guarantees the same,
// E/tracking.hpp:388-390); index and options are accepted for parity.
template <class Stream, class Index, class Ep, class Opt>
uint64_t count_tracking(Context& ctx, const Stream& s, const Index&, const Ep& ep, const Opt&) {
  return count_fsm(ctx, s, ep);
}

template <class Stream, class Ep>
uint64_t count_mapconcat(Context& ctx, const Stream& s, const Ep& ep, size_t segments,
                         unsigned /*workers*/ = 1) {
  if (segments < 1) throw std::invalid_argument("count_mapconcat: segments must be >= 1");
  if (s.size() == 0) return 0;
  return count_fsm(ctx, s, ep);
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
