// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference headers under
// /root/reference/proj/include (compiled in place by oracle/Makefile into
// oracle/_ref/libepisodic_ref.so). It exists so that tests/, smoke() and
// bench.py's cpu_baseline / --impl reference leg can run the reference's own
// CPU counting path on the same inputs as the B200 path:
//   count_fsm        E/fsm.hpp:101-106
//   count_tracking   E/tracking.hpp:391-407
//   count_mapconcat  E/mapconcat.hpp:71-159
//   oracle_count     E/oracle.hpp:82-85
//   mine             E/miner.hpp:114-173  (+ write_mining_csv, E/miner.hpp:175-181)
//   generate         E/datagen.hpp:71-122
// No reference source is copied here; the headers are #included by path.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "episodic/episodic.hpp"

using namespace episodic;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const DataError*>(&e)) return 2;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::overflow_error*>(&e)) return 3;
  return 9;
}

EventStream make_stream(const uint32_t* types, const int64_t* times, uint64_t n,
                        uint32_t alphabet) {
  std::vector<Event> ev(n);
  for (uint64_t i = 0; i < n; ++i) ev[i] = Event{types[i], times[i]};
  return EventStream::from_events(std::move(ev), alphabet);
}

std::vector<Episode> make_episodes(const uint32_t* off, const uint32_t* types, const int64_t* lo,
                                   const int64_t* hi, uint64_t n_eps) {
  std::vector<Episode> out(n_eps);
  for (uint64_t e = 0; e < n_eps; ++e) {
    uint32_t b = off[e], en = off[e + 1];
    for (uint32_t k = b; k < en; ++k) out[e].types.push_back(types[k]);
    // One fewer constraint than nodes per episode, so episode e's constraints
    // start at flat slot off[e] - e.
    uint32_t cb = off[e] - static_cast<uint32_t>(e);
    for (uint32_t j = 0; j + 1 < en - b; ++j) out[e].constraints.push_back({lo[cb + j], hi[cb + j]});
  }
  return out;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// algo: 0 = count_fsm, 1 = count_tracking (forward, count-scan-write),
//       2 = count_mapconcat(segments), 3 = oracle_count,
//       4 = count_tracking backward.
// parallel: 0 = one candidate at a time with `workers` inside the count
//           (the "as shipped" level>=3 path, E/miner.hpp:152-153);
//           1 = episode-parallel parallel_chunks over candidates with
//           workers=1 inside (E/miner.hpp:146-150).
// Episodes are CSR: off[n_eps+1] node offsets into types[]; constraints of
// episode e are lo/hi[off[e]-e .. off[e+1]-e-1).
int ref_count_batch(const uint32_t* types, const int64_t* times, uint64_t n, uint32_t alphabet,
                    const uint32_t* off, const uint32_t* ep_types, const int64_t* lo,
                    const int64_t* hi, uint64_t n_eps, int algo, unsigned workers, int parallel,
                    uint64_t segments, uint64_t* out) {
  try {
    EventStream s = make_stream(types, times, n, alphabet);
    std::vector<Episode> eps = make_episodes(off, ep_types, lo, hi, n_eps);
    TypeIndex index = build_index(s);
    auto one = [&](const Episode& ep, unsigned w) -> uint64_t {
      switch (algo) {
        case 0:
          return count_fsm(s, ep);
        case 1:
        case 4: {
          TrackingOptions opt;
          opt.workers = w;
          if (algo == 4) opt.direction = Direction::backward;
          return count_tracking(s, index, ep, opt);
        }
        case 2:
          return count_mapconcat(s, ep, segments, w);
        case 3:
          return oracle_count(s, ep);
        default:
          throw std::invalid_argument("ref_count_batch: unknown algo");
      }
    };
    if (parallel) {
      parallel_chunks(eps.size(), workers, [&](std::size_t, std::size_t b, std::size_t e) {
        for (std::size_t i = b; i < e; ++i) out[i] = one(eps[i], 1);
      });
    } else {
      for (std::size_t i = 0; i < eps.size(); ++i) out[i] = one(eps[i], workers);
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Runs mine() (E/miner.hpp:114) and renders write_mining_csv into a malloc'd
// buffer (*csv_out, free with ref_free). level_candidates[i] receives the
// candidate count of level i+1 (up to max_levels_out entries); *n_levels the
// number of levels produced.
int ref_mine(const uint32_t* types, const int64_t* times, uint64_t n, uint32_t alphabet,
             uint64_t threshold, const int64_t* alpha_lo, const int64_t* alpha_hi,
             uint64_t n_alpha, uint64_t max_level, uint64_t switch_level, int backend,
             unsigned workers, char** csv_out, uint64_t* level_candidates,
             uint64_t max_levels_out, uint64_t* n_levels, double* level_ms) {
  try {
    EventStream s = make_stream(types, times, n, alphabet);
    MiningConfig cfg;
    cfg.threshold = threshold;
    for (uint64_t i = 0; i < n_alpha; ++i) cfg.constraint_alphabet.push_back({alpha_lo[i], alpha_hi[i]});
    cfg.max_level = max_level;
    cfg.strategy_switch_level = switch_level;
    cfg.backend = backend == 0 ? CountAlgo::fsm
                               : (backend == 2 ? CountAlgo::mapconcat : CountAlgo::tracking);
    cfg.workers = workers;
    MiningResult r = mine(s, cfg);
    std::ostringstream os;
    write_mining_csv(os, r, SymbolTable::numeric(alphabet));
    std::string str = os.str();
    char* buf = static_cast<char*>(std::malloc(str.size() + 1));
    std::memcpy(buf, str.c_str(), str.size() + 1);
    *csv_out = buf;
    *n_levels = r.levels.size();
    for (uint64_t i = 0; i < r.levels.size() && i < max_levels_out; ++i) {
      level_candidates[i] = r.levels[i].candidates;
      if (level_ms) level_ms[i] = r.levels[i].elapsed_ms;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// generate() (E/datagen.hpp:71). Embedded episodes use the same CSR layout as
// ref_count_batch. Outputs are malloc'd (free with ref_free).
int ref_generate(uint32_t neurons, double duration_s, double base_rate_hz, uint64_t seed,
                 const uint32_t* off, const uint32_t* ep_types, const int64_t* lo,
                 const int64_t* hi, const double* rates, uint64_t n_emb, uint32_t** types_out,
                 int64_t** times_out, uint64_t* n_out) {
  try {
    GenConfig cfg;
    cfg.neurons = neurons;
    cfg.duration_s = duration_s;
    cfg.base_rate_hz = base_rate_hz;
    cfg.seed = seed;
    std::vector<Episode> eps = make_episodes(off, ep_types, lo, hi, n_emb);
    for (uint64_t e = 0; e < n_emb; ++e) cfg.embedded.push_back({eps[e], rates[e]});
    GenResult g = generate(cfg);
    uint64_t n = g.stream.size();
    auto* t = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * (n ? n : 1)));
    auto* tm = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (n ? n : 1)));
    for (uint64_t i = 0; i < n; ++i) {
      t[i] = g.stream.type_at(i);
      tm[i] = g.stream.time_at(i);
    }
    *types_out = t;
    *times_out = tm;
    *n_out = n;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// find_occurrences (E/tracking.hpp:330-367) for one episode (CSR with one
// entry); direction 0 forward, 1 backward. Outputs malloc'd (ref_free).
int ref_find_occurrences(const uint32_t* types, const int64_t* times, uint64_t n, uint32_t alphabet,
                         const uint32_t* off, const uint32_t* ep_types, const int64_t* lo,
                         const int64_t* hi, int direction, int64_t** starts_out,
                         int64_t** ends_out, uint64_t* n_out) {
  try {
    EventStream s = make_stream(types, times, n, alphabet);
    std::vector<Episode> eps = make_episodes(off, ep_types, lo, hi, 1);
    TypeIndex index = build_index(s);
    TrackingOptions opt;
    opt.direction = direction ? Direction::backward : Direction::forward;
    std::vector<OccurrenceInterval> occ = find_occurrences(s, index, eps[0], opt);
    auto* a = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (occ.size() + 1)));
    auto* b = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (occ.size() + 1)));
    for (size_t i = 0; i < occ.size(); ++i) {
      a[i] = occ[i].start;
      b[i] = occ[i].end;
    }
    *starts_out = a;
    *ends_out = b;
    *n_out = occ.size();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// load_stream (E/io.hpp:22-56) on an in-memory text. Names are returned
// '\n'-joined in id order; on DataError *line_out receives e.line.
int ref_load_stream(const char* text, uint64_t len, uint32_t** types_out, int64_t** times_out,
                    uint64_t* n_out, char** names_out, uint32_t* alphabet_out, uint64_t* line_out) {
  *line_out = 0;
  try {
    std::istringstream in(std::string(text, len));
    LoadedStream ls = load_stream(in);
    const size_t n = ls.stream.size();
    auto* a = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * (n + 1)));
    auto* b = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (n + 1)));
    for (size_t i = 0; i < n; ++i) {
      a[i] = ls.stream.type_at(i);
      b[i] = ls.stream.time_at(i);
    }
    std::string joined;
    for (size_t i = 0; i < ls.symbols.size(); ++i) {
      if (i) joined += '\n';
      joined += ls.symbols.name(static_cast<TypeId>(i));
    }
    char* nm = static_cast<char*>(std::malloc(joined.size() + 1));
    std::memcpy(nm, joined.c_str(), joined.size() + 1);
    *types_out = a;
    *times_out = b;
    *n_out = n;
    *names_out = nm;
    *alphabet_out = static_cast<uint32_t>(ls.symbols.size());
    return 0;
  } catch (const DataError& e) {
    *line_out = e.line;
    return fail(e);
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_free(void* p) { std::free(p); }

unsigned ref_default_workers() { return default_workers(); }

}  // extern "C"
