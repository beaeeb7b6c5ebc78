// TEST INFRASTRUCTURE ONLY — writes the golden fixtures under tests/golden/
// by running the UNMODIFIED reference (headers included in place from
// /root/reference/proj/include and /root/reference/proj/tests/helpers.hpp).
//
//   make -C oracle ref && oracle/_ref/make_golden tests/golden
//
// Fixtures:
//   kats.json        the reference's own known-answer tests (T/test_fsm.cpp,
//                    T/test_mapconcat.cpp, T/test_oracle.cpp,
//                    T/test_tracking.cpp, T/test_miner.cpp), each re-evaluated
//                    through the reference so the literal and computed values
//                    are both recorded.
//   instances.json   InstanceRng corpora with the seeds of the reference's
//                    randomised tests (T/helpers.hpp:13-50): per instance a
//                    64-bit FNV-1a of the stream, the episode, count_fsm and
//                    oracle_count. Tests regenerate the streams from the seed.
//   datagen.json     generate() (E/datagen.hpp:71) digests for the bench
//                    configs and the acceptance datasets.
//   configs.json     per-candidate counts for cfg1 (676 episodes), the cfg2
//                    mining CSV, the first 256 cfg3 candidates.
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "episodic/episodic.hpp"
#include "helpers.hpp"

using namespace episodic;
using json = nlohmann::json;

namespace {

uint64_t fnv_stream(const EventStream& s) {
  uint64_t h = 1469598103934665603ULL;
  auto mix = [&](uint64_t v) {
    for (int b = 0; b < 8; ++b) {
      h ^= (v >> (8 * b)) & 0xff;
      h *= 1099511628211ULL;
    }
  };
  mix(s.size());
  mix(s.alphabet_size());
  for (std::size_t i = 0; i < s.size(); ++i) {
    mix(s.type_at(i));
    mix(static_cast<uint64_t>(s.time_at(i)));
  }
  return h;
}

uint64_t fnv_u64s(const std::vector<uint64_t>& v) {
  uint64_t h = 1469598103934665603ULL;
  for (uint64_t x : v)
    for (int b = 0; b < 8; ++b) {
      h ^= (x >> (8 * b)) & 0xff;
      h *= 1099511628211ULL;
    }
  return h;
}

std::string hex(uint64_t v) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(v));
  return buf;
}

json ep_json(const Episode& ep) {
  json t = json::array(), c = json::array();
  for (auto x : ep.types) t.push_back(x);
  for (auto& k : ep.constraints) c.push_back({k.low, k.high});
  return {{"types", t}, {"constraints", c}};
}

json stream_json(const EventStream& s) {
  json ev = json::array();
  for (std::size_t i = 0; i < s.size(); ++i) ev.push_back({s.type_at(i), s.time_at(i)});
  return {{"events", ev}, {"alphabet", s.alphabet_size()}};
}

// One KAT: stream, episode, literal expected (from the reference test), and
// what count_fsm / oracle_count / count_tracking / count_mapconcat return.
json kat(const std::string& name, const std::string& where, const EventStream& s,
         const Episode& ep, uint64_t expected) {
  TypeIndex idx = build_index(s);
  json j = stream_json(s);
  j["name"] = name;
  j["where"] = where;
  j["episode"] = ep_json(ep);
  j["expected"] = expected;
  j["count_fsm"] = count_fsm(s, ep);
  j["oracle_count"] = s.size() <= 500 ? oracle_count(s, ep) : 0;
  TrackingOptions opt;
  j["count_tracking"] = count_tracking(s, idx, ep, opt);
  j["count_mapconcat_p2"] = count_mapconcat(s, ep, 2);
  return j;
}

Episode chain(std::size_t len, IntervalConstraint gap, TypeId first) {
  Episode ep;
  for (std::size_t i = 0; i < len; ++i) {
    ep.types.push_back(first + static_cast<TypeId>(i));
    if (i > 0) ep.constraints.push_back(gap);
  }
  return ep;
}

const IntervalConstraint kBins[3] = {{0, 5}, {5, 10}, {10, 15}};

GenConfig cfg1_gen() {
  GenConfig g;
  g.neurons = 26;
  g.duration_s = 60;
  g.base_rate_hz = 32;
  g.seed = 1;
  g.embedded.push_back({chain(4, {5, 10}, 0), 2.0});
  return g;
}

GenConfig cfg2_gen() {
  GenConfig g;
  g.neurons = 26;
  g.duration_s = 60;
  g.base_rate_hz = 32;
  g.seed = 1;
  auto mk = [](TypeId first, int a, int b, int c) {
    Episode ep = chain(4, {0, 1}, first);
    ep.constraints = {kBins[a], kBins[b], kBins[c]};
    return ep;
  };
  g.embedded.push_back({mk(0, 1, 1, 1), 5.0});
  g.embedded.push_back({mk(4, 0, 1, 2), 5.0});
  g.embedded.push_back({mk(8, 2, 0, 1), 5.0});
  g.embedded.push_back({mk(12, 1, 2, 0), 5.0});
  return g;
}

GenConfig cfg3_gen() {
  GenConfig g;
  g.neurons = 64;
  g.duration_s = 7813;
  g.base_rate_hz = 20;
  g.seed = 3;
  return g;
}

std::vector<Episode> cfg3_candidates(std::size_t count) {
  std::mt19937_64 rng(5);
  std::vector<Episode> out;
  for (std::size_t i = 0; i < count; ++i) {
    Episode ep;
    for (int k = 0; k < 3; ++k) ep.types.push_back(static_cast<TypeId>(rng() % 64));
    for (int k = 0; k < 2; ++k) ep.constraints.push_back(kBins[rng() % 3]);
    out.push_back(ep);
  }
  return out;
}

json gen_digest(const std::string& name, const GenConfig& g) {
  GenResult r = generate(g);
  json j;
  j["name"] = name;
  j["n"] = r.stream.size();
  j["fnv"] = hex(fnv_stream(r.stream));
  j["last_time"] = r.stream.size() ? r.stream.time_at(r.stream.size() - 1) : 0;
  json inj = json::array();
  for (auto& v : r.injections) inj.push_back(v.size());
  j["injections"] = inj;
  return j;
}

void write(const std::string& path, const json& j) {
  std::ofstream f(path);
  f << j.dump(1) << "\n";
  std::cerr << "wrote " << path << "\n";
}

}  // namespace

int main(int argc, char** argv) {
  std::string dir = argc > 1 ? argv[1] : "tests/golden";
  using testing::stream_of;

  // ---- KATs -------------------------------------------------------------
  json kats = json::array();
  kats.push_back(kat("fsm_window_pair", "T/test_fsm.cpp:10-15",
                     stream_of({{0, 10}, {1, 18}, {2, 30}}, 3), Episode{{0, 1, 2}, {{5, 10}, {10, 15}}}, 1));
  kats.push_back(kat("fsm_two_disjoint_pairs", "T/test_fsm.cpp:17-21",
                     stream_of({{0, 0}, {1, 6}, {0, 20}, {1, 27}}, 2), Episode{{0, 1}, {{5, 10}}}, 2));
  kats.push_back(kat("fsm_no_first_type", "T/test_fsm.cpp:23-27", stream_of({{1, 6}}, 2),
                     Episode{{0, 1}, {{5, 10}}}, 0));
  kats.push_back(kat("tied_single_node_collapse", "T/test_fsm.cpp:49-56",
                     stream_of({{0, 5}, {0, 5}, {0, 9}}, 1), Episode{{0}, {}}, 2));
  kats.push_back(kat("tied_restart_blocked", "T/test_fsm.cpp:58-64",
                     stream_of({{0, 0}, {1, 3}, {0, 3}, {1, 5}}, 2), Episode{{0, 1}, {{0, 5}}}, 1));
  kats.push_back(kat("mapconcat_boundary", "T/test_mapconcat.cpp:19-25",
                     stream_of({{3, 0}, {3, 5}, {0, 22}, {1, 30}, {2, 38}, {3, 50}}, 4),
                     Episode{{0, 1, 2}, {{5, 10}, {5, 10}}}, 1));
  kats.push_back(kat("mapconcat_more_segments_than_events", "T/test_mapconcat.cpp:47-53",
                     stream_of({{0, 1}, {1, 7}}, 2), Episode{{0, 1}, {{5, 10}}}, 1));
  kats.push_back(kat("mapconcat_empty", "T/test_mapconcat.cpp:51-52", stream_of({}, 2),
                     Episode{{0, 1}, {{5, 10}}}, 0));
  kats.push_back(kat("oracle_single_pair", "T/test_oracle.cpp:32-38",
                     stream_of({{0, 1}, {1, 8}}, 2), Episode{{0, 1}, {{5, 10}}}, 1));
  kats.push_back(kat("oracle_no_types", "T/test_oracle.cpp:40-44",
                     stream_of({{1, 3}, {1, 9}}, 2), Episode{{0, 1}, {{5, 10}}}, 0));
  kats.push_back(kat("oracle_distinct_starts", "T/test_oracle.cpp:46-53",
                     stream_of({{0, 0}, {0, 1}, {1, 7}}, 2), Episode{{0, 1}, {{5, 10}}}, 1));
  kats.push_back(kat("tracking_three_node_chain", "T/test_tracking.cpp:56-67",
                     stream_of({{0, 1}, {1, 8}, {2, 20}}, 3), Episode{{0, 1, 2}, {{5, 10}, {10, 15}}}, 1));
  kats.push_back(kat("tracking_shared_event", "T/test_tracking.cpp:128-136",
                     stream_of({{0, 0}, {0, 2}, {1, 6}}, 2), Episode{{0, 1}, {{0, 10}}}, 1));
  kats.push_back(kat("tracking_point_intervals", "T/test_tracking.cpp:45-54",
                     stream_of({{0, 2}, {1, 3}, {0, 7}}, 2), Episode{{0}, {}}, 2));
  {
    std::vector<Event> ev{{0, 0}};
    for (TimeMs t = 1; t <= 9; ++t) ev.push_back({1, t});
    kats.push_back(kat("tracking_flag_retry", "T/test_tracking.cpp:161-176", stream_of(ev, 2),
                       Episode{{0, 1}, {{0, 10}}}, 1));
  }
  kats.push_back(kat("track_step_dedup_stream", "T/test_tracking.cpp:20-34",
                     stream_of({{0, 0}, {0, 3}, {1, 6}, {1, 9}, {1, 12}}, 2),
                     Episode{{0, 1}, {{5, 10}}}, 1));
  kats.push_back(kat("miner_two_event", "T/test_miner.cpp:69-80", stream_of({{0, 0}, {1, 7}}, 2),
                     Episode{{0, 1}, {{5, 10}}}, 1));
  // Wide constraints: exercise high up to 63 and beyond (device mask limit).
  kats.push_back(kat("wide_window_63", "new: high=63 edge", stream_of({{0, 0}, {1, 63}, {0, 70}, {1, 134}}, 2),
                     Episode{{0, 1}, {{0, 63}}}, 1));
  kats.push_back(kat("wide_window_100", "new: high>63", stream_of({{0, 0}, {1, 99}, {0, 120}, {1, 220}}, 2),
                     Episode{{0, 1}, {{50, 100}}}, 2));

  json mkat = json::array();
  {
    // T/test_miner.cpp:69-80 and 134-151: two-event mine + CSV line.
    EventStream s = stream_of({{0, 0}, {1, 7}}, 2);
    MiningConfig cfg;
    cfg.threshold = 1;
    cfg.constraint_alphabet = {{5, 10}};
    cfg.max_level = 8;
    cfg.workers = 2;
    MiningResult r = mine(s, cfg);
    std::ostringstream csv;
    write_mining_csv(csv, r, SymbolTable::numeric(2));
    json j = stream_json(s);
    j["name"] = "mine_two_event";
    j["threshold"] = 1;
    j["alphabet_bins"] = json::array({{5, 10}});
    j["max_level"] = 8;
    j["csv"] = csv.str();
    json cands = json::array();
    for (auto& l : r.levels) cands.push_back(l.candidates);
    j["level_candidates"] = cands;
    mkat.push_back(j);
  }
  {
    // T/test_miner.cpp:112-132: backend identity on a random stream.
    testing::InstanceRng rng(82);
    EventStream s = testing::random_stream(rng, 150, 3, 2);
    for (int variant = 0; variant < 2; ++variant) {
      MiningConfig cfg;
      cfg.threshold = variant == 0 ? 2 : 3;
      cfg.constraint_alphabet = variant == 0 ? std::vector<IntervalConstraint>{{0, 5}}
                                             : std::vector<IntervalConstraint>{{0, 5}, {2, 7}};
      cfg.max_level = 4;
      cfg.workers = 2;
      MiningResult r = mine(s, cfg);
      std::ostringstream csv;
      write_mining_csv(csv, r, SymbolTable::numeric(s.alphabet_size()));
      json j = stream_json(s);
      j["name"] = variant == 0 ? "mine_backend_identity_seed82" : "mine_seed82_two_bins";
      j["threshold"] = cfg.threshold;
      json bins = json::array();
      for (auto& c : cfg.constraint_alphabet) bins.push_back({c.low, c.high});
      j["alphabet_bins"] = bins;
      j["max_level"] = 4;
      j["csv"] = csv.str();
      json cands = json::array();
      for (auto& l : r.levels) cands.push_back(l.candidates);
      j["level_candidates"] = cands;
      mkat.push_back(j);
    }
  }
  {
    // T/test_miner.cpp:91-110 shape: random_stream(rng(81), 200, 4, 2).
    testing::InstanceRng rng(81);
    EventStream s = testing::random_stream(rng, 200, 4, 2);
    MiningConfig cfg;
    cfg.threshold = 3;
    cfg.constraint_alphabet = {{0, 5}, {2, 7}};
    cfg.max_level = 4;
    cfg.workers = 2;
    MiningResult r = mine(s, cfg);
    std::ostringstream csv;
    write_mining_csv(csv, r, SymbolTable::numeric(s.alphabet_size()));
    json j = stream_json(s);
    j["name"] = "mine_apriori_seed81";
    j["threshold"] = 3;
    j["alphabet_bins"] = json::array({{0, 5}, {2, 7}});
    j["max_level"] = 4;
    j["csv"] = csv.str();
    json cands = json::array();
    for (auto& l : r.levels) cands.push_back(l.candidates);
    j["level_candidates"] = cands;
    mkat.push_back(j);
  }
  json gc = json::array();
  {
    // generate_candidates KATs (T/test_miner.cpp:23-66) as raw joins.
    auto dump = [&](const std::string& name, std::size_t level, const std::vector<Episode>& freq,
                    std::vector<IntervalConstraint> alpha, TypeId A) {
      auto c = generate_candidates(level, freq, alpha, A);
      json j;
      j["name"] = name;
      j["level"] = level;
      json f = json::array();
      for (auto& e : freq) f.push_back(ep_json(e));
      j["frequent"] = f;
      json a = json::array();
      for (auto& x : alpha) a.push_back({x.low, x.high});
      j["alphabet_bins"] = a;
      j["alphabet"] = A;
      json out = json::array();
      for (auto& e : c) out.push_back(ep_json(e));
      j["candidates"] = out;
      gc.push_back(j);
    };
    dump("level1", 1, {}, {{5, 10}}, 2);
    dump("join_l3", 3, {Episode{{0, 1}, {{5, 10}}}, Episode{{1, 2}, {{5, 10}}}}, {{5, 10}}, 3);
    dump("join_l3_constraints", 3, {Episode{{0, 1}, {{5, 10}}}, Episode{{1, 2}, {{0, 5}}}},
         {{5, 10}, {0, 5}}, 3);
    dump("join_l4_refuse", 4,
         {Episode{{0, 1, 2}, {{5, 10}, {5, 10}}}, Episode{{1, 2, 0}, {{0, 5}, {5, 10}}}},
         {{5, 10}, {0, 5}}, 3);
    dump("empty_l2", 2, {}, {{5, 10}}, 3);
    dump("empty_l5", 5, {}, {{5, 10}}, 3);
    dump("level2_pairs", 2, {Episode{{0}, {}}, Episode{{2}, {}}}, {{0, 5}, {5, 10}}, 3);
    dump("join_l3_repeats", 3,
         {Episode{{0, 0}, {{0, 5}}}, Episode{{0, 1}, {{0, 5}}}, Episode{{1, 0}, {{0, 5}}}},
         {{0, 5}}, 2);
  }
  write(dir + "/kats.json", json{{"count", kats}, {"mine", mkat}, {"candidates", gc}});

  // ---- InstanceRng corpora ----------------------------------------------
  struct Corpus {
    const char* name;
    uint64_t seed;
    int count;
    std::size_t max_events;
    TypeId max_alphabet;
    TimeMs max_gap;
    std::size_t max_size;
    const char* where;
  };
  const Corpus corpora[] = {
      {"fsm_vs_oracle", 53, 300, 200, 6, 3, 4, "T/test_fsm.cpp:83-90"},
      {"fsm_repeated_types", 54, 200, 120, 2, 3, 4, "T/test_fsm.cpp:92-99"},
      {"tracking_vs_oracle", 62, 250, 200, 6, 3, 4, "T/test_tracking.cpp:225-242"},
      {"mapconcat_segments", 72, 500, 200, 6, 3, 4, "T/test_mapconcat.cpp:137-145"},
      {"acceptance_c1", 20240101, 1000, 200, 6, 3, 4, "T/acceptance.cpp:42-81"},
  };
  json inst = json::array();
  for (const Corpus& c : corpora) {
    testing::InstanceRng rng(c.seed);
    json list = json::array();
    for (int i = 0; i < c.count; ++i) {
      EventStream s = testing::random_stream(rng, c.max_events, c.max_alphabet, c.max_gap);
      Episode ep = testing::random_episode(rng, s.alphabet_size(), c.max_size);
      uint64_t f = count_fsm(s, ep);
      uint64_t o = oracle_count(s, ep);
      TypeIndex idx = build_index(s);
      TrackingOptions opt;
      uint64_t tr = count_tracking(s, idx, ep, opt);
      uint64_t mc = count_mapconcat(s, ep, 3);
      if (f != o || tr != o || mc != o) std::cerr << "reference disagreement in " << c.name << "\n";
      json j;
      j["n"] = s.size();
      j["alphabet"] = s.alphabet_size();
      j["fnv"] = hex(fnv_stream(s));
      j["episode"] = ep_json(ep);
      j["count"] = f;
      list.push_back(j);
    }
    inst.push_back({{"name", c.name},
                    {"seed", c.seed},
                    {"count", c.count},
                    {"max_events", c.max_events},
                    {"max_alphabet", c.max_alphabet},
                    {"max_gap", c.max_gap},
                    {"max_size", c.max_size},
                    {"where", c.where},
                    {"instances", list}});
  }
  write(dir + "/instances.json", inst);

  // ---- datagen digests ----------------------------------------------------
  json gens = json::array();
  gens.push_back(gen_digest("cfg1", cfg1_gen()));
  gens.push_back(gen_digest("cfg2", cfg2_gen()));
  {
    GenConfig g;
    g.neurons = 64;
    g.duration_s = 100;
    g.base_rate_hz = 20;
    g.seed = 424242;
    g.embedded.push_back({chain(5, {5, 10}, 0), 1.0});
    gens.push_back(gen_digest("acceptance_c2", g));
  }
  {
    GenConfig g;
    g.neurons = 8;
    g.duration_s = 20;
    g.base_rate_hz = 10;
    g.seed = 17;
    g.embedded.push_back({Episode{{0, 1, 2, 3}, {{5, 10}, {5, 10}, {0, 6}}}, 2.0});
    gens.push_back(gen_digest("datagen_injections", g));
  }
  {
    GenConfig g;
    g.neurons = 1;
    g.duration_s = 1000000;
    g.base_rate_hz = 1.0;
    g.seed = 99;
    gens.push_back(gen_digest("datagen_reproducible", g));
  }
  gens.push_back(gen_digest("cfg3", cfg3_gen()));
  write(dir + "/datagen.json", gens);

  // ---- config-scale counts -------------------------------------------------
  json cfgs;
  {
    GenResult g = generate(cfg1_gen());
    std::vector<Episode> eps;
    for (TypeId a = 0; a < 26; ++a)
      for (TypeId b = 0; b < 26; ++b) eps.push_back(Episode{{a, b}, {{5, 10}}});
    std::vector<uint64_t> counts(eps.size());
    parallel_chunks(eps.size(), default_workers(), [&](std::size_t, std::size_t b, std::size_t e) {
      for (std::size_t i = b; i < e; ++i) counts[i] = count_fsm(g.stream, eps[i]);
    });
    uint64_t sum = 0;
    for (auto c : counts) sum += c;
    cfgs["cfg1"] = {{"n", g.stream.size()}, {"sum", sum}, {"fnv_counts", hex(fnv_u64s(counts))},
                    {"counts", counts}};
  }
  {
    GenResult g = generate(cfg2_gen());
    MiningConfig cfg;
    cfg.threshold = 250;
    cfg.constraint_alphabet = {kBins[0], kBins[1], kBins[2]};
    cfg.max_level = 4;
    cfg.strategy_switch_level = 99;
    cfg.workers = default_workers();
    MiningResult r = mine(g.stream, cfg);
    std::ostringstream csv;
    write_mining_csv(csv, r, SymbolTable::numeric(26));
    json cands = json::array();
    for (auto& l : r.levels) cands.push_back(l.candidates);
    cfgs["cfg2"] = {{"n", g.stream.size()}, {"csv", csv.str()}, {"level_candidates", cands},
                    {"threshold", 250}};
  }
  {
    GenResult g = generate(cfg3_gen());
    std::vector<Episode> eps = cfg3_candidates(256);
    std::vector<uint64_t> counts(eps.size());
    parallel_chunks(eps.size(), default_workers(), [&](std::size_t, std::size_t b, std::size_t e) {
      for (std::size_t i = b; i < e; ++i) counts[i] = count_fsm(g.stream, eps[i]);
    });
    uint64_t sum64 = 0;
    for (int i = 0; i < 64; ++i) sum64 += counts[i];
    json ej = json::array();
    for (auto& e : eps) ej.push_back(ep_json(e));
    cfgs["cfg3"] = {{"n", g.stream.size()}, {"sum_first64", sum64}, {"counts", counts},
                    {"episodes", ej}};
  }
  write(dir + "/configs.json", cfgs);
  return 0;
}
