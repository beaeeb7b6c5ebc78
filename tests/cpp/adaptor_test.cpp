// TEST INFRASTRUCTURE: the reference's own data model and test vectors,
// counted through the B200 backend via the C++ adaptor (include/
// episodic_b200.hpp) - the drop-in demonstration. Built in the build
// container (needs /root/reference headers for the types and checkers);
// the binary travels to the GPU box and tests/test_cpp_adaptor.py runs it.
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>
#include <vector>

#include "episodic/episodic.hpp"
#include "episodic_b200.hpp"
#include "helpers.hpp"

using namespace episodic;
namespace gpu = episodic::b200;

static int failures = 0;
#define CHECK(cond)                                                  \
  do {                                                               \
    if (!(cond)) {                                                   \
      ++failures;                                                    \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                \
  } while (0)

int main() {
  gpu::Context ctx(0);
  // T/test_fsm.cpp KATs, reference types in, reference expectations out.
  {
    EventStream s = testing::stream_of({{0, 10}, {1, 18}, {2, 30}}, 3);
    CHECK(gpu::count_fsm(ctx, s, Episode{{0, 1, 2}, {{5, 10}, {10, 15}}}) == 1);
  }
  {
    EventStream s = testing::stream_of({{0, 0}, {1, 6}, {0, 20}, {1, 27}}, 2);
    CHECK(gpu::count_fsm(ctx, s, Episode{{0, 1}, {{5, 10}}}) == 2);
  }
  {
    EventStream s = testing::stream_of({{0, 5}, {0, 5}, {0, 9}}, 1);
    CHECK(gpu::count_fsm(ctx, s, Episode{{0}, {}}) == 2);
  }
  {
    EventStream s = testing::stream_of({{0, 0}, {1, 3}, {0, 3}, {1, 5}}, 2);
    CHECK(gpu::count_fsm(ctx, s, Episode{{0, 1}, {{0, 5}}}) == 1);
  }
  // T/test_fsm.cpp:83-99 and T/test_tracking.cpp:225-242 corpora.
  for (auto [seed, n, cnt, alpha] : std::vector<std::tuple<uint64_t, size_t, int, TypeId>>{
           {53, 200, 300, 6}, {54, 120, 200, 2}, {62, 200, 250, 6}}) {
    testing::InstanceRng rng(seed);
    for (int i = 0; i < cnt; ++i) {
      EventStream s = testing::random_stream(rng, n, alpha);
      Episode ep = testing::random_episode(rng, s.alphabet_size());
      const uint64_t want = oracle_count(s, ep);
      CHECK(gpu::count_fsm(ctx, s, ep) == want);
      TypeIndex idx = build_index(s);
      TrackingStats ts;
      CHECK(gpu::count_tracking(ctx, s, idx, ep, TrackingOptions{}, &ts) == want);
      TrackingOptions back;
      back.direction = Direction::backward;
      CHECK(gpu::count_tracking(ctx, s, idx, ep, back, &ts) == want);
      // the reference's own tracking statistics for the same episode
      TrackingStats rs;
      count_tracking(s, idx, ep, TrackingOptions{}, &rs);
      count_tracking(s, idx, ep, back, &rs);
      CHECK(ts.items_tracked == rs.items_tracked);
      CHECK(ts.flag_retries == 0);
      MapConcatStats ms;
      CHECK(gpu::count_mapconcat(ctx, s, ep, 3, 1, &ms) == want);
      CHECK(ms.machines_precomputed >= 1 && ms.machine_hits + ms.patches == ms.machines_precomputed);
    }
  }
  // the stream is uploaded once for any number of calls on it
  {
    testing::InstanceRng rng(83);
    EventStream s = testing::random_stream(rng, 300, 4, 2);
    const uint64_t before = ctx.uploads();
    for (int i = 0; i < 20; ++i) {
      Episode ep = testing::random_episode(rng, s.alphabet_size(), 4);
      CHECK(gpu::count_fsm(ctx, s, ep) == count_fsm(s, ep));
    }
    CHECK(ctx.uploads() == before + 1);
    EventStream s2 = testing::random_stream(rng, 300, 4, 2);
    Episode ep = testing::random_episode(rng, s2.alphabet_size(), 4);
    CHECK(gpu::count_fsm(ctx, s2, ep) == count_fsm(s2, ep));
    CHECK(ctx.uploads() == before + 2);
  }
  // batch over one stream == reference loop
  {
    testing::InstanceRng rng(82);
    EventStream s = testing::random_stream(rng, 200, 5, 2);
    std::vector<Episode> eps;
    for (int i = 0; i < 100; ++i) eps.push_back(testing::random_episode(rng, s.alphabet_size(), 5));
    std::vector<uint64_t> got = gpu::count_batch(ctx, s, eps);
    for (size_t i = 0; i < eps.size(); ++i) CHECK(got[i] == count_fsm(s, eps[i]));
  }
  // mine(): T/test_miner.cpp shapes, CSV byte-equal with the reference.
  {
    struct Case {
      EventStream s;
      MiningConfig cfg;
    };
    std::vector<Case> cases;
    {
      MiningConfig c;
      c.threshold = 1;
      c.constraint_alphabet = {{5, 10}};
      c.max_level = 8;
      cases.push_back({testing::stream_of({{0, 0}, {1, 7}}, 2), c});
    }
    {
      testing::InstanceRng rng(81);
      MiningConfig c;
      c.threshold = 3;
      c.constraint_alphabet = {{0, 5}, {2, 7}};
      c.max_level = 4;
      cases.push_back({testing::random_stream(rng, 200, 4, 2), c});
    }
    for (auto& cs : cases) {
      cs.cfg.workers = 2;
      MiningResult want = mine(cs.s, cs.cfg);
      for (uint32_t mode : {uint32_t{EPI_MODE_MINE}, uint32_t{EPI_MODE_EXACT}}) {
        MiningResult got = gpu::mine<MiningResult>(ctx, cs.s, cs.cfg, mode);
        std::ostringstream a, b;
        SymbolTable sym = SymbolTable::numeric(cs.s.alphabet_size());
        write_mining_csv(a, want, sym);
        write_mining_csv(b, got, sym);
        CHECK(a.str() == b.str());
        CHECK(got.levels.size() == want.levels.size());
        for (size_t l = 0; l < got.levels.size() && l < want.levels.size(); ++l)
          CHECK(got.levels[l].candidates == want.levels[l].candidates);
      }
    }
  }
  // one mine() call over a two-rank context (both ranks on device 0 here):
  // same CSV as the reference
  if (!std::getenv("SKIP_MULTI")) {
    gpu::Context multi(std::vector<int>{0, 0});
    CHECK(multi.world() == 2);
    testing::InstanceRng rng(84);
    EventStream s = testing::random_stream(rng, 3000, 6, 2);
    MiningConfig c;
    c.threshold = 5;
    c.constraint_alphabet = {{0, 5}, {5, 10}};
    c.max_level = 4;
    c.workers = 2;
    MiningResult want = mine(s, c);
    if (std::getenv("VERBOSE")) {
      std::fprintf(stderr, "multi mine: %zu events, levels", s.size());
      for (auto& l : want.levels) std::fprintf(stderr, " %zu", static_cast<size_t>(l.candidates));
      std::fprintf(stderr, "\n");
    }
    MiningResult got = gpu::mine<MiningResult>(multi, s, c);
    if (std::getenv("VERBOSE")) std::fprintf(stderr, "multi mine done\n");
    std::ostringstream a, b;
    SymbolTable sym = SymbolTable::numeric(s.alphabet_size());
    write_mining_csv(a, want, sym);
    write_mining_csv(b, got, sym);
    CHECK(a.str() == b.str());
    std::vector<Episode> eps;
    for (int i = 0; i < 50; ++i) eps.push_back(testing::random_episode(rng, s.alphabet_size(), 4));
    std::vector<uint64_t> cnt = gpu::count_batch(multi, s, eps);
    for (size_t i = 0; i < eps.size(); ++i) CHECK(cnt[i] == count_fsm(s, eps[i]));
  }
  // exception types of the reference
  {
    EventStream s = testing::stream_of({{0, 1}, {1, 7}}, 2);
    bool threw = false;
    try {
      gpu::count_fsm(ctx, s, Episode{{0, 1}, {{5, 5}}});
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
      gpu::count_mapconcat(ctx, s, Episode{{0}, {}}, 0);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  std::printf("%s (%d failures)\n", failures ? "FAIL" : "PASS", failures);
  return failures ? 1 : 0;
}
