// Synthetic spike-train generator: a bit-exact restatement of generate()
// (E/datagen.hpp:71-122) so the bench and the parity tests build the same
// streams as the reference without linking it.
//   * per neuron: Rng(splitmix64(seed ^ (0x42 + neuron))), exponential
//     inter-spike gaps, times truncated to ms   (E/datagen.hpp:91-98)
//   * per embedded episode: Rng(splitmix64(seed ^ (0xE1BEDDED + (e << 20)))),
//     exponential start gaps, uniform gaps inside each constraint window
//                                                (E/datagen.hpp:100-115)
//   * events sorted by (time, type)            (E/datagen.hpp:117-119)
// The reference sorts stably; entries that compare equal under (time, type)
// are identical values, so any sort yields the same stream. Neurons are
// generated in parallel (each owns its RNG) and the sort is a parallel
// chunk-sort + merge, so 10M-event streams build in well under a second.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <thread>
#include <vector>

#include "../../include/episodic_b200.h"
#include "common.cuh"

namespace epi {
namespace {

uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

class Rng {
 public:
  explicit Rng(uint64_t seed) : gen_(seed) {}
  double uniform01() { return (static_cast<double>(gen_() >> 11) + 1.0) * 0x1.0p-53; }
  double exponential(double rate) { return -std::log(uniform01()) / rate; }
  int64_t uniform_gap(int64_t lo, int64_t hi) {
    return lo + 1 + static_cast<int64_t>(gen_() % static_cast<uint64_t>(hi - lo));
  }

 private:
  std::mt19937_64 gen_;
};

struct Ev {
  int64_t time;
  uint32_t type;
  bool operator<(const Ev& o) const { return time != o.time ? time < o.time : type < o.type; }
};

unsigned workers() {
  unsigned hw = std::thread::hardware_concurrency();
  return hw ? std::min(hw, 64u) : 1u;
}

template <class F>
void parallel_for(size_t n, F&& f) {
  unsigned w = std::min<size_t>(workers(), n ? n : 1);
  std::vector<std::thread> th;
  for (unsigned i = 1; i < w; ++i) th.emplace_back([&, i] {
    for (size_t j = i; j < n; j += w) f(j);
  });
  for (size_t j = 0; j < n; j += w) f(j);
  for (auto& t : th) t.join();
}

void parallel_sort(std::vector<Ev>& v) {
  const size_t n = v.size();
  unsigned w = workers();
  if (n < (1u << 16) || w == 1) {
    std::sort(v.begin(), v.end());
    return;
  }
  size_t parts = 1;
  while (parts * 2 <= w) parts *= 2;
  std::vector<size_t> b(parts + 1);
  for (size_t i = 0; i <= parts; ++i) b[i] = n * i / parts;
  parallel_for(parts, [&](size_t i) { std::sort(v.begin() + b[i], v.begin() + b[i + 1]); });
  std::vector<Ev> tmp(n);
  std::vector<Ev>* src = &v;
  std::vector<Ev>* dst = &tmp;
  for (size_t width = 1; width < parts; width *= 2) {
    const size_t pairs = parts / (2 * width);
    parallel_for(pairs, [&](size_t p) {
      size_t lo = b[2 * width * p], mid = b[2 * width * p + width], hi = b[2 * width * (p + 1)];
      std::merge(src->begin() + lo, src->begin() + mid, src->begin() + mid, src->begin() + hi,
                 dst->begin() + lo);
    });
    std::swap(src, dst);
  }
  if (src != &v) v.swap(*src);
}

// validate(Episode) + rate + neuron checks of generate() (E/datagen.hpp:75-80).
void validate_embedded(uint32_t neurons, const epi_episode_batch* emb, const double* rates) {
  const uint64_t ne = emb ? emb->n_episodes : 0;
  for (uint64_t e = 0; e < ne; ++e) {
    uint32_t b0 = emb->offsets[e], N = emb->offsets[e + 1] - b0;
    if (N == 0) throw Error(EPI_EINVAL, "episode must have at least one node");
    uint64_t cb = b0 - e;
    for (uint32_t k = 0; k + 1 < N; ++k)
      if (emb->low[cb + k] < 0 || emb->low[cb + k] >= emb->high[cb + k])
        throw Error(EPI_EINVAL, "interval constraint requires 0 <= low < high");
    if (!(rates[e] > 0)) throw Error(EPI_EINVAL, "generate: injection rate must be > 0");
    for (uint32_t k = 0; k < N; ++k)
      if (emb->types[b0 + k] >= neurons)
        throw Error(EPI_EINVAL, "generate: embedded episode references unknown neuron");
  }
}

}  // namespace

// Returns the generated stream; throws Error(EPI_EINVAL) with the
// reference's messages (E/datagen.hpp:72-80).
void generate_stream(uint32_t neurons, double duration_s, double base_rate_hz, uint64_t seed,
                     const epi_episode_batch* emb, const double* rates, std::vector<uint32_t>& types,
                     std::vector<int64_t>& times) {
  if (neurons < 1) throw Error(EPI_EINVAL, "generate: need at least one neuron");
  if (duration_s < 0) throw Error(EPI_EINVAL, "generate: negative duration");
  if (!(base_rate_hz > 0)) throw Error(EPI_EINVAL, "generate: base rate must be > 0");
  validate_embedded(neurons, emb, rates);
  const uint64_t ne = emb ? emb->n_episodes : 0;

  std::vector<std::vector<Ev>> per(neurons + ne);
  parallel_for(neurons + ne, [&](size_t j) {
    std::vector<Ev>& out = per[j];
    if (j < neurons) {
      const uint32_t neuron = static_cast<uint32_t>(j);
      Rng rng(splitmix64(seed ^ (0x42ULL + neuron)));
      out.reserve(static_cast<size_t>(duration_s * base_rate_hz * 1.05) + 16);
      double t = rng.exponential(base_rate_hz);
      while (t < duration_s) {
        out.push_back({static_cast<int64_t>(t * 1000.0), neuron});
        t += rng.exponential(base_rate_hz);
      }
    } else {
      const uint64_t e = j - neurons;
      const uint32_t b0 = emb->offsets[e], N = emb->offsets[e + 1] - b0;
      const uint64_t cb = b0 - e;
      Rng rng(splitmix64(seed ^ (0xE1BEDDEDULL + (e << 20))));
      double start_s = rng.exponential(rates[e]);
      while (start_s < duration_s) {
        int64_t t = static_cast<int64_t>(start_s * 1000.0);
        out.push_back({t, emb->types[b0]});
        for (uint32_t k = 1; k < N; ++k) {
          t += rng.uniform_gap(emb->low[cb + k - 1], emb->high[cb + k - 1]);
          out.push_back({t, emb->types[b0 + k]});
        }
        start_s += rng.exponential(rates[e]);
      }
    }
  });
  size_t total = 0;
  for (auto& v : per) total += v.size();
  std::vector<Ev> all;
  all.reserve(total);
  for (auto& v : per) {
    all.insert(all.end(), v.begin(), v.end());
    std::vector<Ev>().swap(v);
  }
  parallel_sort(all);
  types.resize(total);
  times.resize(total);
  for (size_t i = 0; i < total; ++i) {
    types[i] = all[i].type;
    times[i] = all[i].time;
  }
}

// The embedded-episode events of generate() alone (E/datagen.hpp:100-115),
// unsorted, after the same validation: the device generator (gen_dev.cu)
// produces the neurons' Poisson background and merges these in.
void generate_embedded_events(uint32_t neurons, double duration_s, uint64_t seed, const epi_episode_batch* emb,
                              const double* rates, std::vector<uint32_t>& types, std::vector<int64_t>& times) {
  validate_embedded(neurons, emb, rates);
  types.clear();
  times.clear();
  const uint64_t ne = emb ? emb->n_episodes : 0;
  for (uint64_t e = 0; e < ne; ++e) {
    const uint32_t b0 = emb->offsets[e], N = emb->offsets[e + 1] - b0;
    const uint64_t cb = b0 - e;
    Rng rng(splitmix64(seed ^ (0xE1BEDDEDULL + (e << 20))));
    double start_s = rng.exponential(rates[e]);
    while (start_s < duration_s) {
      int64_t t = static_cast<int64_t>(start_s * 1000.0);
      types.push_back(emb->types[b0]);
      times.push_back(t);
      for (uint32_t k = 1; k < N; ++k) {
        t += rng.uniform_gap(emb->low[cb + k - 1], emb->high[cb + k - 1]);
        types.push_back(emb->types[b0 + k]);
        times.push_back(t);
      }
      start_s += rng.exponential(rates[e]);
    }
  }
}

// The host-side parts of generate_bursty for the device generator
// (gen_dev.cu): the per-electrode rates (the first two draws of each
// electrode's Rng, Box-Muller, exp - computed here so that libm decides them
// exactly as in generate_bursty) and the shared burst schedule.
void bursty_plan(uint32_t electrodes, double duration_s, double base_rate_hz, double rate_sigma,
                 double burst_rate_hz, double burst_min_ms, double burst_max_ms, double burst_gain, uint64_t seed,
                 std::vector<double>& rates, std::vector<double>& burst_lo, std::vector<double>& burst_hi) {
  if (electrodes < 1) throw Error(EPI_EINVAL, "generate: need at least one neuron");
  if (duration_s < 0) throw Error(EPI_EINVAL, "generate: negative duration");
  if (!(base_rate_hz > 0)) throw Error(EPI_EINVAL, "generate: base rate must be > 0");
  if (!(burst_gain >= 1) || burst_rate_hz < 0 || burst_min_ms < 0 || burst_max_ms < burst_min_ms)
    throw Error(EPI_EINVAL, "generate_bursty: invalid burst parameters");
  burst_lo.clear();
  burst_hi.clear();
  if (burst_rate_hz > 0) {
    Rng rb(splitmix64(seed ^ 0xB1257ULL));
    double t = rb.exponential(burst_rate_hz);
    while (t < duration_s) {
      const double len = (burst_min_ms + (burst_max_ms - burst_min_ms) * rb.uniform01()) / 1000.0;
      burst_lo.push_back(t);
      burst_hi.push_back(std::min(t + len, duration_s));
      t += len + rb.exponential(burst_rate_hz);
    }
  }
  rates.resize(electrodes);
  for (uint32_t e = 0; e < electrodes; ++e) {
    Rng rng(splitmix64(seed ^ (0xB0B5ULL + e)));
    const double u1 = rng.uniform01(), u2 = rng.uniform01();
    const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    rates[e] = base_rate_hz * std::exp(rate_sigma * z);
  }
}

// MEA-culture-shaped bursty generator (the reference
// generator has no burst model, E/datagen.hpp:91-98). Deterministic under a
// seed, with the reference's Rng (mt19937_64 raw output + splitmix64 seeds):
//   * electrode e fires as a homogeneous Poisson process at
//     r_e = base_rate * exp(rate_sigma * z_e), z_e ~ N(0,1) (Box-Muller),
//     Rng(splitmix64(seed ^ (0xB0B5 + e)));
//   * network bursts start as a Poisson process at burst_rate_hz and last
//     uniform [burst_min_ms, burst_max_ms], Rng(splitmix64(seed ^ 0xB1257));
//     inside a burst every electrode fires additionally at
//     r_e * (burst_gain - 1) (so the total rate is burst_gain * r_e);
//   * embedded episodes exactly as generate(): exponential starts, uniform
//     gaps inside each constraint window;
//   * events sorted by (time, type); times truncated to ms.
void generate_bursty(uint32_t electrodes, double duration_s, double base_rate_hz, double rate_sigma,
                     double burst_rate_hz, double burst_min_ms, double burst_max_ms,
                     double burst_gain, uint64_t seed, const epi_episode_batch* emb,
                     const double* rates, std::vector<uint32_t>& types,
                     std::vector<int64_t>& times) {
  if (electrodes < 1) throw Error(EPI_EINVAL, "generate: need at least one neuron");
  if (duration_s < 0) throw Error(EPI_EINVAL, "generate: negative duration");
  if (!(base_rate_hz > 0)) throw Error(EPI_EINVAL, "generate: base rate must be > 0");
  if (!(burst_gain >= 1) || burst_rate_hz < 0 || burst_min_ms < 0 || burst_max_ms < burst_min_ms)
    throw Error(EPI_EINVAL, "generate_bursty: invalid burst parameters");
  // burst schedule (shared by every electrode)
  std::vector<std::pair<double, double>> bursts;  // [start, end) in seconds
  if (burst_rate_hz > 0) {
    Rng rb(splitmix64(seed ^ 0xB1257ULL));
    double t = rb.exponential(burst_rate_hz);
    while (t < duration_s) {
      const double len = (burst_min_ms + (burst_max_ms - burst_min_ms) * rb.uniform01()) / 1000.0;
      bursts.emplace_back(t, std::min(t + len, duration_s));
      t += len + rb.exponential(burst_rate_hz);
    }
  }
  validate_embedded(electrodes, emb, rates);
  // background + bursts per electrode
  std::vector<std::vector<Ev>> per(electrodes);
  parallel_for(electrodes, [&](size_t j) {
    const uint32_t e = static_cast<uint32_t>(j);
    Rng rng(splitmix64(seed ^ (0xB0B5ULL + e)));
    const double u1 = rng.uniform01(), u2 = rng.uniform01();
    const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    const double r = base_rate_hz * std::exp(rate_sigma * z);
    std::vector<Ev>& out = per[j];
    double t = rng.exponential(r);
    while (t < duration_s) {
      out.push_back({static_cast<int64_t>(t * 1000.0), e});
      t += rng.exponential(r);
    }
    const double extra = r * (burst_gain - 1.0);
    if (extra > 0)
      for (const auto& b : bursts) {
        double s = b.first + rng.exponential(extra);
        while (s < b.second) {
          out.push_back({static_cast<int64_t>(s * 1000.0), e});
          s += rng.exponential(extra);
        }
      }
  });
  size_t total = 0;
  for (auto& v : per) total += v.size();
  std::vector<Ev> all;
  all.reserve(total);
  for (auto& v : per) {
    all.insert(all.end(), v.begin(), v.end());
    std::vector<Ev>().swap(v);
  }
  // embedded episodes: same RNG streams as generate()
  const uint64_t ne = emb ? emb->n_episodes : 0;
  for (uint64_t e = 0; e < ne; ++e) {
    const uint32_t b0 = emb->offsets[e], N = emb->offsets[e + 1] - b0;
    const uint64_t cb = b0 - e;
    Rng rng(splitmix64(seed ^ (0xE1BEDDEDULL + (e << 20))));
    double start_s = rng.exponential(rates[e]);
    while (start_s < duration_s) {
      int64_t t = static_cast<int64_t>(start_s * 1000.0);
      all.push_back({t, emb->types[b0]});
      for (uint32_t k = 1; k < N; ++k) {
        t += rng.uniform_gap(emb->low[cb + k - 1], emb->high[cb + k - 1]);
        all.push_back({t, emb->types[b0 + k]});
      }
      start_s += rng.exponential(rates[e]);
    }
  }
  parallel_sort(all);
  types.resize(all.size());
  times.resize(all.size());
  for (size_t i = 0; i < all.size(); ++i) {
    types[i] = all[i].type;
    times[i] = all[i].time;
  }
}

}  // namespace epi
