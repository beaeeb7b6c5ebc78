// extern "C" boundary (include/episodic_b200.h). Every entry point catches
// and maps exceptions to epi_status; messages follow the reference's.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/episodic_b200.h"
#include "engine.h"
#include "multi.h"

struct CandStore {
  std::vector<uint32_t> gc_off, gc_types;
  std::vector<int64_t> gc_lo, gc_hi;
};

struct epi_ctx {
  epi::Engine engine;  // the (first) device's engine
  CandStore cands;
  std::unique_ptr<epi::MultiGroup> multi;  // epi_create_multi: every rank
  explicit epi_ctx(int device) : engine(device) {}
};

namespace epi {
void generate_stream(uint32_t neurons, double duration_s, double base_rate_hz, uint64_t seed,
                     const epi_episode_batch* emb, const double* rates, std::vector<uint32_t>& types,
                     std::vector<int64_t>& times);
void parse_event_text(const char* text, size_t len, std::vector<uint32_t>& types,
                      std::vector<int64_t>& times, std::vector<std::string>& names);
void generate_bursty(uint32_t electrodes, double duration_s, double base_rate_hz, double rate_sigma,
                     double burst_rate_hz, double burst_min_ms, double burst_max_ms,
                     double burst_gain, uint64_t seed, const epi_episode_batch* emb,
                     const double* rates, std::vector<uint32_t>& types, std::vector<int64_t>& times);
}

namespace {

thread_local std::string g_free_err;

// malloc'd copies released by epi_free.
void export_stream(const std::vector<uint32_t>& t, const std::vector<int64_t>& tm,
                   uint32_t** types_out, int64_t** times_out, uint64_t* n_out) {
  const size_t n = t.size();
  auto* a = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * (n ? n : 1)));
  auto* b = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (n ? n : 1)));
  if (!a || !b) {
    std::free(a);
    std::free(b);
    throw std::bad_alloc();
  }
  std::memcpy(a, t.data(), n * sizeof(uint32_t));
  std::memcpy(b, tm.data(), n * sizeof(int64_t));
  *types_out = a;
  *times_out = b;
  *n_out = n;
}

template <class F>
epi_status guarded(std::string& err, F&& f) {
  try {
    f();
    err.clear();
    return EPI_OK;
  } catch (const epi::Error& e) {
    err = e.what();
    return static_cast<epi_status>(e.status);
  } catch (const std::bad_alloc&) {
    err = "host allocation failed";
    return EPI_ENOMEM;
  } catch (const std::exception& e) {
    err = e.what();
    return EPI_EINVAL;
  }
}

// ---- binary event files (EPIEVT01) -----------------------------------------
// 24-byte header {char magic[8]; u64 n; u32 alphabet; u32 flags = 0}, then
// the n u32 types, zero padding to 8 bytes, the n i64 times (little endian):
// the stream's SoA exactly as epi_load_stream takes it, so a load maps the
// file and uploads straight from the mapping (no parse, no per-event work).
constexpr char kEvtMagic[8] = {'E', 'P', 'I', 'E', 'V', 'T', '0', '1'};
constexpr size_t kEvtHeader = 24;
inline size_t evt_times_off(uint64_t n) { return kEvtHeader + (n * 4 + 7) / 8 * 8; }

struct EventFile {
  void* base = nullptr;
  size_t bytes = 0;
  uint64_t n = 0;
  uint32_t alphabet = 0;
  const uint32_t* types = nullptr;
  const int64_t* times = nullptr;
  explicit EventFile(const char* path) {
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) throw epi::Error(EPI_EDATA, std::string("cannot open event file '") + path + "'");
    struct stat sb {};
    if (::fstat(fd, &sb) != 0 || sb.st_size < static_cast<off_t>(kEvtHeader)) {
      ::close(fd);
      throw epi::Error(EPI_EDATA, std::string("not an event file '") + path + "'");
    }
    bytes = static_cast<size_t>(sb.st_size);
    base = ::mmap(nullptr, bytes, PROT_READ, MAP_PRIVATE, fd, 0);
    ::close(fd);
    if (base == MAP_FAILED) {
      base = nullptr;
      throw epi::Error(EPI_EDATA, std::string("cannot map event file '") + path + "'");
    }
    ::madvise(base, bytes, MADV_SEQUENTIAL | MADV_WILLNEED);
    const char* b = static_cast<const char*>(base);
    uint32_t flags = 0;
    std::memcpy(&n, b + 8, 8);
    std::memcpy(&alphabet, b + 16, 4);
    std::memcpy(&flags, b + 20, 4);
    // the destructor does not run for a throwing constructor: unmap first
    auto reject = [&](const char* what) {
      ::munmap(base, bytes);
      base = nullptr;
      throw epi::Error(EPI_EDATA, std::string(what) + " '" + path + "'");
    };
    if (std::memcmp(b, kEvtMagic, 8) != 0 || flags != 0) reject("not an event file");
    if (n > (bytes - kEvtHeader) / 12 || evt_times_off(n) + n * 8 != bytes) reject("truncated event file");
    types = reinterpret_cast<const uint32_t*>(b + kEvtHeader);
    times = reinterpret_cast<const int64_t*>(b + evt_times_off(n));
  }
  ~EventFile() {
    if (base) ::munmap(base, bytes);
  }
};

}  // namespace

extern "C" {

const char* epi_version(void) {
  return "episodic_b200 0.1 sm_100a: bit-sliced tile automaton (32 ms tiles, high<=63, N<=16), "
         "MapConcatenate segments + concat walk, two-pass hull pruning";
}

const char* epi_status_name(epi_status s) {
  switch (s) {
    case EPI_OK: return "EPI_OK";
    case EPI_EINVAL: return "EPI_EINVAL";
    case EPI_EDATA: return "EPI_EDATA";
    case EPI_EOVERFLOW: return "EPI_EOVERFLOW";
    case EPI_ECUDA: return "EPI_ECUDA";
    case EPI_ENCCL: return "EPI_ENCCL";
    case EPI_ENOMEM: return "EPI_ENOMEM";
    case EPI_EUNSUPPORTED: return "EPI_EUNSUPPORTED";
  }
  return "EPI_UNKNOWN";
}

epi_status epi_create(int device, epi_ctx** out) {
  if (!out) return EPI_EINVAL;
  *out = nullptr;
  return guarded(g_free_err, [&] { *out = new epi_ctx(device); });
}

epi_status epi_create_multi(int n_gpus, const int* devices, epi_ctx** out) {
  if (!out || n_gpus < 1) return EPI_EINVAL;
  *out = nullptr;
  return guarded(g_free_err, [&] {
    std::vector<int> devs(static_cast<size_t>(n_gpus));
    for (int r = 0; r < n_gpus; ++r) devs[r] = devices ? devices[r] : r;
    std::unique_ptr<epi_ctx> c(new epi_ctx(devs[0]));
    if (n_gpus > 1) c->multi = std::make_unique<epi::MultiGroup>(c->engine, devs);
    *out = c.release();
  });
}

uint32_t epi_world(const epi_ctx* ctx) {
  return ctx && ctx->multi ? static_cast<uint32_t>(ctx->multi->world()) : 1u;
}

int epi_uses_nccl(const epi_ctx* ctx) { return ctx && ctx->multi && ctx->multi->nccl() ? 1 : 0; }

void epi_destroy(epi_ctx* ctx) { delete ctx; }

const char* epi_last_error(const epi_ctx* ctx) {
  return ctx ? ctx->engine.err.c_str() : g_free_err.c_str();
}

epi_status epi_load_stream(epi_ctx* ctx, const uint32_t* types, const int64_t* times, uint64_t n,
                           uint32_t alphabet) {
  if (!ctx) return EPI_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->engine.mu);
  return guarded(ctx->engine.err, [&] {
    if (ctx->multi) {
      // replicated stream: every device uploads and builds its bitmap
      ctx->multi->run([&](int r, const epi_shard&) { ctx->multi->rank(r).load_stream_host(types, times, n, alphabet); },
                      0);
    } else {
      ctx->engine.load_stream_host(types, times, n, alphabet);
    }
  });
}

epi_status epi_load_stream_device(epi_ctx* ctx, const uint32_t* d_types, const int64_t* d_times,
                                  uint64_t n, uint32_t alphabet) {
  if (!ctx) return EPI_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->engine.mu);
  return guarded(ctx->engine.err,
                 [&] { ctx->engine.load_stream_device(d_types, d_times, n, alphabet); });
}

uint64_t epi_stream_size(const epi_ctx* ctx) { return ctx ? ctx->engine.stream_size() : 0; }

uint64_t epi_stream_upload_bytes(const epi_ctx* ctx) {
  if (!ctx) return 0;
  uint64_t b = ctx->engine.last_load_h2d;
  if (ctx->multi)
    for (int r = 1; r < ctx->multi->world(); ++r) b += ctx->multi->rank(r).last_load_h2d;
  return b;
}

epi_status epi_count(epi_ctx* ctx, const epi_episode_batch* batch, uint64_t threshold,
                     uint32_t mode, uint64_t* counts_out, uint8_t* frequent_out,
                     epi_stats* stats) {
  if (!ctx || !batch) return EPI_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->engine.mu);
  return guarded(ctx->engine.err, [&] {
    if (ctx->multi) {
      // every rank counts its shard; counts all-gathered, every rank holds all
      const int G = ctx->multi->world();
      const uint64_t n = batch->n_episodes;
      std::vector<std::vector<uint64_t>> c(G);
      std::vector<std::vector<uint8_t>> f(G);
      ctx->multi->run(
          [&](int r, const epi_shard& sh) {
            uint64_t* co = counts_out;
            uint8_t* fo = frequent_out;
            if (r > 0) {
              c[r].resize(n);
              co = c[r].data();
              if (frequent_out) {
                f[r].resize(n);
                fo = f[r].data();
              }
            }
            ctx->multi->rank(r).count_batch_sharded(*batch, threshold, mode, sh, co, fo, r == 0 ? stats : nullptr);
          },
          4096ull * static_cast<uint64_t>(G));
    } else {
      ctx->engine.count_batch(*batch, threshold, mode, counts_out, frequent_out, stats);
    }
  });
}

epi_status epi_find_occurrences(epi_ctx* ctx, const epi_episode_batch* batch, uint32_t direction,
                                uint64_t** offsets_out, int64_t** starts_out, int64_t** ends_out) {
  if (!ctx || !batch || !offsets_out || !starts_out || !ends_out) return EPI_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->engine.mu);
  return guarded(ctx->engine.err, [&] {
    std::vector<uint64_t> off;
    std::vector<int64_t> s, e;
    ctx->engine.track_batch(*batch, direction, nullptr, &off, &s, &e, nullptr);
    auto* o = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * off.size()));
    auto* a = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (s.size() ? s.size() : 1)));
    auto* b = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (e.size() ? e.size() : 1)));
    if (!o || !a || !b) {
      std::free(o);
      std::free(a);
      std::free(b);
      throw std::bad_alloc();
    }
    std::memcpy(o, off.data(), off.size() * sizeof(uint64_t));
    std::memcpy(a, s.data(), s.size() * sizeof(int64_t));
    std::memcpy(b, e.data(), e.size() * sizeof(int64_t));
    *offsets_out = o;
    *starts_out = a;
    *ends_out = b;
  });
}

epi_status epi_count_tracking(epi_ctx* ctx, const epi_episode_batch* batch, uint32_t direction,
                              uint64_t* counts_out, epi_stats* stats) {
  if (!ctx || !batch) return EPI_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->engine.mu);
  return guarded(ctx->engine.err, [&] {
    ctx->engine.track_batch(*batch, direction, counts_out, nullptr, nullptr, nullptr, stats);
  });
}

epi_status epi_count_mapconcat(epi_ctx* ctx, const epi_episode_batch* batch, uint64_t segments,
                               uint64_t* counts_out, epi_stats* stats) {
  if (!ctx || !batch) return EPI_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->engine.mu);
  return guarded(ctx->engine.err, [&] { ctx->engine.count_batch_segments(*batch, segments, counts_out, stats); });
}

epi_status epi_mine(epi_ctx* ctx, const epi_mine_config* cfg, epi_mine_result* out) {
  if (!ctx || !cfg || !out) return EPI_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->engine.mu);
  return guarded(ctx->engine.err, [&] {
    if (ctx->multi) {
      // levels of >= 8192 candidates sharded by episode, one all-gather each
      std::vector<epi_mine_result> res(ctx->multi->world());
      ctx->multi->run([&](int r, const epi_shard& sh) { ctx->multi->rank(r).mine(*cfg, r == 0 ? out : &res[r], &sh); },
                      8192);
    } else {
      ctx->engine.mine(*cfg, out, nullptr);
    }
  });
}

epi_status epi_count_sharded(epi_ctx* ctx, const epi_episode_batch* batch, uint64_t threshold,
                             uint32_t mode, const epi_shard* shard, uint64_t* counts_out,
                             uint8_t* frequent_out, epi_stats* stats) {
  if (!ctx || !batch || !shard) return EPI_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->engine.mu);
  return guarded(ctx->engine.err, [&] {
    ctx->engine.count_batch_sharded(*batch, threshold, mode, *shard, counts_out, frequent_out, stats);
  });
}

epi_status epi_mine_sharded(epi_ctx* ctx, const epi_mine_config* cfg, const epi_shard* shard,
                            epi_mine_result* out) {
  if (!ctx || !cfg || !shard || !out) return EPI_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->engine.mu);
  return guarded(ctx->engine.err, [&] { ctx->engine.mine(*cfg, out, shard); });
}

epi_status epi_generate(uint32_t neurons, double duration_s, double base_rate_hz, uint64_t seed,
                        const epi_episode_batch* embedded, const double* rates,
                        uint32_t** types_out, int64_t** times_out, uint64_t* n_out) {
  if (!types_out || !times_out || !n_out) return EPI_EINVAL;
  return guarded(g_free_err, [&] {
    std::vector<uint32_t> t;
    std::vector<int64_t> tm;
    epi::generate_stream(neurons, duration_s, base_rate_hz, seed, embedded, rates, t, tm);
    export_stream(t, tm, types_out, times_out, n_out);
  });
}

void epi_free(void* p) { std::free(p); }

epi_status epi_generate_stream(epi_ctx* ctx, uint32_t neurons, double duration_s, double base_rate_hz,
                               uint64_t seed, const epi_episode_batch* embedded, const double* rates) {
  if (!ctx) return EPI_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->engine.mu);
  return guarded(ctx->engine.err, [&] {
    if (ctx->multi)
      ctx->multi->run(
          [&](int r, const epi_shard&) {
            ctx->multi->rank(r).generate_stream_device(neurons, duration_s, base_rate_hz, seed, embedded, rates);
          },
          0);
    else
      ctx->engine.generate_stream_device(neurons, duration_s, base_rate_hz, seed, embedded, rates);
  });
}

epi_status epi_generate_bursty_stream(epi_ctx* ctx, uint32_t electrodes, double duration_s,
                                      double base_rate_hz, double rate_sigma, double burst_rate_hz,
                                      double burst_min_ms, double burst_max_ms, double burst_gain,
                                      uint64_t seed, const epi_episode_batch* embedded, const double* rates) {
  if (!ctx) return EPI_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->engine.mu);
  return guarded(ctx->engine.err, [&] {
    auto one = [&](epi::Engine& e) {
      e.generate_bursty_device(electrodes, duration_s, base_rate_hz, rate_sigma, burst_rate_hz, burst_min_ms,
                               burst_max_ms, burst_gain, seed, embedded, rates);
    };
    if (ctx->multi)
      ctx->multi->run([&](int r, const epi_shard&) { one(ctx->multi->rank(r)); }, 0);
    else
      one(ctx->engine);
  });
}

epi_status epi_stream_download(epi_ctx* ctx, uint32_t* types_out, int64_t* times_out) {
  if (!ctx) return EPI_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->engine.mu);
  return guarded(ctx->engine.err, [&] { ctx->engine.download_stream(types_out, times_out); });
}

epi_status epi_parse_events(const char* text, uint64_t len, uint32_t** types_out,
                            int64_t** times_out, uint64_t* n_out, char** names_out,
                            uint32_t* alphabet_out) {
  if (!types_out || !times_out || !n_out || !names_out || !alphabet_out || (len && !text))
    return EPI_EINVAL;
  return guarded(g_free_err, [&] {
    std::vector<uint32_t> t;
    std::vector<int64_t> tm;
    std::vector<std::string> names;
    epi::parse_event_text(text, len, t, tm, names);
    std::string joined;
    for (size_t i = 0; i < names.size(); ++i) {
      if (i) joined += '\n';
      joined += names[i];
    }
    char* nm = static_cast<char*>(std::malloc(joined.size() + 1));
    if (!nm) throw std::bad_alloc();
    std::memcpy(nm, joined.c_str(), joined.size() + 1);
    export_stream(t, tm, types_out, times_out, n_out);
    *names_out = nm;
    *alphabet_out = static_cast<uint32_t>(names.size());
  });
}

epi_status epi_generate_bursty(uint32_t electrodes, double duration_s, double base_rate_hz,
                               double rate_sigma, double burst_rate_hz, double burst_min_ms,
                               double burst_max_ms, double burst_gain, uint64_t seed,
                               const epi_episode_batch* embedded, const double* rates,
                               uint32_t** types_out, int64_t** times_out, uint64_t* n_out) {
  if (!types_out || !times_out || !n_out) return EPI_EINVAL;
  return guarded(g_free_err, [&] {
    std::vector<uint32_t> t;
    std::vector<int64_t> tm;
    epi::generate_bursty(electrodes, duration_s, base_rate_hz, rate_sigma, burst_rate_hz,
                         burst_min_ms, burst_max_ms, burst_gain, seed, embedded, rates, t, tm);
    export_stream(t, tm, types_out, times_out, n_out);
  });
}

epi_status epi_random_episodes(uint64_t seed, uint64_t count, uint32_t nodes, uint32_t alphabet,
                               uint32_t n_bins, uint32_t* types_out, uint32_t* bins_out) {
  if ((count && !types_out) || (count && nodes > 1 && !bins_out)) return EPI_EINVAL;
  return guarded(g_free_err, [&] {
    if (nodes < 1 || alphabet < 1 || (nodes > 1 && n_bins < 1))
      throw epi::Error(EPI_EINVAL, "random_episodes: need nodes >= 1, alphabet >= 1, n_bins >= 1");
    // one sequential std::mt19937_64 stream (the reference's Rng engine,
    // E/datagen.hpp:44-62): per episode `nodes` type draws, then nodes-1 bin
    // draws, each raw output modulo the range
    std::mt19937_64 g(seed);
    for (uint64_t e = 0; e < count; ++e) {
      for (uint32_t k = 0; k < nodes; ++k) types_out[e * nodes + k] = static_cast<uint32_t>(g() % alphabet);
      for (uint32_t k = 0; k + 1 < nodes; ++k)
        bins_out[e * (nodes - 1) + k] = static_cast<uint32_t>(g() % n_bins);
    }
  });
}

epi_status epi_generate_candidates(epi_ctx* ctx, uint64_t level, const epi_episode_batch* frequent,
                                   const int64_t* alpha_low, const int64_t* alpha_high,
                                   uint64_t n_alpha, uint32_t alphabet_size,
                                   epi_episode_batch* out) {
  if (!out) return EPI_EINVAL;
  // Host-only: usable without a device. Output storage lives in ctx, or in
  // thread-local storage when ctx is NULL.
  static thread_local CandStore tls;
  CandStore& E = ctx ? ctx->cands : tls;
  std::string& err = ctx ? ctx->engine.err : g_free_err;
  return guarded(err, [&] {
    if (level < 1) throw epi::Error(EPI_EINVAL, "generate_candidates: level must be >= 1");
    epi::EpisodeSet freq;
    freq.N = static_cast<uint32_t>(level > 1 ? level - 1 : 1);
    const uint64_t nf = (level > 1 && frequent) ? frequent->n_episodes : 0;
    for (uint64_t e = 0; e < nf; ++e) {
      const uint32_t b0 = frequent->offsets[e], N = frequent->offsets[e + 1] - b0;
      if (N != freq.N) throw epi::Error(EPI_EINVAL, "generate_candidates: frequent episodes must have level-1 nodes");
      const uint64_t cb = b0 - e;
      freq.types.insert(freq.types.end(), frequent->types + b0, frequent->types + b0 + N);
      freq.lo.insert(freq.lo.end(), frequent->low + cb, frequent->low + cb + N - 1);
      freq.hi.insert(freq.hi.end(), frequent->high + cb, frequent->high + cb + N - 1);
    }
    std::vector<std::pair<int64_t, int64_t>> alpha;
    for (uint64_t i = 0; i < n_alpha; ++i) alpha.emplace_back(alpha_low[i], alpha_high[i]);
    epi::EpisodeSet outset;
    epi::generate_candidates(level, freq, alpha, alphabet_size, outset);
    const size_t n = outset.size();
    const uint32_t N = outset.N;
    E.gc_off.resize(n + 1);
    for (size_t i = 0; i <= n; ++i) E.gc_off[i] = static_cast<uint32_t>(i * N);
    E.gc_types = std::move(outset.types);
    E.gc_lo = std::move(outset.lo);
    E.gc_hi = std::move(outset.hi);
    out->n_episodes = n;
    out->offsets = E.gc_off.data();
    out->types = E.gc_types.data();
    out->low = E.gc_lo.data();
    out->high = E.gc_hi.data();
  });
}

}  // extern "C"

epi_status epi_write_events(const char* path, const uint32_t* types, const int64_t* times,
                            uint64_t n, uint32_t alphabet) {
  if (!path || (n && (!types || !times))) return EPI_EINVAL;
  return guarded(g_free_err, [&] {
    std::FILE* f = std::fopen(path, "wb");
    if (!f) throw epi::Error(EPI_EDATA, std::string("cannot open event file '") + path + "'");
    char hdr[kEvtHeader] = {};
    std::memcpy(hdr, kEvtMagic, 8);
    std::memcpy(hdr + 8, &n, 8);
    std::memcpy(hdr + 16, &alphabet, 4);
    static const char pad[8] = {};
    const size_t padb = evt_times_off(n) - kEvtHeader - n * 4;
    const bool ok = std::fwrite(hdr, 1, kEvtHeader, f) == kEvtHeader &&
                    (n == 0 || std::fwrite(types, 4, n, f) == n) &&
                    std::fwrite(pad, 1, padb, f) == padb &&
                    (n == 0 || std::fwrite(times, 8, n, f) == n);
    if (std::fclose(f) != 0 || !ok)
      throw epi::Error(EPI_EDATA, std::string("cannot write event file '") + path + "'");
  });
}

epi_status epi_read_events(const char* path, uint32_t** types_out, int64_t** times_out,
                           uint64_t* n_out, uint32_t* alphabet_out) {
  if (!path || !types_out || !times_out || !n_out || !alphabet_out) return EPI_EINVAL;
  return guarded(g_free_err, [&] {
    EventFile ef(path);
    std::vector<uint32_t> t(ef.types, ef.types + ef.n);
    std::vector<int64_t> tm(ef.times, ef.times + ef.n);
    export_stream(t, tm, types_out, times_out, n_out);
    *alphabet_out = ef.alphabet;
  });
}

epi_status epi_load_stream_file(epi_ctx* ctx, const char* path) {
  if (!ctx || !path) return EPI_EINVAL;
  std::lock_guard<std::mutex> lk(ctx->engine.mu);
  return guarded(ctx->engine.err, [&] {
    EventFile ef(path);
    ctx->engine.load_stream_host(ef.types, ef.times, ef.n, ef.alphabet);
  });
}
