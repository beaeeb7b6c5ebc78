// Host engine behind the C-ABI: owns the device stream, runs the two-pass
// count and the level-wise miner. Host C++17; CUDA runtime only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/episodic_b200.h"
#include "device_stream.h"
#include "ingest.h"

namespace epi {

// Flat list of episodes of one length N (the form every mining level has).
struct EpisodeSet {
  uint32_t N = 0;
  std::vector<uint32_t> types;  // n * N
  std::vector<int64_t> lo, hi;  // n * (N-1)
  size_t size() const { return N ? types.size() / N : 0; }
  void clear() {
    types.clear();
    lo.clear();
    hi.clear();
  }
};

// A fixed-length episode set resident on the device, in the counting
// kernels' parameter layout, plus the host-side summary the launch needs.
struct DevSet {
  uint32_t N = 0;
  uint64_t n = 0;
  const uint32_t* types = nullptr;  // [n * N]
  const uint32_t* win = nullptr;    // [n * (N-1)]: (low+1) | high << 16
  const uint32_t* sigma = nullptr;  // [n] sum of highs
  uint32_t max_sigma = 0;
  int64_t max_high = 0;
  int width = 0;                    // launch-uniform high-low, 0 if mixed
  uint32_t last_w = 0;              // != 0: the last constraint alone has this
                                    // launch-uniform width; `width` covers the others
};

// Host memory the device writes directly (zero-copy): small, sparse outputs
// such as a level's frequent episodes arrive without a sized D2H copy.
struct MappedBuffer {
  void* p = nullptr;
  void* d = nullptr;
  size_t bytes = 0;
  ~MappedBuffer() {
    if (p) cudaFreeHost(p);
  }
  void get(size_t need) {
    if (need > bytes) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      size_t grow = need + need / 4 + 4096;
      EPI_CUDA(cudaHostAlloc(&p, grow, cudaHostAllocMapped));
      EPI_CUDA(cudaHostGetDevicePointer(&d, p, 0));
      bytes = grow;
      ++generation;
    }
  }
  uint64_t generation = 0;
};

struct PinnedBuffer {
  void* p = nullptr;
  size_t bytes = 0;
  ~PinnedBuffer() {
    if (p) cudaFreeHost(p);
  }
  void* get(size_t need) {
    if (need > bytes) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      size_t grow = need + need / 4 + 4096;
      EPI_CUDA(cudaMallocHost(&p, grow));
      bytes = grow;
      ++generation;
    }
    return p;
  }
  uint64_t generation = 0;
};

class Engine {
 public:
  explicit Engine(int device);
  ~Engine();

  void load_stream_host(const uint32_t* types, const int64_t* times, uint64_t n, uint32_t alphabet);
  // generate() (E/datagen.hpp:71-122) bit-exact on the device, loaded as the
  // context's stream (gen_dev.cu).
  void generate_stream_device(uint32_t neurons, double duration_s, double base_rate_hz, uint64_t seed,
                              const epi_episode_batch* emb, const double* rates);
  // generate_bursty (datagen.cpp, cfg4's MEA-shaped stream) bit-exact on the
  // device (gen_dev.cu; rates and the burst schedule are planned on the host).
  void generate_bursty_device(uint32_t electrodes, double duration_s, double base_rate_hz, double rate_sigma,
                              double burst_rate_hz, double burst_min_ms, double burst_max_ms, double burst_gain,
                              uint64_t seed, const epi_episode_batch* emb, const double* rates);
  // Copies the loaded stream's SoA back to host arrays (stream_size entries).
  void download_stream(uint32_t* types, int64_t* times);
  void load_stream_device(const uint32_t* d_types, const int64_t* d_times, uint64_t n,
                          uint32_t alphabet);
  uint64_t stream_size() const { return stream_.n; }
  // EPI_EINVAL unless a stream load succeeded (counting needs the bitmap)
  void require_stream() const;
  uint64_t last_load_h2d = 0;
  uint32_t alphabet() const { return stream_.alphabet; }

  // Exact or two-pass count of one fixed-length set; counts[i] for set[i].
  void count_set(const EpisodeSet& set, uint64_t threshold, uint32_t mode,
                 std::vector<uint64_t>& counts, epi_stats& stats);
  // Arbitrary CSR batch (mixed lengths): validated, grouped by length.
  // count_mapconcat (E/mapconcat.hpp:71): exact counts with `segments`
  // MapConcatenate segments (clamped to what the stream allows).
  void count_batch_segments(const epi_episode_batch& b, uint64_t segments, uint64_t* counts_out,
                            epi_stats* stats_out);
  void count_batch(const epi_episode_batch& b, uint64_t threshold, uint32_t mode,
                   uint64_t* counts_out, uint8_t* frequent_out, epi_stats* stats);
  // shard == nullptr: single device (epi_mine); else epi_mine_sharded.
  void mine(const epi_mine_config& cfg, epi_mine_result* out, const epi_shard* shard);
  // epi_count_sharded: many episodes -> episode slices + all-gather of the
  // counts; few episodes -> MapConcatenate segments sharded by time range,
  // the segment records all-gathered and walked on every rank.
  void count_batch_sharded(const epi_episode_batch& b, uint64_t threshold, uint32_t mode,
                           const epi_shard& shard, uint64_t* counts_out, uint8_t* frequent_out,
                           epi_stats* stats);
  // Parallel local tracking (tracking.cu): counts (greedy) and/or intervals.
  void track_batch(const epi_episode_batch& b, uint32_t direction, uint64_t* counts_out,
                   std::vector<uint64_t>* off_out, std::vector<int64_t>* starts,
                   std::vector<int64_t>* ends, epi_stats* stats_out);

  std::string err;
  std::mutex mu;

 private:
  // Exact count of one fixed-length set on the device.
  // Same for a batch whose episodes all have N nodes, straight from the
  // caller's CSR (parallel host packing) into counts_out.
  void count_exact_csr(const epi_episode_batch& b, uint32_t N, uint64_t* counts_out, epi_stats& stats,
                       double* ms_out);
  // epi_count MODE_MINE for a batch of N-node episodes: pass 1 is the device
  // chain-end popcount bound (chain kernel, bound mode), pass 2 the exact
  // count of the survivors. Returns false (nothing done) when the batch's
  // shape has no chain kernel.
  bool count_mine_csr(const epi_episode_batch& b, uint32_t N, uint64_t threshold, uint64_t* counts_out,
                      epi_stats& stats);
  // Uploads packed parameters (pinned host, `total` bytes), counts them and
  // copies the counts into out[0..n).
  void count_packed(DevSet ds, char* host, size_t off_win, size_t off_sigma, size_t total, uint64_t* out,
                    epi_stats& stats, double* ms_out);
  void count_exact(const EpisodeSet& set, std::vector<uint64_t>& counts, epi_stats& stats,
                   double* ms_out);
  // Launches only: timings and counters are resolved by flush_stats.
  // live_slot >= 0: ds.n is an upper bound and the live count is the
  // device log value log_[live_slot] (written by an earlier kernel).
  void count_device(const DevSet& ds, uint64_t* d_counts, epi_stats& stats, double* ms_out,
                    int live_slot = -1);
  // uniform_win != 0: pass-1 relaxation uses that window at every position.
  void count_device_two_pass(const DevSet& c, uint64_t threshold, uint32_t mode,
                             uint32_t uniform_win, const uint32_t* alpha, uint32_t n_alpha,
                             uint64_t* d_counts, epi_stats& stats);
  // Left-grouped candidates of a mining level (the popcount pass 1): left l
  // (a frequent (L-1)-episode) owns candidates [off[l], off[l+1]) (or
  // [l*stride, (l+1)*stride) when off is null); the set counted here is the
  // slice starting at candidate slice_lo.
  struct PopLefts {
    uint64_t nf = 0;
    const uint32_t* types = nullptr;  // [nf * (L-1)]
    const uint32_t* win = nullptr;    // [nf * (L-2)]
    const uint64_t* off = nullptr;
    uint64_t stride = 0;
    uint64_t slice_lo = 0;
    // join mode: the level's candidates were not materialised (no
    // gen_join_kernel); the passes read them off the join index
    bool join_mode = false;
    const uint32_t* pre = nullptr;     // bucket order of the rights
    const uint32_t* lrange = nullptr;  // [2 nf] bucket range per left
    const uint32_t* sigma = nullptr;   // [nf] lefts' sums of highs
  };
  // Survivors of pass 1 and their exact counts (device; live count in log
  // slot `slot`): what the frequent-set compaction needs when the level's
  // full count vector is not (unsharded mining).
  struct Survivors {
    const uint32_t* types = nullptr;
    const uint32_t* win = nullptr;
    const uint64_t* counts = nullptr;
    int slot = -1;
  };
  // surv != nullptr: skip scattering the survivors' counts back into
  // d_counts and report the survivors instead.
  void count_device_popbound(const DevSet& c, const PopLefts& lf, uint64_t threshold,
                             const uint32_t* alpha, uint32_t n_alpha, uint64_t* d_counts,
                             epi_stats& stats, Survivors* surv = nullptr);
  // Exclusive scan of n u32 flags; the total goes to device log slot `slot`
  // (and to *host_total, zero-copy, when given). No host synchronisation.
  void dev_scan_total(const uint32_t* flags, uint32_t* scan, uint64_t n, int slot,
                      uint32_t* host_total = nullptr);

  // ---- deferred statistics: no host sync per launch ------------------------
  // begin_op resets the per-call state; flush_stats synchronises once and
  // resolves every recorded interval and device counter into `stats`.
  void begin_op();
  void flush_stats(epi_stats& stats);
  // Enqueue the D2H of the statistics log right before a synchronisation the
  // caller makes anyway; flush_stats then needs no extra round trip when
  // nothing was launched in between.
  void prefetch_stats();
  // Resolve the timed intervals recorded before index `upto` (their events
  // complete): the miner does this for level L-1 while level L runs, so the
  // event-timestamp reads overlap device work instead of trailing the call.
  void resolve_timed(epi_stats& stats, size_t upto);
  size_t timed_done_ = 0;
  uint64_t stat_epoch_ = 0, prefetched_epoch_ = ~0ull;
  const epi_shard* tshard_ = nullptr;  // active time-segment shard (count_device)
  int64_t force_segments_ = 0;         // count_batch_segments: caller's segment count
  bool bound_only_ = false;            // count_device: chain-end popcount bounds (pass 1)
  uint64_t iota_n_ = 0;                 // size of the level-1 type-id buffer

  cudaEvent_t next_event();
  int new_slot();  // a device u32 log slot, unique within the call
  uint32_t* slot_ptr(int s) { return d_log_ + s; }
  struct Timed {
    cudaEvent_t e0, e_map, e1;
    double* ms_out;
    int live_slot;        // -1: n_host episodes
    uint64_t n_host;
    uint64_t tiles_per_ep;
    bool map;             // automaton launch (map_ms / concat_ms split)
    double* ms_out2 = nullptr;  // a second accumulator of the interval
  };
  struct SlotCounter {
    int slot;
    uint64_t* target;
  };
  std::vector<cudaEvent_t> ev_pool_;
  size_t ev_used_ = 0;
  std::vector<Timed> timed_;
  // ---- per-level CUDA graphs (epi_mine) -----------------------------------
  // A mining level's device work (upload, generation, passes, compaction,
  // statistics prefetch) depends on the host only through the values in its
  // key; the second time a key is seen the enqueue is captured into a graph,
  // from then on the graph is relaunched and the enqueue's host-side
  // bookkeeping replayed. The key includes every buffer generation, so a
  // reallocation invalidates it.
  struct LevelGraph {
    cudaGraphExec_t exec = nullptr;
    bool capturable = true;
    int seen = 0;
    epi_stats delta{};
    uint64_t segments_after = 0;
    bool segments_set = false;
    std::vector<Timed> timed;            // ms pointers stored as offsets into epi_stats
    std::vector<SlotCounter> slots;      // targets stored as offsets into epi_stats
    int log_start = 0, log_end = 0;
    size_t ev_start = 0, ev_end = 0;
  };
  std::vector<std::pair<std::string, LevelGraph>> level_graphs_;
  bool capturing_ = false;
  void rec(cudaEvent_t e);  // event record, external node while capturing
  uint64_t buffers_generation() const;
  // Runs `enqueue` (the level's device work) directly, captured, or as a
  // replayed graph; `stats` is the call's accumulator.
  template <class F>
  void run_level(const std::string& key, bool graphable, epi_stats& stats, F&& enqueue);

  std::vector<SlotCounter> slot_counters_;
  uint32_t* d_log_ = nullptr;            // kLogSlots u32
  unsigned long long* d_acc_ = nullptr;  // [0] patches [1] matched pairs [2] pruned
  int log_used_ = 0;
  static constexpr int kLogSlots = 4096;
  std::vector<std::pair<uint64_t, int>> occ_cache_;  // (launch shape key, CTAs/SM)
  void h2d(void* dst, const void* src, size_t bytes);
  void ensure_type_index();

  // per-type index for tracking (built lazily per loaded stream)
  bool csr_valid_ = false;
  std::vector<uint64_t> csr_off_;
  uint64_t csr_cap_ = 0;
  uint64_t* d_csr_off_ = nullptr;
  int64_t* d_csr_time_ = nullptr;

  int device_;
  int num_sms_ = 148;
  cudaStream_t st_ = nullptr;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr, ev2_ = nullptr;
  DeviceStream stream_;
  DeviceScratch scratch_;
  PinnedBuffer pin_up_, pin_down_, pin_small_;
  PinnedRing ingest_ring_;  // compressed stream uploads (ingest.cu)
  MappedBuffer map_out_, map_small_;

  // epi_mine result storage
  std::vector<uint64_t> m_level_cands_, m_level_off_, m_counts_;
  std::vector<double> m_level_ms_;
  std::vector<uint32_t> m_off_, m_types_;
  std::vector<int64_t> m_lo_, m_hi_;
};

// Apriori join, generate_candidates (E/miner.hpp:76-109).
void generate_candidates(size_t level, const EpisodeSet& frequent,
                         const std::vector<std::pair<int64_t, int64_t>>& alphabet,
                         uint32_t alphabet_size, EpisodeSet& out);

}  // namespace epi
