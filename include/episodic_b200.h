/* episodic_b200 — C-ABI of the B200-native frequent-episode counter.
 *
 * This is the drop-in boundary for the reference's counting hot path
 * (paths relative to /root/reference/proj/include/episodic):
 *   EventStream::from_events  types.hpp:102-119  -> epi_load_stream
 *   build_index               index.hpp:20-30    -> (inside epi_load_stream)
 *   count_fsm                 fsm.hpp:101-106    -> epi_count (one episode)
 *   count_tracking            tracking.hpp:391   -> epi_count (same counts)
 *   count_mapconcat           mapconcat.hpp:71   -> epi_count (same counts)
 *   counting block of mine()  miner.hpp:145-154  -> epi_count (one call/level)
 *   mine()                    miner.hpp:114-173  -> epi_mine
 *   generate()                datagen.hpp:71-122 -> epi_generate
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * Every call returns an epi_status; the message of the last failure is
 * available from epi_last_error(ctx). A C++ adaptor that rethrows the
 * reference's exception types lives in episodic_b200.hpp.
 */
#ifndef EPISODIC_B200_H
#define EPISODIC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  EPI_OK = 0,
  EPI_EINVAL = 1,      /* std::invalid_argument in the reference (validate, mine) */
  EPI_EDATA = 2,       /* episodic::DataError (from_events)                       */
  EPI_EOVERFLOW = 3,   /* std::overflow_error                                     */
  EPI_ECUDA = 4,       /* CUDA runtime failure                                    */
  EPI_ENCCL = 5,       /* NCCL failure (multi-GPU allgather)                      */
  EPI_ENOMEM = 6,      /* device or host allocation failed                        */
  EPI_EUNSUPPORTED = 7 /* input outside what this build's kernels support         */
} epi_status;

typedef struct epi_ctx epi_ctx;

/* Episode batch in CSR form. Episode e has nodes types[offsets[e] ..
 * offsets[e+1]) and N-1 interval constraints (low, high] stored at
 * low/high[offsets[e]-e .. offsets[e+1]-e-1) (one fewer constraint than nodes
 * per episode, so no separate constraint offsets are needed). */
typedef struct {
  uint64_t n_episodes;
  const uint32_t* offsets; /* n_episodes + 1 entries, offsets[0] == 0 */
  const uint32_t* types;
  const int64_t* low;
  const int64_t* high;
} epi_episode_batch;

typedef enum {
  EPI_MODE_EXACT = 0, /* every count exact (count_fsm semantics)                  */
  EPI_MODE_MINE = 1   /* pass 1 relaxed upper bound prunes; survivors exact;
                         pruned entries get EPI_COUNT_PRUNED and frequent = 0   */
} epi_mode;

#define EPI_COUNT_PRUNED UINT64_MAX

typedef struct {
  uint64_t episodes;          /* candidates in the call                        */
  uint64_t pass1_groups;      /* relaxed episodes counted by pass 1            */
  uint64_t pass2_episodes;    /* episodes counted exactly by pass 2            */
  uint64_t pruned;            /* candidates eliminated by pass 1               */
  uint64_t segments;          /* MapConcatenate segments per episode           */
  uint64_t patches;           /* boundary machines re-run by the concat walk   */
  uint64_t kernel_launches;   /* device kernels launched by the call           */
  uint64_t map_launches;      /* segment-map (automaton) kernel launches       */
  uint64_t episode_events;    /* sum over device passes of episodes x events   */
  uint64_t matched_pairs;     /* sum over passes of sum_e sum_k n(type_k)      */
  uint64_t tile_steps;        /* (episode, 32 ms tile) automaton steps, map    */
  uint64_t h2d_bytes;         /* host->device bytes moved by the call          */
  uint64_t d2h_bytes;         /* device->host bytes moved by the call          */
  double pass1_ms, pass2_ms;  /* device time of each pass (CUDA events)        */
  double map_ms;              /* device time of the segment-map kernels        */
  double concat_ms;           /* device time of the concat walks               */
  double total_ms;            /* device time of the whole call                 */
  uint64_t bound_words;       /* pass-1 popcount bound: (candidate, 32 ms tile)
                                 AND-POPC word pairs                            */
  double bound_ms;            /* device time of the pass-1 bound kernels       */
  uint64_t chain_launches;    /* map launches that ran the chain kernel         */
  uint64_t items_tracked;     /* tracking: occurrence intervals found (TrackingStats) */
  uint64_t sort_fallbacks;    /* tracking: episodes whose intervals were not end-sorted,
                                 counted by the exact counter instead (TrackingStats) */
} epi_stats;

/* Context bound to one CUDA device. */
epi_status epi_create(int device, epi_ctx** out);

/* One context over n_gpus devices of this process (SURVEY §8b
 * "epi_create(int n_gpus, ...)", §8e): one engine and one CUDA stream per
 * device, the stream replicated on every device, candidates sharded by
 * episode (few candidates over a long stream: by time segment) with one
 * all-gather of the u64 counts per level, so a single epi_count / epi_mine
 * call uses every device (the reference's one-call ThreadPool spread,
 * E/parallel.hpp:28-125, E/miner.hpp:146-150). devices: n_gpus CUDA ordinals
 * (NULL: 0 .. n_gpus-1). The exchange is NCCL (libnccl.so.2 loaded at run
 * time; ncclCommInitAll over the devices) when every device is distinct and
 * NCCL loads, else device-to-device copies between the ranks' buffers (also
 * what a group with a repeated device - e.g. several ranks on one GPU for
 * testing - uses). epi_load_stream / epi_count / epi_mine run on every rank;
 * the other calls run on the first device. Results and stats come from the
 * first rank (every rank holds the same counts). */
epi_status epi_create_multi(int n_gpus, const int* devices, epi_ctx** out);
/* Ranks of a context (1 for epi_create) and whether its exchange is NCCL. */
uint32_t epi_world(const epi_ctx* ctx);
int epi_uses_nccl(const epi_ctx* ctx);
void epi_destroy(epi_ctx* ctx);
/* Message of the last failure on ctx (or of the calling thread's last
 * context-free call when ctx is NULL). */
const char* epi_last_error(const epi_ctx* ctx);
const char* epi_status_name(epi_status s);

/* Load (replace) the event stream: validated exactly like
 * EventStream::from_events (times >= 0, non-decreasing, type < alphabet;
 * the first offending event decides the message). Host arrays are borrowed
 * for the call; the device copy is owned by the context. */
epi_status epi_load_stream(epi_ctx* ctx, const uint32_t* types, const int64_t* times,
                           uint64_t n, uint32_t alphabet);

/* Same, from arrays already resident on the context's device (for callers
 * that keep the stream in HBM). */
epi_status epi_load_stream_device(epi_ctx* ctx, const uint32_t* d_types, const int64_t* d_times,
                                  uint64_t n, uint32_t alphabet);

uint64_t epi_stream_size(const epi_ctx* ctx);
/* Bytes the last epi_load_stream moved host->device: 12 per event for small
 * streams; large ones (>= 4M events) cross PCIe encoded - narrowed types,
 * per-event time deltas against a base every 2048 events, ~2 B/event on the
 * bench configs - and are widened on the device (ingest.cu). */
uint64_t epi_stream_upload_bytes(const epi_ctx* ctx);

/* Count every episode of the batch over the loaded stream. counts_out has
 * n_episodes entries; frequent_out (optional) receives count >= threshold.
 * stats (optional) receives the pass breakdown. Validation of each episode
 * follows validate(Episode) (types.hpp:87-92). */
epi_status epi_count(epi_ctx* ctx, const epi_episode_batch* batch, uint64_t threshold,
                     uint32_t mode, uint64_t* counts_out, uint8_t* frequent_out,
                     epi_stats* stats);

/* Parallel local tracking (the paper's Alg. 2; tracking.hpp:236-407) on the
 * device, a second exact counter with the reference's interval output.
 * direction: 0 forward (tracking from the first type), 1 backward.
 *   epi_find_occurrences  find_occurrences (tracking.hpp:330-367): the
 *                         intervals of episode e are starts/ends[off[e] ..
 *                         off[e+1]) in the reference's order; the three
 *                         arrays are library-allocated (release with epi_free).
 *   epi_count_tracking    count_tracking (tracking.hpp:391-407): tracking +
 *                         greedy_schedule, equal to count_fsm on every input. */
epi_status epi_find_occurrences(epi_ctx* ctx, const epi_episode_batch* batch, uint32_t direction,
                                uint64_t** offsets_out, int64_t** starts_out, int64_t** ends_out);
epi_status epi_count_tracking(epi_ctx* ctx, const epi_episode_batch* batch, uint32_t direction,
                              uint64_t* counts_out, epi_stats* stats);

/* count_mapconcat (mapconcat.hpp:71-159) with the caller's segment count:
 * exact counts with the MapConcatenate map/concat split into `segments`
 * time segments (clamped to what the stream allows: each segment must span
 * the episodes' sum of highs). stats->segments reports the count used,
 * stats->patches the boundary machines the concat walk re-ran
 * (MapConcatStats: machines_precomputed = segments x episodes, patches). */
epi_status epi_count_mapconcat(epi_ctx* ctx, const epi_episode_batch* batch, uint64_t segments,
                               uint64_t* counts_out, epi_stats* stats);

/* Level-wise mining, mine() (miner.hpp:114-173) with one epi_count call per
 * level. The result is owned by the context until the next epi_mine call:
 *   *n_levels                     levels produced
 *   level_candidates[l]           candidates generated at level l+1
 *   level_offsets[l..l+1]         frequent episodes of level l+1 in the flat
 *                                 result list (candidate-generation order)
 *   res_batch                     the flat frequent episodes (CSR, as above)
 *   res_counts                    their exact counts
 * constraint alphabet: n_alpha bins (alpha_low[i], alpha_high[i]]. */
typedef struct {
  uint64_t threshold;
  uint64_t max_level;
  const int64_t* alpha_low;
  const int64_t* alpha_high;
  uint64_t n_alpha;
  uint32_t mode; /* epi_mode used for levels >= 2 */
} epi_mine_config;

typedef struct {
  uint64_t n_levels;
  const uint64_t* level_candidates;
  const uint64_t* level_offsets;
  const double* level_ms; /* wall time per level (host clock, like LevelResult) */
  epi_episode_batch frequent;
  const uint64_t* counts;
  epi_stats totals;
} epi_mine_result;

epi_status epi_mine(epi_ctx* ctx, const epi_mine_config* cfg, epi_mine_result* out);

/* Episode-sharded mining across ranks (one process and one context per GPU,
 * SURVEY §8e). Every rank generates each level's full candidate list on its
 * own device (the join is deterministic, so the lists agree). A level with
 * at least min_shard candidates is cut into `world` contiguous slices of
 * s = ceil(n / world) candidates; rank r counts slice r only, then calls
 * allgather(user, send, recv, s * 8, stream) with send = its s u64 counts
 * and recv = world * s u64 (both device pointers on the context's device),
 * ordered on the context's CUDA stream `stream` (cudaStream_t). The callback
 * must leave recv = the rank-ordered concatenation of every rank's send
 * (an NCCL all-gather) with the work ordered before anything later enqueued
 * on `stream`, and return 0 (nonzero -> EPI_ENCCL). Thresholding and the next
 * join then run identically on every rank: the result equals epi_mine's on
 * every rank. Smaller levels are counted whole on every rank. */
typedef int (*epi_allgather_fn)(void* user, const void* send_dev, void* recv_dev,
                                uint64_t bytes_per_rank, void* cuda_stream);
typedef struct {
  uint32_t rank;
  uint32_t world;
  uint64_t min_shard; /* levels with fewer candidates are not sharded */
  epi_allgather_fn allgather;
  void* user;
} epi_shard;

epi_status epi_mine_sharded(epi_ctx* ctx, const epi_mine_config* cfg, const epi_shard* shard,
                            epi_mine_result* out);

/* epi_count across ranks (same callback contract as epi_mine_sharded; every
 * rank passes the same batch and receives every count). A batch of at least
 * shard->min_shard episodes is split into `world` contiguous episode slices
 * (counts all-gathered). A smaller batch - few episodes over a long stream -
 * is split by TIME instead: every rank runs the MapConcatenate
 * map step for its own contiguous block of segments, the per-segment records
 * are all-gathered, and every rank runs the concat walk over all segments. */
epi_status epi_count_sharded(epi_ctx* ctx, const epi_episode_batch* batch, uint64_t threshold,
                             uint32_t mode, const epi_shard* shard, uint64_t* counts_out,
                             uint8_t* frequent_out, epi_stats* stats);

/* Synthetic spike-train generator, a bit-exact restatement of generate()
 * (datagen.hpp:71-122): per-neuron homogeneous Poisson background plus
 * injected episodes with uniform gaps, ties ordered by neuron id. The
 * embedded episodes use the batch CSR layout (may be NULL); rates[e] is
 * episode e's injection rate in Hz. *types_out / *times_out are allocated by
 * the library (release with epi_free); *n_out receives the event count.
 * Host-side C++, parallel over neurons. Errors are reported through
 * epi_last_error(NULL). */
epi_status epi_generate(uint32_t neurons, double duration_s, double base_rate_hz, uint64_t seed,
                        const epi_episode_batch* embedded, const double* rates,
                        uint32_t** types_out, int64_t** times_out, uint64_t* n_out);
void epi_free(void* p);

/* generate() bit-exact ON THE DEVICE, straight into the context's stream
 * (as if its arrays were passed to epi_load_stream): one
 * CTA per neuron runs the neuron's mt19937_64 stream and accumulates its
 * spike times in the reference's order, the embedded episodes are generated
 * on the host (few events), one device radix sort merges them. A 1B-event
 * stream takes a fraction of a second instead of host minutes. */
epi_status epi_generate_stream(epi_ctx* ctx, uint32_t neurons, double duration_s, double base_rate_hz,
                               uint64_t seed, const epi_episode_batch* embedded, const double* rates);
/* epi_generate_bursty's MEA-shaped stream (cfg4) generated on the device
 * straight into the context, identical to the host generator's output: the
 * per-electrode rates and the burst schedule are planned on the host, each
 * electrode's background and burst events drawn by one CTA. */
epi_status epi_generate_bursty_stream(epi_ctx* ctx, uint32_t electrodes, double duration_s,
                                      double base_rate_hz, double rate_sigma, double burst_rate_hz,
                                      double burst_min_ms, double burst_max_ms, double burst_gain,
                                      uint64_t seed, const epi_episode_batch* embedded, const double* rates);
/* Copies the loaded stream (epi_stream_size events) to host arrays. */
epi_status epi_stream_download(epi_ctx* ctx, uint32_t* types_out, int64_t* times_out);

/* Event-file ingest, load_stream (io.hpp:22-56) restated multi-threaded:
 * `<name>,<int_ms>` per line, '#' comments and blank lines skipped, CRLF
 * tolerated. Type ids are the names' first-seen order; *names_out receives
 * the names joined by '\n' (id order). Errors are EPI_EDATA with the
 * reference's messages and line numbers. Outputs are library-allocated
 * (epi_free). Feed the arrays to epi_load_stream with *alphabet_out. */
epi_status epi_parse_events(const char* text, uint64_t len, uint32_t** types_out,
                            int64_t** times_out, uint64_t* n_out, char** names_out,
                            uint32_t* alphabet_out);

/* Binary event files (no reference counterpart): the
 * stream's SoA as epi_load_stream takes it — a 24-byte header
 * {"EPIEVT01", u64 n, u32 alphabet, u32 flags = 0}, n u32 types, zero
 * padding to 8 bytes, n i64 times (little endian). epi_write_events writes
 * one (no validation; the load validates), epi_read_events returns the
 * arrays (library-allocated, epi_free), epi_load_stream_file maps the file
 * and uploads from the mapping through the pinned double-buffered H2D of
 * epi_load_stream, with the same validation and messages. File errors are
 * EPI_EDATA ("cannot open event file '<path>'", as load_stream_file,
 * io.hpp:58-61; "not an event file", "truncated event file"). */
epi_status epi_write_events(const char* path, const uint32_t* types, const int64_t* times,
                            uint64_t n, uint32_t alphabet);
epi_status epi_read_events(const char* path, uint32_t** types_out, int64_t** times_out,
                           uint64_t* n_out, uint32_t* alphabet_out);
epi_status epi_load_stream_file(epi_ctx* ctx, const char* path);

/* MEA-culture-shaped bursty generator (no reference
 * counterpart): per-electrode lognormal base rates (base_rate_hz *
 * exp(rate_sigma * N(0,1))), network bursts as a Poisson process at
 * burst_rate_hz lasting uniform [burst_min_ms, burst_max_ms] during which
 * every electrode fires burst_gain times faster, plus embedded episodes as in
 * epi_generate. Deterministic under `seed`; same output conventions. */
epi_status epi_generate_bursty(uint32_t electrodes, double duration_s, double base_rate_hz,
                               double rate_sigma, double burst_rate_hz, double burst_min_ms,
                               double burst_max_ms, double burst_gain, uint64_t seed,
                               const epi_episode_batch* embedded, const double* rates,
                               uint32_t** types_out, int64_t** times_out, uint64_t* n_out);

/* Seeded synthetic candidate episodes for the bench configs (no reference
 * counterpart; the draw order of SURVEY §8d config 3): one std::mt19937_64
 * stream seeded with `seed`; per episode `nodes` types (raw output %
 * alphabet) then nodes-1 constraint-bin indices (raw output % n_bins).
 * types_out holds count*nodes entries, bins_out count*(nodes-1). */
epi_status epi_random_episodes(uint64_t seed, uint64_t count, uint32_t nodes, uint32_t alphabet,
                               uint32_t n_bins, uint32_t* types_out, uint32_t* bins_out);

/* generate_candidates (miner.hpp:76-109) exposed for parity tests and for
 * callers that drive their own level loop: `frequent` holds level-1 frequent
 * episodes (all of length level-1; ignored for level 1). Host-only (no device
 * needed). The output batch is owned by ctx (or, when ctx is NULL, by the
 * calling thread) until the next call. */
epi_status epi_generate_candidates(epi_ctx* ctx, uint64_t level, const epi_episode_batch* frequent,
                                   const int64_t* alpha_low, const int64_t* alpha_high,
                                   uint64_t n_alpha, uint32_t alphabet_size,
                                   epi_episode_batch* out);

/* INT32 issue-rate probe (roofline denominator): lane-ops/s in units of
 * 1e12 on `device`; mixed == 1 saturates both integer pipes (LOP3 + IMAD),
 * mixed == 0 the ALU pipe only (LOP3), mixed == 2 the POPC rate (XU pipe). */
epi_status epi_probe_int32(int device, int mixed, double* tops_out);

/* Build/version string (arch, kernel variants). */
const char* epi_version(void);

#ifdef __cplusplus
}
#endif
#endif
