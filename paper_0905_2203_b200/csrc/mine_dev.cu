// Device-resident level-wise miner: mine() (E/miner.hpp:114-173) with the
// candidate join (generate_candidates, E/miner.hpp:76-109), the two-pass
// elimination and the frequency threshold (E/miner.hpp:159-160) on the GPU.
// Only the small per-level join index (sorted prefix order + per-left bucket
// ranges over the FREQUENT set) goes host->device, and only the frequent
// episodes come back; candidate lists never cross PCIe.
//
// Per level L >= 2:
//   1. generate candidates straight into the counting-kernel parameter layout
//      (types [n*L], packed windows [n*(L-1)], sum of highs [n]);
//   2. pass 1 (MINE mode): radix-sort the packed type sequences, one hull
//      episode per distinct sequence (per position min low, max high), count
//      the hulls exactly -> a sound upper bound per candidate; prune
//      bound < threshold; singleton groups are already exact;
//   3. pass 2: gather the survivors, count them exactly, scatter back;
//   4. flag count >= threshold, compact in candidate order, copy back.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cuda/atomic>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cstddef>
#include <cstdio>
#include <string>
#include <cstdlib>
#include <numeric>

#include "common.cuh"
#include "count_impl.cuh"
#include "engine.h"

namespace epi {
namespace {

constexpr uint64_t kPrunedDev = ~0ull;

enum MineSlot : size_t {
  kMTypes = 10,
  kMWin,
  kMSigma,
  kMCounts,
  kMFreq,      // frequent set of the previous level (types, win, sigma)
  kMJoin,      // pre order + per-left ranges + offsets
  kMKeys,
  kMKeysAlt,
  kMIdx,
  kMIdxAlt,
  kMFlags,
  kMScan,
  kMCub,
  kMGroups,    // relaxed params + group meta
  kMGroupCnt,
  kMSurv,      // survivor params
  kMSurvCnt,
  kMGather,    // all-gathered level counts (sharded mining)
  kMBound,     // pass-1 popcount bounds
  kMLookback,  // tile counter + status words of the single-pass compactions
  kMTileCnt,   // per-tile counts of the two-launch compactions
  kMFreqOut,   // compacted frequent set of a small level (copied back)
  kMIota,      // level-1 candidates: type ids 0..A-1
};

inline size_t align256(size_t x) { return (x + 255) / 256 * 256; }

// EPI_TRACE=1: host timestamps of the mining phases on stderr (diagnostics).
struct HostTrace {
  bool on = std::getenv("EPI_TRACE") != nullptr;
  std::vector<std::pair<const char*, std::chrono::steady_clock::time_point>> pts;
  void mark(const char* what) {
    if (on) pts.emplace_back(what, std::chrono::steady_clock::now());
  }
  void dump() {
    if (!on || pts.empty()) return;
    for (size_t i = 1; i < pts.size(); ++i)
      std::fprintf(stderr, "[epi trace] %-18s %8.1f us\n", pts[i].first,
                   std::chrono::duration<double, std::micro>(pts[i].second - pts[i - 1].second).count());
    pts.clear();
  }
};
thread_local HostTrace g_trace;

__global__ void gen_level2_kernel(const uint32_t* __restrict__ f1, uint32_t nf1,
                                  const uint32_t* __restrict__ awin, const uint32_t* __restrict__ ahi,
                                  uint32_t na, uint32_t* types, uint32_t* win, uint32_t* sigma,
                                  uint64_t n) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t c = static_cast<uint32_t>(i % na);
  const uint64_t lr = i / na;
  const uint32_t r = static_cast<uint32_t>(lr % nf1), l = static_cast<uint32_t>(lr / nf1);
  types[2 * i] = f1[l];
  types[2 * i + 1] = f1[r];
  win[i] = awin[c];
  sigma[i] = ahi[c];
}

// One warp per left: candidates left ++ right.last for every right in the
// left's bucket (rights sorted by prefix key, stable -> frequent order).
__global__ void gen_join_kernel(uint32_t L, const uint32_t* __restrict__ ftypes,
                                const uint32_t* __restrict__ fwin,
                                const uint32_t* __restrict__ fsigma, uint32_t nf,
                                const uint32_t* __restrict__ pre, const uint32_t* __restrict__ lrange,
                                const uint64_t* __restrict__ loff, uint32_t* types, uint32_t* win,
                                uint32_t* sigma) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (warp >= nf) return;
  const uint32_t l = warp;
  const uint32_t F = L - 1, FM = L - 2;
  const uint32_t b0 = lrange[2 * l], b1 = lrange[2 * l + 1];
  const uint64_t o0 = loff[l];
  for (uint32_t b = b0 + lane; b < b1; b += 32) {
    const uint32_t r = pre[b];
    const uint64_t o = o0 + (b - b0);
    uint32_t* t = types + o * L;
    for (uint32_t k = 0; k < F; ++k) t[k] = ftypes[static_cast<size_t>(l) * F + k];
    t[F] = ftypes[static_cast<size_t>(r) * F + F - 1];
    uint32_t* w = win + o * (L - 1);
    for (uint32_t k = 0; k < FM; ++k) w[k] = fwin[static_cast<size_t>(l) * FM + k];
    const uint32_t rw = fwin[static_cast<size_t>(r) * FM + FM - 1];
    w[FM] = rw;
    sigma[o] = fsigma[l] + (rw >> 16);
  }
}

// Constraint alphabet by value (window -> index for the grouping keys).
struct AlphaWin {
  uint32_t w[16];
  uint32_t n;
};

// Grouping key of pass 1: the type sequence, plus (with wbits > 0) the
// alphabet indices of every constraint but the last.
__global__ void pack_keys_kernel(const uint32_t* __restrict__ types, const uint32_t* __restrict__ win,
                                 uint32_t L, uint32_t bits, uint32_t wbits, const AlphaWin aw,
                                 uint64_t n, uint64_t* keys, uint32_t* idx) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t k = 0;
  for (uint32_t j = 0; j < L; ++j) k = (k << bits) | types[i * L + j];
  if (wbits)
    for (uint32_t j = 0; j + 2 < L; ++j) {
      const uint32_t w = win[i * (L - 1) + j];
      uint32_t x = 0;
      for (uint32_t a = 0; a < aw.n; ++a)
        if (aw.w[a] == w) x = a;
      k = (k << wbits) | x;
    }
  keys[i] = k;
  idx[i] = static_cast<uint32_t>(i);
}

__global__ void head_flags_kernel(const uint64_t* __restrict__ keys, uint64_t n, uint32_t* flags) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  flags[j] = (j == 0 || keys[j] != keys[j - 1]) ? 1u : 0u;
}

// scan = exclusive scan of head flags: group of sorted position j is
// scan[j] + flags[j] - 1; group g starts at the j with flags[j] && scan[j] == g.
__global__ void group_starts_kernel(const uint32_t* __restrict__ flags,
                                    const uint32_t* __restrict__ scan, uint64_t n, uint32_t* gstart) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  if (flags[j]) gstart[scan[j]] = static_cast<uint32_t>(j);
}

// One thread per group: the relaxed episode of the group. With last_only the
// group shares every constraint but the last (they are part of its key) and
// only the last one is relaxed; with uniform_win != 0 a relaxed constraint
// becomes that window (the hull of the whole constraint alphabet: contains
// every member's window, so still a sound bound, and launch-uniform, so pass
// 1 runs on width-specialised kernels); otherwise the per-position hull of
// the members' windows.
__global__ void hull_kernel(const uint32_t* __restrict__ types, const uint32_t* __restrict__ win,
                            uint32_t L, const uint32_t* __restrict__ idx_sorted,
                            const uint32_t* __restrict__ gstart, uint32_t n_groups, uint64_t n,
                            uint32_t uniform_win, bool last_only, uint32_t* rtypes, uint32_t* rwin,
                            uint32_t* rsigma, uint32_t* gsize) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  const uint32_t j0 = gstart[g];
  const uint32_t j1 = g + 1 < n_groups ? gstart[g + 1] : static_cast<uint32_t>(n);
  const uint32_t M = L - 1;
  const uint32_t first = idx_sorted[j0];
  for (uint32_t k = 0; k < L; ++k) rtypes[static_cast<size_t>(g) * L + k] = types[static_cast<size_t>(first) * L + k];
  uint32_t sig = 0;
  for (uint32_t k = 0; k < M; ++k) {
    uint32_t lo1 = 0xffffu, hi = 0;
    if (last_only && k + 1 < M) {
      // grouped by these windows too: every member has the first's
      const uint32_t w = win[static_cast<size_t>(first) * M + k];
      lo1 = w & 0xffffu;
      hi = w >> 16;
    } else if (uniform_win) {
      lo1 = uniform_win & 0xffffu;
      hi = uniform_win >> 16;
    } else {
      for (uint32_t j = j0; j < j1; ++j) {
        const uint32_t w = win[static_cast<size_t>(idx_sorted[j]) * M + k];
        lo1 = min(lo1, w & 0xffffu);
        hi = max(hi, w >> 16);
      }
    }
    rwin[static_cast<size_t>(g) * M + k] = lo1 | (hi << 16);
    sig += hi;
  }
  rsigma[g] = sig;
  gsize[g] = j1 - j0;
}

// ---- single-CTA flag / scan / compact ---------------------------------------
// Levels of up to kOneBlkMax candidates compact in ONE launch (one CTA: each
// thread owns a contiguous range, one block scan of the per-thread counts,
// ranges are emitted in index order) instead of flag + two-kernel device scan
// + total + compact: the mining levels are launch-latency bound.
constexpr int kOneBlk = 1024;
constexpr uint64_t kOneBlkMax = 1ull << 14;  // beyond, the multi-CTA path is faster

template <class Pred, class Emit>
__device__ __forceinline__ void one_block_compact(uint64_t n, Pred&& pred, Emit&& emit, uint32_t* total_slot,
                                                  uint32_t* host_total) {
  using BS = cub::BlockScan<uint32_t, kOneBlk>;
  __shared__ typename BS::TempStorage ts;
  uint32_t total = 0;
  if (n <= kOneBlkMax) {
    // small: one contiguous chunk per thread, one scan
    const uint64_t chunk = (n + kOneBlk - 1) / kOneBlk;
    const uint64_t b = min(n, threadIdx.x * chunk), e = min(n, b + chunk);
    uint32_t cnt = 0;
    for (uint64_t i = b; i < e; ++i) cnt += pred(i) ? 1u : 0u;
    uint32_t off = 0;
    BS(ts).ExclusiveSum(cnt, off, total);
    for (uint64_t i = b; i < e; ++i)
      if (pred(i)) emit(i, off++);
  } else {
    // large (a device-sized count beyond the small-launch regime): coalesced
    // rounds of kOneBlk items, one block scan each, running offset
    for (uint64_t base = 0; base < n; base += kOneBlk) {
      const uint64_t i = base + threadIdx.x;
      const bool f = i < n && pred(i);
      uint32_t off = 0, agg = 0;
      BS(ts).ExclusiveSum(f ? 1u : 0u, off, agg);
      if (f) emit(i, total + off);
      total += agg;
      __syncthreads();  // TempStorage reuse
    }
  }
  if (threadIdx.x == 0) {
    *total_slot = total;
    if (host_total) *reinterpret_cast<volatile uint32_t*>(host_total) = total;
  }
}

// ---- single-pass stream compaction (decoupled look-back) --------------------
// Order-preserving flag/scan/compact of any size in ONE launch: tiles of
// kLbTile items taken in launch order (atomic tile counter), each CTA scans
// its tile, publishes its aggregate, looks back over its predecessors'
// published aggregates/prefixes and emits. Replaces flag kernel + two-kernel
// device scan + total + compact kernel (5 launches) on the mining levels.
// state[0] is the tile counter, state[1..] the tile status words (flag in the
// top two bits: 1 aggregate, 2 inclusive prefix); zeroed before each launch.
constexpr int kLbThreads = 256;
constexpr int kLbItems = 8;
constexpr uint64_t kLbTile = static_cast<uint64_t>(kLbThreads) * kLbItems;
constexpr unsigned long long kLbAgg = 1ull << 62, kLbIncl = 2ull << 62, kLbVal = (1ull << 62) - 1;

inline uint64_t lb_tiles(uint64_t n) { return (n + kLbTile - 1) / kLbTile; }

template <class Pred, class Emit>
__device__ __forceinline__ void lookback_compact(uint64_t n, Pred&& pred, Emit&& emit, unsigned long long* state,
                                                 uint32_t* total_slot, uint32_t* host_total) {
  using BS = cub::BlockScan<uint32_t, kLbThreads>;
  __shared__ typename BS::TempStorage ts;
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_excl;
  if (threadIdx.x == 0) s_tile = static_cast<uint32_t>(atomicAdd(state, 1ull));
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = static_cast<uint64_t>(tile) * kLbTile;
  if (base >= n && tile > 0) return;  // grid sized for an upper bound of n
  const uint64_t b = base + static_cast<uint64_t>(threadIdx.x) * kLbItems;
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < kLbItems; ++j)
    if (b + j < n && pred(b + j)) bits |= 1u << j;
  uint32_t off = 0, agg = 0;
  BS(ts).ExclusiveSum(static_cast<uint32_t>(__popc(bits)), off, agg);
  if (threadIdx.x < 32) {
    // warp 0: publish the aggregate, then look back 32 predecessors at a time
    const uint32_t lane = threadIdx.x;
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> me(state[1 + tile]);
    unsigned long long excl = 0;
    if (tile == 0) {
      if (lane == 0) me.store(kLbIncl | agg, cuda::memory_order_release);
    } else {
      if (lane == 0) me.store(kLbAgg | agg, cuda::memory_order_release);
      int64_t top = static_cast<int64_t>(tile) - 1;  // newest predecessor not yet summed
      while (true) {
        const int64_t t = top - lane;  // lane 0 = nearest
        unsigned long long v = kLbIncl;  // before tile 0: an empty inclusive prefix
        if (t >= 0) {
          cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> st(state[1 + t]);
          while (((v = st.load(cuda::memory_order_acquire)) >> 62) == 0) {
          }
        }
        const uint32_t incl = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        // sum lanes up to and including the nearest inclusive prefix
        const uint32_t stop = incl ? __ffs(incl) - 1 : 31;
        unsigned long long x = (lane <= stop && t >= 0) ? (v & kLbVal) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        excl += x;
        if (incl) break;
        top -= 32;
      }
      if (lane == 0) me.store(kLbIncl | (excl + agg), cuda::memory_order_release);
    }
    if (lane == 0) {
      s_excl = excl;
      if (base + kLbTile >= n) {  // the last tile knows the total
        const uint32_t total = static_cast<uint32_t>(excl + agg);
        *total_slot = total;
        if (host_total) *reinterpret_cast<volatile uint32_t*>(host_total) = total;
      }
    }
  }
  __syncthreads();
  uint64_t o = s_excl + off;
#pragma unroll
  for (int j = 0; j < kLbItems; ++j)
    if (bits & (1u << j)) emit(b + j, o++);
}

// Join-mode candidate (global index i): its left (binary search over loff)
// and right.
__device__ __forceinline__ void join_pair(const uint64_t* __restrict__ loff, uint32_t nf,
                                          const uint32_t* __restrict__ pre, const uint32_t* __restrict__ lrange,
                                          uint64_t i, uint32_t& l, uint32_t& r) {
  uint32_t lo = 0, hi = nf;  // largest l with loff[l] <= i
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (loff[mid] <= i) lo = mid; else hi = mid;
  }
  l = lo;
  r = pre[lrange[2 * l] + static_cast<uint32_t>(i - loff[l])];
}

// ---- two-launch ordered compaction (count tiles, then emit) ------------------
// For up to kTcMaxTiles tiles: launch 1 evaluates the predicate (with its side
// effects) and writes one count per tile; launch 2 re-evaluates it (pure),
// sums the counts of the preceding tiles (<= kTcMaxTiles values per CTA, no
// inter-CTA protocol or fences) and emits in index order. Cheaper than the
// look-back's release/acquire chain at mining-level sizes.
constexpr uint64_t kTcMaxTiles = 2048;

template <class Pred>
__device__ __forceinline__ void tile_count(uint64_t n, Pred&& pred, uint32_t* tile_cnt) {
  // (callers with a device-side item count pass it as n; tiles past it count 0)
  using BR = cub::BlockReduce<uint32_t, kLbThreads>;
  __shared__ typename BR::TempStorage ts;
  // a count needs no order: interleaved items keep loads and the
  // predicate's side-effect stores coalesced
  const uint64_t b = static_cast<uint64_t>(blockIdx.x) * kLbTile + threadIdx.x;
  uint32_t cnt = 0;
#pragma unroll
  for (int j = 0; j < kLbItems; ++j) {
    const uint64_t i = b + static_cast<uint64_t>(j) * kLbThreads;
    if (i < n && pred(i)) ++cnt;
  }
  const uint32_t total = BR(ts).Sum(cnt);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = total;
}

template <class Pred, class Emit>
__device__ __forceinline__ void tile_emit(uint64_t n, Pred&& pred, Emit&& emit, const uint32_t* tile_cnt,
                                          uint32_t* total_slot, uint32_t* host_total) {
  using BR = cub::BlockReduce<uint32_t, kLbThreads>;
  using BS = cub::BlockScan<uint32_t, kLbThreads>;
  __shared__ typename BR::TempStorage tr;
  __shared__ typename BS::TempStorage ts;
  __shared__ uint32_t s_excl;
  uint32_t part = 0;
  for (uint32_t t = threadIdx.x; t < blockIdx.x; t += kLbThreads) part += tile_cnt[t];
  const uint32_t excl = BR(tr).Sum(part);
  if (threadIdx.x == 0) s_excl = excl;
  // predicate with coalesced (interleaved) loads into a flag tile, then each
  // thread takes kLbItems contiguous flags (index order for the scan)
  __shared__ uint8_t s_flag[kLbTile];
  const uint64_t tb = static_cast<uint64_t>(blockIdx.x) * kLbTile;
#pragma unroll
  for (int j = 0; j < kLbItems; ++j) {
    const uint32_t t = static_cast<uint32_t>(j) * kLbThreads + threadIdx.x;
    s_flag[t] = (tb + t < n && pred(tb + t)) ? 1 : 0;
  }
  __syncthreads();
  const uint64_t b = tb + static_cast<uint64_t>(threadIdx.x) * kLbItems;
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < kLbItems; ++j)
    if (s_flag[threadIdx.x * kLbItems + j]) bits |= 1u << j;
  uint32_t off = 0, agg = 0;
  BS(ts).ExclusiveSum(static_cast<uint32_t>(__popc(bits)), off, agg);
  __syncthreads();
  const uint32_t e0 = s_excl;
  // the tile holding item n-1 (tile 0 when n == 0) knows the total
  const uint64_t last_tile = n ? (n - 1) / kLbTile : 0;
  if (threadIdx.x == 0 && blockIdx.x == last_tile) {
    *total_slot = e0 + agg;
    if (host_total) *reinterpret_cast<volatile uint32_t*>(host_total) = e0 + agg;
  }
  uint64_t o = static_cast<uint64_t>(e0) + off;
#pragma unroll
  for (int j = 0; j < kLbItems; ++j)
    if (bits & (1u << j)) emit(b + j, o++);
}

__global__ void __launch_bounds__(kLbThreads) freq_count_tc(const uint64_t* __restrict__ counts, uint64_t threshold,
                                                            uint64_t n, uint32_t* tile_cnt) {
  tile_count(
      n,
      [&](uint64_t i) {
        const uint64_t x = counts[i];
        return x != kPrunedDev && x >= threshold;
      },
      tile_cnt);
}

__global__ void __launch_bounds__(kLbThreads) freq_emit_tc(const uint64_t* __restrict__ counts, uint64_t threshold,
                                                           uint64_t n, uint32_t L, const uint32_t* __restrict__ types,
                                                           const uint32_t* __restrict__ win, uint32_t* otypes,
                                                           uint32_t* owin, uint64_t* ocounts,
                                                           const uint32_t* __restrict__ tile_cnt, uint32_t* slot,
                                                           uint32_t* host_k) {
  tile_emit(
      n,
      [&](uint64_t i) {
        const uint64_t x = counts[i];
        return x != kPrunedDev && x >= threshold;
      },
      [&](uint64_t i, uint64_t o) {
        for (uint32_t k = 0; k < L; ++k) otypes[o * L + k] = types[i * L + k];
        for (uint32_t k = 0; k + 1 < L; ++k) owin[o * (L - 1) + k] = win[i * (L - 1) + k];
        ocounts[o] = counts[i];
      },
      tile_cnt, slot, host_k);
}

// Frequent episodes among pass-1 survivors (device-side survivor count
// *m_dev; the grid covers an upper bound): survivors are in candidate order,
// and pruned candidates are never frequent, so this is the level's frequent
// set in candidate order.
__global__ void __launch_bounds__(kLbThreads) surv_count_tc(const uint64_t* __restrict__ counts, uint64_t threshold,
                                                            const uint32_t* __restrict__ m_dev, uint32_t* tile_cnt) {
  tile_count(*m_dev, [&](uint64_t i) { return counts[i] >= threshold; }, tile_cnt);
}

__global__ void __launch_bounds__(kLbThreads) surv_emit_tc(const uint64_t* __restrict__ counts, uint64_t threshold,
                                                           const uint32_t* __restrict__ m_dev, uint32_t L,
                                                           const uint32_t* __restrict__ types,
                                                           const uint32_t* __restrict__ win, uint32_t* otypes,
                                                           uint32_t* owin, uint64_t* ocounts,
                                                           const uint32_t* __restrict__ tile_cnt, uint32_t* slot,
                                                           uint32_t* host_k) {
  tile_emit(
      *m_dev, [&](uint64_t i) { return counts[i] >= threshold; },
      [&](uint64_t i, uint64_t o) {
        for (uint32_t k = 0; k < L; ++k) otypes[o * L + k] = types[i * L + k];
        for (uint32_t k = 0; k + 1 < L; ++k) owin[o * (L - 1) + k] = win[i * (L - 1) + k];
        ocounts[o] = counts[i];
      },
      tile_cnt, slot, host_k);
}

// Same, one CTA: the survivors are few whenever pass 1 pays, and when they
// are many pass 2 on them dwarfs a single-CTA pass over them.
__global__ void __launch_bounds__(kOneBlk) surv_compact_1blk(const uint64_t* __restrict__ counts,
                                                             uint64_t threshold, const uint32_t* __restrict__ m_dev,
                                                             uint32_t L, const uint32_t* __restrict__ types,
                                                             const uint32_t* __restrict__ win, uint32_t* otypes,
                                                             uint32_t* owin, uint64_t* ocounts, uint32_t* slot,
                                                             uint32_t* host_k) {
  one_block_compact(
      *m_dev, [&](uint64_t i) { return counts[i] >= threshold; },
      [&](uint64_t i, uint32_t o) {
        for (uint32_t k = 0; k < L; ++k) otypes[static_cast<size_t>(o) * L + k] = types[i * L + k];
        for (uint32_t k = 0; k + 1 < L; ++k) owin[static_cast<size_t>(o) * (L - 1) + k] = win[i * (L - 1) + k];
        ocounts[o] = counts[i];
      },
      slot, host_k);
}

__global__ void __launch_bounds__(kLbThreads) prune_count_tc(const unsigned long long* __restrict__ bound,
                                                             uint64_t threshold, uint64_t n, uint64_t* counts,
                                                             uint32_t* tile_cnt, unsigned long long* pruned) {
  uint32_t np = 0;
  tile_count(
      n,
      [&](uint64_t i) {
        const bool keep = bound[i] >= threshold;
        counts[i] = keep ? 0 : kPrunedDev;
        np += keep ? 0u : 1u;
        return keep;
      },
      tile_cnt);
  // one atomic per warp (per-thread atomics on one address serialise in L2)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) np += __shfl_xor_sync(0xffffffffu, np, o);
  if ((threadIdx.x & 31) == 0 && np) atomicAdd(pruned, static_cast<unsigned long long>(np));
}

// Join index of a level (join mode of the popcount pass): lefts' types and
// windows, their sums of highs, and the bucket order / ranges / offsets.
struct JoinIdx {
  const uint32_t* ftypes;  // [nf * F]
  const uint32_t* fwin;    // [nf * (F-1)]
  const uint32_t* fsigma;  // [nf]
  const uint32_t* pre;
  const uint32_t* lrange;
  const uint64_t* loff;
  uint32_t nf, F;
};

__global__ void __launch_bounds__(kLbThreads) prune_emit_tc(const unsigned long long* __restrict__ bound,
                                                            uint64_t threshold, uint64_t n, uint32_t L,
                                                            const uint32_t* __restrict__ types,
                                                            const uint32_t* __restrict__ win,
                                                            const uint32_t* __restrict__ sigma, uint32_t* stypes,
                                                            uint32_t* swin, uint32_t* ssigma, uint32_t* sidx,
                                                            const uint32_t* __restrict__ tile_cnt, uint32_t* slot,
                                                            const JoinIdx jx) {
  tile_emit(
      n, [&](uint64_t i) { return bound[i] >= threshold; },
      [&](uint64_t i, uint64_t o) {
        if (jx.pre) {
          // survivor generated from the join index (candidates not materialised)
          uint32_t l, r;
          join_pair(jx.loff, jx.nf, jx.pre, jx.lrange, i, l, r);
          const uint32_t F = jx.F;
          for (uint32_t k = 0; k < F; ++k) stypes[o * L + k] = jx.ftypes[static_cast<size_t>(l) * F + k];
          stypes[o * L + F] = jx.ftypes[static_cast<size_t>(r) * F + F - 1];
          for (uint32_t k = 0; k + 1 < F; ++k) swin[o * (L - 1) + k] = jx.fwin[static_cast<size_t>(l) * (F - 1) + k];
          const uint32_t rw = jx.fwin[static_cast<size_t>(r) * (F - 1) + F - 2];
          swin[o * (L - 1) + F - 1] = rw;
          ssigma[o] = jx.fsigma[l] + (rw >> 16);
        } else {
          for (uint32_t k = 0; k < L; ++k) stypes[o * L + k] = types[i * L + k];
          for (uint32_t k = 0; k + 1 < L; ++k) swin[o * (L - 1) + k] = win[i * (L - 1) + k];
          ssigma[o] = sigma[i];
        }
        sidx[o] = static_cast<uint32_t>(i);
      },
      tile_cnt, slot, nullptr);
}

__global__ void __launch_bounds__(kLbThreads) compact_freq_lb(const uint64_t* __restrict__ counts,
                                                              uint64_t threshold, uint64_t n, uint32_t L,
                                                              const uint32_t* __restrict__ types,
                                                              const uint32_t* __restrict__ win, uint32_t* otypes,
                                                              uint32_t* owin, uint64_t* ocounts,
                                                              unsigned long long* state, uint32_t* slot,
                                                              uint32_t* host_k) {
  lookback_compact(
      n,
      [&](uint64_t i) {
        const uint64_t x = counts[i];
        return x != kPrunedDev && x >= threshold;
      },
      [&](uint64_t i, uint64_t o) {
        for (uint32_t k = 0; k < L; ++k) otypes[o * L + k] = types[i * L + k];
        for (uint32_t k = 0; k + 1 < L; ++k) owin[o * (L - 1) + k] = win[i * (L - 1) + k];
        ocounts[o] = counts[i];
      },
      state, slot, host_k);
}

__global__ void __launch_bounds__(kLbThreads) prune_gather_lb(const unsigned long long* __restrict__ bound,
                                                              uint64_t threshold, uint64_t n, uint32_t L,
                                                              const uint32_t* __restrict__ types,
                                                              const uint32_t* __restrict__ win,
                                                              const uint32_t* __restrict__ sigma,
                                                              uint64_t* counts, uint32_t* stypes, uint32_t* swin,
                                                              uint32_t* ssigma, uint32_t* sidx,
                                                              unsigned long long* state, uint32_t* slot,
                                                              unsigned long long* pruned) {
  uint32_t np = 0;
  lookback_compact(
      n,
      [&](uint64_t i) {
        const bool keep = bound[i] >= threshold;
        counts[i] = keep ? 0 : kPrunedDev;
        np += keep ? 0u : 1u;
        return keep;
      },
      [&](uint64_t i, uint64_t o) {
        for (uint32_t k = 0; k < L; ++k) stypes[o * L + k] = types[i * L + k];
        for (uint32_t k = 0; k + 1 < L; ++k) swin[o * (L - 1) + k] = win[i * (L - 1) + k];
        ssigma[o] = sigma[i];
        sidx[o] = static_cast<uint32_t>(i);
      },
      state, slot, nullptr);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) np += __shfl_xor_sync(0xffffffffu, np, o);
  if ((threadIdx.x & 31) == 0 && np) atomicAdd(pruned, static_cast<unsigned long long>(np));
}

// count >= threshold (never the PRUNED sentinel) -> compacted frequent set
__global__ void __launch_bounds__(kOneBlk) compact_freq_1blk(const uint64_t* __restrict__ counts,
                                                             uint64_t threshold, uint64_t n, uint32_t L,
                                                             const uint32_t* __restrict__ types,
                                                             const uint32_t* __restrict__ win, uint32_t* otypes,
                                                             uint32_t* owin, uint64_t* ocounts, uint32_t* slot,
                                                             uint32_t* host_k) {
  one_block_compact(
      n,
      [&](uint64_t i) {
        const uint64_t x = counts[i];
        return x != kPrunedDev && x >= threshold;
      },
      [&](uint64_t i, uint32_t o) {
        for (uint32_t k = 0; k < L; ++k) otypes[static_cast<size_t>(o) * L + k] = types[i * L + k];
        for (uint32_t k = 0; k + 1 < L; ++k) owin[static_cast<size_t>(o) * (L - 1) + k] = win[i * (L - 1) + k];
        ocounts[o] = counts[i];
      },
      slot, host_k);
}


// ---- pass 1, popcount bound ------------------------------------------------
// U(e)[t] = 1 iff some chain of e (no clears, no pe) ends at time t:
//   U(tau) = occ(tau),  U(e ++ w ++ tau) = occ(tau) & dil_w(U(e)).
// Every completion the exact counter makes is the end of a chain at a
// distinct time, so count(c) <= popcount(U(c)): a sound bound. For a
// candidate c = left ++ w ++ tau, popcount(occ(tau) & dil_w(U(left))) is an
// AND-POPC of two bit rows; the dil_w(U(left)) rows are shared by all of the
// left's candidates (one block per left), and there is no automaton state,
// clear or divergence. On cfg2 level 3 it leaves 11 of 142,228 candidates.
// Needs every high <= 32 (one history word).
// Pass 1 only pays when a level is large: smaller levels (< kMinPass1
// candidates) are cheaper to count exactly than to bound, prune and gather.
// (EPI_PASS1_MIN overrides it: tests run pass 1 on small random levels.)
constexpr uint64_t kMinPass1Default = 16384;
uint64_t min_pass1() {
  const char* s = std::getenv("EPI_PASS1_MIN");
  return s ? static_cast<uint64_t>(std::strtoull(s, nullptr, 10)) : kMinPass1Default;
}
constexpr int kBoundThreads = 256;
constexpr int kBoundMaxL = 16;

struct BoundLaunch {
  const uint32_t* occ;
  uint32_t blk_words;
  int32_t n_tiles;
  uint32_t L;                      // candidate length (lefts have L-1 nodes)
  const uint32_t* ltypes;          // [nf * (L-1)]
  const uint32_t* lwin;            // [nf * (L-2)]
  const uint64_t* loff;            // [nf + 1] candidates of left l (or null: l * stride)
  uint64_t stride;
  const uint32_t* ctypes;          // [n * L]
  const uint32_t* cwin;            // [n * (L-1)]
  AlphaWin aw;
  int32_t span;                    // tiles per blockIdx.y split (multiple of kBoundThreads)
  uint32_t uniform_w;              // every alphabet window has width high-low == uniform_w (0: mixed)
  uint32_t sm[5];                  // doubling-smear shifts covering uniform_w
  uint32_t n_sm;                   // steps used
  uint64_t slice_lo, slice_hi;     // candidates counted here (episode shard)
  unsigned long long* bound;       // [slice_hi - slice_lo], zeroed unless direct
  bool direct;                     // one time split: every candidate stored once
  // join mode (jpre != null, level >= 3, unsharded): candidates are not
  // materialised; candidate loff[l] + j of left l is left ++ right
  // jpre[jlrange[2l] + j] (the join index gen_join_kernel would expand)
  const uint32_t* jpre;
  const uint32_t* jlrange;
};



__device__ __forceinline__ uint32_t dil_rt(uint32_t w, uint32_t h, uint32_t c) {
  return impl::window_any<0, true>(c, h, 0u, w & 0xffffu, w >> 16);
}

// Equal-width alphabets (every window high - low == W): S = OR_{b<W} X >> b
// over X = (c : h) once (64-bit doubling smear, shifts p.sm[]), then each
// window [lo+1, hi] is one funnel shift of S by 32 - hi.
struct Smear64 {
  uint32_t lo, hi;
};
__device__ __forceinline__ Smear64 smear64(uint32_t h, uint32_t c, const uint32_t (&sh)[5], uint32_t steps) {
  uint32_t rl = h, rh = c;
  for (uint32_t i = 0; i < steps; ++i) {
    rl |= __funnelshift_r(rl, rh, sh[i]);
    rh |= rh >> sh[i];
  }
  return {rl, rh};
}
__device__ __forceinline__ uint32_t window_of(const Smear64& s, uint32_t w) {
  return __funnelshift_r(s.lo, s.hi, 32u - (w >> 16));
}

// One block per (left, time split). Per chunk of 256 tiles: phase A, one
// thread per tile, rebuilds U(left) from the type bitmaps (no state carried
// across tiles, so any split is exact) and writes dil_w(U(left)) for every
// alphabet window to shared memory; phase B, lane = tile (coalesced bitmap
// rows), each warp accumulates AND-POPC sums for up to kBoundPerWarp of the
// left's candidates in registers; one warp reduction per candidate at the end.
constexpr int kBoundPerWarp = 16;
constexpr int kBoundRound = kBoundPerWarp * (kBoundThreads / 32);

// kF > 0: left length known at compile time (mining levels 2..7: U chain in
// registers, loops unrolled); kF == 0: runtime length up to kBoundMaxL - 1.
template <int kF>
__global__ void __launch_bounds__(kBoundThreads) bound_kernel(const BoundLaunch p) {
  __shared__ uint32_t D[16][kBoundThreads];
  // per round: the candidates' last type row offset and D row offset, the
  // runs of equal last type (the join emits a left's candidates grouped so),
  // and per-candidate per-lane partial sums
  __shared__ uint32_t s_row[kBoundRound], s_drow[kBoundRound];
  __shared__ uint32_t s_run[kBoundRound + 1];
  __shared__ uint32_t s_nrun;
  __shared__ uint32_t s_acc[kBoundRound][32];
  __shared__ uint32_t s_x[kBoundThreads];               // phase A neighbour exchange
  __shared__ uint32_t s_carry[kF > 0 ? kF : 1];         // U_k at the tile before the chunk
  for (uint32_t x = threadIdx.x; x < kBoundRound * 32; x += kBoundThreads) (&s_acc[0][0])[x] = 0;
  const uint32_t l = blockIdx.x;
  const uint64_t c0 = max(p.loff ? p.loff[l] : l * p.stride, p.slice_lo);
  const uint64_t c1 = min(p.loff ? p.loff[l + 1] : (l + 1) * p.stride, p.slice_hi);
  if (c1 <= c0) return;
  const uint32_t m = static_cast<uint32_t>(c1 - c0);
  const uint32_t F = kF > 0 ? static_cast<uint32_t>(kF) : p.L - 1;  // left length
  const int32_t g_lo = static_cast<int32_t>(blockIdx.y) * p.span;
  const int32_t g_hi = min(g_lo + p.span, p.n_tiles);
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr uint32_t kWarps = kBoundThreads / 32;
  for (uint32_t r0 = 0; r0 < m; r0 += kBoundRound) {
    const uint32_t mr = min(m - r0, static_cast<uint32_t>(kBoundRound));
    __syncthreads();  // previous round's table reads are done
    uint32_t my_tau = ~0u;
    for (uint32_t j = tid; j < mr; j += kBoundThreads) {
      const uint64_t cc = c0 + r0 + j;
      uint32_t w;
      if (p.jpre) {
        // candidate = this left ++ right's last node and last constraint
        const uint32_t rr = p.jpre[p.jlrange[2 * l] + static_cast<uint32_t>(cc - p.loff[l])];
        my_tau = p.ltypes[static_cast<size_t>(rr) * F + F - 1];
        w = p.lwin[static_cast<size_t>(rr) * (F - 1) + F - 2];
      } else {
        my_tau = p.ctypes[cc * p.L + p.L - 1];
        w = p.cwin[cc * (p.L - 1) + p.L - 2];
      }
      uint32_t x = 0;
      for (uint32_t a = 0; a < p.aw.n; ++a)
        if (p.aw.w[a] == w) x = a;
      s_row[j] = my_tau * kRowStride;
      s_drow[j] = x * kBoundThreads;
    }
    __syncthreads();
    if (warp == 0) {
      // run starts: j == 0 or a different last type than j - 1 (ballots over
      // the round's <= kBoundRound candidates, in order)
      uint32_t nrun = 0;
      for (uint32_t j0 = 0; j0 < mr; j0 += 32) {
        const uint32_t j = j0 + lane;
        const bool start = j < mr && (j == 0 || s_row[j] != s_row[j - 1]);
        const uint32_t bal = __ballot_sync(0xffffffffu, start);
        if (start) s_run[nrun + __popc(bal & ((1u << lane) - 1))] = j;
        nrun += __popc(bal);
      }
      if (lane == 0) {
        s_run[nrun] = mr;
        s_nrun = nrun;
      }
    }
    __syncthreads();
    const uint32_t nrun = s_nrun;
    for (int32_t gc = g_lo; gc < g_hi; gc += kBoundThreads) {
      // Phase A: dil_w(U(left)) for tile g = gc + tid, every alphabet window w
      if constexpr (kF > 0) {
        // one chain level at a time: thread = tile, U_{k-1} of the previous
        // tile from the neighbour thread (shared memory), thread 0's from
        // the previous chunk (s_carry) or, at a split start, rebuilt
        const int32_t g = gc + static_cast<int32_t>(tid);
        const bool in = g < p.n_tiles;
        const size_t wbase = static_cast<size_t>(g >> 5) * p.blk_words + (g & 31);
        if (tid == 0 && gc == g_lo) {
          // U_k at tile g_lo - 1, k < F: the triangle over tiles g_lo-F .. g_lo-1
          uint32_t u[kF];
          auto occ_at = [&](uint32_t t, int32_t gj) -> uint32_t {
            return (gj >= 0 && gj < p.n_tiles) ? __ldg(p.occ + impl::occ_index(gj, t, p.blk_words)) : 0u;
          };
          const uint32_t t0 = p.ltypes[static_cast<size_t>(l) * F];
#pragma unroll
          for (int j = 0; j < kF; ++j) u[j] = occ_at(t0, g_lo - kF + j);
          s_carry[0] = u[kF - 1];
#pragma unroll
          for (int k = 1; k < kF; ++k) {
            const uint32_t tk = p.ltypes[static_cast<size_t>(l) * F + k];
            const uint32_t wk = p.lwin[static_cast<size_t>(l) * (F - 1) + k - 1];
#pragma unroll
            for (int j = kF - 1; j >= k; --j)
              u[j] = occ_at(tk, g_lo - kF + j) &
                     (p.uniform_w ? window_of(smear64(u[j - 1], u[j], p.sm, p.n_sm), wk) : dil_rt(wk, u[j - 1], u[j]));
            s_carry[k] = u[kF - 1];
          }
        }
        uint32_t u = in ? __ldg(p.occ + wbase + p.ltypes[static_cast<size_t>(l) * F] * kRowStride) : 0u;
#pragma unroll
        for (int k = 1; k <= kF; ++k) {
          s_x[tid] = u;
          __syncthreads();
          const uint32_t prev = tid ? s_x[tid - 1] : s_carry[k - 1];
          __syncthreads();
          if (tid == kBoundThreads - 1) s_carry[k - 1] = u;  // the next chunk's thread 0
          if (k < kF) {
            const uint32_t tk = p.ltypes[static_cast<size_t>(l) * F + k];
            const uint32_t wk = p.lwin[static_cast<size_t>(l) * (F - 1) + k - 1];
            const uint32_t o = in ? __ldg(p.occ + wbase + tk * kRowStride) : 0u;
            u = o & (p.uniform_w ? window_of(smear64(prev, u, p.sm, p.n_sm), wk) : dil_rt(wk, prev, u));
          } else {
            // U(left) at tiles g-1 (prev) and g (u); zero past the split
            const bool live = g < g_hi;
            if (p.uniform_w) {
              const Smear64 sm = smear64(prev, u, p.sm, p.n_sm);
              for (uint32_t a = 0; a < p.aw.n; ++a) D[a][tid] = live ? window_of(sm, p.aw.w[a]) : 0u;
            } else {
              for (uint32_t a = 0; a < p.aw.n; ++a) D[a][tid] = live ? dil_rt(p.aw.w[a], prev, u) : 0u;
            }
          }
        }
      } else {
        const int32_t g = gc + static_cast<int32_t>(tid);
        constexpr int kU = kBoundMaxL;
        uint32_t u[kU];  // u[j] = U at tile g - F + j, j = 0..F
        const uint32_t t0 = p.ltypes[static_cast<size_t>(l) * F];
        // word of type t at tile g - F + j (zero outside the stream)
        auto occ_at = [&](uint32_t t, uint32_t j) -> uint32_t {
          const int32_t gj = g - static_cast<int32_t>(F) + static_cast<int32_t>(j);
          return (gj >= 0 && gj < p.n_tiles) ? __ldg(p.occ + impl::occ_index(gj, t, p.blk_words)) : 0u;
        };
#pragma unroll
        for (uint32_t j = 0; j < static_cast<uint32_t>(kU); ++j)
          if (kF > 0 || j <= F) u[j] = occ_at(t0, j);
#pragma unroll
        for (uint32_t k = 1; k < static_cast<uint32_t>(kU) - 1; ++k) {
          if (kF == 0 && k >= F) break;
          const uint32_t tk = p.ltypes[static_cast<size_t>(l) * F + k];
          const uint32_t wk = p.lwin[static_cast<size_t>(l) * (F - 1) + k - 1];
#pragma unroll
          for (uint32_t j = static_cast<uint32_t>(kU) - 1; j >= k; --j) {
            if (kF > 0 || j <= F)
              u[j] = occ_at(tk, j) &
                     (p.uniform_w ? window_of(smear64(u[j - 1], u[j], p.sm, p.n_sm), wk) : dil_rt(wk, u[j - 1], u[j]));
          }
        }
        // U(left) at tiles g-1 (u[F-1]) and g (u[F])
        // (zero past the split: phase B then reads whole bitmap blocks)
        const bool live = g < g_hi;
        if (p.uniform_w) {
          const Smear64 s = smear64(u[F - 1], u[F], p.sm, p.n_sm);
          for (uint32_t a = 0; a < p.aw.n; ++a) D[a][tid] = live ? window_of(s, p.aw.w[a]) : 0u;
        } else {
          for (uint32_t a = 0; a < p.aw.n; ++a) D[a][tid] = live ? dil_rt(p.aw.w[a], u[F - 1], u[F]) : 0u;
        }
      }
      __syncthreads();
      // Phase B: lane = 4 consecutive tiles (16-byte row loads): lanes 8q..8q+7
      // cover bitmap block q of each group of 4 blocks; D is zero past the
      // split. Per-lane partial sums stay in shared memory (no reduction in
      // the loop).
      const int32_t nk = (min(kBoundThreads, g_hi - gc) + 31) >> 5;  // blocks in chunk
      const uint32_t bw = p.blk_words;
      const uint32_t q = lane >> 3, sub = (lane & 7) * 4;
      const uint32_t* blk0 = p.occ + static_cast<size_t>((gc >> 5) + q) * bw + sub;
      const uint32_t* dbase = &D[0][q * 32 + sub];
      // a warp takes a run: its last type's rows are loaded once, then every
      // candidate of the run (one per alphabet window) ANDs and counts them
      for (uint32_t r = warp; r < nrun; r += kWarps) {
        const uint32_t j0 = s_run[r], j1 = s_run[r + 1];
        const uint32_t* row = blk0 + s_row[j0];
        uint4 o[kBoundThreads / 128];
#pragma unroll
        for (int m = 0; m < kBoundThreads / 128; ++m)
          o[m] = static_cast<int32_t>(q) + 4 * m < nk
                     ? __ldg(reinterpret_cast<const uint4*>(row + 4 * m * bw))
                     : make_uint4(0, 0, 0, 0);
        for (uint32_t j = j0; j < j1; ++j) {
          const uint32_t* drow = dbase + s_drow[j];
          uint32_t a = 0;
#pragma unroll
          for (int m = 0; m < kBoundThreads / 128; ++m) {
            const uint4 d = *reinterpret_cast<const uint4*>(drow + 128 * m);
            a += __popc(o[m].x & d.x) + __popc(o[m].y & d.y) + __popc(o[m].z & d.z) + __popc(o[m].w & d.w);
          }
          s_acc[j][lane] += a;
        }
      }
      __syncthreads();
    }
    // per candidate: sum the 32 lanes' partials (warp per candidate)
    for (uint32_t j = warp; j < mr; j += kWarps) {
      uint32_t v = s_acc[j][lane];
      s_acc[j][lane] = 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) {
        unsigned long long* dst = p.bound + (c0 - p.slice_lo) + r0 + j;
        if (p.direct)
          *dst = v;
        else if (v)
          atomicAdd(dst, static_cast<unsigned long long>(v));
      }
    }
  }
}


// Per sorted position: bound < threshold prunes, the rest survive to pass 2
// (singleton groups are final when their relaxation is the episode itself).
__global__ void prune_kernel(const uint32_t* __restrict__ idx_sorted, const uint32_t* __restrict__ flags,
                             const uint32_t* __restrict__ scan, const uint32_t* __restrict__ gsize,
                             const uint64_t* __restrict__ bound, uint64_t threshold, uint64_t n,
                             bool singletons_exact, uint64_t* counts, uint32_t* surv,
                             unsigned long long* pruned) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  bool pr = false;
  if (j < n) {
    const uint32_t i = idx_sorted[j];
    const uint32_t g = scan[j] + flags[j] - 1;
    uint32_t s = 0;
    if (singletons_exact && gsize[g] == 1) {
      counts[i] = bound[g];
    } else if (bound[g] < threshold) {
      counts[i] = kPrunedDev;
      pr = true;
    } else {
      counts[i] = 0;
      s = 1;
    }
    surv[i] = s;
  }
  // one atomic per warp
  const uint32_t bal = __ballot_sync(0xffffffffu, pr);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(pruned, static_cast<unsigned long long>(__popc(bal)));
}

__global__ void gather_kernel(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ scan,
                              uint64_t n, uint32_t L, const uint32_t* __restrict__ types,
                              const uint32_t* __restrict__ win, const uint32_t* __restrict__ sigma,
                              uint32_t* otypes, uint32_t* owin, uint32_t* osigma, uint32_t* oidx) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || !flags[i]) return;
  const uint32_t o = scan[i];
  for (uint32_t k = 0; k < L; ++k) otypes[static_cast<size_t>(o) * L + k] = types[i * L + k];
  for (uint32_t k = 0; k + 1 < L; ++k) owin[static_cast<size_t>(o) * (L - 1) + k] = win[i * (L - 1) + k];
  osigma[o] = sigma[i];
  oidx[o] = static_cast<uint32_t>(i);
}

__global__ void scatter_counts_kernel(const uint32_t* __restrict__ oidx, const uint64_t* __restrict__ c,
                                      const uint32_t* __restrict__ m_dev, uint64_t* counts) {
  const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o < *m_dev) counts[oidx[o]] = c[o];
}

// total of an exclusive scan = scan[n-1] + flags[n-1] -> device log slot
// (and a zero-copy host word when given)
__global__ void scan_total_kernel(const uint32_t* __restrict__ scan, const uint32_t* __restrict__ flags,
                                  uint64_t n, uint32_t* slot, uint32_t* host) {
  const uint32_t t = scan[n - 1] + flags[n - 1];
  *slot = t;
  if (host) *reinterpret_cast<volatile uint32_t*>(host) = t;
}

__global__ void freq_flags_kernel(const uint64_t* __restrict__ counts, uint64_t threshold, uint64_t n,
                                  uint32_t* flags) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t c = counts[i];
  flags[i] = (c != kPrunedDev && c >= threshold) ? 1u : 0u;
}

__global__ void compact_freq_kernel(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ scan,
                                    uint64_t n, uint32_t L, const uint32_t* __restrict__ types,
                                    const uint32_t* __restrict__ win, const uint64_t* __restrict__ counts,
                                    uint32_t* otypes, uint32_t* owin, uint64_t* ocounts) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || !flags[i]) return;
  const uint32_t o = scan[i];
  for (uint32_t k = 0; k < L; ++k) otypes[static_cast<size_t>(o) * L + k] = types[i * L + k];
  for (uint32_t k = 0; k + 1 < L; ++k) owin[static_cast<size_t>(o) * (L - 1) + k] = win[i * (L - 1) + k];
  ocounts[o] = counts[i];
}

inline unsigned blocks_for(uint64_t n, unsigned t = 256) {
  return static_cast<unsigned>((n + t - 1) / t);
}

}  // namespace

// Exclusive scan of n u32 flags into scan[]; the total lands in device log
// slot `slot` (and in *host_total, zero-copy). No host synchronisation.
void Engine::dev_scan_total(const uint32_t* flags, uint32_t* scan, uint64_t n, int slot,
                            uint32_t* host_total) {
  size_t tmp = 0;
  EPI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flags, scan, static_cast<int>(n), st_));
  void* d_tmp = scratch_.get<char>(kMCub, tmp + 16);
  EPI_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp, flags, scan, static_cast<int>(n), st_));
  scan_total_kernel<<<1, 1, 0, st_>>>(scan, flags, n, slot_ptr(slot), host_total);
  EPI_CUDA(cudaGetLastError());
}

// Counts of the device-resident candidate set `c` into d_counts: exact, or
// two-pass (MINE) with PRUNED sentinels for eliminated candidates. One host
// synchronisation (the group count decides whether pass 1 pays); survivors
// are sized on the device.
void Engine::count_device_two_pass(const DevSet& c, uint64_t threshold, uint32_t mode,
                                   uint32_t uniform_win, const uint32_t* alpha, uint32_t n_alpha,
                                   uint64_t* d_counts, epi_stats& stats) {
  const uint64_t n = c.n;
  const uint32_t L = c.N;
  stats.episodes += n;
  uint32_t bits = 1;
  while ((1ull << bits) < stream_.alphabet + 1ull) ++bits;
  const bool grouping = mode == EPI_MODE_MINE && threshold > 1 && L >= 2 && bits * L <= 64 &&
                        n >= min_pass1() && n < (1ull << 31);
  if (!grouping) {
    stats.pass2_episodes += n;
    count_device(c, d_counts, stats, &stats.pass2_ms);
    return;
  }
  const uint32_t M = L - 1;
  // Relaxation: only the last constraint, to the alphabet hull, grouping by
  // types + the other constraints (tight bounds: on cfg2 level 3 it leaves
  // 51 of 142,228 candidates for pass 2, against 126,512 when every
  // constraint is relaxed); the types-only grouping with every constraint
  // relaxed when the key does not fit 64 bits or the alphabet is large.
  AlphaWin aw{};
  uint32_t wbits = 0;
  if (L >= 3 && uniform_win && n_alpha <= 16) {
    wbits = 1;
    while ((1u << wbits) < n_alpha) ++wbits;
    if (bits * L + wbits * (L - 2) > 64) wbits = 0;
    for (uint32_t a = 0; a < n_alpha; ++a) aw.w[a] = alpha[a];
    aw.n = n_alpha;
  }
  const bool last_only = wbits > 0;
  const uint32_t key_bits = bits * L + wbits * (L >= 2 ? L - 2 : 0);
  uint64_t* keys = scratch_.get<uint64_t>(kMKeys, n);
  uint64_t* keys_alt = scratch_.get<uint64_t>(kMKeysAlt, n);
  uint32_t* idx = scratch_.get<uint32_t>(kMIdx, n);
  uint32_t* idx_alt = scratch_.get<uint32_t>(kMIdxAlt, n);
  pack_keys_kernel<<<blocks_for(n), 256, 0, st_>>>(c.types, c.win, L, bits, wbits, aw, n, keys, idx);
  EPI_CUDA(cudaGetLastError());
  cub::DoubleBuffer<uint64_t> kb(keys, keys_alt);
  cub::DoubleBuffer<uint32_t> vb(idx, idx_alt);
  size_t tmp = 0;
  EPI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, static_cast<int>(n), 0,
                                           static_cast<int>(key_bits), st_));
  void* d_tmp = scratch_.get<char>(kMCub, tmp + 16);
  EPI_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, kb, vb, static_cast<int>(n), 0,
                                           static_cast<int>(key_bits), st_));
  const uint64_t* skeys = kb.Current();
  const uint32_t* sidx = vb.Current();
  uint32_t* flags = scratch_.get<uint32_t>(kMFlags, n);
  uint32_t* scan = scratch_.get<uint32_t>(kMScan, n);
  head_flags_kernel<<<blocks_for(n), 256, 0, st_>>>(skeys, n, flags);
  EPI_CUDA(cudaGetLastError());
  map_small_.get(64);
  uint32_t* h_groups = static_cast<uint32_t*>(map_small_.p);
  dev_scan_total(flags, scan, n, new_slot(), h_groups);
  g_trace.mark("p1 sort launched");
  EPI_CUDA(cudaStreamSynchronize(st_));
  g_trace.mark("p1 groups synced");
  const uint32_t n_groups = *reinterpret_cast<volatile uint32_t*>(h_groups);
  stats.kernel_launches += 5;
  if (2ull * n_groups > n) {
    // type sequences barely repeat: relaxed counts would cost as much as
    // the exact ones, so count everything exactly
    stats.pass2_episodes += n;
    count_device(c, d_counts, stats, &stats.pass2_ms);
    return;
  }

  // group metadata + relaxed (hull) episodes
  const size_t g_types = 0, g_win = align256(static_cast<size_t>(n_groups) * L * 4),
               g_sigma = g_win + align256(static_cast<size_t>(n_groups) * M * 4),
               g_start = g_sigma + align256(n_groups * 4ull), g_size = g_start + align256(n_groups * 4ull),
               g_total = g_size + align256(n_groups * 4ull);
  char* gbuf = scratch_.get<char>(kMGroups, g_total);
  uint32_t* rtypes = reinterpret_cast<uint32_t*>(gbuf + g_types);
  uint32_t* rwin = reinterpret_cast<uint32_t*>(gbuf + g_win);
  uint32_t* rsigma = reinterpret_cast<uint32_t*>(gbuf + g_sigma);
  uint32_t* gstart = reinterpret_cast<uint32_t*>(gbuf + g_start);
  uint32_t* gsize = reinterpret_cast<uint32_t*>(gbuf + g_size);
  group_starts_kernel<<<blocks_for(n), 256, 0, st_>>>(flags, scan, n, gstart);
  hull_kernel<<<blocks_for(n_groups), 256, 0, st_>>>(c.types, c.win, L, sidx, gstart, n_groups, n,
                                                     uniform_win, last_only, rtypes, rwin, rsigma,
                                                     gsize);
  EPI_CUDA(cudaGetLastError());
  stats.kernel_launches += 2;
  DevSet rel = c;
  rel.n = n_groups;
  rel.types = rtypes;
  rel.win = rwin;
  rel.sigma = rsigma;
  // per-group hull widths differ in general; the alphabet hull is uniform
  const int hull_w = uniform_win ? static_cast<int>((uniform_win >> 16) - (uniform_win & 0xffffu) + 1) : 0;
  if (last_only) {
    rel.width = c.width;  // the kept constraints
    rel.last_w = static_cast<uint32_t>(hull_w);
  } else {
    rel.width = hull_w;
  }
  if (uniform_win) rel.max_sigma = (uniform_win >> 16) * (L - 1);
  uint64_t* bound = scratch_.get<uint64_t>(kMGroupCnt, n_groups);
  stats.pass1_groups += n_groups;
  count_device(rel, bound, stats, &stats.pass1_ms);

  // Survivor flags go to the index buffer the sort left free.
  uint32_t* sflags = sidx == idx ? idx_alt : idx;
  // A singleton group's per-group hull is the episode itself (exact); the
  // uniform alphabet hull is only a bound.
  prune_kernel<<<blocks_for(n), 256, 0, st_>>>(sidx, flags, scan, gsize, bound, threshold, n,
                                               uniform_win == 0, d_counts, sflags, d_acc_ + 2);
  EPI_CUDA(cudaGetLastError());
  uint32_t* sscan = scan;
  const int mslot = new_slot();
  dev_scan_total(sflags, sscan, n, mslot);
  slot_counters_.push_back({mslot, &stats.pass2_episodes});
  stats.kernel_launches += 4;
  // Survivors (m <= n, known only on the device): buffers and grids sized
  // for n, kernels read m from the log slot.
  const size_t s_types = 0, s_win = align256(static_cast<size_t>(n) * L * 4),
               s_sigma = s_win + align256(static_cast<size_t>(n) * M * 4),
               s_idx = s_sigma + align256(n * 4ull), s_total = s_idx + align256(n * 4ull);
  char* sbuf = scratch_.get<char>(kMSurv, s_total);
  uint32_t* stypes = reinterpret_cast<uint32_t*>(sbuf + s_types);
  uint32_t* swin = reinterpret_cast<uint32_t*>(sbuf + s_win);
  uint32_t* ssigma = reinterpret_cast<uint32_t*>(sbuf + s_sigma);
  uint32_t* sidx_out = reinterpret_cast<uint32_t*>(sbuf + s_idx);
  gather_kernel<<<blocks_for(n), 256, 0, st_>>>(sflags, sscan, n, L, c.types, c.win, c.sigma, stypes,
                                                swin, ssigma, sidx_out);
  EPI_CUDA(cudaGetLastError());
  DevSet sv = c;
  sv.n = n;
  sv.types = stypes;
  sv.win = swin;
  sv.sigma = ssigma;
  uint64_t* sc = scratch_.get<uint64_t>(kMSurvCnt, n);
  count_device(sv, sc, stats, &stats.pass2_ms, mslot);
  scatter_counts_kernel<<<blocks_for(n), 256, 0, st_>>>(sidx_out, sc, slot_ptr(mslot), d_counts);
  EPI_CUDA(cudaGetLastError());
  stats.kernel_launches += 2;
}

// Pass 1 by the popcount bound (bound_kernel) over the left-grouped
// candidates of one mining level, then pass 2 on the survivors. The host does
// not wait: survivors are sized on the device.
void Engine::count_device_popbound(const DevSet& c, const PopLefts& lf, uint64_t threshold,
                                   const uint32_t* alpha, uint32_t n_alpha, uint64_t* d_counts,
                                   epi_stats& stats, Survivors* surv) {
  const uint64_t n = c.n;
  const uint32_t L = c.N, M = L - 1;
  stats.episodes += n;
  stats.pass1_groups += n;
  unsigned long long* bound = scratch_.get<unsigned long long>(kMBound, n);
  BoundLaunch b{};
  b.occ = stream_.d_occ;
  b.blk_words = stream_.blk_words;
  b.n_tiles = static_cast<int32_t>(stream_.n_tiles);
  b.L = L;
  b.ltypes = lf.types;
  b.lwin = lf.win;
  b.loff = lf.off;
  b.stride = lf.stride;
  b.ctypes = c.types - lf.slice_lo * L;  // the kernel indexes candidates globally
  b.cwin = c.win - lf.slice_lo * M;
  for (uint32_t a = 0; a < n_alpha; ++a) b.aw.w[a] = alpha[a];
  b.aw.n = n_alpha;
  b.slice_lo = lf.slice_lo;
  b.slice_hi = lf.slice_lo + n;
  if (lf.join_mode) {
    if (lb_tiles(n) > kTcMaxTiles || lf.slice_lo != 0)
      throw Error(EPI_EUNSUPPORTED, "join-mode pass 1 needs an unsharded level of <= 4M candidates");
    b.jpre = lf.pre;
    b.jlrange = lf.lrange;
  }
  // equal-width alphabet: one shared smear per tile instead of one per window
  uint32_t uw = n_alpha ? (alpha[0] >> 16) - (alpha[0] & 0xffffu) + 1 : 0;
  for (uint32_t a = 0; a < n_alpha; ++a)
    if ((alpha[a] >> 16) - (alpha[a] & 0xffffu) + 1 != uw) uw = 0;
  b.uniform_w = uw;
  {
    uint32_t cover = 1;
    b.n_sm = 0;
    for (int i = 0; i < 5; ++i) {
      const uint32_t s = cover < uw ? std::min(cover, uw - cover) : 0u;
      b.sm[i] = s;
      cover += s;
      if (s) b.n_sm = static_cast<uint32_t>(i + 1);
    }
  }
  b.bound = bound;
  // split time so that lefts x splits fill the GPU a few times over
  const int64_t chunks = (static_cast<int64_t>(stream_.n_tiles) + kBoundThreads - 1) / kBoundThreads;
  const int64_t want = std::max<int64_t>(1, (static_cast<int64_t>(num_sms_) * 8 + lf.nf - 1) / lf.nf);
  // (<= 2^26 tiles per split keeps the u32 per-lane sums exact)
  const int64_t splits = std::clamp<int64_t>(std::max<int64_t>(want, (stream_.n_tiles >> 26) + 1), 1,
                                             std::max<int64_t>(chunks, 1));
  b.span = static_cast<int32_t>((chunks + splits - 1) / splits * kBoundThreads);
  const int64_t ysplits = (static_cast<int64_t>(stream_.n_tiles) + b.span - 1) / b.span;
  // one CTA per left covers each candidate once: store, no zeroing pass
  b.direct = ysplits <= 1;
  if (!b.direct) EPI_CUDA(cudaMemsetAsync(bound, 0, n * sizeof(unsigned long long), st_));
  Timed t{next_event(), nullptr, next_event(), &stats.pass1_ms, -1, n, 0, false};
  t.e_map = t.e1;
  t.ms_out2 = &stats.bound_ms;
  stats.bound_words += n * static_cast<uint64_t>(stream_.n_tiles);
  rec(t.e0);
  const dim3 grid(static_cast<unsigned>(lf.nf), static_cast<unsigned>(std::max<int64_t>(ysplits, 1)));
  switch (L - 1) {
    case 1: bound_kernel<1><<<grid, kBoundThreads, 0, st_>>>(b); break;
    case 2: bound_kernel<2><<<grid, kBoundThreads, 0, st_>>>(b); break;
    case 3: bound_kernel<3><<<grid, kBoundThreads, 0, st_>>>(b); break;
    case 4: bound_kernel<4><<<grid, kBoundThreads, 0, st_>>>(b); break;
    case 5: bound_kernel<5><<<grid, kBoundThreads, 0, st_>>>(b); break;
    case 6: bound_kernel<6><<<grid, kBoundThreads, 0, st_>>>(b); break;
    default: bound_kernel<0><<<grid, kBoundThreads, 0, st_>>>(b); break;
  }
  EPI_CUDA(cudaGetLastError());
  rec(t.e1);
  timed_.push_back(t);

  const int mslot = new_slot();
  slot_counters_.push_back({mslot, &stats.pass2_episodes});
  const size_t s_types = 0, s_win = align256(static_cast<size_t>(n) * L * 4),
               s_sigma = s_win + align256(static_cast<size_t>(n) * M * 4),
               s_idx = s_sigma + align256(n * 4ull), s_total = s_idx + align256(n * 4ull);
  char* sbuf = scratch_.get<char>(kMSurv, s_total);
  uint32_t* stypes = reinterpret_cast<uint32_t*>(sbuf + s_types);
  uint32_t* swin = reinterpret_cast<uint32_t*>(sbuf + s_win);
  uint32_t* ssigma = reinterpret_cast<uint32_t*>(sbuf + s_sigma);
  uint32_t* sidx_out = reinterpret_cast<uint32_t*>(sbuf + s_idx);
  {
    const uint64_t nt = std::max<uint64_t>(lb_tiles(n), 1);
    if (nt <= kTcMaxTiles) {
      uint32_t* tc = scratch_.get<uint32_t>(kMTileCnt, nt);
      prune_count_tc<<<static_cast<unsigned>(nt), kLbThreads, 0, st_>>>(bound, threshold, n, d_counts, tc,
                                                                         d_acc_ + 2);
      JoinIdx jx{};
      if (lf.join_mode)
        jx = JoinIdx{lf.types, lf.win, lf.sigma, lf.pre, lf.lrange, lf.off, static_cast<uint32_t>(lf.nf), L - 1};
      prune_emit_tc<<<static_cast<unsigned>(nt), kLbThreads, 0, st_>>>(bound, threshold, n, L, c.types, c.win,
                                                                        c.sigma, stypes, swin, ssigma, sidx_out,
                                                                        tc, slot_ptr(mslot), jx);
    } else {
      unsigned long long* lb = scratch_.get<unsigned long long>(kMLookback, nt + 1);
      EPI_CUDA(cudaMemsetAsync(lb, 0, (nt + 1) * sizeof(unsigned long long), st_));
      prune_gather_lb<<<static_cast<unsigned>(nt), kLbThreads, 0, st_>>>(
          bound, threshold, n, L, c.types, c.win, c.sigma, d_counts, stypes, swin, ssigma, sidx_out, lb,
          slot_ptr(mslot), d_acc_ + 2);
    }
    EPI_CUDA(cudaGetLastError());
    stats.kernel_launches += 3;
  }
  DevSet sv = c;
  sv.types = stypes;
  sv.win = swin;
  sv.sigma = ssigma;
  uint64_t* sc = scratch_.get<uint64_t>(kMSurvCnt, n);
  count_device(sv, sc, stats, &stats.pass2_ms, mslot);
  if (surv) {
    surv->types = stypes;
    surv->win = swin;
    surv->counts = sc;
    surv->slot = mslot;
    return;
  }
  scatter_counts_kernel<<<blocks_for(n), 256, 0, st_>>>(sidx_out, sc, slot_ptr(mslot), d_counts);
  EPI_CUDA(cudaGetLastError());
  stats.kernel_launches += 2;
}

// ---- per-level CUDA graphs ---------------------------------------------------

namespace {
// epi_stats as counters (u64 fields, then doubles), for deltas
constexpr size_t kStatU64 = offsetof(epi_stats, pass1_ms) / sizeof(uint64_t);
void stats_axpy(epi_stats& a, const epi_stats& b, int sign) {
  auto* au = reinterpret_cast<uint64_t*>(&a);
  const auto* bu = reinterpret_cast<const uint64_t*>(&b);
  for (size_t i = 0; i < kStatU64; ++i) au[i] += sign > 0 ? bu[i] : (0 - bu[i]);
  double* ad[] = {&a.pass1_ms, &a.pass2_ms, &a.map_ms, &a.concat_ms, &a.total_ms, &a.bound_ms};
  const double bd[] = {b.pass1_ms, b.pass2_ms, b.map_ms, b.concat_ms, b.total_ms, b.bound_ms};
  for (int i = 0; i < 6; ++i) *ad[i] += sign * bd[i];
  a.bound_words += sign > 0 ? b.bound_words : (0 - b.bound_words);
  a.chain_launches += sign > 0 ? b.chain_launches : (0 - b.chain_launches);
  a.items_tracked += sign > 0 ? b.items_tracked : (0 - b.items_tracked);
  a.sort_fallbacks += sign > 0 ? b.sort_fallbacks : (0 - b.sort_fallbacks);
}
}  // namespace

template <class F>
void Engine::run_level(const std::string& key, bool graphable, epi_stats& stats, F&& enqueue) {
  if (!graphable || std::getenv("EPI_NO_GRAPH")) {
    enqueue();
    return;
  }
  LevelGraph* g = nullptr;
  for (auto& kv : level_graphs_)
    if (kv.first == key) g = &kv.second;
  if (!g) {
    if (level_graphs_.size() >= 64) {  // bounded cache
      for (auto& kv : level_graphs_)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      level_graphs_.clear();
    }
    level_graphs_.emplace_back(key, LevelGraph{});
    g = &level_graphs_.back().second;
  }
  char* const base = reinterpret_cast<char*>(&stats);
  auto off_of = [&](const void* ptr) -> ptrdiff_t {
    if (!ptr) return -1;
    const ptrdiff_t o = static_cast<const char*>(ptr) - base;
    return o >= 0 && o < static_cast<ptrdiff_t>(sizeof(epi_stats)) ? o : -2;
  };
  if (g->exec && g->log_start == log_used_ && g->ev_start == ev_used_) {
    // replay: relaunch the graph, then its enqueue's host bookkeeping
    EPI_CUDA(cudaGraphLaunch(g->exec, st_));
    stats_axpy(stats, g->delta, +1);
    if (g->segments_set) stats.segments = g->segments_after;
    for (const Timed& t : g->timed) {
      Timed r = t;
      r.ms_out = t.ms_out ? reinterpret_cast<double*>(base + reinterpret_cast<ptrdiff_t>(t.ms_out)) : nullptr;
      r.ms_out2 = t.ms_out2 ? reinterpret_cast<double*>(base + reinterpret_cast<ptrdiff_t>(t.ms_out2)) : nullptr;
      timed_.push_back(r);
    }
    for (const SlotCounter& sc : g->slots)
      slot_counters_.push_back({sc.slot, reinterpret_cast<uint64_t*>(base + reinterpret_cast<ptrdiff_t>(sc.target))});
    log_used_ = g->log_end;
    ev_used_ = g->ev_end;
    ++stat_epoch_;
    prefetched_epoch_ = stat_epoch_;  // the graph ends with the statistics prefetch
    return;
  }
  if (!g->capturable || g->exec || g->seen == 0) {
    // first sighting (warms every buffer the level needs) or a slot/event
    // position the graph was not captured at: run directly
    ++g->seen;
    enqueue();
    return;
  }
  // capture the enqueue, launch it, remember its bookkeeping
  const epi_stats before = stats;
  const size_t t0 = timed_.size(), s0 = slot_counters_.size();
  const int log0 = log_used_;
  const size_t ev0 = ev_used_;
  const uint64_t gen0 = buffers_generation();
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  bool ok = cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    capturing_ = true;
    try {
      enqueue();
    } catch (...) {
      ok = false;
    }
    capturing_ = false;
    if (cudaStreamEndCapture(st_, &graph) != cudaSuccess || !graph) ok = false;
  }
  if (ok && buffers_generation() != gen0) ok = false;
  if (ok && cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) ok = false;
  if (graph) cudaGraphDestroy(graph);
  for (size_t i = t0; ok && i < timed_.size(); ++i)
    if (off_of(timed_[i].ms_out) == -2 || off_of(timed_[i].ms_out2) == -2) ok = false;
  for (size_t i = s0; ok && i < slot_counters_.size(); ++i)
    if (off_of(slot_counters_[i].target) < 0) ok = false;
  if (!ok) {
    cudaGetLastError();
    if (exec) cudaGraphExecDestroy(exec);
    stats = before;
    timed_.resize(t0);
    slot_counters_.resize(s0);
    log_used_ = log0;
    ev_used_ = ev0;
    g->capturable = false;
    enqueue();
    return;
  }
  EPI_CUDA(cudaGraphLaunch(exec, st_));
  g->exec = exec;
  g->delta = stats;
  stats_axpy(g->delta, before, -1);
  g->segments_set = stats.segments != before.segments;
  g->segments_after = stats.segments;
  g->delta.segments = 0;
  g->timed.assign(timed_.begin() + static_cast<ptrdiff_t>(t0), timed_.end());
  for (Timed& t : g->timed) {
    t.ms_out = t.ms_out ? reinterpret_cast<double*>(off_of(t.ms_out)) : nullptr;
    t.ms_out2 = t.ms_out2 ? reinterpret_cast<double*>(off_of(t.ms_out2)) : nullptr;
  }
  g->slots.assign(slot_counters_.begin() + static_cast<ptrdiff_t>(s0), slot_counters_.end());
  for (SlotCounter& sc : g->slots) sc.target = reinterpret_cast<uint64_t*>(off_of(sc.target));
  g->log_start = log0;
  g->log_end = log_used_;
  g->ev_start = ev0;
  g->ev_end = ev_used_;
}

// mine (E/miner.hpp:114-173), device-resident; with `shard`, each large
// level's counting is split over the ranks and re-assembled by the caller's
// all-gather (epi_mine_sharded).
void Engine::mine(const epi_mine_config& cfg, epi_mine_result* out, const epi_shard* shard) {
  if (cfg.threshold < 1) throw Error(EPI_EINVAL, "mine: threshold must be >= 1");
  if (cfg.max_level < 1) throw Error(EPI_EINVAL, "mine: max_level must be >= 1");
  if (cfg.n_alpha == 0) throw Error(EPI_EINVAL, "mine: constraint alphabet must not be empty");
  const uint32_t W = shard ? shard->world : 1, R = shard ? shard->rank : 0;
  if (shard && (W == 0 || R >= W || (W > 1 && !shard->allgather)))
    throw Error(EPI_EINVAL, "mine: invalid shard (rank, world, allgather)");
  require_stream();
  std::vector<uint32_t> awin(cfg.n_alpha), ahi(cfg.n_alpha);
  int64_t amax = 0, amin_lo = INT64_MAX;
  int awidth = -1;
  for (uint64_t i = 0; i < cfg.n_alpha; ++i) {
    const int64_t lo = cfg.alpha_low[i], hi = cfg.alpha_high[i];
    if (lo < 0 || lo >= hi) throw Error(EPI_EINVAL, "interval constraint requires 0 <= low < high");
    if (hi > kMaxHighWide)
      throw Error(EPI_EUNSUPPORTED, "constraint high > 4095 ms is not supported by the device counter");
    awin[i] = static_cast<uint32_t>(lo + 1) | (static_cast<uint32_t>(hi) << 16);
    ahi[i] = static_cast<uint32_t>(hi);
    amax = std::max(amax, hi);
    amin_lo = std::min(amin_lo, lo);
    const int w = static_cast<int>(hi - lo);
    awidth = awidth == -1 ? w : (awidth == w ? w : 0);
  }
  // Pass-1 relaxation window: the hull (min low, max high] of the alphabet.
  const uint32_t alpha_hull = static_cast<uint32_t>(amin_lo + 1) | (static_cast<uint32_t>(amax) << 16);
  m_level_cands_.clear();
  m_level_off_.assign(1, 0);
  m_level_ms_.clear();
  m_counts_.clear();
  m_off_.assign(1, 0);
  m_types_.clear();
  m_lo_.clear();
  m_hi_.clear();
  epi_stats totals{};
  begin_op();
  g_trace.mark("mine start");
  const uint32_t A = stream_.alphabet;

  // Frequent set of the previous level, host side (types, packed windows).
  std::vector<uint32_t> ftypes, fwin;
  uint32_t F = 0;
  size_t nf = 0;

  auto record_level = [&](size_t cands, uint32_t L, const uint32_t* t, const uint32_t* w,
                          const uint64_t* cnt, size_t k, double ms) {
    const size_t c0 = m_counts_.size(), t0 = m_types_.size(), w0 = m_lo_.size();
    m_counts_.insert(m_counts_.end(), cnt, cnt + k);
    m_types_.insert(m_types_.end(), t, t + k * L);
    m_lo_.resize(w0 + k * (L - 1));
    m_hi_.resize(w0 + k * (L - 1));
    for (size_t j = 0; j < k * (L - 1); ++j) {
      m_lo_[w0 + j] = static_cast<int64_t>(w[j] & 0xffff) - 1;
      m_hi_[w0 + j] = static_cast<int64_t>(w[j] >> 16);
    }
    m_off_.resize(c0 + k + 1);
    for (size_t i = 0; i < k; ++i) m_off_[c0 + i + 1] = static_cast<uint32_t>(t0 + (i + 1) * L);
    m_level_cands_.push_back(cands);
    m_level_off_.push_back(m_counts_.size());
    m_level_ms_.push_back(ms);
  };

  for (size_t level = 1; level <= cfg.max_level; ++level) {
    auto t0 = std::chrono::steady_clock::now();
    const uint32_t L = static_cast<uint32_t>(level);
    // ---- candidate generation on the device ----------------------------
    uint64_t n = 0;
    std::vector<uint32_t> pre, lrange;
    std::vector<uint64_t> loff;
    if (level == 1) {
      n = A;  // every type of the alphabet (E/miner.hpp:81-84)
    } else if (level == 2) {
      n = static_cast<uint64_t>(nf) * nf * cfg.n_alpha;
    } else {
      // Join index over the frequent set: stable sort by the prefix key
      // (first L-2 nodes + their constraints); each left's bucket is the
      // range of rights whose prefix key equals the left's suffix key. Keys
      // are packed into 64 bits (type ids + constraint-alphabet indices)
      // when they fit, else compared field by field.
      const uint32_t K = F - 1;
      uint32_t tbits = 1, wbits = 1;
      while ((1ull << tbits) < A + 1ull) ++tbits;
      while ((1ull << wbits) < cfg.n_alpha) ++wbits;
      const bool packed = K * tbits + (K > 0 ? (K - 1) * wbits : 0) <= 64;
      pre.resize(nf);
      lrange.resize(2 * nf);
      loff.assign(nf + 1, 0);
      g_trace.mark("join alloc");
      if (packed) {
        auto widx = [&](uint32_t w) -> uint64_t {
          for (uint64_t i = 0; i < cfg.n_alpha; ++i)
            if (awin[i] == w) return i;
          return 0;  // frequent windows always come from the alphabet
        };
        auto key = [&](size_t i, uint32_t first) {
          uint64_t k = 0;
          for (uint32_t j = 0; j < K; ++j) k = (k << tbits) | ftypes[i * F + first + j];
          for (uint32_t j = 0; j + 1 < K; ++j) k = (k << wbits) | widx(fwin[i * (F - 1) + first + j]);
          return k;
        };
        const uint32_t kbits = K * tbits + (K > 0 ? (K - 1) * wbits : 0);
        if (kbits <= 16) {
          // small key space: stable counting sort, buckets read off the
          // prefix sums (no comparison sort, no binary search)
          std::vector<uint32_t> start((1u << kbits) + 1, 0);
          std::vector<uint32_t> k0(nf);
          for (size_t i = 0; i < nf; ++i) {
            k0[i] = static_cast<uint32_t>(key(i, 0));
            ++start[k0[i] + 1];
          }
          for (size_t b = 1; b < start.size(); ++b) start[b] += start[b - 1];
          std::vector<uint32_t> fill(start.begin(), start.end() - 1);
          for (size_t i = 0; i < nf; ++i) pre[fill[k0[i]]++] = static_cast<uint32_t>(i);
          g_trace.mark("join sort");
          for (uint32_t l = 0; l < nf; ++l) {
            const uint32_t k = static_cast<uint32_t>(key(l, 1));
            lrange[2 * l] = start[k];
            lrange[2 * l + 1] = start[k + 1];
            loff[l + 1] = loff[l] + (start[k + 1] - start[k]);
          }
        } else {
          std::vector<std::pair<uint64_t, uint32_t>> pk(nf);
          for (size_t i = 0; i < nf; ++i) pk[i] = {key(i, 0), static_cast<uint32_t>(i)};
          std::sort(pk.begin(), pk.end());  // (key, index): ties keep frequent order
          g_trace.mark("join sort");
          for (size_t i = 0; i < nf; ++i) pre[i] = pk[i].second;
          for (uint32_t l = 0; l < nf; ++l) {
            const uint64_t k = key(l, 1);
            auto lo = std::lower_bound(pk.begin(), pk.end(), std::make_pair(k, 0u));
            auto hi = std::upper_bound(lo, pk.end(), std::make_pair(k, UINT32_MAX));
            lrange[2 * l] = static_cast<uint32_t>(lo - pk.begin());
            lrange[2 * l + 1] = static_cast<uint32_t>(hi - pk.begin());
            loff[l + 1] = loff[l] + (hi - lo);
          }
        }
      } else {
        auto cmp_key = [&](uint32_t a, uint32_t fa, uint32_t b, uint32_t fb) -> int {
          for (uint32_t k = 0; k < K; ++k) {
            const uint32_t x = ftypes[static_cast<size_t>(a) * F + fa + k],
                           y = ftypes[static_cast<size_t>(b) * F + fb + k];
            if (x != y) return x < y ? -1 : 1;
          }
          for (uint32_t k = 0; k + 1 < K; ++k) {
            const uint32_t x = fwin[static_cast<size_t>(a) * (F - 1) + fa + k],
                           y = fwin[static_cast<size_t>(b) * (F - 1) + fb + k];
            if (x != y) return x < y ? -1 : 1;
          }
          return 0;
        };
        std::iota(pre.begin(), pre.end(), 0u);
        std::stable_sort(pre.begin(), pre.end(),
                         [&](uint32_t a, uint32_t b) { return cmp_key(a, 0, b, 0) < 0; });
        for (uint32_t l = 0; l < nf; ++l) {
          auto lo = std::lower_bound(pre.begin(), pre.end(), l, [&](uint32_t r, uint32_t left) {
            return cmp_key(r, 0, left, 1) < 0;
          });
          auto hi = std::upper_bound(lo, pre.end(), l, [&](uint32_t left, uint32_t r) {
            return cmp_key(left, 1, r, 0) < 0;
          });
          const uint32_t b0 = static_cast<uint32_t>(lo - pre.begin()), b1 = static_cast<uint32_t>(hi - pre.begin());
          lrange[2 * l] = b0;
          lrange[2 * l + 1] = b1;
          loff[l + 1] = loff[l] + (b1 - b0);
        }
      }
      n = loff[nf];
    }
    g_trace.mark("join index (host)");
    if (n == 0) break;
    if (n >= (1ull << 31)) throw Error(EPI_EUNSUPPORTED, "more than 2^31 candidates in one level");

    // Sharding of this level: rank R counts [R*s, R*s + cnt) of s-wide slices.
    const bool sharded =
        level > 1 && W > 1 && n >= std::max<uint64_t>(shard->min_shard, static_cast<uint64_t>(W) * W);
    const uint64_t s = sharded ? (n + W - 1) / W : n;
    const uint64_t lo_c = sharded ? std::min<uint64_t>(static_cast<uint64_t>(R) * s, n) : 0;
    const uint64_t cnt_c = sharded ? std::min<uint64_t>(s, n - lo_c) : n;

    uint32_t* d_types = scratch_.get<uint32_t>(kMTypes, n * L);
    uint32_t* d_win = scratch_.get<uint32_t>(kMWin, n * (L - 1));
    uint32_t* d_sigma = scratch_.get<uint32_t>(kMSigma, n);
    uint64_t* d_counts = scratch_.get<uint64_t>(kMCounts, sharded ? s * W : n);
    PopLefts lefts;  // the join's lefts on the device (popcount pass 1)
    lefts.nf = nf;
    lefts.slice_lo = lo_c;
    // ---- host prep: the level's upload into pinned memory ------------------
    size_t up_bytes = 0;
    char* h_up = nullptr;
    char* d_up = nullptr;
    size_t o_s = 0, o_p = 0, o_r = 0, o_o = 0;  // join upload layout (level >= 3)
    if (level == 1) {
      // the level-1 candidates are the type ids 0..A-1: a persistent device
      // copy (filled when the alphabet size changes), no per-call upload
      if (iota_n_ != n) {
        uint32_t* d = scratch_.get<uint32_t>(kMIota, n);
        std::vector<uint32_t> h(n);
        std::iota(h.begin(), h.end(), 0u);
        EPI_CUDA(cudaMemcpyAsync(d, h.data(), n * 4, cudaMemcpyHostToDevice, st_));
        EPI_CUDA(cudaStreamSynchronize(st_));
        iota_n_ = n;
      }
      d_types = scratch_.get<uint32_t>(kMIota, n);
    } else if (level == 2) {
      const size_t up = nf + 2 * cfg.n_alpha;
      up_bytes = up * 4;
      uint32_t* h = static_cast<uint32_t*>(pin_up_.get(up_bytes));
      std::copy(ftypes.begin(), ftypes.end(), h);
      std::copy(awin.begin(), awin.end(), h + nf);
      std::copy(ahi.begin(), ahi.end(), h + nf + cfg.n_alpha);
      h_up = reinterpret_cast<char*>(h);
      d_up = reinterpret_cast<char*>(scratch_.get<uint32_t>(kMFreq, up));
      lefts.types = reinterpret_cast<const uint32_t*>(d_up);
      lefts.stride = static_cast<uint64_t>(nf) * cfg.n_alpha;
    } else {
      // frequent types/win/sigma + pre + lrange + loff
      const size_t o_w = align256(nf * F * 4);
      o_s = o_w + align256(nf * (F - 1) * 4);
      o_p = o_s + align256(nf * 4);
      o_r = o_p + align256(nf * 4);
      o_o = o_r + align256(nf * 8);
      up_bytes = o_o + align256((nf + 1) * 8);
      h_up = static_cast<char*>(pin_up_.get(up_bytes));
      std::memcpy(h_up, ftypes.data(), nf * F * 4);
      std::memcpy(h_up + o_w, fwin.data(), nf * (F - 1) * 4);
      uint32_t* hs = reinterpret_cast<uint32_t*>(h_up + o_s);
      for (size_t i = 0; i < nf; ++i) {
        uint32_t sg = 0;
        for (uint32_t k = 0; k + 1 < F; ++k) sg += fwin[i * (F - 1) + k] >> 16;
        hs[i] = sg;
      }
      std::memcpy(h_up + o_p, pre.data(), nf * 4);
      std::memcpy(h_up + o_r, lrange.data(), nf * 8);
      std::memcpy(h_up + o_o, loff.data(), (nf + 1) * 8);
      d_up = scratch_.get<char>(kMJoin, up_bytes);
      lefts.types = reinterpret_cast<const uint32_t*>(d_up);
      lefts.win = reinterpret_cast<const uint32_t*>(d_up + o_w);
      lefts.off = reinterpret_cast<const uint64_t*>(d_up + o_o);
      lefts.pre = reinterpret_cast<const uint32_t*>(d_up + o_p);
      lefts.lrange = reinterpret_cast<const uint32_t*>(d_up + o_r);
      lefts.sigma = reinterpret_cast<const uint32_t*>(d_up + o_s);
    }
    DevSet c;
    c.N = L;
    c.n = cnt_c;
    c.types = d_types + lo_c * L;
    c.win = d_win + lo_c * (L - 1);
    c.sigma = d_sigma + lo_c;
    c.max_high = amax;
    c.max_sigma = static_cast<uint32_t>(amax * (L - 1));
    c.width = awidth > 0 ? awidth : 0;
    // Pass 1 by the popcount bound when the level is large enough to pay
    // and every window fits one history word; else the hull relaxation.
    const bool popbound = cfg.mode == EPI_MODE_MINE && cfg.threshold > 1 && n >= min_pass1() &&
                          amax <= 32 && cfg.n_alpha <= 16 && L <= static_cast<uint32_t>(kBoundMaxL) &&
                          !std::getenv("EPI_PASS1_HULL");
    // Unsharded popcount levels never materialise their candidates: pass 1
    // and the survivor gather read them off the join index, and only
    // survivors can be frequent (compacted from the survivor arrays).
    lefts.join_mode = popbound && !sharded && level >= 3 && lb_tiles(n) <= kTcMaxTiles &&
                      !std::getenv("EPI_MATERIALISE");
    // the hull pass 1 synchronises mid-level (its group count): not graphable
    const bool hull_pass1 = level > 1 && !popbound && cfg.mode == EPI_MODE_MINE && cfg.threshold > 1 &&
                            n >= min_pass1();
    map_small_.get(64);
    uint32_t* h_k = static_cast<uint32_t*>(map_small_.p) + 1;
    const size_t o_ft = 0, o_fw = align256(static_cast<size_t>(n) * L * 4),
                 o_fc = o_fw + align256(static_cast<size_t>(n) * (L - 1) * 4), o_fend = o_fc + align256(n * 8ull);
    map_out_.get(o_fend);
    // Small levels compact into device memory and copy the (bounded) result
    // back in one transfer; large ones write their few frequent episodes
    // straight into mapped host memory (scattered PCIe writes are slow for
    // thousands of entries, a full-size copy is slow for large levels).
    constexpr size_t kCopyBack = 512u << 10;
    const bool copy_back = o_fend <= kCopyBack;
    char* dm = copy_back ? scratch_.get<char>(kMFreqOut, o_fend) : static_cast<char*>(map_out_.d);
    const bool compact_cub = std::getenv("EPI_COMPACT_CUB") != nullptr;
    if (n > kOneBlkMax && !compact_cub) {
      if (lb_tiles(n) <= kTcMaxTiles)
        scratch_.get<uint32_t>(kMTileCnt, lb_tiles(n));
      else
        scratch_.get<unsigned long long>(kMLookback, lb_tiles(n) + 1);
    }

    if (popbound) scratch_.get<uint32_t>(kMTileCnt, std::max<uint64_t>(lb_tiles(n), 1));
    Survivors surv;  // set by the popbound pass on unsharded levels
    // ---- device work of the level ------------------------------------------
    auto enqueue = [&]() {
      surv = Survivors{};
      if (up_bytes) {
        EPI_CUDA(cudaMemcpyAsync(d_up, h_up, up_bytes, cudaMemcpyHostToDevice, st_));
        totals.h2d_bytes += up_bytes;
      }
      if (level == 2) {
        const uint32_t* d = reinterpret_cast<const uint32_t*>(d_up);
        gen_level2_kernel<<<blocks_for(n), 256, 0, st_>>>(d, static_cast<uint32_t>(nf), d + nf,
                                                          d + nf + cfg.n_alpha,
                                                          static_cast<uint32_t>(cfg.n_alpha), d_types,
                                                          d_win, d_sigma, n);
        EPI_CUDA(cudaGetLastError());
        totals.kernel_launches += 1;
      } else if (level > 2 && !lefts.join_mode) {
        const unsigned blocks = static_cast<unsigned>((nf * 32 + 255) / 256);
        gen_join_kernel<<<blocks, 256, 0, st_>>>(
            L, reinterpret_cast<const uint32_t*>(d_up), reinterpret_cast<const uint32_t*>(lefts.win),
            reinterpret_cast<const uint32_t*>(d_up + o_s), static_cast<uint32_t>(nf),
            reinterpret_cast<const uint32_t*>(d_up + o_p), reinterpret_cast<const uint32_t*>(d_up + o_r),
            reinterpret_cast<const uint64_t*>(d_up + o_o), d_types, d_win, d_sigma);
        EPI_CUDA(cudaGetLastError());
        totals.kernel_launches += 1;
      }
      g_trace.mark("gen launched");
      uint64_t* counts_all = d_counts;
      if (level == 1) {
        // single-node episodes: a popcount of each type's bitmap row
        totals.episodes += n;
        totals.pass2_episodes += n;
        count_device(c, d_counts, totals, &totals.pass2_ms);
      } else if (cnt_c > 0 && popbound) {
        count_device_popbound(c, lefts, cfg.threshold, awin.data(), static_cast<uint32_t>(cfg.n_alpha),
                              d_counts + lo_c, totals, sharded ? nullptr : &surv);
      } else if (cnt_c > 0) {
        count_device_two_pass(c, cfg.threshold, cfg.mode, alpha_hull, awin.data(),
                              static_cast<uint32_t>(cfg.n_alpha), d_counts + lo_c, totals);
      }
      g_trace.mark("count launched");
      if (sharded) {
        // every rank's s-wide slice -> the full count vector in candidate order
        uint64_t* d_all = scratch_.get<uint64_t>(kMGather, s * W);
        const int rc = shard->allgather(shard->user, d_counts + static_cast<uint64_t>(R) * s, d_all,
                                        s * sizeof(uint64_t), static_cast<void*>(st_));
        if (rc != 0) throw Error(EPI_ENCCL, "mine: all-gather of level counts failed");
        counts_all = d_all;
      }
      // threshold + compaction in candidate order, straight to host memory
      if (surv.slot >= 0 && n <= kOneBlkMax && !std::getenv("EPI_SURV_TC")) {
        // only pass-1 survivors can be frequent: compact those (in order);
        // one CTA while the level (a bound on its survivors) is small
        surv_compact_1blk<<<1, kOneBlk, 0, st_>>>(
            surv.counts, cfg.threshold, slot_ptr(surv.slot), L, surv.types, surv.win,
            reinterpret_cast<uint32_t*>(dm + o_ft), reinterpret_cast<uint32_t*>(dm + o_fw),
            reinterpret_cast<uint64_t*>(dm + o_fc), slot_ptr(new_slot()), h_k);
        EPI_CUDA(cudaGetLastError());
        totals.kernel_launches += 1;
      } else if (surv.slot >= 0) {
        const uint64_t nt = std::max<uint64_t>(lb_tiles(n), 1);
        uint32_t* tc = scratch_.get<uint32_t>(kMTileCnt, nt);
        surv_count_tc<<<static_cast<unsigned>(nt), kLbThreads, 0, st_>>>(surv.counts, cfg.threshold,
                                                                         slot_ptr(surv.slot), tc);
        surv_emit_tc<<<static_cast<unsigned>(nt), kLbThreads, 0, st_>>>(
            surv.counts, cfg.threshold, slot_ptr(surv.slot), L, surv.types, surv.win,
            reinterpret_cast<uint32_t*>(dm + o_ft), reinterpret_cast<uint32_t*>(dm + o_fw),
            reinterpret_cast<uint64_t*>(dm + o_fc), tc, slot_ptr(new_slot()), h_k);
        EPI_CUDA(cudaGetLastError());
        totals.kernel_launches += 2;
      } else if (n <= kOneBlkMax) {
        compact_freq_1blk<<<1, kOneBlk, 0, st_>>>(counts_all, cfg.threshold, n, L, d_types, d_win,
                                                  reinterpret_cast<uint32_t*>(dm + o_ft),
                                                  reinterpret_cast<uint32_t*>(dm + o_fw),
                                                  reinterpret_cast<uint64_t*>(dm + o_fc), slot_ptr(new_slot()),
                                                  h_k);
        EPI_CUDA(cudaGetLastError());
        totals.kernel_launches += 1;
      } else if (!compact_cub && lb_tiles(n) <= kTcMaxTiles) {
        const uint64_t nt = lb_tiles(n);
        uint32_t* tc = scratch_.get<uint32_t>(kMTileCnt, nt);
        freq_count_tc<<<static_cast<unsigned>(nt), kLbThreads, 0, st_>>>(counts_all, cfg.threshold, n, tc);
        freq_emit_tc<<<static_cast<unsigned>(nt), kLbThreads, 0, st_>>>(
            counts_all, cfg.threshold, n, L, d_types, d_win, reinterpret_cast<uint32_t*>(dm + o_ft),
            reinterpret_cast<uint32_t*>(dm + o_fw), reinterpret_cast<uint64_t*>(dm + o_fc), tc,
            slot_ptr(new_slot()), h_k);
        EPI_CUDA(cudaGetLastError());
        totals.kernel_launches += 2;
      } else if (!compact_cub) {
        const uint64_t nt = lb_tiles(n);
        unsigned long long* lb = scratch_.get<unsigned long long>(kMLookback, nt + 1);
        EPI_CUDA(cudaMemsetAsync(lb, 0, (nt + 1) * sizeof(unsigned long long), st_));
        compact_freq_lb<<<static_cast<unsigned>(nt), kLbThreads, 0, st_>>>(
            counts_all, cfg.threshold, n, L, d_types, d_win, reinterpret_cast<uint32_t*>(dm + o_ft),
            reinterpret_cast<uint32_t*>(dm + o_fw), reinterpret_cast<uint64_t*>(dm + o_fc), lb,
            slot_ptr(new_slot()), h_k);
        EPI_CUDA(cudaGetLastError());
        totals.kernel_launches += 1;
      } else {
        uint32_t* flags = scratch_.get<uint32_t>(kMFlags, n);
        uint32_t* scan = scratch_.get<uint32_t>(kMScan, n);
        freq_flags_kernel<<<blocks_for(n), 256, 0, st_>>>(counts_all, cfg.threshold, n, flags);
        EPI_CUDA(cudaGetLastError());
        dev_scan_total(flags, scan, n, new_slot(), h_k);
        compact_freq_kernel<<<blocks_for(n), 256, 0, st_>>>(
            flags, scan, n, L, d_types, d_win, counts_all, reinterpret_cast<uint32_t*>(dm + o_ft),
            reinterpret_cast<uint32_t*>(dm + o_fw), reinterpret_cast<uint64_t*>(dm + o_fc));
        EPI_CUDA(cudaGetLastError());
        totals.kernel_launches += 5;
      }
      if (copy_back) {
        EPI_CUDA(cudaMemcpyAsync(map_out_.p, dm, o_fend, cudaMemcpyDeviceToHost, st_));
      }
      g_trace.mark("compact launched");
      prefetch_stats();
    };

    // key: every host-side value the enqueue depends on
    std::string key;
    auto put = [&](uint64_t v) { key.append(reinterpret_cast<const char*>(&v), sizeof v); };
    put(level);
    put(n);
    put(nf);
    put(lo_c);
    put(cnt_c);
    put(popbound);
    put(cfg.mode);
    put(cfg.threshold);
    put(cfg.n_alpha);
    for (uint32_t w : awin) put(w);
    put(static_cast<uint64_t>(amax));
    put(static_cast<uint64_t>(awidth));
    put(up_bytes);
    put(stream_.n_tiles);
    put(stream_.blk_words);
    put(stream_.alphabet);
    put(stream_.gap_cap);
    put(buffers_generation());
    put(compact_cub);
    put(std::getenv("EPI_WALK_SEQ") != nullptr);
    put(std::getenv("EPI_SURV_TC") != nullptr);
    put(lefts.join_mode);
    const char* fs = std::getenv("EPI_FORCE_SEGMENTS");
    put(fs ? std::strtoull(fs, nullptr, 10) + 1 : 0);
    const size_t timed_before = timed_.size();
    run_level(key, !sharded && !hull_pass1 && amax <= kMaxHigh, totals, enqueue);
    resolve_timed(totals, timed_before);  // earlier levels', overlapping this one
    EPI_CUDA(cudaStreamSynchronize(st_));
    g_trace.mark("level synced");
    const uint32_t k = *reinterpret_cast<volatile uint32_t*>(h_k);
    const char* hm = static_cast<const char*>(map_out_.p);
    std::vector<uint32_t> ntypes(static_cast<size_t>(k) * L), nwin(static_cast<size_t>(k) * (L - 1));
    std::vector<uint64_t> ncnt(k);
    std::memcpy(ntypes.data(), hm + o_ft, ntypes.size() * 4);
    std::memcpy(nwin.data(), hm + o_fw, nwin.size() * 4);
    std::memcpy(ncnt.data(), hm + o_fc, ncnt.size() * 8);
    totals.d2h_bytes += static_cast<uint64_t>(k) * (8 + 4 * (2 * L - 1)) + 4;
    record_level(n, L, ntypes.data(), nwin.data(), ncnt.data(), k,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    ftypes.swap(ntypes);
    fwin.swap(nwin);
    F = L;
    nf = k;
    g_trace.mark("level recorded");
    if (nf == 0) break;
  }
  g_trace.mark("levels done");
  flush_stats(totals);
  g_trace.mark("stats flushed");
  g_trace.dump();
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
