// Exact non-overlapped episode counting on sm_100a: a bit-sliced counting
// automaton, run segment-parallel (MapConcatenate) and stitched by a
// per-episode concat walk. Included by count.cu / count_w*.cu (narrow
// windows, high <= 63) and count_wide.cu (high <= 4095); see DESIGN.md.
//
// Semantics follow run_fsm / count_fsm (E/fsm.hpp:45-106) exactly:
//   * an event of type tau at time t is admitted at position 0 iff t > pe
//     (pe = time of the last counted completion, E/fsm.hpp:66-68);
//   * at position k >= 1 iff some entry of position k-1 has time in
//     [t-high, t-low)  (E/fsm.hpp:73-79);
//   * admitting the last position counts one occurrence, sets pe = t and
//     clears every list (E/fsm.hpp:83-91).
// Because every admissible gap is >= 1 (low >= 0), admissions at time t only
// read entries older than t. So the automaton's behaviour depends only on the
// set of distinct firing times per type, the order of tied events does not
// matter, and a whole 32 ms tile can be advanced with word-wide bit
// operations:
//
//   C_0 = occ(tau_0) & (times > pe)
//   C_k = occ(tau_k) & OR_{a=low+1..high} (C_{k-1} : history_{k-1}) << a
//
// where history_{k-1} holds the entry bitmaps of the previous tiles. The
// first set bit of C_{N-1} is a completion; the tile is then recomputed above
// it with empty history (the reference's list clear). Rare, so the loop is
// off the hot path.
//
// MapConcatenate (E/mapconcat.hpp:71-159, paper PAPER.md:249-266): the tile
// range is cut into P segments. The automaton state at a segment start T is
// either FRESH (the last completion is older than T - sum(high): no live
// entry can predate the window [T - sum(high), T), so a machine started empty
// at the window start reaches the true state) or RESTART(L) (the last
// completion L lies inside the window: the state is "cleared at L, pe = L").
// The map kernel runs the FRESH machine of every (episode, segment) in
// parallel and records its count, last completion and first kRecorded
// completion times. The concat walk (one thread per episode) chains the
// segments; when a boundary needs RESTART(L) it re-runs that machine inline
// only until it provably coincides with the FRESH machine (same completion,
// or both quiet for sum(high)) and reads the rest of the segment off the
// FRESH record ("patch", cf. E/mapconcat.hpp:144-148).
//
// Bitmap layout (DeviceStream): blocks of kBlkTiles = 32 tiles; inside a
// block, type tau's 32 tile words are contiguous at tau * kRowStride
// (kRowStride = 36: 4 pad words spread the rows over the shared-memory
// banks). A lane fetches 4 consecutive tiles of its type with one 16-byte
// load; a CTA stages one whole block (all types) per bulk copy.
#pragma once

#include "common.cuh"
#include "count.h"

namespace epi {
namespace impl {

constexpr int kMachThreads = 256;
constexpr int kStages = 3;

template <int N>
struct EpParams {
  static constexpr int M = N > 1 ? N - 1 : 1;
  uint32_t type[N];
  uint32_t lo1[M];  // low + 1
  uint32_t hi[M];   // high
  uint32_t sigma;   // sum of highs (MapConcatenate window)
};

template <int N>
__device__ __forceinline__ EpParams<N> load_episode(const CountLaunch& p, uint32_t e) {
  EpParams<N> ep;
#pragma unroll
  for (int k = 0; k < N; ++k) ep.type[k] = p.ep_types[static_cast<size_t>(e) * N + k];
#pragma unroll
  for (int k = 0; k < EpParams<N>::M; ++k) {
    uint32_t w = N > 1 ? p.ep_win[static_cast<size_t>(e) * (N - 1) + k] : 0x10001u;
    ep.lo1[k] = w & 0xffff;
    ep.hi[k] = w >> 16;
  }
  ep.sigma = p.ep_sigma[e];
  return ep;
}

__device__ __forceinline__ int32_t seg_bound(const CountLaunch& p, int q) {
  const int64_t g = static_cast<int64_t>(q) * p.seg_len;
  return g < p.seg_end ? static_cast<int32_t>(g) : p.seg_end;
}

__device__ __forceinline__ uint32_t live_eps(const CountLaunch& p) {
  return p.n_dev ? *p.n_dev : p.n_eps;
}

__device__ __forceinline__ uint32_t out_index(const CountLaunch& p, uint32_t e) {
  return p.out_perm ? p.out_perm[e] : e;
}

__device__ __forceinline__ size_t occ_index(int32_t g, uint32_t type, uint32_t blk_words) {
  return static_cast<size_t>(g >> 5) * blk_words + type * kRowStride + (g & 31);
}

// ---- history policies -------------------------------------------------------

// Window test over X = (c : h1 : h2) (96 bits, c the current tile): bit i of
// the result is set iff X has a set bit at age a in [lo1, hi] from time
// 32*g + i, i.e. at X index 64 + i - a. With Z = X >> (64 - hi) (64 bits,
// Z[j] = X[64 - hi + j]) this is OR_{b < w} Z[i + b], w = hi - lo1 + 1:
// two funnel shifts to extract Z, then a smear of width w. Branch-free;
// requires w <= 32 (wider windows are split in two). kHi32: every high <= 32,
// so X = (c : h1) and the selects disappear.
template <int W, bool kHi32>
__device__ __forceinline__ uint32_t window_any(uint32_t c, uint32_t h1, uint32_t h2, uint32_t lo1,
                                               uint32_t hi) {
  uint32_t zl, zh;
  if constexpr (kHi32 && W >= 9) {
    // wide uniform windows (e.g. the pass-1 hull of a bin alphabet): a
    // compile-time doubling smear over Z = (c : h1) >> (32 - hi) costs
    // ~2 log2(W) + 2 shifts instead of W (the high word is dropped after
    // the last step)
    const uint32_t s = 32u - hi;
    uint32_t rl = __funnelshift_r(h1, c, s), rh = c >> s;
    constexpr int kS1 = 1, kS2 = 2, kS3 = W - 4 < 4 ? W - 4 : 4;  // cover 1 -> 2 -> 4 -> 4 + kS3
    rl |= __funnelshift_r(rl, rh, kS1);
    rh |= rh >> kS1;
    rl |= __funnelshift_r(rl, rh, kS2);
    rh |= rh >> kS2;
    if constexpr (W - 4 - kS3 > 0) {
      rl |= __funnelshift_r(rl, rh, kS3);
      rh |= rh >> kS3;
      rl |= __funnelshift_r(rl, rh, W - 4 - kS3);  // cover 8 -> W (W <= 16)
    } else {
      rl |= __funnelshift_r(rl, rh, kS3);
    }
    return rl;
  } else if constexpr (kHi32 && W > 0) {
    // X = (c : h1); term b of the smear is (c : h1) >> (32 - hi + b), and
    // 32 - hi + b <= 32 - lo1 <= 31, so each term is one funnel shift (ALU
    // pipe). (Moving terms to the FMA pipe as hi32(h1*m + ((c*m) << 32))
    // with m = 2^(hi-b) was measured 33% slower: nvcc kept the shifts and
    // split the 64-bit add onto the ALU pipe.)
    const uint32_t s = 32u - hi;
    uint32_t d = __funnelshift_r(h1, c, s);
#pragma unroll
    for (int b = 1; b < W; ++b) d |= __funnelshift_r(h1, c, s + b);
    return d;
  } else if constexpr (kHi32) {
    const uint32_t s = 32u - hi;  // 0..31
    zl = __funnelshift_r(h1, c, s);
    zh = c >> s;
  } else {
    const uint32_t s = 64u - hi;  // 1..63
    const bool low = s < 32u;
    const uint32_t w0 = low ? h2 : h1;
    const uint32_t w1 = low ? h1 : c;
    const uint32_t w2 = low ? c : 0u;
    zl = __funnelshift_r(w0, w1, s & 31u);
    zh = __funnelshift_r(w1, w2, s & 31u);
  }
  if constexpr (W > 0) {
    uint32_t d = zl;
#pragma unroll
    for (int b = 1; b < W; ++b) d |= __funnelshift_r(zl, zh, b);
    return d;
  } else {
    // runtime width: doubling smear, cover 1 -> 2 -> 4 -> ... -> w
    const uint32_t w = hi - lo1 + 1u;
    uint32_t rl = zl, rh = zh, cover = 1;
#pragma unroll
    for (int step = 0; step < 5; ++step) {
      const uint32_t sh = cover < w ? (cover < w - cover ? cover : w - cover) : 0u;
      rl |= __funnelshift_r(rl, rh, sh);
      rh |= rh >> sh;
      cover += sh;
    }
    return rl;
  }
}

// high <= 63: the entry bitmaps of the previous tiles, in registers (two
// words; one when every high <= 32). W > 0: every window of the launch has
// width high - low == W (compile-time unrolled smear); W == 0: runtime.
// Window test of the last constraint when it alone has a different,
// launch-uniform width (pass 1 relaxes only the last constraint to the
// constraint alphabet's hull, high <= 32): a doubling smear whose four shift
// amounts are kernel parameters (constant bank), so the other positions keep
// the compile-time width W.
__device__ __forceinline__ uint32_t window_last(uint32_t c, uint32_t h1, uint32_t hi,
                                                const CountLaunch& p) {
  const uint32_t s = 32u - hi;
  uint32_t rl = __funnelshift_r(h1, c, s), rh = c >> s;
  rl |= __funnelshift_r(rl, rh, p.last_sh[0]);
  rh |= rh >> p.last_sh[0];
  rl |= __funnelshift_r(rl, rh, p.last_sh[1]);
  rh |= rh >> p.last_sh[1];
  rl |= __funnelshift_r(rl, rh, p.last_sh[2]);
  rh |= rh >> p.last_sh[2];
  return rl | __funnelshift_r(rl, rh, p.last_sh[3]);
}

template <int N, int W = 0, bool kHi32 = false, bool kLast = false>
struct NarrowHist {
  static_assert(!kLast || (kHi32 && W > 0), "last-position smear needs high <= 32 and a uniform W");
  static constexpr bool kQuad = true;  // four tiles per 16-byte load, unrolled
  static constexpr int M = N > 1 ? N - 1 : 1;
  static constexpr int M2 = kHi32 ? 1 : M;
  uint32_t h1[M];
  uint32_t h2[M2];

  __device__ __forceinline__ void reset(int32_t, int) {
#pragma unroll
    for (int k = 0; k < M; ++k) h1[k] = 0;
#pragma unroll
    for (int k = 0; k < M2; ++k) h2[k] = 0;
  }
  __device__ __forceinline__ void on_clear(int32_t g) { reset(g, 0); }
  __device__ __forceinline__ static uint32_t dil(uint32_t c, uint32_t h1, uint32_t h2, uint32_t lo1,
                                                 uint32_t hi) {
    if constexpr (W > 0) {
      return window_any<W, kHi32>(c, h1, h2, lo1, hi);
    } else {
      if (hi - lo1 < 32u) return window_any<0, kHi32>(c, h1, h2, lo1, hi);
      return window_any<0, kHi32>(c, h1, h2, lo1, lo1 + 31u) |
             window_any<0, kHi32>(c, h1, h2, lo1 + 32u, hi);
    }
  }
  __device__ __forceinline__ uint32_t dilate(int k, uint32_t c, uint32_t lo1, uint32_t hi, int32_t,
                                             const CountLaunch& p) const {
    if constexpr (kLast) {
      if (k == N - 2) return window_last(c, h1[k], hi, p);
    }
    return dil(c, h1[k], kHi32 ? 0u : h2[kHi32 ? 0 : k], lo1, hi);
  }
  __device__ __forceinline__ static uint32_t dilate_fresh(int k, uint32_t c, uint32_t lo1, uint32_t hi,
                                                          const CountLaunch& p) {
    if constexpr (kLast) {
      if (k == N - 2) return window_last(c, 0u, hi, p);
    }
    return dil(c, 0u, 0u, lo1, hi);
  }
  __device__ __forceinline__ void push(const uint32_t* C, int32_t) {
#pragma unroll
    for (int k = 0; k < N - 1; ++k) {
      if constexpr (!kHi32) h2[k] = h1[k];
      h1[k] = C[k];
    }
  }
};

// high <= 32*HWMAX: a ring of per-tile entry bitmaps in local memory, `hw`
// words deep (uniform per launch). Tiles older than `clear_tile` read as 0,
// so a clear costs O(1).
template <int N, int HWMAX>
struct WideHist {
  static constexpr bool kQuad = false;  // rare path: one tile per iteration, compact code
  static constexpr int M = N > 1 ? N - 1 : 1;
  static constexpr int kMask = HWMAX - 1;
  uint32_t ring[M][HWMAX];
  int head;          // slot of the newest pushed tile word
  int32_t last;      // tile index of the newest pushed word
  int32_t clear_tile;
  int hw;

  __device__ __forceinline__ void reset(int32_t g_start, int hw_) {
    head = 0;
    last = g_start - 1;
    clear_tile = g_start;
    hw = hw_;
  }
  __device__ __forceinline__ void on_clear(int32_t g) { clear_tile = g; }

  // Word widx in [0, hw] of X = (hw history words, then the current tile):
  // widx == hw is `c`, widx == hw - j is the tile j back.
  __device__ __forceinline__ uint32_t word(int k, int widx, uint32_t c, int32_t g) const {
    if (widx >= hw) return widx == hw ? c : 0u;
    const int j = hw - widx;
    const int32_t tile = g - j;
    if (tile < clear_tile || tile > last) return 0u;
    return ring[k][(head - (last - tile)) & kMask];
  }
  __device__ __forceinline__ uint32_t slice32(int k, int x, uint32_t c, int32_t g) const {
    const int w = x >> 5, s = x & 31;
    return __funnelshift_r(word(k, w, c, g), word(k, w + 1, c, g), s);
  }
  __device__ uint32_t dilate(int k, uint32_t c, uint32_t lo1, uint32_t hi, int32_t g,
                             const CountLaunch&) const {
    const int A = static_cast<int>(lo1), B = static_cast<int>(hi);
    const int P0 = 32 * hw - B, P1 = 32 * hw - A;
    const int w = B - A + 1;  // window width (high - low)
    if (w <= 32) {
      uint64_t r = static_cast<uint64_t>(slice32(k, P0, c, g)) |
                   (static_cast<uint64_t>(slice32(k, P0 + 32, c, g)) << 32);
      int cover = 1;
      while (cover < w) {
        const int sh = cover < w - cover ? cover : w - cover;
        r |= r >> sh;
        cover += sh;
      }
      return static_cast<uint32_t>(r);
    }
    // interior [P0+31, P1] is inside every bit's window
    bool any = false;
    const int lo = P0 + 31, hix = P1;
    for (int wi = lo >> 5; wi <= (hix >> 5) && !any; ++wi) {
      uint32_t m = ~0u;
      if (wi == (lo >> 5)) m &= ~0u << (lo & 31);
      if (wi == (hix >> 5)) m &= (hix & 31) == 31 ? ~0u : ((1u << ((hix & 31) + 1)) - 1u);
      any = (word(k, wi, c, g) & m) != 0;
    }
    uint32_t sl = slice32(k, P0, c, g) & 0x7fffffffu;  // left edge: any(X[P0+i .. P0+30])
    sl |= sl >> 1;
    sl |= sl >> 2;
    sl |= sl >> 4;
    sl |= sl >> 8;
    sl |= sl >> 16;
    uint32_t sr = (slice32(k, P1 + 1, c, g) & 0x7fffffffu) << 1;  // right: any(X[P1+1 .. P1+i])
    sr |= sr << 1;
    sr |= sr << 2;
    sr |= sr << 4;
    sr |= sr << 8;
    sr |= sr << 16;
    return (any ? ~0u : 0u) | sl | sr;
  }
  __device__ __forceinline__ static uint32_t dilate_fresh(int, uint32_t c, uint32_t lo1, uint32_t hi,
                                                          const CountLaunch&) {
    uint32_t d = 0;
    const uint32_t e1 = hi < 31u ? hi : 31u;
    for (uint32_t a = lo1; a <= e1; ++a) d |= c << a;
    return d;
  }
  __device__ __forceinline__ void push(const uint32_t* C, int32_t g) {
    head = (head + 1) & kMask;
    last = g;
#pragma unroll
    for (int k = 0; k < N - 1; ++k) ring[k][head] = C[k];
  }
};

template <int N, class Hist>
struct Machine {
  Hist hist;
  int32_t thr_tile;   // position 0 admits only times > thr:
  uint32_t thr_mask;  // tiles < thr_tile none, tile == thr_tile thr_mask

  __device__ __forceinline__ void set_threshold(int64_t thr) {
    if (thr < 0) {
      thr_tile = -1;
      thr_mask = ~0u;
    } else {
      thr_tile = static_cast<int32_t>(thr >> 5);
      uint32_t b = static_cast<uint32_t>(thr & 31);
      thr_mask = b == 31 ? 0u : (~0u << (b + 1));
    }
  }
};

// Advance one tile. on_completion(time) returns true to stop the machine.
// kMask: the tile may lie at or before the position-0 threshold tile.
template <int N, class Hist, bool kMask, class OnC>
__device__ __forceinline__ bool tile_step(Machine<N, Hist>& m, const EpParams<N>& ep,
                                          const uint32_t (&occ)[N], int32_t g, const CountLaunch& p,
                                          OnC&& on_c) {
  uint32_t C[N];
  C[0] = occ[0];
  if constexpr (kMask) {
    if (g <= m.thr_tile) C[0] &= (g < m.thr_tile) ? 0u : m.thr_mask;
  }
#pragma unroll
  for (int k = 1; k < N; ++k)
    C[k] = occ[k] & m.hist.dilate(k - 1, C[k - 1], ep.lo1[k - 1], ep.hi[k - 1], g, p);
  if (C[N - 1]) {
    uint32_t last = C[N - 1];
    do {
      const int b = __ffs(last) - 1;
      const uint64_t tc = static_cast<uint64_t>(g) * 32 + b;
      if (on_c(tc)) return true;
      const uint32_t msk = b == 31 ? 0u : (~0u << (b + 1));
      m.thr_tile = g;
      m.thr_mask = msk;
      C[0] = occ[0] & msk;
#pragma unroll
      for (int k = 1; k < N; ++k)
        C[k] = occ[k] & Hist::dilate_fresh(k - 1, C[k - 1], ep.lo1[k - 1], ep.hi[k - 1], p);
      last = C[N - 1];
    } while (last);
    m.hist.on_clear(g);  // the clear also empties older history
  }
  m.hist.push(C, g);
  return false;
}

// Four consecutive tiles g..g+3 from 16-byte loads (v[k] = tiles of type k).
// (A speculative no-completion fast path per quad was measured slower: with
// 32 episodes per warp about half of all quads hold some lane's completion,
// so the warp replays the quad anyway.)
template <int N, class Hist, bool kMask, class OnC>
__device__ __forceinline__ void quad_step(Machine<N, Hist>& m, const EpParams<N>& ep,
                                          const uint4 (&v)[N], int32_t g, const CountLaunch& p,
                                          OnC&& on_c) {
  uint32_t o[N];
#pragma unroll
  for (int k = 0; k < N; ++k) o[k] = v[k].x;
  tile_step<N, Hist, kMask>(m, ep, o, g, p, on_c);
#pragma unroll
  for (int k = 0; k < N; ++k) o[k] = v[k].y;
  tile_step<N, Hist, kMask>(m, ep, o, g + 1, p, on_c);
#pragma unroll
  for (int k = 0; k < N; ++k) o[k] = v[k].z;
  tile_step<N, Hist, kMask>(m, ep, o, g + 2, p, on_c);
#pragma unroll
  for (int k = 0; k < N; ++k) o[k] = v[k].w;
  tile_step<N, Hist, kMask>(m, ep, o, g + 3, p, on_c);
}

// Map step: FRESH machine of (episode, segment). The CTA walks the bitmap
// blocks covering its segment (plus window); with p.stages > 0 each block is
// staged into shared memory by one bulk copy (TMA engine) in a ring of
// p.stages buffers, otherwise (very large alphabets) lanes read their rows
// from global memory through L1. Every thread of the CTA walks the same
// tiles, so one staged block serves all 256 episodes of the block.
template <int N, class Hist>
__global__ void __launch_bounds__(kMachThreads) machines_kernel(const CountLaunch p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint32_t* stage = reinterpret_cast<uint32_t*>(smem + 128);
  const uint32_t bw = p.blk_words;
  const int stages = p.stages;

  // Grid: (episode blocks, segments) - CTAs resident together walk the same
  // segments, so each staged bitmap block is reused from L2 across episode
  // blocks. Launches sized for an upper bound (device-side live count) use
  // (segments, episode blocks) instead: the live episode blocks come first in
  // dispatch order and start before the idle CTAs are retired.
  const int q = static_cast<int>(p.n_dev ? blockIdx.x : blockIdx.y) + p.q_base;
  const uint32_t eblk = p.n_dev ? blockIdx.y : blockIdx.x;
  const uint32_t n_live = live_eps(p);
  // launches sized for an upper bound (device-side count): idle CTAs leave
  if (eblk * kMachThreads >= n_live) return;
  const uint32_t e = eblk * kMachThreads + threadIdx.x;
  const bool active = e < n_live;
  // warps without a live episode (a CTA's tail in small launches) keep the
  // CTA's barrier protocol but skip the automaton: in small or device-sized
  // launches they would otherwise multiply the SM's issue load
  const bool warp_live = __any_sync(0xffffffffu, active);
  const int32_t gq = seg_bound(p, q);
  const int32_t gend = seg_bound(p, q + 1);
  const int32_t g0 = (gq - p.window_tiles > 0 ? gq - p.window_tiles : 0) & ~3;

  EpParams<N> ep = load_episode<N>(p, active ? e : 0);
  if (q == 0 && p.matched) {
    // matched-pair work of the launch (statistics): the first segment's
    // CTAs add their episodes' sum_k events(type_k)
    unsigned long long mp = 0;
    if (active) {
#pragma unroll
      for (int k = 0; k < N; ++k) mp += p.hist[ep.type[k]];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mp += __shfl_xor_sync(0xffffffffu, mp, o);
    if ((threadIdx.x & 31) == 0 && mp) atomicAdd(p.matched, mp);
  }
  Machine<N, Hist> m;
  m.hist.reset(g0, p.hist_words);
  const int64_t tq = static_cast<int64_t>(gq) * 32;
  int64_t s0 = q == 0 ? 0 : tq - static_cast<int64_t>(ep.sigma);
  if (s0 < 0) s0 = 0;
  m.set_threshold(s0 - 1);

  uint32_t cnt = 0, ncomp = 0;
  uint64_t last = ~0ull;
  // first completions are recorded for the concat walk only (P > 1; with one
  // segment the record arrays are not allocated per episode)
  const bool record = active && p.P > 1;
  uint64_t* first = p.f_first + (static_cast<size_t>(q) * p.n_eps + e) * kRecorded;

  uint32_t row_off[N];
#pragma unroll
  for (int k = 0; k < N; ++k) row_off[k] = ep.type[k] * kRowStride;

  const int32_t blk0 = g0 >> 5;
  const int32_t nblk = ((gend - 1) >> 5) - blk0 + 1;

  auto issue = [&](int32_t c) {
    uint64_t* bar = &bars[c % stages];
    dev::fence_proxy_async();
    dev::mbar_arrive_expect_tx(bar, bw * 4u);
    dev::bulk_g2s(stage + static_cast<size_t>(c % stages) * bw,
                  p.occ + static_cast<size_t>(blk0 + c) * bw, bw * 4u, bar);
  };

  if (stages > 0) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < stages; ++s) dev::mbar_init(&bars[s], 1);
      dev::fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int32_t c = 0; c < stages - 1 && c < nblk; ++c) issue(c);
  }

  auto on_c = [&](uint64_t tc) -> bool {
    if (ncomp < kRecorded && record) first[ncomp] = tc;
    ++ncomp;
    if (static_cast<int64_t>(tc) >= tq) {
      ++cnt;
      last = tc;
    }
    return false;
  };

  // One bitmap block: tiles [t0, t1) of block starting at tile gb, rows read
  // through `rd(k, t)` (shared-memory or global flavour).
  auto run_block = [&](int32_t gb, int32_t t0, int32_t t1, auto&& rd4, auto&& rd1) {
    if constexpr (Hist::kQuad) {
      for (int32_t t = t0; t < t1; t += 4) {
        uint4 v[N];
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] = rd4(k, t);
        const int32_t g = gb + t;
        // warp-uniform choice: the masked variant is exact for every lane,
        // so a warp with any lane at or before its threshold tile runs it
        // once instead of diverging into both variants
        if (__any_sync(0xffffffffu, g <= m.thr_tile))
          quad_step<N, Hist, true>(m, ep, v, g, p, on_c);
        else
          quad_step<N, Hist, false>(m, ep, v, g, p, on_c);
      }
    } else {
      for (int32_t t = t0; t < t1; ++t) {
        uint32_t o[N];
#pragma unroll
        for (int k = 0; k < N; ++k) o[k] = rd1(k, t);
        tile_step<N, Hist, true>(m, ep, o, gb + t, p, on_c);
      }
    }
  };

  for (int32_t c = 0; c < nblk; ++c) {
    const int32_t gb = (blk0 + c) * 32;
    const int32_t t0 = g0 > gb ? g0 - gb : 0;
    const int32_t t1 = gend - gb < 32 ? gend - gb : 32;
    if (stages > 0) {
      if (threadIdx.x == 0 && c + stages - 1 < nblk) issue(c + stages - 1);
      dev::mbar_wait(&bars[c % stages], static_cast<uint32_t>(c / stages) & 1u);
      // index the extern __shared__ array directly so the loads are LDS
      const uint32_t sbase = static_cast<uint32_t>(c % stages) * bw;
      if (warp_live)
        run_block(
            gb, t0, t1,
            [&](int k, int32_t t) { return *reinterpret_cast<const uint4*>(&stage[sbase + row_off[k] + t]); },
            [&](int k, int32_t t) { return stage[sbase + row_off[k] + t]; });
      __syncthreads();
    } else if (warp_live) {
      const uint32_t* gbuf = p.occ + static_cast<size_t>(blk0 + c) * bw;
      run_block(
          gb, t0, t1,
          [&](int k, int32_t t) { return __ldg(reinterpret_cast<const uint4*>(gbuf + row_off[k] + t)); },
          [&](int k, int32_t t) { return __ldg(gbuf + row_off[k] + t); });
    }
  }

  if (active) {
    if (p.P == 1) {
      p.counts[out_index(p, e)] = cnt;  // one segment from the stream start: exact, no walk
    } else {
      const size_t idx = static_cast<size_t>(q) * p.n_eps + e;
      p.f_count[idx] = cnt;
      p.f_ncomp[idx] = ncomp;
      p.f_last[idx] = last;
    }
  }
}

// Segment q of episode e entered in RESTART(L) (the previous segment's last
// completion L lies inside q's window): re-run the machine from L, cleared
// with pe = L, only until it provably coincides with the FRESH machine (same
// completion, or both quiet for sum(high)) and read the rest of the segment
// off the FRESH record ("patch", cf. E/mapconcat.hpp:144-148). Returns the
// segment's count and last in-segment completion (~0 if none).
template <int N, class Hist>
__device__ __forceinline__ void patch_segment(const CountLaunch& p, const EpParams<N>& ep, uint32_t e,
                                              int q, uint64_t L, uint32_t fcnt, uint64_t flast,
                                              uint32_t& cnt, uint64_t& last) {
  const int32_t gq = seg_bound(p, q);
  const int32_t gn = seg_bound(p, q + 1);
  const size_t idx = static_cast<size_t>(q) * p.n_eps + e;
  const uint64_t tq = static_cast<uint64_t>(gq) * 32;
  const uint32_t nf = p.f_ncomp[idx];
  const uint32_t nrec = nf < kRecorded ? nf : kRecorded;
  uint64_t first[kRecorded];
#pragma unroll
  for (int j = 0; j < kRecorded; ++j)
    first[j] = j < static_cast<int>(nrec) ? p.f_first[idx * kRecorded + j] : ~0ull;
  Machine<N, Hist> m;
  const int32_t gL = static_cast<int32_t>(L >> 5);
  m.hist.reset(gL, p.hist_words);
  m.set_threshold(static_cast<int64_t>(L));
  uint32_t rc = 0;
  uint64_t rl = ~0ull;
  bool synced = false;
  // Quiet-window sync: once both machines' last clear (R: its restart or
  // last completion; F: its fresh start at the window or its last
  // completion) lies more than sum(high) before T, every live entry at T
  // comes from chains starting in [T - sum(high), T), which both machines
  // hold identically, and pe no longer matters: from T on, R == F.
  const int64_t sigma = static_cast<int64_t>(ep.sigma);
  const int64_t f_start = static_cast<int64_t>(tq) - sigma - 1;  // F admits starts >= window
  int64_t last_r = static_cast<int64_t>(L);
  auto quiet = [&](int64_t T) -> bool {
    if (last_r + sigma >= T) return false;
    if (nf > static_cast<uint32_t>(kRecorded) && static_cast<int64_t>(first[kRecorded - 1]) < T)
      return false;  // F completions before T not all recorded
    int64_t last_f = f_start;
    uint32_t f_before = 0;  // F in-segment completions before T
#pragma unroll
    for (int j = 0; j < kRecorded; ++j)
      if (j < static_cast<int>(nrec) && static_cast<int64_t>(first[j]) < T) {
        last_f = static_cast<int64_t>(first[j]);
        if (first[j] >= tq) ++f_before;
      }
    if (last_f + sigma >= T) return false;
    const uint32_t rest = fcnt - f_before;
    cnt = rc + rest;
    last = rest ? flast : rl;
    return true;
  };
  auto on_c = [&](uint64_t tc) -> bool {
    if (tc >= tq) {
      ++rc;
      rl = tc;
    }
    last_r = static_cast<int64_t>(tc);
    uint32_t inseg = 0;
#pragma unroll
    for (int j = 0; j < kRecorded; ++j) {
      if (j < static_cast<int>(nrec)) {
        if (first[j] >= tq) ++inseg;
        if (first[j] == tc) {
          const uint32_t rest = fcnt - inseg;
          cnt = rc + rest;
          last = rest ? flast : rl;
          synced = true;
          return true;
        }
      }
    }
    return false;
  };
  for (int32_t g = gL; g < gn; ++g) {
    if (g > gL && quiet(static_cast<int64_t>(g) * 32)) {
      synced = true;
      break;
    }
    uint32_t occ[N];
#pragma unroll
    for (int k = 0; k < N; ++k) occ[k] = __ldg(p.occ + occ_index(g, ep.type[k], p.blk_words));
    if (tile_step<N, Hist, true>(m, ep, occ, g, p, on_c)) break;
  }
  if (!synced) {
    cnt = rc;
    last = rl;
  }
}

// Whether segment q's successor starts in RESTART: q has an in-segment
// completion inside the successor's window.
__device__ __forceinline__ bool restarts_next(const CountLaunch& p, int q, uint32_t cnt, uint64_t last,
                                              uint32_t sigma) {
  const int64_t wn = static_cast<int64_t>(seg_bound(p, q + 1)) * 32 - static_cast<int64_t>(sigma);
  return (q + 1 < p.P) && cnt > 0 && static_cast<int64_t>(last) >= wn;
}

// Concat step: one thread per episode chains the P segment records.
template <int N, class Hist>
__global__ void __launch_bounds__(128) walk_kernel(const CountLaunch p) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= live_eps(p)) return;
  const EpParams<N> ep = load_episode<N>(p, e);
  uint64_t total = 0;
  bool restart = false;
  uint64_t L = 0;
  uint32_t patches = 0;
  // Segment records do not depend on the walk state: fetch them kPrefetch
  // segments at a time so the loads overlap instead of serialising.
  constexpr int kPrefetch = 8;
  uint32_t pf_cnt[kPrefetch];
  uint64_t pf_last[kPrefetch];
  for (int q = 0; q < p.P; ++q) {
    if (q % kPrefetch == 0) {
#pragma unroll
      for (int j = 0; j < kPrefetch; ++j) {
        const int qq = q + j;
        const size_t ix = static_cast<size_t>(qq) * p.n_eps + e;
        pf_cnt[j] = qq < p.P ? p.f_count[ix] : 0u;
        pf_last[j] = qq < p.P ? p.f_last[ix] : ~0ull;
      }
    }
    const uint32_t fcnt = pf_cnt[q % kPrefetch];
    const uint64_t flast = pf_last[q % kPrefetch];
    uint32_t cnt = fcnt;
    uint64_t last = flast;
    if (restart) {
      ++patches;
      patch_segment<N, Hist>(p, ep, e, q, L, fcnt, flast, cnt, last);
    }
    total += cnt;
    restart = restarts_next(p, q, cnt, last, ep.sigma);
    L = last;
  }
  p.counts[out_index(p, e)] = total;
  // statistics: one atomic per warp (per-thread atomics on one address
  // serialise in L2)
  const unsigned mask = __activemask();
  const unsigned sum = __reduce_add_sync(mask, patches);
  if (static_cast<int>(threadIdx.x & 31) == __ffs(mask) - 1 && sum)
    atomicAdd(p.patches, static_cast<unsigned long long>(sum));
}

// Concat step, warp-parallel (few episodes, many segments): one warp per
// episode, lane j owns segments j, j+32, ... Every segment's outcome is first
// taken to be its FRESH record; then, in rounds, each segment whose
// predecessor's current outcome ends inside its window is re-patched from
// that completion, until no outcome changes (the chain's fixpoint, i.e. the
// sequential walk's result; usually one or two rounds). The walk's latency
// drops from P dependent steps to a few parallel rounds.
constexpr int kWalkWarpSegs = 4;  // segments per lane (P <= 128)

template <int N, class Hist>
__device__ __forceinline__ void walk_warp_episode(const CountLaunch& p, uint32_t e, int lane) {
  const EpParams<N> ep = load_episode<N>(p, e);
  uint32_t fc[kWalkWarpSegs], cnt[kWalkWarpSegs];
  uint64_t fl[kWalkWarpSegs], last[kWalkWarpSegs], from[kWalkWarpSegs];
#pragma unroll
  for (int i = 0; i < kWalkWarpSegs; ++i) {
    const int q = lane + 32 * i;
    const size_t ix = static_cast<size_t>(q) * p.n_eps + e;
    fc[i] = q < p.P ? p.f_count[ix] : 0u;
    fl[i] = q < p.P ? p.f_last[ix] : ~0ull;
    cnt[i] = fc[i];
    last[i] = fl[i];
    from[i] = ~0ull;  // FRESH
  }
  uint32_t patches = 0;
  for (int round = 0; round <= p.P; ++round) {
    // predecessor outcome of each owned segment (segment q-1 is owned by
    // lane (q-1) & 31, slot (q-1) >> 5)
    bool changed = false;
#pragma unroll
    for (int i = 0; i < kWalkWarpSegs; ++i) {
      const int q = lane + 32 * i;
      const int src_lane = (lane + 31) & 31;
      const int src_slot = lane == 0 ? i - 1 : i;
      uint32_t pc = 0;
      uint64_t pl = 0;
#pragma unroll
      for (int j = 0; j < kWalkWarpSegs; ++j) {
        const uint32_t c_j = __shfl_sync(0xffffffffu, cnt[j], src_lane);
        const uint64_t l_j = __shfl_sync(0xffffffffu, last[j], src_lane);
        if (j == src_slot) {
          pc = c_j;
          pl = l_j;
        }
      }
      const bool rs = q > 0 && q < p.P && restarts_next(p, q - 1, pc, pl, ep.sigma);
      const uint64_t want = rs ? pl : ~0ull;
      if (q < p.P && want != from[i]) {
        uint32_t c2 = fc[i];
        uint64_t l2 = fl[i];
        if (rs) {
          ++patches;
          patch_segment<N, Hist>(p, ep, e, q, pl, fc[i], fl[i], c2, l2);
        }
        changed |= c2 != cnt[i] || l2 != last[i];
        cnt[i] = c2;
        last[i] = l2;
        from[i] = want;
      }
    }
    if (!__any_sync(0xffffffffu, changed)) break;
  }
  uint64_t total = 0;
#pragma unroll
  for (int i = 0; i < kWalkWarpSegs; ++i) total += cnt[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
  if (lane == 0) p.counts[out_index(p, e)] = total;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) patches += __shfl_xor_sync(0xffffffffu, patches, o);
  if (lane == 0 && patches) atomicAdd(p.patches, static_cast<unsigned long long>(patches));
}

template <int N, class Hist>
__global__ void __launch_bounds__(128) walk_warp_kernel(const CountLaunch p) {
  const int lane = static_cast<int>(threadIdx.x & 31);
  const uint32_t n_live = live_eps(p);
  const uint32_t n_warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < n_live; e += n_warps)
    walk_warp_episode<N, Hist>(p, e, lane);
}


inline size_t machines_smem(const CountLaunch& p) {
  return 128 + static_cast<size_t>(p.stages) * p.blk_words * 4;
}

template <int N, class Hist>
void configure_machines() {
  static bool configured = false;
  if (!configured) {
    EPI_CUDA(cudaFuncSetAttribute(machines_kernel<N, Hist>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    configured = true;
  }
}

// With p.occ_query set, report resident map CTAs per SM for this launch
// shape (the segment planner's input) instead of launching.
template <int N, class Hist>
void launch_machines_n(const CountLaunch& p, cudaStream_t st) {
  configure_machines<N, Hist>();
  if (p.occ_query) {
    int blocks = 0;
    EPI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, machines_kernel<N, Hist>,
                                                           kMachThreads, machines_smem(p)));
    *p.occ_query = blocks > 0 ? blocks : 1;
    return;
  }
  // (a time shard launches only its own segments: p.map_segs of them)
  const unsigned segs = static_cast<unsigned>(p.map_segs > 0 ? p.map_segs : p.P);
  const unsigned eblks = (p.n_eps + kMachThreads - 1) / kMachThreads;
  const dim3 grid = p.n_dev ? dim3(segs, eblks) : dim3(eblks, segs);
  machines_kernel<N, Hist><<<grid, kMachThreads, machines_smem(p), st>>>(p);
  EPI_CUDA(cudaGetLastError());
}

template <int N, class Hist>
void launch_walk_n(const CountLaunch& p, cudaStream_t st) {
  if (p.walk_warp && p.P <= 32 * kWalkWarpSegs) {
    // one warp per live episode, grid-stride (the live count may be known
    // only on the device)
    const uint64_t blocks = std::min<uint64_t>((static_cast<uint64_t>(p.n_eps) * 32 + 127) / 128, 4096);
    walk_warp_kernel<N, Hist><<<static_cast<unsigned>(blocks), 128, 0, st>>>(p);
  } else {
    walk_kernel<N, Hist><<<(p.n_eps + 127) / 128, 128, 0, st>>>(p);
  }
  EPI_CUDA(cudaGetLastError());
}

// Runtime N -> template N dispatch for a history policy family H<N>.
template <template <int> class H, int... Ns>
struct Dispatch;

template <template <int> class H>
struct Dispatch<H> {
  static void machines(int, const CountLaunch&, cudaStream_t) {
    throw Error(7, "episode length not supported by the device counter");
  }
  static void walk(int, const CountLaunch&, cudaStream_t) {
    throw Error(7, "episode length not supported by the device counter");
  }
};

template <template <int> class H, int N, int... Rest>
struct Dispatch<H, N, Rest...> {
  static void machines(int n, const CountLaunch& p, cudaStream_t st) {
    if (n == N)
      launch_machines_n<N, H<N>>(p, st);
    else
      Dispatch<H, Rest...>::machines(n, p, st);
  }
  static void walk(int n, const CountLaunch& p, cudaStream_t st) {
    if (n == N)
      launch_walk_n<N, H<N>>(p, st);
    else
      Dispatch<H, Rest...>::walk(n, p, st);
  }
};

template <int W, bool kHi32>
struct NarrowW {
  template <int N>
  using H = NarrowHist<N, W, kHi32>;
};

// Uniform-window-width map kernels (N 2..8, every high <= 32), instantiated
// per W in count_w*.cu so the compile parallelises.
template <int W>
void launch_machines_w(int n, const CountLaunch& p, cudaStream_t st) {
  Dispatch<NarrowW<W, true>::template H, 2, 3, 4, 5, 6, 7, 8>::machines(n, p, st);
}

template <int W>
struct NarrowL {
  template <int N>
  using H = NarrowHist<N, W, true, true>;
};

// Pass-1 map kernels: width W at every position but the last, whose window
// (launch-uniform width <= 16, high <= 32) uses window_last (count_l*.cu).
template <int W>
void launch_machines_l(int n, const CountLaunch& p, cudaStream_t st) {
  Dispatch<NarrowL<W>::template H, 3, 4, 5, 6>::machines(n, p, st);
}
}  // namespace impl
}  // namespace epi
