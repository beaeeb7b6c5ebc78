// Exact counting by greedy scan of the chain-end bitmap, with the chain's
// prefix shared across episodes ("chain" map kernel). Same
// launch interface and segment records as machines_kernel (count_impl.cuh),
// so the MapConcatenate concat walk is unchanged; used for host-sized
// launches whose windows all have the same width W and high <= 32.
//
// For an episode e = tau_0 -w_0- tau_1 ... tau_{N-1} let U_k be the bitmap of
// times at which SOME chain of its first k+1 nodes ends, with no clears:
//   U_0 = occ(tau_0),  U_k = occ(tau_k) & dil_{w_{k-1}}(U_{k-1})
// (dil_w(X)(t) = any X in [t-high, t-low)). run_fsm (E/fsm.hpp:45-106) is
// greedy by earliest end: after a completion at pe it clears every list and
// admits position 0 only at t > pe (E/fsm.hpp:66-68, 83-91), so its next
// completion is the first t > pe with a chain ending at t that starts after
// pe. Such a chain starts in [t - sigma, t - L] (sigma = sum of highs, L = sum
// of (low + 1), the longest and shortest chain spans). Hence, after pe:
//   * U_{N-1} bits in (pe, pe + L] are never completions;
//   * bits after pe + sigma always are (the first one is the next completion);
//   * a bit in (pe + L, pe + sigma] is decided exactly by rebuilding the
//     chain bitmaps from starts after pe over those few tiles
//     (chain_validate).
// The bulk of the work is a pure bitmap AND/dilate chain plus an "any bit"
// test, with no automaton state, masks or clears.
//
// Prefix sharing: the engine sorts the episodes (chain_sort.cu) so that a
// CTA's 256 episodes share few depth-d prefixes (tau_0, w_0, ..., tau_{d-1},
// w_{d-1}). Per staged bitmap block, phase A computes each group's row
// DD = dil_{w_{d-1}}(U_{d-1}) once (one warp per group, lane = tile, the
// previous tile's word by shuffle). Phase B then depends on d:
//   * d = N-1 ("row mode": U_{N-1} = occ(tau_{N-1}) & DD): lane = tile; the
//     warp walks its 32 episodes, one coalesced row load, AND and ballot per
//     (episode, block); the ballots are the per-episode masks of tiles with a
//     chain end, which phase C (lane = episode) turns into completions;
//   * d < N-1 ("chain mode"): lane = episode, four tiles per 16-byte load,
//     the remaining N-1-d dilations per tile, completions taken inline.
// d is chosen per CTA from its group counts with a cost model.
#pragma once

#include <type_traits>

#include "count_impl.cuh"

namespace epi {
namespace impl {

constexpr int kChainGroups = 32;  // max shared prefixes per CTA (phase A rows)
constexpr int kChainMaxN = 8;

template <int N>
struct ChainSmem {
  static constexpr int M = N > 1 ? N - 1 : 1;
  uint32_t gtype[kChainGroups][M];  // prefix rows (type * kRowStride) of the CTA's groups
  uint32_t ghi[kChainGroups][M];
  uint32_t carry[kChainGroups][M];  // U_k word of the previous block's last tile
  uint32_t edge[8][2 * N];          // last lane of each warp: its episode (prefix compare)
  uint32_t wheads[8];
  // row mode: per episode the byte offset of its last type's row in a staged
  // block and of its group's DD row; the per-block ballots
  __align__(16) uint32_t erow[kMachThreads];
  __align__(16) uint32_t egrp[kMachThreads];
  __align__(16) uint32_t nz[2][kMachThreads];
};

inline size_t chain_smem(const CountLaunch& p) {
  // bars + stage ring + DD rows + ChainSmem<N> (bounded by N = kChainMaxN)
  return 128 + static_cast<size_t>(p.stages) * p.blk_words * 4 +
         2 * static_cast<size_t>(kChainGroups) * kRowStride * 4 + sizeof(ChainSmem<kChainMaxN>);
}

// Greedy state of one (episode, segment) machine, times relative to
// T0 = 32 * g0 (the segment's window start; the engine keeps segments short
// enough for 32-bit offsets).
struct ChainState {
  int32_t pe;      // last clear (completion, or the FRESH start - 1)
  int32_t floor;   // bits at or before floor are resolved
  int32_t ready;   // bits in (floor, ready] need the exact check
  uint32_t cnt;    // completions inside the segment
  uint32_t ncomp;  // completions including the window
  int32_t last;    // last in-segment completion (-1: none)
};

template <int N, int W>
struct ChainCtx {
  const CountLaunch& p;
  const EpParams<N>& ep;
  int64_t T0;
  int32_t g0, gend, tq, lsum;
  uint64_t* first;
};

template <int N, int W>
__device__ __forceinline__ void chain_record(const ChainCtx<N, W>& x, ChainState& s, int32_t t) {
  if (s.ncomp < kRecorded && x.first) x.first[s.ncomp] = static_cast<uint64_t>(x.T0 + t);
  ++s.ncomp;
  if (t >= x.tq) {
    ++s.cnt;
    s.last = t;
  }
}

// The next completion after s.pe, when a chain end falls in (pe + L, pe + sigma]:
// run_fsm cleared at pe holds, at position k, exactly the ends of chains of
// the first k+1 nodes that start after pe (E/fsm.hpp:66-68, 83-91), so its
// next completion is the first bit of U'_{N-1}, the chain bitmaps rebuilt
// with U'_0 = occ(tau_0) restricted to (pe, inf). Any chain ending after
// pe + sigma starts after pe, so only tiles up to pe + sigma are rebuilt
// (at most 1 + sigma/32 tiles; the segment's tiles only). One completion per
// call: the caller's greedy continues from it.
template <int N, int W>
__device__ __forceinline__ void chain_validate(const ChainCtx<N, W>& x, ChainState& s) {
  const int64_t start = x.T0 + s.pe + 1;  // first admissible chain start (absolute ms)
  const int64_t lim = x.T0 + s.pe + static_cast<int64_t>(x.ep.sigma);
  int32_t g = static_cast<int32_t>(start >> 5);
  const int32_t gl = static_cast<int32_t>(lim >> 5) + 1 < x.gend ? static_cast<int32_t>(lim >> 5) + 1 : x.gend;
  uint32_t h[N > 1 ? N - 1 : 1];
#pragma unroll
  for (int k = 0; k < N - 1; ++k) h[k] = 0;
  uint32_t u0mask = ~0u << (start & 31);
  for (; g < gl; ++g) {
    uint32_t cw = __ldg(x.p.occ + occ_index(g, x.ep.type[0], x.p.blk_words)) & u0mask;
    u0mask = ~0u;
#pragma unroll
    for (int k = 1; k < N; ++k) {
      const uint32_t hi = x.ep.hi[k - 1];
      const uint32_t o = __ldg(x.p.occ + occ_index(g, x.ep.type[k], x.p.blk_words));
      const uint32_t nx = o & window_any<W, true>(cw, h[k - 1], 0u, hi - W + 1, hi);
      h[k - 1] = cw;
      cw = nx;
    }
    if (cw) {
      const int32_t t = 32 * (g - x.g0) + (__ffs(cw) - 1);
      chain_record(x, s, t);
      s.pe = t;
      s.floor = t + x.lsum;
      s.ready = t + static_cast<int32_t>(x.ep.sigma);
      return;
    }
  }
  // no chain from after pe ends by pe + sigma: the first chain end after it
  // is the next completion
  s.floor = s.pe + static_cast<int32_t>(x.ep.sigma);
  s.ready = s.floor;
}

// Completions among the chain ends of one tile word (tile base `base`,
// relative ms), in time order.
template <int N, int W>
__device__ __forceinline__ void chain_word(const ChainCtx<N, W>& x, ChainState& s, uint32_t w, int32_t base) {
  auto above = [&](int32_t f) -> uint32_t {  // bits of this tile after time f
    const int32_t d = f - base;
    return d < 0 ? ~0u : (d >= 31 ? 0u : (~0u << (d + 1)));
  };
  w &= above(s.floor);
  while (w) {
    const int32_t t = base + (__ffs(w) - 1);
    if (t > s.ready) {
      chain_record(x, s, t);
      s.pe = t;
      s.floor = t + x.lsum;
      s.ready = t + static_cast<int32_t>(x.ep.sigma);
    } else {
      chain_validate<N, W>(x, s);
    }
    w &= above(s.floor);
  }
}

template <int N, int W>
__global__ void __launch_bounds__(kMachThreads) chain_kernel(const CountLaunch p) {
  static_assert(N >= 2 && N <= kChainMaxN, "chain kernel: 2..8 nodes");
  constexpr int M = N - 1;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint32_t* stage = reinterpret_cast<uint32_t*>(smem + 128);
  const uint32_t bw = p.blk_words;
  const int stages = p.stages;
  uint32_t* dd = stage + static_cast<size_t>(stages) * bw;
  ChainSmem<N>& cs = *reinterpret_cast<ChainSmem<N>*>(dd + 2 * kChainGroups * kRowStride);
  const bool bound = p.bound_only != 0;
  const uint32_t stage_s = dev::smem_addr(stage);  // shared-window addresses
  const uint32_t dd_s = dev::smem_addr(dd);

  const int q = static_cast<int>(blockIdx.y) + p.q_base;
  const uint32_t eblk = blockIdx.x;
  const uint32_t n_live = p.n_eps;
  const int tid = static_cast<int>(threadIdx.x), lane = tid & 31, warp = tid >> 5;
  const uint32_t e = eblk * kMachThreads + tid;
  const bool active = e < n_live;
  const int32_t gq = seg_bound(p, q);
  const int32_t gend = seg_bound(p, q + 1);
  const int32_t g0 = (gq - p.window_tiles > 0 ? gq - p.window_tiles : 0) & ~3;

  const EpParams<N> ep = load_episode<N>(p, active ? e : (n_live ? n_live - 1 : 0));
  if (q == 0 && p.matched) {
    unsigned long long mp = 0;
    if (active) {
#pragma unroll
      for (int k = 0; k < N; ++k) mp += p.hist[ep.type[k]];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mp += __shfl_xor_sync(0xffffffffu, mp, o);
    if (lane == 0 && mp) atomicAdd(p.matched, mp);
  }

  // ---- prologue: group heads per prefix depth, choice of d ----------------
  if (lane == 31) {
#pragma unroll
    for (int k = 0; k < N; ++k) cs.edge[warp][k] = ep.type[k];
#pragma unroll
    for (int k = 0; k < M; ++k) cs.edge[warp][N + k] = ep.hi[k];
  }
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) dev::mbar_init(&bars[s], 1);
    dev::fence_barrier_init();
  }
  __syncthreads();
  bool same = tid > 0;  // same depth-d prefix as the previous thread
  uint32_t heads_at[N];
#pragma unroll
  for (int d = 1; d < N; ++d) {
    const uint32_t pt = __shfl_up_sync(0xffffffffu, ep.type[d - 1], 1);
    const uint32_t ph = __shfl_up_sync(0xffffffffu, ep.hi[d - 1], 1);
    const uint32_t qt = lane == 0 && warp > 0 ? cs.edge[warp - 1][d - 1] : pt;
    const uint32_t qh = lane == 0 && warp > 0 ? cs.edge[warp - 1][N + d - 1] : ph;
    same = same && qt == ep.type[d - 1] && qh == ep.hi[d - 1];
    heads_at[d] = active && !same ? 1u : 0u;
  }
  heads_at[0] = 0;
  // Per-CTA cost model, warp-instructions per staged block: phase A costs
  // ceil(G_d / 8) group rows of d levels; phase B for d < N-1 is 8 quads of
  // the remaining N-1-d dilations and the test, for d = N-1 about 8
  // instructions per (episode, block) over the warp's 32 episodes.
  int dsel = 0;
  {
    const int force = p.chain_depth - 1;  // test knob: chain_depth = d + 1 forces depth d
    float best = 8.0f * (12.0f + 36.0f * M);
    bool forced = force == 0;
#pragma unroll
    for (int d = 1; d < N; ++d) {
      const int G = __syncthreads_count(heads_at[d]);
      const float b = d == M ? 32.0f * 8.0f : 8.0f * (14.0f + 36.0f * (M - d));
      const float cost = static_cast<float>((G + 7) / 8) * (12.0f * d + 8.0f) + b;
      if (G <= kChainGroups && d == force) {
        dsel = d;
        forced = true;
      }
      if (G <= kChainGroups && cost < best && !forced) {
        best = cost;
        dsel = d;
      }
    }
  }
  uint32_t head = 0;
#pragma unroll
  for (int d = 1; d < N; ++d)
    if (d == dsel) head = heads_at[d];
  const uint32_t bal = __ballot_sync(0xffffffffu, head);
  if (lane == 0) cs.wheads[warp] = __popc(bal);
  __syncthreads();
  uint32_t before = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kMachThreads / 32; ++w) {
    const uint32_t c = cs.wheads[w];
    before += w < warp ? c : 0u;
    total += c;
  }
  const int grp = static_cast<int>(before + __popc(bal & ((2u << lane) - 1u))) - 1;
  const int G = dsel > 0 ? static_cast<int>(total) : 0;
  if (dsel > 0 && head) {
#pragma unroll
    for (int k = 0; k < M; ++k) {
      cs.gtype[grp][k] = ep.type[k] * kRowStride;
      cs.ghi[grp][k] = ep.hi[k];
      cs.carry[grp][k] = 0;
    }
  }
  // row mode: the warp's episodes fall into runs of one group (sorted): the
  // run heads (segmask) let phase B load each run's DD word once
  const uint32_t my_go = static_cast<uint32_t>(grp > 0 ? grp : 0) * kRowStride * 4u;
  const uint32_t my_ro = ep.type[N - 1] * kRowStride * 4u;
  // (the shuffle runs on every lane: a full-mask shuffle inside the
  // short-circuit below would leave lanes out of the exchange)
  const uint32_t prev_go = __shfl_up_sync(0xffffffffu, my_go, 1);
  const uint32_t segmask = __ballot_sync(0xffffffffu, active && (lane == 0 || prev_go != my_go));
  if (dsel == M) {
    cs.erow[tid] = my_ro;
    cs.egrp[tid] = my_go;
  }

  // ---- per-segment greedy state ---------------------------------------------
  const int64_t T0 = static_cast<int64_t>(g0) * 32;
  uint32_t lsum = 0;
#pragma unroll
  for (int k = 0; k < M; ++k) lsum += ep.lo1[k];
  const ChainCtx<N, W> cx{p, ep, T0, g0, gend, 32 * (gq - g0), static_cast<int32_t>(lsum),
                          // first completions feed the concat walk only (P > 1)
                          p.P > 1 && active ? p.f_first + (static_cast<size_t>(q) * p.n_eps + e) * kRecorded
                                            : nullptr};
  ChainState st;
  {
    const int64_t tqa = static_cast<int64_t>(gq) * 32;
    int64_t s0 = q == 0 ? 0 : tqa - static_cast<int64_t>(ep.sigma);
    if (s0 < 0) s0 = 0;
    st.pe = static_cast<int32_t>(s0 - 1 - T0);
    // U is built from tile g0 with empty history: it holds every chain that
    // starts at or after 32*g0 <= s0; the FRESH machine admits only chains
    // starting at >= s0 (none start earlier when s0 == 0)
    st.floor = s0 == 0 ? -1 : st.pe + static_cast<int32_t>(lsum);
    st.ready = s0 == 0 ? -1 : st.pe + static_cast<int32_t>(ep.sigma);
  }
  st.cnt = 0;
  st.ncomp = 0;
  st.last = -1;

  const int32_t blk0 = g0 >> 5;
  const int32_t nblk = ((gend - 1) >> 5) - blk0 + 1;
  auto issue = [&](int32_t c) {
    uint64_t* bar = &bars[c % stages];
    dev::fence_proxy_async();
    dev::mbar_arrive_expect_tx(bar, bw * 4u);
    dev::bulk_g2s(stage + static_cast<size_t>(c % stages) * bw, p.occ + static_cast<size_t>(blk0 + c) * bw,
                  bw * 4u, bar);
  };
  // Row mode with >= 4 stages takes two bitmap blocks per iteration (half the
  // per-block bookkeeping, one row-table read per two blocks): the ring then
  // runs stages - 2 blocks ahead.
  const bool pair = dsel == M && stages >= 4;
  const int ahead = pair ? stages - 2 : stages - 1;
  __syncthreads();  // group table written; barriers initialised
  if (tid == 0)
    for (int32_t c = 0; c < ahead && c < nblk; ++c) issue(c);
  // episodes of this warp (row mode walks them with lane = tile)
  const int wbase = warp * 32;
  const int nact = static_cast<int>(n_live) - (static_cast<int>(eblk) * kMachThreads + wbase) < 32
                       ? max(0, static_cast<int>(n_live) - (static_cast<int>(eblk) * kMachThreads + wbase))
                       : 32;

  auto phase_a = [&](auto dtag, uint32_t sbase_s, int32_t t0, uint32_t* ddw) {
    constexpr int D = decltype(dtag)::value;
    for (int gi = warp; gi < G; gi += kMachThreads / 32) {
      const bool live = lane >= t0;
      uint32_t x = live ? dev::lds_u32(sbase_s + (cs.gtype[gi][0] + lane) * 4u) : 0u;
      uint32_t nc[D];
      nc[0] = x;
#pragma unroll
      for (int k = 1; k < D; ++k) {
        uint32_t prev = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane == 0) prev = cs.carry[gi][k - 1];
        const uint32_t hi = cs.ghi[gi][k - 1];
        const uint32_t o = live ? dev::lds_u32(sbase_s + (cs.gtype[gi][k] + lane) * 4u) : 0u;
        x = o & window_any<W, true>(x, prev, 0u, hi - W + 1, hi);
        nc[k] = x;
      }
      uint32_t prev = __shfl_up_sync(0xffffffffu, x, 1);
      if (lane == 0) prev = cs.carry[gi][D - 1];
      const uint32_t hi = cs.ghi[gi][D - 1];
      ddw[gi * kRowStride + lane] = window_any<W, true>(x, prev, 0u, hi - W + 1, hi);
      __syncwarp();
      if (lane == 31) {
#pragma unroll
        for (int k = 0; k < D; ++k) cs.carry[gi][k] = nc[k];
      }
    }
  };

  auto run = [&](auto dtag) {
    constexpr int D = decltype(dtag)::value;
    // chain mode: lane's rows from position D on, the history of its
    // remaining dilations
    uint32_t h[M];
#pragma unroll
    for (int k = 0; k < M; ++k) h[k] = 0;
    const uint32_t grow4 = static_cast<uint32_t>(grp > 0 ? grp : 0) * kRowStride * 4u;

    if constexpr (D == M) {
      if (pair) {
        for (int32_t c = 0; c < nblk; c += 2) {
          const bool two = c + 1 < nblk;
          if (tid == 0) {
            if (c + ahead < nblk) issue(c + ahead);
            if (c + ahead + 1 < nblk) issue(c + ahead + 1);
          }
          int32_t gbs[2], t0s[2], t1s[2];
          uint32_t sb[2];
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int32_t cb = two ? c + b : c;
            gbs[b] = (blk0 + cb) * 32;
            t0s[b] = g0 > gbs[b] ? g0 - gbs[b] : 0;
            t1s[b] = gend - gbs[b] < 32 ? gend - gbs[b] : 32;
            sb[b] = stage_s + static_cast<uint32_t>(cb % stages) * bw * 4u;
          }
          dev::mbar_wait(&bars[c % stages], static_cast<uint32_t>(c / stages) & 1u);
          if (two) dev::mbar_wait(&bars[(c + 1) % stages], static_cast<uint32_t>((c + 1) / stages) & 1u);
          phase_a(dtag, sb[0], t0s[0], dd);
          if (two) phase_a(dtag, sb[1], t0s[1], dd + kChainGroups * kRowStride);
          __syncthreads();
          // phase B, lane = tile, both blocks per row-table read
          const uint32_t l0 = sb[0] + lane * 4u, l1 = sb[1] + lane * 4u;
          const uint32_t d0 = dd_s + lane * 4u, d1 = d0 + kChainGroups * kRowStride * 4u;
          const uint32_t m0 = lane >= t0s[0] && lane < t1s[0] ? ~0u : 0u;
          const uint32_t m1 = two && lane >= t0s[1] && lane < t1s[1] ? ~0u : 0u;
          // runs of one group: the run's DD words once, then per episode
          // its last type's row (offset by shuffle) AND DD and a ballot
          uint32_t* nz0 = &cs.nz[0][wbase];
          uint32_t* nz1 = &cs.nz[1][wbase];
          for (uint32_t sm = segmask; sm;) {
            const int s0 = __ffs(sm) - 1;
            sm &= sm - 1u;
            const int s1 = sm ? __ffs(sm) - 1 : nact;
            const uint32_t go = __shfl_sync(0xffffffffu, my_go, s0);
            const uint32_t dA = dev::lds_u32(d0 + go) & m0;
            const uint32_t dB = dev::lds_u32(d1 + go) & m1;
            int j = s0;
            for (; j + 1 < s1; j += 2) {
              const uint32_t r0 = __shfl_sync(0xffffffffu, my_ro, j);
              const uint32_t r1 = __shfl_sync(0xffffffffu, my_ro, j + 1);
              const uint32_t a0 = __ballot_sync(0xffffffffu, (dev::lds_u32(l0 + r0) & dA) != 0u);
              const uint32_t b0 = __ballot_sync(0xffffffffu, (dev::lds_u32(l1 + r0) & dB) != 0u);
              const uint32_t a1 = __ballot_sync(0xffffffffu, (dev::lds_u32(l0 + r1) & dA) != 0u);
              const uint32_t b1 = __ballot_sync(0xffffffffu, (dev::lds_u32(l1 + r1) & dB) != 0u);
              if (lane == 0) {
                nz0[j] = a0;
                nz1[j] = b0;
                nz0[j + 1] = a1;
                nz1[j + 1] = b1;
              }
            }
            if (j < s1) {
              const uint32_t r0 = __shfl_sync(0xffffffffu, my_ro, j);
              const uint32_t a0 = __ballot_sync(0xffffffffu, (dev::lds_u32(l0 + r0) & dA) != 0u);
              const uint32_t b0 = __ballot_sync(0xffffffffu, (dev::lds_u32(l1 + r0) & dB) != 0u);
              if (lane == 0) {
                nz0[j] = a0;
                nz1[j] = b0;
              }
            }
          }
          __syncwarp();
          // phase C, lane = episode: block c's chain ends, then block c+1's
          if (active) {
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              uint32_t mine = cs.nz[b][tid];
              const uint32_t ro4 = sb[b] + cs.erow[tid];
              const uint32_t go4 = dd_s + b * kChainGroups * kRowStride * 4u + cs.egrp[tid];
              const int32_t base_rel = gbs[b] - g0;
              while (mine) {
                const int t = __ffs(mine) - 1;
                mine &= mine - 1u;
                const uint32_t w = dev::lds_u32(ro4 + t * 4u) & dev::lds_u32(go4 + t * 4u);
                if (bound)
                  st.cnt += 32 * (base_rel + t) >= cx.tq ? __popc(w) : 0u;
                else
                  chain_word<N, W>(cx, st, w, 32 * (base_rel + t));
              }
            }
          }
          __syncthreads();  // stage slots and DD rows free for reuse
        }
        return;
      }
    }
    for (int32_t c = 0; c < nblk; ++c) {
      const int32_t gb = (blk0 + c) * 32;
      const int32_t t0 = g0 > gb ? g0 - gb : 0;
      const int32_t t1 = gend - gb < 32 ? gend - gb : 32;
      if (tid == 0 && c + ahead < nblk) issue(c + ahead);
      dev::mbar_wait(&bars[c % stages], static_cast<uint32_t>(c / stages) & 1u);
      const uint32_t sbase_s = stage_s + static_cast<uint32_t>(c % stages) * bw * 4u;
      if constexpr (D > 0) {
        phase_a(dtag, sbase_s, t0, dd);
        __syncthreads();
      }
      const int32_t base_rel = gb - g0 * 1;  // tile offset of this block from g0
      if constexpr (D == M) {
        // row mode, phase B: lane = tile; chunks of 4 episodes, their row
        // offsets read by broadcast, one coalesced row load + AND + ballot
        // per (episode, block); lane 0 stores the 4 ballots
        const bool in_rng = lane >= t0 && lane < t1;
        const uint32_t lane_s = sbase_s + lane * 4u, dlane_s = dd_s + lane * 4u;
        const uint32_t erow_s = dev::smem_addr(&cs.erow[wbase]), egrp_s = dev::smem_addr(&cs.egrp[wbase]);
        // (lanes outside [t0, t1) read word 0 of the rows, masked away)
        const uint32_t msk = in_rng ? ~0u : 0u;
        for (int j = 0; j < nact; j += 4) {
          const uint4 ro = dev::lds_v4(erow_s + j * 4u);
          const uint4 go = dev::lds_v4(egrp_s + j * 4u);
          uint4 m;
          m.x = __ballot_sync(0xffffffffu, (dev::lds_u32(lane_s + ro.x) & dev::lds_u32(dlane_s + go.x) & msk) != 0u);
          m.y = __ballot_sync(0xffffffffu, (dev::lds_u32(lane_s + ro.y) & dev::lds_u32(dlane_s + go.y) & msk) != 0u);
          m.z = __ballot_sync(0xffffffffu, (dev::lds_u32(lane_s + ro.z) & dev::lds_u32(dlane_s + go.z) & msk) != 0u);
          m.w = __ballot_sync(0xffffffffu, (dev::lds_u32(lane_s + ro.w) & dev::lds_u32(dlane_s + go.w) & msk) != 0u);
          if (lane == 0) *reinterpret_cast<uint4*>(&cs.nz[0][wbase + j]) = m;
        }
        __syncwarp();
        // phase C: lane = episode, its chain-end tiles in time order
        if (active) {
          uint32_t mine = cs.nz[0][tid];
          const uint32_t ro4 = sbase_s + cs.erow[tid];
          const uint32_t go4 = dd_s + cs.egrp[tid];
          while (mine) {
            const int t = __ffs(mine) - 1;
            mine &= mine - 1u;
            const uint32_t w = dev::lds_u32(ro4 + t * 4u) & dev::lds_u32(go4 + t * 4u);
            if (bound)
              st.cnt += 32 * (base_rel + t) >= cx.tq ? __popc(w) : 0u;
            else
              chain_word<N, W>(cx, st, w, 32 * (base_rel + t));
          }
        }
      } else if (nact > 0) {
        // chain mode: lane = episode, four tiles per 16-byte load
        uint32_t ra[N];
#pragma unroll
        for (int k = 0; k < N; ++k) ra[k] = sbase_s + ep.type[k] * kRowStride * 4u + t0 * 4u;
        uint32_t da = dd_s + grow4 + t0 * 4u;
        // chain-end words are queued (two per lane, in time order) and taken
        // through the greedy after the block, when every lane's queue is
        // drained together instead of once per lane that has a chain end
        uint32_t qw0 = 0, qw1 = 0;
        int32_t qt0 = 0, qt1 = 0;
        int qn = 0;
        auto quads = [&](auto btag) {
          constexpr bool kBound = decltype(btag)::value;
          for (int32_t t = t0; t < t1; t += 4) {
            uint4 v[N];
#pragma unroll
            for (int k = D; k < N; ++k) v[k] = dev::lds_v4(ra[k]);
            uint4 dv = make_uint4(0, 0, 0, 0);
            if constexpr (D > 0) dv = dev::lds_v4(da);
#pragma unroll
            for (int k = D; k < N; ++k) ra[k] += 16u;
            da += 16u;
            uint32_t u[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              auto pick = [&](const uint4& a) { return j == 0 ? a.x : j == 1 ? a.y : j == 2 ? a.z : a.w; };
              uint32_t cw = D > 0 ? (pick(v[D]) & pick(dv)) : pick(v[0]);
#pragma unroll
              for (int k = D + 1; k < N; ++k) {
                const uint32_t hi = ep.hi[k - 1];
                const uint32_t nx = pick(v[k]) & window_any<W, true>(cw, h[k - 1], 0u, hi - W + 1, hi);
                h[k - 1] = cw;
                cw = nx;
              }
              u[j] = cw;
            }
            if constexpr (kBound) {
              if (32 * (base_rel + t) >= cx.tq)  // the segment proper (the quad is 4-aligned)
                st.cnt += __popc(u[0]) + __popc(u[1]) + __popc(u[2]) + __popc(u[3]);
            } else if ((u[0] | u[1] | u[2] | u[3]) && active) {
              uint32_t wm = (u[0] ? 1u : 0u) | (u[1] ? 2u : 0u) | (u[2] ? 4u : 0u) | (u[3] ? 8u : 0u);
              while (wm) {
                const int j = __ffs(wm) - 1;
                wm &= wm - 1u;
                const uint32_t w = j == 0 ? u[0] : j == 1 ? u[1] : j == 2 ? u[2] : u[3];
                const int32_t base = 32 * (base_rel + t + j);
                if (qn == 0) {
                  qw0 = w;
                  qt0 = base;
                  qn = 1;
                } else if (qn == 1) {
                  qw1 = w;
                  qt1 = base;
                  qn = 2;
                } else {
                  // queue full (dense streams): drain it, then this word
                  chain_word<N, W>(cx, st, qw0, qt0);
                  chain_word<N, W>(cx, st, qw1, qt1);
                  chain_word<N, W>(cx, st, w, base);
                  qn = 0;
                }
              }
            }
          }
        };
        if (bound)
          quads(std::true_type{});
        else
          quads(std::false_type{});
        if (qn > 0) {
          chain_word<N, W>(cx, st, qw0, qt0);
          if (qn > 1) chain_word<N, W>(cx, st, qw1, qt1);
        }
      }
      __syncthreads();  // stage slot and DD rows free for reuse
    }
  };
  switch (dsel) {
    case 0: run(std::integral_constant<int, 0>{}); break;
    case 1: if constexpr (N > 1) run(std::integral_constant<int, 1>{}); break;
    case 2: if constexpr (N > 2) run(std::integral_constant<int, (N > 2 ? 2 : 0)>{}); break;
    case 3: if constexpr (N > 3) run(std::integral_constant<int, (N > 3 ? 3 : 0)>{}); break;
    case 4: if constexpr (N > 4) run(std::integral_constant<int, (N > 4 ? 4 : 0)>{}); break;
    case 5: if constexpr (N > 5) run(std::integral_constant<int, (N > 5 ? 5 : 0)>{}); break;
    case 6: if constexpr (N > 6) run(std::integral_constant<int, (N > 6 ? 6 : 0)>{}); break;
    default: if constexpr (N > 7) run(std::integral_constant<int, (N > 7 ? 7 : 0)>{}); break;
  }

  if (active && bound) {
    // upper bound: the chain ends of every segment proper add up
    if (st.cnt) atomicAdd(reinterpret_cast<unsigned long long*>(p.counts + out_index(p, e)), st.cnt);
  } else if (active) {
    if (p.P == 1) {
      p.counts[out_index(p, e)] = st.cnt;
    } else {
      const size_t idx = static_cast<size_t>(q) * p.n_eps + e;
      p.f_count[idx] = st.cnt;
      p.f_ncomp[idx] = st.ncomp;
      p.f_last[idx] = st.last >= 0 ? static_cast<uint64_t>(T0 + st.last) : ~0ull;
    }
  }
}

template <int N, int W>
void launch_chain_n(const CountLaunch& p, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    EPI_CUDA(cudaFuncSetAttribute(chain_kernel<N, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    configured = true;
  }
  const size_t sm = chain_smem(p);
  if (p.occ_query) {
    int blocks = 0;
    EPI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, chain_kernel<N, W>, kMachThreads, sm));
    *p.occ_query = blocks > 0 ? blocks : 1;
    return;
  }
  const unsigned segs = static_cast<unsigned>(p.map_segs > 0 ? p.map_segs : p.P);
  const unsigned eblks = (p.n_eps + kMachThreads - 1) / kMachThreads;
  chain_kernel<N, W><<<dim3(eblks, segs), kMachThreads, sm, st>>>(p);
  EPI_CUDA(cudaGetLastError());
}

template <int W>
bool launch_chain_w(int n, const CountLaunch& p, cudaStream_t st) {
  switch (n) {
    case 2: launch_chain_n<2, W>(p, st); return true;
    case 3: launch_chain_n<3, W>(p, st); return true;
    case 4: launch_chain_n<4, W>(p, st); return true;
    case 5: launch_chain_n<5, W>(p, st); return true;
    case 6: launch_chain_n<6, W>(p, st); return true;
    case 7: launch_chain_n<7, W>(p, st); return true;
    case 8: launch_chain_n<8, W>(p, st); return true;
  }
  return false;
}

}  // namespace impl
}  // namespace epi
