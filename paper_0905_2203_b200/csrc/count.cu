// Exact non-overlapped episode counting on sm_100a: a bit-sliced counting
// automaton, run segment-parallel (MapConcatenate) and stitched by a
// per-episode concat walk.
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
//   C_k = occ(tau_k) & OR_{a=low+1..high} (C_{k-1} : H1_{k-1} : H2_{k-1}) << a
//
// where H1/H2 are the entry bitmaps of the two previous tiles (high <= 63).
// The first set bit of C_{N-1} is a completion; the tile is then recomputed
// above it with empty history (the reference's list clear). Rare, so the
// loop is off the hot path.
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
// only until it completes at a time where the FRESH machine also completed -
// from there both are identical, so the rest of the segment is read off the
// FRESH record ("patch", cf. E/mapconcat.hpp:144-148).
#include "common.cuh"
#include "count.h"

namespace epi {
namespace {

constexpr int kMachThreads = 256;
constexpr int kStages = 3;
constexpr uint32_t kStageBytes = 8192;

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
    uint32_t w = N > 1 ? p.ep_win[static_cast<size_t>(e) * (N - 1) + k] : 0x0101u;
    ep.lo1[k] = w & 0xff;
    ep.hi[k] = (w >> 8) & 0xff;
  }
  ep.sigma = p.ep_sigma[e];
  return ep;
}

template <int N>
struct Machine {
  static constexpr int M = N > 1 ? N - 1 : 1;
  uint32_t h1[M];
  uint32_t h2[M];
  int32_t thr_tile;   // position 0 admits only times > thr:
  uint32_t thr_mask;  // tiles < thr_tile none, tile == thr_tile thr_mask

  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int k = 0; k < M; ++k) h1[k] = h2[k] = 0;
  }
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

// Window test for one position: bit i set iff an entry of the previous
// position lies at age a in [lo1, hi] from time 32*g + i.
__device__ __forceinline__ uint32_t dilate(uint32_t c, uint32_t h1, uint32_t h2, uint32_t lo1,
                                           uint32_t hi) {
  uint32_t d = 0;
  const uint32_t e1 = hi < 32u ? hi : 32u;
  for (uint32_t a = lo1; a <= e1; ++a) d |= __funnelshift_lc(h1, c, a);
  for (uint32_t a = lo1 > 33u ? lo1 : 33u; a <= hi; ++a) d |= __funnelshift_lc(h2, h1, a - 32);
  return d;
}

// Advance one tile. on_completion(time) returns true to stop the machine.
template <int N, class OnC>
__device__ __forceinline__ bool tile_step(Machine<N>& m, const EpParams<N>& ep,
                                          const uint32_t (&occ)[N], int32_t g, OnC&& on_c) {
  uint32_t C[N];
  C[0] = occ[0];
  if (g <= m.thr_tile) C[0] &= (g < m.thr_tile) ? 0u : m.thr_mask;
#pragma unroll
  for (int k = 1; k < N; ++k)
    C[k] = occ[k] & dilate(C[k - 1], m.h1[k - 1], m.h2[k - 1], ep.lo1[k - 1], ep.hi[k - 1]);
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
      for (int k = 1; k < N; ++k) C[k] = occ[k] & dilate(C[k - 1], 0u, 0u, ep.lo1[k - 1], ep.hi[k - 1]);
      last = C[N - 1];
    } while (last);
#pragma unroll
    for (int k = 0; k < N - 1; ++k) m.h1[k] = 0;  // the clear also empties older history
  }
#pragma unroll
  for (int k = 0; k < N - 1; ++k) {
    m.h2[k] = m.h1[k];
    m.h1[k] = C[k];
  }
  return false;
}

// Map step: FRESH machine of (episode, segment). Tiles of the segment (plus
// its window) are staged through shared memory with bulk copies; every
// thread of the CTA walks the same tiles, so one staged row serves all 256
// episodes of the block.
template <int N>
__global__ void __launch_bounds__(kMachThreads) machines_kernel(const CountLaunch p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint32_t* stage = reinterpret_cast<uint32_t*>(smem + 128);
  const uint32_t a_pad = p.a_pad;
  const uint32_t ch = static_cast<uint32_t>(p.chunk_tiles);
  const uint32_t stage_words = ch * a_pad;

  const int q = blockIdx.y;
  const uint32_t e = blockIdx.x * kMachThreads + threadIdx.x;
  const bool active = e < p.n_eps;
  const int32_t gq = p.seg_g[q];
  const int32_t gend = p.seg_g[q + 1];
  const int32_t g0 = gq - p.window_tiles > 0 ? gq - p.window_tiles : 0;

  EpParams<N> ep = load_episode<N>(p, active ? e : 0);
  Machine<N> m;
  m.clear();
  const int64_t tq = static_cast<int64_t>(gq) * 32;
  int64_t s0 = q == 0 ? 0 : tq - static_cast<int64_t>(ep.sigma);
  if (s0 < 0) s0 = 0;
  m.set_threshold(s0 - 1);

  uint32_t cnt = 0, ncomp = 0;
  uint64_t last = ~0ull;
  uint64_t* first = p.f_first + (static_cast<size_t>(q) * p.n_eps + e) * kRecorded;

  const int32_t total_tiles = gend - g0;
  const int32_t nchunks = (total_tiles + static_cast<int32_t>(ch) - 1) / static_cast<int32_t>(ch);

  auto issue = [&](int32_t c) {
    const int32_t tg = g0 + c * static_cast<int32_t>(ch);
    int32_t nt = gend - tg;
    if (nt > static_cast<int32_t>(ch)) nt = static_cast<int32_t>(ch);
    const uint32_t bytes = static_cast<uint32_t>(nt) * a_pad * 4u;
    uint64_t* bar = &bars[c % kStages];
    dev::fence_proxy_async();
    dev::mbar_arrive_expect_tx(bar, bytes);
    dev::bulk_g2s(stage + static_cast<size_t>(c % kStages) * stage_words,
                  p.occ + static_cast<size_t>(tg) * a_pad, bytes, bar);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) dev::mbar_init(&bars[s], 1);
    dev::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int32_t c = 0; c < kStages - 1 && c < nchunks; ++c) issue(c);

  auto on_c = [&](uint64_t tc) -> bool {
    if (ncomp < kRecorded && active) first[ncomp] = tc;
    ++ncomp;
    if (static_cast<int64_t>(tc) >= tq) {
      ++cnt;
      last = tc;
    }
    return false;
  };

  for (int32_t c = 0; c < nchunks; ++c) {
    if (threadIdx.x == 0 && c + kStages - 1 < nchunks) issue(c + kStages - 1);
    dev::mbar_wait(&bars[c % kStages], static_cast<uint32_t>(c / kStages) & 1u);
    const uint32_t* buf = stage + static_cast<size_t>(c % kStages) * stage_words;
    const int32_t tg = g0 + c * static_cast<int32_t>(ch);
    int32_t nt = gend - tg;
    if (nt > static_cast<int32_t>(ch)) nt = static_cast<int32_t>(ch);
    for (int32_t t = 0; t < nt; ++t) {
      const uint32_t* row = buf + static_cast<size_t>(t) * a_pad;
      uint32_t occ[N];
#pragma unroll
      for (int k = 0; k < N; ++k) occ[k] = row[ep.type[k]];
      tile_step<N>(m, ep, occ, tg + t, on_c);
    }
    __syncthreads();
  }

  if (active) {
    const size_t idx = static_cast<size_t>(q) * p.n_eps + e;
    p.f_count[idx] = cnt;
    p.f_ncomp[idx] = ncomp;
    p.f_last[idx] = last;
  }
}

// Concat step: one thread per episode chains the P segment records.
template <int N>
__global__ void __launch_bounds__(128) walk_kernel(const CountLaunch p) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p.n_eps) return;
  const EpParams<N> ep = load_episode<N>(p, e);
  uint64_t total = 0;
  bool restart = false;
  uint64_t L = 0;
  uint32_t patches = 0;
  for (int q = 0; q < p.P; ++q) {
    const int32_t gq = p.seg_g[q];
    const int32_t gn = p.seg_g[q + 1];
    const size_t idx = static_cast<size_t>(q) * p.n_eps + e;
    const uint32_t fcnt = p.f_count[idx];
    const uint64_t flast = p.f_last[idx];
    uint32_t cnt = fcnt;
    uint64_t last = flast;
    if (restart) {
      ++patches;
      const uint64_t tq = static_cast<uint64_t>(gq) * 32;
      const uint32_t nf = p.f_ncomp[idx];
      const uint32_t nrec = nf < kRecorded ? nf : kRecorded;
      uint64_t first[kRecorded];
#pragma unroll
      for (int j = 0; j < kRecorded; ++j)
        first[j] = j < static_cast<int>(nrec) ? p.f_first[idx * kRecorded + j] : ~0ull;
      Machine<N> m;
      m.clear();
      m.set_threshold(static_cast<int64_t>(L));
      uint32_t rc = 0;
      uint64_t rl = ~0ull;
      bool synced = false;
      auto on_c = [&](uint64_t tc) -> bool {
        if (tc >= tq) {
          ++rc;
          rl = tc;
        }
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
      for (int32_t g = static_cast<int32_t>(L >> 5); g < gn; ++g) {
        const uint32_t* row = p.occ + static_cast<size_t>(g) * p.a_pad;
        uint32_t occ[N];
#pragma unroll
        for (int k = 0; k < N; ++k) occ[k] = __ldg(row + ep.type[k]);
        if (tile_step<N>(m, ep, occ, g, on_c)) break;
      }
      if (!synced) {
        cnt = rc;
        last = rl;
      }
    }
    total += cnt;
    const int64_t wn = static_cast<int64_t>(gn) * 32 - static_cast<int64_t>(ep.sigma);
    restart = (q + 1 < p.P) && cnt > 0 && static_cast<int64_t>(last) >= wn;
    L = last;
  }
  p.counts[e] = total;
  if (patches) atomicAdd(p.patches, static_cast<unsigned long long>(patches));
}

template <int N>
void launch_n(const CountLaunch& p, cudaStream_t st) {
  const uint32_t stage_words = static_cast<uint32_t>(p.chunk_tiles) * p.a_pad;
  const size_t smem = 128 + static_cast<size_t>(kStages) * stage_words * 4;
  static bool configured = false;
  if (!configured) {
    EPI_CUDA(cudaFuncSetAttribute(machines_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024));
    configured = true;
  }
  dim3 grid((p.n_eps + kMachThreads - 1) / kMachThreads, p.P);
  machines_kernel<N><<<grid, kMachThreads, smem, st>>>(p);
  EPI_CUDA(cudaGetLastError());
}

template <int N>
void launch_walk_n(const CountLaunch& p, cudaStream_t st) {
  walk_kernel<N><<<(p.n_eps + 127) / 128, 128, 0, st>>>(p);
  EPI_CUDA(cudaGetLastError());
}

template <int... Ns>
struct Dispatch;

template <>
struct Dispatch<> {
  static void machines(int, const CountLaunch&, cudaStream_t) {
    throw Error(7, "episode length not supported by the device counter");
  }
  static void walk(int, const CountLaunch&, cudaStream_t) {
    throw Error(7, "episode length not supported by the device counter");
  }
};

template <int N, int... Rest>
struct Dispatch<N, Rest...> {
  static void machines(int n, const CountLaunch& p, cudaStream_t st) {
    if (n == N)
      launch_n<N>(p, st);
    else
      Dispatch<Rest...>::machines(n, p, st);
  }
  static void walk(int n, const CountLaunch& p, cudaStream_t st) {
    if (n == N)
      launch_walk_n<N>(p, st);
    else
      Dispatch<Rest...>::walk(n, p, st);
  }
};

using AllN = Dispatch<1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>;

}  // namespace

uint32_t chunk_tiles_for(uint32_t a_pad) {
  uint32_t row = a_pad * 4u;
  uint32_t ch = kStageBytes / row;
  return ch ? ch : 1u;
}

void launch_machines(int n_nodes, const CountLaunch& p, cudaStream_t st) {
  AllN::machines(n_nodes, p, st);
}

void launch_walk(int n_nodes, const CountLaunch& p, cudaStream_t st) { AllN::walk(n_nodes, p, st); }

}  // namespace epi
