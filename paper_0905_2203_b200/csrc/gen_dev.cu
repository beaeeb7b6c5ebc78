// Device-side synthetic generator: generate() (E/datagen.hpp:71-122)
// bit-exact, straight into the context's stream.
//
// Per neuron the reference draws from Rng(splitmix64(seed ^ (0x42 + neuron)))
// (std::mt19937_64 raw output, uniform01 = ((x >> 11) + 1) * 2^-53,
// exponential = -log(u) / rate) and accumulates the spike times
// sequentially in double precision: t = e1, then t += e_k while t < duration,
// each event at (int64)(t * 1000). One CTA per neuron reproduces that stream:
// the 312-word mt19937_64 state lives in shared memory and is twisted by the
// CTA in two parallel phases (the words a phase reads are never the ones it
// writes), every thread tempers one word and computes its gap, and one
// thread accumulates the gaps in the reference's order (floating-point
// addition is not associative, so the sum stays sequential; it is ~8 cycles
// per event). Events are written as sort keys (time << tb | neuron); the
// embedded episodes (few events, host-generated exactly as generate() does)
// join them, and one device radix sort yields the reference's
// (time, type) order.
#include <cub/device/device_radix_sort.cuh>

#include <cmath>
#include <vector>

#include "common.cuh"
#include "engine.h"

namespace epi {

void generate_embedded_events(uint32_t neurons, double duration_s, uint64_t seed, const epi_episode_batch* emb,
                              const double* rates, std::vector<uint32_t>& types, std::vector<int64_t>& times);
void bursty_plan(uint32_t electrodes, double duration_s, double base_rate_hz, double rate_sigma,
                 double burst_rate_hz, double burst_min_ms, double burst_max_ms, double burst_gain, uint64_t seed,
                 std::vector<double>& rates, std::vector<double>& burst_lo, std::vector<double>& burst_hi);

namespace {

constexpr int kMtN = 312, kMtM = 156;
constexpr int kGenThreads = 320;
constexpr uint64_t kMatrixA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull;

__host__ __device__ inline uint64_t splitmix64_d(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__device__ __forceinline__ uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

__global__ void __launch_bounds__(kGenThreads)
    poisson_kernel(uint64_t seed, double duration_s, double rate, uint32_t tb, uint64_t cap, uint64_t* keys,
                   unsigned long long* counts, unsigned int* overflow) {
  __shared__ uint64_t mt[kMtN];
  __shared__ double gap[kMtN];
  __shared__ int done;
  const uint32_t neuron = blockIdx.x;
  const int tid = threadIdx.x;
  if (tid == 0) {
    // std::mt19937_64 seeding
    mt[0] = splitmix64_d(seed ^ (0x42ull + neuron));
    for (int i = 1; i < kMtN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
    done = 0;
  }
  __syncthreads();
  uint64_t* out = keys + static_cast<uint64_t>(neuron) * cap;
  double t = 0.0;
  uint64_t cnt = 0;
  bool first = true;
  for (;;) {
    // twist, phase 1: words 0..155 from old words (i + 1, i + 156)
    uint64_t nv = 0;
    if (tid < kMtN - kMtM) {
      const uint64_t x = (mt[tid] & kUpper) | (mt[tid + 1] & kLower);
      nv = mt[tid + kMtM] ^ (x >> 1) ^ ((x & 1ull) ? kMatrixA : 0ull);
    }
    __syncthreads();
    if (tid < kMtN - kMtM) mt[tid] = nv;
    __syncthreads();
    // phase 2: words 156..311 from old word i + 1 (word 0 is new for i = 311)
    // and new word i - 156
    if (tid >= kMtN - kMtM && tid < kMtN) {
      const uint64_t x = (mt[tid] & kUpper) | (mt[(tid + 1) % kMtN] & kLower);
      nv = mt[tid - (kMtN - kMtM)] ^ (x >> 1) ^ ((x & 1ull) ? kMatrixA : 0ull);
    }
    __syncthreads();
    if (tid >= kMtN - kMtM && tid < kMtN) mt[tid] = nv;
    __syncthreads();
    if (tid < kMtN) {
      const double u = (static_cast<double>(temper(mt[tid]) >> 11) + 1.0) * 0x1.0p-53;
      gap[tid] = -log(u) / rate;
    }
    __syncthreads();
    if (tid == 0) {
      for (int i = 0; i < kMtN; ++i) {
        t = first ? gap[i] : t + gap[i];
        first = false;
        if (!(t < duration_s)) {
          done = 1;
          break;
        }
        const uint64_t ms = static_cast<uint64_t>(static_cast<int64_t>(t * 1000.0));
        if (cnt < cap) out[cnt] = (ms << tb) | neuron;
        ++cnt;
      }
    }
    __syncthreads();
    if (done) break;
  }
  if (tid == 0) {
    counts[neuron] = cnt;
    if (cnt > cap) atomicOr(overflow, 1u);
  }
}

// generate_bursty (datagen.cpp) per electrode: the first
// two draws went into the electrode's rate (computed on the host), then the
// background Poisson process at rate r until the duration, then, burst after
// burst, extra events at r * (gain - 1) inside each burst window - one draw
// stream, consumed in exactly that order.
__global__ void __launch_bounds__(kGenThreads)
    bursty_kernel(uint64_t seed, double duration_s, const double* __restrict__ rates, double gain,
                  const double* __restrict__ blo, const double* __restrict__ bhi, uint32_t nb, uint32_t tb, uint64_t cap,
                  uint64_t* keys, unsigned long long* counts, unsigned int* overflow) {
  __shared__ uint64_t mt[kMtN];
  __shared__ double gbg[kMtN], gbu[kMtN];
  __shared__ int done;
  const uint32_t el = blockIdx.x;
  const int tid = threadIdx.x;
  const double r = rates[el];
  const double extra = r * (gain - 1.0);
  if (tid == 0) {
    mt[0] = splitmix64_d(seed ^ (0xB0B5ull + el));
    for (int i = 1; i < kMtN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
    done = 0;
  }
  __syncthreads();
  uint64_t* out = keys + static_cast<uint64_t>(el) * cap;
  // sequential state (thread 0): phase 0 background, 1 bursts, 2 done
  int phase = 0, skip = 2;
  bool first = true, bstart = true;
  double t = 0.0, s_t = 0.0;
  uint32_t bi = 0;
  uint64_t cnt = 0;
  auto push = [&](double x) {
    const uint64_t ms = static_cast<uint64_t>(static_cast<int64_t>(x * 1000.0));
    if (cnt < cap) out[cnt] = (ms << tb) | el;
    ++cnt;
  };
  for (;;) {
    uint64_t nv = 0;
    if (tid < kMtN - kMtM) {
      const uint64_t x = (mt[tid] & kUpper) | (mt[tid + 1] & kLower);
      nv = mt[tid + kMtM] ^ (x >> 1) ^ ((x & 1ull) ? kMatrixA : 0ull);
    }
    __syncthreads();
    if (tid < kMtN - kMtM) mt[tid] = nv;
    __syncthreads();
    if (tid >= kMtN - kMtM && tid < kMtN) {
      const uint64_t x = (mt[tid] & kUpper) | (mt[(tid + 1) % kMtN] & kLower);
      nv = mt[tid - (kMtN - kMtM)] ^ (x >> 1) ^ ((x & 1ull) ? kMatrixA : 0ull);
    }
    __syncthreads();
    if (tid >= kMtN - kMtM && tid < kMtN) mt[tid] = nv;
    __syncthreads();
    if (tid < kMtN) {
      const double u = (static_cast<double>(temper(mt[tid]) >> 11) + 1.0) * 0x1.0p-53;
      const double lg = -log(u);
      gbg[tid] = lg / r;                           // exponential(r)
      gbu[tid] = extra > 0 ? lg / extra : 0.0;     // exponential(extra)
    }
    __syncthreads();
    if (tid == 0) {
      for (int i = skip; i < kMtN && phase < 2; ++i) {
        if (phase == 0) {
          t = first ? gbg[i] : t + gbg[i];
          first = false;
          if (!(t < duration_s)) {
            phase = extra > 0 && nb > 0 ? 1 : 2;
            continue;
          }
          push(t);
        } else {
          s_t = bstart ? blo[bi] + gbu[i] : s_t + gbu[i];
          bstart = false;
          if (!(s_t < bhi[bi])) {
            bstart = true;
            if (++bi == nb) phase = 2;
            continue;
          }
          push(s_t);
        }
      }
      skip = 0;
      if (phase == 2) done = 1;
    }
    __syncthreads();
    if (done) break;
  }
  if (tid == 0) {
    counts[el] = cnt;
    if (cnt > cap) atomicOr(overflow, 1u);
  }
}

__global__ void decode_keys_kernel(const uint64_t* __restrict__ keys, uint64_t n, uint32_t tb, uint32_t* types,
                                   int64_t* times) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  types[i] = static_cast<uint32_t>(k & ((1ull << tb) - 1));
  times[i] = static_cast<int64_t>(k >> tb);
}

inline size_t align256(size_t x) { return (x + 255) / 256 * 256; }

constexpr size_t kSlotGen = 62;      // engine scratch slots (see engine.cpp's slot map)
constexpr size_t kSlotGenPlan = 63;

}  // namespace

// Key layout, sort and load shared by both device generators: `launch`
// fills keys [0, units * cap) (per-unit event counts into counts[], an
// overflow flag into *ovf) on the engine stream; the embedded events join at
// the end; one radix sort over the key bits orders (time, type).
template <class Launch>
void gen_finish(Engine& eng, DeviceScratch& scratch, DeviceStream& stream, cudaStream_t st, uint32_t units,
                uint32_t alphabet, uint64_t cap, int64_t max_ms, const std::vector<uint32_t>& et,
                const std::vector<int64_t>& etm, uint64_t& h2d, Launch&& launch) {
  uint32_t tb = 1;
  while ((1ull << tb) < alphabet) ++tb;
  for (int64_t x : etm) max_ms = std::max(max_ms, x);
  uint32_t time_bits = 1;
  while ((1ull << time_bits) <= static_cast<uint64_t>(max_ms) + 1) ++time_bits;
  const uint32_t key_bits = time_bits + tb;
  if (key_bits > 64) throw Error(EPI_EUNSUPPORTED, "generate: stream span too long for the device generator");
  const uint64_t ne = et.size();
  for (int attempt = 0;; ++attempt) {
    const uint64_t slots = static_cast<uint64_t>(units) * cap + ne;
    if (slots >= (1ull << 31)) throw Error(EPI_EUNSUPPORTED, "generate: more than 2^31 event slots on the device");
    size_t temp_bytes = 0;
    EPI_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, temp_bytes, static_cast<const uint64_t*>(nullptr),
                                            static_cast<uint64_t*>(nullptr), static_cast<int>(slots), 0,
                                            static_cast<int>(key_bits)));
    const size_t o_a = 0, o_b = align256(slots * 8), o_cnt = o_b + align256(slots * 8),
                 o_tmp = o_cnt + align256((units + 1) * 8ull), total = o_tmp + align256(temp_bytes);
    char* d = scratch.get<char>(kSlotGen, total);
    uint64_t* ka = reinterpret_cast<uint64_t*>(d + o_a);
    uint64_t* kb = reinterpret_cast<uint64_t*>(d + o_b);
    unsigned long long* counts = reinterpret_cast<unsigned long long*>(d + o_cnt);
    unsigned int* ovf = reinterpret_cast<unsigned int*>(counts + units);
    // all-ones keys sort after every event key over the key bits
    EPI_CUDA(cudaMemsetAsync(ka, 0xff, slots * 8, st));
    EPI_CUDA(cudaMemsetAsync(ovf, 0, 4, st));
    launch(tb, cap, ka, counts, ovf);
    EPI_CUDA(cudaGetLastError());
    if (ne) {
      std::vector<uint64_t> ek(ne);
      for (uint64_t i = 0; i < ne; ++i) ek[i] = (static_cast<uint64_t>(etm[i]) << tb) | et[i];
      EPI_CUDA(cudaMemcpyAsync(ka + static_cast<uint64_t>(units) * cap, ek.data(), ne * 8, cudaMemcpyHostToDevice, st));
    }
    std::vector<unsigned long long> hc(units + 1);
    EPI_CUDA(cudaMemcpyAsync(hc.data(), counts, (units + 1) * 8ull, cudaMemcpyDeviceToHost, st));
    EPI_CUDA(cudaStreamSynchronize(st));
    if (reinterpret_cast<const unsigned int*>(&hc[units])[0] != 0) {
      if (attempt >= 3) throw Error(EPI_EUNSUPPORTED, "generate: per-unit event capacity exceeded");
      cap *= 2;
      continue;
    }
    uint64_t n = ne;
    for (uint32_t i = 0; i < units; ++i) n += hc[i];
    cub::DoubleBuffer<uint64_t> db(ka, kb);
    size_t tb_bytes = temp_bytes;
    EPI_CUDA(cub::DeviceRadixSort::SortKeys(d + o_tmp, tb_bytes, db, static_cast<int>(slots), 0,
                                            static_cast<int>(key_bits), st));
    stream.reserve_raw(n);
    if (n)
      decode_keys_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(db.Current(), n, tb,
                                                                                  stream.d_types_raw,
                                                                                  stream.d_times_raw);
    EPI_CUDA(cudaGetLastError());
    h2d = ne * 8;
    stream.load(n, alphabet, st, scratch);
    (void)eng;
    return;
  }
}

void Engine::generate_stream_device(uint32_t neurons, double duration_s, double base_rate_hz, uint64_t seed,
                                    const epi_episode_batch* emb, const double* rates) {
  if (neurons < 1) throw Error(EPI_EINVAL, "generate: need at least one neuron");
  if (duration_s < 0) throw Error(EPI_EINVAL, "generate: negative duration");
  if (!(base_rate_hz > 0)) throw Error(EPI_EINVAL, "generate: base rate must be > 0");
  // embedded episodes: host, exactly as generate() (validates them too)
  std::vector<uint32_t> et;
  std::vector<int64_t> etm;
  generate_embedded_events(neurons, duration_s, seed, emb, rates, et, etm);
  const double lambda = base_rate_hz * duration_s;  // per neuron: mean + 10 sigma
  const uint64_t cap = static_cast<uint64_t>(lambda + 10.0 * std::sqrt(lambda) + 1024.0);
  csr_valid_ = false;
  gen_finish(*this, scratch_, stream_, st_, neurons, neurons, cap, static_cast<int64_t>(duration_s * 1000.0) + 1,
             et, etm, last_load_h2d,
             [&](uint32_t tb, uint64_t c, uint64_t* keys, unsigned long long* counts, unsigned int* ovf) {
               poisson_kernel<<<neurons, kGenThreads, 0, st_>>>(seed, duration_s, base_rate_hz, tb, c, keys, counts,
                                                                ovf);
             });
}

void Engine::generate_bursty_device(uint32_t electrodes, double duration_s, double base_rate_hz, double rate_sigma,
                                    double burst_rate_hz, double burst_min_ms, double burst_max_ms, double burst_gain,
                                    uint64_t seed, const epi_episode_batch* emb, const double* rates) {
  std::vector<double> er, blo, bhi;
  bursty_plan(electrodes, duration_s, base_rate_hz, rate_sigma, burst_rate_hz, burst_min_ms, burst_max_ms,
              burst_gain, seed, er, blo, bhi);
  std::vector<uint32_t> et;
  std::vector<int64_t> etm;
  generate_embedded_events(electrodes, duration_s, seed, emb, rates, et, etm);
  // capacity: the busiest electrode's background + burst events, + 10 sigma
  double burst_s = 0;
  for (size_t b = 0; b < blo.size(); ++b) burst_s += bhi[b] - blo[b];
  double rmax = 0;
  for (double r : er) rmax = std::max(rmax, r);
  const double lambda = rmax * duration_s + rmax * (burst_gain - 1.0) * burst_s;
  const uint64_t cap = static_cast<uint64_t>(lambda + 10.0 * std::sqrt(lambda) + 1024.0);
  // plan arrays on the device (rates, burst windows)
  const size_t nb = blo.size();
  std::vector<double> plan(electrodes + 2 * nb);
  std::copy(er.begin(), er.end(), plan.begin());
  std::copy(blo.begin(), blo.end(), plan.begin() + electrodes);
  std::copy(bhi.begin(), bhi.end(), plan.begin() + electrodes + nb);
  double* d_plan = scratch_.get<double>(kSlotGenPlan, plan.size() + 1);
  EPI_CUDA(cudaMemcpyAsync(d_plan, plan.data(), plan.size() * 8, cudaMemcpyHostToDevice, st_));
  csr_valid_ = false;
  gen_finish(*this, scratch_, stream_, st_, electrodes, electrodes, cap,
             static_cast<int64_t>(duration_s * 1000.0) + 1, et, etm, last_load_h2d,
             [&](uint32_t tb, uint64_t c, uint64_t* keys, unsigned long long* counts, unsigned int* ovf) {
               bursty_kernel<<<electrodes, kGenThreads, 0, st_>>>(seed, duration_s, d_plan, burst_gain,
                                                                  d_plan + electrodes, d_plan + electrodes + nb,
                                                                  static_cast<uint32_t>(nb), tb, c, keys, counts, ovf);
             });
  last_load_h2d += plan.size() * 8;
}

}  // namespace epi
