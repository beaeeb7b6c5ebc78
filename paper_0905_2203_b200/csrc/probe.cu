// INT32 issue-rate microbenchmark: the roofline denominator for the integer
// counting kernels (MEASURED_PEAKS.json has no integer peak). Every thread
// runs independent chains of LOP3 (ALU pipe) and IMAD (FMA pipe) so both
// integer pipes are saturated; the result is lane-ops per second.
#include "../../include/episodic_b200.h"
#include "common.cuh"

namespace epi {
namespace {

constexpr int kProbeIters = 4096;
constexpr int kChains = 8;

template <bool kMixed>
__global__ void __launch_bounds__(256) int32_probe_kernel(uint32_t seed, uint32_t* sink) {
  uint32_t a[kChains], b[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    a[c] = seed * (threadIdx.x + c + 1);
    b[c] = seed ^ (blockIdx.x * 977u + c);
  }
  for (int i = 0; i < kProbeIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(b[c]), "r"(seed));
      if (kMixed)
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(b[c]) : "r"(seed), "r"(a[c]));
      else
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x1e;" : "+r"(b[c]) : "r"(a[c]), "r"(seed));
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) x ^= a[c] ^ b[c];
  if (x == 0x12345678u) sink[0] = x;
}

// POPC issue rate (XU pipe): the denominator of the pass-1 bound kernel
// (one POPC per candidate per 32 ms tile word). Each chain step is one POPC
// fed through one LOP3 (ALU pipe, not the bottleneck); POPCs are counted.
__global__ void __launch_bounds__(256) popc_probe_kernel(uint32_t seed, uint32_t* sink) {
  uint32_t a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) a[c] = seed * (threadIdx.x + c + 1);
  for (int i = 0; i < kProbeIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      uint32_t t;
      asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(t) : "r"(a[c]), "r"(seed), "r"(i));
      asm volatile("popc.b32 %0, %1;" : "=r"(a[c]) : "r"(t));
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) x ^= a[c];
  if (x == 0x12345678u) sink[0] = x;
}

}  // namespace
}  // namespace epi

extern "C" epi_status epi_probe_int32(int device, int mixed, double* tops_out) {
  try {
    EPI_CUDA(cudaSetDevice(device));
    int sms = 0;
    EPI_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    uint32_t* sink = nullptr;
    EPI_CUDA(cudaMalloc(&sink, 4));
    cudaEvent_t e0, e1;
    EPI_CUDA(cudaEventCreate(&e0));
    EPI_CUDA(cudaEventCreate(&e1));
    const int blocks = sms * 8;
    auto launch = [&] {
      if (mixed == 2)
        epi::popc_probe_kernel<<<blocks, 256>>>(0x9e3779b9u, sink);
      else if (mixed)
        epi::int32_probe_kernel<true><<<blocks, 256>>>(0x9e3779b9u, sink);
      else
        epi::int32_probe_kernel<false><<<blocks, 256>>>(0x9e3779b9u, sink);
    };
    launch();
    EPI_CUDA(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      EPI_CUDA(cudaEventRecord(e0));
      launch();
      EPI_CUDA(cudaEventRecord(e1));
      EPI_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      EPI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    const double ops = static_cast<double>(blocks) * 256 * epi::kProbeIters * epi::kChains * (mixed == 2 ? 1 : 2);
    *tops_out = ops / (best * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    return EPI_OK;
  } catch (const epi::Error& e) {
    return static_cast<epi_status>(e.status);
  }
}
