// Multi-device contexts: see multi.h. NCCL is loaded at run time
// (libnccl.so.2): the library itself has no link-time NCCL dependency, and a
// process that already loaded NCCL (e.g. through PyTorch) shares that copy.
#include "multi.h"

#include <dlfcn.h>

#include <cstdlib>
#include <exception>
#include <thread>

namespace epi {
namespace {

// The few NCCL entry points used (nccl.h, stable C ABI).
using nccl_result = int;  // ncclResult_t, ncclSuccess == 0
constexpr int kNcclUint8 = 1;  // ncclDataType_t ncclUint8
struct NcclApi {
  void* lib = nullptr;
  nccl_result (*comm_init_all)(void** comms, int ndev, const int* devlist) = nullptr;
  nccl_result (*all_gather)(const void* send, void* recv, size_t count, int dtype, void* comm,
                            cudaStream_t st) = nullptr;
  nccl_result (*comm_destroy)(void* comm) = nullptr;
  const char* (*error_string)(nccl_result) = nullptr;
  bool ok() const { return comm_init_all && all_gather && comm_destroy; }
};

NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    if (std::getenv("EPI_NO_NCCL")) return a;
    a.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.lib) return a;
    a.comm_init_all = reinterpret_cast<decltype(a.comm_init_all)>(dlsym(a.lib, "ncclCommInitAll"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(a.lib, "ncclAllGather"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.lib, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.lib, "ncclGetErrorString"));
    return a;
  }();
  return api;
}

}  // namespace

MultiGroup::MultiGroup(Engine& rank0, const std::vector<int>& devices) : rank0_(rank0), devices_(devices) {
  const int G = world();
  int count = 0;
  EPI_CUDA(cudaGetDeviceCount(&count));
  for (int d : devices_)
    if (d < 0 || d >= count) throw Error(EPI_EINVAL, "epi_create_multi: no such CUDA device");
  for (int r = 1; r < G; ++r) others_.push_back(std::make_unique<Engine>(devices_[r]));
  bool distinct = true;
  for (int a = 0; a < G; ++a)
    for (int b = a + 1; b < G; ++b) distinct = distinct && devices_[a] != devices_[b];
  NcclApi& api = nccl_api();
  if (G > 1 && distinct && api.ok()) {
    comms_.assign(G, nullptr);
    const nccl_result rc = api.comm_init_all(comms_.data(), G, devices_.data());
    if (rc != 0) {
      comms_.clear();
    } else {
      nccl_ = true;
    }
  }
  send_.assign(G, nullptr);
  recv_.assign(G, nullptr);
  done_.assign(G, nullptr);
  for (int r = 0; r < G; ++r) {
    EPI_CUDA(cudaSetDevice(devices_[r]));
    EPI_CUDA(cudaEventCreateWithFlags(&done_[r], cudaEventDisableTiming));
    users_.push_back({this, r});
  }
  if (!nccl_ && G > 1) {
    // direct peer access where the topology allows it (copies work either way)
    for (int a = 0; a < G; ++a)
      for (int b = 0; b < G; ++b) {
        if (devices_[a] == devices_[b]) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, devices_[a], devices_[b]);
        if (can) {
          cudaSetDevice(devices_[a]);
          cudaDeviceEnablePeerAccess(devices_[b], 0);
          cudaGetLastError();  // already enabled is fine
        }
      }
  }
  EPI_CUDA(cudaSetDevice(devices_[0]));
}

MultiGroup::~MultiGroup() {
  NcclApi& api = nccl_api();
  for (void* c : comms_)
    if (c && api.comm_destroy) api.comm_destroy(c);
  for (size_t r = 0; r < done_.size(); ++r)
    if (done_[r]) {
      cudaSetDevice(devices_[r]);
      cudaEventDestroy(done_[r]);
    }
}

bool MultiGroup::barrier() {
  std::unique_lock<std::mutex> lk(mu_);
  if (abort_) return false;
  const uint64_t g = gen_;
  if (++arrived_ == world()) {
    arrived_ = 0;
    ++gen_;
    cv_.notify_all();
    return true;
  }
  cv_.wait(lk, [&] { return gen_ != g || abort_; });
  return !abort_;
}

int MultiGroup::allgather_cb(void* user, const void* send, void* recv, uint64_t bytes, void* stream) {
  auto* u = static_cast<RankUser*>(user);
  return u->g->allgather(u->r, send, recv, bytes, static_cast<cudaStream_t>(stream));
}

// Every rank's `bytes` slice lands at recv + rank * bytes on every rank,
// ordered on each rank's stream.
int MultiGroup::allgather(int r, const void* send, void* recv, uint64_t bytes, cudaStream_t st) {
  if (nccl_) {
    return nccl_api().all_gather(send, recv, static_cast<size_t>(bytes), kNcclUint8, comms_[r], st) == 0 ? 0 : 1;
  }
  send_[r] = send;
  recv_[r] = recv;
  if (!barrier()) return 1;
  // push this rank's slice into every rank's receive buffer
  for (int q = 0; q < world(); ++q) {
    char* dst = static_cast<char*>(recv_[q]) + static_cast<size_t>(r) * bytes;
    if (cudaMemcpyPeerAsync(dst, devices_[q], send, devices_[r], bytes, st) != cudaSuccess) return 1;
  }
  if (cudaEventRecord(done_[r], st) != cudaSuccess) return 1;
  if (!barrier()) return 1;
  for (int q = 0; q < world(); ++q)
    if (cudaStreamWaitEvent(st, done_[q], 0) != cudaSuccess) return 1;
  // nobody re-records its event before every rank has enqueued its waits
  return barrier() ? 0 : 1;
}

void MultiGroup::run(const std::function<void(int, const epi_shard&)>& f, uint64_t min_shard) {
  const int G = world();
  {
    std::lock_guard<std::mutex> lk(mu_);
    abort_ = false;
    arrived_ = 0;
  }
  std::vector<std::exception_ptr> errs(G);
  int first = -1;  // the rank that failed first (the others may then fail in the exchange)
  auto body = [&](int r) {
    try {
      cudaSetDevice(devices_[r]);
      const epi_shard sh{static_cast<uint32_t>(r), static_cast<uint32_t>(G), min_shard, &MultiGroup::allgather_cb,
                         &users_[r]};
      f(r, sh);
    } catch (...) {
      errs[r] = std::current_exception();
      std::lock_guard<std::mutex> lk(mu_);
      if (first < 0) first = r;
      abort_ = true;
      cv_.notify_all();
    }
  };
  std::vector<std::thread> th;
  for (int r = 1; r < G; ++r) th.emplace_back(body, r);
  body(0);
  for (auto& t : th) t.join();
  cudaSetDevice(devices_[0]);
  if (first >= 0) std::rethrow_exception(errs[first]);
}

}  // namespace epi
