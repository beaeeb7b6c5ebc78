// Multi-device contexts (epi_create_multi): one Engine per device of the
// process, the candidate sets sharded over them through the engines' shard
// contract (epi_shard), the per-level all-gather done by NCCL or by
// device-to-device copies. See include/episodic_b200.h.
#pragma once

#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <vector>

#include "engine.h"

namespace epi {

class MultiGroup {
 public:
  // rank0 is the context's own engine (device devices[0]); the others are
  // created here.
  MultiGroup(Engine& rank0, const std::vector<int>& devices);
  ~MultiGroup();
  int world() const { return static_cast<int>(devices_.size()); }
  bool nccl() const { return nccl_; }
  Engine& rank(int r) { return r == 0 ? rank0_ : *others_[r - 1]; }
  // Runs f(rank, shard) on every rank concurrently (one host thread each);
  // rethrows the first failure.
  void run(const std::function<void(int, const epi_shard&)>& f, uint64_t min_shard);

 private:
  static int allgather_cb(void* user, const void* send, void* recv, uint64_t bytes, void* stream);
  int allgather(int r, const void* send, void* recv, uint64_t bytes, cudaStream_t st);
  bool barrier();  // false: a rank failed (abort)

  Engine& rank0_;
  std::vector<int> devices_;
  std::vector<std::unique_ptr<Engine>> others_;
  bool nccl_ = false;
  std::vector<void*> comms_;  // ncclComm_t
  // device-copy exchange
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  uint64_t gen_ = 0;
  bool abort_ = false;
  std::vector<const void*> send_;
  std::vector<void*> recv_;
  std::vector<cudaEvent_t> done_;
  struct RankUser {
    MultiGroup* g;
    int r;
  };
  std::vector<RankUser> users_;
};

}  // namespace epi
