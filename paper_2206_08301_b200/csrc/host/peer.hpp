// Peer-memory rendezvous of the ranks of one job on one node.
//
// The reference's ranks are loop indices in one address space
// (proj/src/executor.cpp:213); its "collectives" read the other ranks' blocks
// directly (allreduce, executor.cpp:80-108; apply_plan,
// redistribute.cpp:185-206).  On one B200 node the same direct access exists
// between GPUs: every GPU maps every peer's HBM over NVLink/NVSwitch.  A
// PeerComm gives a rank
//   * a host barrier (no kernel ever waits on another rank's kernel: each
//     rank synchronises its own stream, then meets the others on the host),
//   * the exchange of device buffers: CUDA IPC handles between processes
//     (one process per GPU, or several processes on one GPU in the tests),
//     raw pointers between the host threads of one process (einplan_run_json
//     with one thread per GPU; peer access enabled between distinct devices).
// Shared state lives in a named POSIX shared-memory segment (processes) or
// in one heap object shared by the threads.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

namespace einplan {
namespace gpu {

constexpr int kMaxPeers = 64;

struct PeerHeader {
  std::atomic<std::uint32_t> arrived;
  std::atomic<std::uint32_t> generation;
  std::atomic<std::uint32_t> aborted;
  std::uint32_t pad[13];
  struct Slot {
    cudaIpcMemHandle_t handle;
    std::uint64_t ptr;
    std::int32_t device;
    std::int32_t valid;
  } slot[kMaxPeers];
};

class PeerShared {
 public:
  // one process per rank: the named segment (created by whichever rank comes
  // first; the name is unlinked once every rank has attached)
  static std::shared_ptr<PeerShared> attach_shm(const std::string& name, int nranks);
  // the host threads of one process
  static std::shared_ptr<PeerShared> for_threads(int nranks);
  ~PeerShared();
  PeerShared(const PeerShared&) = delete;
  PeerShared& operator=(const PeerShared&) = delete;

  int nranks() const { return nranks_; }
  bool ipc() const { return ipc_; }
  PeerHeader* header() { return hdr_; }
  double timeout_s() const { return timeout_s_; }
  const std::string& name() const { return name_; }
  void abort();  // wake every waiter with an error (a rank failed)

 private:
  PeerShared() = default;
  PeerHeader* hdr_ = nullptr;
  int nranks_ = 0;
  bool ipc_ = false;
  std::string name_;
  double timeout_s_ = 600.0;
};

class PeerComm {
 public:
  PeerComm(std::shared_ptr<PeerShared> shared, int rank);
  int rank() const { return rank_; }
  int nranks() const { return shared_->nranks(); }
  bool ipc() const { return shared_->ipc(); }
  // all ranks meet; throws after the timeout or when a rank aborted
  void barrier();
  // Collective: every rank passes its buffer (a cudaMalloc base pointer, or
  // nullptr); returns every rank's buffer as a pointer usable on this rank's
  // current device (element rank() is `mine`).
  std::vector<char*> exchange(void* mine);
  // release what exchange() mapped (IPC handles); not collective
  void unmap(std::vector<char*>& peers);
  void abort() { shared_->abort(); }

 private:
  std::shared_ptr<PeerShared> shared_;
  int rank_;
};

}  // namespace gpu
}  // namespace einplan
