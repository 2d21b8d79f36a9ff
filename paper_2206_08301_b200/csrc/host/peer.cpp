// See peer.hpp.
#include "peer.hpp"

#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "status.hpp"

namespace einplan {
namespace gpu {

namespace {

double env_timeout() {
  if (const char* v = std::getenv("EB_PEER_TIMEOUT_S")) {
    const double t = std::atof(v);
    if (t > 0) return t;
  }
  return 600.0;
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw eb::DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

std::shared_ptr<PeerShared> PeerShared::attach_shm(const std::string& name, int nranks) {
  if (nranks < 1 || nranks > kMaxPeers) throw eb::InvalidError("peer group: 1..64 ranks");
  if (name.empty() || name[0] != '/' || name.find('/', 1) != std::string::npos)
    throw eb::InvalidError("peer group: name must look like \"/something\" (POSIX shm name)");
  const int fd = shm_open(name.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0) throw eb::DeviceError("peer group: shm_open(" + name + ") failed");
  if (ftruncate(fd, sizeof(PeerHeader)) != 0) {
    close(fd);
    throw eb::DeviceError("peer group: ftruncate failed");
  }
  void* p = mmap(nullptr, sizeof(PeerHeader), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) throw eb::DeviceError("peer group: mmap failed");
  std::shared_ptr<PeerShared> s(new PeerShared());
  s->hdr_ = static_cast<PeerHeader*>(p);  // a fresh segment is zero-filled
  s->nranks_ = nranks;
  s->ipc_ = true;
  s->name_ = name;
  s->timeout_s_ = env_timeout();
  return s;
}

std::shared_ptr<PeerShared> PeerShared::for_threads(int nranks) {
  if (nranks < 1 || nranks > kMaxPeers) throw eb::InvalidError("peer group: 1..64 ranks");
  std::shared_ptr<PeerShared> s(new PeerShared());
  s->hdr_ = new PeerHeader();
  std::memset(static_cast<void*>(s->hdr_), 0, sizeof(PeerHeader));
  s->nranks_ = nranks;
  s->ipc_ = false;
  s->timeout_s_ = env_timeout();
  return s;
}

PeerShared::~PeerShared() {
  if (!hdr_) return;
  if (ipc_)
    munmap(hdr_, sizeof(PeerHeader));
  else
    delete hdr_;
}

void PeerShared::abort() { hdr_->aborted.store(1, std::memory_order_release); }

PeerComm::PeerComm(std::shared_ptr<PeerShared> shared, int rank)
    : shared_(std::move(shared)), rank_(rank) {
  if (rank_ < 0 || rank_ >= shared_->nranks()) throw eb::InvalidError("peer group: bad rank");
  barrier();  // every rank attached
  if (shared_->ipc() && rank_ == 0) shm_unlink(shared_->name().c_str());
}

void PeerComm::barrier() {
  PeerHeader* h = shared_->header();
  const std::uint32_t n = static_cast<std::uint32_t>(shared_->nranks());
  const std::uint32_t gen = h->generation.load(std::memory_order_acquire);
  if (h->arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == n) {
    h->arrived.store(0, std::memory_order_relaxed);
    h->generation.fetch_add(1, std::memory_order_release);
    return;
  }
  const auto deadline = std::chrono::steady_clock::now() +
                        std::chrono::duration<double>(shared_->timeout_s());
  for (unsigned spin = 0; h->generation.load(std::memory_order_acquire) == gen; ++spin) {
    if (h->aborted.load(std::memory_order_acquire))
      throw eb::DeviceError("peer group: another rank failed");
    if (spin < 2000) {
      sched_yield();
      continue;
    }
    if (std::chrono::steady_clock::now() > deadline) {
      shared_->abort();
      throw eb::DeviceError("peer group: barrier timed out (EB_PEER_TIMEOUT_S)");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

std::vector<char*> PeerComm::exchange(void* mine) {
  PeerHeader* h = shared_->header();
  PeerHeader::Slot& s = h->slot[rank_];
  int dev = 0;
  cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
  s.device = dev;
  s.ptr = reinterpret_cast<std::uint64_t>(mine);
  s.valid = mine != nullptr;
  if (shared_->ipc() && mine) cuda_ok(cudaIpcGetMemHandle(&s.handle, mine), "cudaIpcGetMemHandle");
  barrier();
  std::vector<char*> out(static_cast<std::size_t>(nranks()), nullptr);
  for (int r = 0; r < nranks(); ++r) {
    const PeerHeader::Slot& o = h->slot[r];
    if (r == rank_) {
      out[static_cast<std::size_t>(r)] = static_cast<char*>(mine);
      continue;
    }
    if (!o.valid) continue;
    if (shared_->ipc()) {
      void* p = nullptr;
      cuda_ok(cudaIpcOpenMemHandle(&p, o.handle, cudaIpcMemLazyEnablePeerAccess),
              "cudaIpcOpenMemHandle");
      out[static_cast<std::size_t>(r)] = static_cast<char*>(p);
    } else {
      if (o.device != dev) {
        int can = 0;
        cuda_ok(cudaDeviceCanAccessPeer(&can, dev, o.device), "cudaDeviceCanAccessPeer");
        if (!can)
          throw eb::DeviceError("peer group: device " + std::to_string(dev) +
                                " cannot access device " + std::to_string(o.device));
        const cudaError_t e = cudaDeviceEnablePeerAccess(o.device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled)
          (void)cudaGetLastError();
        else
          cuda_ok(e, "cudaDeviceEnablePeerAccess");
      }
      out[static_cast<std::size_t>(r)] = reinterpret_cast<char*>(o.ptr);
    }
  }
  barrier();  // slots may be rewritten only after every rank has read them
  return out;
}

void PeerComm::unmap(std::vector<char*>& peers) {
  if (shared_->ipc())
    for (int r = 0; r < static_cast<int>(peers.size()); ++r)
      if (r != rank_ && peers[static_cast<std::size_t>(r)])
        cudaIpcCloseMemHandle(peers[static_cast<std::size_t>(r)]);
  peers.clear();
}

}  // namespace gpu
}  // namespace einplan
