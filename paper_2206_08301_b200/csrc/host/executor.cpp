// GPU executor for an einplan schedule: the B200 replacement of
// einplan::run() (proj/src/executor.cpp:156-263).
//
// Same term loop and the same accounting as the reference:
//   stage inputs per placement (scatter, 48-65)  -> host-to-device block copies
//   local_contract per step (126-154)            -> eb_contract (DMMA/TMA) for
//        fused MTTKRP terms and TTM / GEMM steps, eb_step_generic otherwise
//   allreduce over reduction groups (80-108)     -> eb_group_sum (virtual ranks
//        on one device, ascending-rank order) or ncclAllReduce on a
//        ncclCommSplit communicator per output block (one process per GPU)
//   apply_plan redistribution (redistribute.cpp:185-206) -> eb_copy_box per
//        message, or grouped ncclSend/ncclRecv of packed boxes
//   gather canonical replicas (67-78)            -> device-to-host block copies
// Communication volumes follow the reference conventions exactly
// (allreduce: block elements x (group size - 1); redistribute: transmitted
// volume of the plan; per-rank sends as in executor.cpp:103-105, 193-198).
#include "executor.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <random>
#include <set>
#include <thread>

#include "status.hpp"

#ifdef EB_HAVE_NCCL
#include <nccl.h>
#endif

namespace einplan {
namespace gpu {

namespace {

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw eb::DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

void eb_ok(int status, const char* what) {
  if (status != EB_OK) {
    const std::string msg = std::string(what) + ": " + eb_last_error();
    if (status == EB_E_INVALID) throw eb::InvalidError(msg);
    throw eb::DeviceError(msg);
  }
}

bool contains(const std::string& s, char c) { return s.find(c) != std::string::npos; }

std::int64_t prod(const std::vector<std::int64_t>& v) {
  std::int64_t n = 1;
  for (auto x : v) n *= x;
  return n;
}

// Copy the dense device block (shape, base) to / from its box inside the
// row-major host tensor of shape gshape (scatter / gather, executor.cpp:48-78).
// Trailing dims the block spans completely collapse into one contiguous run;
// the next dim becomes the height of a pitched 2D copy; only the dims above
// it are looped over on the host.
void copy_box_host(bool h2d, double* host, const std::vector<std::int64_t>& gshape,
                   const std::vector<std::int64_t>& shape, const std::vector<std::int64_t>& base,
                   double* dev, cudaStream_t st) {
  const std::size_t nd = gshape.size();
  const cudaMemcpyKind kind = h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  if (nd == 0 || prod(shape) == 0) {
    if (nd == 0)
      cuda_ok(h2d ? cudaMemcpyAsync(dev, host, 8, kind, st) : cudaMemcpyAsync(host, dev, 8, kind, st),
              "box copy");
    return;
  }
  std::vector<std::int64_t> gstr(nd, 1);
  for (std::size_t d = nd; d-- > 1;) gstr[d - 1] = gstr[d] * gshape[d];
  std::size_t d0 = nd - 1;  // every dim after d0 is spanned completely
  while (d0 > 0 && shape[d0] == gshape[d0]) --d0;
  const std::int64_t run = shape[d0] * gstr[d0];
  const std::size_t run_b = static_cast<std::size_t>(run) * 8;
  if (d0 == 0) {
    double* h = host + base[0] * gstr[0];
    cuda_ok(h2d ? cudaMemcpyAsync(dev, h, run_b, kind, st) : cudaMemcpyAsync(h, dev, run_b, kind, st),
            "box copy");
    return;
  }
  const std::size_t dh = d0 - 1;  // pitched-copy dim
  const std::int64_t height = shape[dh];
  const std::size_t hpitch = static_cast<std::size_t>(gstr[dh]) * 8;
  std::int64_t groups = 1;
  for (std::size_t d = 0; d < dh; ++d) groups *= shape[d];
  std::vector<std::int64_t> idx(dh, 0);
  for (std::int64_t gi = 0; gi < groups; ++gi) {
    std::int64_t off = base[dh] * gstr[dh] + base[d0] * gstr[d0];
    for (std::size_t d = 0; d < dh; ++d) off += (base[d] + idx[d]) * gstr[d];
    double* dv = dev + gi * height * run;
    double* h = host + off;
    cuda_ok(h2d ? cudaMemcpy2DAsync(dv, run_b, h, hpitch, run_b, static_cast<std::size_t>(height),
                                    kind, st)
                : cudaMemcpy2DAsync(h, hpitch, dv, run_b, run_b, static_cast<std::size_t>(height),
                                    kind, st),
            "box copy 2D");
    for (std::size_t d = dh; d-- > 0;) {
      if (++idx[d] < shape[d]) break;
      idx[d] = 0;
    }
  }
}

}  // namespace

// ------------------------------------------------------------- buffers --

double* DeviceArena::alloc(std::int64_t elems, cudaStream_t st, bool zero) {
  void* p = nullptr;
  const std::size_t bytes = static_cast<std::size_t>(std::max<std::int64_t>(elems, 1)) * 8;
  for (std::size_t i = 0; recycle_ && i < kept_.size(); ++i)
    if (kept_[i].first == bytes) {
      p = kept_[i].second;
      kept_.erase(kept_.begin() + static_cast<std::ptrdiff_t>(i));
      break;
    }
  if (!p) {
    cuda_ok(cudaMallocAsync(&p, bytes, st), "cudaMallocAsync");
    ++mallocs_;
  }
  if (zero) cuda_ok(cudaMemsetAsync(p, 0, bytes, st), "cudaMemsetAsync");
  live_.emplace_back(bytes, p);
  return static_cast<double*>(p);
}

void DeviceArena::release(cudaStream_t st) {
  if (recycle_) {
    kept_.insert(kept_.end(), live_.begin(), live_.end());
  } else {
    for (auto& b : live_) cudaFreeAsync(b.second, st);
  }
  live_.clear();
}

void DeviceArena::set_recycle(bool on, cudaStream_t st) {
  if (!on)
    for (auto& b : kept_) cudaFreeAsync(b.second, st);
  if (!on) kept_.clear();
  recycle_ = on;
}

DeviceArena::~DeviceArena() {
  for (auto& b : live_) cudaFree(b.second);
  for (auto& b : kept_) cudaFree(b.second);
}

// ------------------------------------------------------- transports --

Transport::~Transport() {
  if (comm_stream_) {
    cudaStreamSynchronize(comm_stream_);
    cudaStreamDestroy(comm_stream_);
  }
}

cudaStream_t Transport::comm_stream() {
  if (!comm_stream_)
    cuda_ok(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking), "comm stream");
  return comm_stream_;
}

namespace {

// Reduction groups of a placement: ranks holding the same output block
// (executor.cpp:84-86), ascending; accounts the reference's volumes
// (elements x (group - 1), per-rank sends, executor.cpp:103-105).
std::map<std::vector<std::int64_t>, std::vector<std::int64_t>> reduction_groups(
    const TensorPlacement& place, std::vector<std::int64_t>& per_rank_sent, std::int64_t& volume) {
  std::map<std::vector<std::int64_t>, std::vector<std::int64_t>> groups;
  const std::int64_t procs = place.term_grid.total();
  for (std::int64_t r = 0; r < procs; ++r) groups[place.block_coords_of(r)].push_back(r);
  volume = 0;
  for (auto& kv : groups) {
    const std::int64_t n = prod(place.dist.shape_of(kv.first));
    for (std::int64_t r : kv.second) per_rank_sent[static_cast<std::size_t>(r)] += n;
    volume += n * (static_cast<std::int64_t>(kv.second.size()) - 1);
  }
  return groups;
}

}  // namespace

std::int64_t VirtualTransport::allreduce(const TensorPlacement& place, const ReductionGroup& grp,
                                         std::vector<DevBlock>& blocks,
                                         std::vector<std::int64_t>& per_rank_sent,
                                         cudaStream_t st) {
  if (grp.depth <= 1) return 0;
  std::int64_t volume = 0;
  const auto groups = reduction_groups(place, per_rank_sent, volume);
  for (auto& kv : groups) {
    const auto& members = kv.second;
    std::vector<double*> ptrs;
    const std::int64_t n = blocks[static_cast<std::size_t>(members.front())].size();
    for (std::int64_t r : members) {
      const DevBlock& b = blocks[static_cast<std::size_t>(r)];
      if (b.size() != n)
        fail(errc::invalid_argument,
             "allreduce: shape divergence within a group of \"" + place.tensor + "\"");
      ptrs.push_back(b.ptr);
    }
    eb_ok(eb_group_sum(ptrs.data(), static_cast<int>(ptrs.size()), n, st), "eb_group_sum");
  }
  return volume;
}

void VirtualTransport::redistribute(const RedistributionPlan& plan,
                                    const std::vector<DevBlock>& src, std::vector<DevBlock>& dst,
                                    cudaStream_t st) {
  for (const Message& m : plan.messages) {
    const DevBlock& s = src[static_cast<std::size_t>(m.src_rank)];
    DevBlock& d = dst[static_cast<std::size_t>(m.dst_rank)];
    if (!s.ptr && m.elements > 0)
      fail(errc::invalid_argument,
           "apply_plan: missing source block on rank " + std::to_string(m.src_rank));
    eb_ok(eb_copy_box(static_cast<int>(m.oy_lo.size()), s.ptr, s.shape.data(), d.ptr,
                      d.shape.data(), m.oy_lo.data(), m.oy_hi.data(), m.ox_lo.data(), st),
          "eb_copy_box");
  }
}

// ---- peer memory ----

PeerTransport::PeerTransport(std::shared_ptr<PeerComm> comm, std::int64_t nranks,
                             std::unique_ptr<Transport> allreduce_via)
    : comm_(std::move(comm)), nranks_(nranks), allreduce_via_(std::move(allreduce_via)) {
  if (comm_->nranks() != nranks)
    fail(errc::invalid_argument, "peer transport: group of " + std::to_string(comm_->nranks()) +
                                     " ranks for a schedule of " + std::to_string(nranks));
}

std::int64_t PeerTransport::allreduce(const TensorPlacement& place, const ReductionGroup& grp,
                                      std::vector<DevBlock>& blocks,
                                      std::vector<std::int64_t>& per_rank_sent, cudaStream_t st) {
  if (grp.depth <= 1) return 0;
  if (allreduce_via_)  // hybrid: NCCL on the split communicator, in place, asynchronous
    return allreduce_via_->allreduce(place, grp, blocks, per_rank_sent, st);
  std::int64_t volume = 0;
  const auto groups = reduction_groups(place, per_rank_sent, volume);
  const std::int64_t me = comm_->rank();
  const auto& members = groups.at(place.block_coords_of(me));
  DevBlock& mine = blocks[static_cast<std::size_t>(me)];
  const std::int64_t n = mine.size();
  std::vector<const double*> ptrs;
  for (std::int64_t r : members) {
    const DevBlock& b = blocks[static_cast<std::size_t>(r)];
    if (!b.ptr || b.size() != n)
      fail(errc::invalid_argument,
           "allreduce: rank " + std::to_string(r) + " block of \"" + place.tensor + "\" not mapped");
    ptrs.push_back(b.ptr);
  }
  cuda_ok(cudaStreamSynchronize(st), "allreduce: sync");
  comm_->barrier();  // every partial of every group is complete
  double* sum = nullptr;
  if (n > 0 && members.size() > 1) {
    cuda_ok(cudaMallocAsync(reinterpret_cast<void**>(&sum), static_cast<std::size_t>(n) * 8, st),
            "allreduce: scratch");
    eb_ok(eb_group_sum_into(ptrs.data(), static_cast<int>(ptrs.size()), n, sum, st),
          "eb_group_sum_into");
  }
  cuda_ok(cudaStreamSynchronize(st), "allreduce: sync");
  comm_->barrier();  // every member has read every partial: overwrite own block
  if (sum) {
    cuda_ok(cudaMemcpyAsync(mine.ptr, sum, static_cast<std::size_t>(n) * 8,
                            cudaMemcpyDeviceToDevice, st),
            "allreduce: write back");
    cuda_ok(cudaFreeAsync(sum, st), "allreduce: scratch");
  }
  // readers of the sum (a redistribution, the gather) start with a sync +
  // barrier of their own, after which this write is complete
  return volume;
}

void PeerTransport::redistribute(const RedistributionPlan& plan, const std::vector<DevBlock>& src,
                                 std::vector<DevBlock>& dst, cudaStream_t st) {
  const std::int64_t me = comm_->rank();
  cuda_ok(cudaStreamSynchronize(st), "redistribute: sync");
  comm_->barrier();  // every source block is complete
  DevBlock& d = dst[static_cast<std::size_t>(me)];
  for (const Message& m : plan.messages) {
    if (m.dst_rank != me) continue;
    const DevBlock& s = src[static_cast<std::size_t>(m.src_rank)];
    if (!s.ptr && m.elements > 0)
      fail(errc::invalid_argument,
           "apply_plan: source block of rank " + std::to_string(m.src_rank) + " not mapped");
    eb_ok(eb_copy_box(static_cast<int>(m.oy_lo.size()), s.ptr, s.shape.data(), d.ptr,
                      d.shape.data(), m.oy_lo.data(), m.oy_hi.data(), m.ox_lo.data(), st),
          "eb_copy_box (peer pull)");
  }
  cuda_ok(cudaStreamSynchronize(st), "redistribute: sync");
  comm_->barrier();  // every destination has pulled: sources may be reused
}

void PeerTransport::gather_to_root(const TensorPlacement&, std::vector<DevBlock>&, cudaStream_t st) {
  cuda_ok(cudaStreamSynchronize(st), "gather: sync");
  comm_->barrier();  // canonical blocks final; rank 0 reads them from the peers' heaps
}

void PeerTransport::gather_done(std::vector<DevBlock>&, cudaStream_t st) {
  cuda_ok(cudaStreamSynchronize(st), "gather: sync");
  comm_->barrier();
}

#ifdef EB_HAVE_NCCL

namespace {
void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw eb::DeviceError(std::string(what) + ": " + ncclGetErrorString(r));
}
}  // namespace

NcclTransport::NcclTransport(const void* unique_id, std::int64_t nranks, std::int64_t rank)
    : rank_(rank), nranks_(nranks) {
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t c = nullptr;
  nccl_ok(ncclCommInitRank(&c, static_cast<int>(nranks), id, static_cast<int>(rank)),
          "ncclCommInitRank");
  world_ = c;
}

NcclTransport::NcclTransport(void* comm, std::int64_t nranks, std::int64_t rank)
    : rank_(rank), nranks_(nranks), world_(comm) {}

NcclTransport::~NcclTransport() {
  if (staging_done_) cudaEventSynchronize(staging_done_);
  if (staging_) cudaFree(staging_);
  if (staging_done_) cudaEventDestroy(staging_done_);
  for (auto& kv : split_) ncclCommDestroy(static_cast<ncclComm_t>(kv.second));
  if (world_) ncclCommDestroy(static_cast<ncclComm_t>(world_));
}

double* NcclTransport::staging(std::int64_t elems, cudaStream_t st) {
  if (!staging_done_)
    cuda_ok(cudaEventCreateWithFlags(&staging_done_, cudaEventDisableTiming), "event");
  else
    cuda_ok(cudaStreamWaitEvent(st, staging_done_, 0), "staging: wait for its last use");
  if (elems > staging_elems_) {
    if (staging_) cuda_ok(cudaFreeAsync(staging_, st), "staging free");
    staging_ = nullptr;
    cuda_ok(cudaMallocAsync(reinterpret_cast<void**>(&staging_),
                            static_cast<std::size_t>(elems) * 8, st),
            "staging alloc");
    staging_elems_ = elems;
  }
  return staging_;
}

std::int64_t NcclTransport::allreduce(const TensorPlacement& place, const ReductionGroup& grp,
                                      std::vector<DevBlock>& blocks,
                                      std::vector<std::int64_t>& per_rank_sent, cudaStream_t st) {
  if (grp.depth <= 1) return 0;
  // Group = ranks holding the same output block; color it by the block's
  // index among the groups so ncclCommSplit reproduces executor.cpp:84-86.
  std::int64_t volume = 0;
  const auto groups = reduction_groups(place, per_rank_sent, volume);
  const auto mine = place.block_coords_of(rank_);
  int color = 0, idx = 0;
  for (auto& kv : groups) {
    if (kv.first == mine) color = idx;
    ++idx;
  }
  // One split communicator per (placement signature); cached across runs.
  std::string key = place.tensor + "|";
  for (auto d : place.term_grid.dims) key += std::to_string(d) + ",";
  for (auto a : place.axes) key += std::to_string(a) + ";";
  auto it = split_.find(key);
  if (it == split_.end()) {
    ncclComm_t sub = nullptr;
    nccl_ok(ncclCommSplit(static_cast<ncclComm_t>(world_), color, static_cast<int>(rank_), &sub,
                          nullptr),
            "ncclCommSplit");
    it = split_.emplace(key, sub).first;
  }
  DevBlock& b = blocks[static_cast<std::size_t>(rank_)];
  nccl_ok(ncclAllReduce(b.ptr, b.ptr, static_cast<std::size_t>(b.size()), ncclFloat64, ncclSum,
                        static_cast<ncclComm_t>(it->second), st),
          "ncclAllReduce");
  return volume;
}

void NcclTransport::redistribute(const RedistributionPlan& plan, const std::vector<DevBlock>& src,
                                 std::vector<DevBlock>& dst, cudaStream_t st) {
  // Pack every outgoing box into one reused staging buffer, exchange with
  // grouped point-to-point calls, unpack every incoming box; self messages
  // copy in place.
  struct Pending {
    const Message* m;
    std::int64_t off;
  };
  std::vector<Pending> sends, recvs;
  std::int64_t total = 0;
  for (const Message& m : plan.messages) {
    if (m.src_rank != rank_ && m.dst_rank != rank_) continue;
    if (m.src_rank == rank_ && m.dst_rank == rank_) continue;
    (m.src_rank == rank_ ? sends : recvs).push_back({&m, total});
    total += m.elements;
  }
  double* buf = total > 0 ? staging(total, st) : nullptr;
  for (const Message& m : plan.messages) {
    if (m.src_rank != rank_ || m.dst_rank != rank_) continue;
    const DevBlock& s = src[static_cast<std::size_t>(rank_)];
    DevBlock& d = dst[static_cast<std::size_t>(rank_)];
    eb_ok(eb_copy_box(static_cast<int>(m.oy_lo.size()), s.ptr, s.shape.data(), d.ptr,
                      d.shape.data(), m.oy_lo.data(), m.oy_hi.data(), m.ox_lo.data(), st),
          "eb_copy_box");
  }
  if (total == 0) return;
  for (auto& p : sends) {
    const Message& m = *p.m;
    const std::size_t nd = m.oy_lo.size();
    std::vector<std::int64_t> box(nd), zeros(nd, 0);
    for (std::size_t d = 0; d < nd; ++d) box[d] = m.oy_hi[d] - m.oy_lo[d];
    const DevBlock& s = src[static_cast<std::size_t>(rank_)];
    eb_ok(eb_copy_box(static_cast<int>(nd), s.ptr, s.shape.data(), buf + p.off, box.data(),
                      m.oy_lo.data(), m.oy_hi.data(), zeros.data(), st),
          "pack");
  }
  nccl_ok(ncclGroupStart(), "ncclGroupStart");
  for (auto& p : sends)
    nccl_ok(ncclSend(buf + p.off, static_cast<std::size_t>(p.m->elements), ncclFloat64,
                     static_cast<int>(p.m->dst_rank), static_cast<ncclComm_t>(world_), st),
            "ncclSend");
  for (auto& p : recvs)
    nccl_ok(ncclRecv(buf + p.off, static_cast<std::size_t>(p.m->elements), ncclFloat64,
                     static_cast<int>(p.m->src_rank), static_cast<ncclComm_t>(world_), st),
            "ncclRecv");
  nccl_ok(ncclGroupEnd(), "ncclGroupEnd");
  for (auto& p : recvs) {
    const Message& m = *p.m;
    const std::size_t nd = m.oy_lo.size();
    std::vector<std::int64_t> box(nd), zeros(nd, 0);
    for (std::size_t d = 0; d < nd; ++d) box[d] = m.oy_hi[d] - m.oy_lo[d];
    DevBlock& d = dst[static_cast<std::size_t>(rank_)];
    eb_ok(eb_copy_box(static_cast<int>(nd), buf + p.off, box.data(), d.ptr, d.shape.data(),
                      zeros.data(), box.data(), m.ox_lo.data(), st),
          "unpack");
  }
  cuda_ok(cudaEventRecord(staging_done_, st), "event record");
}

void NcclTransport::gather_to_root(const TensorPlacement& place, std::vector<DevBlock>& blocks,
                                   cudaStream_t st) {
  // Canonical owners send their block to rank 0, which receives every
  // non-local canonical block into buffers released by gather_done().
  const std::int64_t procs = place.term_grid.total();
  nccl_ok(ncclGroupStart(), "ncclGroupStart");
  for (std::int64_t r = 1; r < procs; ++r) {
    if (!place.is_canonical(r)) continue;
    const std::int64_t n = prod(place.dist.shape_of(place.block_coords_of(r)));
    if (rank_ == r)
      nccl_ok(ncclSend(blocks[static_cast<std::size_t>(r)].ptr, static_cast<std::size_t>(n),
                       ncclFloat64, 0, static_cast<ncclComm_t>(world_), st),
              "ncclSend");
    if (rank_ == 0) {
      DevBlock& b = blocks[static_cast<std::size_t>(r)];
      double* p = nullptr;
      cuda_ok(cudaMallocAsync(reinterpret_cast<void**>(&p),
                              static_cast<std::size_t>(std::max<std::int64_t>(n, 1)) * 8, st),
              "gather buffer");
      gathered_.push_back(p);
      b.ptr = p;
      nccl_ok(ncclRecv(b.ptr, static_cast<std::size_t>(n), ncclFloat64, static_cast<int>(r),
                       static_cast<ncclComm_t>(world_), st),
              "ncclRecv");
    }
  }
  nccl_ok(ncclGroupEnd(), "ncclGroupEnd");
}

void NcclTransport::gather_done(std::vector<DevBlock>& blocks, cudaStream_t st) {
  if (gathered_.empty()) return;
  for (double* p : gathered_) {
    for (DevBlock& b : blocks)
      if (b.ptr == p) b.ptr = nullptr;
    cudaFreeAsync(p, st);
  }
  gathered_.clear();
}

#endif  // EB_HAVE_NCCL

// --------------------------------------------------------- executor --

ScheduleExecutor::ScheduleExecutor(Pipeline pipe, Transport* transport, cudaStream_t stream)
    : pipe_(std::move(pipe)), transport_(transport), stream_(stream) {
  const std::int64_t procs = pipe_.schedule.procs;
  for (std::int64_t r = 0; r < procs; ++r)
    if (transport_->owns(r)) owned_.push_back(r);
  comm_.per_rank_sent.assign(static_cast<std::size_t>(procs), 0);
  // Keep freed stream-ordered blocks in the pool: repeated execute() calls
  // reuse them instead of returning memory to the driver at every sync.
  int dev = 0;
  cudaMemPool_t pool = nullptr;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    std::uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
}

ScheduleExecutor::~ScheduleExecutor() {
  if (comm_pending_) cudaStreamWaitEvent(stream_, ev_comm_, 0);  // no throwing in a destructor
  cudaStreamSynchronize(stream_);
  if (ev_compute_) cudaEventDestroy(ev_compute_);
  if (ev_comm_) cudaEventDestroy(ev_comm_);
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  run_arena_.release(stream_);
  run_arena_.set_recycle(false, stream_);
  input_arena_.release(stream_);
  cudaFreeAsync(workspace_, stream_);
  cudaStreamSynchronize(stream_);
  if (heap_) {
    if (auto* pt = dynamic_cast<PeerTransport*>(transport_)) pt->comm().unmap(heap_peers_);
    cudaFree(heap_);
  }
}

std::int64_t ScheduleExecutor::local_lo(const TermPlan& t, char c, std::int64_t rank) const {
  const int axis = t.grid.axis_of(c);
  return t.grid.coords_of(rank)[static_cast<std::size_t>(axis)] * t.blocks.at(c);
}

std::int64_t ScheduleExecutor::local_len(const TermPlan& t, char c, std::int64_t rank) const {
  return std::min(t.blocks.at(c), pipe_.spec.extent(c) - local_lo(t, c, rank));
}

void ScheduleExecutor::stage_inputs(const std::vector<const double*>& globals) {
  const auto& spec = pipe_.spec;
  if (globals.size() != spec.inputs.size())
    fail(errc::invalid_argument, "stage: operand count mismatch");
  // Device blocks are allocated on the first stage and reused afterwards, so
  // that blocks aliased by another executor (share_input) stay valid.  A
  // null host pointer keeps the operand's current device contents.
  for (const TermPlan& term : pipe_.schedule.terms) {
    for (const AccessArray& arr : term.statement.arrays) {
      if (arr.tensor.rfind("in", 0) != 0) continue;
      const std::size_t k = static_cast<std::size_t>(std::stoi(arr.tensor.substr(2)));
      const TensorPlacement& place = term.placement_of(arr.tensor);
      const auto gshape = spec.shape_of(spec.inputs[k]);
      const auto key = std::make_pair(term.index, arr.tensor);
      auto it = inputs_.find(key);
      if (it == inputs_.end()) {
        std::vector<DevBlock> blocks(static_cast<std::size_t>(pipe_.schedule.procs));
        for (std::int64_t r : owned_) {
          DevBlock& b = blocks[static_cast<std::size_t>(r)];
          const auto bc = place.block_coords_of(r);
          b.base = place.dist.base_of(bc);
          b.shape = place.dist.shape_of(bc);
          b.ptr = input_arena_.alloc(prod(b.shape), stream_, false);
        }
        it = inputs_.emplace(key, std::move(blocks)).first;
      }
      if (globals[k] == nullptr) continue;
      if (aliased_.count(key))
        fail(errc::invalid_argument, "stage: operand " + arr.tensor +
                                         " is shared from another executor; pass NULL for it");
      for (std::int64_t r : owned_) copy_block_h2d(globals[k], gshape, it->second[r]);
    }
  }
  staged_ = true;
}

void ScheduleExecutor::local_block(int k, std::vector<std::int64_t>& base,
                                   std::vector<std::int64_t>& shape) const {
  if (owned_.size() != 1)
    fail(errc::invalid_argument, "local_block: needs exactly one owned rank (one process per GPU)");
  const std::string name = "in" + std::to_string(k);
  bool found = false;
  for (const TermPlan& term : pipe_.schedule.terms)
    for (const AccessArray& arr : term.statement.arrays) {
      if (arr.tensor != name) continue;
      const TensorPlacement& place = term.placement_of(name);
      const auto bc = place.block_coords_of(owned_[0]);
      const auto b = place.dist.base_of(bc), s = place.dist.shape_of(bc);
      if (found && (b != base || s != shape))
        fail(errc::invalid_argument, "local_block: " + name + " is placed differently by two terms");
      base = b;
      shape = s;
      found = true;
    }
  if (!found) fail(errc::invalid_argument, "local_block: no operand in" + std::to_string(k));
}

void ScheduleExecutor::stage_block(int k, const double* host_block) {
  std::vector<std::int64_t> base, shape;
  local_block(k, base, shape);
  const std::string name = "in" + std::to_string(k);
  const std::int64_t r = owned_[0];
  for (const TermPlan& term : pipe_.schedule.terms)
    for (const AccessArray& arr : term.statement.arrays) {
      if (arr.tensor != name) continue;
      const auto key = std::make_pair(term.index, name);
      if (aliased_.count(key))
        fail(errc::invalid_argument, "stage_block: " + name + " is shared from another executor");
      auto it = inputs_.find(key);
      if (it == inputs_.end()) {
        std::vector<DevBlock> blocks(static_cast<std::size_t>(pipe_.schedule.procs));
        DevBlock& b = blocks[static_cast<std::size_t>(r)];
        b.base = base;
        b.shape = shape;
        b.ptr = input_arena_.alloc(prod(shape), stream_, false);
        it = inputs_.emplace(key, std::move(blocks)).first;
      }
      const DevBlock& b = it->second[static_cast<std::size_t>(r)];
      cuda_ok(cudaMemcpyAsync(b.ptr, host_block, static_cast<std::size_t>(prod(shape)) * 8,
                              cudaMemcpyHostToDevice, stream_),
              "H2D block");
    }
  // staged once every operand has device blocks on this rank
  bool all = true;
  for (const TermPlan& term : pipe_.schedule.terms)
    for (const AccessArray& arr : term.statement.arrays)
      if (arr.tensor.rfind("in", 0) == 0 && !inputs_.count({term.index, arr.tensor})) all = false;
  staged_ = all;
}

int ScheduleExecutor::stage_region(int k, const std::vector<std::int64_t>& rbase,
                                   const std::vector<std::int64_t>& rshape, const double* host) {
  const auto& spec = pipe_.spec;
  if (k < 0 || static_cast<std::size_t>(k) >= spec.inputs.size())
    fail(errc::invalid_argument, "stage_region: no operand " + std::to_string(k));
  const std::string name = "in" + std::to_string(k);
  const auto gshape = spec.shape_of(spec.inputs[static_cast<std::size_t>(k)]);
  if (rbase.size() != gshape.size() || rshape.size() != gshape.size())
    fail(errc::invalid_argument, "stage_region: region rank differs from the operand's");
  for (std::size_t d = 0; d < gshape.size(); ++d)
    if (rbase[d] < 0 || rshape[d] < 0 || rbase[d] + rshape[d] > gshape[d])
      fail(errc::invalid_argument, "stage_region: region outside the operand");
  int staged = 0;
  for (const TermPlan& term : pipe_.schedule.terms)
    for (const AccessArray& arr : term.statement.arrays) {
      if (arr.tensor != name) continue;
      const auto key = std::make_pair(term.index, name);
      if (aliased_.count(key))
        fail(errc::invalid_argument, "stage_region: " + name + " is shared from another executor");
      const TensorPlacement& place = term.placement_of(name);
      auto it = inputs_.find(key);
      if (it == inputs_.end()) {
        std::vector<DevBlock> blocks(static_cast<std::size_t>(pipe_.schedule.procs));
        for (std::int64_t r : owned_) {
          DevBlock& b = blocks[static_cast<std::size_t>(r)];
          const auto bc = place.block_coords_of(r);
          b.base = place.dist.base_of(bc);
          b.shape = place.dist.shape_of(bc);
          b.ptr = input_arena_.alloc(prod(b.shape), stream_, false);
        }
        it = inputs_.emplace(key, std::move(blocks)).first;
      }
      for (std::int64_t r : owned_) {
        const DevBlock& b = it->second[static_cast<std::size_t>(r)];
        bool inside = true;
        std::vector<std::int64_t> rel(b.base.size());
        for (std::size_t d = 0; d < b.base.size(); ++d) {
          rel[d] = b.base[d] - rbase[d];
          inside = inside && rel[d] >= 0 && rel[d] + b.shape[d] <= rshape[d];
        }
        if (!inside) continue;
        copy_box_host(true, const_cast<double*>(host), rshape, b.shape, rel, b.ptr, stream_);
        ++staged;
      }
    }
  bool all = true;
  for (const TermPlan& term : pipe_.schedule.terms)
    for (const AccessArray& arr : term.statement.arrays)
      if (arr.tensor.rfind("in", 0) == 0 && !inputs_.count({term.index, arr.tensor})) all = false;
  staged_ = all;
  return staged;
}

void ScheduleExecutor::share_input(int k, const ScheduleExecutor& src, int k_src) {
  const std::string name = "in" + std::to_string(k), sname = "in" + std::to_string(k_src);
  if (!src.staged_) fail(errc::invalid_argument, "share_input: source executor not staged");
  if (pipe_.spec.shape_of(pipe_.spec.inputs[static_cast<std::size_t>(k)]) !=
      src.pipe_.spec.shape_of(src.pipe_.spec.inputs[static_cast<std::size_t>(k_src)]))
    fail(errc::invalid_argument, "share_input: operand shapes differ");
  const std::vector<DevBlock>* from = nullptr;
  for (const auto& kv : src.inputs_)
    if (kv.first.second == sname) from = &kv.second;
  if (!from) fail(errc::invalid_argument, "share_input: source holds no " + sname);
  for (const TermPlan& term : pipe_.schedule.terms) {
    for (const AccessArray& arr : term.statement.arrays) {
      if (arr.tensor != name) continue;
      const TensorPlacement& place = term.placement_of(name);
      std::vector<DevBlock> blocks(static_cast<std::size_t>(pipe_.schedule.procs));
      for (std::int64_t r : owned_) {
        const auto bc = place.block_coords_of(r);
        const DevBlock& sb = (*from)[static_cast<std::size_t>(r)];
        if (sb.base != place.dist.base_of(bc) || sb.shape != place.dist.shape_of(bc))
          fail(errc::invalid_argument,
               "share_input: the two schedules place " + name + " differently on rank " +
                   std::to_string(r));
        blocks[static_cast<std::size_t>(r)] = sb;
      }
      const auto key = std::make_pair(term.index, name);
      inputs_[key] = std::move(blocks);
      aliased_.insert(key);
    }
  }
}

void ScheduleExecutor::copy_block_h2d(const double* global, const std::vector<std::int64_t>& gshape,
                                      const DevBlock& b) {
  copy_box_host(true, const_cast<double*>(global), gshape, b.shape, b.base, b.ptr, stream_);
}

const RedistRecord* ScheduleExecutor::find_redist(int to_term, const std::string& t) const {
  for (const RedistRecord& r : pipe_.schedule.redistributions)
    if (r.to_term == to_term && r.tensor == t) return &r;
  return nullptr;
}

void* ScheduleExecutor::workspace(std::size_t bytes) {
  if (bytes > workspace_bytes_) {
    if (workspace_) cudaFreeAsync(workspace_, stream_);
    workspace_bytes_ = std::max(bytes, workspace_bytes_ * 2);
    cuda_ok(cudaMallocAsync(&workspace_, workspace_bytes_, stream_), "workspace");
  }
  return workspace_;
}

namespace {

// The n-ary view of a fused MTTKRP term: X[s_0..s_{N-1}], factors
// F_n[s_n, r] for every n except the output mode m, out[s_m, r].
struct MttkrpMatch {
  bool ok = false;
  std::string x_name, x_idx;
  char rank_sym = 0;
  int out_mode = -1;
  std::vector<std::string> factor_of;  // per mode: tensor name ("" for the output mode)
};

MttkrpMatch match_mttkrp(const FusedStatement& st) {
  MttkrpMatch mm;
  std::string out_idx;
  std::vector<const AccessArray*> ins;
  for (const AccessArray& a : st.arrays) {
    if (a.tensor == st.output)
      out_idx = a.indices;
    else
      ins.push_back(&a);
  }
  if (out_idx.size() != 2 || ins.size() < 2) return mm;
  const AccessArray* x = nullptr;
  for (const AccessArray* a : ins)
    if (a->indices.size() >= 2 && !contains(a->indices, out_idx[1])) {
      if (x) return mm;  // two candidates for X
      x = a;
    }
  if (!x) return mm;
  const char r = out_idx[1];
  if (!contains(x->indices, out_idx[0])) return mm;
  mm.factor_of.assign(x->indices.size(), std::string());
  for (const AccessArray* a : ins) {
    if (a == x) continue;
    if (a->indices.size() != 2 || a->indices[1] != r) return mm;
    const auto pos = x->indices.find(a->indices[0]);
    if (pos == std::string::npos || a->indices[0] == out_idx[0] || !mm.factor_of[pos].empty())
      return mm;
    mm.factor_of[pos] = a->tensor;
  }
  for (std::size_t d = 0; d < x->indices.size(); ++d) {
    const bool is_out = x->indices[d] == out_idx[0];
    if (is_out != mm.factor_of[d].empty()) return mm;
  }
  mm.ok = true;
  mm.x_name = x->tensor;
  mm.x_idx = x->indices;
  mm.rank_sym = r;
  mm.out_mode = static_cast<int>(x->indices.find(out_idx[0]));
  return mm;
}

}  // namespace

DevBlock ScheduleExecutor::new_block(const TermPlan& term, const std::string& idx,
                                     std::int64_t rank, bool zero, bool is_output) {
  DevBlock b;
  for (char c : idx) {
    b.shape.push_back(local_len(term, c, rank));
    b.base.push_back(local_lo(term, c, rank));
  }
  const auto slot = heap_slot_.find(term.index);
  if (is_output && heap_ && slot != heap_slot_.end()) {
    b.ptr = reinterpret_cast<double*>(heap_ + slot->second);
    if (zero)
      cuda_ok(cudaMemsetAsync(b.ptr, 0, static_cast<std::size_t>(prod(b.shape)) * 8, stream_),
              "cudaMemsetAsync");
  } else {
    b.ptr = run_arena_.alloc(prod(b.shape), stream_, zero);
  }
  return b;
}

void ScheduleExecutor::prepare_heap() {
  if (!transport_->peer_mapped()) return;
  auto* pt = static_cast<PeerTransport*>(transport_);
  const auto& terms = pipe_.schedule.terms;
  const std::int64_t procs = pipe_.schedule.procs;
  heap_slot_.clear();
  std::size_t off = 0;
  for (const TermPlan& t : terms) {
    bool leaves = t.reduction.depth > 1 || &t == &terms.back();
    for (const RedistRecord& rec : pipe_.schedule.redistributions)
      if (rec.from_term == t.index && rec.tensor == t.statement.output) leaves = true;
    if (!leaves) continue;
    const std::string& idx = t.placement_of(t.statement.output).indices;
    std::int64_t most = 1;
    for (std::int64_t r = 0; r < procs; ++r) {
      std::int64_t n = 1;
      for (char c : idx) n *= local_len(t, c, r);
      most = std::max(most, n);
    }
    heap_slot_[t.index] = off;
    off += (static_cast<std::size_t>(most) * 8 + 255) / 256 * 256;
  }
  heap_in_slot_.clear();
  for (const TermPlan& t : terms)
    if (const RedistRecord* rec = push_record(t)) {  // fused redistribution target
      std::int64_t n = 1;
      for (auto bsz : rec->plan.destination.dist.blocks) n *= bsz;
      heap_in_slot_[rec->to_term] = off;
      off += (static_cast<std::size_t>(n) * 8 + 255) / 256 * 256;
    }
  // identical on every rank (same schedule), so the decision is collective
  if (off <= heap_bytes_) return;
  cuda_ok(cudaStreamSynchronize(stream_), "heap: sync");
  pt->comm().unmap(heap_peers_);
  pt->comm().barrier();  // no rank maps the old heaps any more
  if (heap_) cuda_ok(cudaFree(heap_), "heap free");
  heap_ = nullptr;
  heap_bytes_ = 0;
  cuda_ok(cudaMalloc(reinterpret_cast<void**>(&heap_), off), "exchange heap");
  heap_bytes_ = off;
  heap_peers_ = pt->comm().exchange(heap_);
}

void ScheduleExecutor::map_peer_blocks(const TermPlan& term, std::vector<DevBlock>& blocks) {
  const auto slot = heap_slot_.find(term.index);
  if (!heap_ || slot == heap_slot_.end()) return;
  const std::string& idx = term.placement_of(term.statement.output).indices;
  for (std::int64_t r = 0; r < pipe_.schedule.procs; ++r) {
    if (transport_->owns(r)) continue;
    DevBlock& b = blocks[static_cast<std::size_t>(r)];
    b.shape.clear();
    b.base.clear();
    for (char c : idx) {
      b.shape.push_back(local_len(term, c, r));
      b.base.push_back(local_lo(term, c, r));
    }
    char* base = heap_peers_[static_cast<std::size_t>(r)];
    b.ptr = base ? reinterpret_cast<double*>(base + slot->second) : nullptr;
  }
}

bool ScheduleExecutor::try_fused_mttkrp(const TermPlan& term, std::int64_t rank,
                                        const std::map<std::string, const DevBlock*>& at_hand,
                                        DevBlock& out) {
  const MttkrpMatch mm = match_mttkrp(term.statement);
  if (!mm.ok) return false;
  const int N = static_cast<int>(mm.x_idx.size());
  const int m = mm.out_mode;
  std::vector<std::int64_t> ext(N);
  for (int d = 0; d < N; ++d) ext[d] = local_len(term, mm.x_idx[static_cast<std::size_t>(d)], rank);
  const std::int64_t R = local_len(term, mm.rank_sym, rank);
  eb_contract_desc d;
  std::memset(&d, 0, sizeof(d));
  d.mode = EB_REDUCE;
  d.R = R;
  d.X = at_hand.at(mm.x_name)->ptr;
  auto factor = [&](int mode) {
    const DevBlock* f = at_hand.at(mm.factor_of[static_cast<std::size_t>(mode)]);
    eb_factor e;
    e.ptr = f->ptr;
    e.extent = f->shape[0];
    e.ld = f->shape[1];
    return e;
  };
  if (m < N - 1) {
    d.variant = EB_ROW;
    d.P = 1;
    for (int k = 0; k < m; ++k) d.P *= ext[k];
    d.M = ext[m];
    d.Q = 1;
    for (int k = m + 1; k < N - 1; ++k) d.Q *= ext[k];
    d.L = ext[N - 1];
    for (int k = 0; k < m; ++k) d.pre[d.n_pre++] = factor(k);
    for (int k = m + 1; k < N - 1; ++k) d.mid[d.n_mid++] = factor(k);
    const eb_factor u = factor(N - 1);
    d.U = u.ptr;
    d.ldu = u.ld;
    if (d.L % 2) {  // odd contiguous extent: zero-padded X rows and U (TMA pitch)
      d.X = padded_rows(d.X, d.P * d.M * d.Q, d.L);
      d.U = padded_factor(u.ptr, d.L, u.ld);
      d.L += 1;
    }
  } else {
    d.variant = EB_COL;
    d.P = 1;
    for (int k = 0; k < N - 2; ++k) d.P *= ext[k];
    d.Q = ext[N - 2];
    d.M = ext[N - 1];
    for (int k = 0; k < N - 2; ++k) d.pre[d.n_pre++] = factor(k);
    const eb_factor u = factor(N - 2);
    d.U = u.ptr;
    d.ldu = u.ld;
  }
  if (d.n_pre > 8 || d.n_mid > 8) return false;
  out = new_block(term, term.placement_of(term.statement.output).indices, rank, false, true);
  d.out = out.ptr;
  const std::int64_t M0 = d.M;
  if (d.variant == EB_COL && d.M % 2) {  // odd contiguous (output) extent: pad, copy back
    d.X = padded_rows(d.X, d.P * d.Q, d.M);
    d.M += 1;
    d.out = run_arena_.alloc(d.M * d.R, stream_, false);
  }
  const std::size_t wb = eb_contract_workspace(&d);
  if (wb == 0) return false;
  eb_ok(eb_contract(&d, workspace(wb), wb, stream_), "eb_contract (MTTKRP term)");
  if (d.out != out.ptr)  // rows 0..M0-1 of [M0+1][R] are the first M0*R elements
    cuda_ok(cudaMemcpyAsync(out.ptr, d.out, static_cast<std::size_t>(M0 * d.R) * 8,
                            cudaMemcpyDeviceToDevice, stream_),
            "unpad");
  ++launches_fused_;
  return true;
}

const double* ScheduleExecutor::padded_rows(const double* src, std::int64_t rows,
                                            std::int64_t cols) {
  double* p = run_arena_.alloc(rows * (cols + 1), stream_, false);
  eb_ok(eb_pad_rows(src, rows, cols, p, cols + 1, stream_), "eb_pad_rows");
  return p;
}

const double* ScheduleExecutor::padded_factor(const double* u, std::int64_t rows,
                                              std::int64_t ld) {
  double* p = run_arena_.alloc((rows + 1) * ld, stream_, false);
  cuda_ok(cudaMemcpyAsync(p, u, static_cast<std::size_t>(rows * ld) * 8, cudaMemcpyDeviceToDevice,
                          stream_),
          "pad factor");
  cuda_ok(cudaMemsetAsync(p + rows * ld, 0, static_cast<std::size_t>(ld) * 8, stream_),
          "pad factor");
  return p;
}

// A term of exactly two TTM steps chained through their intermediate,
//   s0: X[P j k R], U1[j b] -> t0[P k R b]    s1: t0[P k R b], U2[k c] -> out[P R b c]
// (both TTMc-O5 terms; executor.cpp:220-235 runs them back to back) goes to
// eb_ttm2 with t0 kept on chip.
bool ScheduleExecutor::ttm2_shape(const TermPlan& term, std::int64_t rank, eb_ttm2_desc& d,
                                  std::string& natural, int& n_pre, int& n_rest) const {
  if (term.step_ids.size() != 2) return false;
  const ContractionTree& tree = pipe_.tree;
  const ContractionStep& s0 = tree.steps[static_cast<std::size_t>(term.step_ids[0])];
  const ContractionStep& s1 = tree.steps[static_cast<std::size_t>(term.step_ids[1])];
  if (s0.rhs < 0 || s1.rhs < 0 || s0.rhs_indices.size() != 2 || s1.rhs_indices.size() != 2)
    return false;
  if (tree.tensor_name(s1.lhs) != tree.tensor_name(tree.result_id(term.step_ids[0])))
    return false;
  if (tree.tensor_name(tree.result_id(term.step_ids[1])) != term.statement.output) return false;
  const std::string& xi = s0.lhs_indices;
  const char j = s0.rhs_indices[0], b = s0.rhs_indices[1];
  const char k = s1.rhs_indices[0], c = s1.rhs_indices[1];
  const auto pj = xi.find(j);
  if (pj == std::string::npos || pj + 1 >= xi.size() || xi[pj + 1] != k) return false;
  if (contains(xi, b) || contains(xi, c) || b == c) return false;
  const std::string pre = xi.substr(0, pj), rest = xi.substr(pj + 2);
  if (s0.result_indices != pre + k + rest + b || s1.lhs_indices != s0.result_indices ||
      s1.result_indices != pre + rest + b + c)
    return false;
  std::memset(&d, 0, sizeof(d));
  d.P = 1;
  for (char sy : pre) d.P *= local_len(term, sy, rank);
  d.M = 1;
  for (char sy : rest) d.M *= local_len(term, sy, rank);
  d.Q1 = local_len(term, j, rank);
  d.Q2 = local_len(term, k, rank);
  d.N1 = local_len(term, b, rank);
  d.N2 = local_len(term, c, rank);
  if (d.Q1 > 64 || d.N1 > 16 || d.N2 > 16 || d.M % 2 != 0) return false;
  natural = s1.result_indices;
  n_pre = static_cast<int>(pre.size());
  n_rest = static_cast<int>(rest.size());
  return true;
}

bool ScheduleExecutor::try_fused_ttm2(const TermPlan& term, std::int64_t rank,
                                      const std::map<std::string, const DevBlock*>& at_hand,
                                      DevBlock& out) {
  eb_ttm2_desc d;
  std::string natural;
  int n_pre = 0, n_rest = 0;
  if (!ttm2_shape(term, rank, d, natural, n_pre, n_rest)) return false;
  const ContractionTree& tree = pipe_.tree;
  const ContractionStep& s0 = tree.steps[static_cast<std::size_t>(term.step_ids[0])];
  const ContractionStep& s1 = tree.steps[static_cast<std::size_t>(term.step_ids[1])];
  const DevBlock* x = at_hand.at(tree.tensor_name(s0.lhs));
  const DevBlock* u1 = at_hand.at(tree.tensor_name(s0.rhs));
  const DevBlock* u2 = at_hand.at(tree.tensor_name(s1.rhs));
  d.X = x->ptr;
  d.U1 = u1->ptr;
  d.ldu1 = u1->shape[1];
  d.U2 = u2->ptr;
  d.ldu2 = u2->shape[1];
  if (push_rec_) {  // fused redistribution: the epilogue stores into the next term's blocks
    eb_scatter sc;
    scatter_desc(term, rank, natural, n_pre, n_rest, sc);
    out = DevBlock{};
    eb_ok(eb_ttm2_scatter(&d, &sc, stream_), "eb_ttm2_scatter (fused TTM pair + redistribution)");
  } else {
    out = new_block(term, s1.result_indices, rank, false, true);
    d.out = out.ptr;
    eb_ok(eb_ttm2(&d, stream_), "eb_ttm2 (fused TTM pair)");
  }
  ++launches_fused_;
  return true;
}

const TermPlan* ScheduleExecutor::chain_next(const TermPlan& a) const {
  const bool chain = eb::options().chain_terms != 0;
  if (!eb::options().fuse_ttm2 || !(chain || eb::options().fold_terms) || a.reduction.depth > 1)
    return nullptr;
  const TermPlan* b = nullptr;
  for (const TermPlan& t : pipe_.schedule.terms)
    if (t.index == a.index + 1) b = &t;
  if (!b || b->reduction.depth > 1) return nullptr;
  const RedistRecord* rec = find_redist(b->index, a.statement.output);
  if (!rec) return nullptr;
  // every rank's t1 block is the same block in both terms: whole self messages
  const TensorPlacement& sp = rec->plan.source;
  const TensorPlacement& dp = rec->plan.destination;
  if (sp.dist.blocks != dp.dist.blocks || sp.dist.extents != dp.dist.extents) return nullptr;
  for (std::int64_t r = 0; r < pipe_.schedule.procs; ++r)
    if (sp.block_coords_of(r) != dp.block_coords_of(r)) return nullptr;
  for (const Message& m : rec->plan.messages)
    if (!m.self) return nullptr;
  eb_ttm2_desc da, db;
  std::string na, nb;
  int p0 = 0, r0 = 0;
  for (std::int64_t r : owned_) {
    if (!ttm2_shape(a, r, da, na, p0, r0) || !ttm2_shape(*b, r, db, nb, p0, r0)) return nullptr;
    const ContractionStep& b0 = pipe_.tree.steps[static_cast<std::size_t>(b->step_ids[0])];
    if (b0.lhs_indices != na || pipe_.tree.tensor_name(b0.lhs) != a.statement.output)
      return nullptr;
    if (da.P != db.P || db.Q1 * db.Q2 * db.M != da.M * da.N1 * da.N2) return nullptr;
    if (!chain && !fold_shape(da, db)) return nullptr;
  }
  return b;
}

// eb_ttmc_fold: term B's second contraction (mode m, Q2b) is the innermost
// mode of term A's rows and term B's rows are term A's (b, c) (ttmc_fold.cu)
bool ScheduleExecutor::fold_shape(const eb_ttm2_desc& da, const eb_ttm2_desc& db) {
  return db.Q2 % 16 == 0 && db.Q2 <= 64 && da.M % db.Q2 == 0 && db.M == da.N1 * da.N2 &&
         db.N1 <= 16 && db.N2 <= 16;
}

void ScheduleExecutor::run_chain(const TermPlan& a, const TermPlan& b, std::int64_t rank,
                                 const std::map<std::string, const DevBlock*>& at_hand,
                                 DevBlock& t1, DevBlock& out) {
  eb_ttm2_desc da, db;
  std::string na, nb;
  int np = 0, nr = 0;
  ttm2_shape(a, rank, da, na, np, nr);
  ttm2_shape(b, rank, db, nb, np, nr);
  const ContractionTree& tree = pipe_.tree;
  const ContractionStep& a0 = tree.steps[static_cast<std::size_t>(a.step_ids[0])];
  const ContractionStep& a1 = tree.steps[static_cast<std::size_t>(a.step_ids[1])];
  const ContractionStep& b0 = tree.steps[static_cast<std::size_t>(b.step_ids[0])];
  const ContractionStep& b1 = tree.steps[static_cast<std::size_t>(b.step_ids[1])];
  auto input = [&](const TermPlan& t, int id) -> const DevBlock& {
    const std::string name = tree.tensor_name(id);
    const auto it = at_hand.find(name);
    if (it != at_hand.end()) return *it->second;
    return inputs_.at({t.index, name})[static_cast<std::size_t>(rank)];
  };
  const DevBlock& x = input(a, a0.lhs);
  const DevBlock& u1 = input(a, a0.rhs);
  const DevBlock& u2 = input(a, a1.rhs);
  const DevBlock& u3 = input(b, b0.rhs);
  const DevBlock& u4 = input(b, b1.rhs);
  t1 = new_block(a, na, rank, false, true);
  out = new_block(b, nb, rank, false, true);
  da.X = x.ptr;
  da.U1 = u1.ptr;
  da.ldu1 = u1.shape[1];
  da.U2 = u2.ptr;
  da.ldu2 = u2.shape[1];
  da.out = t1.ptr;
  db.X = t1.ptr;
  db.U1 = u3.ptr;
  db.ldu1 = u3.shape[1];
  db.U2 = u4.ptr;
  db.ldu2 = u4.shape[1];
  db.out = out.ptr;
  if (!eb::options().chain_terms) {  // fold: t1 (the block above) is never written
    const std::size_t fb = eb_ttmc_fold_workspace(&da, &db);
    eb_ok(eb_ttmc_fold(&da, &db, workspace(fb), fb, stream_),
          "eb_ttmc_fold (both TTMc terms, m folded into term A)");
    launches_fused_ += 2;
    return;
  }
  const std::size_t wb = eb_ttm2_chain_workspace(&da);
  eb_ok(eb_ttm2_chain(&da, &db, workspace(wb), wb, stream_), "eb_ttm2_chain (both TTMc terms)");
  ++launches_fused_;
}

namespace {
bool uniform_blocks(const TensorPlacement& pl) {
  for (std::size_t d = 0; d < pl.indices.size(); ++d) {
    const std::int64_t g = pl.term_grid.dims[static_cast<std::size_t>(pl.axes[d])];
    if (pl.dist.blocks[d] * g != pl.dist.extents[d]) return false;
    if (pl.dist.extents[d] >= (std::int64_t(1) << 31)) return false;
  }
  return true;
}
}  // namespace

const RedistRecord* ScheduleExecutor::push_record(const TermPlan& t) const {
  if (!eb::options().fuse_redistribution || t.reduction.depth > 1) return nullptr;
  if (chain_next(t)) return nullptr;  // the two terms run as one chained launch
  // the producer stores into every destination block: all of them must be
  // addressable here (one device, or the peers' mapped heaps — not NCCL)
  if (!transport_->is_virtual() && !transport_->peer_mapped()) return nullptr;
  const RedistRecord* rec = nullptr;
  for (const RedistRecord& r : pipe_.schedule.redistributions)
    if (r.from_term == t.index && r.tensor == t.statement.output) rec = &r;
  if (!rec || pipe_.schedule.procs > 64) return nullptr;
  const TensorPlacement& src = t.placement_of(t.statement.output);
  const TensorPlacement& dst = rec->plan.destination;
  if (!uniform_blocks(src) || !uniform_blocks(dst)) return nullptr;
  // every rank keeps its own block (whole self messages): the executor
  // aliases the producer's buffer, nothing to push
  bool all_self = src.dist.blocks == dst.dist.blocks && src.dist.extents == dst.dist.extents;
  for (const Message& m : rec->plan.messages) all_self = all_self && m.self;
  for (std::int64_t r = 0; all_self && r < pipe_.schedule.procs; ++r)
    all_self = src.block_coords_of(r) == dst.block_coords_of(r);
  if (all_self) return nullptr;
  std::int64_t reps = 1;
  for (std::size_t a = 0; a < dst.term_grid.dims.size(); ++a)
    if (std::find(dst.axes.begin(), dst.axes.end(), static_cast<int>(a)) == dst.axes.end())
      reps *= dst.term_grid.dims[a];
  if (reps > 8) return nullptr;
  if (match_mttkrp(t.statement).ok) return nullptr;
  // uniform source blocks: every rank's producing step has the same shape,
  // so rank 0 decides for all (and every process decides alike)
  eb_ttm2_desc d;
  std::string natural;
  int n_pre = 0, n_rest = 0;
  if (eb::options().fuse_ttm2 && ttm2_shape(t, 0, d, natural, n_pre, n_rest)) return rec;
  const ContractionStep& s = pipe_.tree.steps[static_cast<std::size_t>(t.step_ids.back())];
  if (s.rhs < 0 || s.rhs_indices.size() != 2) return nullptr;
  const std::string& xi = s.lhs_indices;
  const char j = s.rhs_indices[0], b = s.rhs_indices[1];
  const auto pos = xi.find(j);
  if (pos == std::string::npos || contains(xi, b)) return nullptr;
  std::string want = xi;
  want.erase(pos, 1);
  want.push_back(b);
  std::string sw = want, sr = s.result_indices;
  std::sort(sw.begin(), sw.end());
  std::sort(sr.begin(), sr.end());
  if (sw != sr) return nullptr;
  std::int64_t M = 1;
  for (std::size_t k = pos + 1; k < xi.size(); ++k) M *= local_len(t, xi[k], 0);
  if (M < 2 || M % 2) return nullptr;  // the COL BATCHED kernel without padding
  return rec;
}

void ScheduleExecutor::scatter_desc(const TermPlan& term, std::int64_t rank,
                                    const std::string& natural, int n_outer, int n_row,
                                    eb_scatter& sc) const {
  const TensorPlacement& dst = push_rec_->plan.destination;
  std::memset(&sc, 0, sizeof(sc));
  sc.nd = static_cast<int>(natural.size());
  sc.n_outer = n_outer;
  sc.n_row = n_row;
  const std::size_t ng = dst.term_grid.dims.size();
  std::vector<std::int64_t> gstride(ng, 1);
  for (std::size_t a = ng; a-- > 1;) gstride[a - 1] = gstride[a] * dst.term_grid.dims[a];
  for (int d = 0; d < sc.nd; ++d) {
    const char sym = natural[static_cast<std::size_t>(d)];
    const auto t = dst.indices.find(sym);
    if (t == std::string::npos) fail(errc::invalid_argument, "scatter: symbol not in destination");
    sc.ext[d] = local_len(term, sym, rank);
    sc.gbase[d] = local_lo(term, sym, rank);
    sc.block[d] = dst.dist.blocks[t];
    sc.rank_stride[d] = gstride[static_cast<std::size_t>(dst.axes[t])];
    std::int64_t ls = 1;
    for (std::size_t u = t + 1; u < dst.indices.size(); ++u) ls *= dst.dist.blocks[u];
    sc.local_stride[d] = ls;
  }
  // replicas: every combination of the destination grid axes the tensor does not span
  std::vector<std::int64_t> reps{0};
  for (std::size_t a = 0; a < ng; ++a) {
    if (std::find(dst.axes.begin(), dst.axes.end(), static_cast<int>(a)) != dst.axes.end())
      continue;
    std::vector<std::int64_t> next;
    for (std::int64_t r0 : reps)
      for (std::int64_t c = 0; c < dst.term_grid.dims[a]; ++c) next.push_back(r0 + c * gstride[a]);
    reps.swap(next);
  }
  sc.n_rep = static_cast<int>(reps.size());
  for (std::size_t k = 0; k < reps.size(); ++k) sc.rep_offset[k] = reps[k];
  for (std::int64_t r = 0; r < pipe_.schedule.procs; ++r)
    sc.dest[r] = push_dst_[static_cast<std::size_t>(r)].ptr;
}

void ScheduleExecutor::arm_push() {
  const TensorPlacement& dst = push_rec_->plan.destination;
  const std::int64_t procs = pipe_.schedule.procs;
  const bool peer = transport_->peer_mapped();
  if (peer) {
    // no rank may still read its destination block from the previous run
    cuda_ok(cudaStreamSynchronize(stream_), "push: sync");
    static_cast<PeerTransport*>(transport_)->comm().barrier();
  }
  push_dst_.assign(static_cast<std::size_t>(procs), DevBlock{});
  const std::size_t off = heap_in_slot_.count(push_rec_->to_term) ? heap_in_slot_.at(push_rec_->to_term) : 0;
  for (std::int64_t r = 0; r < procs; ++r) {
    DevBlock& b = push_dst_[static_cast<std::size_t>(r)];
    const auto bc = dst.block_coords_of(r);
    b.shape = dst.dist.shape_of(bc);
    b.base = dst.dist.base_of(bc);
    if (peer) {
      char* base = heap_peers_[static_cast<std::size_t>(r)];
      if (!base || !heap_in_slot_.count(push_rec_->to_term))
        fail(errc::invalid_argument, "push: destination heap not mapped");
      b.ptr = reinterpret_cast<double*>(base + off);
    } else if (transport_->owns(r)) {
      // (option zero_push: zeroed first, so a missing store shows in the result)
      b.ptr = run_arena_.alloc(prod(b.shape), stream_, eb::options().zero_push != 0);
    }
  }
}

DevBlock ScheduleExecutor::run_step(const TermPlan& term, int sid, std::int64_t rank,
                                    const std::map<std::string, const DevBlock*>& at_hand) {
  const ContractionStep& s = pipe_.tree.steps[static_cast<std::size_t>(sid)];
  const ContractionTree& tree = pipe_.tree;
  auto operand = [&](int id) -> const DevBlock* {
    const auto it = at_hand.find(tree.tensor_name(id));
    if (it == at_hand.end() || !it->second || !it->second->ptr)
      fail(errc::invalid_argument,
           "local_contract: missing operand block \"" + tree.tensor_name(id) + "\"");
    return it->second;
  };
  const bool is_output =
      tree.tensor_name(tree.result_id(sid)) == term.statement.output;
  // with a fused redistribution armed the output step writes no block of its own
  const bool pushing = is_output && push_rec_ != nullptr;
  DevBlock out = pushing ? DevBlock{} : new_block(term, s.result_indices, rank, false, is_output);
  const DevBlock* lhs = operand(s.lhs);
  const DevBlock* rhs = s.rhs >= 0 ? operand(s.rhs) : nullptr;

  // TTM / GEMM: X[pre, j, post] x U[j, b] -> [pre, post, b] on the DMMA kernel.
  if (rhs && s.rhs_indices.size() == 2) {
    const std::string& xi = s.lhs_indices;
    const char j = s.rhs_indices[0], b = s.rhs_indices[1];
    const auto pos = xi.find(j);
    std::string want = xi;
    if (pos != std::string::npos) want.erase(pos, 1);
    want.push_back(b);
    std::string sorted_want = want, sorted_res = s.result_indices;
    std::sort(sorted_want.begin(), sorted_want.end());
    std::sort(sorted_res.begin(), sorted_res.end());
    if (pos != std::string::npos && !contains(xi, b) && sorted_res == sorted_want) {
      std::int64_t P = 1, M = 1;
      for (std::size_t k = 0; k < pos; ++k) P *= local_len(term, xi[k], rank);
      for (std::size_t k = pos + 1; k < xi.size(); ++k) M *= local_len(term, xi[k], rank);
      const std::int64_t Q = local_len(term, j, rank), N = local_len(term, b, rank);
      // the kernel writes [pre, post, b]; a result in another order (e.g. the
      // chain's last step writing the einsum's output order) is permuted after
      const bool permuted = s.result_indices != want;
      double* natural =
          permuted && !pushing ? run_arena_.alloc(P * M * N, stream_, false) : out.ptr;
      eb_contract_desc d;
      std::memset(&d, 0, sizeof(d));
      d.R = N;
      d.X = lhs->ptr;
      d.U = rhs->ptr;
      d.ldu = N;
      d.out = natural;
      bool ok = false, unpad = false;
      if (M > 1 && pushing && M % 2 == 0) {
        // fused redistribution: the epilogue stores the natural [pre, post, b]
        // elements straight into the next term's destination blocks
        d.variant = EB_COL;
        d.mode = EB_BATCHED;
        d.P = P;
        d.Q = Q;
        d.M = M;
        eb_scatter sc;
        scatter_desc(term, rank, want, static_cast<int>(pos),
                     static_cast<int>(xi.size() - pos - 1), sc);
        d.out = sc.dest[0];  // not written (the workspace query wants a non-null output)
        const std::size_t wb = eb_contract_workspace(&d);
        if (wb == 0) fail(errc::invalid_argument, "scatter TTM: no contraction plan");
        eb_ok(eb_contract_scatter(&d, &sc, workspace(wb), wb, stream_),
              "eb_contract_scatter (TTM step + redistribution)");
        ++launches_ttm_;
        return DevBlock{};
      }
      if (pushing)
        fail(errc::invalid_argument, "fused redistribution: the output step has no scatter path");
      if (M > 1) {  // contract a strided mode: batched COL
        d.variant = EB_COL;
        d.mode = EB_BATCHED;
        d.P = P;
        d.Q = Q;
        d.M = M;
        if (M % 2) {  // odd contiguous extent: padded X rows, output unpadded after
          d.X = padded_rows(d.X, P * Q, M);
          d.M = M + 1;
          d.out = run_arena_.alloc(P * (M + 1) * N, stream_, false);
          unpad = true;
        }
        ok = true;
      } else {  // contract the last mode: GEMM (ROW)
        d.variant = EB_ROW;
        d.mode = EB_REDUCE;
        d.P = 1;
        d.M = P;
        d.Q = 1;
        d.L = Q;
        if (Q % 2) {  // odd contracted extent: zero-padded rows of X and U
          d.X = padded_rows(d.X, P, Q);
          d.U = padded_factor(rhs->ptr, Q, N);
          d.L = Q + 1;
        }
        ok = true;
      }
      if (ok) {
        const std::size_t wb = eb_contract_workspace(&d);
        if (wb > 0) {
          eb_ok(eb_contract(&d, workspace(wb), wb, stream_), "eb_contract (TTM step)");
          if (unpad) {
            const std::int64_t sshape[3] = {P, M + 1, N}, dshape[3] = {P, M, N};
            const std::int64_t lo[3] = {0, 0, 0}, hi[3] = {P, M, N};
            eb_ok(eb_copy_box(3, d.out, sshape, natural, dshape, lo, hi, lo, stream_), "unpad");
          }
          if (permuted) {
            // out dim k is natural dim want.find(result[k])
            const int nd = static_cast<int>(want.size());
            std::vector<std::int64_t> nshape(static_cast<std::size_t>(nd));
            std::vector<int> perm(static_cast<std::size_t>(nd));
            for (int k = 0; k < nd; ++k) {
              nshape[static_cast<std::size_t>(k)] = local_len(term, want[static_cast<std::size_t>(k)], rank);
              perm[static_cast<std::size_t>(k)] =
                  static_cast<int>(want.find(s.result_indices[static_cast<std::size_t>(k)]));
            }
            eb_ok(eb_permute(nd, natural, nshape.data(), perm.data(), out.ptr, stream_),
                  "eb_permute");
          }
          ++launches_ttm_;
          return out;
        }
      }
    }
  }
  if (pushing)
    fail(errc::invalid_argument, "fused redistribution: the output step has no scatter path");
  std::int64_t ext[256] = {0};
  for (char c : s.lhs_indices) ext[static_cast<unsigned char>(c)] = local_len(term, c, rank);
  for (char c : s.rhs_indices) ext[static_cast<unsigned char>(c)] = local_len(term, c, rank);
  eb_ok(eb_step_generic(s.lhs_indices.c_str(), rhs ? s.rhs_indices.c_str() : "",
                        s.result_indices.c_str(), ext, lhs->ptr, rhs ? rhs->ptr : nullptr, out.ptr,
                        stream_),
        "eb_step_generic");
  ++launches_generic_;
  return out;
}

void ScheduleExecutor::join() {
  if (!comm_pending_) return;
  cuda_ok(cudaStreamWaitEvent(stream_, ev_comm_, 0), "join: wait for the reduction");
  comm_pending_ = false;
}

void ScheduleExecutor::capture() {
  if (transport_->peer_mapped())
    fail(errc::invalid_argument,
         "capture: the peer transport meets its peers on the host between kernels; "
         "graphs need the virtual or NCCL transport");
  if (stream_ == nullptr || stream_ == cudaStreamLegacy || stream_ == cudaStreamPerThread)
    fail(errc::invalid_argument, "capture: needs an explicitly created stream");
  if (graph_exec_) {
    cuda_ok(cudaGraphExecDestroy(graph_exec_), "graph destroy");
    graph_exec_ = nullptr;
  }
  // warm run: the recycling arena keeps every block of the run, the
  // workspace and the transport's buffers reach their final sizes
  run_arena_.set_recycle(true, stream_);
  execute();
  join();
  cuda_ok(cudaStreamSynchronize(stream_), "capture: warm run");
  const long long mallocs0 = run_arena_.mallocs();
  const std::size_t ws0 = workspace_bytes_;
  const long long n0 = eb_launch_count();
  eb::set_capturing(true);
  cuda_ok(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
  cudaGraph_t g = nullptr;
  try {
    execute();
    join();
  } catch (...) {
    cudaStreamEndCapture(stream_, &g);
    if (g) cudaGraphDestroy(g);
    eb::set_capturing(false);
    throw;
  }
  const cudaError_t e = cudaStreamEndCapture(stream_, &g);
  eb::set_capturing(false);
  cuda_ok(e, "end capture");
  graph_launches_ = eb_launch_count() - n0;
  if (run_arena_.mallocs() != mallocs0 || workspace_bytes_ != ws0) {
    cudaGraphDestroy(g);
    fail(errc::invalid_argument, "capture: the captured run allocated memory (blocks differ "
                                 "from the warm run)");
  }
  const cudaError_t ie = cudaGraphInstantiateWithFlags(&graph_exec_, g, 0);
  cudaGraphDestroy(g);
  cuda_ok(ie, "graph instantiate");
}

void ScheduleExecutor::replay() {
  if (!graph_exec_) fail(errc::invalid_argument, "replay: no captured run (call capture)");
  join();
  cuda_ok(cudaGraphLaunch(graph_exec_, stream_), "graph launch");
  eb::count_launches(graph_launches_);
}

std::int64_t ScheduleExecutor::reduce(const TensorPlacement& place, const ReductionGroup& grp,
                                      std::vector<DevBlock>& blocks, bool last_term) {
  if (!async_reduce_ || grp.depth <= 1)
    return transport_->allreduce(place, grp, blocks, comm_.per_rank_sent, stream_);
  // the transport's one communication stream: every executor of this
  // process issues its collectives there, in program order
  cudaStream_t cs = transport_->comm_stream();
  if (!ev_compute_) {
    cuda_ok(cudaEventCreateWithFlags(&ev_compute_, cudaEventDisableTiming), "event");
    cuda_ok(cudaEventCreateWithFlags(&ev_comm_, cudaEventDisableTiming), "event");
  }
  join();  // one reduction in flight per executor
  cuda_ok(cudaEventRecord(ev_compute_, stream_), "event record");
  cuda_ok(cudaStreamWaitEvent(cs, ev_compute_, 0), "stream wait");
  const std::int64_t v = transport_->allreduce(place, grp, blocks, comm_.per_rank_sent, cs);
  cuda_ok(cudaEventRecord(ev_comm_, cs), "event record");
  comm_pending_ = true;
  if (!last_term) join();  // the next term reads it on the compute stream
  return v;
}

void ScheduleExecutor::execute() {
  if (!staged_) fail(errc::invalid_argument, "execute: inputs not staged");
  join();  // the previous run's reduction still owns its output blocks
  run_arena_.release(stream_);
  store_.clear();
  comm_ = CommStats{};
  comm_.per_rank_sent.assign(static_cast<std::size_t>(pipe_.schedule.procs), 0);
  launches_fused_ = launches_ttm_ = launches_generic_ = 0;
  redistributions_fused_ = 0;
  const std::int64_t procs = pipe_.schedule.procs;
  pushed_.clear();
  chain_out_.clear();
  push_rec_ = nullptr;
  prepare_heap();

  for (const TermPlan& term : pipe_.schedule.terms) {
    std::map<std::string, std::vector<DevBlock>*> arrays;
    for (const AccessArray& a : term.statement.arrays) {
      if (a.tensor == term.statement.output) continue;
      if (a.tensor.rfind("in", 0) == 0) {
        arrays[a.tensor] = &inputs_.at({term.index, a.tensor});
        continue;
      }
      if (const RedistRecord* rec = find_redist(term.index, a.tensor)) {
        if (pushed_.count({term.index, a.tensor})) {
          // fused into the producer's epilogue (push): only the accounting
          // of apply_plan remains (redistribute.cpp:185-206, executor.cpp:193-198)
          comm_.events.push_back(
              {"redistribute", term.index, a.tensor, rec->plan.transmitted_volume});
          comm_.redistribute_volume += rec->plan.transmitted_volume;
          for (const Message& m : rec->plan.messages)
            if (!m.self) comm_.per_rank_sent[static_cast<std::size_t>(m.src_rank)] += m.elements;
          arrays[a.tensor] = &store_.at({term.index, a.tensor});
          continue;
        }
        const auto& src = store_.at({rec->from_term, a.tensor});
        std::vector<DevBlock> dst(static_cast<std::size_t>(procs));
        const TensorPlacement& dp = rec->plan.destination;
        // A rank whose only incoming message is a self message covering its
        // whole (identically shaped) block keeps the producer's buffer: the
        // reference copies it (apply_plan), the result is the same block.
        std::vector<int> incoming(static_cast<std::size_t>(procs), 0);
        std::vector<const Message*> only(static_cast<std::size_t>(procs), nullptr);
        for (const Message& m : rec->plan.messages) {
          ++incoming[static_cast<std::size_t>(m.dst_rank)];
          only[static_cast<std::size_t>(m.dst_rank)] = &m;
        }
        std::vector<char> alias(static_cast<std::size_t>(procs), 0);
        for (std::int64_t r : owned_) {
          DevBlock& b = dst[static_cast<std::size_t>(r)];
          const auto bc = dp.block_coords_of(r);
          b.shape = dp.dist.shape_of(bc);
          b.base = dp.dist.base_of(bc);
          const Message* m = only[static_cast<std::size_t>(r)];
          const DevBlock& sb = src[static_cast<std::size_t>(r)];
          bool whole = incoming[static_cast<std::size_t>(r)] == 1 && m->self &&
                       m->src_rank == r && sb.ptr && sb.shape == b.shape;
          for (std::size_t d = 0; whole && d < b.shape.size(); ++d)
            whole = m->oy_lo[d] == 0 && m->ox_lo[d] == 0 && m->oy_hi[d] == b.shape[d] &&
                    m->ox_hi[d] == b.shape[d];
          if (whole) {
            alias[static_cast<std::size_t>(r)] = 1;
            b.ptr = sb.ptr;
          } else {
            b.ptr = run_arena_.alloc(prod(b.shape), stream_, true);
          }
        }
        RedistributionPlan todo = rec->plan;
        todo.messages.clear();
        for (const Message& m : rec->plan.messages)
          if (!(m.self && alias[static_cast<std::size_t>(m.dst_rank)])) todo.messages.push_back(m);
        // (collective for the peer transport: its barriers need every rank)
        if (!todo.messages.empty() || transport_->peer_mapped())
          transport_->redistribute(todo, src, dst, stream_);
        comm_.events.push_back(
            {"redistribute", term.index, a.tensor, rec->plan.transmitted_volume});
        comm_.redistribute_volume += rec->plan.transmitted_volume;
        for (const Message& m : rec->plan.messages)
          if (!m.self) comm_.per_rank_sent[static_cast<std::size_t>(m.src_rank)] += m.elements;
        store_[{term.index, a.tensor}] = std::move(dst);
        arrays[a.tensor] = &store_.at({term.index, a.tensor});
        continue;
      }
      int from = -1;
      for (const TermPlan& prev : pipe_.schedule.terms)
        if (prev.index < term.index && prev.statement.output == a.tensor) from = prev.index;
      if (from < 0) fail(errc::invalid_argument, "run: no producer for \"" + a.tensor + "\"");
      store_[{term.index, a.tensor}] = store_.at({from, a.tensor});
      arrays[a.tensor] = &store_.at({term.index, a.tensor});
    }

    const TensorPlacement& out_place = term.placement_of(term.statement.output);
    std::vector<DevBlock> out_blocks(static_cast<std::size_t>(procs));
    push_rec_ = push_record(term);
    if (push_rec_) arm_push();
    const TermPlan* chained = chain_next(term);
    for (std::int64_t rank : owned_) {
      std::map<std::string, const DevBlock*> at_hand;
      for (auto& kv : arrays) at_hand[kv.first] = &(*kv.second)[static_cast<std::size_t>(rank)];
      if (chain_out_.count({term.index, rank})) {  // computed with the previous term
        out_blocks[static_cast<std::size_t>(rank)] = chain_out_.at({term.index, rank});
        continue;
      }
      DevBlock result;
      if (chained) {
        DevBlock out_next;
        run_chain(term, *chained, rank, at_hand, result, out_next);
        out_blocks[static_cast<std::size_t>(rank)] = result;
        chain_out_[{chained->index, rank}] = out_next;
        continue;
      }
      if (try_fused_mttkrp(term, rank, at_hand, result) ||
          (eb::options().fuse_ttm2 && try_fused_ttm2(term, rank, at_hand, result))) {
        out_blocks[static_cast<std::size_t>(rank)] = result;
        continue;
      }
      std::map<std::string, DevBlock> scratch;
      for (int sid : term.step_ids) {
        DevBlock r = run_step(term, sid, rank, at_hand);
        const std::string name = pipe_.tree.tensor_name(pipe_.tree.result_id(sid));
        if (name == term.statement.output) {
          out_blocks[static_cast<std::size_t>(rank)] = r;
        } else {
          scratch[name] = r;
          at_hand[name] = &scratch[name];
        }
      }
    }
    if (push_rec_) {  // the term's output is already in the next term's blocks
      if (transport_->peer_mapped()) {
        cuda_ok(cudaStreamSynchronize(stream_), "push: sync");
        static_cast<PeerTransport*>(transport_)->comm().barrier();  // every block complete
      }
      store_[{push_rec_->to_term, push_rec_->tensor}] = push_dst_;
      pushed_.insert({push_rec_->to_term, push_rec_->tensor});
      ++redistributions_fused_;
      push_rec_ = nullptr;
    }
    map_peer_blocks(term, out_blocks);
    const std::int64_t v = reduce(out_place, term.reduction, out_blocks,
                                  &term == &pipe_.schedule.terms.back());
    if (term.reduction.depth > 1) {
      comm_.events.push_back({"allreduce", term.index, term.statement.output, v});
      comm_.allreduce_volume += v;
    }
    store_[{term.index, term.statement.output}] = std::move(out_blocks);
  }
}

bool ScheduleExecutor::execute_pair(ScheduleExecutor& m1) {
  if (!staged_ || !m1.staged_) fail(errc::invalid_argument, "execute_pair: inputs not staged");
  if (pipe_.schedule.terms.size() != 1 || m1.pipe_.schedule.terms.size() != 1) return false;
  if (pipe_.schedule.procs != m1.pipe_.schedule.procs || owned_ != m1.owned_) return false;
  if (m1.stream_ != stream_) return false;  // one stream orders the kernel and both reductions
  const TermPlan& t0 = pipe_.schedule.terms[0];
  const TermPlan& t1 = m1.pipe_.schedule.terms[0];
  const MttkrpMatch a = match_mttkrp(t0.statement), b = match_mttkrp(t1.statement);
  if (!a.ok || !b.ok || a.x_idx.size() != 3 || a.x_idx != b.x_idx || a.out_mode != 0 ||
      b.out_mode != 1 || a.rank_sym != b.rank_sym)
    return false;
  // same grid over the same iteration dims: identical X / factor blocks per rank
  if (t0.grid.order != t1.grid.order || t0.grid.dims != t1.grid.dims || t0.blocks != t1.blocks)
    return false;
  const auto& in0 = inputs_;
  const auto& in1 = m1.inputs_;
  auto blocks_of = [](const std::map<std::pair<int, std::string>, std::vector<DevBlock>>& m,
                      const std::string& name) -> const std::vector<DevBlock>* {
    const auto it = m.find({0, name});
    return it == m.end() ? nullptr : &it->second;
  };
  const auto* x0 = blocks_of(in0, a.x_name);
  const auto* x1 = blocks_of(in1, b.x_name);
  const auto* c0 = blocks_of(in0, a.factor_of[2]);
  const auto* c1 = blocks_of(in1, b.factor_of[2]);
  const auto* bf = blocks_of(in0, a.factor_of[1]);
  const auto* af = blocks_of(in1, b.factor_of[0]);
  if (!x0 || !x1 || !c0 || !c1 || !bf || !af) return false;
  for (std::int64_t r : owned_) {  // X and C must be the very same device blocks
    const auto i = static_cast<std::size_t>(r);
    if ((*x0)[i].ptr != (*x1)[i].ptr || (*c0)[i].ptr != (*c1)[i].ptr) return false;
  }
  // kernel preconditions, per owned rank
  std::vector<eb_contract_desc> descs;
  for (std::int64_t r : owned_) {
    const auto i = static_cast<std::size_t>(r);
    eb_contract_desc d;
    std::memset(&d, 0, sizeof(d));
    d.variant = EB_ROW;
    d.mode = EB_REDUCE;
    d.P = 1;
    d.M = local_len(t0, a.x_idx[0], r);
    d.Q = local_len(t0, a.x_idx[1], r);
    d.L = local_len(t0, a.x_idx[2], r);
    d.R = local_len(t0, a.rank_sym, r);
    d.X = (*x0)[i].ptr;
    d.U = (*c0)[i].ptr;
    d.ldu = (*c0)[i].shape[1];
    d.n_mid = 1;
    d.mid[0].ptr = (*bf)[i].ptr;
    d.mid[0].extent = (*bf)[i].shape[0];
    d.mid[0].ld = (*bf)[i].shape[1];
    d.out = (*x0)[i].ptr;  // placeholder for the shape query (set per launch below)
    if (d.L % 2 || eb_mttkrp2_workspace(&d) == 0) return false;
    descs.push_back(d);
  }

  for (ScheduleExecutor* e : {this, &m1}) {
    e->join();
    e->prepare_heap();
    e->run_arena_.release(e->stream_);
    e->store_.clear();
    e->comm_ = CommStats{};
    e->comm_.per_rank_sent.assign(static_cast<std::size_t>(pipe_.schedule.procs), 0);
    e->launches_fused_ = e->launches_ttm_ = e->launches_generic_ = 0;
  }
  const std::int64_t procs = pipe_.schedule.procs;
  std::vector<DevBlock> out0(static_cast<std::size_t>(procs)), out1(static_cast<std::size_t>(procs));
  std::size_t k = 0;
  for (std::int64_t r : owned_) {
    eb_contract_desc& d = descs[k++];
    const auto i = static_cast<std::size_t>(r);
    out0[i] = new_block(t0, t0.placement_of(t0.statement.output).indices, r, false, true);
    out1[i] = m1.new_block(t1, t1.placement_of(t1.statement.output).indices, r, false, true);
    d.out = out0[i].ptr;
    const std::size_t wb = eb_mttkrp2_workspace(&d);
    eb_ok(eb_mttkrp2(&d, (*af)[i].ptr, (*af)[i].shape[1], out1[i].ptr, workspace(wb), wb, stream_),
          "eb_mttkrp2 (dimension-tree pair)");
    ++launches_fused_;
  }
  struct Side {
    ScheduleExecutor* e;
    const TermPlan* t;
    std::vector<DevBlock>* out;
  };
  map_peer_blocks(t0, out0);
  m1.map_peer_blocks(t1, out1);
  for (const Side& sd : {Side{this, &t0, &out0}, Side{&m1, &t1, &out1}}) {
    const TensorPlacement& place = sd.t->placement_of(sd.t->statement.output);
    const std::int64_t v = sd.e->reduce(place, sd.t->reduction, *sd.out, true);
    if (sd.t->reduction.depth > 1) {
      sd.e->comm_.events.push_back({"allreduce", sd.t->index, sd.t->statement.output, v});
      sd.e->comm_.allreduce_volume += v;
    }
    sd.e->store_[{sd.t->index, sd.t->statement.output}] = std::move(*sd.out);
  }
  return true;
}

std::vector<std::int64_t> ScheduleExecutor::output_shape() const {
  return pipe_.spec.shape_of(pipe_.spec.output);
}

void ScheduleExecutor::gather(double* host_out) {
  join();
  const TermPlan& last = pipe_.schedule.terms.back();
  const TensorPlacement& place = last.placement_of(last.statement.output);
  auto& blocks = store_.at({last.index, last.statement.output});
  transport_->gather_to_root(place, blocks, stream_);
  if (!transport_->owns(0) && !transport_->is_virtual()) {
    cuda_ok(cudaStreamSynchronize(stream_), "sync");
    transport_->gather_done(blocks, stream_);
    return;  // only rank 0 assembles
  }
  if (!host_out) fail(errc::invalid_argument, "gather: rank 0 needs an output buffer");
  const auto gshape = place.dist.extents;
  const std::int64_t procs = place.term_grid.total();
  for (std::int64_t r = 0; r < procs; ++r) {
    if (!place.is_canonical(r)) continue;
    const DevBlock& b = blocks[static_cast<std::size_t>(r)];
    const auto shape = place.dist.shape_of(place.block_coords_of(r));
    const auto base = place.dist.base_of(place.block_coords_of(r));
    if (!b.ptr) fail(errc::invalid_argument, "gather: canonical block of rank " +
                                                 std::to_string(r) + " not available");
    copy_box_host(false, host_out, gshape, shape, base, b.ptr, stream_);
  }
  cuda_ok(cudaStreamSynchronize(stream_), "sync");
  transport_->gather_done(blocks, stream_);
}

void ScheduleExecutor::verify(const std::vector<const double*>& globals, const double* host_out,
                              double tol, SimulationReport& rep) {
  // Device-side naive evaluation of the whole kernel (evaluate.cpp:7-63 on
  // the GPU), compared elementwise with the gathered output.
  const auto& spec = pipe_.spec;
  std::vector<double*> dev;
  std::vector<std::string> idx;
  for (std::size_t k = 0; k < spec.inputs.size(); ++k) {
    const std::int64_t n = shape_product(spec.shape_of(spec.inputs[k]));
    double* p = run_arena_.alloc(n, stream_, false);
    cuda_ok(cudaMemcpyAsync(p, globals[k], static_cast<std::size_t>(n) * 8, cudaMemcpyHostToDevice,
                            stream_),
            "H2D");
    dev.push_back(p);
    idx.push_back(spec.inputs[k]);
  }
  const std::int64_t on = shape_product(spec.shape_of(spec.output));
  double* want_d = run_arena_.alloc(on, stream_, false);
  std::int64_t ext[256] = {0};
  for (const auto& kv : spec.extents) ext[static_cast<unsigned char>(kv.first)] = kv.second;
  std::vector<const char*> cidx;
  for (auto& s : idx) cidx.push_back(s.c_str());
  std::vector<const double*> cdev(dev.begin(), dev.end());
  eb_ok(eb_einsum_generic(static_cast<int>(cidx.size()), cidx.data(), spec.output.c_str(), ext,
                          cdev.data(), want_d, stream_),
        "eb_einsum_generic (verify)");
  DenseTensor want(spec.shape_of(spec.output));
  cuda_ok(cudaMemcpyAsync(want.data.data(), want_d, static_cast<std::size_t>(on) * 8,
                          cudaMemcpyDeviceToHost, stream_),
          "D2H");
  cuda_ok(cudaStreamSynchronize(stream_), "sync");
  DenseTensor got(spec.shape_of(spec.output));
  std::memcpy(got.data.data(), host_out, static_cast<std::size_t>(on) * 8);
  rep.verified = true;
  rep.tolerance = tol;
  rep.max_error = max_rel_error(got, want);
  rep.pass = rep.max_error <= tol;
}

}  // namespace gpu

namespace {

// How einplan::run / einplan_run_json place the ranks (procs =
// GPU count).  Runtime configuration of the outer ABI, read per call like the
// reference's EINPLAN_MAX_POINTS (capi.cpp:80-87):
//   EINPLAN_EXEC      "virtual" forces every rank onto the current device;
//   EINPLAN_DEVICES   "d0,d1,..." explicit rank -> device map (cycled), e.g.
//                     "0,0" runs two rank threads on one GPU (peer transport);
//   EINPLAN_TRANSPORT "nccl" | "hybrid" | "peer" for the one-thread-per-GPU mode.
// Default: one host thread per GPU on devices 0..procs-1 when procs <= the
// visible GPU count (hybrid when the devices are distinct), else virtual ranks.
struct ExecChoice {
  bool threads = false;
  std::vector<int> dev;
  std::string transport = "virtual";
};

ExecChoice choose_execution(std::int64_t procs) {
  ExecChoice c;
  const char* mode = std::getenv("EINPLAN_EXEC");
  if (mode && std::string(mode) == "virtual") return c;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
    (void)cudaGetLastError();
    ndev = 0;
  }
  std::vector<int> list;
  if (const char* v = std::getenv("EINPLAN_DEVICES")) {
    std::string s(v);
    std::size_t pos = 0;
    while (pos <= s.size()) {
      const std::size_t q = s.find(',', pos);
      const std::string item = s.substr(pos, q == std::string::npos ? std::string::npos : q - pos);
      if (!item.empty()) {
        const int d = std::atoi(item.c_str());
        if (d < 0 || d >= ndev)
          fail(errc::invalid_argument, "EINPLAN_DEVICES: no device " + item);
        list.push_back(d);
      }
      if (q == std::string::npos) break;
      pos = q + 1;
    }
  }
  if (list.empty()) {
    if (procs > ndev || procs > gpu::kMaxPeers) return c;  // more ranks than GPUs: virtual
    for (int r = 0; r < procs; ++r) list.push_back(r);
  }
  if (procs > gpu::kMaxPeers) fail(errc::invalid_argument, "run: at most 64 rank threads");
  c.threads = true;
  for (std::int64_t r = 0; r < procs; ++r) c.dev.push_back(list[static_cast<std::size_t>(r) % list.size()]);
  const std::set<int> distinct(c.dev.begin(), c.dev.end());
  c.transport = "peer";
#ifdef EB_HAVE_NCCL
  if (procs > 1 && distinct.size() == c.dev.size()) c.transport = "hybrid";
#endif
  if (const char* t = std::getenv("EINPLAN_TRANSPORT")) {
    const std::string ts(t);
    if (ts == "peer") {
      c.transport = "peer";
    } else if (ts == "nccl" || ts == "hybrid") {
#ifndef EB_HAVE_NCCL
      fail(errc::invalid_argument, "EINPLAN_TRANSPORT=nccl: built without NCCL");
#endif
      if (distinct.size() != c.dev.size())
        fail(errc::invalid_argument, "EINPLAN_TRANSPORT=" + ts + " needs one distinct GPU per rank");
      c.transport = ts;
    } else {
      fail(errc::invalid_argument, "EINPLAN_TRANSPORT: \"nccl\", \"hybrid\" or \"peer\"");
    }
  }
  return c;
}

using gpu::cuda_ok;

// The tail of run() on the rank that holds the gathered output.
void finish_report(gpu::ScheduleExecutor& ex, const std::vector<const double*>& globals,
                   const RunOptions& opts, SimulationReport& rep) {
  rep.comm = ex.comm();
  if (opts.corrupt_output && !rep.output.data.empty()) rep.output.data[0] += 1.0;
  if (opts.verify) ex.verify(globals, rep.output.data.data(), opts.tolerance, rep);
}

// One host thread per GPU (rank r on device dev[r]); every thread owns its
// rank's blocks, the collectives run over NCCL or peer memory.
void run_threads(const Pipeline& pipe, const std::vector<const double*>& globals,
                 const RunOptions& opts, const ExecChoice& ch, SimulationReport& rep) {
  const int procs = static_cast<int>(pipe.schedule.procs);
  std::shared_ptr<gpu::PeerShared> shared;
  std::vector<void*> comms(static_cast<std::size_t>(procs), nullptr);
  if (ch.transport == "peer" || ch.transport == "hybrid") shared = gpu::PeerShared::for_threads(procs);
  if (ch.transport != "peer") {
#ifdef EB_HAVE_NCCL
    std::vector<ncclComm_t> c(static_cast<std::size_t>(procs));
    const ncclResult_t r = ncclCommInitAll(c.data(), procs, ch.dev.data());
    if (r != ncclSuccess)
      throw eb::DeviceError(std::string("ncclCommInitAll: ") + ncclGetErrorString(r));
    for (int k = 0; k < procs; ++k) comms[static_cast<std::size_t>(k)] = c[static_cast<std::size_t>(k)];
#endif
  }
  std::vector<std::exception_ptr> errs(static_cast<std::size_t>(procs));
  std::vector<std::string> msgs(static_cast<std::size_t>(procs));
  auto body = [&](int r) {
    std::unique_ptr<gpu::Transport> tp;
    try {
      cuda_ok(cudaSetDevice(ch.dev[static_cast<std::size_t>(r)]), "cudaSetDevice");
      std::unique_ptr<gpu::Transport> nccl;
#ifdef EB_HAVE_NCCL
      if (comms[static_cast<std::size_t>(r)]) {
        nccl = std::make_unique<gpu::NcclTransport>(comms[static_cast<std::size_t>(r)], procs, r);
        comms[static_cast<std::size_t>(r)] = nullptr;  // owned by the transport now
      }
#endif
      if (shared)  // peer, or hybrid: NCCL allreduce + fused redistribution over peer memory
        tp = std::make_unique<gpu::PeerTransport>(std::make_shared<gpu::PeerComm>(shared, r),
                                                  procs, std::move(nccl));
      else
        tp = std::move(nccl);
      cudaStream_t st = nullptr;
      cuda_ok(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
      {
        gpu::ScheduleExecutor ex(pipe, tp.get(), st);
        ex.stage_inputs(globals);
        ex.execute();
        if (r == 0) {
          rep.output = DenseTensor(pipe.spec.shape_of(pipe.spec.output));
          ex.gather(rep.output.data.data());
          finish_report(ex, globals, opts, rep);
        } else {
          ex.gather(nullptr);
        }
      }
      cudaStreamDestroy(st);
    } catch (const std::exception& e) {
      errs[static_cast<std::size_t>(r)] = std::current_exception();
      msgs[static_cast<std::size_t>(r)] = e.what();
      if (shared) shared->abort();
    } catch (...) {
      errs[static_cast<std::size_t>(r)] = std::current_exception();
      if (shared) shared->abort();
    }
  };
  int prev = 0;
  cudaGetDevice(&prev);
  std::vector<std::thread> th;
  for (int r = 0; r < procs; ++r) th.emplace_back(body, r);
  for (auto& t : th) t.join();
  cudaSetDevice(prev);
#ifdef EB_HAVE_NCCL
  for (void* c : comms)
    if (c) ncclCommDestroy(static_cast<ncclComm_t>(c));
#endif
  // report the failing rank's own error, not a peer's "another rank failed"
  std::exception_ptr first;
  for (int r = 0; r < procs; ++r) {
    const auto& e = errs[static_cast<std::size_t>(r)];
    if (!e) continue;
    if (!first) first = e;
    if (msgs[static_cast<std::size_t>(r)].find("another rank failed") == std::string::npos) {
      first = e;
      break;
    }
  }
  if (first) std::rethrow_exception(first);
  rep.exec_mode = "devices";
  rep.devices = ch.dev;
  rep.transport = ch.transport;
}

}  // namespace

// The reference's C++ entry point (executor.cpp:156-263) on the GPUs: one
// host thread per GPU when procs fits the visible devices, else every
// virtual rank on the current device (choose_execution).
SimulationReport run(const Schedule& schedule, const EinsumSpec& spec, const ContractionTree& tree,
                     const std::vector<DenseTensor>& inputs, const RunOptions& opts) {
  if (inputs.size() != static_cast<std::size_t>(tree.n_inputs))
    fail(errc::invalid_argument, "run: operand count mismatch");
  for (std::size_t k = 0; k < inputs.size(); ++k)
    if (inputs[k].shape != spec.shape_of(spec.inputs[k]))
      fail(errc::invalid_argument,
           "run: operand " + std::to_string(k) + " does not match \"" + spec.inputs[k] + "\"");
  Pipeline pipe;
  pipe.spec = spec;
  pipe.tree = tree;
  pipe.schedule = schedule;
  std::vector<const double*> globals;
  for (const auto& t : inputs) globals.push_back(t.data.data());
  SimulationReport rep;
  rep.seed = opts.seed;
  const ExecChoice ch = choose_execution(schedule.procs);
  if (ch.threads) {
    run_threads(pipe, globals, opts, ch, rep);
    return rep;
  }
  gpu::VirtualTransport vt(schedule.procs);
  cudaStream_t st = nullptr;
  gpu::ScheduleExecutor ex(pipe, &vt, st);
  ex.stage_inputs(globals);
  ex.execute();
  rep.output = DenseTensor(spec.shape_of(spec.output));
  ex.gather(rep.output.data.data());
  finish_report(ex, globals, opts, rep);
  int dev = 0;
  cudaGetDevice(&dev);
  rep.exec_mode = "virtual";
  rep.devices = {dev};
  rep.transport = "virtual";
  return rep;
}

std::int64_t CommStats::max_rank_sent() const {
  std::int64_t m = 0;
  for (auto v : per_rank_sent) m = std::max(m, v);
  return m;
}

}  // namespace einplan
