// GPU schedule executor (see executor.cpp).
#pragma once

#include <cstdlib>

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "einplan_b200.h"
#include "einplan_host.hpp"
#include "peer.hpp"

namespace einplan {
namespace gpu {

// One rank's block of a tensor in device memory (row-major, global base).
struct DevBlock {
  double* ptr = nullptr;
  std::vector<std::int64_t> shape;
  std::vector<std::int64_t> base;
  std::int64_t size() const {
    std::int64_t n = 1;
    for (auto d : shape) n *= d;
    return n;
  }
};

// Stream-ordered device allocations released together.
class DeviceArena {
 public:
  ~DeviceArena();
  double* alloc(std::int64_t elems, cudaStream_t st, bool zero);
  void release(cudaStream_t st);
  // Recycling: release() keeps the blocks and alloc() hands back a kept
  // block of the same size before allocating — a captured CUDA graph then
  // replays on fixed addresses (and a run allocates nothing).
  void set_recycle(bool on, cudaStream_t st);
  long long mallocs() const { return mallocs_; }

 private:
  std::vector<std::pair<std::size_t, void*>> live_, kept_;
  bool recycle_ = false;
  long long mallocs_ = 0;
};

// How ranks exchange data: all virtual ranks on one device; one rank per
// process (or host thread) over NCCL; or one rank per process / thread over
// peer memory (PeerTransport: CUDA IPC or P2P pointers plus a host barrier).
// Executors built `like=` another share its transport, and with it one
// communication stream: every rank then issues its collectives in the same
// order on one stream (NCCL's rule for operations on several communicators).
class Transport {
 public:
  virtual ~Transport();
  virtual bool owns(std::int64_t rank) const = 0;
  virtual bool is_virtual() const = 0;
  // blocks of non-owned ranks are peer-mapped device pointers (PeerTransport)
  virtual bool peer_mapped() const { return false; }
  virtual std::int64_t allreduce(const TensorPlacement& place, const ReductionGroup& grp,
                                 std::vector<DevBlock>& blocks,
                                 std::vector<std::int64_t>& per_rank_sent, cudaStream_t st) = 0;
  virtual void redistribute(const RedistributionPlan& plan, const std::vector<DevBlock>& src,
                            std::vector<DevBlock>& dst, cudaStream_t st) = 0;
  // make the canonical output blocks readable by rank 0 (collective)
  virtual void gather_to_root(const TensorPlacement& place, std::vector<DevBlock>& blocks,
                              cudaStream_t st) = 0;
  // after rank 0 copied them out: release staging (collective)
  virtual void gather_done(std::vector<DevBlock>& blocks, cudaStream_t st) {
    (void)blocks;
    (void)st;
  }
  // the process's communication stream (created on first use, on the
  // current device)
  cudaStream_t comm_stream();

 private:
  cudaStream_t comm_stream_ = nullptr;
};

class VirtualTransport final : public Transport {
 public:
  explicit VirtualTransport(std::int64_t procs) : procs_(procs) {}
  bool owns(std::int64_t r) const override { return r >= 0 && r < procs_; }
  bool is_virtual() const override { return true; }
  std::int64_t allreduce(const TensorPlacement& place, const ReductionGroup& grp,
                         std::vector<DevBlock>& blocks, std::vector<std::int64_t>& per_rank_sent,
                         cudaStream_t st) override;
  void redistribute(const RedistributionPlan& plan, const std::vector<DevBlock>& src,
                    std::vector<DevBlock>& dst, cudaStream_t st) override;
  void gather_to_root(const TensorPlacement&, std::vector<DevBlock>&, cudaStream_t) override {}

 private:
  std::int64_t procs_;
};

// One rank per process or host thread; every rank's exchanged blocks live in
// its executor's exchange heap, mapped by every peer (peer.hpp).
//   allreduce: each member sums the group's partials in ascending rank order
//     from 0.0 straight out of the peers' heaps (executor.cpp:91-98), then
//     writes the sum over its own partial once every member has read it;
//   redistribute: each destination pulls its boxes from the canonical
//     source's heap with strided box copies (redistribute.cpp:185-206) —
//     no pack, no unpack, one pass over the link;
//   gather: rank 0 reads the canonical blocks from the peers' heaps.
//
// Hybrid (the default for one process per GPU): a PeerTransport whose
// allreduces go to an NCCL communicator (ncclCommSplit groups, asynchronous
// on the communication stream) while the redistributions stay fused into the
// producing kernels over the mapped heaps.
class PeerTransport final : public Transport {
 public:
  PeerTransport(std::shared_ptr<PeerComm> comm, std::int64_t nranks,
                std::unique_ptr<Transport> allreduce_via = nullptr);
  bool owns(std::int64_t r) const override { return r == comm_->rank(); }
  bool is_virtual() const override { return false; }
  bool peer_mapped() const override { return true; }
  std::int64_t allreduce(const TensorPlacement& place, const ReductionGroup& grp,
                         std::vector<DevBlock>& blocks, std::vector<std::int64_t>& per_rank_sent,
                         cudaStream_t st) override;
  void redistribute(const RedistributionPlan& plan, const std::vector<DevBlock>& src,
                    std::vector<DevBlock>& dst, cudaStream_t st) override;
  void gather_to_root(const TensorPlacement& place, std::vector<DevBlock>& blocks,
                      cudaStream_t st) override;
  void gather_done(std::vector<DevBlock>& blocks, cudaStream_t st) override;
  PeerComm& comm() { return *comm_; }
  bool hybrid() const { return allreduce_via_ != nullptr; }

 private:
  std::shared_ptr<PeerComm> comm_;
  std::int64_t nranks_;
  std::unique_ptr<Transport> allreduce_via_;
};

#ifdef EB_HAVE_NCCL
class NcclTransport final : public Transport {
 public:
  // one process per GPU: communicator from a 128-byte ncclUniqueId
  NcclTransport(const void* unique_id, std::int64_t nranks, std::int64_t rank);
  // one host thread per GPU: a communicator of ncclCommInitAll (owned)
  NcclTransport(void* comm, std::int64_t nranks, std::int64_t rank);
  ~NcclTransport() override;
  bool owns(std::int64_t r) const override { return r == rank_; }
  bool is_virtual() const override { return false; }
  std::int64_t allreduce(const TensorPlacement& place, const ReductionGroup& grp,
                         std::vector<DevBlock>& blocks, std::vector<std::int64_t>& per_rank_sent,
                         cudaStream_t st) override;
  void redistribute(const RedistributionPlan& plan, const std::vector<DevBlock>& src,
                    std::vector<DevBlock>& dst, cudaStream_t st) override;
  void gather_to_root(const TensorPlacement& place, std::vector<DevBlock>& blocks,
                      cudaStream_t st) override;
  void gather_done(std::vector<DevBlock>& blocks, cudaStream_t st) override;

 private:
  // packing buffer for the messages of one redistribution, reused across
  // runs (grown on demand; stream-ordered)
  double* staging(std::int64_t elems, cudaStream_t st);

  std::int64_t rank_, nranks_;
  void* world_ = nullptr;
  std::map<std::string, void*> split_;
  double* staging_ = nullptr;
  std::int64_t staging_elems_ = 0;
  cudaEvent_t staging_done_ = nullptr;  // last use of staging_ (any stream)
  std::vector<double*> gathered_;  // rank 0: receive buffers of one gather
};
#endif

class ScheduleExecutor {
 public:
  ScheduleExecutor(Pipeline pipe, Transport* transport, cudaStream_t stream);
  ~ScheduleExecutor();

  // scatter (executor.cpp:48-65): every owned rank's input blocks to device.
  void stage_inputs(const std::vector<const double*>& global_inputs);
  // One process = one rank: the box (global base, shape) of operand k this
  // rank holds, and staging from a host buffer holding just that box — no
  // process needs the global tensor (e.g. C5's 69 GB X at P = 8).
  void local_block(int k, std::vector<std::int64_t>& base, std::vector<std::int64_t>& shape) const;
  void stage_block(int k, const double* host_block);
  // Virtual ranks without the global tensor: stage operand k from a host
  // buffer holding the global sub-box [base, base + shape) of it; every owned
  // rank's block lying inside the region is copied (returns how many).  E.g.
  // C5 at P = 8 on one GPU, one 8.6 GB i-slab at a time instead of 69 GB.
  int stage_region(int k, const std::vector<std::int64_t>& base,
                   const std::vector<std::int64_t>& shape, const double* host);
  // Use another executor's staged device blocks for operand k (same tensor,
  // same placement on every owned rank): e.g. one X for the three MTTKRP
  // modes of a CP-ALS sweep.
  void share_input(int k, const ScheduleExecutor& src, int k_src);
  // All terms: local contractions, reductions, redistributions (device only).
  void execute();
  // CP-sweep dimension tree: this executor (order-3 MTTKRP mode 0) and `mode1`
  // (mode 1 over the same X and mode-2 factor, both shared from this one)
  // in ONE pass over X — T = X x_k C is contracted once and folded into both
  // outputs (eb_mttkrp2); each output is then reduced over its own reference
  // reduction group.  Returns false (nothing run) when the pair does not
  // qualify; the caller then runs both executors separately.
  bool execute_pair(ScheduleExecutor& mode1);
  // Reductions on a side stream (opt-in): a term's allreduce then overlaps
  // whatever the caller queues next on the compute stream (e.g. the next
  // mode of a sweep); join() orders the compute stream after it.  Later terms
  // of the same schedule, gather() and the next execute() join implicitly.
  void set_async_reduce(bool on) { async_reduce_ = on; }
  void join();
  // CUDA graph of one run: execute() once eagerly (the run arena switches
  // to recycling, so every block of the run keeps its address), then
  // capture a second execute() on the executor's stream and instantiate it.
  // replay() launches that graph: the same kernels, copies and collectives
  // with one host call.  Virtual and NCCL transports (the peer transport
  // meets its peers on the host between kernels); re-staging inputs keeps
  // the graph valid (input blocks never move).
  void capture();
  void replay();
  bool captured() const { return graph_exec_ != nullptr; }
  // Canonical output blocks to host (virtual, or rank 0 over NCCL).
  void gather(double* host_out);
  void verify(const std::vector<const double*>& global_inputs, const double* host_out,
              double tol, SimulationReport& rep);

  const CommStats& comm() const { return comm_; }
  const Pipeline& pipeline() const { return pipe_; }
  std::vector<std::int64_t> output_shape() const;
  Transport* transport() const { return transport_; }
  int launches_fused() const { return launches_fused_; }
  int launches_ttm() const { return launches_ttm_; }
  int launches_generic() const { return launches_generic_; }
  // redistributions of the last run fused into their producer's epilogue
  int redistributions_fused() const { return redistributions_fused_; }
  cudaStream_t stream() const { return stream_; }

 private:
  std::int64_t local_lo(const TermPlan& t, char c, std::int64_t rank) const;
  std::int64_t local_len(const TermPlan& t, char c, std::int64_t rank) const;
  void copy_block_h2d(const double* global, const std::vector<std::int64_t>& gshape,
                      const DevBlock& b);
  const RedistRecord* find_redist(int to_term, const std::string& t) const;
  void* workspace(std::size_t bytes);
  // is_output: the term's output block — placed in the exchange heap when
  // the transport maps peers' blocks and the tensor leaves the rank
  DevBlock new_block(const TermPlan& term, const std::string& idx, std::int64_t rank, bool zero,
                     bool is_output = false);
  // Exchange heap (PeerTransport): one slot per term output that is reduced,
  // redistributed or gathered, sized for the largest rank's block so every
  // rank computes the same offsets; (re)allocated collectively.
  void prepare_heap();
  void map_peer_blocks(const TermPlan& term, std::vector<DevBlock>& blocks);
  // The fused TTM pair of a term (shape only: pointers unset), its natural
  // output index order and the pre / rest dim counts; false if not that shape.
  bool ttm2_shape(const TermPlan& term, std::int64_t rank, eb_ttm2_desc& d, std::string& natural,
                  int& n_pre, int& n_rest) const;
  // Fused redistribution ("push"): the record of term t's output when its
  // producing kernel can store straight into the next term's blocks (depth-1
  // term, uniform source and destination blocks, a TTM / TTM-pair producer),
  // else nullptr.  A function of the schedule only: every rank agrees.
  const RedistRecord* push_record(const TermPlan& t) const;
  void arm_push();  // destination blocks of every rank (push_dst_)
  // Term chaining: the next term when both are TTM pairs joined by a
  // whole-block self hand-over of the intermediate (eb_ttm2_chain), else
  // nullptr; run_chain launches both for one rank.
  const TermPlan* chain_next(const TermPlan& a) const;
  static bool fold_shape(const eb_ttm2_desc& da, const eb_ttm2_desc& db);
  void run_chain(const TermPlan& a, const TermPlan& b, std::int64_t rank,
                 const std::map<std::string, const DevBlock*>& at_hand, DevBlock& t1,
                 DevBlock& out);
  void scatter_desc(const TermPlan& term, std::int64_t rank, const std::string& natural,
                    int n_outer, int n_row, eb_scatter& sc) const;
  bool try_fused_mttkrp(const TermPlan& term, std::int64_t rank,
                        const std::map<std::string, const DevBlock*>& at_hand, DevBlock& out);
  // Two chained TTM steps of one term on the fused eb_ttm2 kernel.
  bool try_fused_ttm2(const TermPlan& term, std::int64_t rank,
                      const std::map<std::string, const DevBlock*>& at_hand, DevBlock& out);
  // zero-padded copies (run arena) for odd contiguous extents: X rows to
  // cols + 1 columns, a factor [rows][ld] to rows + 1 rows
  const double* padded_rows(const double* src, std::int64_t rows, std::int64_t cols);
  const double* padded_factor(const double* u, std::int64_t rows, std::int64_t ld);
  DevBlock run_step(const TermPlan& term, int sid, std::int64_t rank,
                    const std::map<std::string, const DevBlock*>& at_hand);
  std::int64_t reduce(const TensorPlacement& place, const ReductionGroup& grp,
                      std::vector<DevBlock>& blocks, bool last_term);

  Pipeline pipe_;
  Transport* transport_;
  cudaStream_t stream_;
  std::vector<std::int64_t> owned_;
  std::map<std::pair<int, std::string>, std::vector<DevBlock>> inputs_;
  std::map<std::pair<int, std::string>, std::vector<DevBlock>> store_;
  std::set<std::pair<int, std::string>> aliased_;
  bool staged_ = false;
  DeviceArena input_arena_, run_arena_;
  void* workspace_ = nullptr;
  std::size_t workspace_bytes_ = 0;
  CommStats comm_;
  int launches_fused_ = 0, launches_ttm_ = 0, launches_generic_ = 0;
  int redistributions_fused_ = 0;
  bool async_reduce_ = false, comm_pending_ = false;
  cudaEvent_t ev_compute_ = nullptr, ev_comm_ = nullptr;
  cudaGraphExec_t graph_exec_ = nullptr;
  long long graph_launches_ = 0;  // kernel launches inside the captured run
  // exchange heap (PeerTransport only)
  char* heap_ = nullptr;
  std::size_t heap_bytes_ = 0;
  std::vector<char*> heap_peers_;
  std::map<int, std::size_t> heap_slot_;  // term index -> byte offset
  std::map<int, std::size_t> heap_in_slot_;  // term index -> its pushed input block
  // fused redistribution state of the term being executed / done this run
  const RedistRecord* push_rec_ = nullptr;
  std::vector<DevBlock> push_dst_;
  std::set<std::pair<int, std::string>> pushed_;
  std::map<std::pair<int, std::int64_t>, DevBlock> chain_out_;  // (term, rank) -> output
};

}  // namespace gpu
}  // namespace einplan
