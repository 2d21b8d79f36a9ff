// einplan host C++ API, restated for the B200 build.
//
// Same public names and semantics as the reference headers
// (proj/include/einplan/{einsum,tensor,planner,soap,distribution,
// redistribute,schedule,executor}.hpp) so existing callers of the C++ API
// recompile unchanged; the implementation is this repo's own.  Planning is
// host work (it decides the processor grid bit for bit like the reference);
// execution (run) drives the sm_100a kernels in ../kernels through the inner
// C ABI (include/einplan_b200.h).
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace einplan {

// ---------------------------------------------------------------- errors --
// error.hpp:8-25
enum class errc { invalid_argument, parse, infeasible, grid, resource };

class Error : public std::runtime_error {
 public:
  Error(errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
  errc code() const { return code_; }

 private:
  errc code_;
};

[[noreturn]] inline void fail(errc code, const std::string& msg) { throw Error(code, msg); }

// ---------------------------------------------------------------- einsum --
// einsum.hpp:14-53
struct EinsumSpec {
  std::vector<std::string> inputs;
  std::string output;
  std::map<char, std::int64_t> extents;

  bool bound() const;
  std::vector<char> symbols() const;  // first-appearance order, inputs then output
  std::int64_t extent(char sym) const;
  std::vector<std::int64_t> shape_of(const std::string& indices) const;
  std::string text() const;
};

EinsumSpec parse(const std::string& text);
EinsumSpec bind_extents(const EinsumSpec& spec,
                        const std::vector<std::vector<std::int64_t>>& shapes);
EinsumSpec bind_extents(const EinsumSpec& spec, const std::map<char, std::int64_t>& extents);
std::int64_t flop_count_naive(const EinsumSpec& spec);
EinsumSpec make_matricization(int order, int mode);
EinsumSpec make_ttm(int order, int mode);
EinsumSpec make_krp();
EinsumSpec make_ttmc(int order, int mode);
EinsumSpec make_mttkrp(int order, int mode);

// ---------------------------------------------------------------- tensor --
// tensor.hpp:11-37 (host tensors: inputs, gathered outputs)
struct DenseTensor {
  std::vector<std::int64_t> shape;
  std::vector<double> data;

  DenseTensor() = default;
  explicit DenseTensor(std::vector<std::int64_t> s);
  std::int64_t size() const;
  std::vector<std::int64_t> strides() const;
  std::int64_t offset_of(const std::vector<std::int64_t>& idx) const;
  double& at(const std::vector<std::int64_t>& idx);
  double at(const std::vector<std::int64_t>& idx) const;
};

std::int64_t shape_product(const std::vector<std::int64_t>& shape);
DenseTensor random_tensor(const std::vector<std::int64_t>& shape, std::uint64_t seed);
double max_rel_error(const DenseTensor& got, const DenseTensor& want);
void write_tensor(const std::string& path, const DenseTensor& t);
DenseTensor read_tensor(const std::string& path);

// --------------------------------------------------------------- planner --
// planner.hpp:13-59
enum class OpClass { KRP, TTM, TDOT, GEMM, OUTER, ELEMENTWISE };
const char* to_string(OpClass c);

struct ContractionStep {
  int lhs = -1;
  int rhs = -1;
  std::string lhs_indices;
  std::string rhs_indices;
  std::string result_indices;
  std::int64_t flops = 0;
  OpClass op_class = OpClass::TDOT;
};

struct ContractionTree {
  int n_inputs = 0;
  std::vector<ContractionStep> steps;
  std::int64_t total_flops = 0;

  int result_id(int step) const { return n_inputs + step; }
  std::string tensor_name(int id) const;
  const std::string& indices_of(int id, const EinsumSpec& spec) const;
};

std::int64_t step_flops(const std::string& lhs_indices, const std::string& rhs_indices,
                        const std::string& result_indices,
                        const std::map<char, std::int64_t>& extents);
OpClass classify(const std::string& lhs_indices, const std::string& rhs_indices,
                 const std::string& result_indices);
ContractionTree optimal_path(const EinsumSpec& spec);

// ------------------------------------------------------------------ soap --
// soap.hpp:11-84
struct SdgVertex {
  enum class Role { input, intermediate, output };
  std::string name;
  Role role = Role::input;
  std::string indices;
  int step = -1;
};

struct Sdg {
  std::vector<SdgVertex> vertices;
  std::vector<std::pair<int, int>> edges;
  std::vector<int> non_input_ids() const;
  std::vector<int> consumers_of(int id) const;
};

Sdg build_sdg(const ContractionTree& tree, const EinsumSpec& spec);
std::vector<std::vector<std::vector<int>>> enumerate_partitions(const Sdg& sdg);

struct AccessArray {
  std::string tensor;
  std::string indices;
};

struct FusedStatement {
  std::vector<char> iteration;
  std::map<char, std::int64_t> extents;
  std::vector<AccessArray> arrays;
  std::string output;
  std::vector<int> step_ids;
  double volume = 0.0;
};

FusedStatement fuse(const std::vector<int>& block, const Sdg& sdg, const ContractionTree& tree,
                    const EinsumSpec& spec);
std::map<char, double> max_tiles(const FusedStatement& stmt, double budget);

struct IoBound {
  double rho = 0.0;
  double x0 = 0.0;
  double q_bound = 0.0;
  std::map<char, double> tiles;
  bool fits_fast_memory = false;
};

IoBound intensity(const FusedStatement& stmt, double fast_mem);

struct PartitionResult {
  std::vector<std::vector<int>> blocks;
  std::vector<FusedStatement> statements;
  std::vector<IoBound> bounds;
  double total_q = 0.0;
  int partitions_considered = 0;
};

PartitionResult best_partition(const Sdg& sdg, const ContractionTree& tree,
                               const EinsumSpec& spec, double fast_mem);

// ---------------------------------------------------------- distribution --
// distribution.hpp:15-96
struct ProcessGrid {
  std::vector<char> order;
  std::vector<std::int64_t> dims;

  std::int64_t total() const;
  std::int64_t rank_of(const std::vector<std::int64_t>& coords) const;
  std::vector<std::int64_t> coords_of(std::int64_t rank) const;
  int axis_of(char sym) const;
  std::int64_t dim_of(char sym) const;
};

struct BlockDistribution {
  ProcessGrid grid;
  std::vector<std::int64_t> extents;
  std::vector<std::int64_t> blocks;

  std::vector<std::int64_t> base_of(const std::vector<std::int64_t>& coords) const;
  std::vector<std::int64_t> shape_of(const std::vector<std::int64_t>& coords) const;
};

BlockDistribution make_block_distribution(const ProcessGrid& grid,
                                          const std::vector<std::int64_t>& extents);
BlockDistribution block_distribution_from_blocks(const std::vector<char>& order,
                                                 const std::vector<std::int64_t>& extents,
                                                 const std::vector<std::int64_t>& blocks);

struct OwnerInfo {
  std::vector<std::int64_t> coords, offsets, bases;
};
OwnerInfo owner_of(const std::vector<std::int64_t>& index, const BlockDistribution& dist);

struct TensorPlacement {
  std::string tensor;
  std::string indices;
  ProcessGrid term_grid;
  std::vector<int> axes;
  BlockDistribution dist;

  std::int64_t replication() const;
  std::vector<std::int64_t> block_coords_of(std::int64_t rank) const;
  std::vector<std::int64_t> replica_ranks(const std::vector<std::int64_t>& block) const;
  std::int64_t canonical_rank(const std::vector<std::int64_t>& block) const;
  bool is_canonical(std::int64_t rank) const;
};

TensorPlacement placement(const std::string& tensor, const std::string& indices,
                          const ProcessGrid& term_grid,
                          const std::map<char, std::int64_t>& extents);
TensorPlacement placement_with_dist(const std::string& tensor, const std::string& indices,
                                    const ProcessGrid& term_grid, const BlockDistribution& dist);

struct ReductionGroup {
  std::vector<char> dims;
  std::int64_t depth = 1;
};

ReductionGroup reduction_group(const std::string& output_indices, const ProcessGrid& grid);
ProcessGrid choose_grid(const FusedStatement& stmt, const std::map<char, double>& tiles,
                        std::int64_t procs);

// ---------------------------------------------------------- redistribute --
// redistribute.hpp:13-76
struct DimSegment {
  std::int64_t p_x = 0;
  std::int64_t oy_lo = 0, oy_hi = 0;
  std::int64_t ox_lo = 0, ox_hi = 0;
};

struct DimPartition {
  std::int64_t xi = 0;
  std::int64_t lambda = 0;
  std::vector<DimSegment> segments;
};

DimPartition dim_partition(std::int64_t block_y, std::int64_t p_y, std::int64_t block_x,
                           std::int64_t extent);
std::pair<std::int64_t, std::int64_t> matching_ranks(std::int64_t p_x, std::int64_t block_x,
                                                     std::int64_t block_y);

struct Message {
  std::int64_t src_rank = 0;
  std::int64_t dst_rank = 0;
  std::vector<std::int64_t> src_block, dst_block;
  std::vector<std::int64_t> oy_lo, oy_hi, ox_lo, ox_hi;
  std::int64_t elements = 0;
  bool self = false;
};

struct RedistributionPlan {
  std::string tensor;
  TensorPlacement source;
  TensorPlacement destination;
  std::vector<Message> messages;
  std::int64_t transmitted_volume = 0;
  std::int64_t logical_volume = 0;
  std::int64_t self_messages = 0;
};

RedistributionPlan plan_redistribution(const std::string& tensor, const TensorPlacement& source,
                                       const TensorPlacement& destination);

// -------------------------------------------------------------- schedule --
// schedule.hpp:12-57
struct TermPlan {
  int index = 0;
  FusedStatement statement;
  IoBound bound;
  ProcessGrid grid;
  std::map<char, std::int64_t> blocks;
  std::vector<TensorPlacement> placements;
  std::vector<int> step_ids;
  ReductionGroup reduction;

  const TensorPlacement& placement_of(const std::string& tensor) const;
};

struct RedistRecord {
  std::string tensor;
  int from_term = 0;
  int to_term = 0;
  RedistributionPlan plan;
};

struct Schedule {
  std::int64_t procs = 1;
  std::vector<TermPlan> terms;
  std::vector<RedistRecord> redistributions;
};

Schedule build_schedule(const ContractionTree& tree, const PartitionResult& partition,
                        const EinsumSpec& spec, std::int64_t procs);

struct Pipeline {
  EinsumSpec spec;
  ContractionTree tree;
  Sdg sdg;
  PartitionResult partition;
  Schedule schedule;
};

Pipeline make_pipeline(const EinsumSpec& spec, std::int64_t procs, double fast_mem);

// -------------------------------------------------------------- executor --
// executor.hpp:13-73; run() executes on the GPU (see executor.cpp).
struct CommEvent {
  std::string kind;
  int term = 0;
  std::string tensor;
  std::int64_t elements = 0;
};

struct CommStats {
  std::vector<CommEvent> events;
  std::int64_t allreduce_volume = 0;
  std::int64_t redistribute_volume = 0;
  std::vector<std::int64_t> per_rank_sent;

  std::int64_t total() const { return allreduce_volume + redistribute_volume; }
  std::int64_t max_rank_sent() const;
};

struct SimulationReport {
  DenseTensor output;
  CommStats comm;
  bool verified = false;
  double max_error = 0.0;
  double tolerance = 0.0;
  bool pass = true;
  std::uint64_t seed = 0;
  // B200 build: how the ranks ran ("virtual": every rank on one device;
  // "devices": one host thread per GPU), on which devices, over which
  // transport ("virtual", "peer", "nccl").  Reported as "execution".
  std::string exec_mode;
  std::vector<int> devices;
  std::string transport;
};

struct RunOptions {
  bool verify = true;
  double tolerance = 1e-10;
  std::uint64_t seed = 0;
  bool corrupt_output = false;
};

SimulationReport run(const Schedule& schedule, const EinsumSpec& spec,
                     const ContractionTree& tree, const std::vector<DenseTensor>& inputs,
                     const RunOptions& opts);

}  // namespace einplan
