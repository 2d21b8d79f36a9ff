// C ABI of the B200 build.
//
// Outer ABI (include/einplan/einplan.h): the reference's session/report
// interface (proj/src/capi.cpp:13-256) with execution on the GPU.
// Inner ABI (include/einplan_b200.h): eb_exec_* — a rank-local executor
// handle used by the Python host mirror and bench.py, one process per GPU
// over NCCL or all ranks virtual on one device.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <sstream>

#include "einplan/einplan.h"
#include "einplan_b200.h"
#include "executor.hpp"
#include "report_json.hpp"
#include "status.hpp"

#ifdef EB_HAVE_NCCL
#include <nccl.h>
#endif

using namespace einplan;

struct einplan_session {
  EinsumSpec spec;
};

namespace {

thread_local std::string g_outer_error;

char* heap_copy(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (p) std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

einplan_status code_of(errc c) {
  switch (c) {
    case errc::parse: return EINPLAN_E_PARSE;
    case errc::infeasible: return EINPLAN_E_INFEASIBLE;
    case errc::grid: return EINPLAN_E_GRID;
    case errc::resource: return EINPLAN_E_RESOURCE;
    case errc::invalid_argument: return EINPLAN_E_INVALID;
  }
  return EINPLAN_E_INTERNAL;
}

// Exceptions never cross the C boundary (capi.cpp:27-49 convention).
template <typename Fn>
einplan_status shielded(Fn&& fn) {
  try {
    return fn();
  } catch (const Error& e) {
    g_outer_error = e.what();
    return code_of(e.code());
  } catch (const std::exception& e) {
    g_outer_error = e.what();
    return EINPLAN_E_INTERNAL;
  }
}

std::map<char, std::int64_t> dims_list(const char* dims) {
  std::map<char, std::int64_t> out;
  if (!dims) return out;
  std::stringstream in(dims);
  std::string item;
  while (std::getline(in, item, ',')) {
    if (item.empty()) continue;
    if (item.size() < 3 || item[1] != '=')
      fail(errc::parse, "dims: expected symbol=extent, got \"" + item + "\"");
    char* end = nullptr;
    const long long v = std::strtoll(item.c_str() + 2, &end, 10);
    if (!end || *end != '\0' || v < 1) fail(errc::parse, "dims: bad extent in \"" + item + "\"");
    out[item[0]] = v;
  }
  return out;
}

std::vector<std::string> csv_paths(const char* csv) {
  std::vector<std::string> out;
  if (!csv) return out;
  std::stringstream in(csv);
  std::string item;
  while (std::getline(in, item, ','))
    if (!item.empty()) out.push_back(item);
  return out;
}

std::int64_t env_cap(std::int64_t dflt) {
  if (const char* env = std::getenv("EINPLAN_MAX_POINTS")) {
    char* end = nullptr;
    const long long v = std::strtoll(env, &end, 10);
    if (end && *end == '\0' && v > 0) return v;
  }
  return dflt;
}

EinsumSpec make_spec(const char* einsum, const char* dims) {
  const auto given = dims_list(dims);
  EinsumSpec spec = bind_extents(parse(einsum), given);
  for (const auto& kv : given)
    if (!spec.extents.count(kv.first))
      fail(errc::parse, std::string("dims: symbol '") + kv.first + "' does not appear in the einsum");
  return spec;
}

SimulationReport run_on_gpu(const Pipeline& pipe, const std::vector<DenseTensor>& inputs,
                            const RunOptions& opts) {
  return run(pipe.schedule, pipe.spec, pipe.tree, inputs, opts);
}

}  // namespace

extern "C" {

const char* einplan_version(void) { return "1.0.0-b200"; }

const char* einplan_status_name(einplan_status s) {
  switch (s) {
    case EINPLAN_OK: return "ok";
    case EINPLAN_E_VERIFY: return "verification failed";
    case EINPLAN_E_PARSE: return "parse error";
    case EINPLAN_E_INFEASIBLE: return "infeasible fast memory";
    case EINPLAN_E_GRID: return "invalid process grid";
    case EINPLAN_E_RESOURCE: return "resource cap exceeded";
    case EINPLAN_E_INVALID: return "invalid argument";
    case EINPLAN_E_INTERNAL: return "internal error";
  }
  return "unknown";
}

const char* einplan_last_error(void) { return g_outer_error.c_str(); }

void einplan_free(char* str) { std::free(str); }

einplan_status einplan_session_create(const char* einsum, const char* dims,
                                      einplan_session** out) {
  if (!einsum || !out) {
    g_outer_error = "einplan_session_create: null argument";
    return EINPLAN_E_INVALID;
  }
  *out = nullptr;
  return shielded([&] {
    *out = new einplan_session{make_spec(einsum, dims)};
    return EINPLAN_OK;
  });
}

void einplan_session_destroy(einplan_session* s) { delete s; }

einplan_status einplan_bound_json(einplan_session* s, double fast_mem, char** json_out) {
  if (!s || !json_out) {
    g_outer_error = "einplan_bound_json: null argument";
    return EINPLAN_E_INVALID;
  }
  return shielded([&] {
    Pipeline p;
    p.spec = s->spec;
    p.tree = optimal_path(p.spec);
    p.sdg = build_sdg(p.tree, p.spec);
    p.partition = best_partition(p.sdg, p.tree, p.spec, fast_mem);
    *json_out = heap_copy(bound_report(p, fast_mem).dump(2));
    return EINPLAN_OK;
  });
}

einplan_status einplan_plan_json(einplan_session* s, int64_t procs, double fast_mem,
                                 int include_messages, char** json_out) {
  if (!s || !json_out) {
    g_outer_error = "einplan_plan_json: null argument";
    return EINPLAN_E_INVALID;
  }
  return shielded([&] {
    const Pipeline p = make_pipeline(s->spec, procs, fast_mem);
    *json_out = heap_copy(plan_report(p, fast_mem, include_messages != 0).dump(2));
    return EINPLAN_OK;
  });
}

einplan_status einplan_run_json(einplan_session* s, int64_t procs, double fast_mem,
                                uint64_t seed, int verify, const char* input_paths,
                                const char* dump_output, char** json_out) {
  if (!s || !json_out) {
    g_outer_error = "einplan_run_json: null argument";
    return EINPLAN_E_INVALID;
  }
  return shielded([&] {
    const EinsumSpec& spec = s->spec;
    std::int64_t points = 1;
    for (char c : spec.symbols()) points *= spec.extent(c);
    const std::int64_t cap = env_cap(100'000'000);
    if (points > cap)
      fail(errc::resource, "run: iteration space of " + std::to_string(points) +
                               " points exceeds the cap (" + std::to_string(cap) +
                               "; override with EINPLAN_MAX_POINTS)");
    const Pipeline pipe = make_pipeline(spec, procs, fast_mem);
    std::vector<DenseTensor> inputs;
    const auto paths = csv_paths(input_paths);
    if (!paths.empty()) {
      if (paths.size() != spec.inputs.size())
        fail(errc::invalid_argument, "run: expected " + std::to_string(spec.inputs.size()) +
                                         " input tensors, got " + std::to_string(paths.size()));
      for (std::size_t i = 0; i < paths.size(); ++i) {
        DenseTensor t = read_tensor(paths[i]);
        if (t.shape != spec.shape_of(spec.inputs[i]))
          fail(errc::invalid_argument,
               "run: tensor \"" + paths[i] + "\" does not match \"" + spec.inputs[i] + "\"");
        inputs.push_back(std::move(t));
      }
    } else {
      for (std::size_t i = 0; i < spec.inputs.size(); ++i)
        inputs.push_back(random_tensor(spec.shape_of(spec.inputs[i]), seed + i));
    }
    RunOptions ro;
    ro.verify = verify != 0;
    ro.seed = seed;
    ro.corrupt_output = std::getenv("EINPLAN_TEST_CORRUPT") != nullptr;
    const SimulationReport sim = run_on_gpu(pipe, inputs, ro);
    if (dump_output) write_tensor(dump_output, sim.output);
    *json_out = heap_copy(run_report(pipe, fast_mem, sim).dump(2));
    if (sim.verified && !sim.pass) {
      g_outer_error = "verification failed: max relative error " + std::to_string(sim.max_error);
      return EINPLAN_E_VERIFY;
    }
    return EINPLAN_OK;
  });
}

einplan_status einplan_bench_json(double scale, int64_t procs, double fast_mem, uint64_t seed,
                                  char** json_out) {
  if (!json_out) {
    g_outer_error = "einplan_bench_json: null argument";
    return EINPLAN_E_INVALID;
  }
  return shielded([&] {
    if (scale <= 0.0) fail(errc::invalid_argument, "bench: scale must be positive");
    // The Table-III suite (bench.cpp:20-47), extents scaled with a floor of 2.
    struct Fixture {
      const char* name;
      const char* einsum;
      std::vector<std::pair<char, std::int64_t>> ext;
    };
    const std::vector<std::pair<char, std::int64_t>> mt3 = {
        {'i', 1024}, {'j', 1024}, {'k', 1024}, {'a', 24}};
    const std::vector<std::pair<char, std::int64_t>> mt5 = {
        {'i', 1024}, {'j', 1024}, {'k', 1024}, {'l', 1024}, {'m', 1024}, {'a', 24}};
    const std::vector<Fixture> suite = {
        {"1MM", "ij,jk->ik", {{'i', 4096}, {'j', 4096}, {'k', 4096}}},
        {"2MM", "ij,jk,kl->il", {{'i', 4096}, {'j', 4096}, {'k', 4096}, {'l', 4096}}},
        {"3MM", "ij,jk,kl,lm->im", {{'i', 4096}, {'j', 4096}, {'k', 4096}, {'l', 4096}, {'m', 4096}}},
        {"MTTKRP-O3-M0", "ijk,ja,ka->ia", mt3},
        {"MTTKRP-O3-M1", "ijk,ia,ka->ja", mt3},
        {"MTTKRP-O3-M2", "ijk,ia,ja->ka", mt3},
        {"MTTKRP-O5-M0", "ijklm,ja,ka,la,ma->ia", mt5},
        {"MTTKRP-O5-M2", "ijklm,ia,ja,la,ma->ka", mt5},
        {"MTTKRP-O5-M4", "ijklm,ia,ja,ka,la->ma", mt5},
        {"TTMc-O5-M0", "ijklm,jb,kc,ld,me->ibcde",
         {{'i', 60}, {'j', 60}, {'k', 60}, {'l', 60}, {'m', 60},
          {'b', 24}, {'c', 24}, {'d', 24}, {'e', 24}}},
    };
    const std::int64_t cap = env_cap(4'000'000'000LL);
    bool all_pass = true;
    ojson kernels = ojson::array();
    for (const Fixture& fx : suite) {
      std::map<char, std::int64_t> ext;
      for (const auto& kv : fx.ext)
        ext[kv.first] = std::max<std::int64_t>(2, std::llround(static_cast<double>(kv.second) * scale));
      ojson k;
      k["name"] = fx.name;
      k["einsum"] = fx.einsum;
      ojson ej = ojson::object();
      for (const auto& kv : ext) ej[std::string(1, kv.first)] = kv.second;
      k["extents"] = std::move(ej);
      try {
        const EinsumSpec spec = bind_extents(parse(fx.einsum), ext);
        std::int64_t points = 1;
        for (char c : spec.symbols()) points *= spec.extent(c);
        if (points > cap)
          fail(errc::resource, std::string(fx.name) + ": iteration space exceeds the configured cap");
        const Pipeline pipe = make_pipeline(spec, procs, fast_mem);
        std::vector<DenseTensor> inputs;
        for (std::size_t i = 0; i < spec.inputs.size(); ++i)
          inputs.push_back(random_tensor(spec.shape_of(spec.inputs[i]), seed + i));
        RunOptions ro;
        ro.verify = true;
        ro.tolerance = 1e-10;
        ro.seed = seed;
        const SimulationReport sim = run_on_gpu(pipe, inputs, ro);
        k["pass"] = sim.pass;
        k["max_rel_error"] = sim.max_error;
        k["volume_total"] = sim.comm.total();
        k["allreduce_volume"] = sim.comm.allreduce_volume;
        k["redistribute_volume"] = sim.comm.redistribute_volume;
        k["q_bound_total"] = pipe.partition.total_q;
        if (pipe.partition.total_q > 0.0)
          k["volume_to_bound_ratio"] =
              static_cast<double>(sim.comm.total()) / pipe.partition.total_q;
        else
          k["volume_to_bound_ratio"] = nullptr;
        all_pass = all_pass && sim.pass;
      } catch (const std::exception& e) {
        k["pass"] = false;
        k["error"] = e.what();
        all_pass = false;
      }
      kernels.push_back(std::move(k));
    }
    ojson j;
    j["format"] = "einplan/v1";
    j["command"] = "bench";
    j["suite"] = "table3";
    j["scale"] = scale;
    j["procs"] = procs;
    j["fast_mem"] = fast_mem;
    j["seed"] = seed;
    j["kernels"] = std::move(kernels);
    j["all_pass"] = all_pass;
    *json_out = heap_copy(j.dump(2));
    if (!all_pass) {
      g_outer_error = "bench: at least one kernel failed";
      return EINPLAN_E_VERIFY;
    }
    return EINPLAN_OK;
  });
}

}  // extern "C"

// ===================================================== inner eb_exec ABI --

struct eb_exec {
  std::shared_ptr<gpu::Transport> transport;  // shared by executors of one process group
  int64_t procs = 1;
  std::unique_ptr<gpu::ScheduleExecutor> exec;
  cudaStream_t stream = nullptr;
  double fast_mem = 1024.0;
};

namespace {

int exec_guard(const std::function<void()>& fn) {
  try {
    fn();
    return EB_OK;
  } catch (const Error& e) {
    eb::set_error(e.what());
    return EB_E_INVALID;
  } catch (const eb::InvalidError& e) {
    eb::set_error(e.what());
    return EB_E_INVALID;
  } catch (const std::exception& e) {
    eb::set_error(e.what());
    return EB_E_DEVICE;
  }
}

}  // namespace

extern "C" {

const char* eb_build_info(void) {
  return "einplan_b200: sm_100a (-gencode arch=compute_100a,code=sm_100a), FP64 DMMA + TMA "
         "kernels"
#ifdef EB_HAVE_NCCL
         ", NCCL transport"
#endif
      ;
}

void eb_free(void* p) { std::free(p); }

int eb_mem_in_use(int64_t* bytes) {
  return exec_guard([&] {
    if (!bytes) throw eb::InvalidError("eb_mem_in_use: null argument");
    int dev = 0;
    cudaMemPool_t pool = nullptr;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess)
      throw eb::DeviceError("eb_mem_in_use: no device");
    std::uint64_t used = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) != cudaSuccess)
      throw eb::DeviceError("eb_mem_in_use: pool query failed");
    *bytes = static_cast<int64_t>(used);
  });
}

int eb_plan_json(const char* einsum, const char* dims, int64_t procs, double fast_mem,
                 int include_messages, char** json_out) {
  return exec_guard([&] {
    const Pipeline p = make_pipeline(make_spec(einsum, dims), procs, fast_mem);
    *json_out = heap_copy(plan_report(p, fast_mem, include_messages != 0).dump(2));
  });
}

int eb_nccl_unique_id(void* out128) {
  return exec_guard([&] {
#ifdef EB_HAVE_NCCL
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) throw eb::DeviceError("ncclGetUniqueId failed");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
#else
    (void)out128;
    throw eb::DeviceError("built without NCCL");
#endif
  });
}

int eb_exec_create(const char* einsum, const char* dims, int64_t procs, double fast_mem,
                   int64_t rank, const void* nccl_id, void* stream, eb_exec** out) {
  return exec_guard([&] {
    if (!out) throw eb::InvalidError("eb_exec_create: null out");
    *out = nullptr;
    auto h = std::make_unique<eb_exec>();
    h->fast_mem = fast_mem;
    h->stream = static_cast<cudaStream_t>(stream);
    Pipeline pipe = make_pipeline(make_spec(einsum, dims), procs, fast_mem);
    if (rank < 0) {
      h->transport = std::make_shared<gpu::VirtualTransport>(procs);
    } else {
#ifdef EB_HAVE_NCCL
      if (!nccl_id) throw eb::InvalidError("eb_exec_create: rank >= 0 needs an NCCL unique id");
      h->transport = std::make_shared<gpu::NcclTransport>(nccl_id, procs, rank);
#else
      throw eb::DeviceError("built without NCCL");
#endif
    }
    h->procs = procs;
    h->exec = std::make_unique<gpu::ScheduleExecutor>(std::move(pipe), h->transport.get(),
                                                      h->stream);
    *out = h.release();
  });
}

int eb_exec_create_peer(const char* einsum, const char* dims, int64_t procs, double fast_mem,
                        int64_t rank, const char* group, void* stream, eb_exec** out) {
  return exec_guard([&] {
    if (!out || !group) throw eb::InvalidError("eb_exec_create_peer: null argument");
    *out = nullptr;
    if (rank < 0 || rank >= procs) throw eb::InvalidError("eb_exec_create_peer: rank outside 0..procs-1");
    auto h = std::make_unique<eb_exec>();
    h->fast_mem = fast_mem;
    h->stream = static_cast<cudaStream_t>(stream);
    Pipeline pipe = make_pipeline(make_spec(einsum, dims), procs, fast_mem);
    auto shared = gpu::PeerShared::attach_shm(group, static_cast<int>(procs));
    h->transport = std::make_shared<gpu::PeerTransport>(
        std::make_shared<gpu::PeerComm>(shared, static_cast<int>(rank)), procs);
    h->procs = procs;
    h->exec = std::make_unique<gpu::ScheduleExecutor>(std::move(pipe), h->transport.get(),
                                                      h->stream);
    *out = h.release();
  });
}

int eb_exec_create_hybrid(const char* einsum, const char* dims, int64_t procs, double fast_mem,
                          int64_t rank, const char* group, const void* nccl_id, void* stream,
                          eb_exec** out) {
  return exec_guard([&] {
    if (!out || !group || !nccl_id) throw eb::InvalidError("eb_exec_create_hybrid: null argument");
    *out = nullptr;
    if (rank < 0 || rank >= procs)
      throw eb::InvalidError("eb_exec_create_hybrid: rank outside 0..procs-1");
#ifdef EB_HAVE_NCCL
    auto h = std::make_unique<eb_exec>();
    h->fast_mem = fast_mem;
    h->stream = static_cast<cudaStream_t>(stream);
    Pipeline pipe = make_pipeline(make_spec(einsum, dims), procs, fast_mem);
    auto shared = gpu::PeerShared::attach_shm(group, static_cast<int>(procs));
    auto comm = std::make_shared<gpu::PeerComm>(shared, static_cast<int>(rank));
    h->transport = std::make_shared<gpu::PeerTransport>(
        comm, procs, std::make_unique<gpu::NcclTransport>(nccl_id, procs, rank));
    h->procs = procs;
    h->exec = std::make_unique<gpu::ScheduleExecutor>(std::move(pipe), h->transport.get(),
                                                      h->stream);
    *out = h.release();
#else
    (void)einsum; (void)dims; (void)fast_mem; (void)stream;
    throw eb::DeviceError("built without NCCL");
#endif
  });
}

int eb_exec_create_like(const char* einsum, const char* dims, double fast_mem, eb_exec* peer,
                        void* stream, eb_exec** out) {
  return exec_guard([&] {
    if (!out || !peer) throw eb::InvalidError("eb_exec_create_like: null argument");
    *out = nullptr;
    auto h = std::make_unique<eb_exec>();
    h->fast_mem = fast_mem;
    h->stream = stream ? static_cast<cudaStream_t>(stream) : peer->stream;
    h->procs = peer->procs;
    h->transport = peer->transport;  // same ranks, same NCCL communicator (and split cache)
    Pipeline pipe = make_pipeline(make_spec(einsum, dims), h->procs, fast_mem);
    h->exec = std::make_unique<gpu::ScheduleExecutor>(std::move(pipe), h->transport.get(),
                                                      h->stream);
    *out = h.release();
  });
}

void eb_exec_destroy(eb_exec* h) { delete h; }

int eb_exec_stage(eb_exec* h, const double* const* host_inputs) {
  return exec_guard([&] {
    const auto n = h->exec->pipeline().spec.inputs.size();
    std::vector<const double*> g(host_inputs, host_inputs + n);
    h->exec->stage_inputs(g);
  });
}

int eb_exec_block(eb_exec* h, int k, int64_t* base, int64_t* shape, int* nd) {
  return exec_guard([&] {
    if (!h || !base || !shape || !nd) throw eb::InvalidError("eb_exec_block: null argument");
    std::vector<std::int64_t> b, s;
    h->exec->local_block(k, b, s);
    *nd = static_cast<int>(b.size());
    std::copy(b.begin(), b.end(), base);
    std::copy(s.begin(), s.end(), shape);
  });
}

int eb_exec_stage_block(eb_exec* h, int k, const double* host_block) {
  return exec_guard([&] {
    if (!h || !host_block) throw eb::InvalidError("eb_exec_stage_block: null argument");
    h->exec->stage_block(k, host_block);
  });
}

int eb_exec_stage_region(eb_exec* h, int k, const int64_t* base, const int64_t* shape, int nd,
                         const double* host_region, int* staged) {
  return exec_guard([&] {
    if (!h || !base || !shape || !host_region || nd < 0 || nd > 16)
      throw eb::InvalidError("eb_exec_stage_region: bad argument");
    const int n = h->exec->stage_region(k, std::vector<std::int64_t>(base, base + nd),
                                        std::vector<std::int64_t>(shape, shape + nd), host_region);
    if (staged) *staged = n;
  });
}

int eb_exec_share_input(eb_exec* dst, int k_dst, eb_exec* src, int k_src) {
  return exec_guard([&] {
    if (!dst || !src) throw eb::InvalidError("eb_exec_share_input: null handle");
    dst->exec->share_input(k_dst, *src->exec, k_src);
  });
}

int eb_exec_run(eb_exec* h) {
  return exec_guard([&] { h->exec->execute(); });
}

int eb_exec_set_async_reduce(eb_exec* h, int on) {
  return exec_guard([&] {
    if (!h) throw eb::InvalidError("eb_exec_set_async_reduce: null handle");
    h->exec->set_async_reduce(on != 0);
  });
}

int eb_exec_join(eb_exec* h) {
  return exec_guard([&] {
    if (!h) throw eb::InvalidError("eb_exec_join: null handle");
    h->exec->join();
  });
}

int eb_exec_capture(eb_exec* h) {
  return exec_guard([&] {
    if (!h) throw eb::InvalidError("eb_exec_capture: null handle");
    h->exec->capture();
  });
}

int eb_exec_replay(eb_exec* h) {
  return exec_guard([&] {
    if (!h) throw eb::InvalidError("eb_exec_replay: null handle");
    h->exec->replay();
  });
}

int eb_exec_run_pair(eb_exec* mode0, eb_exec* mode1, int* fused) {
  return exec_guard([&] {
    if (!mode0 || !mode1) throw eb::InvalidError("eb_exec_run_pair: null handle");
    const bool ok = mode0->exec->execute_pair(*mode1->exec);
    if (!ok) {
      mode0->exec->execute();
      mode1->exec->execute();
    }
    if (fused) *fused = ok ? 1 : 0;
  });
}

int eb_exec_gather(eb_exec* h, double* host_out) {
  return exec_guard([&] { h->exec->gather(host_out); });
}

int64_t eb_exec_output_elems(eb_exec* h) {
  return shape_product(h->exec->output_shape());
}

int eb_exec_stats(eb_exec* h, int64_t* out8) {
  return exec_guard([&] {
    const CommStats& c = h->exec->comm();
    out8[0] = c.allreduce_volume;
    out8[1] = c.redistribute_volume;
    out8[2] = c.max_rank_sent();
    out8[3] = h->exec->launches_fused();
    out8[4] = h->exec->launches_ttm();
    out8[5] = h->exec->launches_generic();
    out8[6] = h->exec->pipeline().tree.total_flops;
    out8[7] = static_cast<int64_t>(h->exec->pipeline().schedule.terms.size());
  });
}

int eb_exec_fused_redistributions(eb_exec* h) {
  return h ? h->exec->redistributions_fused() : -1;
}

int eb_exec_report_json(eb_exec* h, const double* host_out, char** json_out) {
  return exec_guard([&] {
    SimulationReport sim;
    sim.output = DenseTensor(h->exec->output_shape());
    if (host_out)
      std::memcpy(sim.output.data.data(), host_out, sim.output.data.size() * sizeof(double));
    sim.comm = h->exec->comm();
    *json_out = heap_copy(run_report(h->exec->pipeline(), h->fast_mem, sim).dump(2));
  });
}

struct eb_rng {
  std::mt19937_64 gen;
};

int eb_rng_create(uint64_t seed, int64_t skip, eb_rng** out) {
  return eb::guard([&] {
    if (!out || skip < 0) throw eb::InvalidError("eb_rng_create: bad argument");
    auto g = std::make_unique<eb_rng>();
    g->gen.seed(seed);
    if (skip > 0) g->gen.discard(static_cast<unsigned long long>(skip));
    *out = g.release();
  });
}

void eb_rng_fill(eb_rng* g, double* out, int64_t n) {
  for (int64_t k = 0; k < n; ++k)
    out[k] = 2.0 * (static_cast<double>(g->gen() >> 11) * 0x1.0p-53) - 1.0;
}

void eb_rng_destroy(eb_rng* g) { delete g; }

void eb_random_fill_host(double* out, int64_t n, uint64_t seed, int64_t skip) {
  std::mt19937_64 gen(seed);
  if (skip > 0) gen.discard(static_cast<unsigned long long>(skip));
  for (int64_t k = 0; k < n; ++k)
    out[k] = 2.0 * (static_cast<double>(gen() >> 11) * 0x1.0p-53) - 1.0;
}

int eb_random_fill_block(double* out, uint64_t seed, int nd, const int64_t* gshape,
                         const int64_t* base, const int64_t* shape) {
  return eb::guard([&] {
    if (nd < 1 || nd > 16 || !out || !gshape || !base || !shape)
      throw eb::InvalidError("eb_random_fill_block: bad arguments");
    for (int d = 0; d < nd; ++d)
      if (shape[d] < 0 || base[d] < 0 || base[d] + shape[d] > gshape[d])
        throw eb::InvalidError("eb_random_fill_block: block outside the tensor");
    std::int64_t n = 1;
    for (int d = 0; d < nd; ++d) n *= shape[d];
    if (n == 0) return;
    std::vector<std::int64_t> gstr(nd, 1);
    for (int d = nd - 1; d > 0; --d) gstr[d - 1] = gstr[d] * gshape[d];
    // walk the block's rows in stream order: skip the gap, draw the row
    std::mt19937_64 gen(seed);
    std::int64_t pos = 0;  // next stream index gen will produce
    const std::int64_t run = shape[nd - 1];
    std::vector<std::int64_t> idx(nd - 1, 0);
    for (std::int64_t row = 0; row < n / run; ++row) {
      std::int64_t off = base[nd - 1];
      for (int d = 0; d + 1 < nd; ++d) off += (base[d] + idx[d]) * gstr[d];
      if (off > pos) gen.discard(static_cast<unsigned long long>(off - pos));
      double* o = out + row * run;
      for (std::int64_t k = 0; k < run; ++k)
        o[k] = 2.0 * (static_cast<double>(gen() >> 11) * 0x1.0p-53) - 1.0;
      pos = off + run;
      for (int d = nd - 2; d >= 0; --d) {
        if (++idx[static_cast<std::size_t>(d)] < shape[d]) break;
        idx[static_cast<std::size_t>(d)] = 0;
      }
    }
  });
}

}  // extern "C"
