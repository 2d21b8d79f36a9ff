// TEST INFRASTRUCTURE ONLY.  An extern "C" shim over the reference einplan
// C++ API (/root/reference/proj), compiled together with the reference's own
// sources into oracle/_ref/libeinplan_ref.so by oracle/Makefile.  Used by
// tests/ (oracle pinning, golden generation, schedule parity) and by
// bench.py's reference arm.  Nothing here is product code.
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "einplan/einsum.hpp"
#include "einplan/evaluate.hpp"
#include "einplan/executor.hpp"
#include "einplan/report.hpp"
#include "einplan/schedule.hpp"
#include "einplan/tensor.hpp"

using namespace einplan;

namespace {
thread_local std::string g_err;

std::map<char, std::int64_t> dims_of(const char* dims) {
  std::map<char, std::int64_t> out;
  std::string s(dims);
  std::size_t pos = 0;
  while (pos < s.size()) {
    std::size_t comma = s.find(',', pos);
    std::string item = s.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
    if (item.size() >= 3) out[item[0]] = std::stoll(item.substr(2));
    if (comma == std::string::npos) break;
    pos = comma + 1;
  }
  return out;
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_free(char* p) { std::free(p); }

// Reference random_tensor (tensor.cpp:55-63) into a caller buffer.
void ref_random_fill(double* out, std::int64_t n, std::uint64_t seed) {
  DenseTensor t = random_tensor({n}, seed);
  std::memcpy(out, t.data.data(), sizeof(double) * n);
}

// plan_report(make_pipeline(...)).dump(2) — the reference's plan JSON.
char* ref_plan_json(const char* einsum, const char* dims, std::int64_t procs,
                    double fast_mem, int include_messages) {
  try {
    auto spec = bind_extents(parse(einsum), dims_of(dims));
    auto pipe = make_pipeline(spec, procs, fast_mem);
    return dup(plan_report(pipe, fast_mem, include_messages != 0).dump(2));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// naive_evaluate (evaluate.cpp:7-63) on explicit operands (row-major, shapes
// implied by the einsum and dims).
int ref_naive_evaluate(const char* einsum, const char* dims, const double* const* ops,
                       double* out) {
  try {
    auto spec = bind_extents(parse(einsum), dims_of(dims));
    std::vector<DenseTensor> in;
    for (std::size_t k = 0; k < spec.inputs.size(); ++k) {
      DenseTensor t(spec.shape_of(spec.inputs[k]));
      std::memcpy(t.data.data(), ops[k], sizeof(double) * t.data.size());
      in.push_back(std::move(t));
    }
    DenseTensor r = naive_evaluate(spec, in);
    std::memcpy(out, r.data.data(), sizeof(double) * r.data.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Plan with make_pipeline, then run() (executor.cpp:156-263) with verify off
// on explicit operands.  Wall seconds of run() alone go to *run_seconds;
// comm volumes to comm[0..2] = allreduce, redistribute, max_rank_sent.
int ref_run(const char* einsum, const char* dims, std::int64_t procs, double fast_mem,
            const double* const* ops, double* out, double* run_seconds,
            std::int64_t* comm) {
  try {
    auto spec = bind_extents(parse(einsum), dims_of(dims));
    auto pipe = make_pipeline(spec, procs, fast_mem);
    std::vector<DenseTensor> in;
    for (std::size_t k = 0; k < spec.inputs.size(); ++k) {
      DenseTensor t(spec.shape_of(spec.inputs[k]));
      std::memcpy(t.data.data(), ops[k], sizeof(double) * t.data.size());
      in.push_back(std::move(t));
    }
    RunOptions opts;
    opts.verify = false;
    auto t0 = std::chrono::steady_clock::now();
    SimulationReport rep = run(pipe.schedule, spec, pipe.tree, in, opts);
    auto t1 = std::chrono::steady_clock::now();
    if (run_seconds) *run_seconds = std::chrono::duration<double>(t1 - t0).count();
    std::memcpy(out, rep.output.data.data(), sizeof(double) * rep.output.data.size());
    if (comm) {
      comm[0] = rep.comm.allreduce_volume;
      comm[1] = rep.comm.redistribute_volume;
      comm[2] = rep.comm.max_rank_sent();
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // extern "C"
