#include "status.hpp"

namespace eb {

namespace {
thread_local std::string g_error;
}

void set_error(const std::string& msg) { g_error = msg; }
const char* error_cstr() { return g_error.c_str(); }

}  // namespace eb

extern "C" const char* eb_last_error(void) { return eb::error_cstr(); }

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>
#include <vector>

namespace eb {

namespace {
std::atomic<long long> g_launches{0};
std::atomic<bool> g_timing{false};
std::mutex g_mu;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_events;
thread_local cudaEvent_t g_open = nullptr;  // one open bracket per launching thread
thread_local bool g_capturing = false;

Options read_env() {
  Options o;
  auto flag = [](const char* n) {
    const char* v = std::getenv(n);
    return v && v[0] && v[0] != '0';
  };
  o.no_fused_tma = flag("EB_NO_FUSED_TMA");
  o.no_rf = flag("EB_NO_RF");
  if (const char* v = std::getenv("EB_RF_CFG")) std::sscanf(v, "%dx%d", &o.rf_rt, &o.rf_os);
  if (const char* v = std::getenv("EB_TTM2_VARIANT")) o.ttm2_variant = std::atoi(v);
  if (const char* v = std::getenv("EB_FUSE_TTM2")) o.fuse_ttm2 = v[0] != '0';
  if (const char* v = std::getenv("EB_GEMM")) o.gemm = std::atoi(v);
  if (const char* v = std::getenv("EB_FUSE_REDIST")) o.fuse_redistribution = v[0] != '0';
  if (const char* v = std::getenv("EB_CHAIN_TERMS")) o.chain_terms = v[0] != '0';
  if (const char* v = std::getenv("EB_FOLD_TERMS")) o.fold_terms = v[0] != '0';
  if (const char* v = std::getenv("EB_CHAIN_FLAGS")) o.chain_flags = std::atoi(v);
  if (const char* v = std::getenv("EB_CHAIN_LAG")) o.chain_lag = std::atoi(v);
  if (const char* v = std::getenv("EB_PDL")) o.pdl = v[0] != '0';
  if (const char* v = std::getenv("EB_SCATTER_FAST")) o.scatter_fast = v[0] != '0';
  if (const char* v = std::getenv("EB_ZERO_PUSH")) o.zero_push = v[0] != '0';
  return o;
}

Options g_opts = read_env();  // at library load
std::mutex g_attr_mu;
std::set<std::pair<const void*, int>> g_attr_done;
}  // namespace

const Options& options() { return g_opts; }

void set_smem_attr_once(const void* kernel, int bytes) {
  int dev = 0;
  EB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (g_attr_done.count({kernel, dev})) return;
  EB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  g_attr_done.insert({kernel, dev});
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
void set_capturing(bool on) { g_capturing = on; }

void main_kernel_begin(cudaStream_t st) {
  if (!g_timing.load() || g_capturing) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEventCreate(&g_open);
  cudaEventRecord(g_open, st);
}

void main_kernel_end(cudaStream_t st) {
  if (!g_timing.load() || g_capturing) return;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_open) return;
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  g_events.emplace_back(g_open, e);
  g_open = nullptr;
}

}  // namespace eb

extern "C" long long eb_launch_count(void) { return eb::g_launches.load(); }

// Options (status.hpp): not thread-safe against concurrent launches; set
// them between runs.
extern "C" int eb_set_option(const char* name, const char* value) {
  return eb::guard([&] {
    if (!name || !value) throw eb::InvalidError("eb_set_option: null argument");
    eb::Options& o = eb::g_opts;
    const int v = std::atoi(value);
    if (!std::strcmp(name, "no_fused_tma")) {
      o.no_fused_tma = v != 0;
    } else if (!std::strcmp(name, "no_rf")) {
      o.no_rf = v != 0;
    } else if (!std::strcmp(name, "rf_cfg")) {
      int rt = 0, os = 0;
      if (value[0] && std::strcmp(value, "auto") && std::sscanf(value, "%dx%d", &rt, &os) != 2)
        throw eb::InvalidError("eb_set_option: rf_cfg is \"RTxOS\" or \"auto\"");
      o.rf_rt = rt;
      o.rf_os = os;
    } else if (!std::strcmp(name, "ttm2_variant")) {
      if (v < 0 || v > 2) throw eb::InvalidError("eb_set_option: ttm2_variant is 0, 1 or 2");
      o.ttm2_variant = v;
    } else if (!std::strcmp(name, "fuse_ttm2")) {
      o.fuse_ttm2 = v != 0;
    } else if (!std::strcmp(name, "zero_push")) {
      o.zero_push = v != 0;
    } else if (!std::strcmp(name, "scatter_fast")) {
      o.scatter_fast = v != 0;
    } else if (!std::strcmp(name, "pdl")) {
      o.pdl = v != 0;
    } else if (!std::strcmp(name, "chain_terms")) {
      o.chain_terms = v != 0;
    } else if (!std::strcmp(name, "fold_terms")) {
      o.fold_terms = v != 0;
    } else if (!std::strcmp(name, "fuse_redistribution")) {
      o.fuse_redistribution = v != 0;
    } else if (!std::strcmp(name, "gemm")) {
      if (v < 0 || v > 2) throw eb::InvalidError("eb_set_option: gemm is 0, 1 or 2");
      o.gemm = v;
    } else {
      throw eb::InvalidError(std::string("eb_set_option: unknown option \"") + name + "\"");
    }
  });
}

extern "C" void eb_timer_enable(int on) { eb::g_timing.store(on != 0); }

// Sum of the bracketed main-kernel durations since the last collect (ms),
// and how many launches they cover.  Synchronises on the recorded events.
extern "C" int eb_timer_collect(double* total_ms, long long* launches) {
  std::lock_guard<std::mutex> lk(eb::g_mu);
  double sum = 0.0;
  long long n = 0;
  for (auto& pr : eb::g_events) {
    cudaEventSynchronize(pr.second);
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) {
      sum += ms;
      ++n;
    }
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  eb::g_events.clear();
  if (total_ms) *total_ms = sum;
  if (launches) *launches = n;
  return 0;
}
