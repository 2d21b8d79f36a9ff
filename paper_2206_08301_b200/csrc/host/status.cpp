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
#include <mutex>
#include <utility>
#include <vector>

namespace eb {

namespace {
std::atomic<long long> g_launches{0};
std::atomic<bool> g_timing{false};
std::mutex g_mu;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_events;
cudaEvent_t g_open = nullptr;
}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void main_kernel_begin(cudaStream_t st) {
  if (!g_timing.load()) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEventCreate(&g_open);
  cudaEventRecord(g_open, st);
}

void main_kernel_end(cudaStream_t st) {
  if (!g_timing.load()) return;
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
