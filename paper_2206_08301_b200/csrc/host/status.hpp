// Error plumbing shared by the host layer and the kernel launchers.
// The planner throws einplan::Error (errc carries the einplan_status); the
// inner C ABI returns eb_status codes with a thread-local message.
#pragma once

#include <stdexcept>
#include <string>

#include "einplan_b200.h"

namespace eb {

void set_error(const std::string& msg);
const char* error_cstr();

// Thrown inside the launchers, mapped to eb_status at the C boundary.
struct DeviceError : std::runtime_error {
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};
struct InvalidError : std::runtime_error {
  explicit InvalidError(const std::string& m) : std::runtime_error(m) {}
};

#define EB_CUDA(call)                                                               \
  do {                                                                              \
    cudaError_t eb_err_ = (call);                                                   \
    if (eb_err_ != cudaSuccess)                                                     \
      throw ::eb::DeviceError(std::string(#call) + ": " + cudaGetErrorString(eb_err_)); \
  } while (0)

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return EB_OK;
  } catch (const InvalidError& e) {
    set_error(e.what());
    return EB_E_INVALID;
  } catch (const DeviceError& e) {
    set_error(e.what());
    return EB_E_DEVICE;
  } catch (const std::exception& e) {
    set_error(e.what());
    return EB_E_DEVICE;
  }
}

}  // namespace eb

#include <cuda_runtime.h>

namespace eb {
// Every kernel launch of the library is counted (bench.py's gpu_launches);
// the dominant contraction kernel can additionally be bracketed by CUDA
// events on its own stream (bench.py's live roofline timing).
void count_launch();
void count_launches(long long n);  // a CUDA-graph replay of n captured launches
// While this thread captures a CUDA graph the main-kernel events are skipped
// (they would become graph nodes).
void set_capturing(bool on);
void main_kernel_begin(cudaStream_t st);
void main_kernel_end(cudaStream_t st);

// Path-selection options.  Read ONCE from the environment when the library
// loads (EB_NO_FUSED_TMA, EB_NO_RF, EB_RF_CFG, EB_TTM2_VARIANT, EB_FUSE_TTM2)
// and changeable afterwards only through eb_set_option — no getenv on the
// launch path.  Defaults are the shipped kernels; the others exist for the
// parity tests of every path and for A/B measurements.
struct Options {
  int no_fused_tma = 0;   // per-16-column TMA boxes instead of one box per stage
  int no_rf = 0;          // general contraction kernel instead of the resident-factor one
  int rf_rt = 0, rf_os = 0;  // resident-factor tiling override (0 = automatic)
  int ttm2_variant = 0;   // 0 auto, 1 / 2 = ttm2_ws_kernel<1> / <2>
  int fuse_ttm2 = 1;      // executor: TTM pairs on eb_ttm2 (0: two eb_contract launches)
  int gemm = 0;           // wide GEMM steps: 0 auto, 1 GEMM mode forced, 2 split-K chunks
  int fuse_redistribution = 1;  // executor: push TTM outputs into the next term's blocks
  // executor: chained TTM-pair terms in one launch (eb_ttm2_chain).  Off by
  // default: measured 1.73 vs 1.60 ms on C5 although t1 never
  // reaches HBM (DRAM writes 534 MB -> 20 MB)
  int chain_terms = 0;
  // executor: TTMc-O5 terms joined by a self hand-over run as eb_ttmc_fold —
  // term B's m contraction folded into term A's epilogue, t1 never stored
  // (ttmc_fold.cu).  Off by default: measured 1.657 vs 1.589 ms on C5 (the
  // folded contraction's 2.15 GFLOP lands on the DMMA-saturated term-A
  // kernel).  chain_terms takes precedence when both are on.
  int fold_terms = 0;
  int chain_flags = 7;    // eb_ttm2_chain cache policy bits (ttm2.cu ChainParams::flags)
  int chain_lag = 1;      // eb_ttm2_chain: term B of slab p runs in group p + lag
  int pdl = 1;            // programmatic dependent launch for the chained kernels
  int scatter_fast = 1;   // ttm2 scatter: single-block fast tail path
  int zero_push = 0;      // zero the pushed destination blocks first (tests: missing stores)
};
const Options& options();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device).
void set_smem_attr_once(const void* kernel, int bytes);
template <typename K>
inline void set_smem_once(K* kernel, int bytes) {
  set_smem_attr_once(reinterpret_cast<const void*>(kernel), bytes);
}
}  // namespace eb
