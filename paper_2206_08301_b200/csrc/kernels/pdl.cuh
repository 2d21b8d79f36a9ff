// Programmatic dependent launch (sm_90+): a kernel launched with
// launch_pdl may be scheduled while the previous kernel in the stream is
// still draining; it must call grid_dep_wait() before its first global
// memory access (read or write), which returns once the previous grid has
// completed and its writes are visible.  Hides the launch latency and the
// barrier-init / descriptor-prefetch prologue between the dependent kernels
// of one contraction (factor staging -> contraction -> partial reduction).
#pragma once

#include <cuda_runtime.h>

#include <utility>

#include "../host/status.hpp"

namespace eb {

__device__ __forceinline__ void grid_dep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = options().pdl ? 1 : 0;
  EB_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

}  // namespace eb
