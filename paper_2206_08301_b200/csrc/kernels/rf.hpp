// Resident-factor MTTKRP term (mttkrp_rf.cu) and the partial-slot reduction
// it shares with the general contraction kernel (contract.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "einplan_b200.h"

namespace eb {

// Workspace the resident-factor path needs for d, or 0 when it does not
// apply (then eb_contract runs the general kernel).
size_t rf_workspace(const eb_contract_desc* d);
// Runs d on the resident-factor kernel; false (nothing launched) when it does
// not apply.
bool rf_run(const eb_contract_desc* d, void* ws, size_t ws_bytes, cudaStream_t st);

void launch_reduce(const double* ws, double* out, int64_t M, int R, int col0, int64_t ldo, int NP,
                   int MT, int SPL, int64_t per_tile, int64_t items, int G, int segmax,
                   cudaStream_t st);

}  // namespace eb
