// Host helpers shared by the sm_100a kernel launchers: TMA tensor-map
// encoding (cuTensorMapEncodeTiled through the runtime's driver entry point,
// FP64, SWIZZLE_128B), SM count and the sm_100 device check.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace eb {

// rank <= 5 dims (dims[0] contiguous), strides_bytes for dims 1..rank-1.
CUtensorMap make_map(const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                     const uint32_t* box);
int sm_count();
void check_device();  // throws DeviceError unless the current device is CC 10.x

}  // namespace eb
