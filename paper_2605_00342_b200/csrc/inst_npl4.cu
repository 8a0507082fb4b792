// Instantiation unit: trees with 64 < N ≤ 128 (4 nodes per lane).
#include "evict_kernels.cuh"
#include "evict_launch.h"

namespace evict {
template evict_status_t launch_select<4>(EVICT_SELECT_ARGS);
template evict_status_t launch_build<4>(EVICT_BUILD_ARGS);
template evict_status_t launch_union<4>(EVICT_UNION_ARGS);
template evict_status_t launch_fused<4>(EVICT_FUSED_ARGS);
}  // namespace evict
