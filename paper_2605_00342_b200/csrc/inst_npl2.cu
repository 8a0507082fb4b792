// Instantiation unit: trees with N ≤ 64 (2 nodes per lane).
#include "evict_kernels.cuh"
#include "evict_launch.h"

namespace evict {
template evict_status_t launch_select<2>(EVICT_SELECT_ARGS);
template evict_status_t launch_build<2>(EVICT_BUILD_ARGS);
template evict_status_t launch_union<2>(EVICT_UNION_ARGS);
template evict_status_t launch_fused<2>(EVICT_FUSED_ARGS);
}  // namespace evict
