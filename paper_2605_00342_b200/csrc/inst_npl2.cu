// Instantiation unit: trees with N ≤ 64 (2 nodes per lane).
#include "evict_kernels.cuh"
#include "evict_launch.h"

namespace evict {
template evict_status_t launch_select<2>(EVICT_SELECT_ARGS);
template evict_status_t launch_build<2>(EVICT_BUILD_ARGS);
template evict_status_t launch_union<2>(EVICT_UNION_ARGS);
template evict_status_t launch_fused<2>(EVICT_FUSED_ARGS);
}  // namespace evict

#ifdef EVICT_PHASE_TIMING
// profiling variant only (not in include/evict.h): read and clear k_fused's per-phase cycle
// sums of this unit (N ≤ 64): [0] select, [1] publish + early look-back, [2] union,
// [3] late look-back, [4] emit
extern "C" int evict_debug_phase_cycles(unsigned long long *out)
{
    if (cudaMemcpyFromSymbol(out, evict::g_phase_cycles, 8 * sizeof(unsigned long long)) != cudaSuccess) return 1;
    static const unsigned long long zero[8] = {};
    return cudaMemcpyToSymbol(evict::g_phase_cycles, zero, sizeof(zero)) != cudaSuccess;
}
#endif
