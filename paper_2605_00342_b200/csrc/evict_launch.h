// evict_launch.h — internal declarations shared by evict_api.cu and the
// per-NPL instantiation units (inst_npl2.cu, inst_npl4.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "evict.h"

#define EVICT_SELECT_ARGS                                                                       \
    const evict_trees_t *, const float *, int, evict_policy_t, int32_t *, float *, float *,     \
        uint64_t *, int32_t *, float *, uint32_t *, cudaStream_t
#define EVICT_BUILD_ARGS                                                                        \
    const evict_trees_t *, const uint64_t *, const int32_t *, int32_t *, int32_t *, int32_t *,  \
        int32_t *, int32_t *, int32_t *, uint64_t *, uint32_t *, uint64_t *, int, cudaStream_t
#define EVICT_UNION_ARGS                                                                        \
    const evict_trees_t *, const uint64_t *, const evict_routing_t *, int32_t *, int32_t *,     \
        uint64_t *, int64_t *, uint32_t *, cudaStream_t
#define EVICT_FUSED_ARGS                                                                        \
    const evict_trees_t *, const float *, int, evict_policy_t, const evict_routing_t *,         \
        const evict_fused_out_t *, uint64_t *, int, cudaStream_t

namespace evict {
constexpr int kTileTrees = 8;        // trees per CTA tile of k_build (= warps per CTA)
constexpr int kFusedTileTrees = 4;   // trees per warp tile of k_fused
constexpr int kFusedSmallBatch = 2048;   // k_fused LEAN takes one-tree tiles up to this batch
int dev_sms();
bool dev_supported();   // the current device is sm_100 (B200); else every entry point returns UNSUPPORTED
template <int NPL> evict_status_t launch_select(EVICT_SELECT_ARGS);
template <int NPL> evict_status_t launch_build(EVICT_BUILD_ARGS);
template <int NPL> evict_status_t launch_union(EVICT_UNION_ARGS);
template <int NPL> evict_status_t launch_fused(EVICT_FUSED_ARGS);
extern template evict_status_t launch_select<2>(EVICT_SELECT_ARGS);
extern template evict_status_t launch_select<4>(EVICT_SELECT_ARGS);
extern template evict_status_t launch_build<2>(EVICT_BUILD_ARGS);
extern template evict_status_t launch_build<4>(EVICT_BUILD_ARGS);
extern template evict_status_t launch_union<2>(EVICT_UNION_ARGS);
extern template evict_status_t launch_union<4>(EVICT_UNION_ARGS);
extern template evict_status_t launch_fused<2>(EVICT_FUSED_ARGS);
extern template evict_status_t launch_fused<4>(EVICT_FUSED_ARGS);
}  // namespace evict
