// router.cu — A8: router logits on tcgen05 tensor cores + TopK + expert union.
#include <cuda_runtime.h>
#include <stdint.h>

#include "evict.h"

extern "C" evict_status_t evict_router_union(const evict_trees_t *trees, const int32_t *verify_offsets,
                                             const int32_t *retrieve_index, const evict_router_t *router,
                                             int32_t *union_count, int32_t *union_total,
                                             uint64_t *union_bits, int32_t *topk_ids, void *stream)
{
    (void)trees; (void)verify_offsets; (void)retrieve_index; (void)router; (void)union_count;
    (void)union_total; (void)union_bits; (void)topk_ids; (void)stream;
    return EVICT_ERR_UNSUPPORTED;
}
