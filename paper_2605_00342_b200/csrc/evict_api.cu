// evict_api.cu — C-ABI entry points of libevict.so: host-side argument checks,
// device check (sm_100), workspace clearing and dispatch to the per-NPL
// launchers (inst_npl2.cu, inst_npl4.cu).  No host sync, no allocation: every
// call is stream-ordered and CUDA-graph capturable.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "evict.h"
#include "evict_launch.h"

namespace evict {

namespace {
struct DevInfo {
    int sms = 0;
    int ok = 0;
};

DevInfo dev_info()
{
    static DevInfo cache[64];
    static std::once_flag flags[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return DevInfo{};
    std::call_once(flags[dev], [dev] {
        int major = 0, minor = 0, sms = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cache[dev].sms = sms;
        cache[dev].ok = (major == 10 && minor == 0);
    });
    return cache[dev];
}

evict_status_t check_trees(const evict_trees_t *t)
{
    if (!t || !t->parent || !t->q) return EVICT_ERR_INVALID_ARG;
    if (t->batch < 1 || t->max_nodes < 1 || t->max_nodes > EVICT_MAX_NODES || (t->max_nodes % 4))
        return EVICT_ERR_INVALID_ARG;
    if (((uintptr_t)t->parent | (uintptr_t)t->q) & 15) return EVICT_ERR_INVALID_ARG;
    return EVICT_OK;
}

evict_status_t check_routing(const evict_routing_t *r)
{
    if (!r || !r->ids) return EVICT_ERR_INVALID_ARG;
    if (r->num_layers < 1 || r->num_layers > EVICT_MAX_LAYERS) return EVICT_ERR_INVALID_ARG;
    if (r->num_experts < 1 || r->num_experts > EVICT_MAX_EXPERTS) return EVICT_ERR_INVALID_ARG;
    if (r->id_format != EVICT_ID_U8 && r->id_format != EVICT_ID_I32 && r->id_format != EVICT_ID_MASK)
        return EVICT_ERR_INVALID_ARG;
    if (r->id_format != EVICT_ID_MASK &&
        (r->top_k < 1 || r->top_k > EVICT_MAX_TOPK || r->top_k > r->num_experts))
        return EVICT_ERR_INVALID_ARG;
    if ((uintptr_t)r->ids & 15) return EVICT_ERR_INVALID_ARG;
    return EVICT_OK;
}

bool wide(int N) { return N > 64; }  // 4 nodes per lane, else 2
}  // namespace

int dev_sms() { return dev_info().sms; }
bool dev_supported() { return dev_info().ok != 0; }

}  // namespace evict

using namespace evict;

extern "C" {

int evict_abi_version(void) { return EVICT_ABI_VERSION; }

const char *evict_status_string(evict_status_t s)
{
    switch (s) {
    case EVICT_OK: return "ok";
    case EVICT_ERR_INVALID_ARG: return "invalid argument";
    case EVICT_ERR_UNSUPPORTED: return "unsupported shape or device (needs sm_100)";
    case EVICT_ERR_CUDA: return "CUDA launch error";
    }
    return "unknown status";
}

size_t evict_workspace_bytes(int32_t batch)
{
    if (batch < 1) return 0;
    // one state word per tile of the finest tiling: k_fused takes one-tree warp tiles up to
    // kFusedSmallBatch trees (serving batches), 4-tree tiles above; k_build 8-tree CTA tiles
    const int tt = batch <= kFusedSmallBatch ? 1 : (kTileTrees < kFusedTileTrees ? kTileTrees : kFusedTileTrees);
    const size_t ntiles = ((size_t)batch + tt - 1) / tt;
    return 8 * (1 + ntiles);
}

static bool policy_ok(const evict_policy_t *p, evict_policy_t *out)
{
    *out = evict_policy_t{EVICT_POLICY_COST, 0.f, 0};
    if (!p) return true;
    if (p->kind == EVICT_POLICY_COST) return true;
    if (p->kind == EVICT_POLICY_COVERAGE) {
        if (!(p->rho > 0.f && p->rho <= 1.f)) return false;   // also rejects NaN
    } else if (p->kind == EVICT_POLICY_FIXED) {
        if (p->k_fixed < 1) return false;
    } else {
        return false;
    }
    *out = *p;
    return true;
}

evict_status_t evict_select(const evict_trees_t *trees, const float *cost, int32_t cost_stride,
                            int32_t *k_star, float *e_hat, float *utility, uint64_t *keep_bits,
                            int32_t *order, float *prefix_sums, uint32_t *status, void *stream)
{
    return evict_select_policy(trees, cost, cost_stride, nullptr, k_star, e_hat, utility, keep_bits,
                               order, prefix_sums, status, stream);
}

evict_status_t evict_select_policy(const evict_trees_t *trees, const float *cost, int32_t cost_stride,
                                   const evict_policy_t *policy, int32_t *k_star, float *e_hat,
                                   float *utility, uint64_t *keep_bits, int32_t *order,
                                   float *prefix_sums, uint32_t *status, void *stream)
{
    evict_policy_t pol;
    if (!policy_ok(policy, &pol)) return EVICT_ERR_INVALID_ARG;
    evict_status_t rc = check_trees(trees);
    if (rc) return rc;
    if (!cost || !k_star || !e_hat || !utility || !keep_bits || cost_stride < 0) return EVICT_ERR_INVALID_ARG;
    if (((uintptr_t)cost & 15) || (cost_stride % 4)) return EVICT_ERR_INVALID_ARG;
    if ((order == nullptr) != (prefix_sums == nullptr)) return EVICT_ERR_INVALID_ARG;
    if (!dev_info().ok) return EVICT_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    if (wide(trees->max_nodes))
        return launch_select<4>(trees, cost, cost_stride, pol, k_star, e_hat, utility, keep_bits, order,
                                prefix_sums, status, s);
    return launch_select<2>(trees, cost, cost_stride, pol, k_star, e_hat, utility, keep_bits, order,
                            prefix_sums, status, s);
}

evict_status_t evict_build_verify_tree(const evict_trees_t *trees, const uint64_t *keep_bits,
                                       const int32_t *pos_offset, int32_t *verify_offsets,
                                       int32_t *kept_index, int32_t *retrieve_index,
                                       int32_t *positions, int32_t *next_token,
                                       int32_t *next_sibling, uint64_t *tree_mask,
                                       uint32_t *status, void *workspace, size_t workspace_bytes,
                                       void *stream)
{
    evict_status_t rc = check_trees(trees);
    if (rc) return rc;
    if (!keep_bits || !verify_offsets || !workspace) return EVICT_ERR_INVALID_ARG;
    if (workspace_bytes < evict_workspace_bytes(trees->batch) || ((uintptr_t)workspace & 7))
        return EVICT_ERR_INVALID_ARG;
    if (!dev_info().ok) return EVICT_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    const int ntiles = (trees->batch + kTileTrees - 1) / kTileTrees;
    if (cudaMemsetAsync(workspace, 0, evict_workspace_bytes(trees->batch), s) != cudaSuccess)
        return EVICT_ERR_CUDA;
    uint64_t *ws = (uint64_t *)workspace;
    if (wide(trees->max_nodes))
        return launch_build<4>(trees, keep_bits, pos_offset, verify_offsets, kept_index, retrieve_index,
                               positions, next_token, next_sibling, tree_mask, status, ws, ntiles, s);
    return launch_build<2>(trees, keep_bits, pos_offset, verify_offsets, kept_index, retrieve_index,
                           positions, next_token, next_sibling, tree_mask, status, ws, ntiles, s);
}

evict_status_t evict_expert_union(const evict_trees_t *trees, const uint64_t *keep_bits,
                                  const evict_routing_t *routing, int32_t *union_count,
                                  int32_t *union_total, uint64_t *union_bits,
                                  int64_t *expert_hist, uint32_t *status, void *stream)
{
    if (!trees || trees->batch < 1 || trees->max_nodes < 1 || trees->max_nodes > EVICT_MAX_NODES ||
        (trees->max_nodes % 4))
        return EVICT_ERR_INVALID_ARG;
    evict_status_t rc = check_routing(routing);
    if (rc) return rc;
    if (!keep_bits || !union_count) return EVICT_ERR_INVALID_ARG;
    if (!dev_info().ok) return EVICT_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    if (wide(trees->max_nodes))
        return launch_union<4>(trees, keep_bits, routing, union_count, union_total, union_bits, expert_hist, status, s);
    return launch_union<2>(trees, keep_bits, routing, union_count, union_total, union_bits, expert_hist, status, s);
}

evict_status_t evict_select_build_union(const evict_trees_t *trees, const float *cost,
                                        int32_t cost_stride, const evict_routing_t *routing,
                                        const evict_fused_out_t *out, void *workspace,
                                        size_t workspace_bytes, void *stream)
{
    return evict_select_build_union_policy(trees, cost, cost_stride, nullptr, routing, out, workspace,
                                           workspace_bytes, stream);
}

evict_status_t evict_select_build_union_policy(const evict_trees_t *trees, const float *cost,
                                               int32_t cost_stride, const evict_policy_t *policy,
                                               const evict_routing_t *routing,
                                               const evict_fused_out_t *out, void *workspace,
                                               size_t workspace_bytes, void *stream)
{
    evict_policy_t pol;
    if (!policy_ok(policy, &pol)) return EVICT_ERR_INVALID_ARG;
    evict_status_t rc = check_trees(trees);
    if (rc) return rc;
    if (!cost || cost_stride < 0 || !out || !workspace) return EVICT_ERR_INVALID_ARG;
    if (((uintptr_t)cost & 15) || (cost_stride % 4)) return EVICT_ERR_INVALID_ARG;
    if ((out->order == nullptr) != (out->prefix_sums == nullptr)) return EVICT_ERR_INVALID_ARG;
    if (workspace_bytes < evict_workspace_bytes(trees->batch) || ((uintptr_t)workspace & 7))
        return EVICT_ERR_INVALID_ARG;
    evict_routing_t none{1, 1, 1, EVICT_ID_MASK, nullptr};
    const evict_routing_t *rt = &none;
    if (out->union_count) {
        rc = check_routing(routing);
        if (rc) return rc;
        rt = routing;
    }
    // A9 (ABI 8): statistics over the call's own outputs
    const bool want_stats = out->stats || out->dstats;
    if (want_stats && (!out->stats || !out->dstats || !out->k_star || !out->e_hat || !out->utility ||
                       !out->status))
        return EVICT_ERR_INVALID_ARG;
    if (!dev_info().ok) return EVICT_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    const int tt = trees->batch <= kFusedSmallBatch ? 1 : kFusedTileTrees;
    const int ntiles = (trees->batch + tt - 1) / tt;
    if (cudaMemsetAsync(workspace, 0, 8 * (1 + (size_t)ntiles), s) != cudaSuccess)
        return EVICT_ERR_CUDA;
    // folded into the launch for the single-pass E = 128 serving union (k_fused kFold), else the
    // statistics kernel runs after it
    const int L = out->union_count ? rt->num_layers : 0;
    const bool fold = want_stats && trees->batch > kFusedSmallBatch && out->union_count &&
                      rt->id_format == EVICT_ID_U8 && rt->top_k == 8 &&
                      rt->num_experts == 128 && L <= 64 && !out->order && !out->union_bits && !out->expert_hist;
    evict_fused_out_t o = *out;
    if (want_stats) {
        if (!fold) {
            o.stats = nullptr;
            o.dstats = nullptr;
        } else if (cudaMemsetAsync(out->stats, 0, sizeof(int64_t) * (6 + (size_t)trees->max_nodes + L), s) != cudaSuccess ||
                   cudaMemsetAsync(out->dstats, 0, 2 * sizeof(double), s) != cudaSuccess) {
            return EVICT_ERR_CUDA;
        }
    }
    uint64_t *ws = (uint64_t *)workspace;
    rc = wide(trees->max_nodes) ? launch_fused<4>(trees, cost, (int)cost_stride, pol, rt, &o, ws, ntiles, s)
                                : launch_fused<2>(trees, cost, (int)cost_stride, pol, rt, &o, ws, ntiles, s);
    if (rc || !want_stats || fold) return rc;
    return evict_batch_stats(trees->batch, trees->max_nodes, L, trees->n_nodes, out->k_star, out->e_hat,
                             out->utility, L ? out->union_count : nullptr, out->status, out->stats,
                             out->dstats, stream);
}

}  // extern "C"

