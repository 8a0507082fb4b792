#pragma once
// evict_kernels.cuh — kernels of libevict.so (sm_100a), instantiated per
// nodes-per-lane (NPL) in inst_npl2.cu / inst_npl4.cu and called from the
// C-ABI in evict_api.cu.
//
// Launch model: one warp per draft tree, 8 trees per 256-thread CTA tile.
//  - k_select:  A1–A5, a plain grid over trees.
//  - k_build:   A6, persistent CTAs pulling tiles from a ticket counter; the
//               packed-row offsets are a single-pass decoupled look-back scan
//               over tiles (tile state words in the caller's workspace).
//  - k_union:   A7, a plain grid over trees.
//  - k_fused:   A1–A7 in one persistent launch; the tree never leaves the SM
//               between select, build and union.
//  - k_stats:   A9 batch statistics (smem partials + global atomics).
// The router GEMM (A8) lives in router.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include "evict.h"
#include "evict_tree.cuh"

namespace evict {

// ------------------------------------------------------------ tile scan
// Workspace: [0] uint32 ticket (8-byte slot), [1..] uint64 tile states.
// state = flag << 62 | value; flag 1 = tile aggregate, 2 = inclusive prefix.
constexpr uint64_t kAgg = 1ull << 62;
constexpr uint64_t kInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_acquire(const uint64_t *p)
{
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint64_t *p, uint64_t v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Called by all threads of the CTA after every warp stored its tree's row
// count in s_cnt[warp].  Returns (in s_off[warp]) the packed-row offset of
// each warp's tree.  Thread 0 publishes and looks back.
__device__ __forceinline__ void tile_scan(int tile, uint64_t *states, int *s_cnt, int *s_off)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        int agg = 0;
        for (int w = 0; w < kWarps; w++) {
            s_off[w] = agg;
            agg += s_cnt[w];
        }
        uint64_t prefix = 0;
        if (tile == 0) {
            st_release(states + tile, kInc | (uint64_t)agg);
        } else {
            st_release(states + tile, kAgg | (uint64_t)agg);
            int j = tile - 1;
            while (true) {
                uint64_t s = ld_acquire(states + j);
                if ((s >> 62) == 0) continue;           // predecessor not published yet
                prefix += s & kValMask;
                if ((s >> 62) == 2) break;
                j--;
            }
            st_release(states + tile, kInc | (prefix + (uint64_t)agg));
        }
        for (int w = 0; w < kWarps; w++) s_off[w] += (int)prefix;
    }
    __syncthreads();
}

__device__ __forceinline__ int next_tile(unsigned *ticket, int *s_tile)
{
    __syncthreads();
    if (threadIdx.x == 0) *s_tile = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    return *s_tile;
}

// ------------------------------------------------------------ select
template <int NPL>
__global__ void __launch_bounds__(kWarps * 32) k_select(evict_trees_t tr, const float *cost,
                                                        int cost_stride, int32_t *k_star,
                                                        float *e_hat, float *utility,
                                                        uint64_t *keep_bits, int32_t *order,
                                                        float *prefix_sums, uint32_t *status)
{
    __shared__ WarpSlab<NPL> slab[kWarps];
    constexpr int W = Shape<NPL>::W;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int b = blockIdx.x * kWarps + warp;
    if (b >= tr.batch) return;
    const int N = tr.max_nodes;
    TreeState<NPL> t;
    WarpSlab<NPL> &sm = slab[warp];
    tree_load_validate<NPL>(t, tr, tr.parent, tr.q, tr.n_nodes, b, N);
    float c[NPL];
    if (!(t.status & EVICT_TREE_BAD_SIZE)) tree_load_cost<NPL>(c, t, cost + (size_t)b * cost_stride);
    int32_t *orow = order ? order + (size_t)b * N : nullptr;
    float *prow = prefix_sums ? prefix_sums + (size_t)b * N : nullptr;
    if (!t.status) {
        tree_levels<NPL, true>(t, sm);
        tree_rank_argmax<NPL>(t, sm, c, N, orow, prow);
    } else {
        t.kstar = 0; t.ehat = 0.f; t.util = 0.f;
#pragma unroll
        for (int w = 0; w < W; w++) t.keep[w] = 0ull;
        if (orow)
            for (int p = lane; p < N; p += 32) { orow[p] = -1; prow[p] = 0.f; }
    }
    if (lane == 0) {
        k_star[b] = t.kstar;
        e_hat[b] = t.ehat;
        utility[b] = t.util;
        if (status) status[b] = t.status;
    }
    // keep_bits row has ceil(N/64) words; write them (NMAX ≥ N)
    const int WN = (N + 63) / 64;
    if (lane < WN) keep_bits[(size_t)b * WN + lane] = t.keep[lane < W ? lane : 0];
}

// ------------------------------------------------------------ build
template <int NPL>
__global__ void __launch_bounds__(kWarps * 32) k_build(evict_trees_t tr, const uint64_t *keep_bits,
                                                       const int32_t *pos_offset,
                                                       int32_t *verify_offsets, int32_t *kept_index,
                                                       int32_t *retrieve_index, int32_t *positions,
                                                       int32_t *next_token, int32_t *next_sibling,
                                                       uint64_t *tree_mask, uint32_t *status,
                                                       uint64_t *ws, int ntiles)
{
    __shared__ WarpSlab<NPL> slab[kWarps];
    __shared__ int s_cnt[kWarps], s_off[kWarps], s_tile;
    constexpr int W = Shape<NPL>::W;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int N = tr.max_nodes;
    const int WN = (N + 63) / 64;
    unsigned *ticket = reinterpret_cast<unsigned *>(ws);
    uint64_t *states = ws + 1;
    WarpSlab<NPL> &sm = slab[warp];
    while (true) {
        const int tile = next_tile(ticket, &s_tile);
        if (tile >= ntiles) break;
        const int b = tile * kWarps + warp;
        TreeState<NPL> t;
        int k = 0;
        if (b < tr.batch) {
            tree_load_validate<NPL>(t, tr, tr.parent, tr.q, tr.n_nodes, b, N);
            t.status &= ~(uint32_t)EVICT_TREE_BAD_PROB;      // q is not an input of A6
#pragma unroll
            for (int w = 0; w < W; w++) t.keep[w] = (w < WN) ? __ldg(keep_bits + (size_t)b * WN + w) : 0ull;
            if (!t.status) {
                tree_levels<NPL, false>(t, sm);
                k = tree_check_keep<NPL>(t);
                if (t.status) k = 0;
            }
        }
        if (lane == 0) s_cnt[warp] = k;
        tile_scan(tile, states, s_cnt, s_off);
        if (b < tr.batch) {
            const int off = s_off[warp];
            if (lane == 0) {
                verify_offsets[b] = off;
                if (b == tr.batch - 1) verify_offsets[tr.batch] = off + k;
                if (status) status[b] = t.status;
            }
            if (k > 0)
                tree_build_emit<NPL>(t, sm, k, b, N, off, pos_offset ? __ldg(pos_offset + b) : 0,
                                     kept_index, retrieve_index, positions, next_token,
                                     next_sibling, tree_mask);
        }
    }
}

// ------------------------------------------------------------ union
template <int NPL>
__device__ __forceinline__ void tree_fill_klist(const TreeState<NPL> &t, WarpSlab<NPL> &sm)
{
    constexpr int W = Shape<NPL>::W;
    const int base = lane_id() * NPL;
#pragma unroll
    for (int r = 0; r < NPL; r++) {
        const int i = base + r;
        if (i < t.n && bit_of<W>(t.keep, i)) sm.klist[popc_below<W>(t.keep, i)] = (uint8_t)i;
    }
    __syncwarp();
}

template <int NPL, int IDF, int KT, int EW, int CL>
__global__ void __launch_bounds__(kWarps * 32) k_union(evict_trees_t tr, const uint64_t *keep_bits,
                                                       evict_routing_t rt, int32_t *union_count,
                                                       int32_t *union_total, uint64_t *union_bits,
                                                       int64_t *expert_hist, uint32_t *status)
{
    __shared__ WarpSlab<NPL> slab[kWarps];
    constexpr int W = Shape<NPL>::W;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int b = blockIdx.x * kWarps + warp;
    if (b >= tr.batch) return;
    const int N = tr.max_nodes;
    const int WN = (N + 63) / 64;
    WarpSlab<NPL> &sm = slab[warp];
    TreeState<NPL> t;
    t.n = tr.n_nodes ? __ldg(tr.n_nodes + b) : N;
    t.status = (t.n < 1 || t.n > N) ? EVICT_TREE_BAD_SIZE : 0u;
#pragma unroll
    for (int w = 0; w < W; w++) {
        uint64_t m = (w < WN) ? __ldg(keep_bits + (size_t)b * WN + w) : 0ull;
        const int lo = w * 64;
        // nodes past n are not part of the tree (same as the oracle)
        uint64_t valid = t.n >= lo + 64 ? ~0ull : (t.n <= lo ? 0ull : ((1ull << (t.n - lo)) - 1ull));
        t.keep[w] = m & valid;
    }
    int k = 0;
#pragma unroll
    for (int w = 0; w < W; w++) k += __popcll(t.keep[w]);
    if (!t.status) tree_fill_klist<NPL>(t, sm);
    uint32_t st = t.status;
    tree_union<NPL, IDF, KT, EW, CL>(st, sm, k, b, N, rt.num_layers, rt.top_k, rt.num_experts,
                                     rt.id_format, rt.ids, union_count, union_total, union_bits, expert_hist);
    if (status && lane == 0) status[b] = st;
}

// ------------------------------------------------------------ fused
template <int NPL, int IDF, int KT, int EW, int CL>
__global__ void __launch_bounds__(kWarps * 32) k_fused(evict_trees_t tr, const float *cost,
                                                       int cost_stride, evict_routing_t rt,
                                                       evict_fused_out_t out, uint64_t *ws,
                                                       int ntiles)
{
    __shared__ WarpSlab<NPL> slab[kWarps];
    __shared__ int s_cnt[kWarps], s_off[kWarps], s_tile;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int N = tr.max_nodes;
    const int WN = (N + 63) / 64;
    unsigned *ticket = reinterpret_cast<unsigned *>(ws);
    uint64_t *states = ws + 1;
    WarpSlab<NPL> &sm = slab[warp];
    constexpr int W = Shape<NPL>::W;
    while (true) {
        const int tile = next_tile(ticket, &s_tile);
        if (tile >= ntiles) break;
        const int b = tile * kWarps + warp;
        TreeState<NPL> t;
        int k = 0;
        if (b < tr.batch) {
            tree_load_validate<NPL>(t, tr, tr.parent, tr.q, tr.n_nodes, b, N);
            float c[NPL];
            if (!(t.status & EVICT_TREE_BAD_SIZE)) tree_load_cost<NPL>(c, t, cost + (size_t)b * cost_stride);
            int32_t *orow = out.order ? out.order + (size_t)b * N : nullptr;
            float *prow = out.prefix_sums ? out.prefix_sums + (size_t)b * N : nullptr;
            if (!t.status) {
                tree_levels<NPL, true>(t, sm);
                tree_rank_argmax<NPL>(t, sm, c, N, orow, prow);
                k = t.kstar;
            } else {
                t.kstar = 0; t.ehat = 0.f; t.util = 0.f;
#pragma unroll
                for (int w = 0; w < W; w++) t.keep[w] = 0ull;
                if (orow)
                    for (int p = lane; p < N; p += 32) { orow[p] = -1; prow[p] = 0.f; }
            }
            if (lane == 0) {
                if (out.k_star) out.k_star[b] = t.kstar;
                if (out.e_hat) out.e_hat[b] = t.ehat;
                if (out.utility) out.utility[b] = t.util;
            }
            if (out.keep_bits && lane < WN) out.keep_bits[(size_t)b * WN + lane] = t.keep[lane < W ? lane : 0];
        }
        if (lane == 0) s_cnt[warp] = k;
        tile_scan(tile, states, s_cnt, s_off);
        if (b < tr.batch) {
            const int off = s_off[warp];
            if (lane == 0 && out.verify_offsets) {
                out.verify_offsets[b] = off;
                if (b == tr.batch - 1) out.verify_offsets[tr.batch] = off + k;
            }
            if (k > 0)
                tree_build_emit<NPL>(t, sm, k, b, N, off,
                                     out.pos_offset ? __ldg(out.pos_offset + b) : 0, out.kept_index,
                                     out.retrieve_index, out.positions, out.next_token,
                                     out.next_sibling, out.tree_mask);
            __syncwarp();
            uint32_t st = t.status;
            if (out.union_count)
                tree_union<NPL, IDF, KT, EW, CL>(st, sm, k, b, N, rt.num_layers, rt.top_k,
                                                 rt.num_experts, rt.id_format, rt.ids, out.union_count,
                                                 out.union_total, out.union_bits, out.expert_hist);
            if (out.status && lane == 0) out.status[b] = st;
        }
    }
}

// ------------------------------------------------------------ launchers
int dev_sms();  // evict_api.cu

inline evict_status_t launched() { return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA; }

template <typename K>
inline int persistent_blocks(K kernel, int ntiles)
{
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kWarps * 32, 0);
    if (per_sm < 1) per_sm = 1;
    long g = (long)dev_sms() * per_sm;
    return (int)(g < ntiles ? g : ntiles);
}

// dispatch over (IDF, KT, EW, CL); IDF 1 = u8 K=8, 4 = i32 K=8, 8 = masks,
// 0 = generic ids (any K ≤ 16, u8 or i32, scalar loads)
template <int NPL, template <int, int, int, int, int> class Launcher, typename... Args>
inline evict_status_t dispatch_union(const evict_routing_t *rt, Args... args)
{
    const int CL = rt->num_layers <= 64 ? 2 : 4;
    const int EW = rt->num_experts <= 128 ? 2 : 4;
#define EVICT_CL(IDF, EWV)                                                    \
    if (CL == 2) return Launcher<NPL, IDF, IDF == 1 || IDF == 4 ? 8 : 0, EWV, 2>::run(args...); \
    return Launcher<NPL, IDF, IDF == 1 || IDF == 4 ? 8 : 0, EWV, 4>::run(args...);
#define EVICT_EW(IDF)                     \
    if (EW == 2) { EVICT_CL(IDF, 2) }     \
    else { EVICT_CL(IDF, 4) }
    if (rt->id_format == EVICT_ID_MASK) { EVICT_EW(8) }
    if (rt->top_k == 8 && rt->id_format == EVICT_ID_U8) { EVICT_EW(1) }
    if (rt->top_k == 8 && rt->id_format == EVICT_ID_I32) { EVICT_EW(4) }
    EVICT_EW(0)
#undef EVICT_EW
#undef EVICT_CL
}

template <int NPL, int IDF, int KT, int EW, int CL>
struct UnionLauncher {
    static evict_status_t run(const evict_trees_t *tr, const uint64_t *keep, const evict_routing_t *rt,
                              int32_t *uc, int32_t *ut, uint64_t *ub, int64_t *eh, uint32_t *st,
                              cudaStream_t s)
    {
        const int blocks = (tr->batch + kWarps - 1) / kWarps;
        k_union<NPL, IDF, KT, EW, CL><<<blocks, kWarps * 32, 0, s>>>(*tr, keep, *rt, uc, ut, ub, eh, st);
        return launched();
    }
};

template <int NPL, int IDF, int KT, int EW, int CL>
struct FusedLauncher {
    static evict_status_t run(const evict_trees_t *tr, const float *cost, int cs,
                              const evict_routing_t *rt, const evict_fused_out_t *o, uint64_t *ws,
                              int ntiles, cudaStream_t s)
    {
        auto kern = k_fused<NPL, IDF, KT, EW, CL>;
        const int blocks = persistent_blocks(kern, ntiles);
        kern<<<blocks, kWarps * 32, 0, s>>>(*tr, cost, cs, *rt, *o, ws, ntiles);
        return launched();
    }
};

template <int NPL>
evict_status_t launch_select(const evict_trees_t *tr, const float *cost, int cs, int32_t *k_star,
                             float *e_hat, float *utility, uint64_t *keep_bits, int32_t *order,
                             float *prefix_sums, uint32_t *status, cudaStream_t s)
{
    const int blocks = (tr->batch + kWarps - 1) / kWarps;
    k_select<NPL><<<blocks, kWarps * 32, 0, s>>>(*tr, cost, cs, k_star, e_hat, utility, keep_bits,
                                                   order, prefix_sums, status);
    return launched();
}

template <int NPL>
evict_status_t launch_build(const evict_trees_t *tr, const uint64_t *keep_bits,
                            const int32_t *pos_offset, int32_t *verify_offsets, int32_t *kept_index,
                            int32_t *retrieve_index, int32_t *positions, int32_t *next_token,
                            int32_t *next_sibling, uint64_t *tree_mask, uint32_t *status,
                            uint64_t *ws, int ntiles, cudaStream_t s)
{
    auto kern = k_build<NPL>;
    kern<<<persistent_blocks(kern, ntiles), kWarps * 32, 0, s>>>(
        *tr, keep_bits, pos_offset, verify_offsets, kept_index, retrieve_index, positions,
        next_token, next_sibling, tree_mask, status, ws, ntiles);
    return launched();
}

template <int NPL>
evict_status_t launch_union(const evict_trees_t *tr, const uint64_t *keep, const evict_routing_t *rt,
                            int32_t *uc, int32_t *ut, uint64_t *ub, int64_t *eh, uint32_t *st,
                            cudaStream_t s)
{
    return dispatch_union<NPL, UnionLauncher>(rt, tr, keep, rt, uc, ut, ub, eh, st, s);
}

template <int NPL>
evict_status_t launch_fused(const evict_trees_t *tr, const float *cost, int cs,
                            const evict_routing_t *rt, const evict_fused_out_t *o, uint64_t *ws,
                            int ntiles, cudaStream_t s)
{
    return dispatch_union<NPL, FusedLauncher>(rt, tr, cost, cs, rt, o, ws, ntiles, s);
}

}  // namespace evict
