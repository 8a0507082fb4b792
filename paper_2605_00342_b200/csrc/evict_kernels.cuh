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

// The tile state word carries its own payload (flag + count in one aligned
// 64-bit word), so relaxed GPU-scope accesses suffice: no acquire (which would
// invalidate L1) and no release fence.
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t *p)
{
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint64_t *p, uint64_t v)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled look-back over CTA tiles (8 trees each), split in two halves so the
// wait for predecessors overlaps useful work:
//  tile_publish  — after every warp stored its tree's row count in s_cnt[warp]:
//                  warp 0 scans the 8 counts and publishes the tile aggregate
//                  (tile 0 publishes its inclusive prefix directly).
//  tile_lookback — later: warp 0 walks back over 32 predecessor states per
//                  L2 round trip; the nearest inclusive prefix ends the walk,
//                  unpublished predecessors in front of it are re-polled.
// s_off[warp] = packed-row offset of the warp's tree after tile_lookback.
__device__ __forceinline__ void tile_publish(int tile, uint64_t *states, const int *s_cnt, int *s_off,
                                             int *s_agg)
{
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) {
        const int lane = lane_id();
        const int c = lane < kWarps ? s_cnt[lane] : 0;
        int inc = c;
#pragma unroll
        for (int o = 1; o < kWarps; o <<= 1) {
            int v = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += v;
        }
        const int agg = __shfl_sync(kFull, inc, kWarps - 1);
        if (lane < kWarps) s_off[lane] = inc - c;
        if (lane == 0) {
            *s_agg = agg;
            st_release(states + tile, (tile == 0 ? kInc : kAgg) | (uint64_t)agg);
        }
    }
}

__device__ __forceinline__ void tile_lookback(int tile, uint64_t *states, int *s_off, const int *s_agg)
{
    __syncthreads();
    if ((threadIdx.x >> 5) == 0 && tile > 0) {
        const int lane = lane_id();
        unsigned prefix = 0;
        int end = tile;
        while (true) {
            const int j = end - 1 - lane;          // lane 0 = nearest predecessor
            const uint64_t s = j >= 0 ? ld_acquire(states + j) : kInc;
            const unsigned flag = (unsigned)(s >> 62);
            const unsigned inc_mask = __ballot_sync(kFull, flag == 2);
            const unsigned zero_mask = __ballot_sync(kFull, flag == 0);
            const int first_inc = inc_mask ? __ffs(inc_mask) - 1 : 32;
            const unsigned before = first_inc == 32 ? kFull : ((1u << first_inc) - 1u);
            if (zero_mask & before) continue;      // a predecessor is not published yet
            const unsigned v = lane <= first_inc ? (unsigned)(s & kValMask) : 0u;
            prefix += __reduce_add_sync(kFull, v);
            if (first_inc < 32) break;
            end -= 32;
        }
        if (lane == 0) st_release(states + tile, kInc | (uint64_t)(prefix + (unsigned)*s_agg));
        if (lane < kWarps) s_off[lane] += (int)prefix;
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
    __shared__ int s_cnt[kWarps], s_off[kWarps], s_tile, s_agg;
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
        tile_publish(tile, states, s_cnt, s_off, &s_agg);
        tile_lookback(tile, states, s_off, &s_agg);
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

// Flag bytes per warp for the shared-memory union (IDF 1/4): L × Epad.
__host__ __device__ inline int union_epad(int E) { return E <= 128 ? 128 : 256; }

template <int NPL, int IDF, int KT, int EW, int CL>
__global__ void __launch_bounds__(kWarps * 32) k_union(evict_trees_t tr, const uint64_t *keep_bits,
                                                       evict_routing_t rt, int32_t *union_count,
                                                       int32_t *union_total, uint64_t *union_bits,
                                                       int64_t *expert_hist, uint32_t *status)
{
    extern __shared__ __align__(16) uint8_t dsm[];
    __shared__ WarpSlab<NPL> slab[kWarps];
    constexpr int W = Shape<NPL>::W;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int Epad = union_epad(rt.num_experts);
    uint8_t *flags = dsm + (size_t)warp * rt.num_layers * Epad;
    if constexpr (IDF == 1 || IDF == 4) {
        uint4 *f4 = reinterpret_cast<uint4 *>(flags);
        for (int i = lane; i < rt.num_layers * Epad / 16; i += 32) f4[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
    }
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
                                     rt.id_format, rt.ids, flags, Epad, union_count, union_total,
                                     union_bits, expert_hist);
    if (status && lane == 0) status[b] = st;
}

// ------------------------------------------------------------ fused
// One CTA tile = 32 consecutive trees, 4 per warp (warp w owns trees w, w+8,
// w+16, w+24 of the tile), processed in three phases:
//   A  per tree: A1–A5 select (outputs written), A7 union (outputs written),
//      and an emit record (parent, depth, keep) parked in shared memory;
//   B  one barrier: warp 0 scans the 32 row counts, publishes the tile
//      aggregate, looks back for the tile prefix and fetches the next ticket;
//   C  per tree: A6 build from the record at the packed offset.
// Two barriers per 32 trees; union-time variance averages over 4 trees/warp.
constexpr int kTreesPerWarp = 4;
constexpr int kTile = kWarps * kTreesPerWarp;

template <int NPL>
struct EmitRec {
    static constexpr int NMAX = Shape<NPL>::NMAX;
    static constexpr int W = Shape<NPL>::W;
    uint64_t keep[W];
    int8_t par[NMAX];
    uint8_t dep[NMAX];
    int n, k;
    uint32_t status;
};

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }
template <int NPL>
__host__ __device__ constexpr size_t fused_rec_offset() { return align16(sizeof(WarpSlab<NPL>) * kWarps); }
template <int NPL>
__host__ __device__ constexpr size_t fused_flags_offset()
{
    return align16(fused_rec_offset<NPL>() + sizeof(EmitRec<NPL>) * kTile);
}

template <int NPL, int IDF, int KT, int EW, int CL>
__global__ void __launch_bounds__(kWarps * 32, 2) k_fused(evict_trees_t tr, const float *cost,
                                                       int cost_stride, evict_routing_t rt,
                                                       evict_fused_out_t out, uint64_t *ws,
                                                       int ntiles)
{
    extern __shared__ __align__(16) uint8_t dsm[];
    // dynamic shared memory: [warp slabs][emit records][union flags]
    WarpSlab<NPL> *slab = reinterpret_cast<WarpSlab<NPL> *>(dsm);
    EmitRec<NPL> *rec = reinterpret_cast<EmitRec<NPL> *>(dsm + fused_rec_offset<NPL>());
    __shared__ int s_cnt[kTile], s_off[kTile], s_tile;
    constexpr int W = Shape<NPL>::W;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int N = tr.max_nodes;
    const int WN = (N + 63) / 64;
    const int base = lane * NPL;
    unsigned *ticket = reinterpret_cast<unsigned *>(ws);
    uint64_t *states = ws + 1;
    WarpSlab<NPL> &sm = slab[warp];
    const int Epad = union_epad(rt.num_experts);
    uint8_t *flags = dsm + fused_flags_offset<NPL>() + (size_t)warp * rt.num_layers * Epad;
    if constexpr (IDF == 1 || IDF == 4) {
        if (out.union_count) {
            uint4 *f4 = reinterpret_cast<uint4 *>(flags);
            for (int i = lane; i < rt.num_layers * Epad / 16; i += 32) f4[i] = make_uint4(0u, 0u, 0u, 0u);
            __syncwarp();
        }
    }
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    int tile = s_tile;
    while (tile < ntiles) {
        // ---------------- phase A1: select per tree (+ emit record)
#pragma unroll 1
        for (int it = 0; it < kTreesPerWarp; it++) {
            const int slot = warp + kWarps * it;
            const int b = tile * kTile + slot;
            int k = 0;
            if (b < tr.batch) {
                TreeState<NPL> t;
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
                EmitRec<NPL> &er = rec[slot];
#pragma unroll
                for (int r = 0; r < NPL; r++) {
                    er.par[base + r] = (int8_t)t.par[r];
                    er.dep[base + r] = (uint8_t)t.dep[r];
                }
                if (lane < W) er.keep[lane] = t.keep[lane];
                if (lane == 0) { er.n = t.n; er.k = k; er.status = t.status; }
            }
            if (lane == 0) s_cnt[slot] = k;
        }
        // ---------------- tile aggregate published as soon as every tree is selected
        __syncthreads();
        int incl = 0;
        if (warp == 0) {
            const int c = s_cnt[lane];             // kTile == 32 == warp size
            incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int v = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += v;
            }
            s_off[lane] = incl - c;
            if (lane == 31) st_release(states + tile, (tile == 0 ? kInc : kAgg) | (uint64_t)incl);
        }
        // ---------------- phase A2: expert union per tree (the look-back latency hides here)
        if (out.union_count) {
#pragma unroll 1
            for (int it = 0; it < kTreesPerWarp; it++) {
                const int slot = warp + kWarps * it;
                const int b = tile * kTile + slot;
                if (b >= tr.batch) break;
                EmitRec<NPL> &er = rec[slot];
                const int k = er.k;
                uint32_t st = er.status;
                TreeState<NPL> t;
                t.n = er.n;
#pragma unroll
                for (int w = 0; w < W; w++) t.keep[w] = er.keep[w];
                if (k > 0) tree_fill_klist<NPL>(t, sm);
                tree_union<NPL, IDF, KT, EW, CL>(st, sm, k, b, N, rt.num_layers, rt.top_k,
                                                 rt.num_experts, rt.id_format, rt.ids, flags, Epad,
                                                 out.union_count, out.union_total, out.union_bits,
                                                 out.expert_hist);
                if (lane == 0) er.status = st;
            }
        }
        // ---------------- look-back for the tile prefix + next ticket
        if (warp == 0) {
            const int agg = __shfl_sync(kFull, incl, 31);
            unsigned prefix = 0;
            if (tile > 0) {
                int end = tile;
                while (true) {
                    const int j = end - 1 - lane;
                    const uint64_t sv = j >= 0 ? ld_acquire(states + j) : kInc;
                    const unsigned flag = (unsigned)(sv >> 62);
                    const unsigned inc_mask = __ballot_sync(kFull, flag == 2);
                    const unsigned zero_mask = __ballot_sync(kFull, flag == 0);
                    const int first_inc = inc_mask ? __ffs(inc_mask) - 1 : 32;
                    const unsigned before = first_inc == 32 ? kFull : ((1u << first_inc) - 1u);
                    if (zero_mask & before) continue;
                    const unsigned v = lane <= first_inc ? (unsigned)(sv & kValMask) : 0u;
                    prefix += __reduce_add_sync(kFull, v);
                    if (first_inc < 32) break;
                    end -= 32;
                }
                if (lane == 0) st_release(states + tile, kInc | (uint64_t)(prefix + (unsigned)agg));
            }
            s_off[lane] += (int)prefix;
            if (lane == 0) s_tile = (int)atomicAdd(ticket, 1u);
        }
        __syncthreads();
        const int next = s_tile;
        // ---------------- phase C: verify-tree build per tree
#pragma unroll 1
        for (int it = 0; it < kTreesPerWarp; it++) {
            const int slot = warp + kWarps * it;
            const int b = tile * kTile + slot;
            if (b >= tr.batch) break;
            const EmitRec<NPL> &er = rec[slot];
            const int k = er.k;
            const int off = s_off[slot];
            if (lane == 0 && out.status) out.status[b] = er.status;
            if (lane == 0 && out.verify_offsets) {
                out.verify_offsets[b] = off;
                if (b == tr.batch - 1) out.verify_offsets[tr.batch] = off + k;
            }
            if (k > 0) {
                TreeState<NPL> t;
                t.n = er.n;
#pragma unroll
                for (int r = 0; r < NPL; r++) {
                    t.par[r] = er.par[base + r];
                    t.dep[r] = er.dep[base + r];
                }
#pragma unroll
                for (int w = 0; w < W; w++) t.keep[w] = er.keep[w];
                tree_build_emit<NPL>(t, sm, k, b, N, off,
                                     out.pos_offset ? __ldg(out.pos_offset + b) : 0, out.kept_index,
                                     out.retrieve_index, out.positions, out.next_token,
                                     out.next_sibling, out.tree_mask);
            }
        }
        tile = next;
    }
}

// ------------------------------------------------------------ launchers
int dev_sms();  // evict_api.cu

inline evict_status_t launched() { return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA; }

template <typename K>
inline int persistent_blocks(K kernel, int ntiles, size_t dyn = 0)
{
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kWarps * 32, dyn);
    if (per_sm < 1) per_sm = 1;
    long g = (long)dev_sms() * per_sm;
    return (int)(g < ntiles ? g : ntiles);
}

// dispatch over (IDF, KT, EW, CL); IDF 1 = u8 K=8, 4 = i32 K=8, 8 = masks,
// 0 = generic ids (any K ≤ 16, u8 or i32, scalar loads)
template <int NPL, template <int, int, int, int, int> class Launcher, typename... Args>
inline evict_status_t dispatch_union(const evict_routing_t *rt, Args... args)
{
    // Fast slot layout (evict_tree.cuh tree_union_fast) for top-8 ids and 1/2/4-word masks:
    // L·P slots in R register rounds (R·32 ≥ L·P).  Otherwise the lane-per-layer layout
    // with R/2 rounds (R/2·32 ≥ L).
    const int L = rt->num_layers;
    const int EWr = (rt->num_experts + 63) / 64;
    const int EW = rt->num_experts <= 128 ? 2 : 4;
    int IDF = 0;
    if (rt->id_format == EVICT_ID_MASK) IDF = (EWr == 3) ? 9 : 8;
    else if (rt->top_k == 8) IDF = rt->id_format;
    const int P = IDF == 8 ? EWr : 2;
    int R = (IDF == 1 || IDF == 4 || IDF == 8) ? (L * P <= 96 ? 3 : (L * P <= 128 ? 4 : 8))
                                               : (L <= 64 ? 4 : 8);
    if ((IDF == 1 || IDF == 4 || IDF == 8) && L * P > 256) {
        if (IDF == 8) IDF = 9; else IDF = 0;
        R = L <= 64 ? 4 : 8;
    }
#define EVICT_R(IDFV, EWV)                                                            \
    if (R == 3) return Launcher<NPL, IDFV, (IDFV == 1 || IDFV == 4) ? 8 : 0, EWV, 3>::run(args...); \
    if (R == 4) return Launcher<NPL, IDFV, (IDFV == 1 || IDFV == 4) ? 8 : 0, EWV, 4>::run(args...); \
    return Launcher<NPL, IDFV, (IDFV == 1 || IDFV == 4) ? 8 : 0, EWV, 8>::run(args...);
#define EVICT_EW(IDFV)                  \
    if (EW == 2) { EVICT_R(IDFV, 2) }   \
    else { EVICT_R(IDFV, 4) }
    switch (IDF) {
    case 1: EVICT_EW(1)
    case 4: EVICT_EW(4)
    case 8: EVICT_EW(8)
    case 9: EVICT_EW(9)
    default: EVICT_EW(0)
    }
#undef EVICT_EW
#undef EVICT_R
}

template <int NPL, int IDF, int KT, int EW, int CL>
struct UnionLauncher {
    static evict_status_t run(const evict_trees_t *tr, const uint64_t *keep, const evict_routing_t *rt,
                              int32_t *uc, int32_t *ut, uint64_t *ub, int64_t *eh, uint32_t *st,
                              cudaStream_t s)
    {
        const int blocks = (tr->batch + kWarps - 1) / kWarps;
        const size_t dyn = (IDF == 1 || IDF == 4) ? (size_t)kWarps * rt->num_layers * union_epad(rt->num_experts) : 0;
        auto kern = k_union<NPL, IDF, KT, EW, CL>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        kern<<<blocks, kWarps * 32, dyn, s>>>(*tr, keep, *rt, uc, ut, ub, eh, st);
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
        const size_t dyn = fused_flags_offset<NPL>() +
                           ((IDF == 1 || IDF == 4) && o->union_count
                                ? (size_t)kWarps * rt->num_layers * union_epad(rt->num_experts) : 0);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        const int blocks = persistent_blocks(kern, ntiles, dyn);
        kern<<<blocks, kWarps * 32, dyn, s>>>(*tr, cost, cs, *rt, *o, ws, ntiles);
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
