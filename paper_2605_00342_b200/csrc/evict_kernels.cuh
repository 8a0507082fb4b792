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
#include "evict_group.cuh"
#include "evict_launch.h"

#ifndef EVICT_UCOLS_UB
#define EVICT_UCOLS_UB 4   // kept rows per load batch of tree_union_cols (8 measured slower)
#endif

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
                                                        int cost_stride, evict_policy_t pol, int32_t *k_star,
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
        tree_rank_argmax<NPL>(t, sm, c, N, orow, prow, pol);
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
__host__ __device__ inline int union_epad_u(int E) { return E <= 128 ? 128 : 256; }

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
    const int Epad = union_epad_u(rt.num_experts);
    const int fbytes = union_flag_bytes(rt.num_layers, rt.num_experts);
    uint8_t *flags = dsm + (size_t)warp * fbytes;
    if constexpr (IDF == 1 || IDF == 4) {
        uint4 *f4 = reinterpret_cast<uint4 *>(flags);
        for (int i = lane; i < fbytes / 16; i += 32) f4[i] = make_uint4(0u, 0u, 0u, 0u);
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
    tree_union<NPL, IDF, KT, EW, CL>(st, sm.klist, k, b, N, rt.num_layers, rt.top_k, rt.num_experts,
                                     rt.id_format, rt.ids, flags, Epad, union_count, union_total,
                                     union_bits, expert_hist);
    if (status && lane == 0) status[b] = st;
}

// ------------------------------------------------------------ fused
// Tiles are per WARP: a warp takes a ticket for kWT = 4 consecutive trees and
// carries them through every phase with no CTA-wide barrier.  A1–A5 and A6 run
// sub-warp-per-tree (evict_group.cuh: G lanes per tree); A7 runs one warp per
// tree.  Phases per warp tile:
//   A1  select the 4 trees (outputs written), park an emit record (parent,
//       keep, kept list) in shared memory;
//   --  publish the tile's row count (decoupled look-back state) and take the
//       next ticket early;
//   A2  expert union, one tree at a time;
//   --  look back for the tile prefix (its wait overlapped A2);
//   C   verify-tree emit (A6) at the packed offsets.
// Predecessor tiles always belong to warps that took their ticket earlier and
// are resident, so the look-back cannot deadlock.
#ifdef EVICT_PHASE_TIMING
// profiling variant only: per-phase SM cycles of k_fused summed over warps (lane 0)
static __device__ unsigned long long g_phase_cycles[8];   // per translation unit
#define EVICT_PHASE(i)                                                                     \
    do {                                                                                   \
        const long long now_ = clock64();                                                  \
        if (lane == 0) atomicAdd(&g_phase_cycles[i], (unsigned long long)(now_ - ph_t));   \
        ph_t = now_;                                                                       \
    } while (0)
#else
#define EVICT_PHASE(i) do {} while (0)
#endif
constexpr int kWT = 4;                 // trees per warp tile (throughput batches)
constexpr int kSmallBatch = 2048;      // up to here (serving batches, LEAN path): one tree per warp
                                       // tile, so batch 64 spreads over 64 warps instead of 16

// Warp-level decoupled look-back for tile `tile` (lane j reads the state of tile end − 1 − j per
// round).  WAIT: re-poll unpublished predecessors until the walk ends; otherwise give up (return
// false, prefix untouched) at the first unpublished predecessor or after kEarlyRounds rounds.
// On success the tile's inclusive prefix (prefix + agg) is published and prefix holds the sum of
// every predecessor's count.
constexpr int kEarlyRounds = 4;
template <bool WAIT>
__device__ __forceinline__ bool lookback_walk(int tile, uint64_t *states, int agg, unsigned &prefix, int lane)
{
    unsigned acc = 0;
    int end = tile, rounds = 0;
    while (true) {
        const int j = end - 1 - lane;
        const uint64_t sv = j >= 0 ? ld_acquire(states + j) : kInc;
        const unsigned flag = (unsigned)(sv >> 62);
        const unsigned inc_mask = __ballot_sync(kFull, flag == 2);
        const unsigned zero_mask = __ballot_sync(kFull, flag == 0);
        const int first_inc = inc_mask ? __ffs(inc_mask) - 1 : 32;
        const unsigned before = first_inc == 32 ? kFull : ((1u << first_inc) - 1u);
        if (zero_mask & before) {
            if (!WAIT) return false;
            continue;
        }
        const unsigned v = lane <= first_inc ? (unsigned)(sv & kValMask) : 0u;
        acc += __reduce_add_sync(kFull, v);
        if (first_inc < 32) break;
        end -= 32;
        if (!WAIT && ++rounds >= kEarlyRounds) return false;
    }
    if (lane == 0) st_release(states + tile, kInc | (uint64_t)(acc + (unsigned)agg));
    prefix = acc;
    return true;
}

template <int G>
struct EmitRec {
    static constexpr int NMAX = grp::GShape<G>::NMAX;
    static constexpr int W = grp::GShape<G>::W;
    uint64_t keep[W];
    alignas(8) int8_t par[NMAX];
    alignas(8) uint8_t klist[NMAX];   // kept nodes, ascending (slot order), built once in A1
    alignas(8) uint8_t slot[NMAX];    // node → slot for kept nodes (W = 1 only: the emit's ancestor walk)
    int n, k;
    uint32_t status;
    float ehat, util;                 // for the folded A9 statistics
};

// Folded A9 statistics (LEAN, E = 128, L ≤ 64): per-CTA accumulators at the end of the dynamic
// shared memory, flushed to the global stats vector (evict_batch_stats layout) when the CTA ends.
struct FusedStats {
    unsigned sc[kWarps][4];     // per warp (no contention): trees, Σk*, Σn, errored trees
    double d[kWarps][2];        // per warp: Σe_hat, Σutility (status 0)
    unsigned hist[129];         // k* histogram, bin 0 = errored trees
    unsigned lay[64];           // Σ union_count per layer (status 0)
};
constexpr size_t kStatsSmem = (sizeof(FusedStats) + 15) & ~(size_t)15;

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// Per-warp scratch: union flags (A2), or sweep state (A1), or emit rows/child (C).
template <int G>
__host__ __device__ constexpr size_t fused_scratch_fixed()
{
    // sweeps: TPW × (NMAX + 8) floats; emit: TPW × NMAX × W child words (+ slack)
    return align16(grp::GShape<G>::TPW * grp::GShape<G>::NMAX *
                   (sizeof(int2) > 2 * 8 * grp::GShape<G>::W ? sizeof(int2) : 2 * 8 * grp::GShape<G>::W));
}
// bytes of the scratch the sweeps (padded score arrays) and emit (child masks) write
template <int G>
__host__ __device__ constexpr size_t fused_scratch_dirty()
{
    constexpr size_t sw = (size_t)grp::GShape<G>::TPW * (grp::GShape<G>::NMAX + 8) * 4;
    constexpr size_t ch = (size_t)grp::GShape<G>::TPW * grp::GShape<G>::NMAX * grp::GShape<G>::W * 8;
    return align16(sw > ch ? sw : ch);
}
__host__ __device__ inline int union_epad(int E) { return E <= 128 ? 128 : 256; }
template <int G>
__host__ __device__ inline size_t fused_scratch_bytes(int L, int E, bool flags)
{
    const size_t f = flags ? (size_t)union_flag_bytes(L, E) : 0;
    const size_t x = fused_scratch_fixed<G>();
    return align16(f > x ? f : x);
}
template <int G, int WT = kWT, int NW = kWarps>
__host__ __device__ inline size_t fused_smem_bytes(int L, int E, bool flags, bool ranks = true)
{
    return (size_t)NW * fused_scratch_bytes<G>(L, E, flags)              // scratch
           + align16(sizeof(EmitRec<G>) * NW * WT)                       // records
           + (ranks ? align16((size_t)NW * grp::GShape<G>::TPW * grp::GShape<G>::NMAX) : 0)  // ranks (order row)
           + kStatsSmem;                                                  // folded A9 statistics
}

// LEAN: the serving / bench configuration (u8 top-8 ids, E = 128 or 128 < E ≤ 256, no order row, no
// union bit rows, no histogram) compiled without the other paths — with warps in
// different phases the full kernel's code footprint thrashes the instruction cache.
// PRE (two-kernel throughput path, LEAN only): k_select_g already wrote k*, e_hat, utility, keep
// bits, select status and the packed offsets (scanned in the same launch); this kernel rebuilds
// each tree's emit record from them (parent row, keep bits) and runs A6 + A7 (+ A9) only.
// NW: warps per CTA — 8, or 4 for the PRE union/emit kernel, whose 4 × 8 KB flag blocks then sit in
// the first 32 KB of the dynamic shared memory: warp w's byte-store address is the CTA-uniform block
// base (an STS uniform-register operand) + one PRMT result (tree_union_cols)
template <int NPL, int IDF, int KT, int EW, int CL, bool LEAN = false, int WT = kWT, bool PRE = false, int NW = kWarps>
__global__ void __launch_bounds__(NW * 32, NW == 4 ? 6 : 3) k_fused(evict_trees_t tr, const float *cost,
                                                       int cost_stride, evict_policy_t pol, evict_routing_t rt,
                                                       evict_fused_out_t out, uint64_t *ws,
                                                       int ntiles)
{
    static_assert(!LEAN || IDF == 1, "LEAN is the u8 top-8 configuration");
    constexpr int G = NPL == 2 ? 8 : 16;
    constexpr int TPW = grp::GShape<G>::TPW;
    constexpr int NMAX = grp::GShape<G>::NMAX;
    constexpr int W = grp::GShape<G>::W;
    constexpr int PASSES = WT > TPW ? WT / TPW : 1;   // 1 (G=8, or WT = 1) or 2 (G=16, WT = 4)
    constexpr bool FLAGS = IDF == 1 || IDF == 4;
    extern __shared__ __align__(16) uint8_t dsm[];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int gi = grp::gidx<G>(), g = grp::gl<G>();
    const int N = tr.max_nodes;
    const int WN = (N + 63) / 64;
    const int L = rt.num_layers, E = rt.num_experts;
    const bool do_union = out.union_count != nullptr;
    const size_t scratch = fused_scratch_bytes<G>(L, E, FLAGS && do_union);
    // NW == 4: the 4 scratch (= flag) blocks are static shared memory, so their address is a link-time
    // constant the compiler folds into every byte store's immediate; the dynamic block holds the rest
    uint8_t *scr_base = dsm;
    uint32_t sfold_static = 0u;
    EmitRec<G> *rec_base = reinterpret_cast<EmitRec<G> *>(dsm + (size_t)NW * scratch);
    uint8_t *ranks = reinterpret_cast<uint8_t *>(dsm + (size_t)NW * scratch) + align16(sizeof(EmitRec<G>) * NW * WT);
    FusedStats *fs = reinterpret_cast<FusedStats *>(ranks + (LEAN ? 0 : align16((size_t)NW * TPW * NMAX)));
    if constexpr (NW == 4) {
        // the 4 × 8 KB flag blocks are the kernel's only static shared memory (offset 0 of the
        // CTA's window: the base add vanishes from every byte store); records + stats dynamic
        __shared__ __align__(16) uint8_t s_scr4[4 * 8192];
        scr_base = s_scr4;
        sfold_static = (uint32_t)__cvta_generic_to_shared(s_scr4);   // the symbol itself: a constant
        rec_base = reinterpret_cast<EmitRec<G> *>(dsm);
        fs = reinterpret_cast<FusedStats *>(dsm + align16(sizeof(EmitRec<G>) * NW * WT));
    }
    uint8_t *wscr = scr_base + (size_t)warp * scratch;
    EmitRec<G> *rec = rec_base + warp * WT;
    uint8_t *rk = ranks + ((size_t)warp * TPW + gi) * NMAX;
    // A9 folded into the launch: the single-pass E = 128 LEAN union (the caller passes out.stats
    // only for that configuration; it runs evict_batch_stats after the launch otherwise)
    constexpr bool kFold = LEAN && EW == 2 && CL <= 4;
    const bool fstats = kFold && out.stats != nullptr;
    uint32_t lsum[4] = {0u, 0u, 0u, 0u};   // folded A9: this lane's output layers ulane.l0 + m
    unsigned rs_tr = 0u, rs_k = 0u, rs_n = 0u, rs_err = 0u;   // folded A9 scalars (lane 0, registers)
    double rs_e = 0.0, rs_u = 0.0;
    bool emit_dirty = false;   // PRE: the last tile's emit wrote child masks into the flag prefix
    const UColsLane ulane = ucols_lane<CL == 4 ? 2 : 1>(lane, rt.num_layers);
    // NW == 4 (the PRE launch: union_count given, E = 128, so every scratch block is the 8 KB flag
    // block): byte stores at the CTA-uniform base sfold + a PRMT result whose row byte carries 32·warp
    // (hfold); otherwise at this warp's block (sfold = its address, hfold = 0)
    constexpr bool fold = NW == 4;
    const uint32_t sfold = fold ? sfold_static : (uint32_t)__cvta_generic_to_shared(wscr);
    const uint32_t hfold = fold ? (32u * (uint32_t)warp) * 0x01010101u : 0u;
    if constexpr (kFold) {
        if (fstats) {
            uint32_t *z = reinterpret_cast<uint32_t *>(fs);
            for (int i = threadIdx.x; i < (int)(sizeof(FusedStats) / 4); i += blockDim.x) z[i] = 0u;
            __syncthreads();
        }
    }
    const int Epad = union_epad(E);
    unsigned *ticket = reinterpret_cast<unsigned *>(ws);
    uint64_t *states = ws + 1;
    int tile = 0;
    if (lane == 0) tile = (int)atomicAdd(ticket, 1u);
    tile = __shfl_sync(kFull, tile, 0);
    bool first = true;
    int epoch = 0;   // LEAN union marker window (tree_union_flags64)
#ifdef EVICT_PHASE_TIMING
    long long ph_t = clock64();
#endif
    while (tile < ntiles) {
        const int b0 = tile * WT;
        // ---------------- A1: select, sub-warp per tree
#pragma unroll 1
        for (int pass = 0; pass < PASSES; pass++) {
            const int slot = pass * TPW + gi;
            const int b = b0 + slot;
            const bool active = slot < WT && b < tr.batch;
            grp::GTree<G> t;
            if constexpr (PRE) {
                // the select's outputs (this stream, earlier launch)
                grp::g_load_par<G>(t, tr.parent, tr.n_nodes, b, N, active);
#pragma unroll
                for (int w = 0; w < W; w++) t.keep[w] = (active && w < WN) ? out.keep_bits[(size_t)b * WN + w] : 0ull;
                t.kstar = active ? out.k_star[b] : 0;
                t.status = active ? out.status[b] : 0u;
                t.ehat = active ? out.e_hat[b] : 0.f;
                t.util = active ? out.utility[b] : 0.f;
            } else {
            float4 cr[2];
            grp::g_fetch_cost<G>(cr, cost + (size_t)(active ? b : 0) * cost_stride, N, active);
            grp::g_load<G>(t, tr.parent, tr.q, tr.n_nodes, b, N, active);
            float c[grp::NP];
            grp::g_apply_cost<G>(c, t, cr);
            // per-tree score arrays 8 floats apart in bank space: the 4 trees' reads of
            // their roots (and other equal node ids) land on different banks
            float *sd = reinterpret_cast<float *>(wscr) + gi * (NMAX + 8);
            grp::g_levels<G, true>(t, sd);
            int32_t *orow = (active && out.order) ? out.order + (size_t)b * N : nullptr;
            float *prow = (active && out.prefix_sums) ? out.prefix_sums + (size_t)b * N : nullptr;
            if (!LEAN && out.order) grp::g_rank_argmax<G>(t, rk, c, N, orow, prow, pol);   // kernel-uniform
            else grp::g_select_values<G>(t, c, N, prow, pol);
            }
            const int k = t.kstar;
            EmitRec<G> &er = rec[slot < WT ? slot : 0];
            if (active) {
                if (!PRE && g == 0) {
                    if (out.k_star) out.k_star[b] = t.kstar;
                    if (out.e_hat) out.e_hat[b] = t.ehat;
                    if (out.utility) out.utility[b] = t.util;
                }
                if (!PRE && out.keep_bits && g < WN) out.keep_bits[(size_t)b * WN + g] = t.keep[g < W ? g : 0];
                const int base = g * grp::NP;
                uint32_t pw[2] = {0u, 0u};
#pragma unroll
                for (int r = 0; r < grp::NP; r++) pw[r >> 2] |= (uint32_t)(t.par[r] & 0xff) << (8 * (r & 3));
                *reinterpret_cast<uint2 *>(&er.par[base]) = make_uint2(pw[0], pw[1]);
                if (g < W) er.keep[g] = t.keep[g];
                if constexpr (W == 1) {
                    // this lane's 8 keep bits and the slot of its first node: 32-bit work per node
                    const uint32_t kb = (uint32_t)(t.keep[0] >> base) & 0xffu & ((t.n - base) >= grp::NP ? 0xffu : ((1u << (t.n - base > 0 ? t.n - base : 0)) - 1u));
                    const int sb = __popcll(t.keep[0] & ((1ull << base) - 1ull));
#pragma unroll
                    for (int r = 0; r < grp::NP; r++)
                        if ((kb >> r) & 1u) {
                            const int sl = sb + __popc(kb & ((1u << r) - 1u));
                            er.klist[sl] = (uint8_t)(base + r);
                            er.slot[base + r] = (uint8_t)sl;
                        }
                } else {
#pragma unroll
                    for (int r = 0; r < grp::NP; r++) {
                        const int i = base + r;
                        if (i < t.n && grp::bit_w<W>(t.keep, i)) er.klist[grp::popc_below_w<W>(t.keep, i)] = (uint8_t)i;
                    }
                }
                if (g == 0) { er.n = t.n; er.k = k; er.status = t.status; er.ehat = t.ehat; er.util = t.util; }
            } else if (g == 0 && slot < WT) {
                er.k = 0;
            }
            __syncwarp();
        }
        EVICT_PHASE(0);
        // ---------------- tile aggregate (lanes 0..3 = the tile's trees) + next ticket
        const int cnt = lane < WT ? rec[lane].k : 0;
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < WT; o <<= 1) {
            const int v = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += v;
        }
        const int agg = __shfl_sync(kFull, incl, WT - 1);
        int off_local = incl - cnt;
        if (!PRE && lane == 0) st_release(states + tile, (tile == 0 ? kInc : kAgg) | (uint64_t)agg);
        int next = 0;
        if (lane == 0) next = (int)atomicAdd(ticket, 1u);
        // ---------------- look-back, first attempt right after the publish: walk back over at most
        // kEarlyRounds × 32 predecessor states without waiting; success publishes this tile's
        // inclusive prefix now, so successors find one close by.  If a predecessor is still
        // unpublished the attempt is dropped and the full look-back runs after the union (whose
        // duration hides the wait).  (Only after the union, the walk crossed every tile still in
        // its union — ~300 instructions of polling per tree; only before it, warps spun on
        // predecessors still in their select: 2.5x slower.)
        unsigned prefix = 0;
        bool have = tile == 0 || PRE;   // PRE: the select launch scanned the offsets
        if (!have) have = lookback_walk<false>(tile, states, agg, prefix, lane);
        EVICT_PHASE(1);
        // ---------------- A2: expert union, one warp per tree
        if (do_union) {
            if constexpr (FLAGS) {
                // every union path leaves its flag block zero after each tree; only the
                // prefix the sweeps / emit scribbled on needs clearing (all of it once)
                uint4 *f4 = reinterpret_cast<uint4 *>(wscr);
                const int nflag = union_flag_bytes(L, E) / 16;   // uint4 words
                constexpr int dirty = (int)(fused_scratch_dirty<G>() / 16);
                // (PRE: only the emit writes the prefix, and only for kept sets > 16 — its child masks)
                const int nz = first ? nflag : ((PRE && !emit_dirty) ? 0 : (dirty < nflag ? dirty : nflag));
                for (int i = lane; i < nz; i += 32) f4[i] = make_uint4(0u, 0u, 0u, 0u);
                __syncwarp();
                first = false;
            }
#pragma unroll 1
            // cross-tree prefetch of the tile's first kept rows (a tree's first batch is in flight
            // during the previous tree's read-back)
            UColsBatch<EVICT_UCOLS_UB> pfb;
#ifdef EVICT_UPF   // measured 12% slower: the prefetched registers spill (a spill store waits for its load)
            UColsBatch<EVICT_UCOLS_UB> *pfp = &pfb;
#else
            UColsBatch<EVICT_UCOLS_UB> *pfp = nullptr;
#endif
            if constexpr (LEAN && EW == 2 && CL <= 4) {
                if (pfp) {
                const EmitRec<G> &e0 = rec[0];
                if (b0 < tr.batch && e0.status == 0u && e0.k > 0)
                    ucols_load<CL == 4 ? 2 : 1, EVICT_UCOLS_UB>(pfb, e0.klist, e0.k, 0, b0, N, L, rt.ids, lane);
                }
            }
            for (int slot = 0; slot < WT; slot++) {
                const int b = b0 + slot;
                if (b >= tr.batch) break;
                EmitRec<G> &er = rec[slot];
                uint32_t st = er.status;
                if constexpr (LEAN && EW == 2 && CL <= 4) {
                    // lane-owned flag columns (conflict-free byte stores); CL = 3: L ≤ 48, CL = 4: L ≤ 64
                    const bool nx = slot + 1 < WT && b + 1 < tr.batch && rec[slot + 1].status == 0u;
                    const int nk = nx ? rec[slot + 1].k : 0;
                    tree_union_cols<CL == 4 ? 2 : 1, EVICT_UCOLS_UB>(st, er.klist, er.k, b, N, L, rt.ids, wscr,
                                                                   out.union_count, out.union_total, &epoch,
                                                                   fstats ? lsum : nullptr, ulane, sfold, hfold,
                                                                   pfp, rec[nx ? slot + 1 : slot].klist, nk, b + 1);
                    if constexpr (kFold) {
                        if (fstats && lane == 0) {
                            rs_tr += 1u;
                            if (st) {
                                rs_err += 1u;
                                atomicAdd(&fs->hist[0], 1u);
                            } else {
                                rs_k += (unsigned)er.k;
                                rs_n += (unsigned)er.n;
                                rs_e += (double)er.ehat;
                                rs_u += (double)er.util;
                                atomicAdd(&fs->hist[er.k], 1u);
                            }
                        }
                    }
                }
                else if constexpr (LEAN && EW == 2)
                    tree_union_flags64<1, CL, true, false, false, WT == 1 ? 8 : 4>(
                        st, er.klist, er.k, b, N, L, E, rt.ids, wscr, out.union_count, out.union_total, nullptr,
                        &epoch, nullptr);
                else if constexpr (LEAN)   // 128 < E ≤ 256 (Ling-flash-2.0): 32-byte expert rows
                    tree_union_flags64<1, CL, false, false, true, WT == 1 ? 8 : 4>(
                        st, er.klist, er.k, b, N, L, E, rt.ids, wscr, out.union_count, out.union_total, nullptr,
                        &epoch);
                else
                    tree_union<NPL, IDF, KT, EW, CL>(st, er.klist, er.k, b, N, L, rt.top_k, E, rt.id_format,
                                                     rt.ids, wscr, Epad, out.union_count, out.union_total,
                                                     out.union_bits, out.expert_hist);
                if (lane == 0) er.status = st;
                __syncwarp();
            }
        }
        EVICT_PHASE(2);
        if (!have) lookback_walk<true>(tile, states, agg, prefix, lane);
        EVICT_PHASE(3);
        off_local += (int)prefix;
        next = __shfl_sync(kFull, next, 0);
        // ---------------- C: verify-tree emit, sub-warp per tree
#pragma unroll 1
        for (int pass = 0; pass < PASSES; pass++) {
            const int slot = pass * TPW + gi;
            const int b = b0 + slot;
            const bool active = slot < WT && b < tr.batch;
            const EmitRec<G> &er = rec[slot < WT ? slot : 0];
            const int k = active ? er.k : 0;
            const int off = PRE ? (active ? __ldg(out.verify_offsets + b) : 0)
                                : __shfl_sync(kFull, off_local, slot < WT ? slot : 0);
            if (active && g == 0) {
                if (out.status) out.status[b] = er.status;
                if (!PRE && out.verify_offsets) {
                    out.verify_offsets[b] = off;
                    if (b == tr.batch - 1) out.verify_offsets[tr.batch] = off + k;
                }
            }
            uint64_t keep[W];
#pragma unroll
            for (int w = 0; w < W; w++) keep[w] = active ? er.keep[w] : 0ull;
            uint64_t *child = reinterpret_cast<uint64_t *>(wscr) + (size_t)gi * NMAX * W;
            grp::g_emit<G>(keep, active ? er.n : 0, active && k > 0, k, b, N, off,
                           (active && out.pos_offset) ? __ldg(out.pos_offset + b) : 0, er.par,
                           child, er.klist, out.kept_index, out.retrieve_index, out.positions,
                           out.next_token, out.next_sibling, out.tree_mask, W == 1 ? er.slot : nullptr);
            // (g_emit writes child masks into the prefix unless W = 1 and k ≤ 16)
            if (pass == 0) emit_dirty = false;
            emit_dirty |= __any_sync(kFull, W != 1 || (active && k > 16));
            __syncwarp();
        }
        EVICT_PHASE(4);
        tile = next;
    }
    if constexpr (kFold) {
        if (fstats) {
            if (lane == 0) {
                fs->sc[warp][0] = rs_tr; fs->sc[warp][1] = rs_k; fs->sc[warp][2] = rs_n; fs->sc[warp][3] = rs_err;
                fs->d[warp][0] = rs_e; fs->d[warp][1] = rs_u;
            }
            // per-lane layer sums (tree_union_cols' output layers)
#pragma unroll
            for (int m = 0; m < 4; m++)
                if (m < ulane.nl && lsum[m]) atomicAdd(&fs->lay[ulane.l0 + m], lsum[m]);
            __syncthreads();
            unsigned long long *gs = reinterpret_cast<unsigned long long *>(out.stats);
            if (threadIdx.x == 0) {
                unsigned long long su = 0, sc[4] = {0ull, 0ull, 0ull, 0ull};
                for (int l = 0; l < L; l++) su += fs->lay[l];
                for (int w = 0; w < NW; w++)
                    for (int i = 0; i < 4; i++) sc[i] += fs->sc[w][i];
                if (sc[0]) atomicAdd(gs + 0, sc[0]);
                if (sc[1]) atomicAdd(gs + 1, sc[1]);
                if (sc[2]) atomicAdd(gs + 2, sc[2]);
                if (su) atomicAdd(gs + 3, su);
                if (sc[3]) atomicAdd(gs + 4, sc[3]);
                double de = 0.0, du = 0.0;
                for (int w = 0; w < NW; w++) { de += fs->d[w][0]; du += fs->d[w][1]; }
                atomicAdd(out.dstats + 0, de);
                atomicAdd(out.dstats + 1, du);
            }
            for (int i = threadIdx.x; i <= N; i += blockDim.x)
                if (fs->hist[i]) atomicAdd(gs + 5 + i, (unsigned long long)fs->hist[i]);
            for (int l = threadIdx.x; l < L; l += blockDim.x)
                if (fs->lay[l]) atomicAdd(gs + 6 + N + l, (unsigned long long)fs->lay[l]);
        }
    }
}


// ------------------------------------------------------------ select (grouped)
// evict_select: G lanes per tree, 32/G trees per warp, 4 warps per CTA (small
// CTAs keep batch-64 latency low: 64 trees → 4 CTAs on 4 SMs).
constexpr int kSelWarps = 4;
constexpr int kScanChunk = 4096;   // trees per chunk of the packed-offset scan (1024 threads × 4)

// Packed verify-row offsets, second half: block c adds the chunk sums before it, then scans its
// chunk's k* (4 per thread, warp shuffles + one smem pass) — verify_offsets[b] = Σ_{b' < b} k*,
// verify_offsets[B] = T.  k* of an errored tree is 0.
static __global__ void __launch_bounds__(1024) k_scan_offsets(int B, const int32_t *__restrict__ k_star,
                                                       const int32_t *__restrict__ chunk_sums,
                                                       int32_t *__restrict__ verify_offsets)
{
    __shared__ int s_w[32];
    __shared__ int s_base;
    const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int pre = 0;
    for (int j = tid; j < c; j += blockDim.x) pre += chunk_sums[j];
    pre = __reduce_add_sync(kFull, pre);
    if (lane == 0) s_w[warp] = pre;
    __syncthreads();
    if (warp == 0) {
        const int v = __reduce_add_sync(kFull, s_w[lane]);
        if (lane == 0) s_base = v;
    }
    __syncthreads();
    const int b0 = c * kScanChunk + tid * 4;
    int k[4];
#pragma unroll
    for (int i = 0; i < 4; i++) k[i] = b0 + i < B ? __ldg(k_star + b0 + i) : 0;
    const int own = k[0] + k[1] + k[2] + k[3];
    int inc = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += v;
    }
    __syncthreads();
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const int x = s_w[lane];
        int xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(kFull, xi, o);
            if (lane >= o) xi += v;
        }
        s_w[lane] = xi - x;                       // exclusive prefix of warp totals
    }
    __syncthreads();
    int run = s_base + s_w[warp] + inc - own;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        if (b0 + i < B) verify_offsets[b0 + i] = run;
        run += k[i];
        if (b0 + i == B - 1) verify_offsets[B] = run;
    }
}

template <int G, bool COST = false>   // COST: the policy is EVICT_POLICY_COST (compile-time argmax epilogue)
__global__ void __launch_bounds__(kSelWarps * 32) k_select_g(evict_trees_t tr, const float *cost,
                                                             int cost_stride, evict_policy_t pol, int32_t *k_star,
                                                             float *e_hat, float *utility,
                                                             uint64_t *keep_bits, int32_t *order,
                                                             float *prefix_sums, uint32_t *status,
                                                             int32_t *chunk_sums = nullptr)
{
    constexpr int TPW = grp::GShape<G>::TPW;
    constexpr int NMAX = grp::GShape<G>::NMAX;
    constexpr int W = grp::GShape<G>::W;
    constexpr int PER = kSelWarps * TPW;               // trees per CTA tile
    __shared__ __align__(16) float sd_all[kSelWarps * TPW * NMAX];
    __shared__ uint8_t rk_all[kSelWarps * TPW * NMAX];
    __shared__ int s_k[PER];
    const int warp = threadIdx.x >> 5;
    const int gi = grp::gidx<G>(), g = grp::gl<G>();
    const int slot = warp * TPW + gi;
    const int b = blockIdx.x * PER + slot;
    const bool active = b < tr.batch;
    const int N = tr.max_nodes;
    const int WN = (N + 63) / 64;
    grp::GTree<G> t;
    float4 cr[2];
    grp::g_fetch_cost<G>(cr, cost + (size_t)(active ? b : 0) * cost_stride, N, active);
    grp::g_load<G>(t, tr.parent, tr.q, tr.n_nodes, b, N, active);
    float c[grp::NP];
    grp::g_apply_cost<G>(c, t, cr);
    grp::g_levels<G, true>(t, sd_all + slot * NMAX);
    int32_t *orow = (active && order) ? order + (size_t)b * N : nullptr;
    float *prow = (active && prefix_sums) ? prefix_sums + (size_t)b * N : nullptr;
    if (order) grp::g_rank_argmax<G>(t, rk_all + slot * NMAX, c, N, orow, prow, pol);   // kernel-uniform
    else grp::g_select_values<G, COST>(t, c, N, prow, pol);
    if (chunk_sums) {
        // packed verify-row offsets, first half: Σk* per chunk of kScanChunk trees (one atomic
        // per CTA); k_scan_offsets turns the chunk sums and k* into the exclusive scan
        if (g == 0) s_k[slot] = active ? t.kstar : 0;
        __syncthreads();
        if (warp == 0) {
            const int lane = lane_id();
            const int v = __reduce_add_sync(kFull, lane < PER ? s_k[lane] : 0);
            if (lane == 0 && v) atomicAdd(chunk_sums + (blockIdx.x * PER) / kScanChunk, v);
        }
    }
    if (!active) return;
    if (g == 0) {
        k_star[b] = t.kstar;
        e_hat[b] = t.ehat;
        utility[b] = t.util;
        if (status) status[b] = t.status;
    }
    if (g < WN) keep_bits[(size_t)b * WN + g] = t.keep[g < W ? g : 0];
}

// ------------------------------------------------------------ launchers
int dev_sms();  // evict_api.cu

inline evict_status_t launched() { return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA; }

template <typename K>
inline int persistent_blocks(K kernel, int ntiles, size_t dyn = 0, int nthreads = kWarps * 32)
{
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, nthreads, dyn);
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
        const size_t dyn = (IDF == 1 || IDF == 4) ? (size_t)kWarps * union_flag_bytes(rt->num_layers,
                                                                                      rt->num_experts) : 0;
        auto kern = k_union<NPL, IDF, KT, EW, CL>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        kern<<<blocks, kWarps * 32, dyn, s>>>(*tr, keep, *rt, uc, ut, ub, eh, st);
        return launched();
    }
};

// ------------------------------------------------------------ fused, serving batches
// Batches up to kSmallBatch in the u8 serving configuration: one warp per tree, the latency
// chain of k_select (32 lanes × NPL nodes: the shortest select) → publish k* → expert union
// (8 kept rows per load batch: one DRAM round trip for a typical tree) → decoupled look-back for
// the packed offset → warp-wide emit (k_build's tree_build_emit).  Tree b is warp b of the grid
// (every warp is resident for B ≤ kSmallBatch), so predecessors always run.  ws[1 + b]: tile
// states.  Statistics are not folded here (the call runs k_stats when they are requested).
template <int NPL, int EW, int CL, int WPC>   // WPC: warps (trees) per CTA
__global__ void __launch_bounds__(WPC * 32) k_fused_lat(evict_trees_t tr, const float *cost, int cost_stride,
                                                         evict_policy_t pol, evict_routing_t rt,
                                                         evict_fused_out_t out, uint64_t *ws)
{
    constexpr int W = Shape<NPL>::W;
    extern __shared__ __align__(16) uint8_t dsm[];       // WPC × 8 KB union flag blocks
    __shared__ WarpSlab<NPL> slab[WPC];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int b = blockIdx.x * WPC + warp;
    if (b >= tr.batch) return;
    uint8_t *flags = dsm + (size_t)warp * 8192;
    uint4 *f4 = reinterpret_cast<uint4 *>(flags);
    for (int i = lane; i < 8192 / 16; i += 32) f4[i] = make_uint4(0u, 0u, 0u, 0u);
    const int N = tr.max_nodes;
    const int WN = (N + 63) / 64;
    const int L = rt.num_layers, E = rt.num_experts;
    WarpSlab<NPL> &sm = slab[warp];
    TreeState<NPL> t;
    tree_load_validate<NPL>(t, tr, tr.parent, tr.q, tr.n_nodes, b, N);
    float c[NPL];
    if (!(t.status & EVICT_TREE_BAD_SIZE)) tree_load_cost<NPL>(c, t, cost + (size_t)b * cost_stride);
    if (!t.status) {
        tree_levels<NPL, true>(t, sm);
        tree_rank_argmax<NPL>(t, sm, c, N, nullptr, nullptr, pol);
    } else {
        t.kstar = 0; t.ehat = 0.f; t.util = 0.f;
#pragma unroll
        for (int w = 0; w < W; w++) t.keep[w] = 0ull;
    }
    const int k = t.kstar;
    uint64_t *states = ws + 1;
    if (lane == 0) {
        st_release(states + b, (b == 0 ? kInc : kAgg) | (uint64_t)k);
        if (out.k_star) out.k_star[b] = t.kstar;
        if (out.e_hat) out.e_hat[b] = t.ehat;
        if (out.utility) out.utility[b] = t.util;
    }
    if (out.keep_bits && lane < WN) out.keep_bits[(size_t)b * WN + lane] = t.keep[lane < W ? lane : 0];
    if (!t.status) tree_fill_klist<NPL>(t, sm);
    uint32_t st = t.status;
    int epoch = 0;
    __syncwarp();
    // (tree_union_cols measured 8% slower here at batch 64: 11.2 vs 10.3 µs per graph replay)
    if constexpr (EW == 2)
        tree_union_flags64<1, CL, true, false, false, 8>(st, sm.klist, k, b, N, L, E, rt.ids, flags,
                                                         out.union_count, out.union_total, nullptr, &epoch);
    else
        tree_union_flags64<1, CL, false, false, true, 8>(st, sm.klist, k, b, N, L, E, rt.ids, flags,
                                                         out.union_count, out.union_total, nullptr, &epoch);
    unsigned prefix = 0;
    if (b > 0) lookback_walk<true>(b, states, k, prefix, lane);
    const int off = (int)prefix;
    if (lane == 0) {
        if (out.status) out.status[b] = st;
        if (out.verify_offsets) {
            out.verify_offsets[b] = off;
            if (b == tr.batch - 1) out.verify_offsets[tr.batch] = off + k;
        }
    }
    if (k > 0)
        tree_build_emit<NPL>(t, sm, k, b, N, off, out.pos_offset ? __ldg(out.pos_offset + b) : 0,
                             out.kept_index, out.retrieve_index, out.positions, out.next_token,
                             out.next_sibling, out.tree_mask);
}

template <int NPL, int IDF, int KT, int EW, int CL>
struct FusedLauncher {
    // the caller cleared 1 + batch tile states when batch ≤ kSmallBatch (else 1 + ⌈batch/4⌉)
    static evict_status_t run(const evict_trees_t *tr, const float *cost, int cs, evict_policy_t pol,
                              const evict_routing_t *rt, const evict_fused_out_t *o, uint64_t *ws,
                              int /*ntiles*/, cudaStream_t s)
    {
        auto kern = k_fused<NPL, IDF, KT, EW, CL, false>;
        constexpr int G = NPL == 2 ? 8 : 16;
        const bool flags = (IDF == 1 || IDF == 4) && o->union_count;
        size_t dyn = fused_smem_bytes<G>(rt->num_layers, rt->num_experts, flags);
        int wt = kWT;
        if constexpr (IDF == 1 && (EW == 2 || EW == 4)) {
            const bool shape = EW == 2 ? rt->num_experts == 128 : rt->num_experts > 128;
            if (shape && !o->order && !o->union_bits && !o->expert_hist && o->union_count) {
                if (tr->batch <= kSmallBatch) {
                    // up to one SM per tree: a CTA per tree while the batch fits the SMs, else 8 per CTA
                    if (tr->batch <= dev_sms()) {
                        k_fused_lat<NPL, EW, CL, 1><<<tr->batch, 32, 8192, s>>>(*tr, cost, cs, pol, *rt, *o, ws);
                    } else {
                        auto lk = k_fused_lat<NPL, EW, CL, kWarps>;
                        const int ldyn = kWarps * 8192;
                        cudaFuncSetAttribute(lk, cudaFuncAttributeMaxDynamicSharedMemorySize, ldyn);
                        lk<<<(tr->batch + kWarps - 1) / kWarps, kWarps * 32, ldyn, s>>>(*tr, cost, cs, pol, *rt, *o, ws);
                    }
                    return launched();
                } else if (o->k_star && o->e_hat && o->utility && o->keep_bits && o->status && o->verify_offsets) {
                    // throughput batches: the select (+ packed-offset scan) as its own launch at full
                    // occupancy, then A6 + A7 (+ A9) reading its outputs — no look-back in the union
                    // kernel (ws[0]: its ticket; ws[1]: the scan's ticket; ws[2..]: scan tile states)
                    constexpr int PER = kSelWarps * grp::GShape<G>::TPW;
                    const int sblocks = (tr->batch + PER - 1) / PER;
                    int32_t *chunk_sums = reinterpret_cast<int32_t *>(ws + 1);   // zeroed by the caller
                    auto sk = pol.kind == EVICT_POLICY_COST ? k_select_g<G, true> : k_select_g<G, false>;
                    sk<<<sblocks, kSelWarps * 32, 0, s>>>(*tr, cost, cs, pol, o->k_star, o->e_hat, o->utility,
                                                         o->keep_bits, nullptr, nullptr, o->status, chunk_sums);
                    k_scan_offsets<<<(tr->batch + kScanChunk - 1) / kScanChunk, 1024, 0, s>>>(
                        tr->batch, o->k_star, chunk_sums, o->verify_offsets);
                    if (cudaGetLastError() != cudaSuccess) return EVICT_ERR_CUDA;
#ifdef EVICT_PRE_NW4   // measured 1.2% slower than 8-warp CTAs (ptxas keeps the static base in a register)
                    if constexpr (EW == 2 && CL <= 4) {
                        // 4-warp CTAs, static flag blocks (tree_union_cols' store addressing)
                        auto pk = k_fused<NPL, IDF, KT, EW, CL, true, kWT, true, 4>;
                        const size_t pdyn = align16(sizeof(EmitRec<G>) * 4 * kWT) + kStatsSmem;   // flags static
                        const int pt = (tr->batch + kWT - 1) / kWT;
                        cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pdyn);
                        pk<<<persistent_blocks(pk, pt, pdyn, 4 * 32), 4 * 32, pdyn, s>>>(*tr, cost, cs, pol, *rt, *o,
                                                                                         ws, pt);
                        return launched();
                    }
#endif
                    kern = k_fused<NPL, IDF, KT, EW, CL, true, kWT, true>;
                } else {
                    kern = k_fused<NPL, IDF, KT, EW, CL, true>;
                }
            }
        }
        const int ntiles = (tr->batch + wt - 1) / wt;
        if (kern != k_fused<NPL, IDF, KT, EW, CL, false>)   // LEAN instantiations: no ranks area
            dyn = fused_smem_bytes<G>(rt->num_layers, rt->num_experts, flags, false);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        const int blocks = persistent_blocks(kern, ntiles, dyn);
        kern<<<blocks, kWarps * 32, dyn, s>>>(*tr, cost, cs, pol, *rt, *o, ws, ntiles);
        return launched();
    }
};

template <int NPL>
evict_status_t launch_select(const evict_trees_t *tr, const float *cost, int cs, evict_policy_t pol, int32_t *k_star,
                             float *e_hat, float *utility, uint64_t *keep_bits, int32_t *order,
                             float *prefix_sums, uint32_t *status, cudaStream_t s)
{
    if (tr->batch <= 4096) {
        // latency regime (serving batches): one warp per tree, shortest dependency chain
        const int blocks = (tr->batch + kWarps - 1) / kWarps;
        k_select<NPL><<<blocks, kWarps * 32, 0, s>>>(*tr, cost, cs, pol, k_star, e_hat, utility, keep_bits,
                                                       order, prefix_sums, status);
        return launched();
    }
    // throughput regime: sub-warp groups, 32/G trees per warp instruction
    constexpr int G = NPL == 2 ? 8 : 16;
    constexpr int per_cta = kSelWarps * grp::GShape<G>::TPW;
    const int blocks = (tr->batch + per_cta - 1) / per_cta;
    auto sk = (pol.kind == EVICT_POLICY_COST && !order) ? k_select_g<G, true> : k_select_g<G, false>;
    sk<<<blocks, kSelWarps * 32, 0, s>>>(*tr, cost, cs, pol, k_star, e_hat, utility, keep_bits,
                                                      order, prefix_sums, status, nullptr);
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
evict_status_t launch_fused(const evict_trees_t *tr, const float *cost, int cs, evict_policy_t pol,
                            const evict_routing_t *rt, const evict_fused_out_t *o, uint64_t *ws,
                            int ntiles, cudaStream_t s)
{
    return dispatch_union<NPL, FusedLauncher>(rt, tr, cost, cs, pol, rt, o, ws, ntiles, s);
}

}  // namespace evict
