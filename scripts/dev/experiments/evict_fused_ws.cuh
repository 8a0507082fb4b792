#pragma once
// evict_fused_ws.cuh — warp-specialised fused select → build → union (A1–A7) for the serving /
// bench configuration (u8 top-8 ids, E = 128 or 128 < E ≤ 256, no order row, no union bit rows,
// no histogram) at throughput batch sizes.  Included by evict_kernels.cuh after k_fused.
//
// One CTA = kWsSel select warps + kWsUni union warps sharing a ring of union records:
//   select warps  take 4-tree tickets (sub-warp per tree, evict_group.cuh): A1–A5, publish the
//                 tile's row count, decoupled look-back for its packed offset, push one union
//                 record per tree (kept list, tree id, status) into the ring, then A6 emit;
//                 tickets are taken after the emit, so a tile's predecessors are in the same
//                 phase and the look-back wait stays short
//   union warps   pop records and run A7 (tree_union_flags64, one warp per tree, an 8 KB
//                 flag block each), writing union_count / union_total / status
// The emit (A6) does not need the union, and the union does not need the packed offsets, so the
// two halves only meet through the ring (mbarrier full/empty pairs per slot).  Each warp runs one
// small loop, so the SM's instruction caches hold both loops instead of thrashing on one long
// body whose phases the warps visit out of step (k_fused: ~20% of stall samples were
// "no instruction"), and union loads are in flight while the select warps compute.
#include "evict_kernels.cuh"

namespace evict {
namespace ws {

constexpr int kWsSel = 4, kWsUni = 4;                 // warps per role
constexpr int kWsThreads = (kWsSel + kWsUni) * 32;
constexpr int kRing = 32;                             // union records in flight per CTA

template <int G>
struct UnionRec {
    alignas(16) uint8_t klist[grp::GShape<G>::NMAX];  // kept nodes, ascending
    int b, k;                                         // k < 0: end of stream (one per select warp)
    uint32_t status;
};

__device__ __forceinline__ uint32_t sptr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t *b, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sptr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sptr(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t parity)
{
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(sptr(b)),
        "r"(parity)
        : "memory");
}

template <int G>
__host__ __device__ constexpr size_t ws_sel_scratch() { return fused_scratch_fixed<G>(); }

template <int G, int WT>
__host__ __device__ constexpr size_t ws_smem_bytes()
{
    return (size_t)kWsUni * 8192                                   // union flag blocks
           + (size_t)kWsSel * ws_sel_scratch<G>()                  // sweeps / emit child masks
           + align16(sizeof(EmitRec<G>) * kWsSel * WT)             // select records
           + align16(sizeof(UnionRec<G>) * kRing)                  // ring
           + 2 * kRing * 8 + 16;                                   // full/empty barriers, heads
}

template <int NPL, int EW, int R>
__global__ void __launch_bounds__(kWsThreads, 3) k_fused_ws(evict_trees_t tr, const float *cost, int cost_stride,
                                                            evict_policy_t pol, evict_routing_t rt,
                                                            evict_fused_out_t out, uint64_t *wsp, int ntiles)
{
    constexpr int G = NPL == 2 ? 8 : 16;
    constexpr int WT = kWT;
    constexpr int TPW = grp::GShape<G>::TPW;
    constexpr int NMAX = grp::GShape<G>::NMAX;
    constexpr int W = grp::GShape<G>::W;
    constexpr int PASSES = WT / TPW;                  // 1 (G=8) or 2 (G=16)
    extern __shared__ __align__(16) uint8_t dsm[];
    uint8_t *flags0 = dsm;
    uint8_t *sel0 = flags0 + (size_t)kWsUni * 8192;
    EmitRec<G> *recs = reinterpret_cast<EmitRec<G> *>(sel0 + (size_t)kWsSel * ws_sel_scratch<G>());
    UnionRec<G> *ring = reinterpret_cast<UnionRec<G> *>(reinterpret_cast<uint8_t *>(recs) +
                                                       align16(sizeof(EmitRec<G>) * kWsSel * WT));
    uint64_t *full = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(ring) + align16(sizeof(UnionRec<G>) * kRing));
    uint64_t *empty = full + kRing;
    int *heads = reinterpret_cast<int *>(empty + kRing);   // [0] producer, [1] consumer
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int N = tr.max_nodes;
    const int L = rt.num_layers, E = rt.num_experts;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kRing; i++) {
            bar_init(full + i, 1);
            bar_init(empty + i, 1);
        }
        heads[0] = 0;
        heads[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp >= kWsSel) {
        // ======================= union warps
        uint8_t *flags = flags0 + (size_t)(warp - kWsSel) * 8192;
        uint4 *f4 = reinterpret_cast<uint4 *>(flags);
        for (int i = lane; i < 8192 / 16; i += 32) f4[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
        int epoch = 0;
        while (true) {
            int idx = 0;
            if (lane == 0) idx = atomicAdd(heads + 1, 1);
            idx = __shfl_sync(kFull, idx, 0);
            const int rs = idx % kRing;
            bar_wait(full + rs, (uint32_t)(idx / kRing) & 1u);
            const UnionRec<G> &r = ring[rs];
            const int k = r.k;
            if (k < 0) {
                __syncwarp();
                if (lane == 0) bar_arrive(empty + rs);
                break;
            }
            const int b = r.b;
            uint32_t st = r.status;
            if constexpr (EW == 2)
                tree_union_flags64<1, R, true, false>(st, r.klist, k, b, N, L, E, rt.ids, flags, out.union_count,
                                                      out.union_total, nullptr, &epoch);
            else
                tree_union_flags64<1, R, false, false, true>(st, r.klist, k, b, N, L, E, rt.ids, flags,
                                                             out.union_count, out.union_total, nullptr, &epoch);
            if (lane == 0 && out.status) out.status[b] = st;
            __syncwarp();
            if (lane == 0) bar_arrive(empty + rs);
        }
        return;
    }

    // ======================= select / emit warps
    const int gi = grp::gidx<G>(), g = grp::gl<G>();
    const int WN = (N + 63) / 64;
    uint8_t *wscr = sel0 + (size_t)warp * ws_sel_scratch<G>();
    EmitRec<G> *rec = recs + warp * WT;
    unsigned *ticket = reinterpret_cast<unsigned *>(wsp);
    uint64_t *states = wsp + 1;
    int tile = 0;
    if (lane == 0) tile = (int)atomicAdd(ticket, 1u);
    tile = __shfl_sync(kFull, tile, 0);
    while (tile < ntiles) {
        const int b0 = tile * WT;
        // ---------------- A1–A5: select, sub-warp per tree
#pragma unroll 1
        for (int pass = 0; pass < PASSES; pass++) {
            const int slot = pass * TPW + gi;
            const int b = b0 + slot;
            const bool active = b < tr.batch;
            grp::GTree<G> t;
            grp::g_load<G>(t, tr.parent, tr.q, tr.n_nodes, b, N, active);
            float c[grp::NP];
            grp::g_load_cost<G>(c, t, cost + (size_t)(active ? b : 0) * cost_stride, N);
            float *sd = reinterpret_cast<float *>(wscr) + gi * (NMAX + 8);
            grp::g_levels<G, true>(t, sd);
            grp::g_select_values<G>(t, c, N, nullptr, pol);
            const int k = t.kstar;
            EmitRec<G> &er = rec[slot];
            if (active) {
                if (g == 0) {
                    if (out.k_star) out.k_star[b] = t.kstar;
                    if (out.e_hat) out.e_hat[b] = t.ehat;
                    if (out.utility) out.utility[b] = t.util;
                }
                if (out.keep_bits && g < WN) out.keep_bits[(size_t)b * WN + g] = t.keep[g < W ? g : 0];
                const int base = g * grp::NP;
                uint32_t pw[2] = {0u, 0u};
#pragma unroll
                for (int r = 0; r < grp::NP; r++) pw[r >> 2] |= (uint32_t)(t.par[r] & 0xff) << (8 * (r & 3));
                *reinterpret_cast<uint2 *>(&er.par[base]) = make_uint2(pw[0], pw[1]);
                if (g < W) er.keep[g] = t.keep[g];
#pragma unroll
                for (int r = 0; r < grp::NP; r++) {
                    const int i = base + r;
                    if (i < t.n && grp::bit_w<W>(t.keep, i)) er.klist[grp::popc_below_w<W>(t.keep, i)] = (uint8_t)i;
                }
                if (g == 0) { er.n = t.n; er.k = k; er.status = t.status; }
            } else if (g == 0) {
                er.k = 0;
            }
            __syncwarp();
        }
        // ---------------- tile aggregate, publish, look-back (predecessors are in this phase too)
        const int cnt = lane < WT ? rec[lane].k : 0;
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < WT; o <<= 1) {
            const int v = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += v;
        }
        const int agg = __shfl_sync(kFull, incl, WT - 1);
        int off_local = incl - cnt;
        if (lane == 0) st_release(states + tile, (tile == 0 ? kInc : kAgg) | (uint64_t)agg);
        unsigned prefix = 0;
        if (tile > 0) lookback_walk<true>(tile, states, agg, prefix, lane);
        off_local += (int)prefix;
        // ---------------- hand the tile's trees to the union warps
        const int nvalid = tr.batch - b0 < WT ? tr.batch - b0 : WT;
        int base_idx = 0;
        if (lane == 0) base_idx = atomicAdd(heads, nvalid);
        base_idx = __shfl_sync(kFull, base_idx, 0);
#pragma unroll 1
        for (int slot = 0; slot < nvalid; slot++) {
            const int idx = base_idx + slot;
            const int rs = idx % kRing;
            if (idx >= kRing) bar_wait(empty + rs, (uint32_t)(idx / kRing - 1) & 1u);
            UnionRec<G> &r = ring[rs];
            const EmitRec<G> &er = rec[slot];
            if (lane < NMAX / 8)
                reinterpret_cast<uint2 *>(r.klist)[lane] = reinterpret_cast<const uint2 *>(er.klist)[lane];
            if (lane == 0) {
                r.b = b0 + slot;
                r.k = er.k;
                r.status = er.status;
            }
            __syncwarp();
            if (lane == 0) bar_arrive(full + rs);
        }
        int next = 0;
        if (lane == 0) next = (int)atomicAdd(ticket, 1u);   // consumed after the emit
        // ---------------- A6: verify-tree emit, sub-warp per tree
#pragma unroll 1
        for (int pass = 0; pass < PASSES; pass++) {
            const int slot = pass * TPW + gi;
            const int b = b0 + slot;
            const bool active = b < tr.batch;
            const EmitRec<G> &er = rec[slot];
            const int k = active ? er.k : 0;
            const int off = __shfl_sync(kFull, off_local, slot);
            if (active && g == 0 && out.verify_offsets) {
                out.verify_offsets[b] = off;
                if (b == tr.batch - 1) out.verify_offsets[tr.batch] = off + k;
            }
            uint64_t keep[W];
#pragma unroll
            for (int w = 0; w < W; w++) keep[w] = active ? er.keep[w] : 0ull;
            uint64_t *child = reinterpret_cast<uint64_t *>(wscr) + (size_t)gi * NMAX * W;
            grp::g_emit<G>(keep, active ? er.n : 0, active && k > 0, k, b, N, off,
                           (active && out.pos_offset) ? __ldg(out.pos_offset + b) : 0, er.par,
                           child, er.klist, out.kept_index, out.retrieve_index, out.positions,
                           out.next_token, out.next_sibling, out.tree_mask);
            __syncwarp();
        }
        tile = __shfl_sync(kFull, next, 0);
    }
    // end of stream: one sentinel per select warp (there are as many union warps)
    int idx = 0;
    if (lane == 0) idx = atomicAdd(heads, 1);
    idx = __shfl_sync(kFull, idx, 0);
    const int rs = idx % kRing;
    if (idx >= kRing) bar_wait(empty + rs, (uint32_t)(idx / kRing - 1) & 1u);
    if (lane == 0) {
        ring[rs].k = -1;
        bar_arrive(full + rs);
    }
}

}  // namespace ws
}  // namespace evict
