// evict_tree.cuh — warp-per-tree device building blocks of the EVICT hot path
// (sm_100a).  One warp owns one draft tree; lane t owns the NPL consecutive
// nodes i = t*NPL + r (blocked layout, so rows load as 8/16-byte vectors).
// The tree is staged in registers + a small per-warp shared-memory slab;
// nothing here touches the host.
//
//   A1 tree_load_validate  PAPER.md:48 (tree), readings Z4/Z9/Z10
//   A2 tree_scores         Eq. 7: level-synchronous fp32
//                          product root→leaf (exact serial order per node)
//   A3 tree_rank           §3.2.1: warp bitonic sort of
//                          64-bit keys (~bits(score) << 32 | index)
//   A4/A5 tree_argmax      Eq. 8–10: shuffle scan,
//                          IEEE division by C(k), argmax via __reduce_max_sync
//   A6 tree_build          Fig. 4(c): __ballot/__popc slot
//                          compaction, ancestor-or-self mask rows, child lists
//   A7 tree_union          Eq. 5: OR of kept nodes' routing
//                          into per-layer expert bitsets, __popcll counts
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "evict.h"

namespace evict {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kWarps = 8;  // warps (= trees) per CTA tile

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <int NPL>
struct Shape {
    static constexpr int NMAX = 32 * NPL;          // nodes per warp
    static constexpr int W = (NMAX + 63) / 64;     // 64-bit mask words
    static constexpr int W32 = (NMAX + 31) / 32;   // 32-bit words
};

// Per-warp shared-memory slab.
template <int NPL>
struct WarpSlab {
    static constexpr int NMAX = Shape<NPL>::NMAX;
    static constexpr int W = Shape<NPL>::W;
    int2 sd[NMAX];              // A2 (score bits, depth) of the previous sweep
    uint8_t rank[NMAX];         // A3 node → rank
    uint8_t klist[NMAX];        // A7 slot → node
    uint64_t row[NMAX][W];      // A6 mask rows by slot
    uint64_t child[NMAX][W];    // A6 kept-children masks by slot
};

// Register state of one tree (per lane: its NPL nodes).
template <int NPL>
struct TreeState {
    static constexpr int W = Shape<NPL>::W;
    int par[NPL];
    float q[NPL];
    float sc[NPL];
    int dep[NPL];
    int n;
    uint32_t status;
    int kstar;
    float ehat, util;
    uint64_t keep[W];  // identical in every lane
};

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ uint64_t shfl_xor64(uint64_t v, int m)
{
    uint32_t lo = __shfl_xor_sync(kFull, (uint32_t)v, m);
    uint32_t hi = __shfl_xor_sync(kFull, (uint32_t)(v >> 32), m);
    return ((uint64_t)hi << 32) | lo;
}

template <int W>
__device__ __forceinline__ bool bit_of(const uint64_t (&m)[W], int i)
{
    bool r = false;
#pragma unroll
    for (int w = 0; w < W; w++)
        if ((i >> 6) == w) r = (m[w] >> (i & 63)) & 1ull;
    return r;
}

// number of set bits of m strictly below position i (0 ≤ i ≤ 64W)
template <int W>
__device__ __forceinline__ int popc_below(const uint64_t (&m)[W], int i)
{
    int c = 0;
#pragma unroll
    for (int w = 0; w < W; w++) {
        int lo = w * 64;
        uint64_t mk = i >= lo + 64 ? ~0ull : (i <= lo ? 0ull : ((1ull << (i - lo)) - 1ull));
        c += __popcll(m[w] & mk);
    }
    return c;
}

// ------------------------------------------------------------ A1: load + validate
// Loads parent/q of tree b (row stride N) into the lane's registers and
// checks the tree (BAD_SIZE / BAD_PARENT / BAD_PROB).  -0.0 → +0.0 (Z9).
template <int NPL>
__device__ __forceinline__ void tree_load_validate(TreeState<NPL> &t, const evict_trees_t &tr,
                                                   const int32_t *__restrict__ parent,
                                                   const float *__restrict__ q,
                                                   const int32_t *__restrict__ n_nodes, int b,
                                                   int N)
{
    const int lane = lane_id();
    const int base = lane * NPL;
    const size_t row = (size_t)b * N;
    if (base < N) {
        if constexpr (NPL == 4) {
            int4 p4 = __ldg(reinterpret_cast<const int4 *>(parent + row + base));
            float4 q4 = __ldg(reinterpret_cast<const float4 *>(q + row + base));
            t.par[0] = p4.x; t.par[1] = p4.y; t.par[2] = p4.z; t.par[3] = p4.w;
            t.q[0] = q4.x; t.q[1] = q4.y; t.q[2] = q4.z; t.q[3] = q4.w;
        } else if constexpr (NPL == 2) {
            int2 p2 = __ldg(reinterpret_cast<const int2 *>(parent + row + base));
            float2 q2 = __ldg(reinterpret_cast<const float2 *>(q + row + base));
            t.par[0] = p2.x; t.par[1] = p2.y;
            t.q[0] = q2.x; t.q[1] = q2.y;
        } else {
            t.par[0] = __ldg(parent + row + base);
            t.q[0] = __ldg(q + row + base);
        }
    } else {
#pragma unroll
        for (int r = 0; r < NPL; r++) { t.par[r] = -1; t.q[r] = 0.f; }
    }
    t.n = n_nodes ? __ldg(n_nodes + b) : N;
    uint32_t st = 0;
    if (t.n < 1 || t.n > N) st = EVICT_TREE_BAD_SIZE;
#pragma unroll
    for (int r = 0; r < NPL; r++) {
        const int i = base + r;
        if (i < t.n) {
            if (i == 0) {
                if (t.par[r] != -1) st |= EVICT_TREE_BAD_PARENT;
            } else {
                if (t.par[r] < 0 || t.par[r] >= i) st |= EVICT_TREE_BAD_PARENT;
                float qq = t.q[r];
                if (!(qq >= 0.f && qq <= 1.f)) st |= EVICT_TREE_BAD_PROB;  // NaN fails both
            }
        }
        if (t.q[r] == 0.f) t.q[r] = 0.f;  // canonicalise -0.0
    }
    t.status = __reduce_or_sync(kFull, st);
    if (t.status & EVICT_TREE_BAD_SIZE) t.status = EVICT_TREE_BAD_SIZE;
}

// cost validation (BAD_COST) for k = 1..n.  cost[k-1] NaN or ≤ 0, or cost[0] = +inf.
template <int NPL>
__device__ __forceinline__ void tree_load_cost(float (&c)[NPL], TreeState<NPL> &t,
                                               const float *__restrict__ cost)
{
    const int base = lane_id() * NPL;
    uint32_t st = 0;
#pragma unroll
    for (int r = 0; r < NPL; r++) {
        const int i = base + r;
        c[r] = 1.f;
        if (i < t.n) {
            c[r] = __ldg(cost + i);
            if (!(c[r] > 0.f)) st |= EVICT_TREE_BAD_COST;           // NaN or ≤ 0
            if (i == 0 && c[r] == __int_as_float(0x7f800000)) st |= EVICT_TREE_BAD_COST;
        }
    }
    t.status |= __reduce_or_sync(kFull, st);
}

// ------------------------------------------------------------ A2: path products
// Synchronous sweeps: every sweep, every node recomputes (score, depth) from
// its parent's value of the previous sweep.  After sweep t every node of
// depth ≤ t holds fl32(Score(parent)·q) computed from its parent's FINAL
// value, i.e. exactly the serial root→leaf product of Eq. 7 (deeper nodes
// hold scratch that later sweeps overwrite).  The loop ends on the first
// sweep that changes nothing: depth+2 sweeps, branch-free per node.
// With SCORES = false only the depth is computed.
template <int NPL, bool SCORES>
__device__ __forceinline__ void tree_levels(TreeState<NPL> &t, WarpSlab<NPL> &sm)
{
    const int base = lane_id() * NPL;
    bool live[NPL];
    int pidx[NPL];
#pragma unroll
    for (int r = 0; r < NPL; r++) {
        const int i = base + r;
        live[r] = (i > 0) && (i < t.n);
        pidx[r] = live[r] ? t.par[r] : 0;
        t.sc[r] = 1.f;
        t.dep[r] = 0;
        sm.sd[i] = make_int2(__float_as_int(1.f), 0);
    }
    __syncwarp();
    while (true) {
        bool changed = false;
        float ns[NPL];
        int nd[NPL];
#pragma unroll
        for (int r = 0; r < NPL; r++) {
            const int2 pv = sm.sd[pidx[r]];
            float sv = t.sc[r];
            if constexpr (SCORES) {
                sv = __fmul_rn(__int_as_float(pv.x), t.q[r]);   // both ≥ +0: never -0
            }
            ns[r] = live[r] ? sv : t.sc[r];
            nd[r] = live[r] ? pv.y + 1 : t.dep[r];
            changed |= (__float_as_int(ns[r]) != __float_as_int(t.sc[r])) | (nd[r] != t.dep[r]);
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < NPL; r++) {
            t.sc[r] = ns[r];
            t.dep[r] = nd[r];
            sm.sd[base + r] = make_int2(__float_as_int(ns[r]), nd[r]);
        }
        __syncwarp();
        if (!__any_sync(kFull, changed)) break;
    }
}

// Selection policy cut (include/evict.h, NEXT-2): does position pos (k = pos + 1)
// qualify?  The caller takes the smallest qualifying position.  COST: the ratio
// bits equal the maximum (Eq. 10); COVERAGE: S_k / S_K ≥ ρ in fp32 IEEE
// division (position n−1 always qualifies); FIXED: k = min(k_fixed, n).
__device__ __forceinline__ bool policy_hit(const evict_policy_t &pol, int pos, int n, uint32_t rb,
                                           uint32_t mx, float s, float SK)
{
    if (pol.kind == EVICT_POLICY_COVERAGE) return pos == n - 1 || __fdiv_rn(s, SK) >= pol.rho;
    if (pol.kind == EVICT_POLICY_FIXED) return pos == (pol.k_fixed < n ? pol.k_fixed : n) - 1;
    return rb == mx;
}

// ------------------------------------------------------------ A3–A5
// Ranks the nodes (bitonic sort), scans S[k], divides by C(k) and takes the
// smallest argmax.  Fills t.kstar/ehat/util/keep; optionally writes order and
// prefix sums (row of N entries).
template <int NPL>
__device__ __forceinline__ void tree_rank_argmax(TreeState<NPL> &t, WarpSlab<NPL> &sm,
                                                 const float (&c)[NPL], int N,
                                                 int32_t *__restrict__ order_row,
                                                 float *__restrict__ prefix_row,
                                                 const evict_policy_t &pol)
{
    constexpr int NMAX = Shape<NPL>::NMAX;
    constexpr int W = Shape<NPL>::W;
    constexpr int W32 = Shape<NPL>::W32;
    const int lane = lane_id();
    const int base = lane * NPL;

    uint64_t key[NPL];
#pragma unroll
    for (int r = 0; r < NPL; r++) {
        const int i = base + r;
        key[r] = (i < t.n) ? (((uint64_t)(~__float_as_uint(t.sc[r])) << 32) | (uint32_t)i) : ~0ull;
    }
    // bitonic sort ascending on key == (score desc, index asc)
#pragma unroll
    for (int k = 2; k <= NMAX; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < NPL) {
#pragma unroll
                for (int r = 0; r < NPL; r++) {
                    const int rp = r ^ j;
                    if (rp > r) {
                        const bool asc = (((base + r) & k) == 0);
                        uint64_t a = key[r], bb = key[rp];
                        const bool sw = asc ? (a > bb) : (a < bb);
                        key[r] = sw ? bb : a;
                        key[rp] = sw ? a : bb;
                    }
                }
            } else {
                const int lj = j / NPL;
#pragma unroll
                for (int r = 0; r < NPL; r++) {
                    const int x = base + r;
                    uint64_t o = shfl_xor64(key[r], lj);
                    const bool take_min = (((x & j) == 0) == ((x & k) == 0));
                    key[r] = take_min ? (o < key[r] ? o : key[r]) : (o > key[r] ? o : key[r]);
                }
            }
        }
    }
    // position p = base + r now holds the p-th ranked node
    float sp[NPL];
    int node[NPL];
#pragma unroll
    for (int r = 0; r < NPL; r++) {
        node[r] = (int)(uint32_t)key[r];   // pads: -1
        sp[r] = __uint_as_float(~(uint32_t)(key[r] >> 32));
        if (base + r < t.n) sm.rank[node[r]] = (uint8_t)(base + r);
    }
    // A4: S[k] = Σ_{j<k} Score(order[j])
    float loc[NPL];
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < NPL; r++) {
        acc = __fadd_rn(acc, sp[r]);
        loc[r] = acc;
    }
    float incl = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        float v = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl = __fadd_rn(incl, v);
    }
    float excl = __shfl_up_sync(kFull, incl, 1);
    if (lane == 0) excl = 0.f;
    float S[NPL];
    uint32_t Rb[NPL];
    uint32_t best = 0;
#pragma unroll
    for (int r = 0; r < NPL; r++) {
        S[r] = __fadd_rn(excl, loc[r]);
        const bool v = base + r < t.n;
        // A5: R[k] = S[k] / C(k), IEEE division (cost +inf ⇒ R = 0)
        float R = v ? __fdiv_rn(S[r], c[r]) : 0.f;
        Rb[r] = v ? __float_as_uint(R) : 0u;   // R ≥ 0 ⇒ bit order = value order
        best = Rb[r] > best ? Rb[r] : best;
    }
    const uint32_t mx = __reduce_max_sync(kFull, best);
    float SK = 0.f;   // S at position n−1 (coverage policy)
    if (pol.kind == EVICT_POLICY_COVERAGE) {
        float sl = 0.f;
#pragma unroll
        for (int r = 0; r < NPL; r++)
            if (base + r == t.n - 1) sl = S[r];
        SK = __shfl_sync(kFull, sl, (t.n - 1) / NPL);
    }
    int rfirst = NPL;
#pragma unroll
    for (int r = NPL - 1; r >= 0; r--)
        if (base + r < t.n && policy_hit(pol, base + r, t.n, Rb[r], mx, S[r], SK)) rfirst = r;
    const unsigned has = __ballot_sync(kFull, rfirst < NPL);
    const int wl = __ffs(has) - 1;               // smallest k wins ties (Z3)
    const int rf = __shfl_sync(kFull, rfirst, wl);
    float Sk = 0.f, Rk = 0.f;
#pragma unroll
    for (int r = 0; r < NPL; r++)
        if (r == rf) { Sk = S[r]; Rk = __uint_as_float(Rb[r]); }
    t.ehat = __shfl_sync(kFull, Sk, wl);
    t.util = __shfl_sync(kFull, Rk, wl);
    t.kstar = wl * NPL + rf + 1;

    if ((order_row != nullptr || prefix_row != nullptr) && base < N) {
#pragma unroll
        for (int r = 0; r < NPL; r++) {
            if (order_row) order_row[base + r] = (base + r < t.n) ? node[r] : -1;
            if (prefix_row) prefix_row[base + r] = (base + r < t.n) ? S[r] : 0.f;
        }
    }
    __syncwarp();
    // keep = order[0 .. k*): node i kept ⇔ rank(i) < k*
    uint32_t local = 0;
#pragma unroll
    for (int r = 0; r < NPL; r++) {
        const int i = base + r;
        if (i < t.n && sm.rank[i] < t.kstar) local |= 1u << ((i & 31));
    }
    uint32_t wd[2 * W];
#pragma unroll
    for (int w = 0; w < 2 * W; w++) {
        uint32_t mine = (w < W32 && (base >> 5) == w) ? local : 0u;
        wd[w] = (w < W32) ? __reduce_or_sync(kFull, mine) : 0u;
    }
#pragma unroll
    for (int w = 0; w < W; w++) t.keep[w] = (uint64_t)wd[2 * w] | ((uint64_t)wd[2 * w + 1] << 32);
}

// ------------------------------------------------------------ A6: verify tree
// Requires t.par/t.dep/t.n and t.keep.  Checks the keep set (BAD_KEEP) and
// returns k = |keep| (0 on error).  Row outputs are written by emit_build.
template <int NPL>
__device__ __forceinline__ int tree_check_keep(TreeState<NPL> &t)
{
    constexpr int W = Shape<NPL>::W;
    const int base = lane_id() * NPL;
    uint32_t bad = 0;
#pragma unroll
    for (int r = 0; r < NPL; r++) {
        const int i = base + r;
        const bool kp = bit_of<W>(t.keep, i);
        if (i >= t.n && kp) bad = 1;
        if (i == 0 && !kp) bad = 1;
        if (i > 0 && i < t.n && kp && !bit_of<W>(t.keep, t.par[r])) bad = 1;
    }
    if (__any_sync(kFull, bad)) t.status |= EVICT_TREE_BAD_KEEP;
    int k = 0;
#pragma unroll
    for (int w = 0; w < W; w++) k += __popcll(t.keep[w]);
    return k;
}

template <int NPL>
__device__ __forceinline__ void tree_build_emit(const TreeState<NPL> &t, WarpSlab<NPL> &sm, int k,
                                                int b, int N, int off, int pos_off,
                                                int32_t *__restrict__ kept_index,
                                                int32_t *__restrict__ retrieve_index,
                                                int32_t *__restrict__ positions,
                                                int32_t *__restrict__ next_token,
                                                int32_t *__restrict__ next_sibling,
                                                uint64_t *__restrict__ tree_mask)
{
    constexpr int W = Shape<NPL>::W;
    const int lane = lane_id();
    const int base = lane * NPL;
    bool kp[NPL];
    int slot[NPL], pslot[NPL];
    int maxd = 0;
#pragma unroll
    for (int r = 0; r < NPL; r++) {
        const int i = base + r;
        kp[r] = i < t.n && bit_of<W>(t.keep, i);
        slot[r] = popc_below<W>(t.keep, i);
        pslot[r] = (i > 0 && kp[r]) ? popc_below<W>(t.keep, t.par[r]) : -1;
        if (kp[r]) {
            maxd = t.dep[r] > maxd ? t.dep[r] : maxd;
            sm.klist[slot[r]] = (uint8_t)i;
        }
    }
    maxd = __reduce_max_sync(kFull, maxd);
    // ancestor-or-self rows, one tree level at a time
    for (int d = 0; d <= maxd; d++) {
#pragma unroll
        for (int r = 0; r < NPL; r++) {
            if (kp[r] && t.dep[r] == d) {
#pragma unroll
                for (int w = 0; w < W; w++) {
                    uint64_t v = (d == 0) ? 0ull : sm.row[pslot[r]][w];
                    if ((slot[r] >> 6) == w) v |= 1ull << (slot[r] & 63);
                    sm.row[slot[r]][w] = v;
                }
            }
        }
        __syncwarp();
    }
    for (int s = lane; s < k; s += 32)
#pragma unroll
        for (int w = 0; w < W; w++) sm.child[s][w] = 0ull;
    __syncwarp();
#pragma unroll
    for (int r = 0; r < NPL; r++)
        if (kp[r] && pslot[r] >= 0)
            atomicOr(reinterpret_cast<unsigned long long *>(&sm.child[pslot[r]][slot[r] >> 6]),
                     1ull << (slot[r] & 63));
    __syncwarp();
#pragma unroll
    for (int r = 0; r < NPL; r++) {
        if (!kp[r]) continue;
        const int s = slot[r];
        const int rowi = off + s;
        int nt = -1, ns = -1;
#pragma unroll
        for (int w = W - 1; w >= 0; w--) {
            uint64_t cm = sm.child[s][w];
            if (cm) nt = w * 64 + __ffsll((long long)cm) - 1;
        }
        if (pslot[r] >= 0) {
#pragma unroll
            for (int w = W - 1; w >= 0; w--) {
                uint64_t cm = sm.child[pslot[r]][w];
                const int lo = w * 64;
                uint64_t above = (s + 1 <= lo) ? ~0ull : (s + 1 >= lo + 64 ? 0ull : (~0ull << (s + 1 - lo)));
                cm &= above;
                if (cm) ns = lo + __ffsll((long long)cm) - 1;
            }
        }
        const int i = base + r;
        if (kept_index) kept_index[rowi] = i;
        if (retrieve_index) retrieve_index[rowi] = b * N + i;
        if (positions) positions[rowi] = pos_off + t.dep[r];
        if (next_token) next_token[rowi] = nt;
        if (next_sibling) next_sibling[rowi] = ns;
        if (tree_mask) {
#pragma unroll
            for (int w = 0; w < W; w++) tree_mask[(size_t)rowi * W + w] = sm.row[s][w];
        }
    }
}

// ------------------------------------------------------------ A7: expert union
// Lane `lane` owns layers l = lane + 32c.  For every kept node (slot order,
// sm.klist), the node's routing row is read and OR-ed into the lane's
// per-layer EW-word expert bitsets; counts are __popcll of the bitsets.
template <int EW>
struct LayerBits {
    uint32_t w[2 * EW];  // 32-bit words: expert e ⇔ bit e%32 of word e/32
};

// 1 << s with PTX clamp semantics: 0 for any s ≥ 32 (s is unsigned, so a
// "negative" s - 32j also gives 0).  One SHF per call.
__device__ __forceinline__ uint32_t shl_clamp(uint32_t s)
{
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(1u), "r"(s));
    return r;
}

// OR expert e into the layer's bitset: word j gets 1 << (e - 32j), which is
// non-zero only for the one word that holds e (no per-word compare/select).
template <int EW>
__device__ __forceinline__ void or_id(LayerBits<EW> &bs, uint32_t e, uint32_t &bad, uint32_t E)
{
    bad |= (e >= E);
#pragma unroll
    for (int j = 0; j < 2 * EW; j++) bs.w[j] |= shl_clamp(e - 32u * j);
}

// Four u8 ids packed in one word (E == 128 fast path: the id is bad iff bit 7 is set).
template <int EW>
__device__ __forceinline__ void or_ids_u8x4(LayerBits<EW> &bs, uint32_t wv, uint32_t &bad, uint32_t E)
{
    if (E == 128) {
        bad |= wv & 0x80808080u;
    } else {
#pragma unroll
        for (int s = 0; s < 4; s++) bad |= (__byte_perm(wv, 0, 0x4440 | s) >= E);
    }
#pragma unroll
    for (int s = 0; s < 4; s++) {
        const uint32_t e = __byte_perm(wv, 0, 0x4440 | s);
#pragma unroll
        for (int j = 0; j < 2 * EW; j++) bs.w[j] |= shl_clamp(e - 32u * j);
    }
}

// IDF: 1 = u8 ids, 4 = i32 ids, 8 = masks.  KT: compile-time K (0 = runtime).
// Generic layout: lane `lane` owns layers l = lane + 32c (any K, any E ≤ 256).
template <int NPL, int IDF, int KT, int EW, int CL>
__device__ __forceinline__ void tree_union_generic(uint32_t &status, const uint8_t *__restrict__ klist, int k,
                                           int b, int N, int L, int K, int E, int idb,
                                           const void *__restrict__ ids,
                                           int32_t *__restrict__ union_count,
                                           int32_t *__restrict__ union_total,
                                           uint64_t *__restrict__ union_bits,
                                           int64_t *__restrict__ expert_hist)
{
    const int lane = lane_id();
    LayerBits<EW> bs[CL];
#pragma unroll
    for (int c = 0; c < CL; c++)
#pragma unroll
        for (int w = 0; w < 2 * EW; w++) bs[c].w[w] = 0u;
    uint32_t bad = 0;
    const int Kr = KT ? KT : K;
    if (!status) {
        constexpr int U = 4;  // rows in flight per lane
        for (int j0 = 0; j0 < k; j0 += U) {
            if constexpr (IDF == 1 && KT == 8) {
                uint2 v[U][CL];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int j = j0 + u;
                    const int node = j < k ? klist[j] : 0;
                    const uint8_t *rowp = (const uint8_t *)ids + ((size_t)b * N + node) * L * 8;
#pragma unroll
                    for (int c = 0; c < CL; c++) {
                        const int l = lane + 32 * c;
                        v[u][c] = (j < k && l < L) ? __ldg(reinterpret_cast<const uint2 *>(rowp + l * 8))
                                                   : make_uint2(0, 0);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++)
#pragma unroll
                    for (int c = 0; c < CL; c++) {
                        if (j0 + u >= k || lane + 32 * c >= L) continue;
#pragma unroll
                        or_ids_u8x4<EW>(bs[c], v[u][c].x, bad, E);
                        or_ids_u8x4<EW>(bs[c], v[u][c].y, bad, E);
                    }
            } else if constexpr (IDF == 4 && KT == 8) {
                int4 v[U][CL][2];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int j = j0 + u;
                    const int node = j < k ? klist[j] : 0;
                    const int32_t *rowp = (const int32_t *)ids + ((size_t)b * N + node) * L * 8;
#pragma unroll
                    for (int c = 0; c < CL; c++) {
                        const int l = lane + 32 * c;
                        const bool ok = j < k && l < L;
#pragma unroll
                        for (int h = 0; h < 2; h++)
                            v[u][c][h] = ok ? __ldg(reinterpret_cast<const int4 *>(rowp + l * 8) + h)
                                            : make_int4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++)
#pragma unroll
                    for (int c = 0; c < CL; c++) {
                        if (j0 + u >= k || lane + 32 * c >= L) continue;
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            or_id<EW>(bs[c], (uint32_t)v[u][c][h].x, bad, E);
                            or_id<EW>(bs[c], (uint32_t)v[u][c][h].y, bad, E);
                            or_id<EW>(bs[c], (uint32_t)v[u][c][h].z, bad, E);
                            or_id<EW>(bs[c], (uint32_t)v[u][c][h].w, bad, E);
                        }
                    }
            } else if constexpr (IDF >= 8) {
                const int EWr = (E + 63) >> 6;   // row stride in 64-bit words
                uint64_t v[U][CL][EW];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int j = j0 + u;
                    const int node = j < k ? klist[j] : 0;
                    const uint64_t *rowp = (const uint64_t *)ids + ((size_t)b * N + node) * L * EWr;
#pragma unroll
                    for (int c = 0; c < CL; c++) {
                        const int l = lane + 32 * c;
                        const bool ok = j < k && l < L;
                        if (EW == 2 && EWr == 2) {
                            ulonglong2 x = ok ? __ldg(reinterpret_cast<const ulonglong2 *>(rowp + l * 2))
                                              : make_ulonglong2(0, 0);
                            v[u][c][0] = x.x;
                            v[u][c][1] = x.y;
                        } else {
#pragma unroll
                            for (int w = 0; w < EW; w++)
                                v[u][c][w] = (ok && w < EWr) ? __ldg(rowp + l * EWr + w) : 0ull;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++)
#pragma unroll
                    for (int c = 0; c < CL; c++)
#pragma unroll
                        for (int w = 0; w < EW; w++) {
                            bs[c].w[2 * w] |= (uint32_t)v[u][c][w];
                            bs[c].w[2 * w + 1] |= (uint32_t)(v[u][c][w] >> 32);
                        }
            } else {
                // generic K (any ≤ 16), u8 or i32: scalar loads
#pragma unroll 1
                for (int u = 0; u < U; u++) {
                    const int j = j0 + u;
                    if (j >= k) break;
                    const int node = klist[j];
#pragma unroll
                    for (int c = 0; c < CL; c++) {
                        const int l = lane + 32 * c;
                        if (l >= L) continue;
                        const size_t o = (((size_t)b * N + node) * L + l) * Kr;
                        for (int x = 0; x < Kr; x++) {
                            uint32_t e = idb == 1 ? (uint32_t)__ldg((const uint8_t *)ids + o + x)
                                                  : (uint32_t)__ldg((const int32_t *)ids + o + x);
                            or_id<EW>(bs[c], e, bad, E);
                        }
                    }
                }
            }
        }
        if constexpr (IDF >= 8) {
            // bits at or above E are not experts
#pragma unroll
            for (int c = 0; c < CL; c++)
#pragma unroll
                for (int w = 0; w < 2 * EW; w++) {
                    const int lo = w * 32;
                    uint32_t valid = E >= lo + 32 ? ~0u : (E <= lo ? 0u : ((1u << (E - lo)) - 1u));
                    if (bs[c].w[w] & ~valid) bad = 1;
                }
        }
        if (__any_sync(kFull, bad)) status |= EVICT_TREE_BAD_EXPERT;
    }
    int tot = 0;
    const bool zero = status != 0;
#pragma unroll
    for (int c = 0; c < CL; c++) {
        const int l = lane + 32 * c;
        if (l >= L) continue;
        int cnt = 0;
#pragma unroll
        for (int w = 0; w < 2 * EW; w++) {
            if (zero) bs[c].w[w] = 0u;
            cnt += __popc(bs[c].w[w]);
        }
        tot += cnt;
        union_count[(size_t)b * L + l] = cnt;
        const int EWr = (E + 63) / 64;
        if (union_bits) {
#pragma unroll
            for (int w = 0; w < EW; w++)
                if (w < EWr)
                    union_bits[((size_t)b * L + l) * EWr + w] =
                        (uint64_t)bs[c].w[2 * w] | ((uint64_t)bs[c].w[2 * w + 1] << 32);
        }
        if (expert_hist && !zero) {
#pragma unroll
            for (int w = 0; w < 2 * EW; w++) {
                uint32_t m = bs[c].w[w];
                while (m) {
                    const int e = w * 32 + __ffs(m) - 1;
                    m &= m - 1;
                    atomicAdd(reinterpret_cast<unsigned long long *>(expert_hist + (size_t)l * E + e), 1ull);
                }
            }
        }
    }
    tot = __reduce_add_sync(kFull, tot);
    if (union_total && lane == 0) union_total[b] = tot;
}

}  // namespace evict

namespace evict {

// Fast layout: a layer's routing row splits into P parts (4 ids = half of a
// top-8 row, or one 64-bit mask word); slot = l·P + part is owned by lane
// slot % 32 in round slot / 32, so every load instruction of the warp reads
// 32 consecutive parts (128 B of u8 ids, 512 B of i32 ids, 256 B of masks) and
// no lane idles.  Parts of one layer sit in adjacent lanes and are merged with
// __shfl_xor_sync at the end.  R = register rounds (≥ ceil(L·P/32)).
template <int NPL, int IDF, int EW, int R>
__device__ __forceinline__ void tree_union_fast(uint32_t &status, const uint8_t *__restrict__ klist, int k,
                                                int b, int N, int L, int E,
                                                const void *__restrict__ ids,
                                                int32_t *__restrict__ union_count,
                                                int32_t *__restrict__ union_total,
                                                uint64_t *__restrict__ union_bits,
                                                int64_t *__restrict__ expert_hist)
{
    constexpr bool MASK = IDF == 8;
    constexpr int NW = MASK ? 2 : 2 * EW;      // 32-bit words held per slot
    const int lane = lane_id();
    const int EWr = (E + 63) >> 6;
    const int P = MASK ? EWr : 2;              // parts per layer (1, 2 or 4)
    const int lp = P == 1 ? 0 : (P == 2 ? 1 : 2);   // log2 P (shifts, not divisions)
    const int S = L * P;                       // slots
    uint32_t bs[R][NW];
#pragma unroll
    for (int c = 0; c < R; c++)
#pragma unroll
        for (int w = 0; w < NW; w++) bs[c][w] = 0u;
    uint32_t bad = 0;
    if (!status) {
        // bytes per node row: u8 L·8, i32 L·32, mask L·EWr·8
        const size_t row_elems = MASK ? (size_t)S : (size_t)L * 8;
        constexpr int U = 4;                    // node rows in flight
        for (int j0 = 0; j0 < k; j0 += U) {
            if constexpr (IDF == 1) {
                uint32_t v[U][R];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int j = j0 + u;
                    const uint32_t *rowp = reinterpret_cast<const uint32_t *>(
                        (const uint8_t *)ids + ((size_t)b * N + (j < k ? klist[j] : 0)) * row_elems);
#pragma unroll
                    for (int c = 0; c < R; c++) {
                        const int sl = lane + 32 * c;
                        v[u][c] = (j < k && sl < S) ? __ldg(rowp + sl) : 0u;
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++)
#pragma unroll
                    for (int c = 0; c < R; c++)
                        if (j0 + u < k && lane + 32 * c < S) {
                            LayerBits<EW> lb;
#pragma unroll
                            for (int w = 0; w < NW; w++) lb.w[w] = bs[c][w];
                            or_ids_u8x4<EW>(lb, v[u][c], bad, E);
#pragma unroll
                            for (int w = 0; w < NW; w++) bs[c][w] = lb.w[w];
                        }
            } else if constexpr (IDF == 4) {
                int4 v[U][R];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int j = j0 + u;
                    const int4 *rowp = reinterpret_cast<const int4 *>(
                        (const int32_t *)ids + ((size_t)b * N + (j < k ? klist[j] : 0)) * row_elems);
#pragma unroll
                    for (int c = 0; c < R; c++) {
                        const int sl = lane + 32 * c;
                        v[u][c] = (j < k && sl < S) ? __ldg(rowp + sl) : make_int4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++)
#pragma unroll
                    for (int c = 0; c < R; c++)
                        if (j0 + u < k && lane + 32 * c < S) {
                            LayerBits<EW> lb;
#pragma unroll
                            for (int w = 0; w < NW; w++) lb.w[w] = bs[c][w];
                            or_id<EW>(lb, (uint32_t)v[u][c].x, bad, E);
                            or_id<EW>(lb, (uint32_t)v[u][c].y, bad, E);
                            or_id<EW>(lb, (uint32_t)v[u][c].z, bad, E);
                            or_id<EW>(lb, (uint32_t)v[u][c].w, bad, E);
#pragma unroll
                            for (int w = 0; w < NW; w++) bs[c][w] = lb.w[w];
                        }
            } else {
                // a batch past k re-reads node k-1 (OR is idempotent); node offsets are
                // 32-bit byte offsets onto this lane's pointer
                uint2 v[U][R];
                const uint2 *lanep = reinterpret_cast<const uint2 *>(ids) + (size_t)b * N * row_elems + lane;
                const uint32_t rowb = (uint32_t)row_elems * 8u;
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const uint32_t node = klist[min(j0 + u, k - 1)];
                    const uint2 *rowp = reinterpret_cast<const uint2 *>(
                        reinterpret_cast<const char *>(lanep) + node * rowb);
#pragma unroll
                    for (int c = 0; c < R; c++) {
                        const int sl = lane + 32 * c;
                        v[u][c] = (sl < S) ? __ldg(rowp + 32 * c) : make_uint2(0u, 0u);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++)
#pragma unroll
                    for (int c = 0; c < R; c++) {
                        bs[c][0] |= v[u][c].x;
                        bs[c][1] |= v[u][c].y;
                    }
            }
        }
        if constexpr (MASK) {
            if (E & 63) {   // bits at or above E are not experts
#pragma unroll
                for (int c = 0; c < R; c++) {
                    const int sl = lane + 32 * c;
                    if (sl < S && (sl & (P - 1)) == P - 1) {
                        const int lo = (P - 1) * 64, rem = E - lo;
                        const uint64_t m = (uint64_t)bs[c][0] | ((uint64_t)bs[c][1] << 32);
                        if (m & ~((1ull << rem) - 1ull)) bad = 1;
                    }
                }
            }
        }
        if (__any_sync(kFull, bad)) status |= EVICT_TREE_BAD_EXPERT;
    }
    const bool zero = status != 0;
    int tot = 0;
#pragma unroll
    for (int c = 0; c < R; c++) {
        const int sl = lane + 32 * c;
        const int l = sl >> lp, h = sl & (P - 1);
        if (zero) {
#pragma unroll
            for (int w = 0; w < NW; w++) bs[c][w] = 0u;
        }
        int cnt;
        if constexpr (!MASK) {
            // merge the two halves of the layer (adjacent lanes)
#pragma unroll
            for (int w = 0; w < NW; w++) bs[c][w] |= __shfl_xor_sync(kFull, bs[c][w], 1);
            cnt = 0;
#pragma unroll
            for (int w = 0; w < NW; w++) cnt += __popc(bs[c][w]);
        } else {
            cnt = __popc(bs[c][0]) + __popc(bs[c][1]);
            if (P >= 2) cnt += __shfl_xor_sync(kFull, cnt, 1);
            if (P >= 4) cnt += __shfl_xor_sync(kFull, cnt, 2);
        }
        if (sl >= S) continue;
        if (h == 0) {
            union_count[(size_t)b * L + l] = cnt;
            tot += cnt;
        }
        // this lane owns 64-bit words w with w % P == h (ids: of the merged set)
        uint64_t *dst = union_bits ? union_bits + ((size_t)b * L + l) * EWr : nullptr;
        if constexpr (!MASK) {
#pragma unroll
            for (int w = 0; w < EW; w++) {
                if (w < EWr && (w & 1) == h) {
                    const uint64_t m = (uint64_t)bs[c][2 * w] | ((uint64_t)bs[c][2 * w + 1] << 32);
                    if (dst) dst[w] = m;
                    if (expert_hist && !zero) {
                        uint64_t mm = m;
                        while (mm) {
                            const int e = w * 64 + __ffsll((long long)mm) - 1;
                            mm &= mm - 1;
                            atomicAdd(reinterpret_cast<unsigned long long *>(expert_hist + (size_t)l * E + e), 1ull);
                        }
                    }
                }
            }
        } else {
            const uint64_t m = (uint64_t)bs[c][0] | ((uint64_t)bs[c][1] << 32);
            if (dst) dst[h] = m;
            if (expert_hist && !zero) {
                uint64_t mm = m;
                while (mm) {
                    const int e = h * 64 + __ffsll((long long)mm) - 1;
                    mm &= mm - 1;
                    atomicAdd(reinterpret_cast<unsigned long long *>(expert_hist + (size_t)l * E + e), 1ull);
                }
            }
        }
    }
    tot = __reduce_add_sync(kFull, tot);
    if (union_total && lane == 0) union_total[b] = tot;
}

// Top-8 ids (u8 or i32) via per-warp shared-memory expert flags.  A layer's
// 8 ids split into two 4-id halves; slot = 2l + half; lane `lane` owns slots
// lane + 32c (round c < R, 16 layers per round).  In round c's flag block the
// byte of (layer j' = lane/2, expert e) lives in 32-bit word (e/4)·16 + j' at
// byte e%4, so a store's bank is 16·((e/4)&1) + j': lanes of different layers
// never collide, only the two halves of one layer can (half the time).  One
// byte store per id (no read-modify-write, duplicates idempotent); then each
// lane counts its half (popc of 0/1 bytes), optionally packs the bits, and
// clears its words.  Region: R·Epad·16 bytes per warp.
template <int NPL, int IDF, int R, bool E128, bool BITS>
__device__ __forceinline__ void tree_union_flags(uint32_t &status, const uint8_t *__restrict__ klist,
                                                 int k, int b, int N, int L, int E,
                                                 const void *__restrict__ ids, uint8_t *flags,
                                                 int Epad, int32_t *__restrict__ union_count,
                                                 int32_t *__restrict__ union_total,
                                                 uint64_t *__restrict__ union_bits)
{
    const int lane = lane_id();
    const int S = 2 * L;
    const int jp = lane >> 1, h = lane & 1;
    const int blk = Epad * 16;                      // bytes per round block
    const int G4 = Epad >> 2;                       // flag words per layer
    const int HW = G4 >> 1;                         // words per half
    const int EWr = (E + 63) >> 6;
    const size_t row = (size_t)L * 8;               // ids per node row
    const uint8_t *tree_u8 = (const uint8_t *)ids + (size_t)b * N * row;
    const int32_t *tree_i32 = (const int32_t *)ids + (size_t)b * N * row;
    uint32_t bad = 0;
    const bool run = status == 0;
    if (run) {
        constexpr int U = 4;
        for (int j0 = 0; j0 < k; j0 += U) {
            if constexpr (IDF == 1) {
                uint32_t v[U][R];
                // warp-uniform fast path: a full batch of U nodes and full 32-slot rounds
                // need no per-store guards (no divergence bookkeeping in the hot loop)
                const bool full = (j0 + U <= k) && ((S & 31) == 0);
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int j = j0 + u;
                    const uint32_t *rowp = reinterpret_cast<const uint32_t *>(
                        tree_u8 + (uint32_t)klist[j < k ? j : 0] * (uint32_t)row);
#pragma unroll
                    for (int c = 0; c < R; c++) {
                        const int sl = lane + 32 * c;
                        v[u][c] = (j < k && sl < S) ? __ldg(rowp + sl) : 0u;
                    }
                }
                if (E128 && full) {
#pragma unroll
                    for (int u = 0; u < U; u++)
#pragma unroll
                        for (int c = 0; c < R; c++) {
                            if (32 * c >= S) continue;          // uniform: round absent
                            uint8_t *fl = flags + c * blk + jp * 4;
                            const uint32_t wv = v[u][c];
                            bad |= wv & 0x80808080u;
                            const uint32_t wm = wv & 0x7F7F7F7Fu;
#pragma unroll
                            for (int q = 0; q < 4; q++) {
                                const uint32_t e = __byte_perm(wm, 0, 0x4440 | q);
                                fl[e * 16u - (e & 3u) * 15u] = 1;
                            }
                        }
                    continue;
                }
#pragma unroll
                for (int u = 0; u < U; u++)
#pragma unroll
                    for (int c = 0; c < R; c++) {
                        if (j0 + u < k && lane + 32 * c < S) {
                            uint8_t *fl = flags + c * blk + jp * 4;
                            uint32_t wv = v[u][c];
                            if constexpr (E128) {
                                bad |= wv & 0x80808080u;
                                wv &= 0x7F7F7F7Fu;
#pragma unroll
                                for (int q = 0; q < 4; q++) {
                                    const uint32_t e = __byte_perm(wv, 0, 0x4440 | q);
                                    fl[e * 16u - (e & 3u) * 15u] = 1;
                                }
                            } else {
#pragma unroll
                                for (int q = 0; q < 4; q++) {
                                    const uint32_t e = __byte_perm(wv, 0, 0x4440 | q);
                                    if (e < (uint32_t)E) fl[e * 16u - (e & 3u) * 15u] = 1;
                                    else bad = 1;
                                }
                            }
                        }
                    }
            } else {
                int4 v[U][R];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int j = j0 + u;
                    const int4 *rowp = reinterpret_cast<const int4 *>(
                        tree_i32 + (uint32_t)(j < k ? klist[j] : 0) * (uint32_t)row);
#pragma unroll
                    for (int c = 0; c < R; c++) {
                        const int sl = lane + 32 * c;
                        v[u][c] = (j < k && sl < S) ? __ldg(rowp + sl) : make_int4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++)
#pragma unroll
                    for (int c = 0; c < R; c++) {
                        if (j0 + u < k && lane + 32 * c < S) {
                            uint8_t *fl = flags + c * blk + jp * 4;
                            const uint32_t e4[4] = {(uint32_t)v[u][c].x, (uint32_t)v[u][c].y,
                                                    (uint32_t)v[u][c].z, (uint32_t)v[u][c].w};
#pragma unroll
                            for (int q = 0; q < 4; q++) {
                                const uint32_t e = e4[q];
                                if (e < (uint32_t)E) fl[e * 16u - (e & 3u) * 15u] = 1;
                                else bad = 1;
                            }
                        }
                    }
            }
        }
    }
    __syncwarp();
    const bool anybad = run && __any_sync(kFull, bad);
    if (anybad) status |= EVICT_TREE_BAD_EXPERT;
    const bool zero = status != 0;
    int tot = 0;
#pragma unroll
    for (int c = 0; c < R; c++) {
        const int sl = lane + 32 * c;
        const bool in = sl < S;
        const int l = sl >> 1;
        const uint32_t *fw = reinterpret_cast<const uint32_t *>(flags + c * blk);
        uint32_t *fwm = reinterpret_cast<uint32_t *>(flags + c * blk);
        int cnt = 0;
        uint64_t bits[2] = {0ull, 0ull};
        if (run && in) {        // flags were written only for good-status trees
            for (int qq = 0; qq < HW; qq++) {
                const int g = h * HW + ((qq + h) & (HW - 1));   // rotated: halves hit different banks
                const uint32_t x = fw[g * 16 + jp];
                cnt += __popc(x);
                if constexpr (BITS) {
                    const uint32_t nib = (x & 1u) | ((x >> 7) & 2u) | ((x >> 14) & 4u) | ((x >> 21) & 8u);
                    const int pos = (g - h * HW) * 4;
                    bits[pos >> 6] |= (uint64_t)nib << (pos & 63);
                }
                fwm[g * 16 + jp] = 0u;
            }
        }
        cnt += __shfl_xor_sync(kFull, cnt, 1);
        if (!in) continue;
        if (zero) { cnt = 0; bits[0] = bits[1] = 0ull; }
        if (h == 0) {
            union_count[(size_t)b * L + l] = cnt;
            tot += cnt;
        }
        if constexpr (BITS) {
            const int w0 = h * (HW >> 4);                // first 64-bit word of this half
#pragma unroll
            for (int w = 0; w < 2; w++)
                if (w < (HW >> 4) && w0 + w < EWr) union_bits[((size_t)b * L + l) * EWr + w0 + w] = bits[w];
        }
    }
    __syncwarp();
    tot = __reduce_add_sync(kFull, tot);
    if (union_total && lane == 0) union_total[b] = tot;
}

// Flag bytes per warp for the top-K id union: the expert-major block below for
// E ≤ 128 (any L ≤ 128, in passes of 64 layers), the older layer-round blocks
// (R · 256 · 16 bytes) for E > 128.
__host__ __device__ inline int union_flag_bytes(int L, int E)
{
    (void)L;
    (void)E;
    return 8192;   // E ≤ 128: 128 experts × 64 layer bytes; E ≤ 256: 256 experts × 32 layer bytes
}

// Top-K ids (u8 or i32, E ≤ 128) via an expert-major shared-memory flag block
// (Eq. 5: |∪_{v kept} TopK_l(v)| per layer l).
//
// Slot = 2l + half (a layer's 8 ids split into two 4-id halves); lane owns
// slots lane + 32c (round c).  Layer l lives in pass l/64, byte (l/16)%4 of
// 32-bit word e·16 + (l%16) for expert e:
//     flag(l, e) at byte  e·64 + 4·(l%16) + (l/16)%4
// so a store's address is one LEA of the id (e << 6) onto a per-lane base, and
// its bank is 16·(e&1) + l%16: lanes of different layers never collide, only
// the two halves of one layer can.  One byte store per id (no read-modify-
// write; duplicates idempotent).  Read-back: lane (q = lane&3, p8 = lane>>2)
// adds 16 uint4 words bytewise (expert e = p8 + 8i, layers-words 4q..4q+3) and
// zeroes them; an xor-shuffle over p8 leaves per-byte counts ≤ 128, i.e. the
// union size of 16 layers per word.  Region: 8 KB per warp.
__device__ __forceinline__ void sts_u8(uint32_t addr, uint32_t v)
{
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ uint4 lds_v4(uint32_t addr)
{
    uint4 x;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "r"(addr));
    return x;
}
__device__ __forceinline__ void sts_v4_zero(uint32_t addr)
{
    asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(addr), "r"(0u));
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// W256 (128 < E ≤ 256, Ling-flash-2.0): the same scheme with 32-byte expert rows — passes
// of 32 layers, flag(l, e) at byte e·32 + 4·(l%8) + (l/8)%4; the read-back widens the byte
// sums to 16-bit lanes before the cross-lane reduction (a layer can hold all 256 experts).
// UB: nodes per load batch for u8 ids (4 for throughput; 8 in the serving-batch kernel, where one
// DRAM round trip covers a typical tree's kept rows and registers are not scarce)
template <int IDF, int R, bool E128, bool BITS, bool W256 = false, int UB = 4>
__device__ __forceinline__ void tree_union_flags64(uint32_t &status, const uint8_t *__restrict__ klist, int k,
                                                   int b, int N, int L, int E, const void *__restrict__ ids,
                                                   uint8_t *flags, int32_t *__restrict__ union_count,
                                                   int32_t *__restrict__ union_total,
                                                   uint64_t *__restrict__ union_bits, int *epoch = nullptr,
                                                   uint32_t *lsum = nullptr)
{
    // lsum (single-pass E ≤ 128 layout only): lsum[hb] += this lane's count of layer
    // 16·(bsel + 2·hb) + 4·(lane & 3) + (lane >> 2 & 3), bsel = lane >> 4 (A9 per-layer sums of
    // good trees, folded into the fused launch)
    static_assert(IDF == 1 || IDF == 4, "flag union takes u8 or i32 ids");
    constexpr int RPP = W256 ? 2 : 4;                  // 16-layer rounds per pass
    constexpr int PASSES = (R + RPP - 1) / RPP;
    constexpr int ESH = W256 ? 5 : 6;                  // log2 bytes per expert row
    // Marker mode (single pass, no bit rows, caller keeps `epoch`): tree t stores the
    // byte 1 << (t mod 4) and counts only that bit, so the block is cleared once per 4
    // trees instead of after every tree (a byte holds its last writer's marker; the 4
    // markers of a window are distinct).  Otherwise: store 1, clear after each read.
    const bool mark = PASSES == 1 && !BITS && epoch != nullptr;
    const int ep = mark ? *epoch : 0;
    const uint32_t marker = 1u << ep;
    constexpr int RP = R < RPP ? R : RPP;              // rounds per pass
    constexpr int U = IDF == 1 ? UB : 1;               // nodes per load batch (i32 rows are 4x wider)
    const int lane = lane_id();
    const int S = 2 * L;
    const uint32_t row = (uint32_t)S;                  // 4-id units per node row
    const uint32_t fbase = (uint32_t)__cvta_generic_to_shared(flags);
    // + (e << ESH) + round byte: layer 16c + j' (j' = lane/2) sits at byte 4·(l%16) + l/16 (E ≤ 128)
    // or 4·(l%8) + l/8 (W256)
    const uint32_t jp = (uint32_t)(lane >> 1);
    const uint32_t lbase = W256 ? fbase + 4u * (jp & 7u) + (jp >> 3) : fbase + 4u * jp;
    constexpr uint32_t CSTEP = W256 ? 2u : 1u;         // byte step of one round
    uint32_t bad = 0;
    const bool run = status == 0;
    int tot = 0;
    uint32_t lcnt[2] = {0u, 0u};
#pragma unroll 1
    for (int pass = 0; pass < PASSES; pass++) {
        if (run) {
            // A batch past k re-reads node k-1 (cheap L1 hits) but stores nothing for it; a slot
            // past 2L stores e = 0 into a layer ≥ L, whose byte is never counted (the read-back
            // still clears it).
            // this lane's first unit of the pass in the tree's node-row block; a node adds
            // node·row units (32-bit: node < 128, row ≤ 256) and a round 32 units
            const uint32_t *lane_u32 = reinterpret_cast<const uint32_t *>(ids) + (size_t)b * N * row + lane + 32 * RPP * pass;
            const int4 *lane_i4 = reinterpret_cast<const int4 *>(ids) + (size_t)b * N * row + lane + 32 * RPP * pass;
            // load a batch of U kept nodes' row parts (a batch past k re-reads node k-1)
            auto load_batch = [&](int j0, uint32_t (&v)[U][RP][IDF]) {
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const uint32_t node = klist[min(j0 + u, k - 1)];
#pragma unroll
                    for (int cc = 0; cc < RP; cc++) {
                        const bool ok = lane + 32 * (RPP * pass + cc) < S;
                        if constexpr (IDF == 1) {
                            const uint32_t *rp = reinterpret_cast<const uint32_t *>(
                                reinterpret_cast<const char *>(lane_u32) + node * (4u * row));
                            v[u][cc][0] = ok ? __ldg(rp + 32 * cc) : 0u;
                        } else {
                            const int4 *rp = reinterpret_cast<const int4 *>(
                                reinterpret_cast<const char *>(lane_i4) + node * (16u * row));
                            const int4 x = ok ? __ldg(rp + 32 * cc) : make_int4(0, 0, 0, 0);
                            v[u][cc][0] = (uint32_t)x.x; v[u][cc][1] = (uint32_t)x.y;
                            v[u][cc][2] = (uint32_t)x.z; v[u][cc][3] = (uint32_t)x.w;
                        }
                    }
                }
            };
            auto store_batch = [&](int j0, const uint32_t (&v)[U][RP][IDF]) {
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if (j0 + u >= k) break;    // warp-uniform: a batch's tail re-read of node k-1 stores nothing
#pragma unroll
                    for (int cc = 0; cc < RP; cc++) {
                        if constexpr (IDF == 1) {
                            const uint32_t wv = v[u][cc][0];
                            const uint32_t wm = W256 ? wv : wv & 0x7F7F7F7Fu;
                            if constexpr (E128) {
                                bad |= wv & 0x80808080u;
                            } else {
                                // SIMD byte compare (E ≤ 255); every u8 id is valid when E = 256
                                if (E < 256) bad |= __vcmpgeu4(wv, 0x01010101u * (uint32_t)E);
                            }
#pragma unroll
                            for (int qb = 0; qb < 4; qb++)
                                sts_u8((__byte_perm(wm, 0, 0x4440 | qb) << ESH) + (lbase + CSTEP * cc), marker);
                        } else {
#pragma unroll
                            for (int qb = 0; qb < 4; qb++) {
                                const uint32_t e = v[u][cc][qb];
                                bad |= e >= (uint32_t)E;
                                sts_u8(((e & (W256 ? 255u : 127u)) << ESH) + (lbase + CSTEP * cc), marker);
                            }
                        }
                    }
                }
            };
#ifdef EVICT_UNION_PREFETCH
            if constexpr (IDF == 1) {
                // two register batches: batch j+1's loads are in flight while batch j stores
                uint32_t va[U][RP][IDF], vb[U][RP][IDF];
                load_batch(0, va);
                for (int j0 = 0;;) {
                    if (j0 + U < k) load_batch(j0 + U, vb);
                    store_batch(j0, va);
                    j0 += U;
                    if (j0 >= k) break;
                    if (j0 + U < k) load_batch(j0 + U, va);
                    store_batch(j0, vb);
                    j0 += U;
                    if (j0 >= k) break;
                }
            } else
#endif
            for (int j0 = 0; j0 < k; j0 += U) {
                uint32_t v[U][RP][IDF];
                load_batch(j0, v);
                store_batch(j0, v);
            }
        }
        __syncwarp();
        if (run) {
            if constexpr (BITS) {
                // per-layer bit rows (test configuration only): lane = layer of this pass
                const int EWr = (E + 63) >> 6;
#pragma unroll 1
                for (int li = lane; li < 16 * RPP; li += 32) {
                    const int l = 16 * RPP * pass + li;
                    if (l >= L) break;
                    const uint32_t fl = W256 ? fbase + 4u * (uint32_t)(li & 7) + (uint32_t)(li >> 3)
                                             : fbase + 4u * (uint32_t)(li & 15) + (uint32_t)(li >> 4);
                    uint64_t wd[4] = {0ull, 0ull, 0ull, 0ull};
                    for (int e = 0; e < E; e++)
                        if (lds_u8(fl + ((uint32_t)e << ESH))) wd[e >> 6] |= 1ull << (e & 63);
                    for (int h = 0; h < EWr; h++) union_bits[((size_t)b * L + l) * EWr + h] = wd[h];
                }
                __syncwarp();
            }
            const int q = lane & 3, p8 = lane >> 2;
            const uint32_t fw = fbase + 16u * (uint32_t)(p8 * 4 + q);
            uint32_t a0 = 0u, a1 = 0u, a2 = 0u, a3 = 0u;
            if (mark) {
                // byte sums of marker bits ≤ 16·8 = 128 per lane: no carry into the next byte
                const uint32_t mk = 0x01010101u << ep;
                const bool wrap = ep == 3;
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    const uint4 x = lds_v4(fw + 512u * i);
                    a0 += x.x & mk; a1 += x.y & mk; a2 += x.z & mk; a3 += x.w & mk;
                    if (wrap) sts_v4_zero(fw + 512u * i);
                }
                a0 >>= ep; a1 >>= ep; a2 >>= ep; a3 >>= ep;
            } else {
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    const uint4 x = lds_v4(fw + 512u * i);
                    a0 += x.x; a1 += x.y; a2 += x.z; a3 += x.w;
                    sts_v4_zero(fw + 512u * i);
                }
            }
            if constexpr (W256) {
                // lane reads expert rows e = lane/2 + 16i, word quad h = lane&1 (words 4h..4h+3 =
                // layers l%8); the cross-lane sum spans 256 experts, so widen bytes to 16-bit lanes
                uint32_t lo[4] = {a0 & 0x00ff00ffu, a1 & 0x00ff00ffu, a2 & 0x00ff00ffu, a3 & 0x00ff00ffu};
                uint32_t hi[4] = {(a0 >> 8) & 0x00ff00ffu, (a1 >> 8) & 0x00ff00ffu, (a2 >> 8) & 0x00ff00ffu,
                                  (a3 >> 8) & 0x00ff00ffu};
#pragma unroll
                for (int o = 2; o < 32; o <<= 1)
#pragma unroll
                    for (int mm = 0; mm < 4; mm++) {
                        lo[mm] += __shfl_xor_sync(kFull, lo[mm], o);
                        hi[mm] += __shfl_xor_sync(kFull, hi[mm], o);
                    }
                const int u = lane >> 1, m = u & 3, beta = u >> 2;     // layer 8β + 4h + m
                const uint32_t wsel = (beta & 1) ? (m == 0 ? hi[0] : m == 1 ? hi[1] : m == 2 ? hi[2] : hi[3])
                                                 : (m == 0 ? lo[0] : m == 1 ? lo[1] : m == 2 ? lo[2] : lo[3]);
                const int l = 32 * pass + 8 * beta + 4 * (lane & 1) + m;
                if (l < L) {
                    const int cnt = (int)((wsel >> (16 * (beta >> 1))) & 0xffffu);
                    union_count[(size_t)b * L + l] = cnt;
                    tot += cnt;
                }
            } else {
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                a0 += __shfl_xor_sync(kFull, a0, o);
                a1 += __shfl_xor_sync(kFull, a1, o);
                a2 += __shfl_xor_sync(kFull, a2, o);
                a3 += __shfl_xor_sync(kFull, a3, o);
            }
            const int m = p8 & 3, bsel = p8 >> 2;
            const uint32_t x = m == 0 ? a0 : m == 1 ? a1 : m == 2 ? a2 : a3;
#pragma unroll
            for (int hb = 0; hb < 2; hb++) {
                const int byte = bsel + 2 * hb;
                const int l = 64 * pass + 16 * byte + 4 * q + m;
                if (l < L) {
                    const int cnt = (int)((x >> (8 * byte)) & 0xffu);
                    union_count[(size_t)b * L + l] = cnt;
                    tot += cnt;
                    if (PASSES == 1 && lsum) lcnt[hb] = (uint32_t)cnt;
                }
            }
            }
        }
        __syncwarp();
    }
    const bool anybad = run && __any_sync(kFull, bad);
    if (anybad) status |= EVICT_TREE_BAD_EXPERT;
    if (!run || anybad) {
        // a bad tree reports zero counts (and zero bit rows), like the oracle
        for (int l = lane; l < L; l += 32) union_count[(size_t)b * L + l] = 0;
        if constexpr (BITS) {
            const int EWr = (E + 63) >> 6;
            for (int i = lane; i < L * EWr; i += 32) union_bits[(size_t)b * L * EWr + i] = 0ull;
        }
        tot = 0;
    }
    __syncwarp();
    if (lsum && run && !anybad) { lsum[0] += lcnt[0]; lsum[1] += lcnt[1]; }
    if (mark && run) *epoch = (ep + 1) & 3;   // the block was cleared when ep == 3
    tot = __reduce_add_sync(kFull, tot);
    if (union_total && lane == 0) union_total[b] = tot;
}

// Top-8 u8 ids, E = 128, L ≤ 64 (the serving / C5 configuration; Eq. 5) with
// lane-owned flag columns: lane c owns byte column c of an 8 KB block of 32 rows × 256 B; row
// r = e >> 2 holds, at byte 4c + (e & 3), the flag of expert e for lane c's layer in region 0
// (bytes 0–127: layer c, all 8 ids of it from one 8-byte load) and region 1 (bytes 128–255:
// MODE 1 (32 < L ≤ 48) the half c & 1 of layer 32 + c/2, MODE 2 (48 < L ≤ 64) layer 32 + c).
// Every byte store of a warp instruction lands on bank c: conflict-free whatever the ids (the
// slot layout of tree_union_flags64 puts the two halves of a layer on one bank group, ≈ 2
// wavefronts per store).  The store offset of id e is one PRMT of two per-word vectors:
// lo = (w & 0x03030303) | column base, hi = (w >> 2) & 0x1F1F1F1F give (e >> 2) << 8 | lo.
// Nibble markers: tree t stores 0x01 (t even) or 0x10 (t odd) and the block is cleared after
// every second read-back, so a byte holds at most one marker of each parity and 8-row byte
// sums keep the two parities in separate nibbles (≤ 8 each): the read-back adds raw words.
// Read-back: lane (q = lane & 7, r0 = lane >> 3) loads rows r0 + 4j (j < 8) as 16-byte vectors
// (8 lanes per 128-byte phase: conflict-free), sums per column, keeps its parity's nibbles, two
// xor-shuffles over r0, one IDP4A per layer.
// Lane outputs (UColsLane, computed once per kernel): lanes 0–7 region 0 layers 4q..4q+3,
// lanes 8–15 region 1 (MODE 1: 32 + 2q, 33 + 2q; MODE 2: 32 + 4q..), others none.
struct UColsLane {
    int l0;          // first output layer (64: none)
    int nl;          // output layers of this lane (0, 2 or 4), all < L
    bool vec;        // one 8/16-byte store covers them (contiguous, aligned)
};
template <int MODE>
__device__ __forceinline__ UColsLane ucols_lane(int lane, int L)
{
    const int q = lane & 7, r0 = lane >> 3;
    UColsLane u{64, 0, false};
    if (r0 == 0) { u.l0 = 4 * q; u.nl = 4; }
    else if (r0 == 1 && MODE == 1) { u.l0 = 32 + 2 * q; u.nl = 2; }
    else if (r0 == 1 && MODE == 2) { u.l0 = 32 + 4 * q; u.nl = 4; }
    int n = L - u.l0;
    n = n < 0 ? 0 : (n > u.nl ? u.nl : n);
    u.vec = n == u.nl && n > 0 && (L % u.nl) == 0;   // b·L + l0 is a multiple of nl
    u.nl = n;
    if (n == 0) u.l0 = 64;
    return u;
}
__device__ __forceinline__ uint32_t prmt_b32(uint32_t a, uint32_t b, uint32_t sel)
{
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}
__device__ __forceinline__ void ucols_store4(uint32_t fb, uint32_t w, uint32_t cb, uint32_t hb, uint32_t marker)
{
    const uint32_t lo = (w & 0x03030303u) | cb;
    const uint32_t hi = ((w >> 2) & 0x1F1F1F1Fu) | hb;   // hb < 128 per byte (row bits 5–6)
    // id j: byte 0 = lo.b_j, byte 1 = hi.b_j, bytes 2–3 = sign of hi.b_j (0)
    sts_u8(fb + prmt_b32(lo, hi, 0xCC40u), marker);
    sts_u8(fb + prmt_b32(lo, hi, 0xDD51u), marker);
    sts_u8(fb + prmt_b32(lo, hi, 0xEE62u), marker);
    sts_u8(fb + prmt_b32(lo, hi, 0xFF73u), marker);
}
// One load batch of UB kept rows (this lane's parts) and the loader: rows j0 .. j0 + UB − 1 of
// the tree (a slot past k re-reads row k − 1); `half` loads only the first UB / 2 when the rest
// lies past k (warp-uniform).
template <int UB>
struct UColsBatch {
    uint2 x0[UB];
    uint32_t x1[UB], x2[UB];
};
template <int MODE, int UB>
__device__ __forceinline__ void ucols_load(UColsBatch<UB> &v, const uint8_t *__restrict__ klist, int k, int j0,
                                           int b, int N, int L, const void *__restrict__ ids, int lane)
{
    const uint32_t rowB = (uint32_t)L * 8u;
    const bool ld0 = lane < L;
    const bool ld1 = MODE == 1 ? lane < 2 * (L - 32) : (MODE == 2 ? lane < L - 32 : false);
    const uint32_t lo0 = ld0 ? 8u * (uint32_t)lane : 0u;
    const uint32_t lo1 = ld1 ? (MODE == 1 ? 256u + 4u * (uint32_t)lane : 256u + 8u * (uint32_t)lane) : 0u;
    const uint8_t *tb = reinterpret_cast<const uint8_t *>(ids) + (size_t)b * N * rowB;
    const uint8_t *p0 = tb + lo0, *p1 = tb + lo1;
#pragma unroll
    for (int u = 0; u < UB; u++) {
        const uint32_t o = (uint32_t)klist[min(j0 + u, k - 1)] * rowB;
        v.x0[u] = __ldg(reinterpret_cast<const uint2 *>(p0 + o));
        v.x1[u] = 0u;
        v.x2[u] = 0u;
        if constexpr (MODE == 1) {
            v.x1[u] = __ldg(reinterpret_cast<const uint32_t *>(p1 + o));
        } else if constexpr (MODE == 2) {
            const uint2 y = __ldg(reinterpret_cast<const uint2 *>(p1 + o));
            v.x1[u] = y.x;
            v.x2[u] = y.y;
        }
    }
}
template <int MODE, int UB>
__device__ __forceinline__ void tree_union_cols(uint32_t &status, const uint8_t *__restrict__ klist, int k,
                                                int b, int N, int L, const void *__restrict__ ids,
                                                uint8_t *flags, int32_t *__restrict__ union_count,
                                                int32_t *__restrict__ union_total, int *epoch,
                                                uint32_t *lsum, const UColsLane &ul, uint32_t sbase, uint32_t hb,
                                                UColsBatch<UB> *pf = nullptr, const uint8_t *nklist = nullptr,
                                                int nk = 0, int nb = 0)
{
    // pf (cross-tree prefetch): on entry it holds this tree's first batch (loaded during the
    // previous tree's read-back); after this tree's stores it receives the next tree's first batch
    // (nklist / nk / nb; nk = 0: none) so that round trip overlaps this read-back.
    // byte stores at sbase + PRMT(lo, hi | hb): sbase = the flag block's shared address (hb = 0), or a
    // CTA-uniform base with the block's 256-byte row offset in hb (the add folds into the STS)
    const int lane = lane_id();
    const int q = lane & 7, r0 = lane >> 3;
    const bool run = status == 0 && k > 0;
    uint32_t cnt[4] = {0u, 0u, 0u, 0u};
    if (run) {
        const int ep = *epoch;                      // 0 or 1
        const uint32_t marker = ep ? 0x10u : 0x01u;
        const uint32_t fb = (uint32_t)__cvta_generic_to_shared(flags);
        const uint32_t rowB = (uint32_t)L * 8u;
        // lanes past the layers re-read byte 0 of the row: their flags land in columns of
        // layers ≥ L (never counted) and the bytes are ids of the same kept row
        const bool ld0 = lane < L;
        const bool ld1 = MODE == 1 ? lane < 2 * (L - 32) : (MODE == 2 ? lane < L - 32 : false);
        const uint32_t lo0 = ld0 ? 8u * (uint32_t)lane : 0u;
        const uint32_t lo1 = ld1 ? (MODE == 1 ? 256u + 4u * (uint32_t)lane : 256u + 8u * (uint32_t)lane) : 0u;
        const uint32_t cb0 = (4u * (uint32_t)lane) * 0x01010101u;
        const uint32_t cb1 = (128u + 4u * (uint32_t)lane) * 0x01010101u;
        const uint8_t *tb = reinterpret_cast<const uint8_t *>(ids) + (size_t)b * N * rowB;
        const uint8_t *p0 = tb + lo0, *p1 = tb + lo1;
        uint32_t badw = 0u;
#pragma unroll 1
        for (int j0 = 0; j0 < k; j0 += UB) {
            if (pf != nullptr && j0 == 0) {
                // the batch arrived during the previous tree; its id check
#pragma unroll
                for (int u = 0; u < UB; u++) badw |= pf->x0[u].x | pf->x0[u].y | pf->x1[u] | pf->x2[u];
#pragma unroll
                for (int u = 0; u < UB; u++) {
                    if (u >= k) break;   // warp-uniform
                    ucols_store4(sbase, pf->x0[u].x, cb0, hb, marker);
                    ucols_store4(sbase, pf->x0[u].y, cb0, hb, marker);
                    if constexpr (MODE >= 1) ucols_store4(sbase, pf->x1[u], cb1, hb, marker);
                    if constexpr (MODE == 2) ucols_store4(sbase, pf->x2[u], cb1, hb, marker);
                }
                continue;
            }
            uint2 x0[UB];
            uint32_t x1[UB], x2[UB];
            auto load = [&](int u) {
                const uint32_t o = (uint32_t)klist[min(j0 + u, k - 1)] * rowB;
                x0[u] = __ldg(reinterpret_cast<const uint2 *>(p0 + o));
                x1[u] = 0u;
                x2[u] = 0u;
                if constexpr (MODE == 1) {
                    x1[u] = __ldg(reinterpret_cast<const uint32_t *>(p1 + o));
                } else if constexpr (MODE == 2) {
                    const uint2 y = __ldg(reinterpret_cast<const uint2 *>(p1 + o));
                    x1[u] = y.x;
                    x2[u] = y.y;
                }
            };
            // every row of the batch is consumed here, in the loads' own block: the compiler
            // cannot sink a row's loads behind the previous rows' stores (the store loop's
            // warp-uniform exits), so one DRAM round trip serves the batch (tail re-reads are
            // rows k − 1 again: harmless for the id check).  The batch's second half is loaded
            // only when the tree has rows there (warp-uniform).
            constexpr int H = UB > 4 ? UB / 2 : UB;
#pragma unroll
            for (int u = 0; u < H; u++) load(u);
            if (UB > H && j0 + H < k) {
#pragma unroll
                for (int u = H; u < UB; u++) load(u);
#pragma unroll
                for (int u = H; u < UB; u++) badw |= x0[u].x | x0[u].y | x1[u] | x2[u];
            }
#pragma unroll
            for (int u = 0; u < H; u++) badw |= x0[u].x | x0[u].y | x1[u] | x2[u];
#pragma unroll
            for (int u = 0; u < UB; u++) {
                if (j0 + u >= k) break;   // warp-uniform: a batch's tail re-read stores nothing
                ucols_store4(sbase, x0[u].x, cb0, hb, marker);
                ucols_store4(sbase, x0[u].y, cb0, hb, marker);
                if constexpr (MODE >= 1) ucols_store4(sbase, x1[u], cb1, hb, marker);
                if constexpr (MODE == 2) ucols_store4(sbase, x2[u], cb1, hb, marker);
            }
        }
        if (pf != nullptr && nk > 0) ucols_load<MODE, UB>(*pf, nklist, nk, 0, nb, N, L, ids, lane);
        __syncwarp();
        const bool clear = ep == 1;
        uint32_t a0 = 0u, a1 = 0u, a2 = 0u, a3 = 0u, c0 = 0u, c1 = 0u, c2 = 0u, c3 = 0u;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t ra = fb + 256u * (uint32_t)(r0 + 4 * j) + 16u * (uint32_t)q;
            const uint4 x = lds_v4(ra);
            a0 += x.x; a1 += x.y; a2 += x.z; a3 += x.w;
            if constexpr (MODE == 1) {
                const uint4 y = lds_v4(ra + 128u);
                c0 += y.x | y.y;   // layer 32 + 2q (both halves)
                c1 += y.z | y.w;   // layer 33 + 2q
            } else if constexpr (MODE == 2) {
                const uint4 y = lds_v4(ra + 128u);
                c0 += y.x; c1 += y.y; c2 += y.z; c3 += y.w;
            }
            if (clear) {
                sts_v4_zero(ra);
                if constexpr (MODE >= 1) sts_v4_zero(ra + 128u);
            }
        }
        *epoch = ep ^ 1;
        // this lane's words (its output region), this parity's nibbles: ≤ 8 per byte, ≤ 32 after
        // the sum over the 4 lanes (r0) of a column quad
        const int sh = 4 * ep;
        uint32_t w0 = ((r0 & 1) ? c0 : a0) >> sh & 0x0F0F0F0Fu, w1 = ((r0 & 1) ? c1 : a1) >> sh & 0x0F0F0F0Fu;
        uint32_t w2 = ((r0 & 1) ? c2 : a2) >> sh & 0x0F0F0F0Fu, w3 = ((r0 & 1) ? c3 : a3) >> sh & 0x0F0F0F0Fu;
        // partners across r0 hold the other region's words for odd r0: exchange both regions
        uint32_t o0 = ((r0 & 1) ? a0 : c0) >> sh & 0x0F0F0F0Fu, o1 = ((r0 & 1) ? a1 : c1) >> sh & 0x0F0F0F0Fu;
        uint32_t o2 = ((r0 & 1) ? a2 : c2) >> sh & 0x0F0F0F0Fu, o3 = ((r0 & 1) ? a3 : c3) >> sh & 0x0F0F0F0Fu;
        // xor 8 swaps r0 parity: the partner's "other" words are this lane's region
        w0 += __shfl_xor_sync(kFull, o0, 8); w1 += __shfl_xor_sync(kFull, o1, 8);
        w2 += __shfl_xor_sync(kFull, o2, 8); w3 += __shfl_xor_sync(kFull, o3, 8);
        w0 += __shfl_xor_sync(kFull, w0, 16); w1 += __shfl_xor_sync(kFull, w1, 16);
        w2 += __shfl_xor_sync(kFull, w2, 16); w3 += __shfl_xor_sync(kFull, w3, 16);
        cnt[0] = (uint32_t)__dp4a(w0, 0x01010101u, 0u);
        cnt[1] = (uint32_t)__dp4a(w1, 0x01010101u, 0u);
        cnt[2] = (uint32_t)__dp4a(w2, 0x01010101u, 0u);
        cnt[3] = (uint32_t)__dp4a(w3, 0x01010101u, 0u);
        if (__any_sync(kFull, badw & 0x80808080u)) {
            status |= EVICT_TREE_BAD_EXPERT;
            cnt[0] = cnt[1] = cnt[2] = cnt[3] = 0u;
        }
    }
    if (!run && pf != nullptr && nk > 0) ucols_load<MODE, UB>(*pf, nklist, nk, 0, nb, N, L, ids, lane);
    // union counts (zeros for an errored tree)
    if (ul.nl < 4) cnt[3] = 0u;
    if (ul.nl < 3) cnt[2] = 0u;
    if (ul.nl < 2) cnt[1] = 0u;
    if (ul.nl < 1) cnt[0] = 0u;
    int32_t *uc = union_count + (size_t)b * L + ul.l0;
    if (ul.vec) {
        if (ul.nl == 4) *reinterpret_cast<int4 *>(uc) = make_int4((int)cnt[0], (int)cnt[1], (int)cnt[2], (int)cnt[3]);
        else *reinterpret_cast<int2 *>(uc) = make_int2((int)cnt[0], (int)cnt[1]);
    } else {
#pragma unroll
        for (int m = 0; m < 4; m++)
            if (m < ul.nl) uc[m] = (int)cnt[m];
    }
    const int tot = __reduce_add_sync(kFull, (int)(cnt[0] + cnt[1] + cnt[2] + cnt[3]));
    if (union_total && lane == 0) union_total[b] = tot;
    if (lsum && status == 0) {
#pragma unroll
        for (int m = 0; m < 4; m++) lsum[m] += cnt[m];
    }
}

// Dispatch: flags for top-8 ids, register OR for 1/2/4-word masks, generic otherwise.
template <int NPL, int IDF, int KT, int EW, int R>
__device__ __forceinline__ void tree_union(uint32_t &status, const uint8_t *__restrict__ klist, int k, int b,
                                           int N, int L, int K, int E, int idb,
                                           const void *__restrict__ ids, uint8_t *flags, int Epad,
                                           int32_t *__restrict__ union_count,
                                           int32_t *__restrict__ union_total,
                                           uint64_t *__restrict__ union_bits,
                                           int64_t *__restrict__ expert_hist)
{
    if constexpr (IDF == 1 || IDF == 4) {
        if (expert_hist == nullptr) {   // the flag path cannot retract a bad tree's histogram rows
            const bool e128 = IDF == 1 && E == 128;
            if (E <= 128) {
                if (union_bits == nullptr) {
                    if (e128) tree_union_flags64<IDF, R, true, false>(status, klist, k, b, N, L, E, ids, flags,
                                                                      union_count, union_total, nullptr);
                    else tree_union_flags64<IDF, R, false, false>(status, klist, k, b, N, L, E, ids, flags,
                                                                  union_count, union_total, nullptr);
                } else {
                    if (e128) tree_union_flags64<IDF, R, true, true>(status, klist, k, b, N, L, E, ids, flags,
                                                                     union_count, union_total, union_bits);
                    else tree_union_flags64<IDF, R, false, true>(status, klist, k, b, N, L, E, ids, flags,
                                                                 union_count, union_total, union_bits);
                }
            } else if (union_bits == nullptr) {   // 128 < E ≤ 256: 32-byte expert rows
                tree_union_flags64<IDF, R, false, false, true>(status, klist, k, b, N, L, E, ids, flags,
                                                               union_count, union_total, nullptr);
            } else {
                tree_union_flags64<IDF, R, false, true, true>(status, klist, k, b, N, L, E, ids, flags,
                                                              union_count, union_total, union_bits);
            }
        } else {
            tree_union_generic<NPL, IDF, KT, EW, (R + 1) / 2>(status, klist, k, b, N, L, K, E, idb, ids,
                                                             union_count, union_total, union_bits,
                                                             expert_hist);
        }
    }
    else if constexpr (IDF == 8)
        tree_union_fast<NPL, IDF, EW, R>(status, klist, k, b, N, L, E, ids, union_count, union_total,
                                         union_bits, expert_hist);
    else
        tree_union_generic<NPL, IDF, KT, EW, R / 2>(status, klist, k, b, N, L, K, E, idb, ids,
                                                    union_count, union_total, union_bits, expert_hist);
}

}  // namespace evict
