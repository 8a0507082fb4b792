// evict_group.cuh — sub-warp-per-tree select (A1–A5) and verify-tree build (A6).
//
// A group of G lanes owns one tree (G = 8 for N ≤ 64, G = 16 for N ≤ 128), so a
// warp works on 32/G trees at once; lane g of a group owns the 8 consecutive
// nodes 8g .. 8g+7 (two 16-byte vector loads per array).  Compared with one
// warp per tree this cuts the per-tree instruction count several-fold: most
// bitonic stages become register compare-exchanges inside a lane, the scan is
// 8 serial adds + log2(G) shuffles, and every warp instruction serves 4 (or 2)
// trees.  All shuffles stay inside the group (xor offsets < G, width G).
//   A1 g_load            PAPER.md:48; readings Z4/Z9/Z10
//   A2 g_levels          Eq. 7: synchronous sweeps, exact
//                        serial root→leaf fp32 products
//   A3–A5 g_rank_argmax  §3.2.1, Eq. 8–10: full
//                        (score desc, index asc) ranking when the order row
//                        is requested; g_select_values otherwise (value sort +
//                        tie-aware threshold, same k*/keep bit for bit)
//   A6 g_emit            Fig. 4(c), layout Z12
#pragma once

#include "evict_tree.cuh"

namespace evict {
namespace grp {

constexpr int NP = 8;  // nodes per lane

template <int G>
struct GShape {
    static constexpr int NMAX = G * NP;   // 64 or 128
    static constexpr int W = NMAX / 64;   // 64-bit mask words
    static constexpr int TPW = 32 / G;    // trees per warp
};

template <int G>
__device__ __forceinline__ int gl() { return threadIdx.x & (G - 1); }
template <int G>
__device__ __forceinline__ int gidx() { return (threadIdx.x & 31) / G; }

template <int G>
__device__ __forceinline__ uint32_t g_or(uint32_t v)
{
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v |= __shfl_xor_sync(kFull, v, o);
    return v;
}
template <int G>
__device__ __forceinline__ uint32_t g_max(uint32_t v)
{
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
        const uint32_t w = __shfl_xor_sync(kFull, v, o);
        v = w > v ? w : v;
    }
    return v;
}
template <int G>
__device__ __forceinline__ int g_sum(int v)
{
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}
template <int G>
__device__ __forceinline__ int g_maxi(int v)
{
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
        const int w = __shfl_xor_sync(kFull, v, o);
        v = w > v ? w : v;
    }
    return v;
}
template <int G>
__device__ __forceinline__ uint64_t g_or64(uint64_t v)
{
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v |= shfl_xor64(v, o);
    return v;
}

template <int W>
__device__ __forceinline__ int popc_below_w(const uint64_t (&m)[W], int i)
{
    if constexpr (W == 1) return __popcll(m[0] & ((1ull << i) - 1ull));   // 0 ≤ i < 64 at every call
    int c = 0;
#pragma unroll
    for (int w = 0; w < W; w++) {
        const int lo = w * 64;
        const uint64_t mk = i >= lo + 64 ? ~0ull : (i <= lo ? 0ull : ((1ull << (i - lo)) - 1ull));
        c += __popcll(m[w] & mk);
    }
    return c;
}
template <int W>
__device__ __forceinline__ bool bit_w(const uint64_t (&m)[W], int i)
{
    bool r = false;
#pragma unroll
    for (int w = 0; w < W; w++)
        if ((i >> 6) == w) r = (m[w] >> (i & 63)) & 1ull;
    return r;
}

template <int G>
struct GTree {
    static constexpr int W = GShape<G>::W;
    int par[NP];
    float q[NP];
    float sc[NP];
    int n;
    uint32_t status;  // EVICT_TREE_* ; inactive groups carry BAD_SIZE
    int kstar;
    float ehat, util;
    uint64_t keep[W];  // identical in every lane of the group
};

// ------------------------------------------------------------ A1
template <int G>
__device__ __forceinline__ void g_load(GTree<G> &t, const int32_t *__restrict__ parent,
                                       const float *__restrict__ q, const int32_t *__restrict__ n_nodes,
                                       int b, int N, bool active)
{
    const int base = gl<G>() * NP;
    const size_t row = (size_t)b * N;
    int4 p0 = make_int4(-1, -1, -1, -1), p1 = p0;
    float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f), q1 = q0;
    if (active && base < N) {
        p0 = __ldg(reinterpret_cast<const int4 *>(parent + row + base));
        q0 = __ldg(reinterpret_cast<const float4 *>(q + row + base));
        if (base + NP <= N) {   // N % 4 == 0: the second half is all in or all out
            p1 = __ldg(reinterpret_cast<const int4 *>(parent + row + base + 4));
            q1 = __ldg(reinterpret_cast<const float4 *>(q + row + base + 4));
        }
    }
    t.par[0] = p0.x; t.par[1] = p0.y; t.par[2] = p0.z; t.par[3] = p0.w;
    t.par[4] = p1.x; t.par[5] = p1.y; t.par[6] = p1.z; t.par[7] = p1.w;
    t.q[0] = q0.x; t.q[1] = q0.y; t.q[2] = q0.z; t.q[3] = q0.w;
    t.q[4] = q1.x; t.q[5] = q1.y; t.q[6] = q1.z; t.q[7] = q1.w;
    t.n = active ? (n_nodes ? __ldg(n_nodes + b) : N) : 0;
    uint32_t st = (t.n < 1 || t.n > N) ? EVICT_TREE_BAD_SIZE : 0u;
#pragma unroll
    for (int r = 0; r < NP; r++) {
        const int i = base + r;
        if (i < t.n) {
            if (i == 0) {
                if (t.par[r] != -1) st |= EVICT_TREE_BAD_PARENT;
            } else {
                if (t.par[r] < 0 || t.par[r] >= i) st |= EVICT_TREE_BAD_PARENT;
                const float qq = t.q[r];
                if (!(qq >= 0.f && qq <= 1.f)) st |= EVICT_TREE_BAD_PROB;
            }
        }
        if (t.q[r] == 0.f) t.q[r] = 0.f;  // canonicalise -0.0 (Z9)
    }
    st = g_or<G>(st);
    t.status = (st & EVICT_TREE_BAD_SIZE) ? EVICT_TREE_BAD_SIZE : st;
}

// A6 input only (the two-kernel throughput path: select already ran): parent row and n
template <int G>
__device__ __forceinline__ void g_load_par(GTree<G> &t, const int32_t *__restrict__ parent,
                                           const int32_t *__restrict__ n_nodes, int b, int N, bool active)
{
    const int base = gl<G>() * NP;
    const size_t row = (size_t)b * N;
    int4 p0 = make_int4(-1, -1, -1, -1), p1 = p0;
    if (active && base < N) {
        p0 = __ldg(reinterpret_cast<const int4 *>(parent + row + base));
        if (base + NP <= N) p1 = __ldg(reinterpret_cast<const int4 *>(parent + row + base + 4));
    }
    t.par[0] = p0.x; t.par[1] = p0.y; t.par[2] = p0.z; t.par[3] = p0.w;
    t.par[4] = p1.x; t.par[5] = p1.y; t.par[6] = p1.z; t.par[7] = p1.w;
    t.n = active ? (n_nodes ? __ldg(n_nodes + b) : N) : 0;
}

// cost row: the loads (g_fetch_cost, independent of the tree — issue them before the tree's own
// loads are consumed) and the validation against n (g_apply_cost)
template <int G>
__device__ __forceinline__ void g_fetch_cost(float4 (&cr)[2], const float *__restrict__ cost, int N, bool active)
{
    const int base = gl<G>() * NP;
    // cost rows are 16-byte aligned with N % 4 == 0 (host-checked): two vector loads
    cr[0] = make_float4(1.f, 1.f, 1.f, 1.f);
    cr[1] = cr[0];
    if (active && base < N) {
        cr[0] = __ldg(reinterpret_cast<const float4 *>(cost + base));
        if (base + 4 < N) cr[1] = __ldg(reinterpret_cast<const float4 *>(cost + base + 4));
    }
}
template <int G>
__device__ __forceinline__ void g_apply_cost(float (&c)[NP], GTree<G> &t, const float4 (&cr)[2])
{
    const int base = gl<G>() * NP;
    c[0] = cr[0].x; c[1] = cr[0].y; c[2] = cr[0].z; c[3] = cr[0].w;
    c[4] = cr[1].x; c[5] = cr[1].y; c[6] = cr[1].z; c[7] = cr[1].w;
    uint32_t st = 0;
#pragma unroll
    for (int r = 0; r < NP; r++) {
        const int i = base + r;
        if (i < t.n && !(t.status & EVICT_TREE_BAD_SIZE)) {
            if (!(c[r] > 0.f)) st |= EVICT_TREE_BAD_COST;
            if (i == 0 && c[r] == __int_as_float(0x7f800000)) st |= EVICT_TREE_BAD_COST;
        } else {
            c[r] = 1.f;
        }
    }
    t.status |= g_or<G>(st);
}
template <int G>
__device__ __forceinline__ void g_load_cost(float (&c)[NP], GTree<G> &t, const float *__restrict__ cost,
                                            int N)
{
    float4 cr[2];
    g_fetch_cost<G>(cr, cost, N, !(t.status & EVICT_TREE_BAD_SIZE));
    g_apply_cost<G>(c, t, cr);
}

// ------------------------------------------------------------ A2
// Score(v) = Π_{u ∈ Path(root, v)} q(u) (Eq. 7) by synchronous
// sweeps: every sweep each node recomputes from its parent's previous score, so
// after sweep t all depth-≤t nodes are exact with the serial root→leaf product
// order (one fp32 rounding per edge).  The first sweep with no change ends the
// loop: the update x(v) = q(v)·x(parent) has a unique fixed point (induction on
// depth), so an unchanged state is the exact one — depth needs no tracking here
// (emit recovers it from the ancestor walk).
// sd: this group's NMAX scores in shared memory, stored swizzled: node i at
// swz(i) = i ^ ((i >> 3) & 4), so the two 16-byte stores of the 8 lanes of a
// quarter-warp land on 8 distinct bank groups.
__device__ __forceinline__ int swz(int i) { return i ^ ((i >> 3) & 4); }

template <int G, bool SCORES>
__device__ __forceinline__ void g_levels(GTree<G> &t, float *sd)
{
    const int g = gl<G>();
    const int base = g * NP;
    // non-live nodes (root, pads, errored tree) read the root's slot (always 1) times 1: their
    // score stays 1 without a select per sweep
    int pidx[NP];
    float qe[NP];
#pragma unroll
    for (int r = 0; r < NP; r++) {
        const int i = base + r;
        const bool live = (t.status == 0) && (i > 0) && (i < t.n);
        pidx[r] = live ? swz(t.par[r]) : 0;
        qe[r] = live ? t.q[r] : 1.f;
        t.sc[r] = 1.f;
    }
    const int c0 = swz(base), c1 = swz(base + 4);
    *reinterpret_cast<float4 *>(&sd[c0]) = make_float4(1.f, 1.f, 1.f, 1.f);
    *reinterpret_cast<float4 *>(&sd[c1]) = make_float4(1.f, 1.f, 1.f, 1.f);
    __syncwarp();
    if constexpr (SCORES) {
        while (true) {
            uint32_t diff = 0u;
            float ns[NP];
#pragma unroll
            for (int r = 0; r < NP; r++) {
                ns[r] = __fmul_rn(sd[pidx[r]], qe[r]);   // both ≥ +0
                diff |= __float_as_uint(ns[r]) ^ __float_as_uint(t.sc[r]);
            }
            const bool changed = diff != 0u;
            __syncwarp();
#pragma unroll
            for (int r = 0; r < NP; r++) t.sc[r] = ns[r];
            *reinterpret_cast<float4 *>(&sd[c0]) = make_float4(ns[0], ns[1], ns[2], ns[3]);
            *reinterpret_cast<float4 *>(&sd[c1]) = make_float4(ns[4], ns[5], ns[6], ns[7]);
            __syncwarp();
            if (!__any_sync(kFull, changed)) break;
        }
    }
}

// ------------------------------------------------------------ A3–A5
// rk: this group's node → rank bytes (NMAX).  Writes order/prefix rows when
// given (row of N entries), fills t.kstar/ehat/util/keep.
template <int G>
__device__ __forceinline__ void g_rank_argmax(GTree<G> &t, uint8_t *rk, const float (&c)[NP], int N,
                                              int32_t *__restrict__ order_row,
                                              float *__restrict__ prefix_row, const evict_policy_t &pol)
{
    constexpr int NMAX = GShape<G>::NMAX;
    constexpr int W = GShape<G>::W;
    const int g = gl<G>();
    const int base = g * NP;
    const bool ok = t.status == 0;
    uint64_t key[NP];
#pragma unroll
    for (int r = 0; r < NP; r++) {
        const int i = base + r;
        key[r] = (ok && i < t.n) ? (((uint64_t)(~__float_as_uint(t.sc[r])) << 32) | (uint32_t)i) : ~0ull;
    }
    // bitonic sort ascending on key == (score desc, index asc); element x = 8g + r.
    // Valid keys are unique (the index is in the low bits; pads are all ~0), so
    // a compare-exchange needs one 64-bit comparison: swap ⇔ (a > b) xor desc.
#pragma unroll
    for (int k = 2; k <= NMAX; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < NP) {
#pragma unroll
                for (int r = 0; r < NP; r++) {
                    const int rp = r ^ j;
                    if (rp > r) {
                        // direction = bit k of x = base + r: base is a multiple of NP, so
                        // k < NP reads r (compile-time), k ≥ NP reads base (lane-uniform)
                        const bool desc = (k < NP) ? ((r & k) != 0) : ((base & k) != 0);
                        const uint64_t a = key[r], bb = key[rp];
                        const bool sw = (a > bb) != desc;
                        key[r] = sw ? bb : a;
                        key[rp] = sw ? a : bb;
                    }
                }
            } else {
                const int lj = j / NP;
                // lane-uniform: lower partner (x & j == 0) keeps the min when ascending
                const bool take_min = ((base & j) == 0) == ((base & k) == 0);
#pragma unroll
                for (int r = 0; r < NP; r++) {
                    const uint64_t o = shfl_xor64(key[r], lj);
                    const bool lt = o < key[r];
                    key[r] = (lt == take_min) ? o : key[r];
                }
            }
        }
    }
    float sp[NP];
    int node[NP];
#pragma unroll
    for (int r = 0; r < NP; r++) {
        node[r] = (int)(uint32_t)key[r];
        sp[r] = __uint_as_float(~(uint32_t)(key[r] >> 32));
        if (ok && base + r < t.n) rk[node[r]] = (uint8_t)(base + r);
    }
    // A4: S[k] = Σ_{j<k} Score(order[j])
    float loc[NP];
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < NP; r++) {
        acc = __fadd_rn(acc, sp[r]);
        loc[r] = acc;
    }
    float incl = acc;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
        const float v = __shfl_up_sync(kFull, incl, o, G);
        if (g >= o) incl = __fadd_rn(incl, v);
    }
    float excl = __shfl_up_sync(kFull, incl, 1, G);
    if (g == 0) excl = 0.f;
    float S[NP];
    uint32_t Rb[NP];
    uint32_t best = 0;
#pragma unroll
    for (int r = 0; r < NP; r++) {
        S[r] = __fadd_rn(excl, loc[r]);
        const bool v = ok && base + r < t.n;
        const float R = v ? __fdiv_rn(S[r], c[r]) : 0.f;   // A5: IEEE division, +inf cost ⇒ 0
        Rb[r] = v ? __float_as_uint(R) : 0u;
        best = Rb[r] > best ? Rb[r] : best;
    }
    const uint32_t mx = g_max<G>(best);
    float SK = 0.f;   // S at position n−1 (coverage policy)
    if (pol.kind == EVICT_POLICY_COVERAGE) {
        float sl = 0.f;
#pragma unroll
        for (int r = 0; r < NP; r++)
            if (base + r == t.n - 1) sl = S[r];
        const int own = ok && t.n >= 1 ? (t.n - 1) / NP : 0;
        SK = __shfl_sync(kFull, sl, (threadIdx.x & 31 & ~(G - 1)) + own);
    }
    int rfirst = NP;
#pragma unroll
    for (int r = NP - 1; r >= 0; r--)
        if (ok && base + r < t.n && policy_hit(pol, base + r, t.n, Rb[r], mx, S[r], SK)) rfirst = r;
    const unsigned has = __ballot_sync(kFull, rfirst < NP);
    const unsigned gm = (G == 32) ? has : ((has >> (gidx<G>() * G)) & ((1u << G) - 1u));
    const int wl = gm ? __ffs(gm) - 1 : 0;                 // smallest k wins ties (Z3)
    const int src = (threadIdx.x & 31 & ~(G - 1)) + wl;
    const int rf = __shfl_sync(kFull, rfirst, src);
    float Sk = 0.f, Rk = 0.f;
#pragma unroll
    for (int r = 0; r < NP; r++)
        if (r == rf) { Sk = S[r]; Rk = __uint_as_float(Rb[r]); }
    Sk = __shfl_sync(kFull, Sk, src);
    Rk = __shfl_sync(kFull, Rk, src);
    if (ok) {
        t.ehat = Sk;
        t.util = Rk;
        t.kstar = wl * NP + rf + 1;
    } else {
        t.ehat = 0.f;
        t.util = 0.f;
        t.kstar = 0;
    }
    if ((order_row != nullptr || prefix_row != nullptr) && base < N) {
#pragma unroll
        for (int r = 0; r < NP; r++) {
            if (base + r < N) {
                const bool v = ok && base + r < t.n;
                if (order_row) order_row[base + r] = v ? node[r] : -1;
                if (prefix_row) prefix_row[base + r] = v ? S[r] : 0.f;
            }
        }
    }
    __syncwarp();
    // keep = order[0 .. k*): node i kept ⇔ rank(i) < k*
    uint64_t local[W];
#pragma unroll
    for (int w = 0; w < W; w++) local[w] = 0ull;
#pragma unroll
    for (int r = 0; r < NP; r++) {
        const int i = base + r;
        if (ok && i < t.n && rk[i] < t.kstar) local[i >> 6] |= 1ull << (i & 63);
    }
#pragma unroll
    for (int w = 0; w < W; w++) t.keep[w] = g_or64<G>(local[w]);
}

// A3–A5 without the order row: the prefix sums S[k] (Eq. 8) need only the
// sorted score VALUES — equal scores add the same fp32 terms whichever of them
// comes first, so S, the ratios and k* are bit-identical to the (score desc,
// index asc) ranking.  Values sort with fmin/fmax (scores are ≥ +0, pads -1),
// one 32-bit shuffle per cross-lane step.  The kept set is then the ranking's
// first k* nodes: every node with score > v (v = the k*-th largest score) plus
// the k* − #{score > v} lowest-index nodes with score == v.  prefix_row may be
// written (values only).
// COST: the launch's policy is EVICT_POLICY_COST (k* = smallest argmax of the ratio; no coverage
// or fixed-k test per position)
template <int G, bool COST = false>
__device__ __forceinline__ void g_select_values(GTree<G> &t, const float (&c)[NP], int N,
                                                float *__restrict__ prefix_row, const evict_policy_t &pol)
{
    constexpr int NMAX = GShape<G>::NMAX;
    constexpr int W = GShape<G>::W;
    const int g = gl<G>();
    const int base = g * NP;
    const bool ok = t.status == 0;
    float key[NP];
#pragma unroll
    for (int r = 0; r < NP; r++) key[r] = (ok && base + r < t.n) ? t.sc[r] : -1.f;
    // bitonic sort, descending; element x = 8g + r
#pragma unroll
    for (int k = 2; k <= NMAX; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < NP) {
#pragma unroll
                for (int r = 0; r < NP; r++) {
                    const int rp = r ^ j;
                    if (rp > r) {
                        const bool desc = (k < NP) ? ((r & k) != 0) : ((base & k) != 0);
                        const float lo = fminf(key[r], key[rp]), hi = fmaxf(key[r], key[rp]);
                        key[r] = desc ? lo : hi;
                        key[rp] = desc ? hi : lo;
                    }
                }
            } else {
                const int lj = j / NP;
                const bool take_hi = ((base & j) == 0) == ((base & k) == 0);
#pragma unroll
                for (int r = 0; r < NP; r++) {
                    const float o = __shfl_xor_sync(kFull, key[r], lj);
                    key[r] = take_hi ? fmaxf(key[r], o) : fminf(key[r], o);
                }
            }
        }
    }
    // A4: S[k] = Σ_{j<k} Score(order[j])
    float loc[NP];
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < NP; r++) {
        acc = __fadd_rn(acc, key[r]);
        loc[r] = acc;
    }
    float incl = acc;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
        const float v = __shfl_up_sync(kFull, incl, o, G);
        if (g >= o) incl = __fadd_rn(incl, v);
    }
    float excl = __shfl_up_sync(kFull, incl, 1, G);
    if (g == 0) excl = 0.f;
    float S[NP];
    uint32_t Rb[NP];
    uint32_t best = 0;
#pragma unroll
    for (int r = 0; r < NP; r++) {
        S[r] = __fadd_rn(excl, loc[r]);
        const bool v = ok && base + r < t.n;
        const float R = v ? __fdiv_rn(S[r], c[r]) : 0.f;   // A5: IEEE division, +inf cost ⇒ 0
        Rb[r] = v ? __float_as_uint(R) : 0u;
        best = Rb[r] > best ? Rb[r] : best;
    }
    const uint32_t mx = g_max<G>(best);
    int rfirst = NP;
    if constexpr (COST) {
        // Rb = 0 past n and for an errored tree: only valid positions can equal mx > 0; mx = 0
        // (every ratio 0) takes position 0
#pragma unroll
        for (int r = NP - 1; r >= 0; r--)
            if (Rb[r] == mx && (mx != 0u || base + r == 0)) rfirst = r;
    } else {
        float SK = 0.f;   // S at position n−1 (coverage policy)
        if (pol.kind == EVICT_POLICY_COVERAGE) {
            float sl = 0.f;
#pragma unroll
            for (int r = 0; r < NP; r++)
                if (base + r == t.n - 1) sl = S[r];
            const int own = ok && t.n >= 1 ? (t.n - 1) / NP : 0;
            SK = __shfl_sync(kFull, sl, (threadIdx.x & 31 & ~(G - 1)) + own);
        }
#pragma unroll
        for (int r = NP - 1; r >= 0; r--)
            if (ok && base + r < t.n && policy_hit(pol, base + r, t.n, Rb[r], mx, S[r], SK)) rfirst = r;
    }
    const unsigned has = __ballot_sync(kFull, rfirst < NP);
    const unsigned gm = (G == 32) ? has : ((has >> (gidx<G>() * G)) & ((1u << G) - 1u));
    const int wl = gm ? __ffs(gm) - 1 : 0;                 // smallest k wins ties (Z3)
    const int src = (threadIdx.x & 31 & ~(G - 1)) + wl;
    const int rf = __shfl_sync(kFull, rfirst, src);
    float Sk = 0.f, Rk = 0.f, vk = 0.f;
#pragma unroll
    for (int r = 0; r < NP; r++)
        if (r == rf) { Sk = S[r]; Rk = __uint_as_float(Rb[r]); vk = key[r]; }
    Sk = __shfl_sync(kFull, Sk, src);
    Rk = __shfl_sync(kFull, Rk, src);
    vk = __shfl_sync(kFull, vk, src);
    const int kstar = wl * NP + rf + 1;
    if (ok) {
        t.ehat = Sk;
        t.util = Rk;
        t.kstar = kstar;
    } else {
        t.ehat = 0.f;
        t.util = 0.f;
        t.kstar = 0;
    }
    if (prefix_row != nullptr && base < N) {
#pragma unroll
        for (int r = 0; r < NP; r++)
            if (base + r < N) prefix_row[base + r] = (ok && base + r < t.n) ? S[r] : 0.f;
    }
    // keep: score > vk, plus the lowest-index ties (score == vk) up to k*
    uint32_t gt = 0u, eq = 0u;
#pragma unroll
    for (int r = 0; r < NP; r++) {
        const bool v = ok && base + r < t.n;
        gt |= (v && t.sc[r] > vk) ? (1u << r) : 0u;
        eq |= (v && t.sc[r] == vk) ? (1u << r) : 0u;
    }
    const int ngt = g_sum<G>(__popc(gt));
    const int neq = __popc(eq);
    int eq_before = neq;                                   // inclusive scan over lanes
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
        const int v = __shfl_up_sync(kFull, eq_before, o, G);
        if (g >= o) eq_before += v;
    }
    eq_before -= neq;
    int take = kstar - ngt - eq_before;                    // ties this lane may keep
    take = take < 0 ? 0 : (take > neq ? neq : take);
    uint32_t keq = eq;
    if (neq > take) {   // rare: more ties at the cut than slots left in this lane
#pragma unroll
        for (int r = 0; r < NP; r++) {
            // drop the highest set bits beyond `take`
            if (__popc(keq) > take) keq &= ~(0x80000000u >> __clz(keq));
        }
    }
    const uint32_t kb = ok ? (gt | keq) : 0u;
    uint64_t local[W];
#pragma unroll
    for (int w = 0; w < W; w++) local[w] = 0ull;
#pragma unroll
    for (int w = 0; w < W; w++)
        if ((base >> 6) == w) local[w] = (uint64_t)kb << (base & 63);
#pragma unroll
    for (int w = 0; w < W; w++) t.keep[w] = g_or64<G>(local[w]);
}

// ------------------------------------------------------------ A6
// Only kept nodes do work, spread over the group by slot so no lane serialises
// a cluster of kept nodes (kept nodes crowd the low indices):
//   1. klist[slot] = node (slot = popc(keep below node)), built once by the select;
//   2. slot s (lane s % G) ORs bit s into its parent's child mask (shared atomics);
//   3. slot s builds its ancestor-or-self row by walking the parent chain of the
//      shared-memory record (depth steps, no level loop), reads next-token /
//      next-sibling from the child masks and emits the packed row.
// par: the tree's shared parent record; klist: its kept nodes (built by the select); child (NMAX × W words)
// (all in shared memory).
// slot_of (optional, N ≤ 64): node → slot for the kept nodes (built with klist) — one byte load per
// ancestor step instead of a 64-bit masked popcount.
template <int G>
__device__ __forceinline__ void g_emit(const uint64_t (&keep)[grp::GShape<G>::W], int n, bool emit,
                                       int k, int b, int N, int off, int pos_off,
                                       const int8_t *par, uint64_t *child,
                                       const uint8_t *klist, int32_t *__restrict__ kept_index,
                                       int32_t *__restrict__ retrieve_index,
                                       int32_t *__restrict__ positions,
                                       int32_t *__restrict__ next_token,
                                       int32_t *__restrict__ next_sibling,
                                       uint64_t *__restrict__ tree_mask, const uint8_t *slot_of = nullptr)
{
    constexpr int W = GShape<G>::W;
    if constexpr (W == 1) {
        if (slot_of != nullptr) {
            const int g = gl<G>();
            const int kk = emit ? k : 0;
            // small kept sets (the cost-effective cut: k* ≈ 8): first child and next sibling by a
            // scan of the later slots (children and later siblings have larger node indices, so
            // larger slots) — no shared atomics; large kept sets build child masks instead
            constexpr int kScanMax = 16;
            const bool scan = kk <= kScanMax;
            if (!scan)
                for (int s = g; s < kk; s += G) child[s] = 0ull;
            __syncwarp();   // (outside the group-dependent branches: every lane of the warp arrives)
            if (!scan) {
                for (int s = g; s < kk; s += G) {
                    const int i = klist[s];
                    if (i > 0)
                        atomicOr(reinterpret_cast<unsigned long long *>(&child[slot_of[par[i]]]), 1ull << s);
                }
            }
            __syncwarp();
            for (int s = g; s < kk; s += G) {
                const int i = klist[s];
                uint64_t row = 1ull << s;
                int depth = 0;
                for (int a = par[i]; a >= 0; a = par[a]) {   // strict ancestors, all kept
                    depth++;
                    row |= 1ull << slot_of[a];
                }
                int nt = -1, ns = -1;
                if (scan) {
                    const int p = i > 0 ? par[i] : -2;
                    for (int t = s + 1; t < kk; t++) {
                        const int pj = par[klist[t]];
                        if (nt < 0 && pj == i) nt = t;
                        if (ns < 0 && pj == p) ns = t;
                    }
                } else {
                    const uint64_t cm = child[s];
                    nt = cm ? __ffsll((long long)cm) - 1 : -1;
                    if (i > 0) {
                        const uint64_t sib = child[slot_of[par[i]]] & (s >= 63 ? 0ull : (~0ull << (s + 1)));
                        ns = sib ? __ffsll((long long)sib) - 1 : -1;
                    }
                }
                const int rowi = off + s;
                if (kept_index) kept_index[rowi] = i;
                if (retrieve_index) retrieve_index[rowi] = b * N + i;
                if (positions) positions[rowi] = pos_off + depth;
                if (next_token) next_token[rowi] = nt;
                if (next_sibling) next_sibling[rowi] = ns;
                if (tree_mask) tree_mask[rowi] = row;
            }
            return;
        }
    }
    const int g = gl<G>();
    const int base = g * NP;
    const int kk = emit ? k : 0;
    if (emit) {
        for (int s = g; s < kk; s += G)
#pragma unroll
            for (int w = 0; w < W; w++) child[s * W + w] = 0ull;
    }
    __syncwarp();
    for (int s = g; s < kk; s += G) {
        const int i = klist[s];
        if (i > 0) {
            const int ps = popc_below_w<W>(keep, par[i]);
            atomicOr(reinterpret_cast<unsigned long long *>(&child[ps * W + (s >> 6)]), 1ull << (s & 63));
        }
    }
    __syncwarp();
    for (int s = g; s < kk; s += G) {
        const int i = klist[s];
        uint64_t row[W];
#pragma unroll
        for (int w = 0; w < W; w++) row[w] = 0ull;
        int depth = -1;
        for (int a = i; a >= 0; a = par[a]) {             // ancestor-or-self chain
            depth++;
            const int sa = popc_below_w<W>(keep, a);
#pragma unroll
            for (int w = 0; w < W; w++)
                if ((sa >> 6) == w) row[w] |= 1ull << (sa & 63);
        }
        int nt = -1, ns = -1;
#pragma unroll
        for (int w = W - 1; w >= 0; w--) {
            const uint64_t cm = child[s * W + w];
            if (cm) nt = w * 64 + __ffsll((long long)cm) - 1;
        }
        if (i > 0) {
            const int ps = popc_below_w<W>(keep, par[i]);
#pragma unroll
            for (int w = W - 1; w >= 0; w--) {
                uint64_t cm = child[ps * W + w];
                const int lo = w * 64;
                const uint64_t above = (s + 1 <= lo) ? ~0ull : (s + 1 >= lo + 64 ? 0ull : (~0ull << (s + 1 - lo)));
                cm &= above;
                if (cm) ns = lo + __ffsll((long long)cm) - 1;
            }
        }
        const int rowi = off + s;
        if (kept_index) kept_index[rowi] = i;
        if (retrieve_index) retrieve_index[rowi] = b * N + i;
        if (positions) positions[rowi] = pos_off + depth;   // depth = ancestor steps
        if (next_token) next_token[rowi] = nt;
        if (next_sibling) next_sibling[rowi] = ns;
        if (tree_mask) {
#pragma unroll
            for (int w = 0; w < W; w++) tree_mask[(size_t)rowi * W + w] = row[w];
        }
    }
}

}  // namespace grp
}  // namespace evict
