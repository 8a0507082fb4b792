// union_emit.cu — k_union_emit: A6 (verify-tree emit) + A7 (expert union) + folded A9 of the
// throughput path, after k_select_g (A1–A5) and k_scan_offsets (packed offsets) have run.
//
// Scope: u8 top-8 routing ids, E = 128, L ≤ 64, N ≤ 64 (the C5 / serving configuration:
// PAPER.md:84–88 Eq. 5 for the union, PAPER.md:48, 92 / Fig. 4(c) for the emit).
//
// One warp per tree, trees strided over the persistent grid (no look-back: the offsets are
// already scanned), software-pipelined across a warp's trees: tree t+1's metadata loads are
// issued when tree t starts, and its first batch of kept rows (kUEB rows) right after tree t's
// byte stores, so both round trips overlap tree t's read-back and emit.
//
// A7 — lane-owned flag columns.  Lane c owns byte column c of a per-warp 8 KB block of 32 rows
// × 256 B: row r = e >> 2 holds, at byte 4c + (e & 3), the flag of expert e for lane c's layer
// in region 0 (bytes 0–127: layer c) and region 1 (bytes 128–255: layer 32 + c, or the half
// (c & 1) of layer 32 + c/2 when L ≤ 48).  A store's bank is therefore c — every byte-store
// instruction of the warp is conflict-free whatever the ids (one wavefront per 32 ids; the
// round-1 layout split a layer over two lanes on one bank group, ≈ 2 wavefronts).  The byte
// address of id e is one PRMT of two per-word precomputed vectors: lo = (w & 0x03030303) | 4c
// and hi = (w >> 2) & 0x1F1F1F1F give (e >> 2) << 8 | (4c + (e & 3)).
// Marker epochs: tree t stores 1 << (t mod 4) and its read-back counts only that bit; the
// block is cleared after every fourth read-back.  Read-back: lane (q = lane & 7, r0 = lane >> 3)
// loads rows r0 + 4j (j < 8) as 16-byte vectors (4 wavefronts per instruction, conflict-free:
// 8 lanes per 128-byte phase), sums marker bits bytewise per column, then two xor-shuffles over
// r0 and one IDP4A per layer give the union size of every layer.
//
// A6 — warp-wide, nodes i = lane and lane + 32: slots by popc below the node; ancestor-or-self
// rows by pointer jumping in slot space (A(i) ∪= A(J(i)), J(i) = J(J(i)); ⌈log2(depth+1)⌉
// rounds), depth = |A| − 1; kept siblings via __match_any_sync on the parent id (same half)
// and per-warp first-child tables (tagged with a per-warp tree counter, never cleared) for the
// first child of a node and for the first sibling in the other half.
#include <cuda_runtime.h>
#include <stdint.h>

#include "evict.h"
#include "evict_launch.h"
#include "evict_tree.cuh"

namespace evict {

constexpr int kUEWarps = 4;          // warps per CTA (the PRMT store address keeps bit 15 clear: see ue_store4)
constexpr int kUEFlagBytes = 8192;   // per warp
constexpr int kUETabBytes = 512;     // per warp: first-child tables F0[64], F1[64] (uint32)
constexpr int kUEKlistBytes = 64;    // per warp: slot → node
constexpr int kUEB = 4;              // kept rows per load batch

// folded A9 accumulators (per CTA), flushed to the evict_batch_stats vector when the CTA ends
struct UEStats {
    unsigned sc[kUEWarps][4];   // per warp: trees, Σk*, Σn, errored trees
    double d[kUEWarps][2];      // per warp: Σe_hat, Σutility (status 0)
    unsigned hist[65];          // k* histogram (N ≤ 64), bin 0 = errored trees
    unsigned lay[64];           // Σ union_count per layer (status 0)
};


__device__ __forceinline__ uint32_t ue_prmt(uint32_t a, uint32_t b, uint32_t sel)
{
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// byte stores of the 4 ids of w.  Warp w's block is bytes [8192·w, 8192·(w+1)) of the dynamic
// shared memory (w < 4), so 32·w fills bits 5–6 of the row byte and the PRMT result is the
// store's offset from the dynamic block; the block's own shared address (a link-time constant)
// goes into the STS immediate: one PRMT + one STS per id.  hb = 32·w·0x01010101.
// Selector for id j: byte 0 = lo.b_j, byte 1 = hi.b_j, bytes 2–3 = sign of hi.b_j (= 0: hi < 128).
__device__ __forceinline__ void ue_store4(uint32_t base, uint32_t hb, uint32_t w, uint32_t cb, uint32_t marker)
{
    const uint32_t lo = (w & 0x03030303u) | cb;
    const uint32_t hi = ((w >> 2) & 0x1F1F1F1Fu) | hb;
    sts_u8(base + ue_prmt(lo, hi, 0xCC40u), marker);
    sts_u8(base + ue_prmt(lo, hi, 0xDD51u), marker);
    sts_u8(base + ue_prmt(lo, hi, 0xEE62u), marker);
    sts_u8(base + ue_prmt(lo, hi, 0xFF73u), marker);
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src)
{
    const uint32_t lo = __shfl_sync(kFull, (uint32_t)v, src), hi = __shfl_sync(kFull, (uint32_t)(v >> 32), src);
    return ((uint64_t)hi << 32) | lo;
}

// A batch of kUEB kept rows of one tree in registers: x0 = region-0 ids (8 bytes: layer `lane`),
// x1/x2 = region-1 ids (MODE 1: 4 bytes, half lane&1 of layer 32 + lane/2; MODE 2: 8 bytes)
template <int MODE>
struct UEBatch {
    uint2 x0[kUEB];
    uint32_t x1[kUEB];
    uint32_t x2[kUEB];
};

// per-tree state: metadata + per-lane row pointers.  Every load is unconditional (clamped
// addresses; validity applied where a value is used) so no select waits on a load in flight.
struct UETree {
    int b, k;
    uint32_t st;
    uint64_t keep;
    int par0, par1;                // raw parent words of nodes lane, lane + 32 (valid: node < N)
    int off, pos_off;              // packed row offset, position offset
    float ehat, util;              // A9 inputs (lane 0)
    int n;
    uint32_t ro0, ro1;             // lane j: byte offset of slot j's / slot j+32's row
    const uint8_t *p0, *p1;        // this lane's part of the tree's node-row block, regions 0 / 1
};

// MODE: region 1 layout — 0 none (L ≤ 32), 1 half-layer columns (32 < L ≤ 48), 2 layer columns (48 < L ≤ 64)
template <int MODE>
__global__ void __launch_bounds__(kUEWarps * 32, 6) k_union_emit(evict_trees_t tr, evict_routing_t rt,
                                                                evict_fused_out_t out)
{
    // static shared memory (36 KB < 48 KB): the flag block's address is a link-time constant,
    // so it rides in the STS immediate (ue_store4)
    __shared__ __align__(16) uint8_t s_flags[kUEWarps * kUEFlagBytes];
    __shared__ __align__(16) uint32_t s_tab[kUEWarps * kUETabBytes / 4];
    __shared__ __align__(16) uint8_t s_klist[kUEWarps * kUEKlistBytes];
    __shared__ __align__(16) UEStats s_stats;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    uint8_t *flags = s_flags + (size_t)warp * kUEFlagBytes;
    uint32_t *ftab = s_tab + warp * (kUETabBytes / 4);
    uint8_t *klist = s_klist + warp * kUEKlistBytes;
    UEStats *fs = &s_stats;
    const bool fstats = out.stats != nullptr;
    {
        uint4 *f4 = reinterpret_cast<uint4 *>(flags);
        for (int i = lane; i < kUEFlagBytes / 16; i += 32) f4[i] = make_uint4(0u, 0u, 0u, 0u);
        for (int i = lane; i < kUETabBytes / 4; i += 32) ftab[i] = 0u;
        if (fstats) {
            uint32_t *z = reinterpret_cast<uint32_t *>(fs);
            for (int i = threadIdx.x; i < (int)(sizeof(UEStats) / 4); i += blockDim.x) z[i] = 0u;
            __syncthreads();
        }
        __syncwarp();
    }
    const int N = tr.max_nodes, L = rt.num_layers;
    const uint32_t rowB = (uint32_t)L * 8u;
    const uint8_t *ids = reinterpret_cast<const uint8_t *>(rt.ids);
    const unsigned long long *keep_bits = reinterpret_cast<const unsigned long long *>(out.keep_bits);
    const uint32_t dsb = (uint32_t)__cvta_generic_to_shared(s_flags);   // STS immediate
    const uint32_t fb = dsb + (uint32_t)warp * kUEFlagBytes;
    const uint32_t hb = (32u * (uint32_t)warp) * 0x01010101u;
    const uint32_t cb0 = (4u * (uint32_t)lane) * 0x01010101u;
    const uint32_t cb1 = (128u + 4u * (uint32_t)lane) * 0x01010101u;
    const int q = lane & 7, r0 = lane >> 3;
    // this lane's row parts: region 0 = bytes 8·lane (layer lane); region 1 = bytes 256 + 4·lane
    // (MODE 1) or 256 + 8·lane (MODE 2)
    // (lanes past the layers re-read byte 0 / 256 of the row: their flags land in columns of
    // layers ≥ L, which are never counted, and the bytes are ids of the same kept row)
    const bool ld0 = lane < L;
    const bool ld1 = MODE == 1 ? lane < 2 * (L - 32) : (MODE == 2 ? lane < L - 32 : false);
    const uint32_t lo0c = ld0 ? 8u * (uint32_t)lane : 0u;
    const uint32_t lo1c = ld1 ? (MODE == 1 ? 256u + 4u * (uint32_t)lane : 256u + 8u * (uint32_t)lane) : 256u;
    // output layers of this lane after the read-back (r0 = 0: region 0; r0 = 1: region 1)
    int lay[4];
#pragma unroll
    for (int m = 0; m < 4; m++)
        lay[m] = r0 == 0 ? 4 * q + m : (r0 == 1 ? (MODE == 1 ? (m < 2 ? 32 + 2 * q + m : 64) : (MODE == 2 ? 32 + 4 * q + m : 64)) : 64);
    int ep = 0;
    uint32_t tag = 0;
    uint32_t lsum[4] = {0u, 0u, 0u, 0u};   // A9 per-layer sums of this lane's output layers
    const int GW = gridDim.x * kUEWarps;

    auto fetch_meta = [&](UETree &t, int b) {
        t.b = b;
        const int bc = b < tr.batch ? b : tr.batch - 1;
        t.k = __ldg(out.k_star + bc);
        t.st = __ldg(out.status + bc);
        t.keep = __ldg(keep_bits + bc);
        const int32_t *prow = tr.parent + (size_t)bc * N;
        t.par0 = __ldg(prow + (lane < N ? lane : 0));
        t.par1 = __ldg(prow + (lane + 32 < N ? lane + 32 : 0));
    };
    // the rest of a tree's inputs, issued when the tree starts (used by its emit / statistics)
    auto fetch_late = [&](UETree &t) {
        const int bc = t.b;
        t.off = __ldg(out.verify_offsets + bc);
        t.pos_off = out.pos_offset ? __ldg(out.pos_offset + bc) : 0;
        if (fstats) {
            t.ehat = __ldg(out.e_hat + bc);
            t.util = __ldg(out.utility + bc);
            t.n = tr.n_nodes ? __ldg(tr.n_nodes + bc) : N;
        }
    };
    // slot → node list (shared, one tree at a time) and the per-lane row offsets / pointers
    auto prepare = [&](UETree &t) {
        const uint32_t klo = (uint32_t)t.keep, khi = (uint32_t)(t.keep >> 32);
        if ((klo >> lane) & 1u) klist[__popc(klo & ((1u << lane) - 1u))] = (uint8_t)lane;
        if ((khi >> lane) & 1u) klist[__popc(klo) + __popc(khi & ((1u << lane) - 1u))] = (uint8_t)(lane + 32);
        __syncwarp();
        t.ro0 = (uint32_t)klist[lane] * rowB;
        t.ro1 = (uint32_t)klist[32 + lane] * rowB;
        const uint8_t *tb = ids + (size_t)t.b * N * rowB;
        t.p0 = tb + lo0c;
        t.p1 = tb + lo1c;
    };
    auto load_row = [&](const UETree &t, int j, UEBatch<MODE> &v, int u) {
        const uint32_t o = __shfl_sync(kFull, j < 32 ? t.ro0 : t.ro1, j & 31);
        v.x0[u] = __ldg(reinterpret_cast<const uint2 *>(t.p0 + o));
        if constexpr (MODE == 1) {
            v.x1[u] = __ldg(reinterpret_cast<const uint32_t *>(t.p1 + o));
        } else if constexpr (MODE == 2) {
            const uint2 y = __ldg(reinterpret_cast<const uint2 *>(t.p1 + o));
            v.x1[u] = y.x;
            v.x2[u] = y.y;
        }
    };
    // rows j0 .. j0 + kUEB − 1 (a slot past k re-reads row k − 1; its stores are skipped)
    auto load_batch = [&](const UETree &t, int j0, UEBatch<MODE> &v) {
#pragma unroll
        for (int u = 0; u < kUEB; u++) load_row(t, min(j0 + u, t.k - 1), v, u);
    };
    auto store_batch = [&](int n, const UEBatch<MODE> &v, uint32_t marker, uint32_t &badw) {
#pragma unroll
        for (int u = 0; u < kUEB; u++) {
            if (u >= n) break;   // warp-uniform
            badw |= v.x0[u].x | v.x0[u].y;
            ue_store4(dsb, hb, v.x0[u].x, cb0, marker);
            ue_store4(dsb, hb, v.x0[u].y, cb0, marker);
            if constexpr (MODE >= 1) {
                badw |= v.x1[u];
                ue_store4(dsb, hb, v.x1[u], cb1, marker);
            }
            if constexpr (MODE == 2) {
                badw |= v.x2[u];
                ue_store4(dsb, hb, v.x2[u], cb1, marker);
            }
        }
    };

    UETree cur, nxt;
    UEBatch<MODE> va, vb;
    fetch_meta(cur, blockIdx.x * kUEWarps + warp);
    if (cur.b < tr.batch) {
        prepare(cur);
        if (cur.st == 0u && cur.k > 0) load_batch(cur, 0, va);
    }
#pragma unroll 1
    while (cur.b < tr.batch) {
        const int b = cur.b, k = cur.k;
        fetch_meta(nxt, b + GW);                 // in flight during this tree
        fetch_late(cur);
        uint32_t st = cur.st;
        const bool run = st == 0u && k > 0;
        uint32_t badw = 0u;
        if (run) {
            // ---------------- A7 stores (batch A was loaded during the previous tree)
            const uint32_t marker = 1u << ep;
            if (k > kUEB) load_batch(cur, kUEB, vb);
            store_batch(k, va, marker, badw);
#pragma unroll 1
            for (int j0 = kUEB; j0 < k; j0 += kUEB) {
                if (j0 > kUEB) load_batch(cur, j0, vb);
                store_batch(k - j0, vb, marker, badw);
            }
        }
        // ---------------- next tree: slot list, row pointers, first row batch
        if (nxt.b < tr.batch) {
            __syncwarp();                        // this tree's klist reads are done
            prepare(nxt);
            if (nxt.st == 0u && nxt.k > 0) load_batch(nxt, 0, va);
        }
        uint32_t cnt[4] = {0u, 0u, 0u, 0u};
        if (run) {
            __syncwarp();
            // read-back: rows r0 + 4j, byte columns 16q..16q+15 of both regions
            const uint32_t mk = 0x01010101u << ep;
            const bool clear = ep == 3;
            uint32_t a0 = 0u, a1 = 0u, a2 = 0u, a3 = 0u, c0 = 0u, c1 = 0u, c2 = 0u, c3 = 0u;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const uint32_t ra = fb + 256u * (uint32_t)(r0 + 4 * j) + 16u * (uint32_t)q;
                const uint4 x = lds_v4(ra);
                a0 += x.x & mk; a1 += x.y & mk; a2 += x.z & mk; a3 += x.w & mk;
                if constexpr (MODE == 1) {
                    const uint4 y = lds_v4(ra + 128u);
                    c0 += (y.x | y.y) & mk;   // layer 32 + 2q (both halves)
                    c1 += (y.z | y.w) & mk;   // layer 33 + 2q
                } else if constexpr (MODE == 2) {
                    const uint4 y = lds_v4(ra + 128u);
                    c0 += y.x & mk; c1 += y.y & mk; c2 += y.z & mk; c3 += y.w & mk;
                }
                if (clear) {
                    sts_v4_zero(ra);
                    if constexpr (MODE >= 1) sts_v4_zero(ra + 128u);
                }
            }
            // bytes ≤ 8 markers each after the shift; the sum over r0 ≤ 32 per byte
            a0 >>= ep; a1 >>= ep; a2 >>= ep; a3 >>= ep;
            a0 += __shfl_xor_sync(kFull, a0, 8);  a1 += __shfl_xor_sync(kFull, a1, 8);
            a2 += __shfl_xor_sync(kFull, a2, 8);  a3 += __shfl_xor_sync(kFull, a3, 8);
            a0 += __shfl_xor_sync(kFull, a0, 16); a1 += __shfl_xor_sync(kFull, a1, 16);
            a2 += __shfl_xor_sync(kFull, a2, 16); a3 += __shfl_xor_sync(kFull, a3, 16);
            if constexpr (MODE >= 1) {
                c0 >>= ep; c1 >>= ep;
                c0 += __shfl_xor_sync(kFull, c0, 8);  c1 += __shfl_xor_sync(kFull, c1, 8);
                c0 += __shfl_xor_sync(kFull, c0, 16); c1 += __shfl_xor_sync(kFull, c1, 16);
            }
            if constexpr (MODE == 2) {
                c2 >>= ep; c3 >>= ep;
                c2 += __shfl_xor_sync(kFull, c2, 8);  c3 += __shfl_xor_sync(kFull, c3, 8);
                c2 += __shfl_xor_sync(kFull, c2, 16); c3 += __shfl_xor_sync(kFull, c3, 16);
            }
            ep = (ep + 1) & 3;
            const uint32_t w0 = r0 == 0 ? a0 : c0, w1 = r0 == 0 ? a1 : c1;
            const uint32_t w2 = r0 == 0 ? a2 : c2, w3 = r0 == 0 ? a3 : c3;
            cnt[0] = lay[0] < L ? (uint32_t)__dp4a(w0, 0x01010101u, 0u) : 0u;
            cnt[1] = lay[1] < L ? (uint32_t)__dp4a(w1, 0x01010101u, 0u) : 0u;
            cnt[2] = lay[2] < L ? (uint32_t)__dp4a(w2, 0x01010101u, 0u) : 0u;
            cnt[3] = lay[3] < L ? (uint32_t)__dp4a(w3, 0x01010101u, 0u) : 0u;
            if (__any_sync(kFull, badw & 0x80808080u)) {
                st |= EVICT_TREE_BAD_EXPERT;
                cnt[0] = cnt[1] = cnt[2] = cnt[3] = 0u;
            }
        }
        // union counts (zeros for an errored tree): lanes 0–7 region 0, lanes 8–15 region 1
        {
            int32_t *uc = out.union_count + (size_t)b * L;
#pragma unroll
            for (int m = 0; m < 4; m++)
                if (lay[m] < L) uc[lay[m]] = (int)cnt[m];
            const int tot = __reduce_add_sync(kFull, (int)(cnt[0] + cnt[1] + cnt[2] + cnt[3]));
            if (out.union_total && lane == 0) out.union_total[b] = tot;
            if (fstats && st == 0u) {
#pragma unroll
                for (int m = 0; m < 4; m++) lsum[m] += cnt[m];
            }
        }
        if (lane == 0 && (st & EVICT_TREE_BAD_EXPERT)) out.status[b] = st;
        // ---------------- A9 scalars
        if (fstats && lane == 0) {
            unsigned *wsc = fs->sc[warp];
            wsc[0] += 1u;
            if (st) {
                wsc[3] += 1u;
                atomicAdd(&fs->hist[0], 1u);
            } else {
                wsc[1] += (unsigned)k;
                wsc[2] += (unsigned)cur.n;
                fs->d[warp][0] += (double)cur.ehat;
                fs->d[warp][1] += (double)cur.util;
                atomicAdd(&fs->hist[k], 1u);
            }
        }
        // ---------------- A6 (k > 0 ⇔ the select succeeded; BAD_EXPERT trees still own their rows)
        if (k > 0) {
            const uint64_t keep = cur.keep;
            const int par0 = lane < N ? cur.par0 : -1, par1 = lane + 32 < N ? cur.par1 : -1;
            const uint32_t klo = (uint32_t)keep, khi = (uint32_t)(keep >> 32);
            const unsigned below = (1u << lane) - 1u;
            const bool kp0 = (klo >> lane) & 1u, kp1 = (khi >> lane) & 1u;
            const int s0 = __popc(klo & below);
            const int s1 = __popc(klo) + __popc(khi & below);
            const int off = cur.off, pos_off = cur.pos_off;
            const bool hi_any = khi != 0u;   // nodes ≥ 32 kept (warp-uniform)
            uint64_t A0 = kp0 ? 1ull << s0 : 0ull, A1 = kp1 ? 1ull << s1 : 0ull;
            int J0 = kp0 ? par0 : -1, J1 = kp1 ? par1 : -1;   // root: par = −1
            if (!hi_any) {
                while (__any_sync(kFull, J0 >= 0)) {
                    const int src = J0 & 31;
                    const uint64_t x = shfl64(A0, src);
                    const int jx = __shfl_sync(kFull, J0, src);
                    if (J0 >= 0) { A0 |= x; J0 = jx; }
                }
            } else {
                while (__any_sync(kFull, J0 >= 0 || J1 >= 0)) {
                    const int s0r = J0 & 31, s1r = J1 & 31;
                    const uint64_t x0 = shfl64(A0, s0r);
                    const int j0x = __shfl_sync(kFull, J0, s0r);
                    const uint64_t y0 = shfl64(A0, s1r), y1 = shfl64(A1, s1r);
                    const int jy0 = __shfl_sync(kFull, J0, s1r), jy1 = __shfl_sync(kFull, J1, s1r);
                    if (J0 >= 0) { A0 |= x0; J0 = j0x; }   // half-0 parents are < 32
                    if (J1 >= 0) {
                        const bool h = J1 >= 32;
                        A1 |= h ? y1 : y0;
                        J1 = h ? jy1 : jy0;
                    }
                }
            }
            // siblings: same-parent groups per half; group leaders record first children
            if (++tag == 0x01000000u) {   // tag wrap: clear the tables once per 2^24 trees
                for (int i = lane; i < kUETabBytes / 4; i += 32) ftab[i] = 0u;
                tag = 1u;
                __syncwarp();
            }
            const uint32_t tg = tag << 8;
            const bool c0k = kp0 && lane > 0;
            const unsigned M0 = __match_any_sync(kFull, c0k ? par0 : 1024 + lane);
            if (c0k && (M0 & below) == 0u) ftab[par0] = tg | (uint32_t)lane;
            unsigned M1 = 0u;
            if (hi_any) {
                M1 = __match_any_sync(kFull, kp1 ? par1 : 1024 + lane);
                if (kp1 && (M1 & below) == 0u) ftab[64 + par1] = tg | (uint32_t)(lane + 32);
            }
            __syncwarp();
            auto slot_of = [&](int node) { return __popcll(keep & ((1ull << node) - 1ull)); };
            auto first_child = [&](int p) {
                const uint32_t f0 = ftab[p], f1 = ftab[64 + p];
                return (f0 >> 8) == tag ? (int)(f0 & 0xffu) : ((f1 >> 8) == tag ? (int)(f1 & 0xffu) : -1);
            };
            if (kp0) {
                const int row = off + s0;
                const int fc = first_child(lane);
                const unsigned above = M0 & ~(below | (1u << lane));
                int nsib = -1;
                if (lane > 0) {
                    if (above) nsib = __ffs(above) - 1;
                    else {
                        const uint32_t f1 = ftab[64 + par0];
                        nsib = (f1 >> 8) == tag ? (int)(f1 & 0xffu) : -1;
                    }
                }
                if (out.kept_index) out.kept_index[row] = lane;
                if (out.retrieve_index) out.retrieve_index[row] = b * N + lane;
                if (out.positions) out.positions[row] = pos_off + __popcll(A0) - 1;
                if (out.next_token) out.next_token[row] = fc < 0 ? -1 : slot_of(fc);
                if (out.next_sibling) out.next_sibling[row] = nsib < 0 ? -1 : slot_of(nsib);
                if (out.tree_mask) out.tree_mask[row] = A0;
            }
            if (hi_any && kp1) {
                const int row = off + s1;
                const int i = lane + 32;
                const int fc = first_child(i);
                const unsigned ab1 = M1 & ~(below | (1u << lane));
                const int nsib = ab1 ? 32 + __ffs(ab1) - 1 : -1;
                if (out.kept_index) out.kept_index[row] = i;
                if (out.retrieve_index) out.retrieve_index[row] = b * N + i;
                if (out.positions) out.positions[row] = pos_off + __popcll(A1) - 1;
                if (out.next_token) out.next_token[row] = fc < 0 ? -1 : slot_of(fc);
                if (out.next_sibling) out.next_sibling[row] = nsib < 0 ? -1 : slot_of(nsib);
                if (out.tree_mask) out.tree_mask[row] = A1;
            }
        }
        __syncwarp();
        cur = nxt;
    }
    if (fstats) {
        // per-lane layer sums → CTA sums → the global statistics vector (evict_batch_stats layout)
#pragma unroll
        for (int m = 0; m < 4; m++)
            if (lay[m] < L && lsum[m]) atomicAdd(&fs->lay[lay[m]], lsum[m]);
        __syncthreads();
        unsigned long long *gs = reinterpret_cast<unsigned long long *>(out.stats);
        if (threadIdx.x == 0) {
            unsigned long long su = 0, sc[4] = {0ull, 0ull, 0ull, 0ull};
            for (int l = 0; l < L; l++) su += fs->lay[l];
            for (int w = 0; w < kUEWarps; w++)
                for (int i = 0; i < 4; i++) sc[i] += fs->sc[w][i];
            if (sc[0]) atomicAdd(gs + 0, sc[0]);
            if (sc[1]) atomicAdd(gs + 1, sc[1]);
            if (sc[2]) atomicAdd(gs + 2, sc[2]);
            if (su) atomicAdd(gs + 3, su);
            if (sc[3]) atomicAdd(gs + 4, sc[3]);
            double de = 0.0, du = 0.0;
            for (int w = 0; w < kUEWarps; w++) { de += fs->d[w][0]; du += fs->d[w][1]; }
            atomicAdd(out.dstats + 0, de);
            atomicAdd(out.dstats + 1, du);
        }
        for (int i = threadIdx.x; i <= N; i += blockDim.x)
            if (fs->hist[i]) atomicAdd(gs + 5 + i, (unsigned long long)fs->hist[i]);
        for (int l = threadIdx.x; l < L; l += blockDim.x)
            if (fs->lay[l]) atomicAdd(gs + 6 + N + l, (unsigned long long)fs->lay[l]);
    }
}

evict_status_t launch_union_emit(const evict_trees_t *tr, const evict_routing_t *rt, const evict_fused_out_t *o,
                                 cudaStream_t s)
{
    const int L = rt->num_layers;
    auto uk = L <= 32 ? k_union_emit<0> : (L <= 48 ? k_union_emit<1> : k_union_emit<2>);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, uk, kUEWarps * 32, 0);
    if (per_sm < 1) per_sm = 1;
    const long need = ((long)tr->batch + kUEWarps - 1) / kUEWarps;
    const long grid = (long)dev_sms() * per_sm;
    uk<<<(int)(grid < need ? grid : need), kUEWarps * 32, 0, s>>>(*tr, *rt, *o);
    return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA;
}

}  // namespace evict
