// curve.cu — NEXT-1: the prefix-union curve along the ranking and the offline
// cost profile built from it (Fig. 1:
// the experts a verify pass activates grow with the number of verified
// tokens; C(k) is profiled offline per k).
//
// k_union_curve: one warp per tree, lane = layer (rounds of 32 layers), the
// layer's expert set in registers (4 words for ids of E ≤ 128; 8 words for ids or masks of
// E ≤ 256), nodes visited in ranking order: each node ORs its ids into its
// layers' sets, counts the new bits, and a warp sum gives curve[k−1].  No
// shared memory, no atomics; each lane owns its layers exclusively.
// k_profile_sum / k_profile_cost: warp per tree row (lane = k), int64 column
// sums in registers → global atomics, then C(k) = c0 + c_union·Ū(k) + c_tok·k.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "evict.h"
#include "evict_launch.h"

namespace evict {
namespace curve {

constexpr int kWarpsC = 8;

// OR expert e into an NW-word set (NW = 4: E ≤ 128, NW = 8: E ≤ 256); returns 1 if it was new.
template <int NW>
__device__ __forceinline__ uint32_t set4(uint32_t (&w)[NW], uint32_t e)
{
    const uint32_t bit = 1u << (e & 31u), q = e >> 5;
    uint32_t cur = 0u;
#pragma unroll
    for (int i = 0; i < NW; i++) cur |= (q == (uint32_t)i) ? w[i] : 0u;
#pragma unroll
    for (int i = 0; i < NW; i++) w[i] |= (q == (uint32_t)i) ? bit : 0u;
    return (cur & bit) ? 0u : 1u;
}

// PTX shl.b32 clamps shift amounts ≥ 32 to 32 (result 0)
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t sh)
{
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(sh));
    return r;
}

template <int IDF, int R, int NW>
__global__ void __launch_bounds__(kWarpsC * 32) k_union_curve(evict_trees_t tr, const int32_t *order,
                                                              evict_routing_t rt, int32_t *curve,
                                                              int32_t *curve_layer, uint32_t *status)
{
    static_assert(IDF != EVICT_ID_MASK || NW == 8, "mask sets span 256 experts");
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * kWarpsC + (threadIdx.x >> 5);
    if (b >= tr.batch) return;
    const int N = tr.max_nodes, L = rt.num_layers, K = rt.top_k, E = rt.num_experts;
    const int n = tr.n_nodes ? __ldg(tr.n_nodes + b) : N;
    int32_t *crow = curve + (size_t)b * N;
    int32_t *lrow = curve_layer ? curve_layer + (size_t)b * N * L : nullptr;
    uint32_t st = (n < 1 || n > N) ? EVICT_TREE_BAD_SIZE : 0u;
    uint32_t w[R][NW];
    int per[R];
#pragma unroll
    for (int c = 0; c < R; c++) {
        per[c] = 0;
#pragma unroll
        for (int i = 0; i < NW; i++) w[c][i] = 0u;
    }
    int tot = 0, kdone = 0;
    const int EW = (E + 63) >> 6;
    if constexpr (IDF == EVICT_ID_U8) {
        if (!st && K == 8) {
            // u8 top-8 fast path: the order row lives in registers, and the routing rows of D
            // nodes are loaded before any is processed (D independent 8-byte loads per lane
            // and layer round in flight instead of one dependent chain per node)
            constexpr int D = 8;
            const int32_t *orow = order + (size_t)b * N;
            int oreg[4];
#pragma unroll
            for (int i = 0; i < 4; i++) oreg[i] = lane + 32 * i < n ? __ldg(orow + lane + 32 * i) : 0;
            const uint8_t *base = reinterpret_cast<const uint8_t *>(rt.ids) + (size_t)b * N * L * 8;
            for (int j0 = 0; j0 < n; j0 += D) {
                uint2 x[D][R];
                bool badk = false;
#pragma unroll
                for (int h = 0; h < D; h++) {
                    const int j = j0 + h;
                    const int sel = (j >> 5) & 3;
                    const int o = sel == 0 ? oreg[0] : sel == 1 ? oreg[1] : sel == 2 ? oreg[2] : oreg[3];
                    const int v = __shfl_sync(0xffffffffu, o, j & 31);
                    bool ok = j < n;
                    if (ok && (v < 0 || v >= n)) { badk = true; ok = false; }
#pragma unroll
                    for (int c = 0; c < R; c++) {
                        const int l = lane + 32 * c;
                        x[h][c] = (ok && l < L) ? __ldg(reinterpret_cast<const uint2 *>(base + ((size_t)v * L + l) * 8))
                                                : make_uint2(0u, 0u);
                    }
                }
                if (badk) { st |= EVICT_TREE_BAD_KEEP; break; }    // v is warp-uniform
                uint32_t bad = 0;
#pragma unroll
                for (int h = 0; h < D; h++) {
                    const int j = j0 + h;
                    if (j >= n) break;
                    uint32_t nw = 0;
#pragma unroll
                    for (int c = 0; c < R; c++) {
                        const int l = lane + 32 * c;
                        if (l >= L) continue;
                        // one-hot words by clamped shifts: shl.b32 by ≥ 32 (incl. a negative
                        // offset seen unsigned) is 0, so word i takes bit e − 32i only when
                        // 32i ≤ e < 32i + 32 — no selects, no per-id "was it new" test
                        uint32_t m[NW];
#pragma unroll
                        for (int i = 0; i < NW; i++) m[i] = 0u;
#pragma unroll
                        for (int q = 0; q < 8; q++) {
                            const uint32_t e = __byte_perm(q < 4 ? x[h][c].x : x[h][c].y, 0, 0x4440 | (q & 3));
                            bad |= e >= (uint32_t)E;
#pragma unroll
                            for (int i = 0; i < NW; i++) m[i] |= shl_clamp(1u, e - 32u * i);
                        }
                        int cnt = 0;
#pragma unroll
                        for (int i = 0; i < NW; i++) {
                            w[c][i] |= m[i];
                            cnt += __popc(w[c][i]);
                        }
                        nw += (uint32_t)(cnt - per[c]);
                        per[c] = cnt;
                        if (lrow) lrow[(size_t)j * L + l] = per[c];
                    }
                    tot += (int)__reduce_add_sync(0xffffffffu, nw);
                    if (lane == 0) crow[j] = tot;
                }
                if (__any_sync(0xffffffffu, bad)) { st |= EVICT_TREE_BAD_EXPERT; break; }
                kdone = min(n, j0 + D);
            }
            goto finish;
        }
    }
    if (!st) {
        for (int j = 0; j < n; j++) {
            const int v = __ldg(order + (size_t)b * N + j);
            if (v < 0 || v >= n) { st |= EVICT_TREE_BAD_KEEP; break; }
            uint32_t nw = 0, bad = 0;
#pragma unroll
            for (int c = 0; c < R; c++) {
                const int l = lane + 32 * c;
                if (l >= L) continue;
                uint32_t got = 0;
                if constexpr (IDF == EVICT_ID_MASK) {
                    const uint64_t *m = reinterpret_cast<const uint64_t *>(rt.ids) +
                                        (((size_t)b * N + v) * L + l) * EW;
#pragma unroll
                    for (int h = 0; h < 4; h++) {
                        if (h >= EW) break;
                        uint64_t x = __ldg(m + h);
                        if (64 * h + 64 > E) {   // bits at or above E are not experts
                            const int r = E - 64 * h;   // 1..64
                            const uint64_t valid = r >= 64 ? ~0ull : ((1ull << r) - 1ull);
                            if (x & ~valid) bad = 1;
                            x &= valid;
                        }
                        const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
                        got += __popc(lo & ~w[c][2 * h]) + __popc(hi & ~w[c][2 * h + 1]);
                        w[c][2 * h] |= lo;
                        w[c][2 * h + 1] |= hi;
                    }
                } else if constexpr (IDF == EVICT_ID_U8) {
                    const uint8_t *p = reinterpret_cast<const uint8_t *>(rt.ids) + (((size_t)b * N + v) * L + l) * K;
                    if (K == 8) {
                        const uint2 x = __ldg(reinterpret_cast<const uint2 *>(p));
#pragma unroll
                        for (int q = 0; q < 8; q++) {
                            const uint32_t e = __byte_perm(q < 4 ? x.x : x.y, 0, 0x4440 | (q & 3));
                            if (e >= (uint32_t)E) { bad = 1; continue; }
                            got += set4(w[c], e);
                        }
                    } else {
                        for (int q = 0; q < K; q++) {
                            const uint32_t e = __ldg(p + q);
                            if (e >= (uint32_t)E) { bad = 1; continue; }
                            got += set4(w[c], e);
                        }
                    }
                } else {
                    const int32_t *p = reinterpret_cast<const int32_t *>(rt.ids) + (((size_t)b * N + v) * L + l) * K;
                    for (int q = 0; q < K; q++) {
                        const uint32_t e = (uint32_t)__ldg(p + q);
                        if (e >= (uint32_t)E) { bad = 1; continue; }
                        got += set4(w[c], e);
                    }
                }
                per[c] += (int)got;
                nw += got;
                if (lrow) lrow[(size_t)j * L + l] = per[c];
            }
            if (__any_sync(0xffffffffu, bad)) { st |= EVICT_TREE_BAD_EXPERT; break; }
            tot += (int)__reduce_add_sync(0xffffffffu, nw);
            if (lane == 0) crow[j] = tot;
            kdone = j + 1;
        }
    }
finish:
    // pads (and, on error, every row) are 0
    const int from = st ? 0 : kdone;
    for (int j = from + lane; j < N; j += 32) crow[j] = 0;
    if (lrow)
        for (size_t i = (size_t)from * L + lane; i < (size_t)N * L; i += 32) lrow[i] = 0;
    if (status && lane == 0) status[b] = st;
}

// Column sums of the curves over trees with n_b ≥ k and status 0: warp per
// tree row (coalesced), lane k (+32i), int64 register accumulators.
__global__ void __launch_bounds__(256) k_profile_sum(int B, int N, const int32_t *n_nodes,
                                                     const int32_t *curve, const uint32_t *status,
                                                     unsigned long long *sums, unsigned long long *cnts)
{
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    unsigned long long s[4] = {0ull, 0ull, 0ull, 0ull}, c[4] = {0ull, 0ull, 0ull, 0ull};
    for (int b = gw; b < B; b += nw) {
        if (status && status[b]) continue;
        const int n = n_nodes ? n_nodes[b] : N;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int k = lane + 32 * i;
            if (k < n && k < N) {
                s[i] += (unsigned long long)curve[(size_t)b * N + k];
                c[i] += 1ull;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int k = lane + 32 * i;
        if (k < N && c[i]) {
            atomicAdd(sums + k, s[i]);
            atomicAdd(cnts + k, c[i]);
        }
    }
}

__global__ void k_profile_cost(int N, int L, const unsigned long long *sums, const unsigned long long *cnts,
                               double c0, double cu, double ct, float *cost)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= N) return;
    const unsigned long long cnt = cnts[k];
    cost[k] = cnt ? (float)(c0 + cu * ((double)sums[k] / ((double)L * (double)cnt)) + ct * (double)(k + 1))
                  : __int_as_float(0x7f800000);
}

}  // namespace curve
}  // namespace evict

using namespace evict::curve;

extern "C" evict_status_t evict_union_curve(const evict_trees_t *trees, const int32_t *order,
                                            const evict_routing_t *rt, int32_t *curve, int32_t *curve_layer,
                                            uint32_t *status, void *stream)
{
    if (!trees || trees->batch < 1 || trees->max_nodes < 1 || trees->max_nodes > EVICT_MAX_NODES)
        return EVICT_ERR_INVALID_ARG;
    if (!order || !curve || !rt || !rt->ids) return EVICT_ERR_INVALID_ARG;
    if (rt->num_layers < 1 || rt->num_layers > EVICT_MAX_LAYERS || rt->num_experts < 1) return EVICT_ERR_INVALID_ARG;
    if (rt->id_format == EVICT_ID_MASK) {
        if (rt->num_experts > EVICT_MAX_EXPERTS) return EVICT_ERR_INVALID_ARG;
    } else if (rt->id_format == EVICT_ID_U8 || rt->id_format == EVICT_ID_I32) {
        if (rt->top_k < 1 || rt->top_k > EVICT_MAX_TOPK || rt->top_k > rt->num_experts) return EVICT_ERR_INVALID_ARG;
        if (rt->num_experts > EVICT_MAX_EXPERTS) return EVICT_ERR_INVALID_ARG;
    } else {
        return EVICT_ERR_INVALID_ARG;
    }
    if ((uintptr_t)rt->ids & 15) return EVICT_ERR_INVALID_ARG;
    if (!evict::dev_supported()) return EVICT_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = (trees->batch + kWarpsC - 1) / kWarpsC;
    const int R = (rt->num_layers + 31) / 32;
#define EVICT_CURVE(IDFV, NWV)                                                                         \
    switch (R) {                                                                                      \
    case 1: k_union_curve<IDFV, 1, NWV><<<blocks, kWarpsC * 32, 0, s>>>(*trees, order, *rt, curve, curve_layer, status); break; \
    case 2: k_union_curve<IDFV, 2, NWV><<<blocks, kWarpsC * 32, 0, s>>>(*trees, order, *rt, curve, curve_layer, status); break; \
    case 3: k_union_curve<IDFV, 3, NWV><<<blocks, kWarpsC * 32, 0, s>>>(*trees, order, *rt, curve, curve_layer, status); break; \
    default: k_union_curve<IDFV, 4, NWV><<<blocks, kWarpsC * 32, 0, s>>>(*trees, order, *rt, curve, curve_layer, status); break; \
    }
    const bool wide = rt->num_experts > 128;   // 8-word register sets (Ling-flash-2.0: 256 experts)
    if (rt->id_format == EVICT_ID_U8) { if (wide) { EVICT_CURVE(EVICT_ID_U8, 8) } else { EVICT_CURVE(EVICT_ID_U8, 4) } }
    else if (rt->id_format == EVICT_ID_I32) { if (wide) { EVICT_CURVE(EVICT_ID_I32, 8) } else { EVICT_CURVE(EVICT_ID_I32, 4) } }
    else { EVICT_CURVE(EVICT_ID_MASK, 8) }
#undef EVICT_CURVE
    return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA;
}

extern "C" size_t evict_profile_workspace_bytes(int32_t max_nodes)
{
    return max_nodes < 1 ? 0 : (size_t)16 * max_nodes;
}

extern "C" evict_status_t evict_profile_cost(int32_t batch, int32_t max_nodes, int32_t num_layers,
                                             const int32_t *n_nodes, const int32_t *curve,
                                             const uint32_t *status, float c0, float c_union, float c_tok,
                                             float *cost, void *workspace, size_t workspace_bytes, void *stream)
{
    if (batch < 1 || max_nodes < 1 || max_nodes > EVICT_MAX_NODES || num_layers < 1) return EVICT_ERR_INVALID_ARG;
    if (!curve || !cost || !workspace || workspace_bytes < evict_profile_workspace_bytes(max_nodes) ||
        ((uintptr_t)workspace & 7))
        return EVICT_ERR_INVALID_ARG;
    if (!isfinite(c0) || !isfinite(c_union) || !isfinite(c_tok)) return EVICT_ERR_INVALID_ARG;
    // every entry must be a valid evict_select cost: C(k) ≥ c0 > 0 and finite in fp32
    // (Ū(k) ≤ E ≤ EVICT_MAX_EXPERTS, k ≤ N)
    if (!(c0 > 0.f) || c_union < 0.f || c_tok < 0.f) return EVICT_ERR_INVALID_ARG;
    if ((double)c0 + (double)c_union * EVICT_MAX_EXPERTS + (double)c_tok * max_nodes > 3.0e38)
        return EVICT_ERR_INVALID_ARG;
    const int sms = evict::dev_sms();
    if (sms <= 0 || !evict::dev_supported()) return EVICT_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long *sums = reinterpret_cast<unsigned long long *>(workspace);
    unsigned long long *cnts = sums + max_nodes;
    if (cudaMemsetAsync(workspace, 0, evict_profile_workspace_bytes(max_nodes), s) != cudaSuccess)
        return EVICT_ERR_CUDA;
    int blocks = (batch + 7) / 8;
    if (blocks > sms * 8) blocks = sms * 8;
    k_profile_sum<<<blocks, 256, 0, s>>>(batch, max_nodes, n_nodes, curve, status, sums, cnts);
    k_profile_cost<<<(max_nodes + 127) / 128, 128, 0, s>>>(max_nodes, num_layers, sums, cnts, c0, c_union, c_tok,
                                                            cost);
    return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA;
}
