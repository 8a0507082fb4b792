// draft.cu — NEXT-4 (P2): the EAGLE-style draft-tree builder on the GPU
// (§2.1 "repeatedly extends a fixed number
// of draft tokens … with the same number of tokens at each layer", then the
// budget cut of §3.2.1, by cumulative score).  It turns the
// drafter's per-step top-k tables into the (parent, q, token) arrays that
// evict_select consumes, on the device (no host round trip between drafting
// and selection).
//
// k_draft: one CTA (256 threads) per tree, the candidate pool in shared memory.
//   step s: thread t < |frontier|·topk creates candidate (slot t / topk, child
//   t % topk) with Score = fl32(Score(parent)·q) (Eq. 7); the step's candidates
//   are sorted by (Score desc, creation index asc) — a bitonic sort of 64-bit
//   keys (~Score bits, index), one per thread, shuffles below stride 32 — and
//   the first topk become the next frontier.  Budget cut: a node's rank in the
//   pool = its index in its step's sorted list + binary-search counts in the
//   other steps' lists; the root and ranks < N−1 are kept and renumbered by
//   creation index with a block-wide prefix count.
#include <cuda_runtime.h>
#include <stdint.h>

#include "evict.h"
#include "evict_launch.h"

namespace evict {
namespace draft {

constexpr int kThreads = 256;
constexpr int kMaxPool = EVICT_DRAFT_MAX_POOL;   // 2048

struct Smem {
    float score[kMaxPool];
    int32_t src[kMaxPool];              // offset of the node's (token, q) in its tree's table; -1 root
    int16_t par[kMaxPool], nid[kMaxPool];
    unsigned long long sk[kThreads];    // bitonic exchange buffer (strides ≥ 32)
    unsigned long long lst[16][EVICT_MAX_NODES];   // each step's sorted keys (first N−1)
    int32_t len[16];
    int16_t frontier[16];
    int32_t wsum[kThreads / 32];
    uint32_t bad;
};

__device__ __forceinline__ unsigned long long node_key(float score, int idx)
{
    // (Score desc, creation index asc) as one ascending 64-bit key; Score ∈ [0, 1], −0 → +0
    return ((unsigned long long)(0x7fffffffu - (__float_as_uint(score) & 0x7fffffffu)) << 32) | (uint32_t)idx;
}

// number of keys < x in the ascending list l[0..n)
__device__ __forceinline__ int lower_bound(const unsigned long long *l, int n, unsigned long long x)
{
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (l[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(kThreads) k_draft(int B, int steps, int topk, int N, const int32_t *ctok,
                                                    const float *cprob, int32_t *parent, float *q,
                                                    int32_t *tokens, int32_t *n_nodes, uint32_t *status)
{
    __shared__ Smem s;
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const size_t tbl = (size_t)b * steps * topk * topk;
    if (tid == 0) {
        s.score[0] = 1.f;
        s.src[0] = -1;
        s.par[0] = -1;
        s.frontier[0] = 0;
        s.bad = 0u;
    }
    __syncthreads();
    int count = 1, nf = 1;
    for (int st = 0; st < steps; st++) {
        const int nnew = nf * topk;
        unsigned long long key = ~0ull;
        if (tid < nnew) {
            const int j = tid / topk, c = tid - j * topk;
            const size_t at = tbl + ((size_t)st * topk + j) * topk + c;
            const float p = __ldg(cprob + at);
            if (!(p >= 0.f && p <= 1.f)) atomicOr(&s.bad, 1u);
            const int u = s.frontier[j];
            const int idx = count + tid;
            const float sc = __fmul_rn(s.score[u], p);
            s.score[idx] = sc;
            s.src[idx] = (int32_t)(at - tbl);
            s.par[idx] = (int16_t)u;
            key = node_key(sc, idx);
        }
        // sort the step's candidates (one key per thread; bitonic over the next power of two):
        // the first topk are the next frontier, the first N−1 the step's share of the cut
        int Kp = 1;
        while (Kp < nnew) Kp <<= 1;
        const bool sorter = w * 32 < Kp;           // warps past Kp only join the barriers
        for (int k = 2; k <= Kp; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                unsigned long long other = key;
                if (j >= 32) {
                    if (sorter) s.sk[tid] = key;
                    __syncthreads();
                    if (sorter) other = s.sk[tid ^ j];
                    __syncthreads();
                } else if (sorter) {
                    other = __shfl_xor_sync(0xffffffffu, key, j);
                }
                if (sorter) {
                    const bool up = (tid & k) == 0, lower = (tid & j) == 0;
                    key = (lower == up) ? (key < other ? key : other) : (key > other ? key : other);
                }
            }
        }
        const int keepn = nnew < N - 1 ? nnew : N - 1;
        if (tid < topk) s.frontier[tid] = (int16_t)(key & 0xffffffffu);
        if (tid < keepn) s.lst[st][tid] = key;
        if (tid == 0) s.len[st] = keepn > 0 ? keepn : 0;
        __syncthreads();
        if (s.bad) break;
        count += nnew;
        nf = nnew < topk ? nnew : topk;
    }
    const bool bad = s.bad != 0u;
    const int n = bad ? 0 : (count < N ? count : N);
    if (!bad) {
        // Budget cut: within a step the kept nodes are a prefix of its sorted list, so a node's
        // rank among all non-root pool nodes is its list index plus, for every other step, the
        // number of that step's keys below it (binary search; lists are cut at N−1, which only
        // ever understates ranks that are ≥ N−1 anyway).  Keep the root and ranks < N−1.
        for (int i = tid; i < count; i += kThreads) s.nid[i] = i == 0 ? 1 : -1;
        __syncthreads();
        const int R = N - 1;
        for (int e = tid; e < steps * R; e += kThreads) {
            const int st = e / R, i = e - st * R;
            if (i >= s.len[st]) continue;
            const unsigned long long x = s.lst[st][i];
            int rank = i;
            for (int o = 0; o < steps && rank < R; o++)
                if (o != st) rank += lower_bound(s.lst[o], s.len[o], x);
            if (rank < R) s.nid[(int)(x & 0xffffffffu)] = 1;
        }
        __syncthreads();
        // renumber kept nodes by creation index: block-wide exclusive prefix count of the flags
        constexpr int PER = kMaxPool / kThreads;   // 8 pool entries per thread
        const int i0 = tid * PER;
        int loc = 0;
#pragma unroll
        for (int e = 0; e < PER; e++) loc += (i0 + e < count && s.nid[i0 + e] == 1) ? 1 : 0;
        int incl = loc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        if (lane == 31) s.wsum[w] = incl;
        __syncthreads();
        int run = incl - loc;
        for (int i = 0; i < w; i++) run += s.wsum[i];
#pragma unroll
        for (int e = 0; e < PER; e++) {
            const int i = i0 + e;
            if (i < count && s.nid[i] == 1) s.nid[i] = (int16_t)(run++);
        }
        __syncthreads();
        for (int i = tid; i < count; i += kThreads) {
            const int k = s.nid[i];
            if (k < 0) continue;
            const size_t o = (size_t)b * N + k;
            const int sr = s.src[i];
            parent[o] = s.par[i] < 0 ? -1 : (int32_t)s.nid[s.par[i]];
            q[o] = sr < 0 ? 1.f : __ldg(cprob + tbl + sr);
            tokens[o] = sr < 0 ? -1 : __ldg(ctok + tbl + sr);
        }
    }
    for (int k = n + tid; k < N; k += kThreads) {
        const size_t o = (size_t)b * N + k;
        parent[o] = -1;
        q[o] = 0.f;
        tokens[o] = -1;
    }
    if (tid == 0) {
        n_nodes[b] = n;
        if (status) status[b] = bad ? EVICT_TREE_BAD_PROB : 0u;
    }
}

// ---------------------------------------------------------------------------
// k_draft_warp: one WARP per tree (4 trees per 128-thread CTA), for pools ≤ 1024 — the
// serving shapes.  Same algorithm, no block barriers: each step's candidates are sorted by a
// register bitonic sort (KPL keys per lane in a blocked layout: strides < KPL inside a lane,
// larger ones by shuffles), the pool / lists live in the warp's dynamic shared-memory slice.
constexpr int kWarpTrees = 4;
constexpr int kWarpPool = 1024;

struct WarpLayout {   // byte offsets inside one warp's slice
    int score, src, par, nid, lst, frontier, len, bytes;
};

__host__ __device__ inline WarpLayout warp_layout(int P, int steps, int lmax)
{
    WarpLayout w;
    w.lst = 0;                                        // u64 [steps][lmax]
    w.score = w.lst + 8 * steps * lmax;               // f32 [P]
    w.src = w.score + 4 * P;                          // i32 [P]
    w.par = w.src + 4 * P;                            // i16 [P]
    w.nid = w.par + 2 * P;                            // i16 [P]
    w.frontier = w.nid + 2 * P;                       // i16 [16]
    w.len = w.frontier + 32;                          // i32 [16]
    w.bytes = (w.len + 64 + 15) & ~15;
    return w;
}

// sort the ≤ 32·KPL keys of one step (blocked: element i = lane·KPL + r), ascending
template <int KPL>
__device__ __forceinline__ void warp_bitonic(unsigned long long (&v)[8], int lane)
{
#pragma unroll
    for (int k = 2; k <= 32 * KPL; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < KPL) {
#pragma unroll
                for (int r = 0; r < KPL; r++) {
                    if (r & j) continue;
                    const int i = lane * KPL + r;
                    const bool up = (i & k) == 0;
                    const unsigned long long x = v[r], y = v[r | j];
                    const bool sw = (x > y) == up;
                    v[r] = sw ? y : x;
                    v[r | j] = sw ? x : y;
                }
            } else {
#pragma unroll
                for (int r = 0; r < KPL; r++) {
                    const unsigned long long o = __shfl_xor_sync(0xffffffffu, v[r], j / KPL);
                    const int i = lane * KPL + r;
                    const bool up = (i & k) == 0, lower = (i & j) == 0;
                    v[r] = (lower == up) ? (v[r] < o ? v[r] : o) : (v[r] > o ? v[r] : o);
                }
            }
        }
    }
}

template <int KPL>
__device__ __forceinline__ void warp_step(int st, int nnew, int topk, int count, int keepn, const float *cprob,
                                          size_t tbl, float *score, int32_t *src, int16_t *par,
                                          int16_t *frontier, unsigned long long *lst_s, uint32_t &bad, int lane)
{
    unsigned long long v[8];
    int16_t fr[8];
#pragma unroll
    for (int r = 0; r < KPL; r++) fr[r] = frontier[(lane * KPL + r) / topk < 16 ? (lane * KPL + r) / topk : 0];
    __syncwarp();   // every lane has read the previous frontier before it is overwritten
#pragma unroll
    for (int r = 0; r < 8; r++) v[r] = ~0ull;
#pragma unroll
    for (int r = 0; r < KPL; r++) {
        const int i = lane * KPL + r;
        if (i < nnew) {
            const int j = i / topk, c = i - j * topk;
            const size_t at = tbl + ((size_t)st * topk + j) * topk + c;
            const float p = __ldg(cprob + at);
            if (!(p >= 0.f && p <= 1.f)) bad = 1u;
            const int u = fr[r];
            const int idx = count + i;
            const float sc = __fmul_rn(score[u], p);
            score[idx] = sc;
            src[idx] = (int32_t)(at - tbl);
            par[idx] = (int16_t)u;
            v[r] = node_key(sc, idx);
        }
    }
    warp_bitonic<KPL>(v, lane);
#pragma unroll
    for (int r = 0; r < KPL; r++) {
        const int i = lane * KPL + r;
        if (i < topk) frontier[i] = (int16_t)(v[r] & 0xffffffffu);
        if (i < keepn) lst_s[i] = v[r];
    }
    __syncwarp();
}

__global__ void __launch_bounds__(kWarpTrees * 32) k_draft_warp(int B, int steps, int topk, int N, int lmax,
                                                                 int wbytes, const int32_t *ctok,
                                                                 const float *cprob, int32_t *parent, float *q,
                                                                 int32_t *tokens, int32_t *n_nodes,
                                                                 uint32_t *status)
{
    extern __shared__ __align__(16) uint8_t dsm[];
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int b = blockIdx.x * kWarpTrees + wi;
    if (b >= B) return;
    const int P = 1 + topk + (steps - 1) * topk * topk;
    const WarpLayout L = warp_layout(P, steps, lmax);
    uint8_t *base = dsm + (size_t)wi * wbytes;
    unsigned long long *lst = reinterpret_cast<unsigned long long *>(base + L.lst);
    float *score = reinterpret_cast<float *>(base + L.score);
    int32_t *src = reinterpret_cast<int32_t *>(base + L.src);
    int16_t *par = reinterpret_cast<int16_t *>(base + L.par);
    int16_t *nid = reinterpret_cast<int16_t *>(base + L.nid);
    int16_t *frontier = reinterpret_cast<int16_t *>(base + L.frontier);
    int32_t *len = reinterpret_cast<int32_t *>(base + L.len);
    const size_t tbl = (size_t)b * steps * topk * topk;
    if (lane == 0) {
        score[0] = 1.f;
        src[0] = -1;
        par[0] = -1;
        frontier[0] = 0;
    }
    __syncwarp();
    uint32_t bad = 0u;
    int count = 1, nf = 1;
    for (int st = 0; st < steps; st++) {
        const int nnew = nf * topk;
        const int keepn = nnew < N - 1 ? nnew : N - 1;
        unsigned long long *lst_s = lst + (size_t)st * lmax;
        if (nnew <= 32) warp_step<1>(st, nnew, topk, count, keepn, cprob, tbl, score, src, par, frontier, lst_s, bad, lane);
        else if (nnew <= 64) warp_step<2>(st, nnew, topk, count, keepn, cprob, tbl, score, src, par, frontier, lst_s, bad, lane);
        else if (nnew <= 128) warp_step<4>(st, nnew, topk, count, keepn, cprob, tbl, score, src, par, frontier, lst_s, bad, lane);
        else warp_step<8>(st, nnew, topk, count, keepn, cprob, tbl, score, src, par, frontier, lst_s, bad, lane);
        if (lane == 0) len[st] = keepn > 0 ? keepn : 0;
        if (__any_sync(0xffffffffu, bad)) { bad = 1u; break; }
        count += nnew;
        nf = nnew < topk ? nnew : topk;
    }
    __syncwarp();
    const int n = bad ? 0 : (count < N ? count : N);
    if (!bad) {
        for (int i = lane; i < count; i += 32) nid[i] = i == 0 ? 1 : -1;
        __syncwarp();
        const int R = N - 1;
        for (int e = lane; e < steps * R; e += 32) {
            const int st = e / R, i = e - st * R;
            if (i >= len[st]) continue;
            const unsigned long long x = lst[(size_t)st * lmax + i];
            int rank = i;
            for (int o = 0; o < steps && rank < R; o++)
                if (o != st) rank += lower_bound(lst + (size_t)o * lmax, len[o], x);
            if (rank < R) nid[(int)(x & 0xffffffffu)] = 1;
        }
        __syncwarp();
        // renumber by creation index: each lane owns a contiguous run of the pool
        const int per = (count + 31) >> 5;
        const int i0 = lane * per, i1 = min(count, i0 + per);
        int loc = 0;
        for (int i = i0; i < i1; i++) loc += nid[i] == 1 ? 1 : 0;
        int incl = loc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        int run = incl - loc;
        for (int i = i0; i < i1; i++)
            if (nid[i] == 1) nid[i] = (int16_t)(run++);
        __syncwarp();
        for (int i = lane; i < count; i += 32) {
            const int k = nid[i];
            if (k < 0) continue;
            const size_t o = (size_t)b * N + k;
            const int sr = src[i];
            parent[o] = par[i] < 0 ? -1 : (int32_t)nid[par[i]];
            q[o] = sr < 0 ? 1.f : __ldg(cprob + tbl + sr);
            tokens[o] = sr < 0 ? -1 : __ldg(ctok + tbl + sr);
        }
    }
    for (int k = n + lane; k < N; k += 32) {
        const size_t o = (size_t)b * N + k;
        parent[o] = -1;
        q[o] = 0.f;
        tokens[o] = -1;
    }
    if (lane == 0) {
        n_nodes[b] = n;
        if (status) status[b] = bad ? EVICT_TREE_BAD_PROB : 0u;
    }
}

}  // namespace draft
}  // namespace evict

extern "C" evict_status_t evict_build_draft_tree(int32_t batch, int32_t steps, int32_t topk, int32_t max_nodes,
                                                 const int32_t *child_tokens, const float *child_probs,
                                                 int32_t *parent, float *q, int32_t *tokens, int32_t *n_nodes,
                                                 uint32_t *status, void *stream)
{
    if (batch < 1 || steps < 1 || steps > 16 || topk < 1 || topk > 16 || max_nodes < 1 || max_nodes > EVICT_MAX_NODES)
        return EVICT_ERR_INVALID_ARG;
    if ((long long)1 + topk + (long long)(steps - 1) * topk * topk > EVICT_DRAFT_MAX_POOL) return EVICT_ERR_INVALID_ARG;
    if (!child_tokens || !child_probs || !parent || !q || !tokens || !n_nodes) return EVICT_ERR_INVALID_ARG;
    if (!evict::dev_supported()) return EVICT_ERR_UNSUPPORTED;
    using namespace evict::draft;
    const int P = 1 + topk + (steps - 1) * topk * topk;
    const int lmax = (topk * topk < max_nodes - 1 ? topk * topk : max_nodes - 1) > 0
                         ? (topk * topk < max_nodes - 1 ? topk * topk : max_nodes - 1) : 1;
    const int wbytes = warp_layout(P, steps, lmax).bytes;
    const size_t dyn = (size_t)kWarpTrees * wbytes;
    if (P <= kWarpPool && dyn <= 96 * 1024 && batch >= 4 * evict::dev_sms()) {
        // warp per tree for throughput batches (no block barriers, 3× fewer instructions per
        // tree); small batches keep a whole CTA per tree, which finishes each tree sooner
        cudaFuncSetAttribute(k_draft_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        k_draft_warp<<<(batch + kWarpTrees - 1) / kWarpTrees, kWarpTrees * 32, dyn, (cudaStream_t)stream>>>(
            batch, steps, topk, max_nodes, lmax, wbytes, child_tokens, child_probs, parent, q, tokens, n_nodes,
            status);
    } else {
        k_draft<<<batch, kThreads, 0, (cudaStream_t)stream>>>(batch, steps, topk, max_nodes, child_tokens,
                                                               child_probs, parent, q, tokens, n_nodes, status);
    }
    return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA;
}
