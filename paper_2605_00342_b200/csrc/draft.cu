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
    if (evict::dev_sms() <= 0) return EVICT_ERR_UNSUPPORTED;
    evict::draft::k_draft<<<batch, evict::draft::kThreads, 0, (cudaStream_t)stream>>>(
        batch, steps, topk, max_nodes, child_tokens, child_probs, parent, q, tokens, n_nodes, status);
    return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA;
}
