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
//   t % topk) with Score = fl32(Score(parent)·q) (Eq. 7); the next frontier is
//   the topk best new candidates by (Score desc, creation index asc), found by
//   rank counting (≤ 256 candidates).  Budget cut: a shared-memory bitonic sort
//   of 64-bit keys (~Score bits, creation index) over the pool (≤ 2048), the
//   first N kept, renumbered by creation index with a block-wide prefix count.
#include <cuda_runtime.h>
#include <stdint.h>

#include "evict.h"
#include "evict_launch.h"

namespace evict {
namespace draft {

constexpr int kThreads = 256;
constexpr int kMaxPool = EVICT_DRAFT_MAX_POOL;   // 2048

struct Smem {
    unsigned long long key[kMaxPool];   // sort keys; later the kept flags / new ids reuse `nid`
    float score[kMaxPool];
    int32_t src[kMaxPool];              // offset of the node's (token, q) in its tree's table; -1 root
    int16_t par[kMaxPool], nid[kMaxPool];
    int16_t frontier[16];
    int32_t wsum[kThreads / 32];
    uint32_t bad;
};

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
        if (tid < nnew) {
            const int j = tid / topk, c = tid - j * topk;
            const size_t at = tbl + ((size_t)st * topk + j) * topk + c;
            const float p = __ldg(cprob + at);
            if (!(p >= 0.f && p <= 1.f)) atomicOr(&s.bad, 1u);
            const int u = s.frontier[j];
            const int idx = count + tid;
            s.score[idx] = __fmul_rn(s.score[u], p);
            s.src[idx] = (int32_t)(at - tbl);
            s.par[idx] = (int16_t)u;
        }
        __syncthreads();
        if (s.bad) break;
        if (tid < nnew) {
            const float v = s.score[count + tid];
            int rank = 0;
            for (int u = 0; u < nnew; u++) {
                const float x = s.score[count + u];
                rank += (x > v || (x == v && u < tid)) ? 1 : 0;
            }
            if (rank < topk) s.frontier[rank] = (int16_t)(count + tid);
        }
        __syncthreads();
        count += nnew;
        nf = nnew < topk ? nnew : topk;
    }
    const bool bad = s.bad != 0u;
    const int n = bad ? 0 : (count < N ? count : N);
    if (!bad) {
        // budget cut: sort (Score desc, creation index asc) — Score ∈ [0, 1] so its bits order it
        int Pp = 1;
        while (Pp < count) Pp <<= 1;
        for (int i = tid; i < Pp; i += kThreads)
            s.key[i] = i < count ? ((unsigned long long)(0x7fffffffu - (__float_as_uint(s.score[i]) & 0x7fffffffu)) << 32) | (uint32_t)i
                                 : ~0ull;
        __syncthreads();
        for (int k = 2; k <= Pp; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < Pp; i += kThreads) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const unsigned long long a = s.key[i], c = s.key[ixj];
                        const bool up = (i & k) == 0;
                        if ((a > c) == up) {
                            s.key[i] = c;
                            s.key[ixj] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int i = tid; i < count; i += kThreads) s.nid[i] = 0;
        __syncthreads();
        for (int i = tid; i < n; i += kThreads) s.nid[(int)(s.key[i] & 0xffffffffu)] = 1;   // kept flags
        __syncthreads();
        // renumber kept nodes by creation index: block-wide exclusive prefix count of the flags
        constexpr int PER = kMaxPool / kThreads;   // 8 entries per thread
        const int i0 = tid * PER;
        int loc = 0;
#pragma unroll
        for (int e = 0; e < PER; e++) loc += (i0 + e < count) ? s.nid[i0 + e] : 0;
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
            if (i < count) {
                const int f = s.nid[i];
                s.nid[i] = f ? (int16_t)run : (int16_t)-1;
                run += f;
            }
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
    if (batch < 1 || steps < 1 || topk < 1 || topk > 16 || max_nodes < 1 || max_nodes > EVICT_MAX_NODES)
        return EVICT_ERR_INVALID_ARG;
    if ((long long)1 + topk + (long long)(steps - 1) * topk * topk > EVICT_DRAFT_MAX_POOL) return EVICT_ERR_INVALID_ARG;
    if (!child_tokens || !child_probs || !parent || !q || !tokens || !n_nodes) return EVICT_ERR_INVALID_ARG;
    if (evict::dev_sms() <= 0) return EVICT_ERR_UNSUPPORTED;
    evict::draft::k_draft<<<batch, evict::draft::kThreads, 0, (cudaStream_t)stream>>>(
        batch, steps, topk, max_nodes, child_tokens, child_probs, parent, q, tokens, n_nodes, status);
    return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA;
}
