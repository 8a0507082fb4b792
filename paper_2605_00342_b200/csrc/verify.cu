// verify.cu — NEXT-3: verify-side tree sampling (
// PAPER.md:64–72, §2.1, Eq. 3), consuming the packed verify tree that
// evict_build_verify_tree emits and the target's next-token rows of the
// single verify pass.
//
// k_verify: one CTA (512 threads) per tree.
//   1. stage the tree's slot lists (next_token / next_sibling / retrieve_index)
//      and draft tokens into shared memory, derive each slot's parent slot,
//      validate the lists (strictly increasing links ⇒ the walk terminates);
//   2. sampling: gather p_{parent}(token(c)) of every kept child in one round
//      trip, then one thread walks the tree in shared memory applying Eq. 3 in
//      fp32 (accept iff u < p·2^32; on rejection p(w) ← p(w)/(1−p(c)), one
//      IEEE division per rejected sibling in visiting order — reading V3);
//      greedy: the CTA takes argmax of each row on the path (reading V5);
//   3. sampling bonus: the final node's row is read once, coalesced, as
//      exact integers X(w) = r(w)·2^149 in 192-bit fixed point (every fp32
//      value in [0,1] is an integer multiple of 2^-149, so sums are exact and
//      association-free — reading V4): per-512-token chunk sums in shared
//      memory, the rejected tokens subtracted exactly, Z = Σ, threshold
//      T = ⌊u_bonus·Z / 2^32⌋, then the crossing chunk is located by a warp scan
//      and re-read (one 2 KB chunk) to find the smallest t with CDF(t) > T.
// HBM traffic per tree: one row of V fp32 (+ the k gathers) — the kernel is
// HBM-bound at V = 151936 (608 KB per tree).
#include <cuda_runtime.h>
#include <stdint.h>

#include "evict.h"
#include "evict_launch.h"

namespace evict {
namespace verify {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 512;                              // tokens per chunk (16 per lane)
constexpr int kMaxChunks = EVICT_MAX_VOCAB / kChunk;     // 512
constexpr int kMaxRej = EVICT_MAX_NODES;

struct U3 {
    unsigned long long a, b, c;   // little-endian 192-bit unsigned
};

__device__ __forceinline__ void add3(U3 &x, const U3 &y)
{
    asm("add.cc.u64 %0, %0, %3;\n\taddc.cc.u64 %1, %1, %4;\n\taddc.u64 %2, %2, %5;"
        : "+l"(x.a), "+l"(x.b), "+l"(x.c)
        : "l"(y.a), "l"(y.b), "l"(y.c));
}

__device__ __forceinline__ void sub3(U3 &x, const U3 &y)
{
    asm("sub.cc.u64 %0, %0, %3;\n\tsubc.cc.u64 %1, %1, %4;\n\tsubc.u64 %2, %2, %5;"
        : "+l"(x.a), "+l"(x.b), "+l"(x.c)
        : "l"(y.a), "l"(y.b), "l"(y.c));
}

__device__ __forceinline__ bool gt3(const U3 &x, const U3 &y)   // x > y
{
    if (x.c != y.c) return x.c > y.c;
    if (x.b != y.b) return x.b > y.b;
    return x.a > y.a;
}

__device__ __forceinline__ bool zero3(const U3 &x) { return (x.a | x.b | x.c) == 0ull; }

// a valid probability: +0/-0 … 1.0 (NaN, negatives and > 1 are not)
__device__ __forceinline__ bool valid_bits(uint32_t u) { return u <= 0x3f800000u || u == 0x80000000u; }

// exact fixed-point value x·2^149 of a valid fp32 probability (bits, sign cleared)
__device__ __forceinline__ U3 fixed(uint32_t u)
{
    u &= 0x7fffffffu;
    const uint32_t e = u >> 23;
    const unsigned long long m = (u & 0x7fffffu) | (e ? 0x800000u : 0u);
    const uint32_t sh = e ? e - 1u : 0u;                       // ≤ 126 for x ≤ 1
    const uint32_t r = sh & 63u;
    const unsigned long long lo = m << r, hi = (m >> 1) >> (63u - r);
    U3 v;
    const bool low = sh < 64u;
    v.a = low ? lo : 0ull;
    v.b = low ? hi : lo;
    v.c = low ? 0ull : hi;
    return v;
}

__device__ __forceinline__ U3 shfl_xor3(const U3 &x, int m)
{
    return U3{__shfl_xor_sync(0xffffffffu, x.a, m), __shfl_xor_sync(0xffffffffu, x.b, m),
              __shfl_xor_sync(0xffffffffu, x.c, m)};
}

__device__ __forceinline__ U3 shfl_up3(const U3 &x, int d)
{
    return U3{__shfl_up_sync(0xffffffffu, x.a, d), __shfl_up_sync(0xffffffffu, x.b, d),
              __shfl_up_sync(0xffffffffu, x.c, d)};
}

__device__ __forceinline__ U3 shfl3(const U3 &x, int src)
{
    return U3{__shfl_sync(0xffffffffu, x.a, src), __shfl_sync(0xffffffffu, x.b, src),
              __shfl_sync(0xffffffffu, x.c, src)};
}

__device__ __forceinline__ U3 warp_sum3(U3 x)
{
#pragma unroll
    for (int m = 16; m; m >>= 1) add3(x, shfl_xor3(x, m));
    return x;
}

__device__ __forceinline__ U3 warp_incl_scan3(U3 x, int lane)
{
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const U3 y = shfl_up3(x, d);
        if (lane >= d) add3(x, y);
    }
    return x;
}

// floor(u · Z / 2^32) for a 32-bit u: Z·u < 2^200 (Z < 2^168), four 64-bit words, shift right by 32.
__device__ __forceinline__ U3 scale_floor(const U3 &z, uint32_t u)
{
    const unsigned long long U = u;
    const unsigned long long w0 = z.a * U, a_hi = __umul64hi(z.a, U);
    const unsigned long long b_lo = z.b * U, b_hi = __umul64hi(z.b, U);
    const unsigned long long c_lo = z.c * U, c_hi = __umul64hi(z.c, U);
    unsigned long long w1, w2, w3;
    asm("add.cc.u64 %0, %3, %4;\n\taddc.cc.u64 %1, %5, %6;\n\taddc.u64 %2, %7, 0;"
        : "=l"(w1), "=l"(w2), "=l"(w3)
        : "l"(a_hi), "l"(b_lo), "l"(b_hi), "l"(c_lo), "l"(c_hi));
    U3 t;
    t.a = (w0 >> 32) | (w1 << 32);
    t.b = (w1 >> 32) | (w2 << 32);
    t.c = (w2 >> 32) | (w3 << 32);
    return t;
}

struct Smem {
    int32_t nt[EVICT_MAX_NODES], ns[EVICT_MAX_NODES], tok[EVICT_MAX_NODES], ps[EVICT_MAX_NODES];
    float pc[EVICT_MAX_NODES];
    int32_t path[EVICT_MAX_NODES];
    int32_t rej[kMaxRej];
    float dv[kMaxRej];  // 1 − p(c) of the rejected siblings, in visiting order
    U3 csum[kMaxChunks];
    unsigned long long red[kWarps];
    U3 pre;             // exclusive prefix before the crossing chunk
    int32_t k, plen, node, nrej, cross, bonus;
    uint32_t st;
};

// CTA-wide argmax over one row: (value desc, index asc); flags invalid entries.
__device__ int row_argmax(const float *row, int V, Smem &s, int tid)
{
    const int lane = tid & 31, w = tid >> 5;
    unsigned long long best = 0ull;
    bool bad = false;
    const int V4 = V >> 2;
    const float4 *r4 = reinterpret_cast<const float4 *>(row);
    for (int i = tid; i < V4; i += kThreads) {
        const float4 x = __ldcs(r4 + i);
        const uint32_t u[4] = {__float_as_uint(x.x), __float_as_uint(x.y), __float_as_uint(x.z),
                               __float_as_uint(x.w)};
#pragma unroll
        for (int j = 0; j < 4; j++) {
            bad |= !valid_bits(u[j]);
            const unsigned long long key = ((unsigned long long)(u[j] & 0x7fffffffu) << 32) |
                                           (0xffffffffu - (uint32_t)(4 * i + j));
            best = key > best ? key : best;
        }
    }
    for (int i = 4 * V4 + tid; i < V; i += kThreads) {
        const uint32_t u = __float_as_uint(__ldcs(row + i));
        bad |= !valid_bits(u);
        const unsigned long long key = ((unsigned long long)(u & 0x7fffffffu) << 32) | (0xffffffffu - (uint32_t)i);
        best = key > best ? key : best;
    }
#pragma unroll
    for (int m = 16; m; m >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, m);
        best = o > best ? o : best;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&s.st, EVICT_TREE_BAD_PROB);
    if (lane == 0) s.red[w] = best;
    __syncthreads();
    unsigned long long b = 0ull;
#pragma unroll
    for (int i = 0; i < kWarps; i++) b = s.red[i] > b ? s.red[i] : b;
    __syncthreads();   // s.red is reused by the next row
    return (int)(0xffffffffu - (uint32_t)(b & 0xffffffffull));
}

__global__ void __launch_bounds__(kThreads) k_verify(evict_verify_batch_t vb, const float *probs, int V,
                                                     long long stride, int mode, const uint32_t *u_accept,
                                                     const uint32_t *u_bonus, int32_t *accept_len,
                                                     int32_t *accepted_slots, int32_t *bonus_token,
                                                     uint32_t *status)
{
    __shared__ Smem s;
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int N = vb.max_nodes;
    const int off = __ldg(vb.verify_offsets + b), k = __ldg(vb.verify_offsets + b + 1) - off;
    if (tid == 0) {
        s.st = k > N ? EVICT_TREE_BAD_SIZE : k < 1 ? EVICT_TREE_BAD_KEEP : 0u;   // k = 0: empty keep set
        s.k = k;
        s.nrej = 0;
    }
    __syncthreads();
    // 1. stage and validate the slot lists
    if (!s.st) {
        for (int q = tid; q < k; q += kThreads) {
            const int nt = __ldg(vb.next_token + off + q), ns = __ldg(vb.next_sibling + off + q);
            const int ri = __ldg(vb.retrieve_index + off + q);
            uint32_t e = 0;
            if ((nt != -1 && (nt <= q || nt >= k)) || (ns != -1 && (ns <= q || ns >= k))) e |= EVICT_TREE_BAD_KEEP;
            if (ri < b * N || ri >= (b + 1) * N) e |= EVICT_TREE_BAD_KEEP;
            int t = -1;
            if (!e) {
                t = __ldg(vb.tokens + ri);
                if (q > 0 && (t < 0 || t >= V)) e |= EVICT_TREE_BAD_TOKEN;
            }
            s.nt[q] = nt;
            s.ns[q] = ns;
            s.tok[q] = t;
            s.ps[q] = -1;
            if (e) atomicOr(&s.st, e);
        }
    }
    __syncthreads();
    if (!s.st) {
        for (int q = tid; q < k; q += kThreads)
            for (int c = s.nt[q]; c != -1; c = s.ns[c]) s.ps[c] = q;
    }
    __syncthreads();
    if (!s.st) {
        for (int q = 1 + tid; q < k; q += kThreads)
            if (s.ps[q] < 0) atomicOr(&s.st, EVICT_TREE_BAD_KEEP);   // an orphan slot
    }
    __syncthreads();
    // status precedence as the oracle: size/keep, then token, then prob
    if (tid == 0 && (s.st & (EVICT_TREE_BAD_SIZE | EVICT_TREE_BAD_KEEP))) s.st &= EVICT_TREE_BAD_SIZE | EVICT_TREE_BAD_KEEP;
    __syncthreads();

    if (mode == EVICT_VERIFY_SAMPLE) {
        // 2a. gather p_{parent}(token(c)) for every kept child c
        if (!s.st) {
            for (int c = 1 + tid; c < k; c += kThreads) {
                const float p = __ldg(probs + (long long)(off + s.ps[c]) * stride + s.tok[c]);
                if (!(p >= 0.f && p <= 1.f)) atomicOr(&s.st, EVICT_TREE_BAD_PROB);
                s.pc[c] = p;
            }
        }
        __syncthreads();
        // 2b. Eq. 3 walk (one thread, shared memory only)
        if (tid == 0 && !s.st) {
            const uint32_t *ua = u_accept + (size_t)b * N;
            int u = 0, plen = 1;
            s.path[0] = 0;
            float *d = s.dv;
            int nd;
            for (;;) {
                nd = 0;
                int nrej = 0, next = -1;
                for (int c = s.nt[u]; c != -1; c = s.ns[c]) {
                    const int t = s.tok[c];
                    bool gone = false;
                    for (int i = 0; i < nrej; i++) gone |= s.rej[i] == t;
                    float v = 0.f;
                    if (!gone) {
                        v = s.pc[c];
                        for (int i = 0; i < nd; i++) v = __fdiv_rn(v, d[i]);
                    }
                    if ((double)__ldg(ua + c) < (double)v * 4294967296.0) { next = c; break; }
                    d[nd++] = __fsub_rn(1.f, v);
                    s.rej[nrej++] = t;
                }
                if (next < 0) { s.nrej = nrej; break; }
                s.path[plen++] = next;
                u = next;
            }
            s.plen = plen;
            s.node = u;
        }
        __syncthreads();
        if (s.st) goto done;
        // 3. bonus from the residual of the final node's row
        {
            const float *row = probs + (long long)(off + s.node) * stride;
            const int nch = (V + kChunk - 1) / kChunk;
            bool bad = false;
            for (int ch = w; ch < nch; ch += kWarps) {
                U3 acc{0ull, 0ull, 0ull};
#pragma unroll
                for (int j = 0; j < kChunk / 128; j++) {
                    const int e0 = ch * kChunk + j * 128 + lane * 4;
                    if (e0 + 3 < V) {
                        const float4 x = __ldcs(reinterpret_cast<const float4 *>(row + e0));
                        const uint32_t uu[4] = {__float_as_uint(x.x), __float_as_uint(x.y), __float_as_uint(x.z),
                                                __float_as_uint(x.w)};
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            const bool ok = valid_bits(uu[q]);
                            bad |= !ok;
                            if (ok) add3(acc, fixed(uu[q]));
                        }
                    } else {
                        for (int q = 0; q < 4; q++) {
                            if (e0 + q >= V) break;
                            const uint32_t uu = __float_as_uint(__ldcs(row + e0 + q));
                            const bool ok = valid_bits(uu);
                            bad |= !ok;
                            if (ok) add3(acc, fixed(uu));
                        }
                    }
                }
                acc = warp_sum3(acc);
                if (lane == 0) s.csum[ch] = acc;
            }
            if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&s.st, EVICT_TREE_BAD_PROB);
            __syncthreads();
            if (s.st) goto done;
            // subtract each distinct rejected token once (exact)
            if (tid == 0) {
                for (int i = 0; i < s.nrej; i++) {
                    const int t = s.rej[i];
                    bool dup = false;
                    for (int j = 0; j < i; j++) dup |= s.rej[j] == t;
                    if (!dup) sub3(s.csum[t / kChunk], fixed(__float_as_uint(row[t])));
                }
            }
            __syncthreads();
            if (w == 0) {
                const int per = (nch + 31) / 32;
                const int c0 = lane * per, c1 = min(nch, c0 + per);
                U3 mine{0ull, 0ull, 0ull};
                for (int c = c0; c < c1; c++) add3(mine, s.csum[c]);
                const U3 incl = warp_incl_scan3(mine, lane);
                const U3 Z = shfl3(incl, 31);
                if (zero3(Z)) {
                    if (lane == 0) s.st |= EVICT_TREE_BAD_PROB;
                } else {
                    const U3 T = scale_floor(Z, __ldg(u_bonus + b));
                    const unsigned hit = __ballot_sync(0xffffffffu, gt3(incl, T));
                    const int L = __ffs(hit) - 1;          // exists: incl(31) = Z > T
                    if (lane == L) {
                        U3 pre = incl;
                        sub3(pre, mine);                   // exclusive prefix of this lane
                        int c = c0;
                        for (; c < c1; c++) {
                            U3 nx = pre;
                            add3(nx, s.csum[c]);
                            if (gt3(nx, T)) break;
                            pre = nx;
                        }
                        s.cross = c;
                        s.pre = pre;
                    }
                    __syncwarp();
                    // re-read the crossing chunk, lane-contiguous 16 tokens, exact in-chunk scan
                    const int cb = s.cross * kChunk + lane * 16;
                    const int nrej = s.nrej;
                    U3 ls{0ull, 0ull, 0ull};
                    for (int q = 0; q < 16; q++) {
                        const int t = cb + q;
                        if (t >= V) break;
                        bool gone = false;
                        for (int i = 0; i < nrej; i++) gone |= s.rej[i] == t;
                        if (!gone) add3(ls, fixed(__float_as_uint(row[t])));
                    }
                    U3 li = warp_incl_scan3(ls, lane);
                    add3(li, s.pre);
                    const unsigned h2 = __ballot_sync(0xffffffffu, gt3(li, T));
                    const int L2 = __ffs(h2) - 1;
                    if (lane == L2) {                      // walk the lane's 16 tokens again
                        U3 run = li;
                        sub3(run, ls);
                        int t = cb;
                        for (; t < cb + 16 && t < V; t++) {
                            bool gone = false;
                            for (int i = 0; i < nrej; i++) gone |= s.rej[i] == t;
                            if (!gone) add3(run, fixed(__float_as_uint(row[t])));
                            if (gt3(run, T)) break;
                        }
                        s.bonus = t;
                    }
                }
            }
            __syncthreads();
        }
    } else {
        // greedy (T = 0): follow argmax through the kept children
        if (!s.st) {
            int u = 0, plen = 1;
            if (tid == 0) s.path[0] = 0;
            for (;;) {
                const int g = row_argmax(probs + (long long)(off + u) * stride, V, s, tid);
                if (s.st) break;
                int next = -1;
                for (int c = s.nt[u]; c != -1; c = s.ns[c])
                    if (s.tok[c] == g) { next = c; break; }
                if (next < 0) {
                    if (tid == 0) s.bonus = g;
                    break;
                }
                if (tid == 0) s.path[plen] = next;
                plen++;
                u = next;
            }
            if (tid == 0) s.plen = plen;
        }
        __syncthreads();
    }
done:
    __syncthreads();
    const bool ok = s.st == 0;
    const int plen = ok ? s.plen : 0;
    for (int q = tid; q < N; q += kThreads) accepted_slots[(size_t)b * N + q] = q < plen ? s.path[q] : -1;
    if (tid == 0) {
        accept_len[b] = plen;
        bonus_token[b] = ok ? s.bonus : -1;
        if (status) status[b] = s.st;
    }
}

}  // namespace verify
}  // namespace evict

using namespace evict::verify;

extern "C" evict_status_t evict_verify_sample(const evict_verify_batch_t *vb, const float *probs, int32_t vocab,
                                              int64_t row_stride, int32_t mode, const uint32_t *u_accept,
                                              const uint32_t *u_bonus, int32_t *accept_len,
                                              int32_t *accepted_slots, int32_t *bonus_token, uint32_t *status,
                                              void *stream)
{
    if (!vb || vb->batch < 1 || vb->max_nodes < 1 || vb->max_nodes > EVICT_MAX_NODES) return EVICT_ERR_INVALID_ARG;
    if (!vb->verify_offsets || !vb->next_token || !vb->next_sibling || !vb->retrieve_index || !vb->tokens)
        return EVICT_ERR_INVALID_ARG;
    if (!probs || !accept_len || !accepted_slots || !bonus_token) return EVICT_ERR_INVALID_ARG;
    if (vocab < 1 || vocab > EVICT_MAX_VOCAB || row_stride < vocab || (row_stride & 3) || ((uintptr_t)probs & 15))
        return EVICT_ERR_INVALID_ARG;
    if (mode == EVICT_VERIFY_SAMPLE) {
        if (!u_accept || !u_bonus) return EVICT_ERR_INVALID_ARG;
    } else if (mode != EVICT_VERIFY_GREEDY) {
        return EVICT_ERR_INVALID_ARG;
    }
    if (evict::dev_sms() <= 0) return EVICT_ERR_UNSUPPORTED;
    k_verify<<<vb->batch, kThreads, 0, (cudaStream_t)stream>>>(*vb, probs, vocab, row_stride, mode, u_accept,
                                                               u_bonus, accept_len, accepted_slots, bonus_token,
                                                               status);
    return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA;
}
