// verify.cu — NEXT-3: verify-side tree sampling (
// PAPER.md:64–72, §2.1, Eq. 3), consuming the packed verify tree that
// evict_build_verify_tree emits and the target's next-token rows of the
// single verify pass.
//
// k_verify: a thread-block cluster of CL CTAs (256 threads each) per tree; CL > 1 only for
// batches too small to fill the GPU (latency).
//   1. stage the tree's slot lists (next_token / next_sibling / retrieve_index)
//      and draft tokens into shared memory, derive each slot's parent slot,
//      validate the lists (strictly increasing links ⇒ the walk terminates);
//   2. sampling: gather p_{parent}(token(c)) of every kept child in one round
//      trip, then one thread walks the tree in shared memory applying Eq. 3 in
//      fp32 (accept iff u < p·2^32; on rejection p(w) ← p(w)/(1−p(c)), one
//      IEEE division per rejected sibling in visiting order — reading V3);
//      greedy: the CTA takes argmax of each row on the path (reading V5);
//   3. sampling bonus: the final node's row is read once, coalesced, into
//      fp64 chunk sums; the token they locate is certified exact when its CDF
//      clears the threshold by more than the fp64 error bound (bonus_fast);
//      otherwise (a near-boundary draw, ~1e-10 of trees) the row is re-read as
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

constexpr int kThreads = 256;
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

// ---- distributed shared memory (thread-block cluster) helpers
__device__ __forceinline__ uint32_t cl_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cl_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t cl_map(const void *p, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(r)
                 : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
    return r;
}

__device__ __forceinline__ void cl_st_f64(uint32_t a, double v)
{
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

__device__ __forceinline__ void cl_st_u64(uint32_t a, unsigned long long v)
{
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

__device__ __forceinline__ void cl_or_u32(uint32_t a, uint32_t v)
{
    asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

struct Smem {
    int32_t nt[EVICT_MAX_NODES], ns[EVICT_MAX_NODES], tok[EVICT_MAX_NODES], ps[EVICT_MAX_NODES];
    float pc[EVICT_MAX_NODES];
    int32_t path[EVICT_MAX_NODES];
    int32_t rej[kMaxRej];
    float dv[kMaxRej];  // 1 − p(c) of the rejected siblings, in visiting order
    U3 csum[kMaxChunks];
    double dsum[kMaxChunks];
    double rsum;
    int32_t cert;
    unsigned long long red[kWarps];
    unsigned long long ckey[2][8];   // greedy: per-CTA partial argmax keys, row-parity double buffer
    uint32_t cbad[2][8];
    U3 pre;             // exclusive prefix before the crossing chunk
    int32_t k, plen, node, nrej, cross, bonus;
    uint32_t st;
    uint32_t rbad;      // bonus row: invalid entries found by any CTA of the cluster (CTA 0's copy),
                        // merged into st by CTA 0 after the cluster barrier (peers never write st)
};

// Cluster-wide argmax over one row: (value desc, index asc); CTA r of CL scans float4 slots
// i ≡ r (mod CL)·kThreads…; every CTA receives all CL partials (DSMEM stores + cluster barrier)
// and reduces them identically.  Flags invalid entries (uniformly across the cluster).
template <int CL>
__device__ int row_argmax(const float *row, int V, Smem &s, int tid, int par)
{
    const int lane = tid & 31, w = tid >> 5;
    const uint32_t r = CL > 1 ? cl_rank() : 0u;
    unsigned long long best = 0ull;
    bool bad = false;
    const int V4 = V >> 2;
    const float4 *r4 = reinterpret_cast<const float4 *>(row);
    // float4 loads per thread in flight per iteration: 8 for a whole-CTA row (throughput batches),
    // 4 when a cluster shares the row (small batches, where the deeper unroll cost latency)
    constexpr int kStep = CL * kThreads;
    constexpr int DEPTH = CL == 1 ? 8 : 4;
    for (int i0 = tid + (int)r * kThreads; i0 < V4; i0 += DEPTH * kStep) {
        float4 x[DEPTH];
#pragma unroll
        for (int h = 0; h < DEPTH; h++)
            x[h] = i0 + h * kStep < V4 ? __ldcs(r4 + i0 + h * kStep) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int h = 0; h < DEPTH; h++) {
            const int i = i0 + h * kStep;
            const uint32_t u[4] = {__float_as_uint(x[h].x), __float_as_uint(x[h].y), __float_as_uint(x[h].z),
                                   __float_as_uint(x[h].w)};
#pragma unroll
            for (int j = 0; j < 4; j++) {
                bad |= !valid_bits(u[j]);
                const unsigned long long key = ((unsigned long long)(u[j] & 0x7fffffffu) << 32) |
                                               (0xffffffffu - (uint32_t)(4 * i + j));
                best = (i < V4 && key > best) ? key : best;
            }
        }
    }
    if (r == 0) {
        for (int i = 4 * V4 + tid; i < V; i += kThreads) {
            const uint32_t u = __float_as_uint(__ldcs(row + i));
            bad |= !valid_bits(u);
            const unsigned long long key = ((unsigned long long)(u & 0x7fffffffu) << 32) | (0xffffffffu - (uint32_t)i);
            best = key > best ? key : best;
        }
    }
#pragma unroll
    for (int m = 16; m; m >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, m);
        best = o > best ? o : best;
    }
    const bool wbad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        s.red[w] = best;
        if (wbad) atomicOr(&s.cbad[par][r], 1u);
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long bb = 0ull;
#pragma unroll
        for (int i = 0; i < kWarps; i++) bb = s.red[i] > bb ? s.red[i] : bb;
        if constexpr (CL == 1) {
            s.ckey[par][0] = bb;
        } else {
            const uint32_t fb = s.cbad[par][r];
            for (int c = 0; c < CL; c++) {
                cl_st_u64(cl_map(&s.ckey[par][r], c), bb);
                if (fb) cl_or_u32(cl_map(&s.cbad[par][r], c), 1u);
            }
        }
    }
    if constexpr (CL > 1) cl_sync(); else __syncthreads();
    unsigned long long bb = 0ull;
    uint32_t anybad = 0;
#pragma unroll
    for (int c = 0; c < CL; c++) {
        bb = s.ckey[par][c] > bb ? s.ckey[par][c] : bb;
        anybad |= s.cbad[par][c];
    }
    __syncthreads();   // every thread has read this parity before anyone clears it
    if (tid < CL) s.cbad[par][tid] = 0u;   // cleared for the row after next (remote writers wait a barrier)
    if (anybad && tid == 0) atomicOr(&s.st, EVICT_TREE_BAD_PROB);
    __syncthreads();
    return anybad ? -1 : (int)(0xffffffffu - (uint32_t)(bb & 0xffffffffull));
}

// Exact bonus (reading V4): 192-bit fixed-point chunk sums, rejected tokens subtracted,
// T = ⌊u·Z/2^32⌋, crossing chunk by a warp scan, then the crossing token.  Called by the
// whole CTA; sets s.bonus or BAD_PROB (invalid entry or empty residual).
__device__ void bonus_exact(const float *row, int V, uint32_t ub, Smem &s, int tid)
{
    const int lane = tid & 31, w = tid >> 5;
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
    if (s.st) return;
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
            const U3 T = scale_floor(Z, ub);
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

// One 512-token chunk, lane-interleaved float4s (coalesced); tokens ≥ V read as +0.
__device__ __forceinline__ void load_chunk(const float *row, int V, int ch, int lane, uint32_t (&u)[16])
{
    const int base = ch * kChunk + lane * 4;
    if ((ch + 1) * kChunk <= V) {
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const float4 x = __ldcs(reinterpret_cast<const float4 *>(row + base + j * 128));
            u[4 * j] = __float_as_uint(x.x);
            u[4 * j + 1] = __float_as_uint(x.y);
            u[4 * j + 2] = __float_as_uint(x.z);
            u[4 * j + 3] = __float_as_uint(x.w);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int e = base + j * 128 + q;
                u[4 * j + q] = e < V ? __float_as_uint(__ldcs(row + e)) : 0u;
            }
    }
}

// Certified fast bonus: fp64 chunk sums (each fp32 value converts exactly; every partial
// sum of the ≤ V + 2048 + 2·nrej fp64 additions/subtractions is within
// E = (V + 2048 + 2·nrej)·2^-52·Z_full of its exact value).  The token found with the fp64
// sums is the exact answer when its CDF clears τ by more than M = 3E on both sides (and
// Z > M); otherwise s.cert = 0 and the caller runs bonus_exact.  Same validity checks.
template <int CL>
__device__ void bonus_fast(const float *row, int V, uint32_t ub, Smem &s, int tid)
{
    const int lane = tid & 31, w = tid >> 5;
    const int nch = (V + kChunk - 1) / kChunk;
    const uint32_t r = CL > 1 ? cl_rank() : 0u;
    constexpr int kStride = CL * kWarps;            // warps of the whole cluster
    bool bad = false;
    // two chunks per warp iteration: 8 × 16 B loads per lane in flight before any arithmetic;
    // CTA r of the cluster takes chunks of its global warp index, sums land in CTA 0 (DSMEM)
    for (int ch = (int)r * kWarps + w; ch < nch; ch += 2 * kStride) {
        const int ch2 = ch + kStride;
        uint32_t u0[16], u1[16];
        load_chunk(row, V, ch, lane, u0);
        if (ch2 < nch) load_chunk(row, V, ch2, lane, u1);
        else {
#pragma unroll
            for (int q = 0; q < 16; q++) u1[q] = 0u;
        }
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
        for (int q = 0; q < 16; q += 2) {
            const bool o0 = valid_bits(u0[q]), o1 = valid_bits(u0[q + 1]);
            const bool p0 = valid_bits(u1[q]), p1 = valid_bits(u1[q + 1]);
            bad |= !(o0 && o1 && p0 && p1);
            a0 += o0 ? (double)__uint_as_float(u0[q] & 0x7fffffffu) : 0.0;
            a1 += o1 ? (double)__uint_as_float(u0[q + 1] & 0x7fffffffu) : 0.0;
            b0 += p0 ? (double)__uint_as_float(u1[q] & 0x7fffffffu) : 0.0;
            b1 += p1 ? (double)__uint_as_float(u1[q + 1] & 0x7fffffffu) : 0.0;
        }
        double accA = a0 + a1, accB = b0 + b1;
#pragma unroll
        for (int m = 16; m; m >>= 1) {
            accA += __shfl_xor_sync(0xffffffffu, accA, m);
            accB += __shfl_xor_sync(0xffffffffu, accB, m);
        }
        if (lane == 0) {
            if constexpr (CL == 1) {
                s.dsum[ch] = accA;
                if (ch2 < nch) s.dsum[ch2] = accB;
            } else {
                cl_st_f64(cl_map(&s.dsum[ch], 0), accA);
                if (ch2 < nch) cl_st_f64(cl_map(&s.dsum[ch2], 0), accB);
            }
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) {
        if constexpr (CL == 1) atomicOr(&s.rbad, EVICT_TREE_BAD_PROB);
        else cl_or_u32(cl_map(&s.rbad, 0), EVICT_TREE_BAD_PROB);
    }
    if constexpr (CL > 1) cl_sync(); else __syncthreads();
    if (r != 0) return;                             // the rest runs in CTA 0
    // s.st was 0 on entry (uniform across the cluster); bad bonus-row entries arrive in rbad
    if (s.rbad) {
        if (tid == 0) s.st |= s.rbad;
        return;
    }
    const int nrej = s.nrej;
    if (tid == 0) {
        double r = 0.0;
        for (int i = 0; i < nrej; i++) {
            const int t = s.rej[i];
            bool dup = false;
            for (int j = 0; j < i; j++) dup |= s.rej[j] == t;
            if (dup) continue;
            const double x = (double)__uint_as_float(__float_as_uint(row[t]) & 0x7fffffffu);
            s.dsum[t / kChunk] -= x;
            r += x;
        }
        s.rsum = r;
    }
    __syncthreads();
    if (w != 0) return;
    const int per = (nch + 31) / 32;
    const int c0 = lane * per, c1 = min(nch, c0 + per);
    double mine = 0.0;
    for (int c = c0; c < c1; c++) mine += s.dsum[c];
    double incl = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    double excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = 0.0;
    const double Zh = __shfl_sync(0xffffffffu, incl, 31);
    const double E = (double)(V + 2048 + 2 * nrej) * 0x1p-52 * (Zh + s.rsum);
    const double M = 3.0 * E;
    const double tau = ((double)ub * 0x1p-32) * Zh;
    const unsigned hit = __ballot_sync(0xffffffffu, incl > tau);
    bool cert = Zh > M && hit != 0u;
    int found = -1;
    if (cert) {
        const int L = __ffs(hit) - 1;
        int cross = -1;
        double pre = excl;
        if (lane == L) {
            for (int c = c0; c < c1; c++) {
                const double nx = pre + s.dsum[c];
                if (nx > tau) { cross = c; break; }
                pre = nx;
            }
        }
        cross = __shfl_sync(0xffffffffu, cross, L);
        pre = __shfl_sync(0xffffffffu, pre, L);
        if (cross < 0) {
            cert = false;
        } else {
            const int cb = cross * kChunk + lane * 16;
            double ls = 0.0;
            for (int q = 0; q < 16; q++) {
                const int t = cb + q;
                if (t >= V) break;
                bool gone = false;
                for (int i = 0; i < nrej; i++) gone |= s.rej[i] == t;
                if (!gone) ls += (double)__uint_as_float(__float_as_uint(row[t]) & 0x7fffffffu);
            }
            double li = ls;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, li, d);
                if (lane >= d) li += y;
            }
            li += pre;
            double ex2 = __shfl_up_sync(0xffffffffu, li, 1);
            if (lane == 0) ex2 = pre;
            const unsigned h2 = __ballot_sync(0xffffffffu, li > tau);
            if (!h2) {
                cert = false;
            } else {
                const int L2 = __ffs(h2) - 1;
                int tt = -1, ok = 0;
                if (lane == L2) {
                    double run = ex2;
                    for (int q = 0; q < 16; q++) {
                        const int t = cb + q;
                        if (t >= V) break;
                        bool gone = false;
                        for (int i = 0; i < nrej; i++) gone |= s.rej[i] == t;
                        const double x = gone ? 0.0 : (double)__uint_as_float(__float_as_uint(row[t]) & 0x7fffffffu);
                        const double prev = run;
                        run += x;
                        if (run > tau) {
                            tt = t;
                            ok = run > tau + M && prev < tau - M;
                            break;
                        }
                    }
                }
                tt = __shfl_sync(0xffffffffu, tt, L2);
                ok = __shfl_sync(0xffffffffu, ok, L2);
                cert = ok && tt >= 0;
                found = tt;
            }
        }
    }
    if (lane == 0) {
        s.cert = cert ? 1 : 0;
        s.bonus = found;
    }
}

template <int CL>
__global__ void __launch_bounds__(kThreads) k_verify(evict_verify_batch_t vb, const float *probs, int V,
                                                     long long stride, int mode, const uint32_t *u_accept,
                                                     const uint32_t *u_bonus, int32_t *accept_len,
                                                     int32_t *accepted_slots, int32_t *bonus_token,
                                                     uint32_t *status)
{
    __shared__ Smem s;
    const int b = blockIdx.x / CL, tid = threadIdx.x;
    const uint32_t rank = CL > 1 ? cl_rank() : 0u;
    const int N = vb.max_nodes;
    const int off = __ldg(vb.verify_offsets + b), k = __ldg(vb.verify_offsets + b + 1) - off;
    if (tid == 0) {
        s.st = k > N ? EVICT_TREE_BAD_SIZE : k < 1 ? EVICT_TREE_BAD_KEEP : 0u;   // k = 0: empty keep set
        s.k = k;
        s.nrej = 0;
        s.rbad = 0u;
    }
    if (tid < 16) (&s.cbad[0][0])[tid] = 0u;
    if constexpr (CL > 1) cl_sync(); else __syncthreads();   // every CTA of the cluster is live
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
    // parent slots and the orphan check run unless size/keep already failed (a bad token alone
    // must not hide a BAD_KEEP: the first failing check in header order is reported)
    if (!(s.st & (EVICT_TREE_BAD_SIZE | EVICT_TREE_BAD_KEEP))) {
        for (int q = tid; q < k; q += kThreads)
            for (int c = s.nt[q]; c != -1; c = s.ns[c]) s.ps[c] = q;
    }
    __syncthreads();
    if (!(s.st & (EVICT_TREE_BAD_SIZE | EVICT_TREE_BAD_KEEP))) {
        for (int q = 1 + tid; q < k; q += kThreads)
            if (s.ps[q] < 0) atomicOr(&s.st, EVICT_TREE_BAD_KEEP);   // an orphan slot
    }
    __syncthreads();
    // status precedence as the oracle: size/keep, then token, then prob
    if (tid == 0 && (s.st & (EVICT_TREE_BAD_SIZE | EVICT_TREE_BAD_KEEP))) s.st &= EVICT_TREE_BAD_SIZE | EVICT_TREE_BAD_KEEP;
    __syncthreads();

    if ((mode & 1) == EVICT_VERIFY_SAMPLE) {
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
            const uint32_t ub = __ldg(u_bonus + b);
            if (mode & EVICT_VERIFY_EXACT) {
                if (tid == 0) s.cert = 0;
            } else {
                bonus_fast<CL>(row, V, ub, s, tid);
            }
            __syncthreads();
            if (rank != 0 || s.st) goto done;
            if (!s.cert) bonus_exact(row, V, ub, s, tid);
        }
    } else {
        // greedy (T = 0): follow argmax through the kept children
        if (!s.st) {
            int u = 0, plen = 1, par = 0;
            if (tid == 0) s.path[0] = 0;
            for (;;) {
                const int g = row_argmax<CL>(probs + (long long)(off + u) * stride, V, s, tid, par);
                par ^= 1;
                if (g < 0) break;
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
    if (rank == 0) {
        const bool ok = s.st == 0;
        const int plen = ok ? s.plen : 0;
        for (int q = tid; q < N; q += kThreads) accepted_slots[(size_t)b * N + q] = q < plen ? s.path[q] : -1;
        if (tid == 0) {
            accept_len[b] = plen;
            bonus_token[b] = ok ? s.bonus : -1;
            if (status) status[b] = s.st;
        }
    }
    // no final cluster barrier: the last DSMEM writes (chunk sums into CTA 0, argmax partials)
    // precede a cluster barrier every CTA has passed, so peers may exit as soon as they are done
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
    if (mode & ~(1 | EVICT_VERIFY_EXACT)) return EVICT_ERR_INVALID_ARG;
    if ((mode & 1) == EVICT_VERIFY_SAMPLE && (!u_accept || !u_bonus)) return EVICT_ERR_INVALID_ARG;
    const int sms = evict::dev_sms();
    if (sms <= 0 || !evict::dev_supported()) return EVICT_ERR_UNSUPPORTED;
    // cluster size: split each tree's row over CL CTAs only until one wave of the 4 resident
    // CTAs per SM is full (64 trees → 8, 300 → 2, ≥ 592 → 1).  Past that a cluster only adds
    // redundant prologues and barriers: at 1024 trees CL = 1 / 2 / 4 / 8 measured 75% / 69% /
    // 60% / 44% of HBM for sampling.
    const long long target = 4LL * sms;
    int CL = 1;
    while (CL < 8 && (long long)vb->batch * CL < target) CL *= 2;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    cfg.gridDim = dim3((unsigned)(vb->batch * CL));
    cfg.blockDim = dim3(kThreads);
    cfg.stream = (cudaStream_t)stream;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    const evict_verify_batch_t v = *vb;
    switch (CL) {
    case 1: e = cudaLaunchKernelEx(&cfg, k_verify<1>, v, probs, (int)vocab, (long long)row_stride, (int)mode, u_accept, u_bonus, accept_len, accepted_slots, bonus_token, status); break;
    case 2: e = cudaLaunchKernelEx(&cfg, k_verify<2>, v, probs, (int)vocab, (long long)row_stride, (int)mode, u_accept, u_bonus, accept_len, accepted_slots, bonus_token, status); break;
    case 4: e = cudaLaunchKernelEx(&cfg, k_verify<4>, v, probs, (int)vocab, (long long)row_stride, (int)mode, u_accept, u_bonus, accept_len, accepted_slots, bonus_token, status); break;
    default: e = cudaLaunchKernelEx(&cfg, k_verify<8>, v, probs, (int)vocab, (long long)row_stride, (int)mode, u_accept, u_bonus, accept_len, accepted_slots, bonus_token, status); break;
    }
    if (e != cudaSuccess) return EVICT_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA;
}
