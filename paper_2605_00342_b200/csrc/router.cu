// router.cu — A8 → A7: router logits of the kept draft nodes on tcgen05 tensor
// cores, TopK, and the per-layer expert union (Eq. 4–5).
//
// One CTA = (layer l, 128 packed verify rows).  D[128 rows][128 experts] =
// H·W_gᵀ accumulates in TMEM (128 fp32 columns) over d in 64-wide k-blocks:
//   warps 0–3  gather the rows' hidden states (cp.async, 16 B per thread,
//              128-byte XOR swizzle) into a 6-stage ring, arriving on the
//              stage barrier asynchronously (cp.async.mbarrier.arrive.noinc),
//              then run the
//              epilogue: tcgen05.ld → per-row TopK (logit desc, expert asc)
//              → warp-aggregated atomicOr into the tree's union bitset
//   warp 4     one elected thread issues tcgen05.mma (M128 N128 K16, bf16 →
//              fp32, both operands K-major SWIZZLE_128B) and tcgen05.commit
//   warp 5     one thread streams W_g k-blocks with TMA (cp.async.bulk.tensor)
// mbarriers: full[s] (128 producer arrivals + TMA tx bytes), empty[s]
// (tcgen05.commit), tmem_full.  A finalize kernel turns bitsets into counts.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <mutex>

#include "evict.h"
#include "evict_launch.h"

namespace evict {
namespace router {

constexpr int BM = 128, BK = 64;   // rows per tile, k-block; the MMA N = E (128 or 256, template NE)
// operand ring depth (template): 6 stages (1 CTA/SM) when the grid fits one wave,
// 3 stages (2 CTAs/SM, 256 of 512 TMEM columns) when tiles × layers exceed the SMs
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
template <int NE> __host__ __device__ constexpr int b_bytes() { return NE * BK * 2; }            // 16 / 32 KB
template <int NE> __host__ __device__ constexpr int stage_bytes() { return A_BYTES + b_bytes<NE>(); }
constexpr int THREADS = 192;
constexpr int NPROD = 128;
constexpr int KMAX = 16;
constexpr int kMaxDev = 64;        // per-device host caches (function attributes, cluster occupancy)
template <int NE>
__host__ __device__ constexpr int smem_bytes(int stages)
{
    return stages * stage_bytes<NE>() + 1024 /*align*/ + 1024 /*barriers, ridx*/ + 512;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// arrive with a count (one thread completes `count` expected arrivals)
__device__ __forceinline__ void mbar_arrive_cnt(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
// raise the phase's expected transaction bytes without arriving
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *m)
{
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(bar),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t src_bytes)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t bar)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int x, int y)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
        : "memory");
}

// W_g k-block as a 3D box {64 cols, NE experts, 1 layer} of the [L][E][d] tensor: expert rows
// ≥ E (E < NE) fall outside the tensor and are zero-filled by TMA (their logits are masked).
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int x, int y, int z)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y), "r"(z)
        : "memory");
}

__device__ __forceinline__ void cluster_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_cluster(uint32_t addr, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ float4 ld_cluster_v4(uint32_t addr)
{
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}
__device__ __forceinline__ float ld_cluster_f32(uint32_t addr)
{
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// TMA row gather (sm_100a): 4 rows × one 64-column box, written as 4 consecutive
// 128-byte smem rows with the map's 128B swizzle.
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap *map, uint32_t bar, int col, int r0,
                                            int r1, int r2, int r3)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr)
{
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// Instruction descriptor: kind::f16, A/B bf16, D fp32, K-major, M=128, N=NE.
template <int NE>
__host__ __device__ constexpr uint32_t idesc() { return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NE >> 3) << 17) | ((uint32_t)(BM >> 4) << 24); }

template <int NE>
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate)
{
    constexpr uint32_t kIdesc = idesc<NE>();
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32])
{
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

// TopK of one row of BN logits under the key (logit desc, expert asc), a sorted
// register list of KL entries (KL compile-time so the list stays in registers).
// Entries j ≥ K hold +inf sentinels that are never displaced, so the list acts
// as length K.  Writes the ids (if out) and ORs them into the 4-word bitset w.
__device__ __forceinline__ long long gtimer()
{
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Expert bitset of one row: NE/32 words (scalars in registers after unrolling).
template <int NE>
struct Bits {
    uint32_t w[NE / 32];
};

template <int KL, int NE>
__device__ __forceinline__ Bits<NE> topk_scan(const float *lg, int K, bool valid, int32_t *out, long long *tr)
{
    constexpr int BN = NE;
    // Candidates are visited in expert order, so a new candidate loses every tie:
    // its rank is p = #{j < K : bv[j] >= v}; p == K never happens for a candidate
    // (it beats the K-th entry or the list is not full).  Insertion is a branch-free shift by
    // rank (independent selects, no dependent compare-swap chain), and a first
    // pass bounds the work: the minimum of the 8 group maxima (16 experts each)
    // is ≤ the 8th largest logit, so only values ≥ it can enter the list.
    float bv[KL];
    int bi[KL];
    const float ninf = -__int_as_float(0x7f800000);
    float gmin = __int_as_float(0x7f800000);
    const float4 *lg4 = reinterpret_cast<const float4 *>(lg);   // 16-byte aligned rows
#pragma unroll 1
    for (int g = 0; g < BN / 16; g++) {
        const float4 a = lg4[4 * g], b = lg4[4 * g + 1], c = lg4[4 * g + 2], d = lg4[4 * g + 3];
        const float m = fmaxf(fmaxf(fmaxf(fmaxf(a.x, a.y), fmaxf(a.z, a.w)), fmaxf(fmaxf(b.x, b.y), fmaxf(b.z, b.w))),
                              fmaxf(fmaxf(fmaxf(c.x, c.y), fmaxf(c.z, c.w)), fmaxf(fmaxf(d.x, d.y), fmaxf(d.z, d.w))));
        gmin = fminf(gmin, m);
    }
    // valid as a lower bound for the K-th largest only when K ≤ BN/16 groups
    // rows past T (zero-filled A tiles) have no candidates: all-equal rows would
    // otherwise walk every element through the candidate loop
    float thr = !valid ? __int_as_float(0x7f800000) : (K <= BN / 16) ? gmin : ninf;
    if (tr) tr[198] = gtimer();
    const long long c0 = tr ? clock64() : 0;
    int nins = 0;
#pragma unroll
    for (int j = 0; j < KL; j++) { bv[j] = ninf; bi[j] = 0x7fffffff; }
    int filled = 0;
    float kth = ninf;   // current K-th entry once the list is full
    // One warp per scheduler leaves no TLP to hide a per-element compare→branch
    // chain, so each 32-expert chunk is screened with independent compares into a
    // bit mask first and only the surviving candidates walk the insertion path.
    // The state only tightens (filled, kth grow), so a screened-out value can never
    // become a candidate again; survivors are re-checked before insertion.
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
        uint32_t cand = 0u;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const float4 x = lg4[(c >> 2) + q];
            const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const float v = xv[j];
                cand |= (v >= thr && (filled < K || v > kth)) ? (1u << (4 * q + j)) : 0u;
            }
        }
        while (cand) {
            const int i = c + __ffs(cand) - 1;
            cand &= cand - 1u;
            const float vi = lg[i];
            if (!(filled < K || vi > kth)) continue;
            int p = 0;
#pragma unroll
            for (int j = 0; j < KL; j++) p += (j < K && j < filled && bv[j] >= vi) ? 1 : 0;
            float nb[KL];
            int ni[KL];
#pragma unroll
            for (int j = 0; j < KL; j++) {
                const float prev = j > 0 ? bv[j - 1] : ninf;
                const int previ = j > 0 ? bi[j - 1] : 0x7fffffff;
                nb[j] = j < p ? bv[j] : (j == p ? vi : prev);
                ni[j] = j < p ? bi[j] : (j == p ? i : previ);
            }
#pragma unroll
            for (int j = 0; j < KL; j++) { bv[j] = nb[j]; bi[j] = ni[j]; }
            filled = filled < K ? filled + 1 : K;
            nins++;
            // sorted descending: the K-th entry is the minimum of the first K
            // (a min-reduction, not a select, so it stays in registers)
            kth = __int_as_float(0x7f800000);
#pragma unroll
            for (int j = 0; j < KL; j++) kth = fminf(kth, j < K ? bv[j] : kth);
        }
    }
    if (tr) { tr[199] = gtimer(); tr[200] = nins; tr[201] = clock64() - c0; }
    // word select by compile-time-unrolled compares (a dynamically indexed word
    // would turn the set into a local-memory array)
    Bits<NE> r;
#pragma unroll
    for (int q = 0; q < NE / 32; q++) r.w[q] = 0u;
#pragma unroll
    for (int j = 0; j < KL; j++) {
        const int e = bi[j];
        const bool ok = j < K && e >= 0 && e < BN;
        const uint32_t bit = ok ? (1u << (e & 31)) : 0u;
        const int q = e >> 5;
#pragma unroll
        for (int qq = 0; qq < NE / 32; qq++) r.w[qq] |= q == qq ? bit : 0u;
        if (ok && valid && out) out[j] = e;
    }
    return r;
}

// TopK of one row by a whole warp (sparse tiles: few valid rows would leave one
// thread per row with no latency hiding).  Lane holds experts lane + 32q; each of
// the K rounds takes the warp max under (logit desc, expert asc) with two
// reductions (orderable logit bits, then the smallest expert among the maxima)
// and retires the winner.  Every lane ends with the same ids and bit words.
__device__ __forceinline__ uint32_t f2ord(float f)
{
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
template <int NE>
__device__ __forceinline__ Bits<NE> topk_warp_row(const float *lgrow, int K, int32_t *out, int lane)
{
    constexpr int Q = NE / 32;
    float v[Q];
#pragma unroll
    for (int q = 0; q < Q; q++) v[q] = lgrow[lane + 32 * q];
    Bits<NE> r;
#pragma unroll
    for (int q = 0; q < Q; q++) r.w[q] = 0u;
    const float ninf = -__int_as_float(0x7f800000);
#pragma unroll 1
    for (int j = 0; j < K; j++) {
        float m = v[0];
#pragma unroll
        for (int q = 1; q < Q; q++) m = fmaxf(m, v[q]);
        const uint32_t u = f2ord(m);
        const uint32_t U = __reduce_max_sync(0xffffffffu, u);
        int el = 0xffff;
#pragma unroll
        for (int q = Q - 1; q >= 0; q--) el = (v[q] == m) ? lane + 32 * q : el;
        const int e = (int)__reduce_min_sync(0xffffffffu, u == U ? (uint32_t)el : 0xffffu);
        if ((e & 31) == lane) {
#pragma unroll
            for (int q = 0; q < Q; q++) v[q] = (q == (e >> 5)) ? ninf : v[q];
        }
        const uint32_t bit = 1u << (e & 31);
        const int qw = e >> 5;
#pragma unroll
        for (int q = 0; q < Q; q++) r.w[q] |= qw == q ? bit : 0u;
        if (out && lane == 0) out[j] = e;
    }
    return r;
}

// TopK of one row by a whole warp as a truncated merge network: lane j holds experts j + 32q as
// 64-bit keys (orderable logit bits << 32 | ~expert: larger key = larger logit, ties → smaller
// expert), sorts its Q keys, then 5 xor-levels each merge two sorted KL-lists into the top KL of
// their union (elementwise max of a and reversed b is bitonic; log2(KL) half-cleaner stages sort
// it).  Every lane ends with the same top-KL; the first K are the TopK in rank order.
__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m)
{
    const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, m);
    const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), m);
    return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t tkey(float v, int e)
{
    return ((uint64_t)f2ord(v) << 32) | (uint32_t)(~(uint32_t)e);
}
__device__ __forceinline__ void ce_desc(uint64_t &x, uint64_t &y)
{
    const uint64_t hi = x > y ? x : y, lo = x > y ? y : x;
    x = hi;
    y = lo;
}
template <int NE, int KL>
__device__ __forceinline__ Bits<NE> topk_warp_merge(const float *lgrow, int K, int32_t *out, int lane)
{
    constexpr int Q = NE / 32;            // 4 (E ≤ 128) or 8 keys per lane
    static_assert(Q <= KL, "a lane's keys fit its list");
    uint64_t a[KL];
#pragma unroll
    for (int j = 0; j < KL; j++) a[j] = j < Q ? tkey(lgrow[lane + 32 * j], lane + 32 * j) : 0ull;
    // local bitonic sort (descending) of the first Q keys; key 0 sorts below every real key
#pragma unroll
    for (int k = 2; k <= Q; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < Q; i++) {
                const int ip = i ^ j;
                if (ip > i) {
                    if ((i & k) == 0) ce_desc(a[i], a[ip]);
                    else ce_desc(a[ip], a[i]);
                }
            }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t c[KL];
#pragma unroll
        for (int j = 0; j < KL; j++) {
            const uint64_t bj = shfl_xor_u64(a[KL - 1 - j], o);
            c[j] = a[j] > bj ? a[j] : bj;
        }
#pragma unroll
        for (int j = KL >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < KL; i++)
                if ((i & j) == 0) ce_desc(c[i], c[i + j]);
#pragma unroll
        for (int j = 0; j < KL; j++) a[j] = c[j];
    }
    Bits<NE> r;
#pragma unroll
    for (int q = 0; q < NE / 32; q++) r.w[q] = 0u;
#pragma unroll
    for (int j = 0; j < KL; j++) {
        if (j < K) {
            const int e = (int)(~(uint32_t)a[j]);
            const uint32_t bit = 1u << (e & 31);
#pragma unroll
            for (int q = 0; q < NE / 32; q++) r.w[q] |= (e >> 5) == q ? bit : 0u;
            if (out && lane == j) out[j] = e;
        }
    }
    return r;
}

struct Params {
    const uint16_t *hidden;        // bf16 [L][BNrows][d]
    const int32_t *verify_offsets; // [B+1]
    const int32_t *retrieve_index; // [cap]
    int L, B, N, d, K;
    int E;                         // real experts (≤ NE): logits of columns ≥ E are masked to -inf
    int EWo;                       // output bit words per (tree, layer) = ceil(E/64)
    int splits;                    // k-splits = cluster size along z (1: no cluster)
    unsigned long long *bits;      // [B][L][EWo]
    int32_t *topk_ids;             // [L][B*N][K] or null
    float *dbg_logits;             // [L][B*N][128] or null (debug entry point only)
    long long *trace;              // [256] globaltimer trace of CTA (0,0) or null (debug only)
};


template <int NE, int STAGES>
__global__ void __launch_bounds__(THREADS, STAGES <= 3 ? 2 : 1)
k_router(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap hmap, Params p)
{
    constexpr int BN = NE, EW = NE / 64;
    constexpr int LS = BN + 4;   // staged logit row stride (floats): 16-byte rows, conflict-free float4 phases
    constexpr int B_BYTES = b_bytes<NE>(), STAGE_BYTES = stage_bytes<NE>();
    static_assert(BM * LS * 4 <= STAGES * STAGE_BYTES, "logit staging must fit the operand ring");
    extern __shared__ uint8_t smem_raw[];
    const int m0 = blockIdx.x * BM;
    const int l = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t *base = smem_raw + (base_u32 - smem_u32(smem_raw));
    uint8_t *meta = base + STAGES * STAGE_BYTES;
    uint64_t *bars = reinterpret_cast<uint64_t *>(meta);   // full[S], empty[S], tmem_full
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(meta + 8 * (2 * STAGES + 1));
    int *ridx = reinterpret_cast<int *>(meta + 256);
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES), tfull = smem_u32(bars + 2 * STAGES);
    auto A = [&](int s) { return base_u32 + s * STAGE_BYTES; };
    auto Bs = [&](int s) { return base_u32 + s * STAGE_BYTES + A_BYTES; };

    const bool tr0 = p.trace && blockIdx.x == 0 && blockIdx.y == 0;
    const int KB = p.d / BK;
    // split z of S takes k-blocks [kb0, kb1); the S CTAs of a cluster share (tile, layer)
    const int S = p.splits, z = blockIdx.z;
    const int kb0 = (int)(((long)KB * z) / S), kb1 = (int)(((long)KB * (z + 1)) / S);
    const int NKB = kb1 - kb0;
    const int first = NKB < STAGES ? NKB : STAGES;
    if (tr0 && threadIdx.x == 0) {
        p.trace[250] = gtimer();
        p.trace[251] = p.splits;
    }
    // full[s] expects NPROD + 1 arrivals: the W_g thread (arrive + its tx bytes) and the hidden
    // rows — 128 cp.async producers (dense tiles) or one gather4 thread arriving with count NPROD
    // after raising the tx bytes (sparse tiles); the same count either way, so the barriers and
    // the first W_g loads go out before T (device-resident) is known
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(full0 + 8 * s, NPROD + 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(tfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 5 && lane == 0) {
        prefetch_tmap(&wmap);
        prefetch_tmap(&hmap);
        for (int i = 0; i < first; i++) {
            mbar_arrive_tx(full0 + 8 * i, B_BYTES);
            tma_load_3d(Bs(i), &wmap, full0 + 8 * i, (kb0 + i) * BK, 0, l);
        }
    }
    const int T = __ldg(p.verify_offsets + p.B);
    if (m0 >= T) {
        // no rows in this tile: complete the issued stages' phases and wait for their W_g bytes
        // (no TMA may land in an exited CTA)
        if (threadIdx.x == 0) {
            for (int s = 0; s < first; s++) mbar_arrive_cnt(full0 + 8 * s, NPROD);
            for (int s = 0; s < first; s++) mbar_wait(full0 + 8 * s, 0);
        }
        return;   // uniform per CTA; TMEM not yet allocated; no cluster peers (splits share T)
    }
    const int nrow = T - m0 < BM ? T - m0 : BM;   // valid rows of this tile
    // sparse tiles gather their few hidden rows with TMA (gather4, one issuing thread);
    // dense tiles use 128 cp.async producers (one TMA thread would serialise 32 gathers)
    const bool sparse = nrow <= 32;
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(NE) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x < BM) {
        const int r = m0 + threadIdx.x;
        ridx[threadIdx.x] = r < T ? __ldg(p.retrieve_index + r) : -1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const size_t BNrows = (size_t)p.B * p.N;
    const int row = warp * 32 + lane;         // epilogue row (warps 0–3)
    float *lg = reinterpret_cast<float *>(base) + (size_t)(row & (BM - 1)) * LS;

    if (warp < 4) {
        if (!sparse) {
            // ---- producers: gather 128 rows × 64 bf16 per stage, 128-byte XOR swizzle
            const int t = threadIdx.x, c = t & 7, r0 = t >> 3;
            const uint16_t *hl = p.hidden + (size_t)l * BNrows * p.d;
            for (int i = 0; i < NKB; i++) {
                const int kb = kb0 + i, s = i % STAGES;
                if (i >= STAGES) mbar_wait(empty0 + 8 * s, ((i / STAGES) - 1) & 1);
                if (tr0 && threadIdx.x == 0 && i < 64) p.trace[128 + i] = gtimer();
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const int rr = r0 + 16 * j;
                    const int rid = ridx[rr];
                    const uint16_t *src = hl + (size_t)(rid < 0 ? 0 : rid) * p.d + kb * BK + c * 8;
                    cp_async16(A(s) + rr * 128 + ((c ^ (rr & 7)) << 4), src, rid < 0 ? 0u : 16u);
                }
                // arrive on full[s] asynchronously once this thread's copies have landed:
                // the producer never blocks on its own loads, only on slot reuse (empty[s])
                cp_async_arrive_noinc(full0 + 8 * s);
            }
            cp_async_wait<0>();
        } else if (warp == 0) {
            // ---- sparse tile: one thread gathers the valid rows (4-row groups) per stage with
            // TMA gather4, while warp 5 streams W_g (two issuers, one stage barrier)
            if (lane == 0) {
                const int ng = (nrow + 3) >> 2;
                const int lrow = l * (int)BNrows;
                for (int i = 0; i < NKB; i++) {
                    const int kb = kb0 + i, s = i % STAGES;
                    if (i >= STAGES) mbar_wait(empty0 + 8 * s, ((i / STAGES) - 1) & 1);
                    mbar_expect_tx(full0 + 8 * s, 512u * ng);
                    for (int g4 = 0; g4 < ng; g4++) {
                        int rr[4];
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            const int row_ = 4 * g4 + u;
                            rr[u] = lrow + ridx[row_ < nrow ? row_ : 0];
                        }
                        tma_gather4(A(s) + g4 * 512, &hmap, full0 + 8 * s, kb * BK, rr[0], rr[1], rr[2], rr[3]);
                    }
                    mbar_arrive_cnt(full0 + 8 * s, NPROD);
                }
            }
            __syncwarp();
        }
        // ---- stage the (partial) accumulator: TMEM → registers → shared memory
        if (tr0 && threadIdx.x == 0) p.trace[192] = gtimer();
        mbar_wait(tfull, 0);
        if (tr0 && threadIdx.x == 0) p.trace[193] = gtimer();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // the operand ring is free now; rows of LS = BN + 4 floats written as float4: an 8-thread
        // phase of a 16-byte store covers 8 distinct 4-bank groups
#pragma unroll 1
        for (int chunk = 0; chunk < BN / 32; chunk++) {
            float v[32];
            tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + chunk * 32, v);
            if (chunk * 32 + 32 > p.E) {   // E < NE: padding experts never enter the TopK
#pragma unroll
                for (int j = 0; j < 32; j++) v[j] = chunk * 32 + j < p.E ? v[j] : -__int_as_float(0x7f800000);
            }
            float4 *l4 = reinterpret_cast<float4 *>(lg + chunk * 32);
#pragma unroll
            for (int q = 0; q < 8; q++) l4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
        if (tr0 && threadIdx.x == 0) p.trace[196] = gtimer();
    } else if (warp == 4) {
        // ---- MMA issuer
        if (lane == 0) {
            for (int i = 0; i < NKB; i++) {
                const int s = i % STAGES;
                mbar_wait(full0 + 8 * s, (i / STAGES) & 1);
                if (tr0 && i < 64) p.trace[i] = gtimer();
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int k = 0; k < BK / 16; k++)
                    umma_bf16<NE>(tmem, umma_desc(A(s) + 32 * k), umma_desc(Bs(s) + 32 * k), (i | k) != 0);
                umma_commit(empty0 + 8 * s);
            }
            umma_commit(tfull);
        }
        __syncwarp();
    } else {
        // ---- W_g k-blocks via TMA (3D box, the first `first` were issued in the prologue); the
        // hidden rows come from warps 0–3 (rows past T in a sparse tile's last gather4 group
        // repeat a valid row — an A row only feeds its own D row, which nobody reads)
        if (lane == 0) {
            for (int i = first; i < NKB; i++) {
                const int kb = kb0 + i, s = i % STAGES;
                mbar_wait(empty0 + 8 * s, ((i / STAGES) - 1) & 1);
                if (tr0 && i < 64) p.trace[64 + i] = gtimer();
                mbar_arrive_tx(full0 + 8 * s, B_BYTES);
                tma_load_3d(Bs(s), &wmap, full0 + 8 * s, kb * BK, 0, l);
            }
        }
        __syncwarp();
    }
    if (tr0 && threadIdx.x == 0) p.trace[194] = gtimer();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tr0 && threadIdx.x == 0) p.trace[195] = gtimer();
    if (warp == 4) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(NE) : "memory");
    }
    if (S > 1) cluster_sync();                // every split's partial is staged

    if (warp < 4 && (S > 1 || z == 0)) {
        // ---- split-K: every split reduces and ranks a contiguous block of ⌈nrow/S⌉ rows (the sum
        // order per element stays split 0 + 1 + … + S−1: deterministic, as one leader would)
        const int r = m0 + row;
        const bool valid = r < T;
        int r0 = 0, r1 = nrow;
        if (S > 1) {
            const int R = (nrow + S - 1) / S;
            r0 = min(nrow, z * R);
            r1 = min(nrow, r0 + R);
            float4 *lg4 = reinterpret_cast<float4 *>(base);
            const uint32_t mine = smem_u32(base);
            const int f0 = (r0 * LS) >> 2, f1 = (r1 * LS) >> 2;   // LS % 4 == 0: whole float4 rows
            uint32_t rem[4];
#pragma unroll
            for (int zz = 0; zz < 4; zz++) rem[zz] = zz < S ? mapa_cluster(mine, (uint32_t)zz) : 0u;
#pragma unroll 1
            for (int f = f0 + threadIdx.x; f < f1; f += BM) {
                float4 acc = ld_cluster_v4(rem[0] + 16u * f);
                float4 t[3];
#pragma unroll
                for (int zz = 1; zz < 4; zz++)
                    if (zz < S) t[zz - 1] = ld_cluster_v4(rem[zz] + 16u * f);
#pragma unroll
                for (int zz = 1; zz < 4; zz++)
                    if (zz < S) {
                        acc.x += t[zz - 1].x; acc.y += t[zz - 1].y; acc.z += t[zz - 1].z; acc.w += t[zz - 1].w;
                    }
                lg4[f] = acc;   // own rows only: no other split reads this block after the barrier
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");   // warps 0–3 only
        }
        if (p.dbg_logits && valid && row >= r0 && row < r1)
            for (int i = 0; i < BN; i++) p.dbg_logits[((size_t)l * BNrows + r) * BN + i] = lg[i];
        if (S > 1 || nrow <= 32) {
            // a warp per row (rows r0 + warp, + 4, …), one atomic group per row: sparse tiles, and
            // every split's block of a split-K tile
#pragma unroll 1
            for (int rr = r0 + warp; rr < r1; rr += 4) {
                const int rg = m0 + rr;
                int32_t *o = p.topk_ids ? p.topk_ids + ((size_t)l * BNrows + rg) * p.K : nullptr;
                const float *lrow = reinterpret_cast<const float *>(base) + (size_t)rr * LS;
                const Bits<NE> wr = p.K <= 8 ? topk_warp_merge<NE, 8>(lrow, p.K, o, lane)
                                             : topk_warp_merge<NE, 16>(lrow, p.K, o, lane);
                if (lane == 0) {
                    unsigned long long *dst = p.bits + ((size_t)(ridx[rr] / p.N) * p.L + l) * p.EWo;
#pragma unroll
                    for (int h = 0; h < EW; h++)
                        if (h < p.EWo) atomicOr(dst + h, (unsigned long long)wr.w[2 * h] | ((unsigned long long)wr.w[2 * h + 1] << 32));
                }
            }
            if (tr0 && threadIdx.x == 0) p.trace[197] = gtimer();
        } else {
        long long *ttr = (tr0 && threadIdx.x == 0) ? p.trace : nullptr;
        int32_t *tk_out = p.topk_ids ? p.topk_ids + ((size_t)l * BNrows + r) * p.K : nullptr;
        const Bits<NE> wq = p.K <= 8 ? topk_scan<8, NE>(lg, p.K, valid, tk_out, ttr)
                                     : topk_scan<KMAX, NE>(lg, p.K, valid, tk_out, ttr);
        if (tr0 && threadIdx.x == 0) p.trace[197] = gtimer();
        const int tree = valid ? ridx[row] / p.N : -1;
        unsigned pending = __ballot_sync(0xffffffffu, valid);
        while (pending) {
            const int leader = __ffs(pending) - 1;
            const int tb = __shfl_sync(0xffffffffu, tree, leader);
            const unsigned grp = __ballot_sync(0xffffffffu, valid && tree == tb);
            const bool in = (grp >> lane) & 1u;
            uint32_t o[NE / 32];
#pragma unroll
            for (int q = 0; q < NE / 32; q++) o[q] = __reduce_or_sync(0xffffffffu, in ? wq.w[q] : 0u);
            if (lane == leader) {
                unsigned long long *dst = p.bits + ((size_t)tb * p.L + l) * p.EWo;
#pragma unroll
                for (int h = 0; h < EW; h++)
                    if (h < p.EWo) atomicOr(dst + h, (unsigned long long)o[2 * h] | ((unsigned long long)o[2 * h + 1] << 32));
            }
            pending &= ~grp;
        }
        }
    }
    if (S > 1) cluster_sync();                // partials stay alive until every split has read them
}

__global__ void k_finalize(int B, int L, int EW, const unsigned long long *bits, int32_t *count, int32_t *total)
{
    const int b = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (b >= B) return;
    int tot = 0;
    for (int l = lane; l < L; l += 32) {
        int c = 0;
        for (int h = 0; h < EW; h++) c += __popcll(bits[((size_t)b * L + l) * EW + h]);
        count[(size_t)b * L + l] = c;
        tot += c;
    }
    tot = __reduce_add_sync(0xffffffffu, tot);
    if (total && lane == 0) total[b] = tot;
}

// ---------------------------------------------------------------- host
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn()
{
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    });
    return fn;
}

}  // namespace router
}  // namespace evict

using namespace evict::router;

static evict_status_t router_impl(const evict_trees_t *trees, const int32_t *verify_offsets,
                                  const int32_t *retrieve_index, const evict_router_t *rt,
                                  int32_t *union_count, int32_t *union_total, uint64_t *union_bits,
                                  int32_t *topk_ids, float *dbg_logits, long long *trace, void *stream);

extern "C" evict_status_t evict_router_union(const evict_trees_t *trees, const int32_t *verify_offsets,
                                             const int32_t *retrieve_index, const evict_router_t *rt,
                                             int32_t *union_count, int32_t *union_total,
                                             uint64_t *union_bits, int32_t *topk_ids, void *stream)
{
    return router_impl(trees, verify_offsets, retrieve_index, rt, union_count, union_total, union_bits,
                       topk_ids, nullptr, nullptr, stream);
}

// Debug entry point (not part of include/evict.h): also dumps the raw fp32 logits.
extern "C" evict_status_t evict_router_union_debug(const evict_trees_t *trees, const int32_t *verify_offsets,
                                                   const int32_t *retrieve_index, const evict_router_t *rt,
                                                   int32_t *union_count, int32_t *union_total,
                                                   uint64_t *union_bits, int32_t *topk_ids, float *logits,
                                                   long long *trace, void *stream)
{
    return router_impl(trees, verify_offsets, retrieve_index, rt, union_count, union_total, union_bits,
                       topk_ids, logits, trace, stream);
}

static evict_status_t router_impl(const evict_trees_t *trees, const int32_t *verify_offsets,
                                  const int32_t *retrieve_index, const evict_router_t *rt,
                                  int32_t *union_count, int32_t *union_total, uint64_t *union_bits,
                                  int32_t *topk_ids, float *dbg_logits, long long *trace, void *stream)
{
    if (!trees || !rt || !verify_offsets || !retrieve_index || !union_count || !union_bits)
        return EVICT_ERR_INVALID_ARG;
    if (trees->batch < 1 || trees->max_nodes < 1 || trees->max_nodes > EVICT_MAX_NODES) return EVICT_ERR_INVALID_ARG;
    if (!rt->hidden || !rt->w_gate || rt->num_layers < 1 || rt->num_layers > EVICT_MAX_LAYERS)
        return EVICT_ERR_INVALID_ARG;
    if (rt->top_k < 1 || rt->top_k > EVICT_MAX_TOPK || rt->top_k > rt->num_experts) return EVICT_ERR_INVALID_ARG;
    if (rt->hidden_dim < 64 || rt->hidden_dim % 64) return EVICT_ERR_INVALID_ARG;
    if (((uintptr_t)rt->hidden | (uintptr_t)rt->w_gate) & 15) return EVICT_ERR_INVALID_ARG;
    if (rt->num_experts < 1 || rt->num_experts > 256) return EVICT_ERR_UNSUPPORTED;
    if (!evict::dev_supported()) return EVICT_ERR_UNSUPPORTED;
    EncodeTiledFn enc = encode_fn();
    if (!enc) return EVICT_ERR_UNSUPPORTED;
    const int L = rt->num_layers, E = rt->num_experts, d = rt->hidden_dim;
    const int B = trees->batch, N = trees->max_nodes;
    // the MMA width: N = 128 for E ≤ 128, N = 256 for 128 < E ≤ 256 (columns ≥ E masked)
    const int wide = E > 128;
    const int NE = wide ? 256 : 128;
    CUtensorMap map;
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)E, (cuuint64_t)L};
    cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)E * d * 2};
    cuuint32_t box[3] = {BK, (cuuint32_t)NE, 1};   // one W_g k-block: NE expert rows, zero-filled past E
    cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(rt->w_gate), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return EVICT_ERR_INVALID_ARG;
    // hidden rows are gathered by TMA with int32 row coordinates over the [L·B·N][d] view
    if ((size_t)L * B * N >= (size_t)1 << 31) return EVICT_ERR_UNSUPPORTED;
    CUtensorMap hmap;
    cuuint64_t hdims[2] = {(cuuint64_t)d, (cuuint64_t)L * B * N};
    cuuint32_t hbox[2] = {BK, 1};
    if (enc(&hmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(rt->hidden), hdims, strides, hbox, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return EVICT_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    // function attributes are per device: opt in to > 48 KB of shared memory once per device
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return EVICT_ERR_UNSUPPORTED;
    static std::once_flag attr_once[kMaxDev];
    std::call_once(attr_once[dev], [] {
        cudaFuncSetAttribute(k_router<128, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<128>(6));
        cudaFuncSetAttribute(k_router<128, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<128>(3));
        cudaFuncSetAttribute(k_router<256, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<256>(4));
    });
    const int EW = (E + 63) / 64;   // output words per (tree, layer)
    if (cudaMemsetAsync(union_bits, 0, sizeof(uint64_t) * (size_t)B * L * EW, s) != cudaSuccess) return EVICT_ERR_CUDA;
    Params p;
    p.hidden = (const uint16_t *)rt->hidden;
    p.verify_offsets = verify_offsets;
    p.retrieve_index = retrieve_index;
    p.L = L; p.B = B; p.N = N; p.d = d; p.K = rt->top_k;
    p.E = E; p.EWo = EW;
    p.bits = reinterpret_cast<unsigned long long *>(union_bits);
    p.topk_ids = topk_ids;
    p.dbg_logits = dbg_logits;
    p.trace = trace;
    // Split the d-reduction over a cluster of S CTAs when the (tile, layer) grid would leave
    // SMs idle (batch-1 serving: one 128-row tile × L layers < #SMs).  The host bounds the
    // active tiles by B·N rows (T is device-resident).
    if (rt->max_rows < 0) return EVICT_ERR_INVALID_ARG;
    const size_t rows_bound = rt->max_rows > 0 && (size_t)rt->max_rows < (size_t)B * N ? (size_t)rt->max_rows
                                                                                          : (size_t)B * N;
    const int tiles = (int)((rows_bound + BM - 1) / BM);
    const int KB = d / BK;
    // Split the d-reduction over a cluster of S CTAs when the (tile, layer) grid would leave SMs
    // idle (batch-1 serving: one 128-row tile × L layers < #SMs).  Every CTA streams its W_g
    // k-blocks as 128-byte rows, so the per-SM request rate, not HBM, bounds a lone CTA: the more
    // SMs stream, the closer the call gets to the HBM roofline.  Candidates: the 6-stage ring
    // (1 CTA/SM, S ≤ SMs/(tiles·L)) and the 3-stage ring (2 CTAs/SM, S ≤ 2·SMs/(tiles·L));
    // clusters are placed GPC by GPC, so a split counts only if all tiles·L clusters are
    // co-resident (cudaOccupancyMaxActiveClusters; a second wave would double the time).
    const int sms = evict::dev_sms();
    const long grid1 = (long)tiles * L;
    static int max_clusters[kMaxDev][2][5] = {};
    static bool mc_known[kMaxDev][2][5] = {};
    static std::mutex mc_mu;
    auto fits = [&](int deep, int S_) -> bool {   // deep: 6-stage (1 CTA/SM), else 3-stage
        std::lock_guard<std::mutex> g(mc_mu);
        if (!mc_known[dev][deep][S_]) {
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3((unsigned)S_, 1u, 1u);
            q.blockDim = dim3(THREADS, 1, 1);
            q.dynamicSmemBytes = deep ? smem_bytes<128>(6) : smem_bytes<128>(3);
            cudaLaunchAttribute a[1];
            a[0].id = cudaLaunchAttributeClusterDimension;
            a[0].val.clusterDim.x = (unsigned)S_;
            a[0].val.clusterDim.y = 1;
            a[0].val.clusterDim.z = 1;
            q.attrs = a;
            q.numAttrs = 1;
            int n = 0;
            const cudaError_t qe = deep ? cudaOccupancyMaxActiveClusters(&n, k_router<128, 6>, &q)
                                        : cudaOccupancyMaxActiveClusters(&n, k_router<128, 3>, &q);
            max_clusters[dev][deep][S_] = qe == cudaSuccess ? n : 0;
            mc_known[dev][deep][S_] = true;
        }
        return max_clusters[dev][deep][S_] >= grid1;
    };
    int S = 1, deep = grid1 <= sms;
    if (wide) {
        // 256 experts: 48 KB stages, 1 CTA/SM, ≤ 4-CTA clusters — placed without the query
        S = (int)(sms / grid1);
        S = S < 1 ? 1 : (S > 4 ? 4 : S);
    } else {
        for (int S_ = 4; S_ >= 2 && S == 1; S_--) {
            if (S_ > KB) continue;
            if ((long)S_ * grid1 <= sms && fits(1, S_)) { S = S_; deep = 1; }
            else if ((long)S_ * grid1 <= 2L * sms && fits(0, S_)) { S = S_; deep = 0; }
        }
    }
    if (const char *ov = getenv("EVICT_ROUTER_SPLITS")) {   // measurement override (dev only)
        const int o = atoi(ov);
        if (o >= 1 && o <= 4 && o <= KB) { S = o; if (!wide) deep = (long)S * grid1 <= sms; }
    }
    p.splits = S;
    if (S == 1) {
        dim3 grid((unsigned)tiles, (unsigned)L, 1u);
        if (wide) k_router<256, 4><<<grid, THREADS, smem_bytes<256>(4), s>>>(map, hmap, p);
        else if (!deep) k_router<128, 3><<<grid, THREADS, smem_bytes<128>(3), s>>>(map, hmap, p);
        else k_router<128, 6><<<grid, THREADS, smem_bytes<128>(6), s>>>(map, hmap, p);
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)tiles, (unsigned)L, (unsigned)S);
        cfg.blockDim = dim3(THREADS, 1, 1);
        cfg.dynamicSmemBytes = wide ? smem_bytes<256>(4) : (deep ? smem_bytes<128>(6) : smem_bytes<128>(3));
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 1;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = (unsigned)S;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const cudaError_t le = wide ? cudaLaunchKernelEx(&cfg, k_router<256, 4>, map, hmap, p)
                               : deep ? cudaLaunchKernelEx(&cfg, k_router<128, 6>, map, hmap, p)
                                      : cudaLaunchKernelEx(&cfg, k_router<128, 3>, map, hmap, p);
        if (le != cudaSuccess) return EVICT_ERR_CUDA;
    }
    if (cudaGetLastError() != cudaSuccess) return EVICT_ERR_CUDA;
    k_finalize<<<(B + 7) / 8, 256, 0, s>>>(B, L, EW, reinterpret_cast<const unsigned long long *>(union_bits),
                                           union_count, union_total);
    return cudaGetLastError() == cudaSuccess ? EVICT_OK : EVICT_ERR_CUDA;
}
