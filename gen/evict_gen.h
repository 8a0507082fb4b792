/*
 * evict_gen.h — seeded synthetic workload generator (single source).
 *
 * This module is the ONLY thing the oracle side and the CUDA side share: it
 * makes inputs (draft trees, routing ids, hidden states, router weights) and
 * holds none of the method's arithmetic.  It is compiled twice: by gcc into
 * gen/libevictgen_host.so (inputs for oracle parity tests) and by nvcc into
 * gen/libevictgen_cuda.so (device-resident inputs for the bench), and both
 * builds produce bit-identical data because every operation here is either
 * integer arithmetic or a correctly-rounded IEEE fp64 operation written
 * without contraction (tests/test_gen.py checks host == device on the GPU).
 *
 * Counter-based: every value is a pure function of (seed, tree_id, ...), so
 * a rank generates its own shard of trees and any sampled tree can be
 * regenerated on the host alone.
 *
 * Recipe:
 *  - Draft trees emulate the EAGLE-2/3 drafter:
 *    the root expands `topk` children; each later step expands the `topk`
 *    best frontier nodes (by the drafter's cumulative probability) into
 *    `topk` children each; every candidate enters a pool; the pool is pruned
 *    to the best N−1 nodes plus the root and renumbered in creation order
 *    (topological).  Child probabilities: sorted top-`topk` of topk+1
 *    weights u^m (u uniform in (0,1), the last weight is "rest of vocab"),
 *    normalised; m is a per-tree difficulty exponent in [m_lo, m_hi]
 *    (m=1: hard/flat, m=16: easy/peaked).
 *  - Routing ids: logit_{l,e}(v) = s·z_{tree,l,e} + 4·ε_{v,l,e} with z, ε
 *    integer Irwin–Hall(4) samples; ids = top-K by (logit desc, e asc).
 *    s = round(4·σ_b) (σ_b = 2.25 ⇒ s = 9).
 *  - Hidden states / router weights: integers in [−2, 2] (mode 0, exact
 *    fp32 logits) or bf16 approx-normal (mode 1).
 */
#ifndef EVICT_GEN_H
#define EVICT_GEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define GEN_FN __host__ __device__ static inline
#else
#define GEN_FN static inline
#endif

#if defined(__CUDA_ARCH__)
#define GEN_DMUL(a, b) __dmul_rn((a), (b))
#define GEN_DADD(a, b) __dadd_rn((a), (b))
#define GEN_DDIV(a, b) __ddiv_rn((a), (b))
#define GEN_D2F(a) __double2float_rn(a)
#else
#define GEN_DMUL(a, b) ((a) * (b))
#define GEN_DADD(a, b) ((a) + (b))
#define GEN_DDIV(a, b) ((a) / (b))
#define GEN_D2F(a) ((float)(a))
#endif

#define GEN_MAX_TOPK 16
#define GEN_MAX_POOL 1024
#define GEN_MAX_NODES 128
#define GEN_MAX_EXPERTS 256
#define GEN_MAX_K 16

/* stream ids keep independent draws apart */
#define GEN_S_DIFF 1u
#define GEN_S_CHILD 2u
#define GEN_S_RZ 3u
#define GEN_S_REPS 4u
#define GEN_S_HID 5u
#define GEN_S_WG 6u

GEN_FN uint64_t gen_mix64(uint64_t z)
{
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

GEN_FN uint64_t gen_hash(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b)
{
    uint64_t h = gen_mix64(seed + 0x9E3779B97F4A7C15ull);
    h = gen_mix64(h ^ (stream * 0xD6E8FEB86659FD93ull + 0x632BE59BD9B4E019ull));
    h = gen_mix64(h ^ (a + 0x8CB92BA72F3D8DD7ull));
    h = gen_mix64(h ^ (b * 0x9E3779B97F4A7C15ull + 0x165667B19E3779F9ull));
    return h;
}

/* uniform in (0,1), exact in fp64 */
GEN_FN double gen_u01(uint64_t h)
{
    return ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

/* Irwin–Hall(4) of 16-bit uniforms, centred: integer in [−131070, 131070] */
GEN_FN int32_t gen_ih4(uint64_t h)
{
    return (int32_t)((h & 0xffffu) + ((h >> 16) & 0xffffu) + ((h >> 32) & 0xffffu) + (h >> 48)) - 131070;
}

/* better(a, b): a ranks before b under (score desc, index asc) */
GEN_FN int gen_better(double sa, int ia, double sb, int ib)
{
    return sa > sb || (sa == sb && ia < ib);
}

/* Child distribution of one expanded drafter node: q_out[0..topk) sorted
 * descending.  key identifies the expanded node inside its tree. */
GEN_FN void gen_child_probs(uint64_t seed, uint64_t tree_id, uint64_t key, int topk, int m,
                            float *q_out)
{
    double w[GEN_MAX_TOPK + 1];
    double sum = 0.0;
    for (int j = 0; j <= topk; j++) {
        double u = gen_u01(gen_hash(seed, GEN_S_CHILD, tree_id, key * 32u + (uint64_t)j));
        double p = u;
        for (int t = 1; t < m; t++) p = GEN_DMUL(p, u);
        w[j] = p;
        sum = GEN_DADD(sum, p);
    }
    /* sort the first topk weights descending (insertion sort); w[topk] = rest */
    for (int i = 1; i < topk; i++) {
        double v = w[i];
        int j = i - 1;
        while (j >= 0 && w[j] < v) {
            w[j + 1] = w[j];
            j--;
        }
        w[j + 1] = v;
    }
    for (int j = 0; j < topk; j++) q_out[j] = GEN_D2F(GEN_DDIV(w[j], sum));
}

/* One EAGLE-style draft tree.  Writes parent[0..N), q[0..N) (pads: parent
 * −1, q 0) and returns the node count n ≤ N.  Scratch arrays live in the
 * caller (host: stack; device: local memory). */
typedef struct {
    int32_t par[GEN_MAX_POOL];  /* candidate parent (candidate index, −1 = root) */
    float q[GEN_MAX_POOL];
    double sc[GEN_MAX_POOL];    /* drafter's cumulative probability */
    int32_t map[GEN_MAX_POOL];  /* candidate → node id, −1 if pruned */
    uint8_t used[GEN_MAX_POOL];
} gen_tree_scratch;

GEN_FN int gen_tree(uint64_t seed, uint64_t tree_id, int steps, int topk, int N, int m_lo,
                    int m_hi, int32_t *parent, float *q, gen_tree_scratch *s)
{
    int m = m_lo + (int)(gen_hash(seed, GEN_S_DIFF, tree_id, 0) % (uint64_t)(m_hi - m_lo + 1));
    float cq[GEN_MAX_TOPK];
    int frontier[GEN_MAX_TOPK];
    int nf = 0, P = 0;

    /* step 1: the root's children */
    gen_child_probs(seed, tree_id, 0, topk, m, cq);
    for (int j = 0; j < topk; j++) {
        s->par[P] = -1;
        s->q[P] = cq[j];
        s->sc[P] = (double)cq[j];
        frontier[nf++] = P;
        P++;
    }
    /* steps 2..steps: expand the frontier, keep the best topk as the next frontier */
    for (int st = 2; st <= steps; st++) {
        int lo = P;
        for (int f = 0; f < nf; f++) {
            int c = frontier[f];
            gen_child_probs(seed, tree_id, (uint64_t)c + 1u, topk, m, cq);
            for (int j = 0; j < topk; j++) {
                s->par[P] = c;
                s->q[P] = cq[j];
                s->sc[P] = GEN_DMUL(s->sc[c], (double)cq[j]);
                P++;
            }
        }
        for (int i = lo; i < P; i++) s->used[i] = 0;
        nf = 0;
        for (int t = 0; t < topk; t++) {
            int best = -1;
            for (int i = lo; i < P; i++)
                if (!s->used[i] && (best < 0 || gen_better(s->sc[i], i, s->sc[best], best))) best = i;
            s->used[best] = 1;
            frontier[nf++] = best;
        }
    }
    /* prune the pool to the best N−1 candidates (ancestors rank first) */
    int keep = N - 1 < P ? N - 1 : P;
    for (int i = 0; i < P; i++) { s->used[i] = 0; s->map[i] = -1; }
    for (int t = 0; t < keep; t++) {
        int best = -1;
        for (int i = 0; i < P; i++)
            if (!s->used[i] && (best < 0 || gen_better(s->sc[i], i, s->sc[best], best))) best = i;
        s->used[best] = 1;
    }
    /* renumber in creation order: root = 0, kept candidates 1.. */
    int n = 1;
    parent[0] = -1;
    q[0] = 1.0f;
    for (int i = 0; i < P; i++) {
        if (!s->used[i]) continue;
        s->map[i] = n;
        parent[n] = s->par[i] < 0 ? 0 : s->map[s->par[i]];
        q[n] = s->q[i];
        n++;
    }
    for (int i = n; i < N; i++) { parent[i] = -1; q[i] = 0.0f; }
    return n;
}

/* Routing top-K of node v of tree tree_id at layer l.  ids_out[0..K). */
GEN_FN void gen_route(uint64_t seed, uint64_t tree_id, int v, int l, int E, int K, int sigma_q4,
                      int32_t *ids_out)
{
    int32_t best_l[GEN_MAX_K];
    int32_t best_e[GEN_MAX_K];
    int cnt = 0;
    uint64_t hz = gen_hash(seed, GEN_S_RZ, tree_id, (uint64_t)l);
    uint64_t he = gen_hash(seed, GEN_S_REPS, tree_id, (uint64_t)v * 4096u + (uint64_t)l);
    for (int e = 0; e < E; e++) {
        int32_t z = gen_ih4(gen_mix64(hz + (uint64_t)e * 0x9E3779B97F4A7C15ull));
        int32_t ep = gen_ih4(gen_mix64(he + (uint64_t)e * 0x9E3779B97F4A7C15ull));
        int32_t lg = sigma_q4 * z + 4 * ep;
        /* insert (lg, e) into the descending list; later e loses ties */
        if (cnt == K && lg <= best_l[K - 1]) continue;
        int j = cnt < K ? cnt : K - 1;
        while (j > 0 && best_l[j - 1] < lg) {
            best_l[j] = best_l[j - 1];
            best_e[j] = best_e[j - 1];
            j--;
        }
        best_l[j] = lg;
        best_e[j] = e;
        if (cnt < K) cnt++;
    }
    for (int j = 0; j < K; j++) ids_out[j] = best_e[j];
}

/* bf16 bits of an element of the hidden states (stream GEN_S_HID) or of the
 * router weights (GEN_S_WG).  mode 0: integer in [−2, 2]; mode 1: approx
 * normal N(0, scale²) with scale given as a power of two exponent. */
GEN_FN uint16_t gen_bf16_value(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b, int mode,
                               int scale_log2)
{
    uint64_t h = gen_hash(seed, stream, a, b);
    if (mode == 0) {
        int v = (int)(h % 5u) - 2;
        /* exact bf16 encodings of −2..2 */
        switch (v) {
        case -2: return 0xC000u;
        case -1: return 0xBF80u;
        case 0: return 0x0000u;
        case 1: return 0x3F80u;
        default: return 0x4000u;
        }
    }
    /* IH4 / 37837 ≈ N(0,1); scale by 2^scale_log2 (exact), round to bf16 */
    double x = GEN_DDIV((double)gen_ih4(h), 37837.0);
    double sc = 1.0;
    if (scale_log2 >= 0)
        for (int t = 0; t < scale_log2; t++) sc = GEN_DMUL(sc, 2.0);
    else
        for (int t = 0; t < -scale_log2; t++) sc = GEN_DMUL(sc, 0.5);
    float f = GEN_D2F(GEN_DMUL(x, sc));
    union { float f; uint32_t u; } cv;
    cv.f = f;
    uint32_t u = cv.u;
    uint32_t r = u + 0x7FFFu + ((u >> 16) & 1u); /* round to nearest even */
    return (uint16_t)(r >> 16);
}

#endif /* EVICT_GEN_H */
