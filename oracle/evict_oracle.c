/*
 * evict_oracle.c — plain, slow CPU oracle for the EVICT hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path under
 * paper_2605_00342_b200/ and includes nothing from it.
 *
 * Every function follows PAPER.md (arxiv 2605.00342, "EVICT") step by step,
 * one tree at a time, with no blocking, fusion or reordering.  Readings of
 * points where the paper is silent are the "Z" readings of DESIGN.md §3
 * (they are SURVEY.md §8(c)'s ambiguity register).
 *
 * Precision (Z6): node scores are fp32 products in root→leaf
 * order, because the score *decides an integer* (the ranking) and such a
 * decision is taken in the kernel's precision on both sides.  Everything
 * that is a value (prefix sums, ratios, router logits) is fp64.
 *
 * Parity pins (tests/test_oracle_pins.py): brute force over every
 * ancestor-closed subset, chain closed form, the worked toy tree, SPEC
 * examples, invariants.  No function here is "parity unpinned".
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -shared -fPIC
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_TREE_BAD_SIZE   0x01u
#define ORACLE_TREE_BAD_PARENT 0x02u
#define ORACLE_TREE_BAD_PROB   0x04u
#define ORACLE_TREE_BAD_COST   0x08u
#define ORACLE_TREE_BAD_EXPERT 0x10u
#define ORACLE_TREE_BAD_KEEP   0x20u

#define ORACLE_MAX_NODES 128
#define ORACLE_TIE_REL 1e-5

int oracle_abi_version(void) { return 1; }

/* ------------------------------------------------------------------ */
/* A1: validation.  PAPER.md:48 (a tree rooted at x_{t+1}); the
 * topological numbering parent[i] < i is reading Z4; q ∈ [0,1] is Z9;
 * cost domain (0, +inf], cost[0] finite, is Z10.                       */
static uint32_t validate_tree(int n, int max_nodes, const int32_t *parent,
                              const float *q)
{
    uint32_t st = 0;
    if (n < 1 || n > max_nodes || n > ORACLE_MAX_NODES) return ORACLE_TREE_BAD_SIZE;
    if (parent[0] != -1) st |= ORACLE_TREE_BAD_PARENT;
    for (int i = 1; i < n; i++) {
        if (parent[i] < 0 || parent[i] >= i) st |= ORACLE_TREE_BAD_PARENT;
        float qi = q[i];
        if (isnan(qi) || qi < 0.0f || qi > 1.0f) st |= ORACLE_TREE_BAD_PROB;
    }
    return st;
}

static uint32_t validate_cost(int n, const float *cost)
{
    uint32_t st = 0;
    for (int k = 1; k <= n; k++) {
        float c = cost[k - 1];
        if (isnan(c) || c <= 0.0f) st |= ORACLE_TREE_BAD_COST;
    }
    if (isinf(cost[0])) st |= ORACLE_TREE_BAD_COST;
    return st;
}

/* ------------------------------------------------------------------ */
/* A2: Score(v) = Π_{u ∈ Path(x_{t+1}, v)} q(u)   (Eq. 7)
 * Score(root) = 1 (reading Z1), computed root → leaf, one fp32 rounding
 * per edge: score[i] = fl32(score[parent[i]] · q[i]).  -0.0 → +0.0 (Z9).
 * depth(v) = |Path| − 1.                                               */
static void path_scores(int n, const int32_t *parent, const float *q,
                        float *score, int32_t *depth)
{
    score[0] = 1.0f;
    depth[0] = 0;
    for (int i = 1; i < n; i++) {
        float qi = q[i];
        if (qi == 0.0f) qi = 0.0f;          /* canonicalise -0.0 */
        float s = score[parent[i]] * qi;   /* parent < i: already final */
        if (s == 0.0f) s = 0.0f;
        score[i] = s;
        depth[i] = depth[parent[i]] + 1;
    }
}

/* A3: ranking by (score desc, node index asc) — the top-k-by-cumulative-
 * score prune of PAPER.md:133–135 (§3.2.1); tie rule is reading Z4.
 * Plain stable insertion sort of indices.                              */
static void rank_nodes(int n, const float *score, int32_t *order)
{
    for (int i = 0; i < n; i++) order[i] = i;
    for (int i = 1; i < n; i++) {
        int32_t v = order[i];
        int j = i - 1;
        while (j >= 0 && score[order[j]] < score[v]) {   /* strict: stable */
            order[j + 1] = order[j];
            j--;
        }
        order[j + 1] = v;
    }
}

/* ------------------------------------------------------------------ */
/* oracle_select_tree: A1–A5 for one tree.
 *   A4: S[k] = Σ_{j<k} Score(order[j]) = Ê[A(T_k)]      (Eq. 8, §3.2.3)
 *   A5: R[k] = S[k] / C(k); k* = argmax_{1≤k≤n} R[k], smallest k on ties
 *       (Eq. 10; tie rule Z3; domain 1..n is Z2)
 *       e_hat = S[k*], utility = R[k*] (C_AR dropped, Z18),
 *       keep = order[0..k*).
 *   Near-tie set (north_star): tie_bits bit (k-1) set iff
 *       R[k] ≥ R[k*]·(1 − 1e-5).
 * Arrays S, R, score, depth, order have room for n entries; keep_bits and
 * tie_bits have W = ceil(max_nodes/64) words.  On a data error every output
 * is written in its defined error state (k*=0, keep=0, S=R=0).          */
/* Selection policies (the cut k* on the same ranking and prefix sums):
 *   ORACLE_POLICY_COST     k* = smallest argmax S[k]/C(k) (Eq. 10, EVICT)
 *   ORACLE_POLICY_COVERAGE k* = smallest k with S_k/S_K ≥ ρ, K = n_b: the
 *                          score-coverage ablation (PAPER.md:290-291,
 *                          §5.4 "Ablating Cost-Aware Selection"); ρ = 1 is
 *                          EAGLE-3 (every node under the budget is verified,
 *                          PAPER.md:292).  If no k qualifies (ρ > 1), k* = n.
 *                          Near ties: k with |S_k/S_K − ρ| ≤ 1e-5·ρ, and the
 *                          k after each (a GPU on the other side of ρ).
 *   ORACLE_POLICY_FIXED    k* = min(k_fixed, n_b): a fixed verify budget on
 *                          the same ranking.
 * e_hat = S[k*] and utility = S[k*]/C(k*) for every policy.             */
#define ORACLE_POLICY_COST 0
#define ORACLE_POLICY_COVERAGE 1
#define ORACLE_POLICY_FIXED 2

uint32_t oracle_select_tree_policy(int n, int max_nodes, const int32_t *parent,
                                   const float *q, const float *cost,
                                   int policy, double rho, int k_fixed,
                                   float *score, int32_t *depth, int32_t *order,
                                   double *S, double *R, int32_t *k_star,
                                   double *e_hat, double *utility,
                                   uint64_t *keep_bits, uint64_t *tie_bits, int W);

uint32_t oracle_select_tree(int n, int max_nodes, const int32_t *parent,
                            const float *q, const float *cost,
                            float *score, int32_t *depth, int32_t *order,
                            double *S, double *R, int32_t *k_star,
                            double *e_hat, double *utility,
                            uint64_t *keep_bits, uint64_t *tie_bits, int W)
{
    return oracle_select_tree_policy(n, max_nodes, parent, q, cost, ORACLE_POLICY_COST, 0.0, 0,
                                     score, depth, order, S, R, k_star, e_hat, utility,
                                     keep_bits, tie_bits, W);
}

uint32_t oracle_select_tree_policy(int n, int max_nodes, const int32_t *parent,
                                   const float *q, const float *cost,
                                   int policy, double rho, int k_fixed,
                                   float *score, int32_t *depth, int32_t *order,
                                   double *S, double *R, int32_t *k_star,
                                   double *e_hat, double *utility,
                                   uint64_t *keep_bits, uint64_t *tie_bits, int W)
{
    for (int w = 0; w < W; w++) { keep_bits[w] = 0; tie_bits[w] = 0; }
    *k_star = 0; *e_hat = 0.0; *utility = 0.0;
    uint32_t st = validate_tree(n, max_nodes, parent, q);
    if (st & ORACLE_TREE_BAD_SIZE) return st;
    st |= validate_cost(n, cost);
    if (st) {
        for (int i = 0; i < n; i++) {
            score[i] = 0.0f; depth[i] = -1; order[i] = -1; S[i] = 0.0; R[i] = 0.0;
        }
        return st;
    }

    path_scores(n, parent, q, score, depth);
    rank_nodes(n, score, order);

    double acc = 0.0;
    for (int k = 1; k <= n; k++) {
        acc += (double)score[order[k - 1]];
        S[k - 1] = acc;
        R[k - 1] = S[k - 1] / (double)cost[k - 1];   /* +inf cost ⇒ R = 0 */
    }
    int kbest = 1;
    if (policy == ORACLE_POLICY_COVERAGE) {
        double SK = S[n - 1];
        kbest = n;
        for (int k = 1; k <= n; k++)
            if (S[k - 1] / SK >= rho) { kbest = k; break; }
    } else if (policy == ORACLE_POLICY_FIXED) {
        kbest = k_fixed < n ? k_fixed : n;
    } else {
        for (int k = 2; k <= n; k++)
            if (R[k - 1] > R[kbest - 1]) kbest = k;      /* strict: smallest k */
    }

    *k_star = kbest;
    *e_hat = S[kbest - 1];
    *utility = R[kbest - 1];
    for (int j = 0; j < kbest; j++) {
        int v = order[j];
        keep_bits[v / 64] |= (uint64_t)1 << (v % 64);
    }
    if (policy == ORACLE_POLICY_COVERAGE) {
        double SK = S[n - 1];
        tie_bits[(kbest - 1) / 64] |= (uint64_t)1 << ((kbest - 1) % 64);
        for (int k = 1; k <= n; k++) {
            if (fabs(S[k - 1] / SK - rho) <= ORACLE_TIE_REL * rho) {
                tie_bits[(k - 1) / 64] |= (uint64_t)1 << ((k - 1) % 64);
                if (k < n) tie_bits[k / 64] |= (uint64_t)1 << (k % 64);
            }
        }
    } else if (policy == ORACLE_POLICY_FIXED) {
        tie_bits[(kbest - 1) / 64] |= (uint64_t)1 << ((kbest - 1) % 64);
    } else {
        double band = R[kbest - 1] * (1.0 - ORACLE_TIE_REL);
        for (int k = 1; k <= n; k++)
            if (R[k - 1] >= band) tie_bits[(k - 1) / 64] |= (uint64_t)1 << ((k - 1) % 64);
    }
    return 0;
}

/* Batched wrapper: trees [b_begin, b_end) of a [B][N] batch.
 * cost_stride 0 ⇒ one shared table.  Per-tree arrays are [B][N].       */
void oracle_select_batch_policy(int b_begin, int b_end, int N, const int32_t *n_nodes,
                                const int32_t *parent, const float *q,
                                const float *cost, int cost_stride,
                                int policy, double rho, int k_fixed,
                                float *score, int32_t *depth, int32_t *order,
                                double *S, double *R, int32_t *k_star, double *e_hat,
                                double *utility, uint64_t *keep_bits,
                                uint64_t *tie_bits, uint32_t *status);

void oracle_select_batch(int b_begin, int b_end, int N, const int32_t *n_nodes,
                         const int32_t *parent, const float *q,
                         const float *cost, int cost_stride,
                         float *score, int32_t *depth, int32_t *order,
                         double *S, double *R, int32_t *k_star, double *e_hat,
                         double *utility, uint64_t *keep_bits,
                         uint64_t *tie_bits, uint32_t *status)
{
    oracle_select_batch_policy(b_begin, b_end, N, n_nodes, parent, q, cost, cost_stride,
                               ORACLE_POLICY_COST, 0.0, 0, score, depth, order, S, R, k_star,
                               e_hat, utility, keep_bits, tie_bits, status);
}

void oracle_select_batch_policy(int b_begin, int b_end, int N, const int32_t *n_nodes,
                                const int32_t *parent, const float *q,
                                const float *cost, int cost_stride,
                                int policy, double rho, int k_fixed,
                                float *score, int32_t *depth, int32_t *order,
                                double *S, double *R, int32_t *k_star, double *e_hat,
                                double *utility, uint64_t *keep_bits,
                                uint64_t *tie_bits, uint32_t *status)
{
    int W = (N + 63) / 64;
    for (int b = b_begin; b < b_end; b++) {
        int n = n_nodes ? n_nodes[b] : N;
        size_t o = (size_t)b * N;
        /* pads: defined values past n */
        for (int i = 0; i < N; i++) {
            score[o + i] = 0.0f; depth[o + i] = -1; order[o + i] = -1;
            S[o + i] = 0.0; R[o + i] = 0.0;
        }
        status[b] = oracle_select_tree_policy(n, N, parent + o, q + o,
                                       cost + (size_t)b * cost_stride, policy, rho, k_fixed,
                                       score + o, depth + o, order + o, S + o,
                                       R + o, &k_star[b], &e_hat[b],
                                       &utility[b], keep_bits + (size_t)b * W,
                                       tie_bits + (size_t)b * W, W);
    }
}

/* ------------------------------------------------------------------ */
/* A6: verify-tree compaction for one tree and one kept set
 * (PAPER.md:48, 92 — Fig. 4(c) tree attention mask; layout is reading
 * Z12).  Slots follow ascending node index among kept nodes.
 *   kept_index[s]   = node of slot s
 *   positions[s]    = pos_offset + depth(node)
 *   tree_mask[s][w] = bit j ⇔ slot j is an ancestor-or-self of slot s
 *   next_token[s]   = smallest slot among kept children, −1 if none
 *   next_sibling[s] = smallest slot > s with the same parent, −1 if none
 * Returns status (BAD_KEEP if the set does not contain the root or is
 * not ancestor-closed); writes k through *k_out (0 on error).           */
uint32_t oracle_build_tree(int n, int max_nodes, const int32_t *parent,
                           const uint64_t *keep_bits, int32_t pos_offset,
                           int32_t *kept_index, int32_t *positions,
                           int32_t *next_token, int32_t *next_sibling,
                           uint64_t *tree_mask, int32_t *k_out)
{
    int W = (max_nodes + 63) / 64;
    int32_t depth[ORACLE_MAX_NODES];
    int32_t slot_of[ORACLE_MAX_NODES];
    int32_t kept[ORACLE_MAX_NODES];
    *k_out = 0;
    uint32_t st = 0;
    if (n < 1 || n > max_nodes || n > ORACLE_MAX_NODES) return ORACLE_TREE_BAD_SIZE;
    if (parent[0] != -1) st |= ORACLE_TREE_BAD_PARENT;
    for (int i = 1; i < n; i++)
        if (parent[i] < 0 || parent[i] >= i) st |= ORACLE_TREE_BAD_PARENT;
    for (int i = 0; i < max_nodes; i++) {
        int bit = (int)((keep_bits[i / 64] >> (i % 64)) & 1u);
        if (i >= n && bit) st |= ORACLE_TREE_BAD_KEEP;     /* kept pad */
        if (i < n) kept[i] = bit;
    }
    if (st) return st;
    if (!kept[0]) return ORACLE_TREE_BAD_KEEP;
    for (int i = 1; i < n; i++)
        if (kept[i] && !kept[parent[i]]) return ORACLE_TREE_BAD_KEEP;

    depth[0] = 0;
    for (int i = 1; i < n; i++) depth[i] = depth[parent[i]] + 1;

    int k = 0;
    for (int i = 0; i < n; i++) slot_of[i] = kept[i] ? k++ : -1;

    for (int i = 0; i < n; i++) {
        if (!kept[i]) continue;
        int s = slot_of[i];
        kept_index[s] = i;
        positions[s] = pos_offset + depth[i];
        for (int w = 0; w < W; w++) tree_mask[(size_t)s * W + w] = 0;
        /* walk the ancestor chain, including self */
        for (int a = i; a != -1; a = parent[a]) {
            int sa = slot_of[a];
            tree_mask[(size_t)s * W + sa / 64] |= (uint64_t)1 << (sa % 64);
        }
        next_token[s] = -1;
        for (int c = i + 1; c < n; c++)
            if (kept[c] && parent[c] == i) { next_token[s] = slot_of[c]; break; }
        next_sibling[s] = -1;
        if (i > 0)
            for (int c = i + 1; c < n; c++)
                if (kept[c] && parent[c] == parent[i]) { next_sibling[s] = slot_of[c]; break; }
    }
    *k_out = k;
    return 0;
}

/* Batched A6 with the packed verify layout: tree b's k_b rows occupy
 * packed rows [off_b, off_b + k_b), off = exclusive scan of k over the
 * batch in tree order; verify_offsets[B] = total rows.
 * retrieve_index[r] = b·N + kept_index[r] (flat index into [B][N] draft
 * arrays; reading Z12).  Trees with a bad status contribute 0 rows.     */
void oracle_build_batch(int B, int N, const int32_t *n_nodes,
                        const int32_t *parent, const uint64_t *keep_bits,
                        const int32_t *pos_offset, int32_t *verify_offsets,
                        int32_t *kept_index, int32_t *retrieve_index,
                        int32_t *positions, int32_t *next_token,
                        int32_t *next_sibling, uint64_t *tree_mask,
                        uint32_t *status)
{
    int W = (N + 63) / 64;
    int32_t off = 0;
    for (int b = 0; b < B; b++) {
        int n = n_nodes ? n_nodes[b] : N;
        int32_t k = 0;
        verify_offsets[b] = off;
        status[b] = oracle_build_tree(n, N, parent + (size_t)b * N,
                                      keep_bits + (size_t)b * W,
                                      pos_offset ? pos_offset[b] : 0,
                                      kept_index + off, positions + off,
                                      next_token + off, next_sibling + off,
                                      tree_mask + (size_t)off * W, &k);
        for (int s = 0; s < k; s++)
            retrieve_index[off + s] = b * N + kept_index[off + s];
        off += k;
    }
    verify_offsets[B] = off;
}

/* ------------------------------------------------------------------ */
/* A7: per-layer expert union over the kept nodes (Eq. 5)
 *   E_l(H) = ∪_{v kept} E_l(h_v);  count[l] = |E_l(H)|; total = Σ_l count.
 * Scope per tree, root included (Z13); duplicate ids are idempotent (Z16).
 * ids: node-major [N][L][K] of id_bytes ∈ {1, 4} (u8 or i32) for one tree.
 * bits: [L][EW] u64 with EW = ceil(E/64).  On an id ≥ E (or < 0) every
 * output of the tree is zero and BAD_EXPERT is returned.                */
uint32_t oracle_union_tree(int n, const uint64_t *keep_bits, const void *ids,
                           int id_bytes, int L, int K, int E,
                           int32_t *count, int32_t *total, uint64_t *bits)
{
    int EW = (E + 63) / 64;
    unsigned char seen[256];
    uint32_t st = 0;
    *total = 0;
    for (int l = 0; l < L; l++) {
        memset(seen, 0, sizeof(seen));
        for (int v = 0; v < n; v++) {
            if (!((keep_bits[v / 64] >> (v % 64)) & 1u)) continue;
            for (int j = 0; j < K; j++) {
                size_t idx = ((size_t)v * L + l) * K + j;
                long e = id_bytes == 1 ? (long)((const uint8_t *)ids)[idx]
                                       : (long)((const int32_t *)ids)[idx];
                if (e < 0 || e >= E) { st |= ORACLE_TREE_BAD_EXPERT; continue; }
                seen[e] = 1;
            }
        }
        int c = 0;
        for (int w = 0; w < EW; w++) bits[(size_t)l * EW + w] = 0;
        for (int e = 0; e < E; e++) {
            if (seen[e]) {
                c++;
                bits[(size_t)l * EW + e / 64] |= (uint64_t)1 << (e % 64);
            }
        }
        count[l] = c;
        *total += c;
    }
    if (st) {
        for (int l = 0; l < L; l++) {
            count[l] = 0;
            for (int w = 0; w < EW; w++) bits[(size_t)l * EW + w] = 0;
        }
        *total = 0;
    }
    return st;
}

/* Batched A7 over trees [b_begin, b_end); ids are [B][N][L][K].          */
void oracle_union_batch(int b_begin, int b_end, int N, const int32_t *n_nodes,
                        const uint64_t *keep_bits, const void *ids,
                        int id_bytes, int L, int K, int E, int32_t *count,
                        int32_t *total, uint64_t *bits, uint32_t *status)
{
    int W = (N + 63) / 64, EW = (E + 63) / 64;
    size_t row = (size_t)L * K * id_bytes;
    for (int b = b_begin; b < b_end; b++) {
        int n = n_nodes ? n_nodes[b] : N;
        status[b] = oracle_union_tree(n, keep_bits + (size_t)b * W,
                                      (const char *)ids + (size_t)b * N * row,
                                      id_bytes, L, K, E,
                                      count + (size_t)b * L, &total[b],
                                      bits + (size_t)b * L * EW);
    }
}

/* ------------------------------------------------------------------ */
/* NEXT-1: the prefix-union curve along the ranking and the offline cost
 * profile built from it (Fig. 1 —
 * activated experts grow with the number of verified tokens
 * — C(k) is profiled offline per k).
 *   curve[k-1]          = Σ_l |∪_{j<k} E_l(order[j])|           (k = 1..n)
 *   curve_layer[k-1][l] = |∪_{j<k} E_l(order[j])|
 * order = the ranking (evict_select's order row); every order[j] must be a
 * node < n (else BAD_KEEP); ids ≥ E give BAD_EXPERT.  On error the tree's
 * curve rows are 0.  Entries past n are 0.                              */
uint32_t oracle_union_curve_tree(int n, const int32_t *order, const void *ids, int id_bytes,
                                 int L, int K, int E, int32_t *curve, int32_t *curve_layer)
{
    unsigned char seen[128][256];
    uint32_t st = 0;
    if (L > 128) return ORACLE_TREE_BAD_SIZE;
    memset(seen, 0, sizeof(seen));
    int32_t tot = 0;
    int32_t per[128];
    for (int l = 0; l < L; l++) per[l] = 0;
    for (int k = 1; k <= n; k++) {
        int v = order[k - 1];
        if (v < 0 || v >= n) { st |= ORACLE_TREE_BAD_KEEP; break; }
        for (int l = 0; l < L; l++) {
            for (int j = 0; j < K; j++) {
                size_t idx = ((size_t)v * L + l) * K + j;
                long e = id_bytes == 1 ? (long)((const uint8_t *)ids)[idx]
                                       : (long)((const int32_t *)ids)[idx];
                if (e < 0 || e >= E) { st |= ORACLE_TREE_BAD_EXPERT; continue; }
                if (!seen[l][e]) { seen[l][e] = 1; per[l]++; tot++; }
            }
            if (curve_layer) curve_layer[(size_t)(k - 1) * L + l] = per[l];
        }
        curve[k - 1] = tot;
    }
    if (st) {
        for (int k = 1; k <= n; k++) {
            curve[k - 1] = 0;
            if (curve_layer)
                for (int l = 0; l < L; l++) curve_layer[(size_t)(k - 1) * L + l] = 0;
        }
    }
    return st;
}

void oracle_union_curve_batch(int b_begin, int b_end, int N, const int32_t *n_nodes,
                              const int32_t *order, const void *ids, int id_bytes, int L, int K,
                              int E, int32_t *curve, int32_t *curve_layer, uint32_t *status)
{
    for (int b = b_begin; b < b_end; b++) {
        int n = n_nodes ? n_nodes[b] : N;
        for (int i = 0; i < N; i++) {
            curve[(size_t)b * N + i] = 0;
            if (curve_layer)
                for (int l = 0; l < L; l++) curve_layer[((size_t)b * N + i) * L + l] = 0;
        }
        if (n < 1 || n > N) { status[b] = ORACLE_TREE_BAD_SIZE; continue; }
        const void *tids = (const uint8_t *)ids + (size_t)b * N * L * K * id_bytes;
        status[b] = oracle_union_curve_tree(n, order + (size_t)b * N, tids, id_bytes, L, K, E,
                                            curve + (size_t)b * N,
                                            curve_layer ? curve_layer + (size_t)b * N * L : NULL);
    }
}

/* Offline cost profile from the curves (reading R2 of DESIGN.md §3 with the
 * analytic Ū(k) = E(1 − (1 − K/E)^k) replaced by the measured mean):
 *   Ū(k) = Σ_{b: n_b ≥ k, status_b = 0} curve_b[k-1] / (L · #{those b})
 *   C(k) = c0 + c_union·Ū(k) + c_tok·k;  C(k) = +inf when no tree has k nodes.
 * fp64 here.                                                            */
void oracle_profile_cost(int B, int N, int L, const int32_t *n_nodes, const int32_t *curve,
                         const uint32_t *status, double c0, double c_union, double c_tok,
                         double *cost)
{
    for (int k = 1; k <= N; k++) {
        double sum = 0.0;
        long cnt = 0;
        for (int b = 0; b < B; b++) {
            int n = n_nodes ? n_nodes[b] : N;
            if ((status && status[b]) || n < k) continue;
            sum += (double)curve[(size_t)b * N + k - 1];
            cnt++;
        }
        cost[k - 1] = cnt ? c0 + c_union * (sum / ((double)L * (double)cnt)) + c_tok * (double)k
                          : INFINITY;
    }
}

/* ------------------------------------------------------------------ */
/* A8: router TopK (Eq. 4): E(h) = TopK(W_g h, K) on raw
 * logits (Z14), ties by expert index ascending; fp64 dot products (Z15).
 * h: d bf16 values (raw uint16 bits); Wg: [E][d] bf16.  ids_out[K] in
 * rank order.  near_tie = 1 when the K-th and (K+1)-th logits are closer
 * than the fp32-accumulation error bound d·2^-24·Σ|h_i w_i| of either.  */
static double bf16_to_double(uint16_t b)
{
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, sizeof(f));
    return (double)f;
}

int oracle_router_topk(int d, const uint16_t *h, const uint16_t *Wg, int E,
                       int K, int32_t *ids_out, double *logits_out)
{
    double logit[256], mag[256];
    int used[256];
    for (int e = 0; e < E; e++) {
        double acc = 0.0, m = 0.0;
        for (int i = 0; i < d; i++) {
            double p = bf16_to_double(h[i]) * bf16_to_double(Wg[(size_t)e * d + i]);
            acc += p;
            m += fabs(p);
        }
        logit[e] = acc;
        mag[e] = m;
        used[e] = 0;
        if (logits_out) logits_out[e] = acc;
    }
    int last = -1;
    for (int j = 0; j < K; j++) {               /* repeated selection */
        int best = -1;
        for (int e = 0; e < E; e++)
            if (!used[e] && (best < 0 || logit[e] > logit[best])) best = e;
        used[best] = 1;
        ids_out[j] = best;
        last = best;
    }
    int near_tie = 0;
    if (K < E) {
        int nxt = -1;
        for (int e = 0; e < E; e++)
            if (!used[e] && (nxt < 0 || logit[e] > logit[nxt])) nxt = e;
        double bound = (double)d * ldexp(1.0, -24) * (mag[last] > mag[nxt] ? mag[last] : mag[nxt]);
        if (logit[last] - logit[nxt] <= bound) near_tie = 1;
    }
    return near_tie;
}

/* Router-mode union for trees [b_begin, b_end): hidden h is [L][B·N][d]
 * (bf16 bits), Wg is [L][E][d].  Produces the same outputs as A7 plus
 * near_tie[b·L + l] = number of kept rows of layer l whose top-K boundary
 * is a near-tie (those rows are excluded from parity, SURVEY §8(c) rule 4). */
void oracle_router_union_batch(int b_begin, int b_end, int B, int N,
                               const int32_t *n_nodes, const uint64_t *keep_bits,
                               int L, int E, int K, int d, const uint16_t *h,
                               const uint16_t *Wg, int32_t *count,
                               int32_t *total, uint64_t *bits,
                               int32_t *near_tie)
{
    int W = (N + 63) / 64, EW = (E + 63) / 64;
    int32_t ids[256];
    unsigned char seen[256];
    for (int b = b_begin; b < b_end; b++) {
        int n = n_nodes ? n_nodes[b] : N;
        total[b] = 0;
        for (int l = 0; l < L; l++) {
            memset(seen, 0, sizeof(seen));
            int nt = 0;
            for (int v = 0; v < n; v++) {
                if (!((keep_bits[(size_t)b * W + v / 64] >> (v % 64)) & 1u)) continue;
                const uint16_t *hv = h + ((size_t)l * B * N + (size_t)b * N + v) * d;
                nt += oracle_router_topk(d, hv, Wg + (size_t)l * E * d, E, K, ids, NULL);
                for (int j = 0; j < K; j++) seen[ids[j]] = 1;
            }
            int c = 0;
            uint64_t *bl = bits + ((size_t)b * L + l) * EW;
            for (int w = 0; w < EW; w++) bl[w] = 0;
            for (int e = 0; e < E; e++)
                if (seen[e]) { c++; bl[e / 64] |= (uint64_t)1 << (e % 64); }
            count[(size_t)b * L + l] = c;
            near_tie[(size_t)b * L + l] = nt;
            total[b] += c;
        }
    }
}

/* ------------------------------------------------------------------ */
/* A9: batch statistics (north_star: "all-reduce aggregate statistics";
 * metrics of PAPER.md:212, 217–219).  Layout of the int64 vector
 * (shared by contract with include/evict.h, restated, not included):
 *   [0] trees  [1] Σk*  [2] Σn  [3] Σunion_total  [4] trees with status≠0
 *   [5 .. 5+N]           k* histogram, bins 0..N
 *   [6+N .. 6+N+L)       Σ union_count per layer
 * dstats[0] = Σ e_hat, dstats[1] = Σ utility (fp64, good trees only).  */
void oracle_batch_stats(int B, int N, int L, const int32_t *n_nodes,
                        const int32_t *k_star, const double *e_hat,
                        const double *utility, const int32_t *union_count,
                        const uint32_t *status, int64_t *stats, double *dstats)
{
    int len = 6 + N + L;
    for (int i = 0; i < len; i++) stats[i] = 0;
    dstats[0] = dstats[1] = 0.0;
    for (int b = 0; b < B; b++) {
        stats[0] += 1;
        if (status[b]) { stats[4] += 1; stats[5 + 0] += 1; continue; }
        int n = n_nodes ? n_nodes[b] : N;
        stats[1] += k_star[b];
        stats[2] += n;
        stats[5 + k_star[b]] += 1;
        for (int l = 0; l < L; l++) {
            stats[3] += union_count[(size_t)b * L + l];
            stats[6 + N + l] += union_count[(size_t)b * L + l];
        }
        dstats[0] += e_hat[b];
        dstats[1] += utility[b];
    }
}
