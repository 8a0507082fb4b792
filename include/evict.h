/*
 * evict.h — C ABI of the B200-native EVICT hot path (libevict.so).
 *
 * EVICT (arxiv 2605.00342, PAPER.md) truncates an EAGLE-style draft tree to
 * its most cost-effective ancestor-closed prefix before MoE verification.
 * Given a batch of draft trees (parent pointers + drafter probabilities q)
 * and the offline-profiled cost table C(k), the calls below compute
 *   evict_select            — Score(v) (Eq. 7), the ancestor-closed ranking
 *                             (§3.2.1), Ê[A(T_k)] prefix sums (Eq. 8) and
 *                             k* = argmax_k Ê[A(T_k)]/C(k) (Eq. 10, §3.2.3)
 *   evict_build_verify_tree — the kept tree T_{k*} compacted into the verify
 *                             batch: tree-attention mask, positions, retrieve
 *                             indices, next-token/next-sibling lists (Fig. 4c)
 *   evict_expert_union      — per-layer union of the MoE experts the kept
 *                             nodes activate (Eq. 5), from routing ids/masks
 *   evict_router_union      — the router logits W_g·h (Eq. 4) of the kept
 *                             nodes on tcgen05 tensor cores, TopK, and the
 *                             same union
 *   evict_select_build_union— the three calls fused into one launch (same
 *                             outputs as calling them in sequence)
 *   evict_batch_stats       — aggregate statistics for the multi-GPU
 *                             all-reduce.
 *
 * Conventions (every call):
 *  - All array arguments are DEVICE pointers owned by the caller; the
 *    library never allocates, frees or retains them.  Descriptor structs are
 *    host memory, read during the call only.  `stream` is a cudaStream_t.
 *  - Calls are stream-ordered and CUDA-graph capturable: no host sync, no
 *    allocation, no device→host read (PAPER.md:198–204 graph fusion).
 *  - Host-checkable argument errors return EVICT_ERR_INVALID_ARG (or
 *    EVICT_ERR_UNSUPPORTED for a shape this build does not implement, or a
 *    device that is not sm_100) and launch nothing.  Launch failures return
 *    EVICT_ERR_CUDA.
 *  - Data errors are reported per tree in `status` (bits EVICT_TREE_*), and
 *    that tree's outputs are written in their defined error state (k* = 0,
 *    empty keep set, zero rows); other trees are unaffected.
 *  - Outputs are fully overwritten except the accumulating expert_hist.
 *  - Layouts: a tree batch is [B][N] row-major with row stride N
 *    (max_nodes); bit i of 64-bit word i/64 of a bitset refers to node
 *    (or slot, or expert) i.  W = ceil(N/64), EW = ceil(E/64).
 *  - Readings of points the paper leaves open (root score 1, tie rules,
 *    cost domain, verify layout, …) are listed in DESIGN.md §3 (Z1–Z20).
 */
#ifndef EVICT_H
#define EVICT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EVICT_ABI_VERSION 8
#define EVICT_MAX_NODES 128   /* N ≤ 128 ⇒ W ≤ 2 mask words */
#define EVICT_MAX_EXPERTS 256 /* Ling-flash-2.0 has 256 experts */
#define EVICT_MAX_TOPK 16
#define EVICT_MAX_LAYERS 128
#define EVICT_MAX_VOCAB 262144  /* target vocabulary bound of evict_verify_sample */

typedef enum {
    EVICT_OK = 0,
    EVICT_ERR_INVALID_ARG = 1,
    EVICT_ERR_UNSUPPORTED = 2,
    EVICT_ERR_CUDA = 3
} evict_status_t;

/* per-tree data-error bits, OR-ed into status[b] */
#define EVICT_TREE_BAD_SIZE 0x01u   /* n_nodes[b] not in [1, N] */
#define EVICT_TREE_BAD_PARENT 0x02u /* parent[0] != -1 or parent[i] not in [0, i) */
#define EVICT_TREE_BAD_PROB 0x04u   /* q[i] NaN, < 0 or > 1 (i ≥ 1) */
#define EVICT_TREE_BAD_COST 0x08u   /* cost[k-1] NaN or ≤ 0 for a k ≤ n, or cost[0] = +inf */
#define EVICT_TREE_BAD_EXPERT 0x10u /* a kept node routes to an expert id outside [0, E) */
#define EVICT_TREE_BAD_KEEP 0x20u   /* keep set misses the root, is not ancestor-closed, or keeps a pad */
#define EVICT_TREE_BAD_TOKEN 0x40u  /* a kept non-root node's draft token is outside [0, V) */

/* A batch of draft trees (the drafter's tree rooted at x_{t+1}).
 * Nodes are numbered topologically: parent[0] = -1, 0 ≤ parent[i] < i.
 * q[i] = q^T(v_i) = P_Md(v_i | x_{<v_i}); q[0] is ignored
 * (the root is already committed, Score(root) = 1, reading Z1).           */
typedef struct {
    int32_t batch;           /* B ≥ 1 */
    int32_t max_nodes;       /* N: row stride, 1..128, multiple of 4 */
    const int32_t *n_nodes;  /* [B] real node count n_b ∈ [1, N], or NULL (= N) */
    const int32_t *parent;   /* [B][N] int32 */
    const float *q;          /* [B][N] fp32 */
} evict_trees_t;

/* ---------------------------------------------------------------------------
 * evict_select — A1–A5 (§3.1–§3.2.3).
 *   Score(v) = Π_{u∈Path(root,v)} q(u), fp32, one rounding per edge in
 *     root→leaf order (Eq. 7; reading Z6).
 *   order    = nodes by (Score desc, index asc): the top-k prune of §3.2.1;
 *     every prefix is ancestor-closed (tie rule Z4).
 *   S[k]     = Σ_{j<k} Score(order[j]) = Ê[A(T_k)] (Eq. 8), fp32.
 *   k*       = smallest argmax_{1≤k≤n_b} S[k]/C(k) (Eq. 10; Z2, Z3).
 * cost: fp32 C(k) at cost[k-1], k = 1..N, per tree at cost + b*cost_stride
 *   (cost_stride 0 = one shared table); 16-byte aligned, cost_stride % 4 == 0.  C(k) ∈ (0, +inf]; +inf marks an
 *   infeasible k (no verify graph of that length, Z10); cost[0] finite.
 * Outputs: k_star [B] (0 on error), e_hat [B] = S[k*], utility [B] =
 *   S[k*]/C(k*) (C_AR dropped, Z18), keep_bits [B][W] = order[0..k*).
 *   Optional (NULL to skip): order [B][N] rank → node (-1 pad),
 *   prefix_sums [B][N] S[k] at [k-1] (0 pad), status [B].
 * ------------------------------------------------------------------------- */
evict_status_t evict_select(const evict_trees_t *trees, const float *cost, int32_t cost_stride,
                            int32_t *k_star, float *e_hat, float *utility, uint64_t *keep_bits,
                            int32_t *order, float *prefix_sums, uint32_t *status, void *stream);

/* ---------------------------------------------------------------------------
 * Selection policies: the same ranking and prefix
 * sums, a different cut k*.
 *   EVICT_POLICY_COST      Eq. 10 (the default; what evict_select does)
 *   EVICT_POLICY_COVERAGE  k* = smallest k with S_k / S_K ≥ rho, K = n_b,
 *                          S_k / S_K an fp32 IEEE division; the score-
 *                          coverage ablation of PAPER.md:290–292 (§5.4),
 *                          rho = 1 is EAGLE-3 (every node verified).
 *                          Requires 0 < rho ≤ 1.
 *   EVICT_POLICY_FIXED     k* = min(k_fixed, n_b), k_fixed ≥ 1.
 * e_hat = S[k*] and utility = S[k*]/C(k*) under every policy; the cost
 * table is still validated (it prices the reported utility).
 * evict_select_policy / evict_select_build_union_policy take the policy
 * (NULL = EVICT_POLICY_COST); otherwise identical to the calls without it.
 * ------------------------------------------------------------------------- */
typedef enum {
    EVICT_POLICY_COST = 0,
    EVICT_POLICY_COVERAGE = 1,
    EVICT_POLICY_FIXED = 2
} evict_policy_kind_t;

typedef struct {
    int32_t kind;     /* evict_policy_kind_t */
    float rho;        /* COVERAGE */
    int32_t k_fixed;  /* FIXED */
} evict_policy_t;

evict_status_t evict_select_policy(const evict_trees_t *trees, const float *cost, int32_t cost_stride,
                                   const evict_policy_t *policy, int32_t *k_star, float *e_hat,
                                   float *utility, uint64_t *keep_bits, int32_t *order,
                                   float *prefix_sums, uint32_t *status, void *stream);

/* ---------------------------------------------------------------------------
 * evict_build_verify_tree — A6 (Fig. 4(c); layout Z12).
 * keep_bits [B][W]: any ancestor-closed node set containing the root.
 * Packed verify layout: tree b owns rows [off_b, off_b + k_b) of every
 * per-row output, k_b = |keep_b|, off = exclusive scan of k over the batch
 * in tree order (single pass, decoupled look-back).  Capacity B*N rows.
 * Within a tree, slots s = 0..k_b-1 follow ascending node index.
 *   verify_offsets [B+1] off_b; verify_offsets[B] = total rows T
 *   kept_index     [T] node index of slot s
 *   retrieve_index [T] b*N + node: flat index of the row's node in [B][N]
 *                      draft arrays (gather index for tokens/hidden states)
 *   positions      [T] pos_offset[b] + depth(node) (pos_offset NULL ⇒ 0)
 *   next_token     [T] smallest kept child slot, -1 if none
 *   next_sibling   [T] smallest slot > s with the same parent, -1 if none
 *   tree_mask      [T][W] bit j ⇔ slot j is an ancestor-or-self of slot s
 *                      (tree part of the attention mask; prefix KV implicit)
 * A tree with a bad status contributes 0 rows.  Any of the per-row outputs
 * may be NULL.  workspace: device scratch of evict_workspace_bytes(B) bytes
 * (cleared by the call itself with cudaMemsetAsync).
 * ------------------------------------------------------------------------- */
evict_status_t evict_build_verify_tree(const evict_trees_t *trees, const uint64_t *keep_bits,
                                       const int32_t *pos_offset, int32_t *verify_offsets,
                                       int32_t *kept_index, int32_t *retrieve_index,
                                       int32_t *positions, int32_t *next_token,
                                       int32_t *next_sibling, uint64_t *tree_mask,
                                       uint32_t *status, void *workspace, size_t workspace_bytes,
                                       void *stream);

size_t evict_workspace_bytes(int32_t batch);

/* ---------------------------------------------------------------------------
 * evict_expert_union — A7 (Eq. 5; scope Z13, Z16).
 * For each tree b and MoE layer l: union_count[b][l] = |∪_{v kept} E_l(v)|,
 * root included; union_total[b] = Σ_l union_count[b][l].
 * Routing input, node-major rows (only the kept nodes' rows are read):
 *   EVICT_ID_U8 / EVICT_ID_I32: ids [B][N][L][K] — top-K expert ids
 *   EVICT_ID_MASK:              masks [B][N][L][EW] uint64 — one-hot top-K
 *                               sets (bit e ⇔ expert e routed)
 * Outputs: union_count [B][L], union_total [B] (or NULL), union_bits
 * [B][L][EW] (or NULL), expert_hist [L][E] int64 (or NULL; ACCUMULATES the
 * number of trees whose layer-l union contains expert e), status [B] (or
 * NULL; only EVICT_TREE_BAD_EXPERT / BAD_KEEP bits are produced here).
 * ------------------------------------------------------------------------- */
#define EVICT_ID_U8 1
#define EVICT_ID_I32 4
#define EVICT_ID_MASK 8

typedef struct {
    int32_t num_layers;  /* L ≥ 1, ≤ 128 */
    int32_t num_experts; /* E ≥ 1, ≤ 256 */
    int32_t top_k;       /* K, 1 ≤ K ≤ min(E, 16) (ignored for EVICT_ID_MASK) */
    int32_t id_format;   /* EVICT_ID_U8 | EVICT_ID_I32 | EVICT_ID_MASK */
    const void *ids;     /* see above; device memory, or page-locked host memory mapped into the
                            device address space (cudaHostAlloc under UVA): only the kept rows
                            are read, so a host-resident routing table costs PCIe traffic for
                            k*·L·K·s bytes per tree instead of a copy of every node's row */
} evict_routing_t;

evict_status_t evict_expert_union(const evict_trees_t *trees, const uint64_t *keep_bits,
                                  const evict_routing_t *routing, int32_t *union_count,
                                  int32_t *union_total, uint64_t *union_bits,
                                  int64_t *expert_hist, uint32_t *status, void *stream);

/* ---------------------------------------------------------------------------
 * evict_select_build_union — evict_select → evict_build_verify_tree →
 * evict_expert_union in ONE launch (the per-tree state stays on chip).
 * Semantics and outputs are exactly those of the three calls in sequence
 * (status is the OR of the three); any optional output may be NULL.
 * workspace: evict_workspace_bytes(B) bytes, 8-byte aligned, cleared by the
 * call (one state word per tile of the packed-offset scan: one tree per
 * tile for B ≤ 2048 — serving batches, spread one tree per warp — else 4).
 * ------------------------------------------------------------------------- */
typedef struct {
    /* select */
    int32_t *k_star;
    float *e_hat;
    float *utility;
    uint64_t *keep_bits;
    int32_t *order;
    float *prefix_sums;
    /* build */
    const int32_t *pos_offset;
    int32_t *verify_offsets;
    int32_t *kept_index;
    int32_t *retrieve_index;
    int32_t *positions;
    int32_t *next_token;
    int32_t *next_sibling;
    uint64_t *tree_mask;
    /* union */
    int32_t *union_count;
    int32_t *union_total;
    uint64_t *union_bits;
    int64_t *expert_hist;
    uint32_t *status;
    /* A9 (ABI 8): if non-NULL, the call also writes the batch statistics of
     * evict_batch_stats over its own outputs (stats int64 [6 + N + L], dstats
     * double [2]; both overwritten).  Requires k_star, e_hat, utility and status
     * (and union_count when routing is given).  The serving configuration
     * (u8 top-8 ids, E = 128, L ≤ 64, no order / bit rows / histogram)
     * accumulates them inside the fused launch; other configurations run the
     * statistics kernel after it. */
    int64_t *stats;
    double *dstats;
} evict_fused_out_t;

evict_status_t evict_select_build_union(const evict_trees_t *trees, const float *cost,
                                        int32_t cost_stride, const evict_routing_t *routing,
                                        const evict_fused_out_t *out, void *workspace,
                                        size_t workspace_bytes, void *stream);

evict_status_t evict_select_build_union_policy(const evict_trees_t *trees, const float *cost,
                                               int32_t cost_stride, const evict_policy_t *policy,
                                               const evict_routing_t *routing,
                                               const evict_fused_out_t *out, void *workspace,
                                               size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * evict_router_union — A8 → A7 (Eq. 4–5; Z14, Z15).
 * For every packed verify row r < verify_offsets[B] (output of
 * evict_build_verify_tree) and layer l: logits = W_g[l] · h[l][retrieve_index[r]]
 * (bf16 × bf16 → fp32 on tcgen05 tensor cores), E(h) = TopK(logits, K) by
 * (logit desc, expert asc); the ids are OR-ed into the union of the row's
 * tree.  Outputs as evict_expert_union (union_bits is required here as the
 * accumulator; it is cleared by the call).
 *   hidden  bf16 [L][B*N][d]  per-layer hidden states of every draft node
 *   w_gate  bf16 [L][E][d]    router weights, rows = expert centroids
 *   topk_ids int32 [L][B*N][K] (or NULL): per packed row r, at [l][r][j]
 *   max_rows: an upper bound on T = verify_offsets[B] known to the caller
 *            (e.g. its verify-token budget), or 0 for B·N.  It sizes the
 *            launch only (grid, k-split, ring depth).  Contract: T ≤
 *            max_rows (T is device-resident, so the host cannot check it;
 *            rows at or past ceil(max_rows/128)·128 would not be routed).
 * Supported: 1 ≤ E ≤ 256 (E ≤ 128: N = 128 MMA; 128 < E ≤ 256, e.g.
 *   Ling-flash-2.0: N = 256 MMA; the expert rows past E are
 *   zero-filled by TMA and their logits masked to -inf before the TopK),
 *   union_bits [B][L][ceil(E/64)], d % 64 == 0, K ≤ min(16, E), L·B·N < 2^31;
 *   E > 256 → EVICT_ERR_UNSUPPORTED.
 * ------------------------------------------------------------------------- */
typedef struct {
    int32_t num_layers;
    int32_t num_experts;
    int32_t top_k;
    int32_t hidden_dim;  /* d */
    const void *hidden;  /* bf16 [L][B*N][d] */
    const void *w_gate;  /* bf16 [L][E][d] */
    int32_t max_rows;    /* upper bound on T, or 0 (= B*N); launch sizing only */
} evict_router_t;

evict_status_t evict_router_union(const evict_trees_t *trees, const int32_t *verify_offsets,
                                  const int32_t *retrieve_index, const evict_router_t *router,
                                  int32_t *union_count, int32_t *union_total,
                                  uint64_t *union_bits, int32_t *topk_ids, void *stream);

/* ---------------------------------------------------------------------------
 * evict_batch_stats — A9 aggregate statistics (north_star: the only
 * cross-GPU exchange is an all-reduce of these).  int64 stats[6 + N + L]:
 *   [0] trees  [1] Σk*  [2] Σn  [3] Σunion_total  [4] trees with status ≠ 0
 *   [5 .. 5+N]      k* histogram, bins 0..N (bin 0 = errored trees)
 *   [6+N .. 6+N+L)  Σ union_count per layer
 * double dstats[2]: Σ e_hat, Σ utility over trees with status 0.
 * Overwrites stats/dstats.  union_count may be NULL (L = 0).
 * ------------------------------------------------------------------------- */
evict_status_t evict_batch_stats(int32_t batch, int32_t max_nodes, int32_t num_layers,
                                 const int32_t *n_nodes, const int32_t *k_star,
                                 const float *e_hat, const float *utility,
                                 const int32_t *union_count, const uint32_t *status,
                                 int64_t *stats, double *dstats, void *stream);

/* ---------------------------------------------------------------------------
 * evict_union_curve — NEXT-1: the prefix-union curve along the ranking
 * (Fig. 1: the experts a verify pass
 * activates grow with the verified tokens).  For k = 1..n_b:
 *   curve[b][k-1]          = Σ_l |∪_{j<k} E_l(order[b][j])|
 *   curve_layer[b][k-1][l] = |∪_{j<k} E_l(order[b][j])|   (NULL: not written)
 * order: int32 [B][N], the ranking (evict_select's order row); every entry
 * below n_b must be a node < n_b (else EVICT_TREE_BAD_KEEP).  routing as in
 * evict_expert_union (ids and masks: E ≤ 256); an id ≥ E gives
 * EVICT_TREE_BAD_EXPERT.  Entries past n_b, and every entry of an errored
 * tree, are 0.  status: uint32 [B] (may be NULL).
 * ------------------------------------------------------------------------- */
evict_status_t evict_union_curve(const evict_trees_t *trees, const int32_t *order,
                                 const evict_routing_t *routing, int32_t *curve,
                                 int32_t *curve_layer, uint32_t *status, void *stream);

/* ---------------------------------------------------------------------------
 * evict_profile_cost — NEXT-1: the offline cost table C(k) from measured
 * curves (PAPER.md:192–194 profiles C(k) offline; reading R2 with
 * the analytic expected union replaced by the measured one):
 *   Ū(k) = Σ_{b: status_b = 0, n_b ≥ k} curve[b][k-1] / (L · #{those b})
 *   cost[k-1] = c0 + c_union·Ū(k) + c_tok·k, fp64 arithmetic, stored fp32;
 *   +inf when no tree has k nodes (an infeasible k, reading Z10).
 * status may be NULL.  workspace: evict_profile_workspace_bytes(N) bytes,
 * 8-byte aligned, overwritten.  Requires c0 > 0, c_union ≥ 0, c_tok ≥ 0 and
 * c0 + 256·c_union + N·c_tok < 3e38 (else EVICT_ERR_INVALID_ARG), so the
 * result is always a valid evict_select cost table (entries ≥ c0, finite
 * or +inf for an infeasible k).
 * ------------------------------------------------------------------------- */
size_t evict_profile_workspace_bytes(int32_t max_nodes);
evict_status_t evict_profile_cost(int32_t batch, int32_t max_nodes, int32_t num_layers,
                                  const int32_t *n_nodes, const int32_t *curve,
                                  const uint32_t *status, float c0, float c_union, float c_tok,
                                  float *cost, void *workspace, size_t workspace_bytes,
                                  void *stream);

/* ---------------------------------------------------------------------------
 * evict_verify_sample — NEXT-3: verify-side tree sampling (PAPER.md:64–72,
 * §2.1, Eq. 3) on the packed verify tree of evict_build_verify_tree, after
 * the target's single verify pass produced one next-token distribution per
 * verified slot (p over the vocabulary after that node).
 *   EVICT_VERIFY_SAMPLE (T > 0): from the root, visit the kept children c of
 *     the current node u in slot order (next_token, then next_sibling);
 *     accept c iff u_accept[b][c] < p_u(token(c))·2^32; on rejection remove
 *     c's mass and renormalise p_u(w) ← p_u(w)/(1 − p_u(c)) (Eq. 3), fp32,
 *     one IEEE division per rejected sibling in visiting order (reading V3).
 *     When every kept child of u is rejected (or u is a leaf) the bonus
 *     token is the inverse CDF of the residual (p_u with the rejected tokens
 *     zeroed) at u_bonus[b]/2^32, computed EXACTLY: the smallest t with
 *     Σ_{w≤t} r(w) > ⌊u_bonus·Σ_w r(w)/2^32⌋ in units of 2^-149 (reading V4).
 *   EVICT_VERIFY_GREEDY (T = 0): accept the first kept child whose token is
 *     argmax_w p_u(w) (smallest w on ties); the bonus is that argmax (V5).
 * Inputs (DEVICE, caller-owned):
 *   vb->verify_offsets [B+1], next_token / next_sibling / retrieve_index [T]:
 *     evict_build_verify_tree's packed outputs (slot links local to a tree;
 *     retrieve_index = b·N + node); vb->tokens [B·N] int32 draft token of
 *     every node (node-indexed, gathered through retrieve_index; the root's is
 *     unused); vb->max_nodes = N.
 *   probs fp32 [T][row_stride]: row off_b + s is the target distribution
 *     after slot s of tree b; entries in [0, 1]; row_stride ≥ vocab, % 4 == 0,
 *     probs 16-byte aligned; vocab ≤ EVICT_MAX_VOCAB.
 *   u_accept uint32 [B][N] (slot-indexed), u_bonus uint32 [B]: the uniforms
 *     (u/2^32), required for SAMPLE, ignored for GREEDY (may be NULL).
 * Outputs: accept_len [B] (nodes on the accepted path, root included; 0 on
 *   error), accepted_slots [B][N] (the path's slots, -1 pad), bonus_token [B]
 *   (-1 on error), status [B] (NULL to skip): BAD_SIZE (k_b > N), BAD_KEEP
 *   (k_b = 0, or links not strictly increasing within [0, k_b), or a slot
 *   with no parent), BAD_TOKEN, BAD_PROB (a gathered child probability, the
 *   bonus row or a greedy row outside [0, 1] or NaN; or an empty residual).
 *   Checks apply in that order; the first failing one is reported.
 * ------------------------------------------------------------------------- */
#define EVICT_VERIFY_SAMPLE 0
#define EVICT_VERIFY_GREEDY 1
#define EVICT_VERIFY_EXACT 0x10  /* OR into SAMPLE: skip the certified fp64 fast path of the bonus and
                                    always run the fixed-point one (same results; a testing aid) */

typedef struct {
    int32_t batch;                  /* B ≥ 1 */
    int32_t max_nodes;              /* N, 1..128: stride of tokens rows, u_accept and accepted_slots */
    const int32_t *verify_offsets;  /* [B+1] */
    const int32_t *next_token;      /* [T] */
    const int32_t *next_sibling;    /* [T] */
    const int32_t *retrieve_index;  /* [T] */
    const int32_t *tokens;          /* [B][N] */
} evict_verify_batch_t;

evict_status_t evict_verify_sample(const evict_verify_batch_t *vb, const float *probs, int32_t vocab,
                                   int64_t row_stride, int32_t mode, const uint32_t *u_accept,
                                   const uint32_t *u_bonus, int32_t *accept_len, int32_t *accepted_slots,
                                   int32_t *bonus_token, uint32_t *status, void *stream);

/* ---------------------------------------------------------------------------
 * On-device verify-graph dispatch — NEXT-4 (one verify
 * graph is pre-captured per verification length and the one matching the
 * selected length is dispatched; done on the host that needs k* on the host,
 * a device→host sync per step).  evict_dispatch_create builds and
 * instantiates ONE CUDA graph
 *     [pre_graph] → k_dispatch → SWITCH { body_graphs[0] | … | [n−1] }
 * k_dispatch reads T = *rows on the device at launch time (e.g.
 * verify_offsets + B: the packed verify row count the step produced), takes
 * i = the smallest index with lengths[i] ≥ T and sets the switch to it (no
 * body runs when T > lengths[n−1]); *chosen (device int32, may be NULL)
 * receives i or −1.  The selection never leaves the device.
 *   n_bodies   1..EVICT_DISPATCH_MAX
 *   lengths    HOST int32 [n_bodies], strictly ascending, ≥ 0
 *   body_graphs HOST array of cudaGraph_t (the caller's captured verify
 *              graphs; CLONED into the switch bodies, the caller keeps
 *              ownership); each may hold kernel, memset, memcpy, empty and
 *              child-graph nodes (CUDA's rule for conditional bodies)
 *   pre_graph  cudaGraph_t or NULL, cloned, runs before the selection
 *   rows, chosen: DEVICE pointers baked into the graph (must outlive it)
 * The handle is a host object owned by the caller: evict_dispatch_destroy.
 * evict_dispatch_launch = cudaGraphLaunch on `stream`.  Errors: INVALID_ARG
 * (bad arguments), UNSUPPORTED (no sm_100 device), CUDA (graph API error).
 * ------------------------------------------------------------------------- */
#define EVICT_DISPATCH_MAX 32
typedef struct evict_dispatch_s *evict_dispatch_t;

evict_status_t evict_dispatch_create(int32_t n_bodies, const int32_t *lengths, void *const *body_graphs,
                                     void *pre_graph, const int32_t *rows, int32_t *chosen,
                                     evict_dispatch_t *out);
evict_status_t evict_dispatch_launch(evict_dispatch_t d, void *stream);
void evict_dispatch_destroy(evict_dispatch_t d);

/* ---------------------------------------------------------------------------
 * evict_build_draft_tree — NEXT-4 (P2): the EAGLE-style draft tree on the
 * device (§2.1: the drafter "repeatedly extends a fixed number of
 * draft tokens … with the same number of tokens at each layer"; the budget
 * cut keeps "the top-k nodes ranked by cumulative scores").
 * Per tree b, from the drafter's per-step top-`topk` tables:
 *   pool = {root}, Score(root) = 1, frontier = [root]
 *   step s: frontier slot j's children c = 0..topk-1 get parent frontier[j],
 *     token child_tokens[b][s][j][c], q = child_probs[b][s][j][c],
 *     Score = fl32(Score(parent)·q) (Eq. 7); the next frontier = the topk
 *     new nodes with the best (Score desc, creation index asc).  Step 0 uses
 *     slot 0 (the root) only.
 *   keep = root + the max_nodes − 1 best pool nodes by (Score desc, creation
 *     index asc); renumbered by creation index (parent < child, reading Z12).
 * Inputs (DEVICE): child_tokens int32 / child_probs fp32 [B][steps][topk][topk].
 * Outputs (DEVICE, [B][N] rows, N = max_nodes): parent (-1 root and pads),
 *   q (1 root, 0 pads), tokens (-1 root — x_{t+1} comes from the target —
 *   and pads), n_nodes [B] = min(N, 1 + topk + (steps−1)·topk²), status [B]
 *   (NULL to skip): BAD_PROB when a read probability is NaN or outside [0,1]
 *   (that tree's outputs are pads, n = 0).  The rows are a valid
 *   evict_trees_t (with N % 4 == 0).
 * Host errors: 1 ≤ steps ≤ 16, 1 ≤ topk ≤ 16, 1 ≤ N ≤ 128, pool
 *   1 + topk + (steps−1)·topk² ≤ EVICT_DRAFT_MAX_POOL.
 * ------------------------------------------------------------------------- */
#define EVICT_DRAFT_MAX_POOL 2048

evict_status_t evict_build_draft_tree(int32_t batch, int32_t steps, int32_t topk, int32_t max_nodes,
                                      const int32_t *child_tokens, const float *child_probs,
                                      int32_t *parent, float *q, int32_t *tokens, int32_t *n_nodes,
                                      uint32_t *status, void *stream);

const char *evict_status_string(evict_status_t s);
int evict_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* EVICT_H */
