"""Pins of the CPU oracle against what PAPER.md and mathematics fix (CPU only).

Every oracle function is pinned by at least one check that does not re-type its
own formula: exact rational brute force over all ancestor-closed subsets, the
chain closed form of Eq. 6 (Appendix A), the worked toy tree, SPEC examples,
library routines (numpy matmul + stable argsort, Python sets) and invariants.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from bruteforce import (ancestor_closed_subsets, best_ratio, best_sum_per_size, exact_scores,
                        is_ancestor_closed)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "toy_tree.json")))


def keep_set(bits, N):
    bits = [int(x) for x in np.atleast_1d(bits)]
    return [i for i in range(min(N, 64 * len(bits))) if (bits[i // 64] >> (i % 64)) & 1]


def rand_tree(rng, n, dyadic=16, allow_ties=True):
    parent = np.full(n, -1, np.int32)
    for i in range(1, n):
        parent[i] = rng.integers(0, i)
    if allow_ties:
        q = rng.integers(0, dyadic + 1, size=n) / dyadic
    else:
        q = rng.integers(1, dyadic, size=n) / dyadic
    q[0] = 1.0
    return parent, q.astype(np.float32)


def select1(parent, q, cost, N=None):
    n = len(parent)
    N = N or n
    P = np.full((1, N), -1, np.int32)
    Q = np.zeros((1, N), np.float32)
    P[0, :n] = parent
    Q[0, :n] = q
    C = np.full(N, 1.0, np.float32)
    C[:len(cost)] = cost
    return oracle.select(P, Q, C, n_nodes=np.array([n], np.int32))


# --------------------------------------------------------------------- toy
def test_toy_tree_golden_is_exact():
    """The golden toy values themselves, re-derived with exact rationals."""
    sc = exact_scores(GOLD["parent"], GOLD["q"])
    assert [float(s) for s in sc] == GOLD["score"]
    best, count = best_sum_per_size(GOLD["parent"], sc)
    assert count == GOLD["ancestor_closed_subsets"]
    assert [float(best[k]) for k in range(1, 9)] == GOLD["S"]
    rstar, ks, _ = best_ratio(GOLD["parent"], sc, GOLD["cost"])
    assert ks == [GOLD["k_star"]]
    assert rstar == Fraction(GOLD["utility_num"]) / Fraction(GOLD["utility_den"])


def test_toy_tree_oracle():
    o = select1(np.array(GOLD["parent"]), np.array(GOLD["q"]), np.array(GOLD["cost"]))
    assert o["status"][0] == 0
    assert o["score"][0].tolist() == GOLD["score"]
    assert o["depth"][0].tolist() == GOLD["depth"]
    assert o["order"][0].tolist() == GOLD["order"]
    assert o["S"][0].tolist() == GOLD["S"]
    assert o["k_star"][0] == GOLD["k_star"]
    assert int(o["keep_bits"][0, 0]) == GOLD["keep_bits"]
    assert o["e_hat"][0] == GOLD["e_hat"]
    assert o["utility"][0] == GOLD["utility_num"] / GOLD["utility_den"]
    assert keep_set(o["tie_bits"][0], 8) == [2]       # k=3 only (bit k-1)


@pytest.mark.parametrize("name", ["constant", "linear", "exact_tie"])
def test_toy_cost_variants(name):
    v = GOLD["cost_variants"][name]
    o = select1(np.array(GOLD["parent"]), np.array(GOLD["q"]), np.array(v["cost"]))
    assert o["k_star"][0] == v["k_star"]
    ties = [b + 1 for b in keep_set(o["tie_bits"][0], 8)]
    assert ties == v.get("tie_ks", [v["k_star"]])


@pytest.mark.parametrize("k", ["3", "5", "8"])
def test_toy_verify_tree(k):
    v = GOLD["verify"][k]
    keep = np.zeros((1, 1), np.uint64)
    for i in v["kept_index"]:
        keep[0, 0] |= np.uint64(1 << i)
    o = oracle.build_verify_tree(np.array([GOLD["parent"]], np.int32), keep)
    kk = int(k)
    assert o["status"][0] == 0
    assert o["verify_offsets"].tolist() == [0, kk]
    assert o["kept_index"][:kk].tolist() == v["kept_index"]
    assert [int(x) for x in o["tree_mask"][:kk, 0]] == v["mask"]
    assert o["positions"][:kk].tolist() == v["positions"]
    assert o["next_token"][:kk].tolist() == v["next_token"]
    assert o["next_sibling"][:kk].tolist() == v["next_sibling"]
    assert o["retrieve_index"][:kk].tolist() == v["kept_index"]


def test_toy_union_along_ranking():
    routing = np.stack([np.array(GOLD["routing_L0"]), np.array(GOLD["routing_L1"])], axis=1)
    ids = routing[None].astype(np.uint8)                     # [1][8][2][2]
    for k in range(1, 9):
        keep = np.zeros((1, 1), np.uint64)
        for v in GOLD["order"][:k]:
            keep[0, 0] |= np.uint64(1 << v)
        o = oracle.expert_union(keep, ids, 8)
        assert o["union_count"][0].tolist() == GOLD["union_along_ranking"][k - 1]
        assert o["union_total"][0] == GOLD["union_total_along_ranking"][k - 1]
        # Python-set definition of Eq. 5
        for l in range(2):
            u = set()
            for v in GOLD["order"][:k]:
                u |= set(routing[v, l].tolist())
            assert sorted(u) == keep_set(o["union_bits"][0, l], 8)


# ------------------------------------------------------------- brute force
@pytest.mark.parametrize("seed", range(40))
def test_ranking_prefix_is_best_subtree_bruteforce(seed):
    """the top-k ranking prefix is ancestor-closed and sum-optimal for every k."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 13))
    parent, q = rand_tree(rng, n, dyadic=8)
    sc = exact_scores(parent, q)
    best, _ = best_sum_per_size(parent, sc)
    o = select1(parent, q, np.ones(n))
    assert o["status"][0] == 0
    assert [Fraction(float(x)) for x in o["score"][0]] == sc     # dyadic, depth ≤ 11: exact in fp32
    order = o["order"][0].tolist()
    for k in range(1, n + 1):
        assert is_ancestor_closed(parent, order[:k])
        assert Fraction(o["S"][0, k - 1]) == best[k]


@pytest.mark.parametrize("seed", range(40))
def test_argmax_equals_bruteforce_ratio(seed):
    """Eq. 10: R[k*] = max over all root-containing ancestor-closed U of Σ/C(|U|), smallest k."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 12))
    parent, q = rand_tree(rng, n, dyadic=8)
    cost = (rng.integers(1, 64, size=n) / 8).astype(np.float32)
    if seed % 5 == 0 and n > 1:
        cost[rng.integers(1, n)] = np.inf               # infeasible k (reading Z10)
    sc = exact_scores(parent, q)
    rstar, ks, _ = best_ratio(parent, sc, cost)
    o = select1(parent, q, cost)
    assert o["k_star"][0] == ks[0]
    assert Fraction(o["utility"][0]) == pytest.approx(rstar, rel=1e-15)
    assert Fraction(o["e_hat"][0]) == best_sum_per_size(parent, sc)[0][ks[0]]
    # every exact tie is inside the reported near-tie set
    ties = [b + 1 for b in keep_set(o["tie_bits"][0], n)]
    assert set(ks) <= set(ties)


def test_subset_enumerator_counts():
    """Enumerator sanity: chain of n has n subsets, star of n has 2^(n-1)."""
    assert sum(1 for _ in ancestor_closed_subsets([-1, 0, 1, 2, 3])) == 5
    assert sum(1 for _ in ancestor_closed_subsets([-1, 0, 0, 0, 0])) == 16


# ------------------------------------------------------ closed forms, SPEC
def test_chain_closed_form():
    """Eq. 6 on a chain (Appendix A): E = Σ_k Π_{i≤k} p_i, with q as p."""
    p = [0.9, 0.8, 0.5]
    o = select1(np.array([-1, 0, 1, 2]), np.array([1] + p), np.array([1, 1, 1, 1.0]))
    closed = 1 + 0.9 + 0.9 * 0.8 + 0.9 * 0.8 * 0.5
    assert o["S"][0, 3] == pytest.approx(closed, rel=1e-7)
    assert o["S"][0, 3] == pytest.approx(2.98, rel=1e-7)


@pytest.mark.parametrize("n", [1, 2, 8, 33, 64, 128])
def test_chain_dyadic_exact(n):
    rng = np.random.default_rng(n)
    q = np.concatenate([[1.0], rng.choice([1.0, 0.5, 0.75, 0.875], size=n - 1)]).astype(np.float32)
    parent = np.arange(-1, n - 1, dtype=np.int32)
    o = select1(parent, q, np.ones(n))
    prod, acc = Fraction(1), Fraction(0)
    for k in range(n):
        if k:
            prod *= Fraction(float(q[k]))
        acc += prod
        assert o["order"][0, k] == k                       # chain: ranking is depth order
    # fp32 products may round beyond 24 bits; compare within fp32 accumulated error
    assert o["S"][0, n - 1] == pytest.approx(float(acc), rel=n * 2 ** -23)


def test_spec_examples():
    # SPEC.md:317 chain root→a→b with q 0.5, 0.5: S = [1, 1.5, 1.75]
    o = select1(np.array([-1, 0, 1]), np.array([1, .5, .5]), np.ones(3))
    assert o["S"][0].tolist() == [1, 1.5, 1.75]
    # SPEC.md:318 root only: S = [1]
    o = select1(np.array([-1]), np.array([1.0]), np.ones(1))
    assert o["S"][0].tolist() == [1] and o["k_star"][0] == 1
    # SPEC.md:327 root with children 0.3 and 0.5: S[3] = 1.8
    o = select1(np.array([-1, 0, 0]), np.array([1, .3, .5]), np.ones(3))
    assert o["S"][0, 2] == pytest.approx(1.8, rel=1e-7)
    # SPEC.md:447 S=[1,1.5,1.6], C=[10,12,20] → k* = 2
    o = select1(np.array([-1, 0, 0]), np.array([1, .5, .1]), np.array([10, 12, 20.]))
    assert o["S"][0].tolist() == pytest.approx([1, 1.5, 1.6], rel=1e-7)
    assert o["k_star"][0] == 2


@pytest.mark.parametrize("seed", range(20))
def test_constant_cost_keeps_full_tree(seed):
    """SPEC.md:448 / north_star invariant (reading Z8: q ∈ [0.5, 1] avoids fp32 absorption)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 129))
    parent = np.array([-1] + [int(rng.integers(0, i)) for i in range(1, n)], np.int32)
    q = np.concatenate([[1], rng.uniform(0.5, 1.0, n - 1)]).astype(np.float32)
    o = select1(parent, q, np.full(n, 3.0))
    assert o["k_star"][0] == n
    assert keep_set(o["keep_bits"][0], 128) == list(range(n))


@pytest.mark.parametrize("seed", range(20))
def test_linear_cost_keeps_root_only(seed):
    """C(k) = c·k ⇒ S[k]/k is a running mean of a non-increasing sequence ⇒ k* = 1."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 129))
    parent = np.array([-1] + [int(rng.integers(0, i)) for i in range(1, n)], np.int32)
    q = np.concatenate([[1], rng.uniform(0.0, 1.0, n - 1)]).astype(np.float32)
    o = select1(parent, q, 0.37 * np.arange(1, n + 1))
    assert o["k_star"][0] == 1
    assert keep_set(o["keep_bits"][0], 128) == [0]


@pytest.mark.parametrize("seed", range(10))
def test_scale_invariance(seed):
    """C_AR (any constant factor on C) does not move k* (SPEC.md:479)."""
    rng = np.random.default_rng(200 + seed)
    n = int(rng.integers(2, 100))
    parent = np.array([-1] + [int(rng.integers(0, i)) for i in range(1, n)], np.int32)
    q = np.concatenate([[1], rng.uniform(0.0, 1.0, n - 1)]).astype(np.float32)
    cost = (10 + rng.uniform(0, 1, n).cumsum()).astype(np.float32)
    a = select1(parent, q, cost)
    b = select1(parent, q, cost * np.float32(8.0))
    assert a["k_star"][0] == b["k_star"][0]
    assert b["utility"][0] == pytest.approx(a["utility"][0] / 8, rel=1e-15)


def test_naive_argmax_loop():
    """k* equals a naive loop over (S, C) pairs."""
    rng = np.random.default_rng(7)
    for _ in range(200):
        n = int(rng.integers(1, 60))
        parent = np.array([-1] + [int(rng.integers(0, i)) for i in range(1, n)], np.int32)
        q = np.concatenate([[1], rng.uniform(0, 1, n - 1)]).astype(np.float32)
        cost = rng.uniform(1, 5, n).astype(np.float32)
        o = select1(parent, q, cost)
        S = o["S"][0, :n]
        best_k, best_r = 1, S[0] / float(cost[0])
        for k in range(2, n + 1):
            r = S[k - 1] / float(cost[k - 1])
            if r > best_r:
                best_k, best_r = k, r
        assert o["k_star"][0] == best_k


def test_q_one_ties_rank_ancestors_first():
    """Reading Z4: with q = 1 a child ties its parent; index order keeps prefixes closed."""
    parent = np.array([-1, 0, 1, 0, 3, 2], np.int32)
    q = np.ones(6, np.float32)
    o = select1(parent, q, np.arange(1, 7.0) ** 0.5)
    assert o["order"][0].tolist() == [0, 1, 2, 3, 4, 5]


def test_zero_and_subnormal_scores():
    """Z9/Z17: q = 0 and −0.0 are legal (score 0 ranks last by index); subnormals are kept."""
    parent = np.arange(-1, 127, dtype=np.int32)
    q = np.full(128, 0.5, np.float32)
    q[0] = 1
    o = select1(parent, q, np.ones(128))
    assert o["score"][0, 127] == np.float32(2.0 ** -127)          # subnormal, exact
    parent = np.array([-1, 0, 0, 1], np.int32)
    q = np.array([1, 0.0, -0.0, 0.5], np.float32)
    o = select1(parent, q, np.ones(4))
    assert o["status"][0] == 0
    assert o["order"][0].tolist() == [0, 1, 2, 3]
    assert np.signbit(o["score"][0]).sum() == 0


def test_invalid_inputs_status():
    base_p = np.array([-1, 0, 0, 1], np.int32)
    base_q = np.array([1, .5, .5, .5], np.float32)
    cases = [
        (np.array([0, 0, 0, 1]), base_q, np.ones(4), oracle.TREE_BAD_PARENT),
        (np.array([-1, 0, 3, 1]), base_q, np.ones(4), oracle.TREE_BAD_PARENT),
        (base_p, np.array([1, .5, 1.5, .5]), np.ones(4), oracle.TREE_BAD_PROB),
        (base_p, np.array([1, .5, np.nan, .5]), np.ones(4), oracle.TREE_BAD_PROB),
        (base_p, np.array([1, -.5, .5, .5]), np.ones(4), oracle.TREE_BAD_PROB),
        (base_p, base_q, np.array([1, 0, 1, 1.]), oracle.TREE_BAD_COST),
        (base_p, base_q, np.array([np.inf, 1, 1, 1.]), oracle.TREE_BAD_COST),
        (base_p, base_q, np.array([1, np.nan, 1, 1.]), oracle.TREE_BAD_COST),
    ]
    for p, q, c, bit in cases:
        o = select1(p, q, c)
        assert o["status"][0] & bit, (p, q, c)
        assert o["k_star"][0] == 0 and int(o["keep_bits"][0, 0]) == 0
    P = np.zeros((2, 4), np.int32)
    o = oracle.select(P, np.zeros((2, 4), np.float32), np.ones(4, np.float32),
                      n_nodes=np.array([0, 5], np.int32))
    assert (o["status"] & oracle.TREE_BAD_SIZE).all()


# ------------------------------------------------------------------ build
@pytest.mark.parametrize("seed", range(30))
def test_verify_tree_invariants(seed):
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(1, 129))
    parent = np.array([-1] + [int(rng.integers(0, i)) for i in range(1, n)], np.int32)
    q = np.concatenate([[1], rng.uniform(0, 1, n - 1)]).astype(np.float32)
    sel = select1(parent, q, np.ones(n), N=128)
    kstar = int(rng.integers(1, n + 1))
    keep = np.zeros((1, 2), np.uint64)
    for v in sel["order"][0, :kstar]:
        keep[0, v // 64] |= np.uint64(1 << int(v % 64))
    P = np.full((1, 128), -1, np.int32)
    P[0, :n] = parent
    o = oracle.build_verify_tree(P, keep, n_nodes=np.array([n], np.int32),
                                 pos_offset=np.array([17], np.int32))
    assert o["status"][0] == 0
    k = o["verify_offsets"][1]
    assert k == kstar
    kept = o["kept_index"][:k].tolist()
    assert kept == sorted(kept) and is_ancestor_closed(parent, kept)
    slot = {v: s for s, v in enumerate(kept)}
    depth = sel["depth"][0]
    rows = [int(o["tree_mask"][s, 0]) | (int(o["tree_mask"][s, 1]) << 64) for s in range(k)]
    for s, v in enumerate(kept):
        assert o["positions"][s] - 17 == depth[v]
        assert bin(rows[s]).count("1") == depth[v] + 1
        assert rows[s] >> (s + 1) == 0                              # lower triangular
        if v:
            assert rows[s] == rows[slot[int(parent[v])]] | (1 << s)
        else:
            assert rows[s] == 1
    # next_token / next_sibling reconstruct exactly the kept parent relation
    rec = {}
    for s in range(k):
        c = o["next_token"][s]
        while c != -1:
            rec[int(c)] = s
            c = o["next_sibling"][c]
    assert rec == {slot[v]: slot[int(parent[v])] for v in kept if v}


def test_verify_tree_chain_and_star():
    n = 70
    P = np.arange(-1, n - 1, dtype=np.int32)[None]
    keep = np.array([[(1 << 64) - 1, (1 << 6) - 1]], np.uint64)
    o = oracle.build_verify_tree(P, keep)
    for s in range(n):
        row = int(o["tree_mask"][s, 0]) | (int(o["tree_mask"][s, 1]) << 64)
        assert row == (1 << (s + 1)) - 1                           # all-ones lower triangle
    P = np.array([[-1] + [0] * 9], np.int32)
    keep = np.array([[(1 << 10) - 1]], np.uint64)
    o = oracle.build_verify_tree(P, keep)
    assert [int(x) for x in o["tree_mask"][:10, 0]] == [1] + [1 | (1 << s) for s in range(1, 10)]
    assert o["next_sibling"][:10].tolist() == [-1] + list(range(2, 10)) + [-1]


def test_verify_tree_batch_offsets_and_bad_keep():
    P = np.array([[-1, 0, 0, 1], [-1, 0, 1, 2], [-1, 0, 0, 0]], np.int32)
    keep = np.array([[0b0011], [0b0101], [0b1111]], np.uint64)
    o = oracle.build_verify_tree(P, keep, pos_offset=np.array([5, 6, 7], np.int32))
    assert o["status"].tolist() == [0, oracle.TREE_BAD_KEEP, 0]     # tree 1: node 2 without parent 1
    assert o["verify_offsets"].tolist() == [0, 2, 2, 6]
    assert o["retrieve_index"][:6].tolist() == [0, 1, 8, 9, 10, 11]
    assert o["positions"][:6].tolist() == [5, 6, 7, 8, 8, 8]


# ------------------------------------------------------------------ union
def rand_routing(rng, N, L, E, K):
    ids = np.stack([np.stack([rng.permutation(E)[:K] for _ in range(L)]) for _ in range(N)])
    return ids[None].astype(np.uint8)


def test_union_single_node_and_idempotence():
    rng = np.random.default_rng(0)
    ids = rand_routing(rng, 6, 5, 128, 8)
    o = oracle.expert_union(np.array([[1]], np.uint64), ids, 128)
    assert o["union_count"][0].tolist() == [8] * 5 and o["union_total"][0] == 40
    dup = ids.copy()
    dup[0, 1] = dup[0, 0]                                          # node 1 routes like node 0
    o1 = oracle.expert_union(np.array([[0b01]], np.uint64), dup, 128)
    o2 = oracle.expert_union(np.array([[0b11]], np.uint64), dup, 128)
    assert (o1["union_bits"] == o2["union_bits"]).all()


@pytest.mark.parametrize("seed", range(10))
def test_union_set_definition_and_bounds(seed):
    rng = np.random.default_rng(seed)
    N, L, E, K = 60, 7, 128 if seed % 2 else 256, 8
    ids = rand_routing(rng, N, L, E, K).astype(np.int32 if seed % 3 == 0 else np.uint8)
    if E == 256 and ids.dtype == np.uint8:
        pass
    keep_nodes = sorted(set([0] + rng.choice(N, int(rng.integers(1, N)), replace=False).tolist()))
    keep = np.zeros((1, 1), np.uint64)
    for v in keep_nodes:
        keep[0, 0] |= np.uint64(1 << v)
    o = oracle.expert_union(keep, ids, E)
    assert o["status"][0] == 0
    for l in range(L):
        u = set()
        for v in keep_nodes:
            u |= set(ids[0, v, l].tolist())
        assert o["union_count"][0, l] == len(u)
        assert keep_set(o["union_bits"][0, l], E) == sorted(u)
        assert K <= len(u) <= min(E, K * len(keep_nodes))
    # order independence: permute node rows together with the keep set
    perm = np.concatenate([[0], rng.permutation(np.arange(1, N))])
    ids2 = ids[:, perm]
    keep2 = np.zeros((1, 1), np.uint64)
    for v in range(N):
        if perm[v] in keep_nodes:
            keep2[0, 0] |= np.uint64(1 << v)
    o2 = oracle.expert_union(keep2, ids2, E)
    assert (o2["union_count"] == o["union_count"]).all()


def test_union_monotone_identical_disjoint():
    N, L, E, K = 16, 3, 128, 8
    same = np.tile(np.arange(K, dtype=np.uint8), (1, N, L, 1))
    disj = np.zeros((1, N, L, K), np.uint8)
    for v in range(N):
        disj[0, v, :, :] = np.arange(v * K, v * K + K) % E
    prev = 0
    for k in range(1, N + 1):
        keep = np.array([[(1 << k) - 1]], np.uint64)
        a = oracle.expert_union(keep, same, E)
        b = oracle.expert_union(keep, disj, E)
        assert a["union_count"][0].tolist() == [K] * L
        assert b["union_count"][0].tolist() == [min(E, K * k)] * L
        assert b["union_total"][0] >= prev
        prev = b["union_total"][0]


def test_union_bad_expert():
    ids = np.zeros((1, 2, 1, 2), np.int32)
    ids[0, 1, 0, 1] = 200
    o = oracle.expert_union(np.array([[0b11]], np.uint64), ids, 128)
    assert o["status"][0] & oracle.TREE_BAD_EXPERT and o["union_total"][0] == 0
    o = oracle.expert_union(np.array([[0b01]], np.uint64), ids, 128)   # bad id on a pruned node
    assert o["status"][0] == 0 and o["union_total"][0] == 1


# ----------------------------------------------------------------- router
def bf16_bits(x):
    x = np.asarray(x, np.float32)
    return (x.view(np.uint32) >> 16).astype(np.uint16)       # exact for the values used here


def test_router_identity_weights():
    """W_g rows e_1..e_N, h = e_j routes to expert j."""
    E, d = 8, 64
    W = np.zeros((E, d), np.float32)
    W[np.arange(E), np.arange(E)] = 1
    for j in range(E):
        h = np.zeros(d, np.float32)
        h[j] = 1
        ids, _, _ = oracle.router_topk(bf16_bits(h), bf16_bits(W), 1)
        assert ids.tolist() == [j]


@pytest.mark.parametrize("seed", range(8))
def test_router_matches_library_matmul_topk(seed):
    """Integer-valued bf16 inputs: logits exact; top-K = stable argsort of numpy matmul."""
    rng = np.random.default_rng(seed)
    E, d, K = 128, 256, 8
    W = rng.integers(-2, 3, size=(E, d)).astype(np.float32)
    h = rng.integers(-2, 3, size=d).astype(np.float32)
    ids, logits, nt = oracle.router_topk(bf16_bits(h), bf16_bits(W), K)
    ref = W.astype(np.float64) @ h.astype(np.float64)
    assert (logits == ref).all()
    expect = np.argsort(-ref, kind="stable")[:K]
    assert ids.tolist() == expect.tolist()
    assert nt == (ref[expect[-1]] == ref[np.argsort(-ref, kind="stable")[K]])


def test_router_toy_construction():
    """one-hot W_g rows and h with 2 at the first, 1 at the second expert."""
    L, E, K, d = 2, 8, 2, 64
    routing = np.stack([np.array(GOLD["routing_L0"]), np.array(GOLD["routing_L1"])], axis=0)
    W = np.zeros((L, E, d), np.float32)
    for l in range(L):
        W[l, np.arange(E), np.arange(E)] = 1
    H = np.zeros((L, 8, d), np.float32)
    for l in range(L):
        for v in range(8):
            H[l, v, routing[l, v, 0]] = 2
            H[l, v, routing[l, v, 1]] = 1
    for k in range(1, 9):
        keep = np.zeros((1, 1), np.uint64)
        for v in GOLD["order"][:k]:
            keep[0, 0] |= np.uint64(1 << v)
        o = oracle.router_union(keep, bf16_bits(H), bf16_bits(W), K)
        assert o["union_count"][0].tolist() == GOLD["union_along_ranking"][k - 1]
        assert o["near_tie"].sum() == 0


# ------------------------------------------------------------------ stats
def test_batch_stats_sums():
    rng = np.random.default_rng(3)
    B, N, L = 50, 60, 4
    k = rng.integers(1, N + 1, B).astype(np.int32)
    st = np.zeros(B, np.uint32)
    st[[3, 7]] = 4
    uc = rng.integers(8, 60, (B, L)).astype(np.int32)
    eh = rng.uniform(1, 4, B)
    ut = rng.uniform(0, 1, B)
    s, d = oracle.batch_stats(N, L, k, eh, ut, uc, st)
    good = st == 0
    assert s[0] == B and s[4] == 2 and s[1] == k[good].sum() and s[2] == N * good.sum()
    assert s[3] == uc[good].sum()
    assert (s[6 + N:] == uc[good].sum(0)).all()
    assert s[5:6 + N].sum() == B and s[5] == 2
    assert np.bincount(k[good], minlength=N + 1)[1:].tolist() == s[6:6 + N].tolist()
    assert d[0] == pytest.approx(eh[good].sum()) and d[1] == pytest.approx(ut[good].sum())


# ----------------------------------------------------------- policies (NEXT-2)
def select1p(parent, q, cost, policy):
    n = len(parent)
    P = np.full((1, n), -1, np.int32)
    Q = np.zeros((1, n), np.float32)
    P[0], Q[0] = parent, q
    return oracle.select(P, Q, np.asarray(cost, np.float32), n_nodes=np.array([n], np.int32),
                         policy=policy)


@pytest.mark.parametrize("seed", range(30))
def test_coverage_policy_bruteforce(seed):
    """k* = the smallest prefix with S_k/S_K ≥ ρ.  Independently of the
    oracle's ranking: the smallest size m for which SOME ancestor-closed subset reaches
    ρ·S_total (exact rationals; dyadic q keeps fp32 scores exact)."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 12))
    parent, q = rand_tree(rng, n, dyadic=8)
    sc = exact_scores(parent, q)
    best, _ = best_sum_per_size(parent, sc)
    total = sum(sc)
    for rho in (0.05, 0.4, 0.7, 0.9, 1.0):
        r = Fraction(float(np.float32(rho)))
        m = min(k for k in range(1, n + 1) if best[k] >= r * total)
        o = select1p(parent, q, np.ones(n), ("coverage", rho))
        assert o["status"][0] == 0
        ties = [k + 1 for k in range(n) if (int(o["tie_bits"][0, 0]) >> k) & 1]
        assert o["k_star"][0] == m or (m in ties and o["k_star"][0] in ties), (rho, m, o["k_star"][0])
        kept = keep_set(o["keep_bits"][0], n)
        assert len(kept) == o["k_star"][0] and is_ancestor_closed(parent, kept)
        assert sum(sc[v] for v in kept) == best[len(kept)]


def test_coverage_rho_one_is_eagle3_full_tree():
    """ρ = 1 verifies every node under the budget (EAGLE-3): k* = the number of
    nodes with a positive score (zero-score nodes add nothing to S_K and rank last)."""
    rng = np.random.default_rng(7)
    for _ in range(40):
        n = int(rng.integers(1, 40))
        parent, q = rand_tree(rng, n, dyadic=4)
        o = select1p(parent, q, np.ones(n), ("coverage", 1.0))
        pos = int((o["score"][0, :n] > 0).sum())
        assert o["k_star"][0] == pos


def test_coverage_chain_closed_form():
    """Chain with q = 1/2: S_k = 2(1 − 2^-k), so the smallest k with S_k/S_n ≥ ρ is
    ceil(−log2(1 − ρ(1 − 2^-n)))."""
    import math
    for n in (1, 2, 5, 12, 30):
        parent = np.arange(-1, n - 1, dtype=np.int32)
        q = np.full(n, 0.5, np.float32)
        for rho in (0.3, 0.5, 0.75, 0.9, 0.99):
            r = float(np.float32(rho))
            x = 1.0 - r * (1.0 - 2.0 ** -n)
            want = max(1, math.ceil(-math.log2(x) - 1e-12))
            o = select1p(parent, q, np.ones(n), ("coverage", rho))
            ties = [k + 1 for k in range(n) if (int(o["tie_bits"][0, 0]) >> k) & 1]
            assert o["k_star"][0] == min(want, n) or o["k_star"][0] in ties


@pytest.mark.parametrize("seed", range(20))
def test_fixed_policy_equals_cost_policy_with_spike_table(seed):
    """fixed-k ≡ the Eq. 10 argmax with C(j) = 1 at j = min(k, n) and 1e30 elsewhere (C(1)
    must stay finite, Z10; S ≥ 1 makes the spike the argmax), which pins it to the
    already-pinned cost path; the kept set is the best ancestor-closed subset of that size."""
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(1, 12))
    parent, q = rand_tree(rng, n, dyadic=8)
    sc = exact_scores(parent, q)
    best, _ = best_sum_per_size(parent, sc)
    for kf in (1, 2, 3, 5, 8, 20):
        o = select1p(parent, q, np.ones(n), ("fixed", kf))
        kk = min(kf, n)
        C = np.full(n, 1e30, np.float32)
        C[kk - 1] = 1.0
        c = select1p(parent, q, C, None)
        assert o["k_star"][0] == kk == c["k_star"][0]
        assert (o["keep_bits"] == c["keep_bits"]).all()
        kept = keep_set(o["keep_bits"][0], n)
        assert sum(sc[v] for v in kept) == best[kk]


# ------------------------------------------------------------ union curve (NEXT-1)
def _curve_sets(order, ids, n):
    """Σ_l |∪_{j<k} E_l(order[j])| by Python set unions (the definition, written out)."""
    L = ids.shape[1]
    seen = [set() for _ in range(L)]
    out = []
    for k in range(n):
        v = int(order[k])
        for l in range(L):
            seen[l].update(int(e) for e in ids[v, l])
        out.append(sum(len(s) for s in seen))
    return out


@pytest.mark.parametrize("seed", range(12))
def test_union_curve_set_definition(seed):
    rng = np.random.default_rng(3000 + seed)
    B, N, L, E, K = 5, 16, 6, 32, 4
    P = np.full((B, N), -1, np.int32)
    Q = np.zeros((B, N), np.float32)
    n = rng.integers(1, N + 1, B).astype(np.int32)
    for b in range(B):
        p, q = rand_tree(rng, int(n[b]), dyadic=8)
        P[b, :n[b]], Q[b, :n[b]] = p, q
    ids = np.stack([rng.permutation(E)[:K] for _ in range(B * N * L)]).reshape(B, N, L, K).astype(np.uint8)
    o = oracle.select(P, Q, np.ones(N, np.float32), n_nodes=n)
    c = oracle.union_curve(o["order"], ids, E, n_nodes=n)
    for b in range(B):
        want = _curve_sets(o["order"][b], ids[b], int(n[b]))
        assert c["curve"][b, :n[b]].tolist() == want
        assert (c["curve"][b, n[b]:] == 0).all()
        assert (c["curve_layer"][b, :n[b]].sum(axis=1) == c["curve"][b, :n[b]]).all()
        full = oracle.expert_union(np.array([[(1 << int(n[b])) - 1 if n[b] < 64 else ~0]], np.uint64),
                                   ids[b:b + 1], E, n_nodes=n[b:b + 1])
        assert c["curve"][b, n[b] - 1] == full["union_total"][0]   # prefix n = the whole tree


def test_union_curve_identical_and_disjoint_routing():
    """Identical routing for every node: curve(k) = L·K.  Node v on experts vK..vK+K−1
    (disjoint): curve(k) = L·min(k·K, E)."""
    N, L, E, K = 12, 3, 32, 4
    P = np.arange(-1, N - 1, dtype=np.int32)[None]
    Q = np.full((1, N), 0.5, np.float32)
    order = oracle.select(P, Q, np.ones(N, np.float32))["order"]
    same = np.tile(np.arange(K, dtype=np.uint8), (1, N, L, 1))
    assert (oracle.union_curve(order, same, E)["curve"][0] == L * K).all()
    disj = np.zeros((1, N, L, K), np.uint8)
    for v in range(N):
        disj[0, v, :, :] = (np.arange(K) + v * K) % E
    got = oracle.union_curve(order, disj, E)["curve"][0]
    assert got.tolist() == [L * min((k + 1) * K, E) for k in range(N)]


def test_profile_cost_matches_independent_routing_closed_form():
    """With independent uniform top-K routing, E[union of k nodes] = E(1 − (1 − K/E)^k) per
    layer (inclusion of each expert is independent across nodes); the profiled Ū(k) must sit
    within 4σ of it, and C(k) = c0 + c_union·Ū(k) + c_tok·k; k beyond every tree is +inf."""
    rng = np.random.default_rng(11)
    B, N, L, E, K = 400, 24, 8, 128, 8
    P = np.tile(np.arange(-1, N - 1, dtype=np.int32), (B, 1))
    Q = np.full((B, N), 0.75, np.float32)
    n = np.full(B, N, np.int32)
    n[:100] = 20                                  # k > 20 averaged over the other 300 trees
    ids = np.argsort(rng.random((B, N, L, E)), axis=3)[..., :K].astype(np.uint8)
    order = oracle.select(P, Q, np.ones(N, np.float32), n_nodes=n)["order"]
    c = oracle.union_curve(order, ids, E, n_nodes=n)
    cost = oracle.profile_cost(c["curve"], L, n_nodes=n, c0=1.0, c_union=0.5, c_tok=0.25)
    for k in range(1, N + 1):
        m = int((n >= k).sum())
        u = E * (1 - (1 - K / E) ** k)
        # per-layer union of k nodes: variance ≤ E·p(1−p) per layer (negatively correlated sums)
        p = 1 - (1 - K / E) ** k
        sd = np.sqrt(E * p * (1 - p) / (L * m))
        ubar = (cost[k - 1] - 1.0 - 0.25 * k) / 0.5
        assert abs(ubar - u) < 4 * sd + 1e-9, (k, ubar, u)
    n2 = np.full(B, 10, np.int32)
    c2 = oracle.union_curve(order, ids, E, n_nodes=n2)
    cost2 = oracle.profile_cost(c2["curve"], L, n_nodes=n2)
    assert np.isinf(cost2[10:]).all() and np.isfinite(cost2[:10]).all()
