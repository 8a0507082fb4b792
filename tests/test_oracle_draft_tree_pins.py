"""Pins of the draft-tree builder oracle (oracle/draft_tree.py) — CPU only.

Checked against what PAPER.md and SPEC.md fix, not against the oracle's own loop: SPEC.md:262's
top-1 chain, the node counts the expansion implies, Eq. 7 scores recomputed edge by edge,
ancestor closure and topological numbering, the "well-structured" layer sizes,
PAPER.md:135's optimality of the kept set over every ancestor-closed subset of the candidate
pool (brute force), and agreement with the separately written A3 ranking of the C oracle.
"""
import itertools

import numpy as np
import pytest

import oracle
from gen.draft import drafter_tables
from oracle import draft_tree as od


def _depths(parent, n):
    d = np.zeros(n, np.int32)
    for i in range(1, n):
        d[i] = d[parent[i]] + 1
    return d


def test_top1_chain():
    """steps = 1, topk = 1 gives a 2-node chain whose child is the drafter's top token."""
    tok = np.array([[[[42]]]], np.int32)
    pr = np.array([[[[0.75]]]], np.float32)
    o = od.build_draft_trees(tok, pr, 1, 1, 8)
    assert o["n_nodes"][0] == 2 and o["parent"][0, :2].tolist() == [-1, 0]
    assert o["tokens"][0, 1] == 42 and o["q"][0, 1] == np.float32(0.75) and o["q"][0, 0] == 1


@pytest.mark.parametrize("steps,topk,N", [(4, 8, 32), (6, 10, 60), (8, 10, 128), (3, 4, 500), (2, 3, 7)])
def test_counts_scores_closure(steps, topk, N):
    tok, pr = drafter_tables(3, 6, steps, topk)
    o = od.build_draft_trees(tok, pr, steps, topk, N)
    pool = 1 + topk + (steps - 1) * topk * topk
    for b in range(6):
        n = int(o["n_nodes"][b])
        assert n == min(N, pool)
        par, q, sc = o["parent"][b], o["q"][b], o["score"][b]
        assert par[0] == -1 and sc[0] == 1
        for i in range(1, n):
            assert 0 <= par[i] < i                                   # topological, ancestor-closed
            assert sc[i] == np.float32(sc[par[i]] * q[i])            # Eq. 7, one fp32 rounding
            assert sc[i] <= sc[par[i]]
            assert q[i] in pr[b]                                     # every q comes from the table
        assert (par[n:] == -1).all() and (o["tokens"][b, n:] == -1).all()


@pytest.mark.parametrize("steps,topk", [(3, 3), (4, 2), (2, 5)])
def test_well_structured_layers(steps, topk):
    """With no budget cut (N ≥ pool): depth 1 holds topk nodes and every deeper layer holds the
    topk² children of exactly topk expanded parents — the same number of expanded tokens per layer."""
    tok, pr = drafter_tables(5, 4, steps, topk)
    o = od.build_draft_trees(tok, pr, steps, topk, 10_000)
    for b in range(4):
        n = int(o["n_nodes"][b])
        par = o["parent"][b, :n]
        d = _depths(par, n)
        assert (d == 1).sum() == topk
        for depth in range(2, steps + 1):
            kids = np.flatnonzero(d == depth)
            assert len(kids) == topk * topk
            assert len(set(par[kids].tolist())) == topk                 # topk frontier parents
        # siblings carry the drafter's children of their parent in table order, with its tokens
        for u in range(n):
            ch = np.flatnonzero(par == u)
            if len(ch):
                assert (np.diff(ch) > 0).all()


def _ancestor_closed_best(pool, k):
    """Brute force over every k-subset containing the root: max Σ score among ancestor-closed ones."""
    n = len(pool)
    best = None
    for sub in itertools.combinations(range(1, n), k - 1):
        s = set(sub) | {0}
        if all(pool[i]["parent"] in s for i in sub):
            v = sum(float(pool[i]["score"]) for i in s)
            best = v if best is None or v > best else best
    return best


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_kept_set_is_the_best_subtree_of_the_pool(seed):
    """the top-k by cumulative score is optimal among all valid k-node subtrees
    of the (unpruned) well-structured tree."""
    steps, topk = 2, 3                       # pool of 1 + 3 + 9 = 13 candidates
    tok, pr = drafter_tables(seed, 1, steps, topk)
    for N in (2, 4, 6, 9):
        st, par, q, t, sc, n, pool = od.build_one(tok[0], pr[0], steps, topk, N)
        assert abs(sum(float(x) for x in sc[:n]) - _ancestor_closed_best(pool, N)) <= 1e-6


def test_kept_set_is_the_a3_ranking_prefix():
    """The builder's budget cut and the C oracle's A3 ranking (oracle.select) of the uncut tree
    agree: the N best nodes of the full pool are exactly order[:N]."""
    steps, topk = 4, 6
    tok, pr = drafter_tables(9, 8, steps, topk)
    full = od.build_draft_trees(tok, pr, steps, topk, 1 + topk + (steps - 1) * topk * topk)
    M = full["parent"].shape[1]
    Mp = (M + 3) // 4 * 4
    P = np.full((8, Mp), 0, np.int32)
    Q = np.zeros((8, Mp), np.float32)
    P[:, :M], Q[:, :M] = full["parent"], full["q"]
    n = full["n_nodes"]
    sel = oracle.select(P[:, :Mp] if Mp <= 128 else P, Q, np.ones(Mp, np.float32), n_nodes=n)
    for N in (16, 32, 60):
        cut = od.build_draft_trees(tok, pr, steps, topk, N)
        for b in range(8):
            kept_full_ids = sorted(sel["order"][b, :N].tolist())
            # the cut tree renumbers the kept nodes by creation index: same tokens in the same order
            assert [int(full["tokens"][b, i]) for i in kept_full_ids] == cut["tokens"][b, :N].tolist()


def test_bad_probability():
    tok, pr = drafter_tables(2, 3, 3, 4)
    pr = pr.copy()
    pr[1, 2, 3, 1] = np.nan
    pr[2, 0, 0, 0] = 1.5
    o = od.build_draft_trees(tok, pr, 3, 4, 32)
    assert o["status"].tolist() == [0, od.TREE_BAD_PROB, od.TREE_BAD_PROB]
    assert o["n_nodes"][1] == 0 and (o["parent"][1] == -1).all()
