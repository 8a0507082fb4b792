"""NEXT-4 (P2): GPU draft-tree builder vs the oracle (oracle/draft_tree.py), bit-exact."""
import numpy as np
import pytest

from gen.draft import drafter_tables
from oracle import draft_tree as od

pytestmark = pytest.mark.gpu


def _gpu(tok, pr, N):
    import torch
    import paper_2605_00342_b200 as ev
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    g = ev.evict_build_draft_tree(cu(tok), cu(pr), N)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in g.items()}


def _compare(o, g):
    for k in ("parent", "tokens", "n_nodes"):
        assert (o[k] == g[k]).all(), k
    assert (o["q"].view(np.uint32) == g["q"].view(np.uint32)).all()
    assert (o["status"] == g["status"].astype(np.uint32)).all()


@pytest.mark.parametrize("steps,topk,N,B", [
    (4, 8, 32, 64),       # the paper's tree configuration, draft_tokens = 32
    (6, 10, 60, 300),     # C2 / C5 trees
    (8, 10, 128, 64),     # C4 trees
    (3, 16, 128, 40),     # topk 16, pool 545
    (1, 1, 8, 10),        # top-1 chain
    (9, 15, 128, 8),      # pool 1 + 15 + 8·225 = 1816 (near the 2048 limit)
    (2, 3, 100, 20),      # budget above the pool: no cut
    (6, 10, 60, 1500),    # ≥ 4·SMs trees: the warp-per-tree kernel (C2 shape)
    (4, 8, 32, 700),      # warp-per-tree, paper shape
    (3, 16, 128, 700),    # warp-per-tree, 256 candidates per step (8 keys per lane)
    (5, 2, 16, 800),      # warp-per-tree, tiny steps (1 key per lane)
])
def test_builder_matches_oracle(steps, topk, N, B):
    tok, pr = drafter_tables(steps * 100 + topk, B, steps, topk)
    _compare(od.build_draft_trees(tok, pr, steps, topk, N), _gpu(tok, pr, N))


def test_builder_ties_and_bad_probs():
    """Exact score ties (dyadic probabilities, many equal products) resolve by creation index;
    NaN / > 1 entries flag BAD_PROB for that tree only."""
    rng = np.random.default_rng(4)
    B, steps, topk, N = 50, 5, 6, 64
    tok, _ = drafter_tables(8, B, steps, topk)
    pr = (rng.integers(0, 5, size=(B, steps, topk, topk)) / 4.0).astype(np.float32)
    pr[3, 2, 1, 1] = np.nan
    pr[7, 0, 0, 2] = 1.25
    pr[9, 1, 4, 4] = -0.0
    o = od.build_draft_trees(tok, pr, steps, topk, N)
    assert o["status"][3] and o["status"][7] and not o["status"][9]
    _compare(o, _gpu(tok, pr, N))


def test_builder_feeds_select():
    """The built rows are a valid evict_select batch: GPU select on them equals the oracle's."""
    import torch
    import gen
    import oracle
    import paper_2605_00342_b200 as ev
    from oracle.parity import compare_select
    B, steps, topk, N = 128, 6, 10, 60
    tok, pr = drafter_tables(11, B, steps, topk)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    g = ev.evict_build_draft_tree(cu(tok), cu(pr), N)
    s = ev.evict_select(g["parent"], g["q"], cu(gen.cost_table(N)), n_nodes=g["n_nodes"], with_order=True)
    o_tree = od.build_draft_trees(tok, pr, steps, topk, N)
    o = oracle.select(o_tree["parent"], o_tree["q"], gen.cost_table(N), n_nodes=o_tree["n_nodes"])
    res, msgs = compare_select(o, {k: v.cpu().numpy() for k, v in s.items()}, n_nodes=o_tree["n_nodes"],
                               check_order=True)
    assert not msgs, msgs[:3]
