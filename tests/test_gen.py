"""The seeded workload generator: shape properties (CPU) and host == device (GPU)."""
import numpy as np
import pytest

import gen


def test_trees_are_valid_eagle_shapes():
    for name in ("c2", "c4", "paper"):
        c = gen.CONFIGS[name]
        p, q, n = gen.trees(c["seed"], 64, c["N"], c["steps"], c["topk"])
        assert (n == c["N"]).all()
        assert (p[:, 0] == -1).all()
        idx = np.arange(c["N"])
        assert ((p[:, 1:] >= 0) & (p[:, 1:] < idx[None, 1:])).all()      # topological
        assert (q[:, 1:] > 0).all() and (q[:, 1:] < 1).all()
        # depth ≤ steps
        depth = np.zeros_like(p)
        for i in range(1, c["N"]):
            depth[:, i] = depth[np.arange(64), p[:, i]] + 1
        assert depth.max() <= c["steps"]


def test_trees_deterministic_and_counter_based():
    a = gen.trees(5, 10, 60, 6, 10, tree_base=100)
    b = gen.trees(5, 20, 60, 6, 10, tree_base=90)
    for x, y in zip(a, b):
        assert (x == y[10:]).all()                  # tree t depends only on (seed, t)
    c = gen.trees(6, 10, 60, 6, 10, tree_base=100)
    assert not (a[1] == c[1]).all()


def test_routing_rows_are_topk_sets():
    ids = gen.routing(5, 4, 60, 48, 128, 8, tree_base=7)
    assert ids.dtype == np.uint8 and ids.max() < 128
    s = np.sort(ids, axis=-1)
    assert (np.diff(s.astype(int), axis=-1) > 0).all()       # K distinct experts per row
    i32 = gen.routing(5, 4, 60, 48, 128, 8, tree_base=7, dtype=np.int32)
    assert (i32 == ids).all()


def test_routing_union_calibration():
    """σ_b = 2.25 targets union(8)/union(32) ≈ 0.68 ≈ 1 − 32.5%."""
    ids = gen.routing(5, 200, 32, 8, 128, 8)
    u8 = np.mean([[len(set(ids[b, :8, l].ravel())) for l in range(8)] for b in range(200)])
    u32 = np.mean([[len(set(ids[b, :32, l].ravel())) for l in range(8)] for b in range(200)])
    assert 0.6 < u8 / u32 < 0.76, u8 / u32


def test_cost_table_calibration():
    """Default C(k) reproduces the paper's −74.7% verified tokens at the paper's
    tree shape steps=4, topk=8, draft_tokens=32: mean k* ≈ 8.1 of 32."""
    import oracle
    c = gen.cost_table(32)
    assert c.dtype == np.float32 and len(c) == 32 and (np.diff(c) > 0).all()
    p, q, n = gen.trees(7, 2000, 32, 4, 8)
    ks = oracle.select(p, q, c, threads=4)["k_star"]
    assert 6.5 < ks.mean() < 9.5, ks.mean()


def test_hidden_and_wgate_integer_mode():
    h = gen.hidden(3, 2, 8, 2, 64)
    w = gen.wgate(3, 2, 8, 64)
    vals = {0x0000, 0x3F80, 0x4000, 0xBF80, 0xC000}
    assert set(np.unique(h).tolist()) <= vals and set(np.unique(w).tolist()) <= vals


@pytest.mark.gpu
def test_device_generator_matches_host():
    import torch
    c = gen.CONFIGS["c2"]
    p, q, n = gen.trees(11, 300, 60, 6, 10, tree_base=12345)
    tp, tq, tn = gen.trees_cuda(11, 300, 60, 6, 10, tree_base=12345)
    assert (tp.cpu().numpy() == p).all() and (tn.cpu().numpy() == n).all()
    assert (tq.cpu().numpy().view(np.uint32) == q.view(np.uint32)).all()
    ids = gen.routing(11, 5, 60, 48, 128, 8, tree_base=999)
    tids = gen.routing_cuda(11, 5, 60, 48, 128, 8, tree_base=999)
    assert (tids.cpu().numpy() == ids).all()
    h = gen.hidden(3, 2, 16, 3, 128, mode=1, tree_base=4)
    th = gen.hidden_cuda(3, 2, 16, 3, 128, mode=1, tree_base=4)
    assert (th.view(torch.int16).cpu().numpy().view(np.uint16) == h).all()
    w = gen.wgate(3, 2, 128, 128, mode=1, scale_log2=-5)
    tw = gen.wgate_cuda(3, 2, 128, 128, mode=1, scale_log2=-5)
    assert (tw.view(torch.int16).cpu().numpy().view(np.uint16) == w).all()


def test_tree_shape_guard():
    """Draft-tree shapes whose candidate pool (topk + (steps − 1)·topk²) exceeds the generator's
    fixed scratch are rejected before any C code runs (8 steps × topk 16 = 1808 > 1024 once
    corrupted the host heap); the benchmark shapes fit."""
    import pytest
    with pytest.raises(ValueError):
        gen.trees(4, 2, 128, 8, 16)
    with pytest.raises(ValueError):
        gen.trees(4, 2, 60, 2, 17)
    for steps, topk in ((6, 10), (8, 10), (1, 16)):
        gen.check_tree_shape(steps, topk)
    P, Q, n = gen.trees(4, 2, 128, 8, 10)
    assert P.shape == (2, 128) and (n >= 1).all()
