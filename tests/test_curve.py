"""NEXT-1: the prefix-union curve along the ranking and the offline cost profile on the GPU,
against the oracle (tests/test_oracle_pins.py pins the oracle)."""
import numpy as np
import pytest

import gen
import oracle
from oracle.parity import compare_select

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ev():
    import paper_2605_00342_b200 as ev
    return ev


def T(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("fmt", ["u8", "i32", "mask"])
@pytest.mark.parametrize("name", ["c2", "c4", "toy_like", "ling"])
def test_union_curve_matches_oracle(ev, fmt, name):
    if name == "toy_like":
        B, N, steps, topk, L, E, K = 50, 8, 3, 2, 2, 8, 2
    elif name == "ling":                  # Ling-flash-2.0: 256 experts, top-8
        B, N, steps, topk, L, E, K = 120, 60, 6, 10, 32, 256, 8
    else:
        c = gen.CONFIGS[name]
        B, N, steps, topk, L, E, K = 120, c["N"], c["steps"], c["topk"], c["L"], c["E"], c["K"]
    P, Q, n = gen.trees(41, B, N, steps, topk)
    n[::9] = np.maximum(1, n[::9] // 3)
    ids = gen.routing(42, B, N, L, E, K, dtype=np.int32 if fmt == "i32" else np.uint8)
    order = oracle.select(P, Q, gen.cost_table(N), n_nodes=n, threads=8)["order"]   # the oracle's ranking
    dev_ids = T(gen.ids_to_mask(ids, E).view(np.int64)) if fmt == "mask" else T(ids)
    g = ev.evict_union_curve(T(order), dev_ids, E, n_nodes=T(n), per_layer=True)
    o = oracle.union_curve(order, ids.astype(np.uint8) if fmt != "i32" else ids, E,
                           n_nodes=n, threads=8)
    assert (g["status"].cpu().numpy() == o["status"].astype(np.int32)).all()
    assert (g["curve"].cpu().numpy() == o["curve"]).all()
    assert (g["curve_layer"].cpu().numpy() == o["curve_layer"]).all()


def test_union_curve_errors(ev):
    import torch
    B, N, L, E, K = 4, 8, 2, 8, 2
    P, Q, n = gen.trees(5, B, N, 3, 2)
    ids = gen.routing(6, B, N, L, E, K)
    order = oracle.select(P, Q, gen.cost_table(N), n_nodes=n)["order"].copy()
    order[1, 0] = 99                      # not a node of tree 1
    bad = ids.copy()
    bad[2, :, 0, 0] = 200                 # id ≥ E in every node of tree 2
    g = ev.evict_union_curve(T(order), T(bad), E, n_nodes=T(n), per_layer=True)
    o = oracle.union_curve(order, bad, E, n_nodes=n)
    assert (g["status"].cpu().numpy() == o["status"].astype(np.int32)).all()
    assert o["status"][1] and o["status"][2]
    assert (g["curve"].cpu().numpy() == o["curve"]).all()
    assert (g["curve_layer"].cpu().numpy() == o["curve_layer"]).all()


def test_profile_cost_matches_oracle_and_feeds_select(ev):
    """C(k) from the measured curves equals the oracle's fp64 value rounded to fp32 (≤ 1 ulp) and
    is a valid cost table for evict_select (the profiled table closes the NEXT-1 loop)."""
    c = gen.CONFIGS["c4"]
    B, N, L, E, K = 64, c["N"], c["L"], c["E"], c["K"]
    P, Q, n = gen.trees(8, B, N, c["steps"], c["topk"])
    ids = gen.routing(9, B, N, L, E, K)
    sel = ev.evict_select(T(P), T(Q), T(gen.cost_table(N)), n_nodes=T(n), with_order=True)
    g = ev.evict_union_curve(sel["order"], T(ids), E, n_nodes=T(n))
    cost = ev.evict_profile_cost(g["curve"], L, n_nodes=T(n), status=g["status"]).cpu().numpy()
    osel = oracle.select(P, Q, gen.cost_table(N), n_nodes=n, threads=8)           # oracle chain end to end
    ocur = oracle.union_curve(osel["order"], ids, E, n_nodes=n, threads=8, per_layer=False)
    oc = oracle.profile_cost(ocur["curve"], L, n_nodes=n, status=ocur["status"])
    fin = np.isfinite(oc)
    assert (np.isfinite(cost) == fin).all()
    assert np.allclose(cost[fin], oc[fin].astype(np.float32), rtol=2 ** -23, atol=0)
    s2 = ev.evict_select(T(P), T(Q), T(cost), n_nodes=T(n), with_order=True)
    o2 = oracle.select(P, Q, oc.astype(np.float32), n_nodes=n, threads=8)
    res, msgs = compare_select(o2, {k: v.cpu().numpy() for k, v in s2.items()}, n_nodes=n, check_order=True)
    assert not msgs, msgs[:3]
