"""CUDA path vs oracle, element by element, through the C ABI (needs a B200).

Inputs are seeded (gen/) or hand-made adversarial trees; the oracle runs on the
same host arrays.  Bar: bit-exact integers; fp32 values within 1e-5 relative;
near-ties reported as ties (oracle/parity.py).
"""
import json
import os

import numpy as np
import pytest

import gen
import oracle
from oracle.parity import downstream_keep, compare_build, compare_select, compare_union

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "toy_tree.json")))


@pytest.fixture(scope="module")
def ev():
    import torch  # noqa: F401
    import paper_2605_00342_b200 as ev
    ev.lib()
    return ev


def T(a, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def npy(d):
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in d.items()}


def pad_batch(trees, N):
    B = len(trees)
    P = np.full((B, N), -1, np.int32)
    Q = np.zeros((B, N), np.float32)
    n = np.zeros(B, np.int32)
    for b, (p, q) in enumerate(trees):
        P[b, :len(p)] = p
        Q[b, :len(q)] = q
        n[b] = len(p)
    return P, Q, n


def adversarial(N, rng):
    out = []
    out.append((np.arange(-1, N - 1, dtype=np.int32), np.full(N, 0.9, np.float32)))        # chain
    out.append((np.array([-1] + [0] * (N - 1), np.int32), rng.uniform(0, 1, N).astype(np.float32)))  # star
    p = np.array([-1] + [int(rng.integers(0, i)) for i in range(1, N)], np.int32)
    out.append((p, np.ones(N, np.float32)))                                                  # q = 1 ties
    out.append((p, np.zeros(N, np.float32)))                                                 # q = 0
    q = np.full(N, 0.5, np.float32)
    q[1:] = rng.choice([0.5, 0.25, 1.0, 0.0, -0.0], N - 1)
    out.append((p, q))                                                                       # dyadic ties, -0
    out.append((np.arange(-1, N - 1, dtype=np.int32), np.full(N, 2.0 ** -10, np.float32)))  # subnormal chain
    for m in (1, 2, 3, N // 2, N - 1):
        pp = np.array([-1] + [int(rng.integers(0, i)) for i in range(1, m)], np.int32)
        out.append((pp, rng.uniform(0, 1, m).astype(np.float32)))                            # ragged n
    for _ in range(10):
        out.append((p, np.concatenate([[1], rng.choice([0.5, 0.25, 0.75, 1.0], N - 1)]).astype(np.float32)))
    for _ in range(10):
        out.append((p, rng.uniform(0, 1, N).astype(np.float32)))
    for q in out:
        q[1][0] = 1.0
    return out


def run_select(ev, P, Q, n, cost, cost_stride=0):
    g = ev.evict_select(T(P), T(Q), T(cost), n_nodes=T(n), cost_stride=cost_stride, with_order=True)
    return npy(g)


def check_select(o, g, n):
    res, msgs = compare_select(o, g, n_nodes=n, check_order=True)
    assert not msgs, msgs[:5]
    return res


# ------------------------------------------------------------------ select
def test_toy_tree(ev):
    P, Q, n = pad_batch([(np.array(GOLD["parent"], np.int32), np.array(GOLD["q"], np.float32))], 8)
    for cost in [GOLD["cost"]] + [v["cost"] for v in GOLD["cost_variants"].values()]:
        c = np.array(cost, np.float32)
        g = run_select(ev, P, Q, n, c)
        o = oracle.select(P, Q, c, n_nodes=n)
        check_select(o, g, n)
    g = run_select(ev, P, Q, n, np.array(GOLD["cost"], np.float32))
    assert g["k_star"][0] == 3 and int(g["keep_bits"][0, 0]) == 11
    assert g["order"][0].tolist() == GOLD["order"]
    assert g["e_hat"][0] == 2.125


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c4_60", "paper"])
def test_select_generated(ev, name):
    c = gen.CONFIGS[name]
    B = max(c["B"], 256)
    P, Q, n = gen.trees(c["seed"], B, c["N"], c["steps"], c["topk"])
    cost = gen.cost_table(c["N"])
    g = run_select(ev, P, Q, n, cost)
    o = oracle.select(P, Q, cost, n_nodes=n, threads=8)
    res = check_select(o, g, n)
    assert res["match"] + res["tie"] == B


@pytest.mark.parametrize("N", [4, 8, 32, 60, 64, 100, 128])
def test_select_adversarial(ev, N):
    rng = np.random.default_rng(N)
    trees = adversarial(N, rng)
    P, Q, n = pad_batch(trees, N)
    # per-tree cost tables: default, constant, linear, infeasible entries
    B = len(trees)
    C = np.tile(gen.cost_table(N), (B, 1))
    C[1::4] = 3.0
    C[2::4] = 0.37 * np.arange(1, N + 1)
    C[3::4, 2::3] = np.inf
    g = run_select(ev, P, Q, n, C.astype(np.float32), cost_stride=N)
    o = oracle.select(P, Q, C, n_nodes=n, cost_stride=N)
    check_select(o, g, n)


def test_select_invalid_inputs(ev):
    N = 8
    base_p = np.array([-1, 0, 0, 1, 1, 2, 3, 4], np.int32)
    base_q = np.array(GOLD["q"], np.float32)
    cases = []
    p = base_p.copy(); p[0] = 0; cases.append((p, base_q))
    p = base_p.copy(); p[5] = 5; cases.append((p, base_q))
    q = base_q.copy(); q[3] = 1.5; cases.append((base_p, q))
    q = base_q.copy(); q[3] = np.nan; cases.append((base_p, q))
    q = base_q.copy(); q[3] = -0.25; cases.append((base_p, q))
    cases.append((base_p, base_q))
    P, Q, n = pad_batch(cases, N)
    n = np.concatenate([n, [0, 9]]).astype(np.int32)
    P = np.concatenate([P, P[:2]])
    Q = np.concatenate([Q, Q[:2]])
    C = np.tile(np.array(GOLD["cost"], np.float32), (len(n), 1))
    g = run_select(ev, P, Q, n, C, cost_stride=N)
    o = oracle.select(P, Q, C, n_nodes=n, cost_stride=N)
    check_select(o, g, n)
    assert (g["status"][:5] != 0).all() and g["status"][5] == 0 and (g["status"][6:] == 1).all()
    # bad cost tables
    C2 = np.tile(np.array(GOLD["cost"], np.float32), (3, 1))
    C2[0, 4] = 0.0
    C2[1, 0] = np.inf
    C2[2, 7] = np.nan
    P3, Q3, n3 = pad_batch([(base_p, base_q)] * 3, N)
    g = run_select(ev, P3, Q3, n3, C2, cost_stride=N)
    assert (g["status"] == 8).all() and (g["k_star"] == 0).all()


def test_select_host_errors(ev):
    import torch
    P = torch.zeros((2, 6), dtype=torch.int32, device="cuda")           # N % 4 != 0
    Q = torch.zeros((2, 6), dtype=torch.float32, device="cuda")
    with pytest.raises(ev.EvictError) as e:
        ev.evict_select(P, Q, torch.ones(6, device="cuda"))
    assert e.value.code == ev.EVICT_ERR_INVALID_ARG


# ------------------------------------------------------------------ build
@pytest.mark.parametrize("name", ["c2", "c4", "c4_60"])
def test_build_generated(ev, name):
    c = gen.CONFIGS[name]
    B = max(c["B"], 300)
    P, Q, n = gen.trees(c["seed"] + 1, B, c["N"], c["steps"], c["topk"])
    o = oracle.select(P, Q, gen.cost_table(c["N"]), n_nodes=n)
    keep = o["keep_bits"]
    pos = np.arange(B, dtype=np.int32) * 3 + 100
    ob = oracle.build_verify_tree(P, keep, n_nodes=n, pos_offset=pos)
    gb = npy(ev.evict_build_verify_tree(T(P), T(keep.view(np.int64)), n_nodes=T(n), pos_offset=T(pos)))
    assert not compare_build(ob, gb)


@pytest.mark.parametrize("N", [8, 60, 128])
def test_build_adversarial_keep_sets(ev, N):
    rng = np.random.default_rng(N + 7)
    trees = adversarial(N, rng)
    P, Q, n = pad_batch(trees, N)
    B = len(trees)
    W = (N + 63) // 64
    keep = np.zeros((B, W), np.uint64)
    for b in range(B):
        nb = int(n[b])
        mode = b % 4
        if mode == 0:
            kept = range(nb)                                   # full tree
        elif mode == 1:
            kept = [0]
        elif mode == 2:                                        # random ancestor-closed
            s = {0}
            for v in range(1, nb):
                if P[b, v] in s and rng.uniform() < 0.6:
                    s.add(v)
            kept = sorted(s)
        else:                                                  # invalid: child without parent
            kept = [0] + ([nb - 1] if nb > 2 and P[b, nb - 1] != 0 else [])
        for v in kept:
            keep[b, v // 64] |= np.uint64(1 << (v % 64))
    ob = oracle.build_verify_tree(P, keep, n_nodes=n)
    gb = npy(ev.evict_build_verify_tree(T(P), T(keep.view(np.int64)), n_nodes=T(n)))
    assert not compare_build(ob, gb)


def test_build_large_batch_offsets(ev):
    """Decoupled look-back across many tiles and persistent CTAs."""
    B, N = 50_000, 60
    P, Q, n = gen.trees(77, B, N, 6, 10)
    o = oracle.select(P, Q, gen.cost_table(N), n_nodes=n, threads=8)
    ob = oracle.build_verify_tree(P, o["keep_bits"], n_nodes=n)
    gb = npy(ev.evict_build_verify_tree(T(P), T(o["keep_bits"].view(np.int64)), n_nodes=T(n)))
    assert not compare_build(ob, gb)


# ------------------------------------------------------------------ union
@pytest.mark.parametrize("fmt", ["u8", "i32", "mask"])
@pytest.mark.parametrize("shape", [(60, 48, 128, 8), (60, 94, 128, 8), (128, 48, 256, 8),
                                   (8, 2, 8, 2), (60, 5, 64, 3), (32, 33, 200, 6)])
def test_union(ev, fmt, shape):
    N, L, E, K = shape
    if fmt == "u8" and E > 256:
        pytest.skip()
    B = 80
    steps, topk = (6, 10) if N >= 32 else (3, 2)
    P, Q, n = gen.trees(5, B, N, steps, topk)
    o = oracle.select(P, Q, gen.cost_table(N), n_nodes=n)
    ids = gen.routing(9, B, N, L, E, K, dtype=np.uint8 if fmt == "u8" else np.int32)
    ou = oracle.expert_union(o["keep_bits"], ids, E, n_nodes=n)
    if fmt == "mask":
        dev_ids = T(gen.ids_to_mask(ids, E).view(np.int64))
    else:
        dev_ids = T(ids)
    gu = npy(ev.evict_expert_union(T(o["keep_bits"].view(np.int64)), dev_ids, E, n_nodes=T(n)))
    assert not compare_union(ou, gu)


def test_union_bad_expert_and_hist(ev):
    import torch
    B, N, L, E, K = 16, 8, 3, 16, 2
    ids = np.zeros((B, N, L, K), np.int32)
    rng = np.random.default_rng(0)
    for b in range(B):
        for v in range(N):
            for l in range(L):
                ids[b, v, l] = rng.permutation(E)[:K]
    ids[3, 0, 1, 0] = 99                      # kept root: bad
    ids[4, 7, 1, 0] = 99                      # pruned node: ignored
    keep = np.full((B, 1), 0b0111_1111, np.uint64)
    ou = oracle.expert_union(keep, ids, E)
    hist = torch.zeros((L, E), dtype=torch.int64, device="cuda")
    gu = npy(ev.evict_expert_union(T(keep.view(np.int64)), T(ids), E, expert_hist=hist))
    assert not compare_union(ou, gu)
    assert gu["status"][3] == 0x10 and gu["status"][4] == 0
    h = np.zeros((L, E), np.int64)
    for b in range(B):
        if ou["status"][b]:
            continue
        for l in range(L):
            for e in range(E):
                if (int(ou["union_bits"][b, l, 0]) >> e) & 1:
                    h[l, e] += 1
    assert (hist.cpu().numpy() == h).all()


# ------------------------------------------------------------------ fused
def _cfg(name):
    """BASELINE configs, plus c2 trees with 56 layers: L·2 = 112 id slots runs the R = 4 register
    rounds of k_fused (L ≤ 48: R = 3; C3's 94 layers: R = 8, two flag passes)."""
    if name == "c2_l56":
        return dict(gen.CONFIGS["c2"], L=56)
    return gen.CONFIGS[name]


@pytest.mark.parametrize("with_order", [True, False])
@pytest.mark.parametrize("name,fmt", [("c2", "u8"), ("c4", "u8"), ("c4_60", "i32"),
                                      ("c4_60", "mask"), ("paper", "u8"), ("ling", "u8"), ("ling", "mask"),
                                      ("c3", "u8"), ("c3", "i32"), ("c3", "mask"), ("c2_l56", "u8"),
                                      ("c2_l56", "i32"), ("c2_l56", "mask")])
def test_fused_equals_oracle(ev, name, fmt, with_order):
    c = _cfg(name)
    B = 333
    N, L, E, K = c["N"], c["L"], c["E"], c["K"]
    P, Q, n = gen.trees(c["seed"] + 11, B, N, c["steps"], c["topk"])
    n[::7] = np.maximum(1, n[::7] // 2)                     # ragged
    cost = gen.cost_table(N)
    ids = gen.routing(c["seed"], B, N, L, E, K, dtype=np.int32 if fmt == "i32" else np.uint8)
    dev_ids = T(gen.ids_to_mask(ids, E).view(np.int64)) if fmt == "mask" else T(ids)
    pos = np.full(B, 5, np.int32)
    g = npy(ev.evict_select_build_union(T(P), T(Q), T(cost), dev_ids, E, n_nodes=T(n),
                                        pos_offset=T(pos), with_bits=True, with_order=with_order))
    o = oracle.select(P, Q, cost, n_nodes=n, threads=8)
    res, msgs = compare_select(o, g, n_nodes=n, check_order=with_order)
    assert not msgs, msgs[:5]
    keep = downstream_keep(o, g)
    ob = oracle.build_verify_tree(P, keep, n_nodes=n, pos_offset=pos)
    assert not compare_build(ob, {k: v for k, v in g.items() if k != "status"})
    ou = oracle.expert_union(keep, ids, E, n_nodes=n, threads=8)
    assert not compare_union(ou, g)


# ------------------------------------------------------------------ stats
def test_batch_stats(ev):
    """Both sides aggregate the same per-tree inputs, produced by the oracle (select + union)."""
    B, N, L, E, K = 5000, 60, 48, 128, 8
    P, Q, n = gen.trees(3, B, N, 6, 10)
    Q[17, 5] = 2.0                                           # one bad tree
    cost = gen.cost_table(N)
    ids = gen.routing(3, B, N, L, E, K)
    o = oracle.select(P, Q, cost, n_nodes=n, threads=8)
    u = oracle.expert_union(o["keep_bits"], ids, E, n_nodes=n, threads=8)
    e_hat = o["e_hat"].astype(np.float32)                    # the kernel's input precision
    util = o["utility"].astype(np.float32)
    s, d = ev.evict_batch_stats(T(o["k_star"]), T(e_hat), T(util), T(u["union_count"]),
                                T(o["status"].view(np.int32)), N, n_nodes=T(n))
    so, do = oracle.batch_stats(N, L, o["k_star"], e_hat.astype(np.float64), util.astype(np.float64),
                                u["union_count"], o["status"], n_nodes=n)
    assert (s.cpu().numpy() == so).all()
    assert np.allclose(d.cpu().numpy(), do, rtol=1e-9)
    assert so[4] == 1


@pytest.mark.parametrize("with_order", [True, False])
@pytest.mark.parametrize("N,steps", [(60, 6), (128, 8)])
def test_select_large_batch_grouped_kernel(ev, N, steps, with_order):
    """B > 4096 takes the sub-warp (grouped) select kernel; ragged trees and a few adversarial rows."""
    B = 6000
    P, Q, n = gen.trees(91, B, N, steps, 10)
    rng = np.random.default_rng(N)
    n[::5] = np.maximum(1, (n[::5] * rng.uniform(0.1, 1.0, len(n[::5]))).astype(np.int32))
    Q[7, 1:] = 1.0                                        # q = 1 ties
    Q[8, 3] = np.nan                                      # bad prob
    C = np.tile(gen.cost_table(N), (B, 1))
    C[9::50, 2::3] = np.inf
    g = npy(ev.evict_select(T(P), T(Q), T(C.astype(np.float32)), n_nodes=T(n), cost_stride=N,
                            with_order=with_order))
    o = oracle.select(P, Q, C, n_nodes=n, cost_stride=N, threads=8)
    res, msgs = compare_select(o, g, n_nodes=n, check_order=with_order)
    assert not msgs, msgs[:5]


@pytest.mark.parametrize("N", [8, 60, 64, 100, 128])
def test_select_values_path_ties(ev, N):
    """Without the order row the grouped kernels sort score values and rebuild the kept set from
    the k*-th score (ties by index): tie-heavy adversarial trees, tiled past the grouped-kernel
    threshold, must give the ranking path's k*, keep bits, ê and utility bit for bit."""
    rng = np.random.default_rng(100 + N)
    trees = adversarial(N, rng)
    P, Q, n = pad_batch(trees, N)
    reps = 4200 // len(trees) + 1
    P, Q, n = np.tile(P, (reps, 1)), np.tile(Q, (reps, 1)), np.tile(n, reps)
    B = len(n)
    C = np.tile(gen.cost_table(N), (B, 1))
    C[1::4] = 3.0                                          # constant cost: keep everything
    C[2::4] = 0.37 * np.arange(1, N + 1)
    C[3::4, 2::3] = np.inf
    C = C.astype(np.float32)
    a = npy(ev.evict_select(T(P), T(Q), T(C), n_nodes=T(n), cost_stride=N, with_order=True))
    v = npy(ev.evict_select(T(P), T(Q), T(C), n_nodes=T(n), cost_stride=N, with_order=False))
    for key in ("k_star", "keep_bits", "status"):
        assert (a[key] == v[key]).all(), key
    for key in ("e_hat", "utility"):
        assert (a[key].view(np.uint32) == v[key].view(np.uint32)).all(), key
    o = oracle.select(P[:len(trees)], Q[:len(trees)], C[:len(trees)], n_nodes=n[:len(trees)],
                      cost_stride=N)
    res, msgs = compare_select(o, {k: x[:len(trees)] for k, x in v.items()}, n_nodes=n[:len(trees)])
    assert not msgs, msgs[:5]


# ------------------------------------------------------------------ policies (NEXT-2)
POLICIES = [("coverage", 0.7), ("coverage", 0.4), ("coverage", 1.0), ("fixed", 1), ("fixed", 5),
            ("fixed", 500)]


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("B,with_order", [(300, True), (300, False), (5000, True), (5000, False)])
def test_select_policy_vs_oracle(ev, policy, B, with_order):
    """Score-coverage and fixed-k cuts on the same ranking: warp kernel
    (B ≤ 4096) and grouped kernels (B > 4096, value-sort path without the order row)."""
    rng = np.random.default_rng(B + len(policy[0]))
    N = 60
    P, Q, n = gen.trees(77, B, N, 6, 10)
    n[::6] = np.maximum(1, (n[::6] * rng.uniform(0.1, 1.0, len(n[::6]))).astype(np.int32))
    adv = adversarial(N, rng)
    Pa, Qa, na = pad_batch(adv, N)
    P[:len(adv)], Q[:len(adv)], n[:len(adv)] = Pa, Qa, na     # ties, zero and subnormal scores
    cost = gen.cost_table(N)
    g = npy(ev.evict_select(T(P), T(Q), T(cost), n_nodes=T(n), with_order=with_order, policy=policy))
    o = oracle.select(P, Q, cost, n_nodes=n, threads=8, policy=policy)
    res, msgs = compare_select(o, g, n_nodes=n, check_order=with_order)
    assert not msgs, msgs[:5]


@pytest.mark.parametrize("policy", [("coverage", 0.7), ("fixed", 6)])
@pytest.mark.parametrize("with_order", [True, False])
def test_fused_policy_vs_oracle(ev, policy, with_order):
    c = gen.CONFIGS["c2"]
    B, N, L, E, K = 333, c["N"], c["L"], c["E"], c["K"]
    P, Q, n = gen.trees(c["seed"] + 5, B, N, c["steps"], c["topk"])
    cost = gen.cost_table(N)
    ids = gen.routing(c["seed"], B, N, L, E, K)
    g = npy(ev.evict_select_build_union(T(P), T(Q), T(cost), T(ids), E, n_nodes=T(n), policy=policy,
                                        with_bits=True, with_order=with_order))
    o = oracle.select(P, Q, cost, n_nodes=n, threads=8, policy=policy)
    res, msgs = compare_select(o, g, n_nodes=n, check_order=with_order)
    assert not msgs, msgs[:5]
    keep = downstream_keep(o, g)
    assert not compare_build(oracle.build_verify_tree(P, keep, n_nodes=n),
                             {k: v for k, v in g.items() if k != "status"})
    assert not compare_union(oracle.expert_union(keep, ids, E, n_nodes=n, threads=8), g)


def test_policy_rejects_bad_arguments(ev):
    import torch
    P = torch.full((2, 8), -1, dtype=torch.int32, device="cuda")
    P[:, 1:] = 0
    Q = torch.full((2, 8), 0.5, device="cuda")
    C = torch.ones(8, device="cuda")
    for bad in (("coverage", 0.0), ("coverage", 1.5), ("coverage", float("nan")), ("fixed", 0)):
        with pytest.raises(ev.EvictError):
            ev.evict_select(P, Q, C, policy=bad)


@pytest.mark.parametrize("B", [1, 64, 777, 5000])
@pytest.mark.parametrize("name", ["c2", "ling", "c3", "c2_l56"])
def test_fused_lean_path(ev, name, B):
    """The serving configuration (u8 top-8 ids, no order row, no bit rows, no histogram) runs the
    LEAN instantiation with marker-epoch flag blocks — E = 128 and the 256-expert layout; C3's
    94 layers (R = 8: two flag passes, no marker epochs) and 56 layers (R = 4).  Batches up to
    2048 take one-tree warp tiles (serving latency), larger ones 4-tree tiles."""
    c = _cfg(name)
    N, L, E, K = c["N"], c["L"], c["E"], c["K"]
    P, Q, n = gen.trees(c["seed"] + 3, B, N, c["steps"], c["topk"])
    n[::5] = np.maximum(1, n[::5] // 3)
    cost = gen.cost_table(N)
    ids = gen.routing(c["seed"] + 1, B, N, L, E, K)
    g = npy(ev.evict_select_build_union(T(P), T(Q), T(cost), T(ids), E, n_nodes=T(n)))
    o = oracle.select(P, Q, cost, n_nodes=n, threads=8)
    res, msgs = compare_select(o, g, n_nodes=n)
    assert not msgs, msgs[:5]
    keep = downstream_keep(o, g)
    ou = oracle.expert_union(keep, ids, E, n_nodes=n, threads=8)
    assert not compare_union(ou, {k: v for k, v in g.items() if k in ("union_count", "union_total")})
    ob = oracle.build_verify_tree(P, keep, n_nodes=n)
    assert not compare_build(ob, {k: v for k, v in g.items() if k != "status"})


@pytest.mark.parametrize("name,fmt,B", [("c2", "u8", 777), ("c2", "u8", 5000), ("c2_l56", "u8", 3000),
                                        ("c3", "u8", 500), ("c4_60", "i32", 300), ("ling", "u8", 300),
                                        ("c4", "u8", 2100)])
def test_fused_stats(ev, name, fmt, B):
    """A9 statistics written by the fused call (ABI 8): folded into the launch for the E = 128,
    L ≤ 64 serving union, the statistics kernel after it otherwise.  They must equal the oracle's
    batch_stats over the call's own outputs (integers exact), errored trees included (NaN q,
    an expert id ≥ E in a kept row)."""
    c = _cfg(name)
    N, L, E, K = c["N"], c["L"], c["E"], c["K"]
    P, Q, n = gen.trees(c["seed"] + 5, B, N, c["steps"], c["topk"])
    Q = Q.copy()
    Q[3, 1] = np.nan                                      # BAD_PROB
    ids = gen.routing(c["seed"] + 2, B, N, L, E, K, dtype=np.int32 if fmt == "i32" else np.uint8)
    if E < 256:
        ids[7, 0, 2, 1] = E + 3 if E + 3 < 256 else 255     # root is always kept: BAD_EXPERT
    g = npy(ev.evict_select_build_union(T(P), T(Q), T(gen.cost_table(N)), T(ids), E, n_nodes=T(n),
                                        with_stats=True))
    assert g["status"][3] != 0 and (E == 256 or g["status"][7] != 0)
    s, d = oracle.batch_stats(N, L, g["k_star"], g["e_hat"].astype(np.float64), g["utility"].astype(np.float64),
                              g["union_count"], g["status"].astype(np.uint32), n_nodes=n)
    assert (g["stats"] == s).all(), np.flatnonzero(g["stats"] != s)[:5]
    assert np.allclose(g["dstats"], d, rtol=1e-9)


@pytest.mark.parametrize("B", [300, 4000])
def test_fused_reads_pinned_host_routing(ev, B):
    """Routing ids in page-locked host memory (mapped, zero-copy): the fused call reads only the
    kept rows over PCIe and must produce exactly the outputs of the device-resident call."""
    import torch
    c = gen.CONFIGS["c2"]
    N, L, E, K = c["N"], c["L"], c["E"], c["K"]
    P, Q, n = gen.trees(c["seed"] + 9, B, N, c["steps"], c["topk"])
    ids = gen.routing(c["seed"] + 9, B, N, L, E, K)
    host = torch.from_numpy(ids).pin_memory()
    cost = T(gen.cost_table(N))
    a = npy(ev.evict_select_build_union(T(P), T(Q), cost, T(ids), E, n_nodes=T(n)))
    b = npy(ev.evict_select_build_union(T(P), T(Q), cost, host, E, n_nodes=T(n)))
    torch.cuda.synchronize()
    for k in ("k_star", "keep_bits", "union_count", "union_total", "status", "verify_offsets"):
        assert (a[k] == b[k]).all(), k


@pytest.mark.parametrize("L,policy", [(7, None), (20, ("fixed", 45)), (32, None), (33, ("fixed", 40)),
                                      (40, None), (48, ("fixed", 50)), (48, ("coverage", 0.9)),
                                      (56, None), (64, ("fixed", 45))])
def test_throughput_union_emit_modes(ev, L, policy):
    """The throughput path's union/emit kernel (k_fused PRE with tree_union_cols; B > 2048, u8
    top-8, E = 128, N ≤ 64) over its flag-column layouts (L ≤ 48: region 1 in half-layer columns,
    empty for L ≤ 32; L ≤ 64: layer columns), ragged trees, kept sets reaching nodes ≥ 32 and
    k > 16 (fixed k / coverage policies: the emit's child-mask path), an errored tree (NaN q) and a
    BAD_EXPERT row; A9 statistics folded into the launch must equal the oracle's batch_stats over
    the call's own outputs."""
    c = gen.CONFIGS["c2"]
    B, N, E, K = 4500, c["N"], 128, 8
    P, Q, n = gen.trees(c["seed"] + L, B, N, c["steps"], c["topk"])
    n[::5] = np.maximum(1, n[::5] // 3)
    Q = Q.copy()
    Q[11, 1] = np.nan                                     # BAD_PROB
    cost = gen.cost_table(N)
    ids = gen.routing(c["seed"] + L, B, N, L, E, K)
    ids[29, 0, L - 1, 5] = 200                            # root is always kept: BAD_EXPERT
    g = npy(ev.evict_select_build_union(T(P), T(Q), T(cost), T(ids), E, n_nodes=T(n), policy=policy,
                                        with_stats=True))
    assert g["status"][11] != 0 and g["status"][29] == 0x10
    o = oracle.select(P, Q, cost, n_nodes=n, threads=8, policy=policy)
    res, msgs = compare_select(o, dict(g, status=g["status"] & ~np.uint32(0x10)), n_nodes=n)
    assert not msgs, msgs[:5]
    keep = downstream_keep(o, g)
    if policy is not None and policy[0] == "fixed":
        assert (g["k_star"] > 32).sum() > 100            # the emit's second half is exercised
    ou = oracle.expert_union(keep, ids, E, n_nodes=n, threads=8)
    assert not compare_union(ou, {k: v for k, v in g.items() if k in ("union_count", "union_total")})
    ob = oracle.build_verify_tree(P, keep, n_nodes=n)
    assert not compare_build(ob, {k: v for k, v in g.items() if k != "status"})
    s, d = oracle.batch_stats(N, L, g["k_star"], g["e_hat"].astype(np.float64), g["utility"].astype(np.float64),
                              g["union_count"], g["status"].astype(np.uint32), n_nodes=n)
    assert (g["stats"] == s).all(), np.flatnonzero(g["stats"] != s)[:5]
    assert np.allclose(g["dstats"], d, rtol=1e-9)
