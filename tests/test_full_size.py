"""Full-size parity: the C5 sweep (1,000,000 trees, u8 routing, device-generated) in the exact
launch configuration bench.py times, checked on sampled tree blocks against the oracle run on
host-regenerated inputs (the generator is counter-based, so any tree id can be rebuilt)."""
import numpy as np
import pytest

import gen
import oracle
from oracle.parity import downstream_keep, compare_build, compare_select, compare_union

pytestmark = pytest.mark.gpu

M, N, STEPS, TOPK, L, E, K, SEED = 1_000_000, 60, 6, 10, 48, 128, 8, 5


@pytest.fixture(scope="module")
def sweep():
    import torch
    import paper_2605_00342_b200 as ev
    P, Q, n = gen.trees_cuda(SEED, M, N, STEPS, TOPK)
    ids = gen.routing_cuda(SEED, M, N, L, E, K)
    cost = torch.from_numpy(gen.cost_table(N)).cuda()
    bench_call = ev.FusedCall(P, Q, cost, ids, E, n_nodes=n)             # bench.py's exact call
    bench_out = {k: v.clone() for k, v in bench_call().items()}
    del bench_call
    call = ev.FusedCall(P, Q, cost, ids, E, n_nodes=n, with_bits=True)   # + union bits
    out = call()
    torch.cuda.synchronize()
    yield dict(P=P, Q=Q, n=n, ids=ids, out=out, ev=ev, bench_out=bench_out)


def test_bench_config_equals_bits_config(sweep):
    a, b = sweep["bench_out"], sweep["out"]
    for k in ("k_star", "keep_bits", "union_count", "union_total", "verify_offsets", "status"):
        assert (a[k] == b[k]).all(), k
    T = int(a["verify_offsets"][-1])
    for k in ("kept_index", "retrieve_index", "positions", "next_token", "next_sibling", "tree_mask"):
        assert (a[k][:T] == b[k][:T]).all(), k


@pytest.mark.parametrize("block", [0, 1, 2, 3])
def test_sampled_blocks_match_oracle(sweep, block):
    rng = np.random.default_rng(block)
    B = 512
    lo = 0 if block == 0 else (M - B if block == 3 else int(rng.integers(0, M - B)))
    P, Q, n = gen.trees(SEED, B, N, STEPS, TOPK, tree_base=lo)
    ids = gen.routing(SEED, B, N, L, E, K, tree_base=lo)
    # device inputs are the same seeded inputs
    assert (sweep["P"][lo:lo + B].cpu().numpy() == P).all()
    assert (sweep["Q"][lo:lo + B].cpu().numpy().view(np.uint32) == Q.view(np.uint32)).all()
    assert (sweep["ids"][lo:lo + B].cpu().numpy() == ids).all()
    out = sweep["out"]
    g = {k: v[lo:lo + B].cpu().numpy() for k, v in out.items()
         if k in ("k_star", "e_hat", "utility", "keep_bits", "status", "union_count", "union_total",
                  "union_bits")}
    o = oracle.select(P, Q, gen.cost_table(N), n_nodes=n, threads=8)
    res, msgs = compare_select(o, g, n_nodes=n)
    assert not msgs, msgs[:3]
    keep = downstream_keep(o, g)
    assert not compare_union(oracle.expert_union(keep, ids, E, n_nodes=n, threads=8), g)
    # packed verify rows of the block, relative to the block's first offset
    off = out["verify_offsets"][lo:lo + B + 1].cpu().numpy().astype(np.int64)
    r0, r1 = int(off[0]), int(off[-1])
    gb = {k: out[k][r0:r1].cpu().numpy() for k in
          ("kept_index", "retrieve_index", "positions", "next_token", "next_sibling", "tree_mask")}
    gb["verify_offsets"] = (off - off[0]).astype(np.int32)
    gb["retrieve_index"] = gb["retrieve_index"] - lo * N
    ob = oracle.build_verify_tree(P, keep, n_nodes=n)
    assert not compare_build(ob, gb)


def test_offsets_cover_every_tree(sweep):
    out = sweep["out"]
    off = out["verify_offsets"].cpu().numpy().astype(np.int64)
    k = out["k_star"].cpu().numpy().astype(np.int64)
    assert off[0] == 0 and (np.diff(off) == k).all()


def test_stats_match_host_sums(sweep):
    import torch
    ev, out = sweep["ev"], sweep["out"]
    s, d = ev.evict_batch_stats(out["k_star"], out["e_hat"], out["utility"], out["union_count"],
                                out["status"], N, n_nodes=sweep["n"])
    s = s.cpu().numpy()
    k = out["k_star"].cpu().numpy().astype(np.int64)
    uc = out["union_count"].cpu().numpy().astype(np.int64)
    assert s[0] == M and s[4] == 0 and s[1] == k.sum() and s[3] == uc.sum()
    assert (s[6 + N:] == uc.sum(0)).all()
    assert (s[5:6 + N] == np.bincount(k, minlength=N + 1)).all()


def test_all_trees_match_oracle(sweep):
    """Every one of the 1,000,000 trees (parity over the whole C5 set): k*,
    keep bits, e_hat / utility and the per-layer union counts against the oracle run on the
    host copies of the same inputs (all host threads)."""
    import os
    P = sweep["P"].cpu().numpy()
    Q = sweep["Q"].cpu().numpy()
    n = sweep["n"].cpu().numpy()
    ids = sweep["ids"].cpu().numpy()
    out = sweep["out"]
    threads = os.cpu_count() or 8
    o = oracle.select(P, Q, gen.cost_table(N), n_nodes=n, threads=threads)
    kg = out["k_star"].cpu().numpy()
    keep_g = out["keep_bits"].cpu().numpy().view(np.uint64)
    diff = np.flatnonzero((kg != o["k_star"]) | (keep_g != o["keep_bits"]).any(axis=1) |
                          (out["status"].cpu().numpy().astype(np.uint32) != o["status"]))
    # the only admissible differences are reported ties (rule 3 of oracle/parity.py)
    if diff.size:
        sub = {k: v[diff] for k, v in o.items()}
        gsub = {k: out[k].cpu().numpy()[diff] for k in ("k_star", "e_hat", "utility", "keep_bits", "status")}
        res, msgs = compare_select(sub, gsub, n_nodes=n[diff])
        assert not msgs, msgs[:3]
        assert res["mismatch"] == 0
    same = (o["status"] == 0)
    same[diff] = False                                    # ties were checked above at the GPU's k*
    for key in ("e_hat", "utility"):
        ref = o[key][same]
        got = out[key].cpu().numpy()[same].astype(np.float64)
        assert np.all(np.abs(got - ref) <= 1e-5 * np.abs(ref)), key
    keep = downstream_keep(o, {"k_star": kg})
    ou = oracle.expert_union(keep, ids, E, n_nodes=n, threads=threads)
    assert (ou["union_count"] == out["union_count"].cpu().numpy()).all()
    assert (ou["union_total"] == out["union_total"].cpu().numpy()).all()
    assert (ou["union_bits"] == out["union_bits"].cpu().numpy().view(np.uint64).reshape(ou["union_bits"].shape)).all()
