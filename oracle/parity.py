"""Parity rules between the CUDA path and the oracle — TEST INFRASTRUCTURE ONLY.

SURVEY.md §8(c) / north_star:
  1. integer outputs bit-exact (keep_bits, k*, order, masks, positions,
     retrieve/next lists, union counts/bits);
  2. fp32 e_hat, utility, prefix sums within 1e-5 relative of the oracle's fp64;
  3. where the oracle's near-tie set (ratios within 1e-5 of the max) holds more
     than one k, a GPU k* inside the set is a *tie*, not a mismatch, and the
     downstream outputs are compared against the oracle at the GPU's k*.
"""
from __future__ import annotations

import numpy as np

REL = 1e-5


def _bits_list(words, n):
    out = []
    for i in range(n):
        if (int(words[i // 64]) >> (i % 64)) & 1:
            out.append(i)
    return out


def _u64(a):
    return np.asarray(a).astype(np.int64).view(np.uint64)


def compare_select(o, g, n_nodes=None, check_order=False):
    """o: oracle.select output; g: dict of numpy arrays from the GPU (k_star, e_hat, utility,
    keep_bits [, order, prefix_sums], status).  Returns (stats, list of mismatch messages)."""
    B, N = o["order"].shape
    W = (N + 63) // 64
    kg = np.asarray(g["k_star"])
    keep_g = _u64(g["keep_bits"]).reshape(B, W)
    st_g = np.asarray(g["status"]).astype(np.uint32)
    res = dict(match=0, tie=0, mismatch=0, error_trees=0)
    msgs = []
    for b in range(B):
        n = int(n_nodes[b]) if n_nodes is not None else N
        if o["status"][b] or st_g[b]:
            if (o["status"][b] != st_g[b]) or kg[b] != 0 or keep_g[b].any():
                res["mismatch"] += 1
                msgs.append(f"tree {b}: status oracle {o['status'][b]} gpu {st_g[b]} k* {kg[b]}")
            else:
                res["error_trees"] += 1
            continue
        ko = int(o["k_star"][b])
        k = int(kg[b])
        ties = _bits_list(o["tie_bits"][b], N)
        if k == ko:
            kind = "match"
        elif 1 <= k <= n and (k - 1) in ties and len(ties) > 1:
            kind = "tie"
        else:
            res["mismatch"] += 1
            msgs.append(f"tree {b}: k* oracle {ko} gpu {k} ties {[t + 1 for t in ties]}")
            continue
        expect = np.zeros(W, np.uint64)
        for v in o["order"][b, :k]:
            expect[v // 64] |= np.uint64(1 << int(v % 64))
        ok = (keep_g[b] == expect).all()
        S = o["S"][b, k - 1]
        R = o["R"][b, k - 1]
        ok &= abs(float(g["e_hat"][b]) - S) <= REL * abs(S)
        ok &= abs(float(g["utility"][b]) - R) <= REL * abs(R)
        if check_order and "order" in g:
            ok &= (np.asarray(g["order"][b]) == o["order"][b]).all()
            ps = np.asarray(g["prefix_sums"][b], np.float64)
            ok &= bool(np.all(np.abs(ps[:n] - o["S"][b, :n]) <= REL * np.abs(o["S"][b, :n])))
            ok &= bool(np.all(ps[n:] == 0))
        if ok:
            res[kind] += 1
        else:
            res["mismatch"] += 1
            msgs.append(f"tree {b}: outputs differ (k*={k}, kind={kind}): e_hat {g['e_hat'][b]} vs {S}, "
                        f"util {g['utility'][b]} vs {R}, keep {keep_g[b]} vs {expect}")
    return res, msgs


def compare_build(o, g):
    """Bit-exact comparison of the packed verify-tree outputs."""
    msgs = []
    off_o = np.asarray(o["verify_offsets"])
    off_g = np.asarray(g["verify_offsets"])
    if not (off_o == off_g).all():
        msgs.append(f"verify_offsets differ: first at {np.argmax(off_o != off_g)}")
        return msgs
    T = int(off_o[-1])
    for f in ("kept_index", "retrieve_index", "positions", "next_token", "next_sibling"):
        a, b_ = np.asarray(o[f])[:T], np.asarray(g[f])[:T]
        if not (a == b_).all():
            i = int(np.argmax(a != b_))
            msgs.append(f"{f} differs at row {i}: oracle {a[i]} gpu {b_[i]}")
    tm_o = np.asarray(o["tree_mask"])[:T]
    tm_g = _u64(g["tree_mask"]).reshape(-1, tm_o.shape[1])[:T]
    if T and not (tm_o == tm_g).all():
        msgs.append("tree_mask differs")
    if "status" in g and not (np.asarray(o["status"]) == np.asarray(g["status"]).astype(np.uint32)).all():
        msgs.append("build status differs")
    return msgs


def compare_union(o, g, with_bits=True):
    msgs = []
    if not (np.asarray(o["union_count"]) == np.asarray(g["union_count"])).all():
        bad = np.argwhere(np.asarray(o["union_count"]) != np.asarray(g["union_count"]))[:3]
        msgs.append(f"union_count differs at {bad.tolist()}")
    if "union_total" in g and not (np.asarray(o["union_total"]) == np.asarray(g["union_total"])).all():
        msgs.append("union_total differs")
    if with_bits and "union_bits" in g and g["union_bits"] is not None:
        if not (np.asarray(o["union_bits"]) == _u64(g["union_bits"]).reshape(o["union_bits"].shape)).all():
            msgs.append("union_bits differ")
    if "status" in g and not (np.asarray(o["status"]) == np.asarray(g["status"]).astype(np.uint32)).all():
        msgs.append("union status differs")
    return msgs


def downstream_keep(o, g, n_nodes=None):
    """Keep sets for the downstream (build / union) comparisons, taken from the ORACLE: its own
    keep bits, except for trees that compare_select classed as a tie (the GPU's k* differs from
    the oracle's but lies in the oracle's near-tie set, rule 3), which use the oracle's ranking
    prefix of the GPU's length — "the oracle evaluated at the GPU's k*".  No node set is taken
    from the GPU."""
    B, N = o["order"].shape
    keep = np.array(o["keep_bits"], dtype=np.uint64, copy=True)
    kg = np.asarray(g["k_star"])
    for b in range(B):
        if o["status"][b] or int(kg[b]) == int(o["k_star"][b]) or int(kg[b]) < 1:
            continue
        keep[b] = 0
        for v in o["order"][b, :int(kg[b])]:
            keep[b, v // 64] |= np.uint64(1 << int(v % 64))
    return keep
