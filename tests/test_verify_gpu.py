"""GPU parity of evict_verify_sample (Eq. 3 tree sampling) against the
oracle (oracle/verify.py): bit-exact accepted paths, bonus tokens and statuses."""
import numpy as np
import pytest

import gen
from gen import verify as gv
from oracle import verify as ov

pytestmark = pytest.mark.gpu


def _case(seed, B, N, V, stride=None, keep="oracle"):
    """Trees, the oracle's keep set (Eq. 10), packed target rows in the oracle's verify layout."""
    import oracle
    P, Q, n = gen.trees(seed, B, N, 6, 10)
    if keep == "oracle":
        keep_bits = oracle.select(P, Q, gen.cost_table(N), n_nodes=n)["keep_bits"]
    else:   # every node kept (EAGLE-3, rho = 1)
        keep_bits = np.zeros((B, (N + 63) // 64), np.uint64)
        for b in range(B):
            for i in range(int(n[b])):
                keep_bits[b, i // 64] |= np.uint64(1 << (i % 64))
    ob = oracle.build_verify_tree(P, keep_bits, n_nodes=n)
    off = ob["verify_offsets"]
    T = int(off[-1])
    row_tree = np.repeat(np.arange(B), np.diff(off))
    row_node = ob["kept_index"][:T]
    tok = gv.draft_tokens(seed, P, V, n_nodes=n)
    rows = gv.target_rows(seed, P, Q, tok, row_tree, row_node, V, n_nodes=n)
    stride = stride or V
    probs = np.zeros((T, stride), np.float32)
    probs[:, :V] = rows
    ua, ub = gv.uniforms(seed, B, N)
    return P, Q, n, keep_bits, off, tok, probs, ua, ub


def _gpu(P, n, keep_bits, tok, probs, ua, ub, V, greedy=False, mutate=None, exact=False):
    import torch
    import paper_2605_00342_b200 as ev
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    vt = ev.evict_build_verify_tree(cu(P), cu(keep_bits.view(np.int64)), n_nodes=cu(n))
    args = dict(verify_offsets=vt["verify_offsets"], next_token=vt["next_token"],
                next_sibling=vt["next_sibling"], retrieve_index=vt["retrieve_index"])
    if mutate:
        mutate(args)
    out = ev.evict_verify_sample(args["verify_offsets"], args["next_token"], args["next_sibling"],
                                 args["retrieve_index"], cu(tok), cu(probs),
                                 u_accept=cu(ua.view(np.int32)), u_bonus=cu(ub.view(np.int32)),
                                 greedy=greedy, vocab=V, exact=exact)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def _compare(o, g):
    for key in ("status", "accept_len", "accepted_slots", "bonus_token"):
        a, b = o[key].astype(np.int64), g[key].astype(np.int64)
        if key == "status":
            b = b & 0xFFFFFFFF
        bad = np.flatnonzero((a != b).reshape(len(a), -1).any(axis=1))
        assert bad.size == 0, (key, bad[:5], a[bad[:3]], b[bad[:3]])


@pytest.mark.parametrize("V,stride,greedy,keep", [
    (1000, None, False, "oracle"),
    (1000, None, "exact", "oracle"),   # the fixed-point bonus path forced for every tree
    (4099, 4100, False, "oracle"),     # ragged vocabulary tail, padded row stride
    (4099, 4100, True, "oracle"),
    (2048, None, False, "all"),        # every node kept: deep walks, many siblings
    (2048, None, True, "all"),
])
def test_parity_small_vocab(V, stride, greedy, keep):
    P, Q, n, kb, off, tok, probs, ua, ub = _case(11, 64, 60, V, stride, keep)
    exact = greedy == "exact"
    greedy = greedy is True
    mode = ov.GREEDY if greedy else ov.SAMPLE
    o = ov.verify_sample(P, kb, tok, probs[:, :V], ua, ub, mode=mode, n_nodes=n, verify_offsets=off)
    g = _gpu(P, n, kb, tok, probs, ua, ub, V, greedy, exact=exact)
    assert (o["status"] == 0).all()
    _compare(o, g)
    if keep == "all" and not greedy:
        assert o["accept_len"].max() >= 3     # the walks really descend


@pytest.mark.parametrize("greedy", [False, True, "exact"])
def test_parity_qwen3_vocab(greedy):
    """Full Qwen3 vocabulary (151936), the bench's launch configuration, 8 trees."""
    V = gv.QWEN3_VOCAB
    P, Q, n, kb, off, tok, probs, ua, ub = _case(12, 8, 60, V)
    exact = greedy == "exact"
    greedy = greedy is True
    mode = ov.GREEDY if greedy else ov.SAMPLE
    o = ov.verify_sample(P, kb, tok, probs, ua, ub, mode=mode, n_nodes=n, verify_offsets=off)
    g = _gpu(P, n, kb, tok, probs, ua, ub, V, greedy, exact=exact)
    _compare(o, g)


def test_parity_uniform_extremes_and_root_only():
    """u = 0 (accept the first child with mass) / u = 2^32-1 (reject all, bonus at the last
    token with residual mass) and root-only keep sets (bonus from the root row)."""
    V = 3000
    P, Q, n, kb, off, tok, probs, ua, ub = _case(13, 32, 60, V, keep="all")
    for fill in (0, 0xFFFFFFFF):
        ua2 = np.full_like(ua, fill)
        ub2 = np.full_like(ub, fill)
        o = ov.verify_sample(P, kb, tok, probs, ua2, ub2, n_nodes=n, verify_offsets=off)
        g = _gpu(P, n, kb, tok, probs, ua2, ub2, V)
        _compare(o, g)
    kb1 = np.zeros_like(kb)
    kb1[:, 0] = 1
    off1 = np.arange(33, dtype=np.int32)
    probs1 = probs[off[:-1]]                  # the root rows
    o = ov.verify_sample(P, kb1, tok, probs1, ua, ub, n_nodes=n, verify_offsets=off1)
    g = _gpu(P, n, kb1, tok, probs1, ua, ub, V)
    _compare(o, g)
    assert (g["accept_len"] == 1).all()


def test_parity_duplicate_sibling_tokens_and_subnormals():
    """Duplicated sibling tokens (the second copy has no mass after a rejection, Eq. 3) and
    rows of subnormal masses (exact fixed-point CDF)."""
    V = 600
    P, Q, n, kb, off, tok, probs, ua, ub = _case(14, 48, 60, V, keep="all")
    rng = np.random.default_rng(1)
    tok = tok.copy()
    for b in range(48):                       # give some nodes their previous sibling's token
        for i in range(2, int(n[b])):
            if P[b, i] == P[b, i - 1] and rng.random() < 0.3:
                tok[b, i] = tok[b, i - 1]
    probs = probs.copy()
    sub = rng.random(probs.shape) < 0.2
    probs[sub] = (rng.integers(1, 1 << 20, size=sub.sum()) * 2.0 ** -149).astype(np.float32)
    o = ov.verify_sample(P, kb, tok, probs, ua, ub, n_nodes=n, verify_offsets=off)
    g = _gpu(P, n, kb, tok, probs, ua, ub, V)
    _compare(o, g)


def test_status_bad_token_and_prob():
    V = 800
    P, Q, n, kb, off, tok, probs, ua, ub = _case(15, 16, 60, V, keep="all")
    tok = tok.copy()
    tok[3, 5] = V + 7                        # a kept node's token out of range
    probs = probs.copy()
    probs[off[6] + 0, 17] = np.nan           # tree 6's root row (bonus row when root-only path)
    probs[off[9] + 0, :] = 0                 # tree 9: empty root row (children masses 0)
    o = ov.verify_sample(P, kb, tok, probs, ua, ub, n_nodes=n, verify_offsets=off)
    g = _gpu(P, n, kb, tok, probs, ua, ub, V)
    assert o["status"][3] == ov.TREE_BAD_TOKEN
    assert o["status"][9] == ov.TREE_BAD_PROB
    _compare(o, g)
    for greedy in (True,):
        o = ov.verify_sample(P, kb, tok, probs, ua, ub, mode=ov.GREEDY, n_nodes=n, verify_offsets=off)
        g = _gpu(P, n, kb, tok, probs, ua, ub, V, greedy)
        _compare(o, g)


def test_bad_links_flag_keep():
    import torch
    V = 256
    P, Q, n, kb, off, tok, probs, ua, ub = _case(16, 4, 60, V, keep="all")

    def loop(args):
        nt = args["next_sibling"].clone()
        nt[int(off[1]) + 2] = 1              # a backwards sibling link in tree 1
        args["next_sibling"] = nt

    g = _gpu(P, n, kb, tok, probs, ua, ub, V, mutate=loop)
    assert int(g["status"][1]) & 0xFFFFFFFF == ov.TREE_BAD_KEEP and g["accept_len"][1] == 0
    assert (g["status"][[0, 2, 3]] == 0).all()
    assert torch.cuda.is_available()


def test_orphan_slot_beats_bad_token():
    """A tree with both an orphan slot and a bad token reports BAD_KEEP (the checks run in header
    order: size/keep, then token, then prob), like the oracle's keep-before-token order."""
    V = 256
    P, Q, n, kb, off, tok, probs, ua, ub = _case(17, 4, 60, V, keep="all")
    tok = tok.copy()
    tok[2, 3] = V + 1                        # a kept node's token out of range

    def cut(args):
        nt = args["next_token"].clone()
        nt[int(off[2])] = -1                 # tree 2: the root loses its child list -> orphan slots
        args["next_token"] = nt

    for greedy in (False, True):
        g = _gpu(P, n, kb, tok, probs, ua, ub, V, greedy=greedy, mutate=cut)
        st = g["status"].astype(np.int64) & 0xFFFFFFFF
        assert st[2] == ov.TREE_BAD_KEEP, (greedy, st)
        assert (st[[0, 1, 3]] == 0).all()


def test_bad_bonus_entry_in_a_peer_cta():
    """Batch 8 runs 8-CTA clusters per tree; a NaN at the last token of every row of trees 1 and 5
    is summed by a peer CTA (chunk 39 of 40), which reports it to CTA 0 without touching CTA 0's
    status word before the cluster barrier.  Status and outputs must equal the oracle."""
    V = 20000
    P, Q, n, kb, off, tok, probs, ua, ub = _case(18, 8, 60, V)
    probs = probs.copy()
    for b in (1, 5):
        probs[off[b]:off[b + 1], V - 1] = np.nan
    o = ov.verify_sample(P, kb, tok, probs, ua, ub, n_nodes=n, verify_offsets=off)
    assert o["status"][1] == ov.TREE_BAD_PROB and o["status"][5] == ov.TREE_BAD_PROB
    for exact in (False, True):
        _compare(o, _gpu(P, n, kb, tok, probs, ua, ub, V, exact=exact))


@pytest.mark.parametrize("exact", [False, True])
def test_parity_threshold_on_a_cdf_boundary(exact):
    """Draws that land exactly on a CDF step (dyadic rows, u = 1/4, 1/2, 3/4, …): the fp64 fast
    path cannot certify them and must hand over to the fixed-point path; the answer is the
    smallest t whose CDF exceeds u (oracle), i.e. the token after the step."""
    V, B, N = 64, 40, 4
    rng = np.random.default_rng(3)
    P = np.tile(np.array([-1, 0, 0, 1], np.int32), (B, 1))
    kb = np.ones((B, 1), np.uint64)                     # root only: the bonus comes from row 0
    tok = np.tile(np.array([0, 1, 2, 3], np.int32), (B, 1))
    probs = np.zeros((B, V), np.float32)
    for b in range(B):
        idx = rng.choice(V, size=4, replace=False)
        probs[b, idx] = [0.25, 0.25, 0.125, 0.375]
    ub = np.array([(1 << 30) * (b % 4) + (b >= 20) for b in range(B)], np.uint32)   # on / just past steps
    ua = np.zeros((B, N), np.uint32)
    off = np.arange(B + 1, dtype=np.int32)
    n = np.full(B, N, np.int32)
    o = ov.verify_sample(P, kb, tok, probs, ua, ub, n_nodes=n, verify_offsets=off)
    g = _gpu(P, n, kb, tok, probs, ua, ub, V, exact=exact)
    _compare(o, g)


@pytest.mark.parametrize("B", [150, 300, 600, 1200, 2400])
@pytest.mark.parametrize("greedy", [False, True])
def test_parity_cluster_sizes(B, greedy):
    """Batch sizes that select 4-, 2- and 1-CTA clusters per tree (the launch splits a tree's
    row over a thread-block cluster until the grid covers 4·SMs CTAs); batches ≤ 64 elsewhere
    use 8."""
    V = 300
    P, Q, n, kb, off, tok, probs, ua, ub = _case(17, B, 60, V, keep="all")
    mode = ov.GREEDY if greedy else ov.SAMPLE
    o = ov.verify_sample(P, kb, tok, probs, ua, ub, mode=mode, n_nodes=n, verify_offsets=off)
    g = _gpu(P, n, kb, tok, probs, ua, ub, V, greedy)
    _compare(o, g)


@pytest.mark.parametrize("greedy", [False, True])
def test_bench_configuration_sampled(greedy):
    """bench.py's verify workload: 1024 trees (16 copies of a 64-tree batch, each copy with its own
    uniforms) at V = 151936 — the 1-CTA-per-tree launch the bench times — with 64 sampled trees
    checked one by one against the oracle."""
    import torch
    import oracle
    import paper_2605_00342_b200 as ev
    V, B0, N, rep = gv.QWEN3_VOCAB, 64, 60, 16
    P, Q, n = gen.trees(21, B0, N, 6, 10)
    keep = oracle.select(P, Q, gen.cost_table(N), n_nodes=n)["keep_bits"]
    ob = oracle.build_verify_tree(P, keep, n_nodes=n)
    off = ob["verify_offsets"]
    T0 = int(off[-1])
    tok = gv.draft_tokens(21, P, V, n_nodes=n)
    rows = gv.target_rows(21, P, Q, tok, np.repeat(np.arange(B0), np.diff(off)), ob["kept_index"][:T0], V, n_nodes=n)
    ua, ub = gv.uniforms(21, B0 * rep, N)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    offs = np.concatenate([off[:-1] + r * T0 for r in range(rep)] + [[rep * T0]]).astype(np.int32)
    tile = lambda a: np.concatenate([a[:T0]] * rep)  # noqa: E731
    ri = np.concatenate([ob["retrieve_index"][:T0] + r * B0 * N for r in range(rep)]).astype(np.int32)
    probs = cu(rows).repeat(rep, 1)
    g = ev.evict_verify_sample(cu(offs), cu(tile(ob["next_token"])), cu(tile(ob["next_sibling"])), cu(ri),
                               cu(np.tile(tok, (rep, 1))), probs, u_accept=cu(ua.view(np.int32)),
                               u_bonus=cu(ub.view(np.int32)), greedy=greedy)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in g.items()}
    mode = ov.GREEDY if greedy else ov.SAMPLE
    sample = np.random.default_rng(3).choice(B0 * rep, 64, replace=False)
    for bb in sample:
        b = int(bb) % B0
        kept = [i for i in range(int(n[b])) if (int(keep[b, 0]) >> i) & 1]
        row_of_slot = [int(off[b]) + s for s in range(len(kept))]
        st, path, bonus = ov.verify_one(P[b].tolist(), int(n[b]), kept, tok[b].tolist(), row_of_slot, rows, mode,
                                        ua[bb].tolist(), int(ub[bb]))
        assert st == 0 and int(g["status"][bb]) == 0
        assert int(g["accept_len"][bb]) == len(path) and g["accepted_slots"][bb, :len(path)].tolist() == path, bb
        assert int(g["bonus_token"][bb]) == bonus, bb
