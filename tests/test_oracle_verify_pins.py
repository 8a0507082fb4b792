"""Pins of the Eq. 3 tree-sampling oracle (oracle/verify.py) — CPU only.

None of these re-types the oracle's formula: they check what PAPER.md and probability
fix — losslessness of the first committed token ("preserves the original
target distribution"), the acceptance probability of every kept node = its Eq. 6 path
product (Appendix A), SPEC.md:522's telescoping example, the
deterministic extremes of the uniforms, and library routines (numpy searchsorted /
argmax / flatnonzero) away from ties.
"""
import numpy as np
import pytest

from oracle import verify as ov

TWO32 = 1 << 32


def bits_of(kept, N):
    w = np.zeros((N + 63) // 64, np.uint64)
    for v in kept:
        w[v // 64] |= np.uint64(1 << (v % 64))
    return w


def run_one(parent, kept, tokens, probs_by_node, ua, ub, mode=ov.SAMPLE):
    """Single tree; probs_by_node[v] = row after node v (node-indexed rows)."""
    N = len(parent)
    rows = [v for v in kept]
    return ov.verify_one(list(parent), N, kept, list(tokens), rows, probs_by_node, mode, list(ua), int(ub))


def mc(parent, kept, tokens, probs, trials, seed):
    rng = np.random.default_rng(seed)
    N = len(parent)
    UA = rng.integers(0, TWO32, size=(trials, N), dtype=np.uint64)
    UB = rng.integers(0, TWO32, size=trials, dtype=np.uint64)
    res = []
    for t in range(trials):
        st, path, bonus = run_one(parent, kept, tokens, probs, UA[t].tolist(), int(UB[t]))
        assert st == 0
        res.append((path, bonus))
    return res


def within(freq, p, n, sig=4.5):
    return abs(freq - p) <= sig * np.sqrt(max(p * (1 - p), 1e-12) / n) + 1e-12


def test_spec_telescoping_two_children():
    """kept children with target probs (0.3, 0.5): child 2 is committed with
    probability (1 - 0.3)·(0.5/0.7) = 0.5, child 1 with 0.3, the bonus with 0.2."""
    parent = [-1, 0, 0]
    tokens = [9, 1, 2]
    probs = np.zeros((3, 4), np.float32)
    probs[0] = [0.2, 0.3, 0.5, 0.0]
    probs[1] = probs[2] = [0.25] * 4
    n = 40000
    res = mc(parent, [0, 1, 2], tokens, probs, n, 1)
    f1 = np.mean([len(p) > 1 and p[1] == 1 for p, _ in res])
    f2 = np.mean([len(p) > 1 and p[1] == 2 for p, _ in res])
    fb = np.mean([len(p) == 1 for p, _ in res])
    assert within(f1, 0.3, n) and within(f2, 0.5, n) and within(fb, 0.2, n), (f1, f2, fb)
    # on the all-rejected branch the bonus can only be token 0 (1 and 2 removed, 3 has no mass)
    assert all(b == 0 for p, b in res if len(p) == 1)


@pytest.mark.parametrize("seed", [2, 3])
def test_losslessness_first_token(seed):
    """the first committed token (accepted child or bonus) is distributed
    exactly as the target's root row, whatever the drafted children."""
    rng = np.random.default_rng(seed)
    V = 6
    parent = [-1, 0, 0, 0, 1, 1]
    tokens = [0, 4, 1, 3, 2, 5]            # root's children: tokens 4, 1, 3
    probs = rng.dirichlet(np.ones(V), size=6).astype(np.float32)
    n = 40000
    res = mc(parent, list(range(6)), tokens, probs, n, seed + 10)
    first = [tokens[p[1]] if len(p) > 1 else b for p, b in res]
    target = probs[0].astype(np.float64) / probs[0].astype(np.float64).sum()
    for t in range(V):
        assert within(np.mean([f == t for f in first]), target[t], n), (t, target[t])


def test_acceptance_is_eq6_path_product():
    """Appendix A / Eq. 6: P(v on the accepted path) = Π of the target probs along its path,
    and E[accept_len] = Σ_v of those products."""
    rng = np.random.default_rng(4)
    V = 8
    parent = [-1, 0, 0, 1, 1, 2, 3, 3, 5, 0]
    N = len(parent)
    tokens = [0] * N
    for u in range(N):                      # distinct sibling tokens
        kids = [v for v in range(1, N) if parent[v] == u]
        for v, t in zip(kids, rng.permutation(V)):
            tokens[v] = int(t)
    probs = rng.dirichlet(np.ones(V) * 0.7, size=N).astype(np.float32)
    kept = list(range(N))
    acc = ov.path_acceptance(parent, kept, tokens, kept, probs)
    n = 30000
    res = mc(parent, kept, tokens, probs, n, 5)
    for v in kept[1:]:
        assert within(np.mean([v in p for p, _ in res]), acc[v], n), v
    mean_len = np.mean([len(p) for p, _ in res])
    sd = np.std([len(p) for p, _ in res])
    assert abs(mean_len - sum(acc.values())) <= 4.5 * sd / np.sqrt(n)


def test_extremes_of_the_uniforms():
    """u_accept = 0 accepts the first kept child with p > 0 at every node (leftmost chain);
    u_accept = 2^32-1 rejects every child with p < 1; u_bonus = 0 / 2^32-1 take the first /
    last token with residual mass (numpy flatnonzero)."""
    rng = np.random.default_rng(6)
    V = 50
    parent = [-1, 0, 0, 1, 1, 3]
    tokens = [0, 7, 8, 9, 10, 11]
    probs = rng.random((6, V)).astype(np.float32) / V
    probs[:, :3] = 0.0                       # leading zero-mass tokens
    probs[:, -2:] = 0.0                      # trailing zero-mass tokens
    st, path, bonus = run_one(parent, list(range(6)), tokens, probs, [0] * 6, 0)
    assert st == 0 and path == [0, 1, 3, 5]
    assert bonus == np.flatnonzero(probs[5])[0] == 3
    st, path, bonus = run_one(parent, list(range(6)), tokens, probs, [TWO32 - 1] * 6, TWO32 - 1)
    res = probs[0].copy()
    res[[7, 8]] = 0
    assert st == 0 and path == [0] and bonus == np.flatnonzero(res)[-1] == V - 3


def test_inverse_cdf_exact_boundaries():
    """Sampling by inversion picks the smallest t whose CDF exceeds u: with row (1/2, 1/2)
    u = 1/2 lies exactly on the boundary and must give token 1; u just below gives 0.
    Subnormal masses count exactly: (2^-149, 0, 1) with u = 0 gives token 0."""
    row = np.array([0.5, 0.5], np.float32)
    assert ov.inverse_cdf(row, [], TWO32 // 2) == 1
    assert ov.inverse_cdf(row, [], TWO32 // 2 - 1) == 0
    tiny = np.array([np.float32(2.0 ** -149), 0.0, 1.0], np.float32)
    assert tiny[0] > 0
    assert ov.inverse_cdf(tiny, [], 0) == 0
    assert ov.inverse_cdf(tiny, [0], 0) == 2
    assert ov.inverse_cdf(np.zeros(4, np.float32), [], 5) == -1


def test_inverse_cdf_vs_searchsorted():
    """Library cross-check away from ties: np.searchsorted on the fp64 normalised CDF."""
    rng = np.random.default_rng(7)
    checked = 0
    for _ in range(300):
        V = int(rng.integers(2, 3000))
        row = (rng.random(V) ** 4).astype(np.float32)
        zeroed = list(rng.choice(V, size=min(3, V - 1), replace=False))
        ub = int(rng.integers(0, TWO32))
        r = row.astype(np.float64)
        r[zeroed] = 0
        cdf = np.cumsum(r) / r.sum()
        u = ub / TWO32
        if np.min(np.abs(cdf - u)) < 1e-9:
            continue
        assert ov.inverse_cdf(row, zeroed, ub) == int(np.searchsorted(cdf, u, side="right"))
        checked += 1
    assert checked > 250


def test_greedy_follows_argmax():
    """T = 0: the accepted path follows np.argmax of each row through the kept children;
    the bonus is np.argmax of the last row (first index on ties)."""
    rng = np.random.default_rng(8)
    V = 40
    parent = [-1, 0, 0, 1, 1, 2, 4]
    tokens = [0, 5, 6, 7, 8, 9, 10]
    probs = rng.random((7, V)).astype(np.float32) * 0.5
    probs[0, 5] = 0.9                        # root → node 1 (token 5)
    probs[1, 8] = 0.8                        # node 1 → node 4 (token 8)
    probs[4, 3] = 0.7                        # node 4: argmax token 3 matches no child (node 6 has 10)
    probs[4, 17] = 0.7                       # tie with 17: first index wins
    st, path, bonus = run_one(parent, list(range(7)), tokens, probs, [0] * 7, 0, ov.GREEDY)
    assert st == 0 and path == [0, 1, 4] and bonus == int(np.argmax(probs[4])) == 3
    # node 4 not kept: the walk stops at node 1 even though argmax matches it
    kept = [0, 1, 2, 3, 5]
    st, path, bonus = run_one(parent, kept, tokens, probs, [0] * 7, 0, ov.GREEDY)
    assert st == 0 and [kept[s] for s in path] == [0, 1] and bonus == 8


def test_status_bits():
    parent = [-1, 0, 0, 1]
    tokens = [0, 1, 2, 3]
    probs = np.full((4, 4), 0.25, np.float32)
    assert run_one(parent, [0, 1, 2, 3], [0, 1, 2, 99], probs, [0] * 4, 0)[0] == ov.TREE_BAD_TOKEN
    assert run_one(parent, [0, 3], tokens, probs, [0] * 4, 0)[0] == ov.TREE_BAD_KEEP
    assert run_one(parent, [1, 3], tokens, probs, [0] * 4, 0)[0] == ov.TREE_BAD_KEEP
    bad = probs.copy()
    bad[0, 2] = np.nan                       # a gathered child prob
    assert run_one(parent, [0, 1, 2, 3], tokens, bad, [0] * 4, 0)[0] == ov.TREE_BAD_PROB
    bad = probs.copy()
    bad[3, 0] = 1.5                          # the bonus row (leaf 3 after accepting 1, 3)
    assert run_one(parent, [0, 1, 2, 3], tokens, bad, [0] * 4, 0)[0] == ov.TREE_BAD_PROB
    zero = probs.copy()
    zero[3] = 0                              # no residual mass on the bonus row
    assert run_one(parent, [0, 1, 2, 3], tokens, zero, [0] * 4, 0)[0] == ov.TREE_BAD_PROB


def test_batch_wrapper_layouts():
    """Packed rows (verify_offsets) and node rows give the same result for the same data."""
    from gen import verify as gv
    import gen
    P, Q, n = gen.trees(2, 6, 60, 6, 10)
    rng = np.random.default_rng(9)
    keep = np.zeros((6, 1), np.uint64)
    for b in range(6):                       # keep the first k nodes (topological ⇒ ancestor-closed)
        k = int(rng.integers(1, int(n[b]) + 1))
        keep[b, 0] = np.uint64((1 << k) - 1) if k < 64 else np.uint64(~0 & ((1 << 64) - 1))
    V = 500
    tok = gv.draft_tokens(3, P, V, n_nodes=n)
    node_probs = gv.target_rows(3, P, Q, tok, np.repeat(np.arange(6), 60), np.tile(np.arange(60), 6), V, n_nodes=n)
    ua, ub = gv.uniforms(3, 6, 60)
    a = ov.verify_sample(P, keep, tok, node_probs, ua, ub, n_nodes=n, node_rows=True)
    ks = [bin(int(keep[b, 0])).count("1") for b in range(6)]
    off = np.concatenate([[0], np.cumsum(ks)]).astype(np.int32)
    packed = np.concatenate([node_probs[b * 60: b * 60 + ks[b]] for b in range(6)])
    c = ov.verify_sample(P, keep, tok, packed, ua, ub, n_nodes=n, verify_offsets=off)
    for key in a:
        assert np.array_equal(a[key], c[key]), key
    assert (a["status"] == 0).all() and (a["accept_len"] >= 1).all()
