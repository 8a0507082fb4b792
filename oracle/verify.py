"""CPU oracle for verify-side tree sampling — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline legs
may import this module; the product path never does and shares no code with it.

What it computes (§2.1, Eq. 3): the kept tree T_{k*} has been
verified in one pass, so every kept node u carries the target's next-token
distribution p_u (one row of ``probs``).  Starting at the root, the verifier
visits the kept children c of the current node u one by one (ascending slot
order = ascending node index, reading Z12/V2) and

  * sampling (T > 0): accepts c with probability p_u(token(c)); on acceptance
    the surviving path moves to c.  On rejection the mass of c is removed and
    every other token w is renormalised, p_u(w) <- p_u(w) / (1 - p_u(c))
    (Eq. 3), and the next sibling is tried with the updated distribution.  If
    every kept child is rejected (or u has none) a fresh "bonus" token is drawn
    from the final residual distribution.
  * greedy (T = 0, Table 1's "Temperature = 0"): accepts the first kept child
    whose token is argmax_w p_u(w) (smallest w on ties); else the bonus is that
    argmax (reading V5).

Random numbers are inputs (uint32): child slot s is decided by u_accept[b][s]
(accept iff u/2^32 < p, i.e. u < p·2^32, exact in fp64), the bonus by
u_bonus[b].  The accept decision and the Eq. 3 renormalisation are taken in
fp32 — the kernel's precision, since they decide an integer (reading V3) — one
IEEE division per rejected sibling, in visiting order.  The bonus is the exact
inverse CDF of the residual (reading V4): with r(w) = p_u(w) for tokens not
rejected at u and 0 for rejected ones, every fp32 value is an exact integer
multiple of 2^-149, so with X(w) = r(w)·2^149 (Python ints) and Z = Σ X(w),
bonus = the smallest t with Σ_{w≤t} X(w) > floor(u_bonus·Z / 2^32), i.e. the
smallest t whose cumulative residual mass exceeds u_bonus/2^32 of the total.
This is the plain definition of sampling a categorical by inversion, with no
rounding at all, so any summation order reaches it.

Pins (tests/test_oracle_verify_pins.py): losslessness of the first committed
token (Monte Carlo), acceptance probability of every kept node =
its Eq. 6 path product (Appendix A), SPEC.md:522's
telescoping example, the deterministic extremes u = 0 / u = 2^32 - 1, inverse
CDF vs numpy searchsorted away from ties, greedy vs numpy argmax.
"""
from __future__ import annotations

import numpy as np

SAMPLE, GREEDY = 0, 1
TREE_BAD_SIZE = 0x01
TREE_BAD_PROB = 0x04
TREE_BAD_KEEP = 0x20
TREE_BAD_TOKEN = 0x40
TWO32 = 1 << 32
SCALE = 2.0 ** 149   # fp32 values are integer multiples of 2^-149


def _bad(x):
    """p entries must be fp32 values in [0, 1] (NaN fails both compares)."""
    return not (x >= 0.0 and x <= 1.0)


def _exact_ints(row):
    """fp32 row -> exact integers X(w) = r(w)·2^149 (fp64 holds every fp32 exactly; ×2^149 is exact)."""
    return [int(v) for v in (np.asarray(row, np.float32).astype(np.float64) * SCALE).tolist()]


def inverse_cdf(row, zeroed, ub):
    """Smallest t with Σ_{w≤t} X(w) > floor(ub·Z/2^32), X = exact residual (zeroed tokens 0).
    Returns -1 when Z = 0 (no residual mass)."""
    X = _exact_ints(row)
    for t in zeroed:
        X[t] = 0
    Z = sum(X)
    if Z == 0:
        return -1
    T = (int(ub) * Z) >> 32
    acc = 0
    for t, x in enumerate(X):
        acc += x
        if acc > T:
            return t
    raise AssertionError("unreachable: T < Z")


def verify_one(parent, n, kept, tokens, row_of_slot, probs, mode, u_accept, u_bonus):
    """One tree.  kept: ascending kept node indices; row_of_slot[s]: row of probs for slot s.
    Returns (status, path_slots, bonus)."""
    V = probs.shape[1]
    if not (1 <= n <= len(parent)):
        return TREE_BAD_SIZE, [], -1
    keep = set(kept)
    if 0 not in keep or any(v >= n or (v != 0 and parent[v] not in keep) for v in kept):
        return TREE_BAD_KEEP, [], -1
    slot = {v: s for s, v in enumerate(kept)}
    # Child(u) restricted to T_{k*}, visited in ascending slot (= node index) order
    children = {u: [v for v in kept if v != 0 and parent[v] == u] for u in kept}
    if any(not (0 <= tokens[v] < V) for v in kept if v != 0):
        return TREE_BAD_TOKEN, [], -1
    if mode == SAMPLE:
        # validated entries: p at (row of the parent's slot, token of c) for every kept child c
        for v in kept:
            if v != 0 and _bad(probs[row_of_slot[slot[parent[v]]], tokens[v]]):
                return TREE_BAD_PROB, [], -1
    path, u = [0], 0
    while True:
        row = probs[row_of_slot[slot[u]]]
        if mode == GREEDY:
            if any(_bad(x) for x in row.tolist()):
                return TREE_BAD_PROB, [], -1
            g = int(np.argmax(row))            # first maximal index
            nxt = next((c for c in children[u] if tokens[c] == g), None)
            if nxt is None:
                return 0, [slot[v] for v in path], g
            path.append(nxt)
            u = nxt
            continue
        # sampling: Eq. 3 over the kept children, current values per sibling token in fp32
        cur = {}
        for c in children[u]:
            cur.setdefault(tokens[c], np.float32(row[tokens[c]]))
        rejected = []
        nxt = None
        for c in children[u]:
            pc = cur[tokens[c]]
            if float(u_accept[slot[c]]) < float(pc) * float(TWO32):   # accept with probability p(c)
                nxt = c
                break
            d = np.float32(np.float32(1.0) - pc)                         # 1 - p(c)
            cur[tokens[c]] = np.float32(0.0)                             # w = c: 0
            for w in cur:                                                # w != c: p(w)/(1 - p(c))
                if w != tokens[c]:
                    cur[w] = np.float32(cur[w] / d)
            rejected.append(tokens[c])
        if nxt is not None:
            path.append(nxt)
            u = nxt
            continue
        if any(_bad(x) for x in row.tolist()):
            return TREE_BAD_PROB, [], -1
        bonus = inverse_cdf(row, rejected, u_bonus)
        if bonus < 0:
            return TREE_BAD_PROB, [], -1
        return 0, [slot[v] for v in path], bonus


def verify_sample(parent, keep_bits, tokens, probs, u_accept, u_bonus, mode=SAMPLE,
                  n_nodes=None, verify_offsets=None, node_rows=False):
    """Batch wrapper.  parent/tokens [B][N] int32 (node-indexed), keep_bits [B][W] uint64,
    probs [R][V] fp32 with slot s of tree b at row verify_offsets[b] + s (verify_offsets
    None ⇒ b·N + s; node_rows ⇒ row b·N + node of slot s), u_accept [B][N] uint32
    (slot-indexed), u_bonus [B] uint32.
    Returns dict(accept_len [B], accepted_slots [B][N], bonus_token [B], status [B])."""
    parent = np.asarray(parent, np.int32)
    tokens = np.asarray(tokens, np.int32)
    keep_bits = np.asarray(keep_bits, np.uint64).reshape(parent.shape[0], -1)
    probs = np.asarray(probs, np.float32)
    u_accept = np.asarray(u_accept, np.uint32)
    u_bonus = np.asarray(u_bonus, np.uint32)
    B, N = parent.shape
    out = dict(accept_len=np.zeros(B, np.int32), accepted_slots=np.full((B, N), -1, np.int32),
               bonus_token=np.full(B, -1, np.int32), status=np.zeros(B, np.uint32))
    for b in range(B):
        n = N if n_nodes is None else int(n_nodes[b])
        words = [int(x) for x in keep_bits[b]]
        kept = [i for i in range(min(max(n, 0), N)) if (words[i >> 6] >> (i & 63)) & 1]
        if any((words[i >> 6] >> (i & 63)) & 1 for i in range(max(n, 0), 64 * len(words))):
            st, path, bonus = TREE_BAD_KEEP, [], -1     # a pad bit is set
        else:
            base = b * N if verify_offsets is None else int(verify_offsets[b])
            rows = [b * N + v for v in kept] if node_rows else [base + s for s in range(len(kept))]
            st, path, bonus = verify_one(parent[b].tolist(), n, kept, tokens[b].tolist(), rows, probs,
                                         mode, u_accept[b].tolist(), int(u_bonus[b]))
        out["status"][b] = st
        if st == 0:
            out["accept_len"][b] = len(path)
            out["accepted_slots"][b, :len(path)] = path
            out["bonus_token"][b] = bonus
    return out


def path_acceptance(parent, kept, tokens, row_of_slot, probs):
    """Eq. 6 / Appendix A: P(node v on the accepted path) = Π_{u on path(root, v), u ≠ root}
    p_{parent(u)}(token(u)), in fp64.  Used by the pins, not by verify_one."""
    slot = {v: s for s, v in enumerate(kept)}
    acc = {0: 1.0}
    for v in kept:
        if v != 0:
            acc[v] = acc[parent[v]] * float(probs[row_of_slot[slot[parent[v]]], tokens[v]])
    return acc
