"""Independent brute-force checks of the oracle (pure Python, exact rationals).

These are the *plain definitions* the method must reach:

* Score(v) = product of q over the root→v path, root factor 1 (Eq. 7, reading Z1)
* For every size k, the best ancestor-closed k-subset maximises the score sum
  (§3.2.1: "optimal among all valid k-node subtrees").
* R* = max over every root-containing ancestor-closed U of sum(U) / C(|U|) (Eq. 10).

They enumerate every ancestor-closed subset, so they only run on tiny trees.
"""
from __future__ import annotations

from fractions import Fraction


def exact_scores(parent, q):
    """Score(v) as exact rationals by walking each path explicitly (no reuse of parent scores)."""
    n = len(parent)
    out = []
    for v in range(n):
        s = Fraction(1)
        u = v
        while u != 0:              # Path(x_{t+1}, v) without the root's own factor
            s *= Fraction(float(q[u]))
            u = int(parent[u])
        out.append(s)
    return out


def ancestor_closed_subsets(parent):
    """All subsets U with root ∈ U and parent(v) ∈ U for every v ∈ U (as sorted tuples)."""
    n = len(parent)
    children = [[] for _ in range(n)]
    for v in range(1, n):
        children[int(parent[v])].append(v)

    def grow(frontier, chosen):
        # frontier: nodes whose parent is chosen but which are undecided
        if not frontier:
            yield tuple(sorted(chosen))
            return
        v, rest = frontier[0], frontier[1:]
        yield from grow(rest, chosen)                                  # exclude v (and its subtree)
        yield from grow(rest + children[v], chosen + [v])              # include v

    yield from grow(children[0], [0])


def best_sum_per_size(parent, scores):
    """best[k] = max sum of scores over ancestor-closed subsets of size k (k = 1..n)."""
    n = len(parent)
    best = [None] * (n + 1)
    count = 0
    for U in ancestor_closed_subsets(parent):
        count += 1
        s = sum(scores[v] for v in U)
        k = len(U)
        if best[k] is None or s > best[k]:
            best[k] = s
    return best, count


def best_ratio(parent, scores, cost):
    """R* = max_U sum(U)/C(|U|) and the set of sizes attaining it."""
    best, _ = best_sum_per_size(parent, scores)
    ratios = {}
    for k in range(1, len(parent) + 1):
        c = float(cost[k - 1])
        ratios[k] = Fraction(0) if c == float("inf") else best[k] / Fraction(c)
    rstar = max(ratios.values())
    return rstar, sorted(k for k, r in ratios.items() if r == rstar), ratios


def is_ancestor_closed(parent, nodes):
    s = set(nodes)
    return 0 in s and all(int(parent[v]) in s for v in s if v != 0)
