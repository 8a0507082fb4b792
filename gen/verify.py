"""Seeded synthetic verify-side inputs for Eq. 3 tree sampling.

Holds none of the method's arithmetic: it draws draft tokens, target next-token
distributions and the uniforms the sampler consumes, all from numpy's PCG64
seeded by (seed, tree_base).  Recipe:

* tokens: the children of every node get distinct token ids drawn without
  replacement from [0, V) (an EAGLE drafter expands the top-k tokens of one
  distribution); the root's token is drawn too (unused).
* target row of node u (the target's next-token distribution after u,
  PAPER.md:49–55): a head on u's children in the full draft tree,
  p(c) = a·q(c)·exp(0.5·z_c) rescaled to at most 0.97 in total (a ~ U(0.6, 1.0):
  drafter and target agree on ranking, not exactly on mass), and a dense tail
  (weights U(0,1)^8, normalised to the rest) over every other token, so that
  every token has non-zero mass like a softmax over the vocabulary.  fp32.
* uniforms: u_accept [B][N] and u_bonus [B], uint32.
"""
from __future__ import annotations

import numpy as np

QWEN3_VOCAB = 151936   # Qwen3-30B-A3B / Qwen3-235B-A22B vocabulary (PAPER.md:551-556 models)


def _rng(seed, tree_base, salt):
    return np.random.default_rng([int(seed), int(tree_base), int(salt)])


def draft_tokens(seed, parent, V, n_nodes=None, tree_base=0):
    """[B][N] int32: siblings carry distinct tokens; pads -1."""
    parent = np.asarray(parent, np.int32)
    B, N = parent.shape
    rng = _rng(seed, tree_base, 1)
    tok = np.full((B, N), -1, np.int32)
    for b in range(B):
        n = N if n_nodes is None else int(n_nodes[b])
        tok[b, 0] = rng.integers(0, V)
        kids = {}
        for i in range(1, n):
            kids.setdefault(int(parent[b, i]), []).append(i)
        for u, cs in kids.items():
            tok[b, cs] = rng.choice(V, size=len(cs), replace=False)
    return tok


def target_rows(seed, parent, q, tokens, row_tree, row_node, V, n_nodes=None, tree_base=0):
    """[R][V] fp32: row r is the target distribution after node row_node[r] of tree row_tree[r]."""
    parent = np.asarray(parent, np.int32)
    q = np.asarray(q, np.float32)
    B, N = parent.shape
    R = len(row_tree)
    out = np.empty((R, V), np.float32)
    for r in range(R):
        b, u = int(row_tree[r]), int(row_node[r])
        rng = _rng(seed, tree_base, 1000 + (b * N + u))
        n = N if n_nodes is None else int(n_nodes[b])
        kids = [i for i in range(1, n) if parent[b, i] == u]
        tail = rng.random(V, dtype=np.float32) ** 8
        head = np.zeros(len(kids))
        if kids:
            head = rng.uniform(0.6, 1.0) * q[b, kids].astype(np.float64) * np.exp(0.5 * rng.standard_normal(len(kids)))
            if head.sum() > 0.97:
                head *= 0.97 / head.sum()
        tail[[tokens[b, c] for c in kids]] = 0
        row = tail.astype(np.float64) * ((1.0 - head.sum()) / max(float(tail.sum(dtype=np.float64)), 1e-30))
        row[[tokens[b, c] for c in kids]] = head
        out[r] = row.astype(np.float32)
    return out


def uniforms(seed, B, N, tree_base=0):
    rng = _rng(seed, tree_base, 2)
    return (rng.integers(0, 1 << 32, size=(B, N), dtype=np.uint64).astype(np.uint32),
            rng.integers(0, 1 << 32, size=B, dtype=np.uint64).astype(np.uint32))
