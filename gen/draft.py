"""Seeded synthetic drafter tables for the draft-tree builder.

Holds none of the method's arithmetic.  For tree b, step s, frontier slot j: the drafter's
top-`topk` children of that node — probabilities = the sorted top-topk of Dirichlet(α) weights
over topk + 1 categories (the extra one is "rest of the vocabulary"), α per tree log-uniform in
[0.05, 1] (easy/hard mix), descending like a drafter's top-k; tokens =
distinct ids in [0, V) (base + c·stride mod V, stride coprime to V).  numpy PCG64 keyed by (seed, tree_base).
"""
from __future__ import annotations

import numpy as np


def drafter_tables(seed, B, steps, topk, V=151936, tree_base=0):
    rng = np.random.default_rng([int(seed), int(tree_base), 7])
    alpha = np.exp(rng.uniform(np.log(0.05), 0.0, size=B))
    w = rng.gamma(np.repeat(alpha, steps * topk * (topk + 1)).reshape(B, steps, topk, topk + 1), 1.0)
    w = w / w.sum(axis=-1, keepdims=True)
    probs = np.sort(w, axis=-1)[..., ::-1][..., :topk].astype(np.float32)
    # distinct tokens per slot: base + c·stride mod V with stride a unit mod V (gcd 1)
    base = rng.integers(0, V, size=(B, steps, topk, 1), dtype=np.int64)
    stride = rng.integers(1, V, size=(B, steps, topk, 1), dtype=np.int64)
    g = np.gcd(stride, V)
    while (g != 1).any():
        stride = np.where(g != 1, stride % (V - 1) + 1, stride)
        g = np.gcd(stride, V)
    toks = ((base + np.arange(topk, dtype=np.int64) * stride) % V).astype(np.int32)
    return toks, np.ascontiguousarray(probs)
