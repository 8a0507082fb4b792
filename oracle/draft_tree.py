"""CPU oracle for the draft-tree builder — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline legs may import
this module; the product path never does and shares no code with it.

What it computes (§2.1: the drafter "repeatedly extends a fixed number of draft
tokens to produce a well-structured token tree ... with the same number of tokens at each
layer", then the tree "is pruned ... to meet a predefined token budget" by "the top-k nodes
ranked by cumulative scores", §3.2.1), one tree at a time, in the paper's
order (reading T1 — EAGLE-2/3 expansion with SGLang's all-candidate reranking):

  pool = [root], Score(root) = 1, frontier = [root]
  for s = 0 .. steps-1:                       # one drafter forward per step
      for j, u in enumerate(frontier):         # frontier slot j (rank order)
          for c in 0 .. topk-1:                # the drafter's top-topk children of u
              add node (parent u, token child_tokens[s][j][c], q = child_probs[s][j][c],
                        Score = fl32(Score(u) · q))          # Eq. 7, one fp32 rounding per edge
      frontier = the topk new nodes of this step with the best (Score desc, creation index asc)
  keep = root + the N-1 best pool nodes by (Score desc, creation index asc)   (§3.2.1, Z4)
  renumber the kept nodes by creation index (parent < child: topological, reading Z12)

Step 0 reads frontier slot 0 only (the root).  Outputs: parent, q (q[0] = 1), token (-1 for
the root: x_{t+1} is sampled by the target, Eq. 1), Score, n = min(N, |pool|).  A probability
outside [0, 1] (or NaN) → status BAD_PROB, zero outputs.

Pins (tests/test_oracle_draft_tree_pins.py): SPEC.md:262's top-1 chain, node counts, every
node's parent/token/q traced back to the drafter table, Eq. 7 scores, ancestor closure, the
"well-structured" layer sizes, the kept set = brute-force best-sum subtree of the pool for
small cases (PAPER.md:135 optimality), and equality with the A3 ranking prefix.
"""
from __future__ import annotations

import numpy as np

TREE_BAD_PROB = 0x04


def build_one(child_tokens, child_probs, steps, topk, N):
    """child_tokens/probs: [steps][topk][topk].  Returns (status, parent, q, token, score, n, pool)."""
    f32 = np.float32
    pool = [dict(score=f32(1.0), parent=-1, token=-1, q=f32(1.0), step=-1)]
    frontier = [0]
    for s in range(steps):
        new = []
        for j, u in enumerate(frontier):
            for c in range(topk):
                q = f32(child_probs[s][j][c])
                if not (q >= 0.0 and q <= 1.0):
                    return TREE_BAD_PROB, None, None, None, None, 0, None
                new.append(len(pool))
                pool.append(dict(score=f32(pool[u]["score"] * q), parent=u,
                                 token=int(child_tokens[s][j][c]), q=q, step=s))
        frontier = sorted(new, key=lambda i: (-float(pool[i]["score"]), i))[:topk]
    ranked = sorted(range(len(pool)), key=lambda i: (-float(pool[i]["score"]), i))
    keep = sorted(ranked[:N])                   # root is first in the ranking (Score 1, index 0)
    new_id = {old: k for k, old in enumerate(keep)}
    parent = np.full(N, -1, np.int32)
    q = np.zeros(N, np.float32)
    tok = np.full(N, -1, np.int32)
    score = np.zeros(N, np.float32)
    for k, old in enumerate(keep):
        p = pool[old]
        parent[k] = -1 if p["parent"] < 0 else new_id[p["parent"]]
        q[k] = p["q"]
        tok[k] = p["token"]
        score[k] = p["score"]
    return 0, parent, q, tok, score, len(keep), pool


def build_draft_trees(child_tokens, child_probs, steps, topk, N):
    """Batch: child_tokens int32 / child_probs fp32 [B][steps][topk][topk].
    Returns dict(parent [B][N], q [B][N], tokens [B][N], score [B][N], n_nodes [B], status [B])."""
    child_tokens = np.asarray(child_tokens, np.int32)
    child_probs = np.asarray(child_probs, np.float32)
    B = child_tokens.shape[0]
    out = dict(parent=np.full((B, N), -1, np.int32), q=np.zeros((B, N), np.float32),
               tokens=np.full((B, N), -1, np.int32), score=np.zeros((B, N), np.float32),
               n_nodes=np.zeros(B, np.int32), status=np.zeros(B, np.uint32))
    for b in range(B):
        st, par, q, tok, sc, n, _ = build_one(child_tokens[b], child_probs[b], steps, topk, N)
        out["status"][b] = st
        if st:
            continue                            # error state: pads, n_nodes 0
        out["parent"][b], out["q"][b], out["tokens"][b], out["score"][b] = par, q, tok, sc
        out["n_nodes"][b] = n
    return out
