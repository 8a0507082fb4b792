"""Per-layer union mismatches of the throughput union/emit kernel vs the oracle (debug)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2605_00342_b200 as ev  # noqa: E402
from oracle.parity import downstream_keep  # noqa: E402

for L in [int(x) for x in sys.argv[1:]] or [56]:
    c = gen.CONFIGS["c2"]
    B, N, E, K = 3000, c["N"], 128, 8
    P, Q, n = gen.trees(3, B, N, c["steps"], c["topk"])
    ids = gen.routing(3, B, N, L, E, K)
    cost = gen.cost_table(N)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    g = ev.evict_select_build_union(T(P), T(Q), T(cost), T(ids), E, n_nodes=T(n))
    g = {k: v.cpu().numpy() for k, v in g.items()}
    o = oracle.select(P, Q, cost, n_nodes=n, threads=8)
    keep = downstream_keep(o, g)
    ou = oracle.expert_union(keep, ids, E, n_nodes=n, threads=8)
    d = g["union_count"] != ou["union_count"]
    print("L", L, "trees with mismatch", d.any(1).sum(), "layers", np.flatnonzero(d.any(0)).tolist())
    bt = np.flatnonzero(d.any(1))[:3]
    for b in bt:
        ls = np.flatnonzero(d[b])[:6]
        print(" tree", b, "k*", g["k_star"][b], [(int(l), int(g["union_count"][b, l]), int(ou["union_count"][b, l])) for l in ls])
