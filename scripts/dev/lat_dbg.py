"""Debug: serving-batch latency configs one by one (+ parity of the fused call for each)."""
import faulthandler
import sys
import numpy as np
import torch
faulthandler.enable()
sys.path.insert(0, ".")
import bench  # noqa: E402
import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2605_00342_b200 as ev  # noqa: E402
from oracle.parity import downstream_keep, compare_select, compare_union, compare_build  # noqa: E402

for B, N, s, t in [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]]:
    P, Q, n = gen.trees(4, B, N, s, t)
    ids = gen.routing(4, B, N, 48, 128, 8)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    g = ev.evict_select_build_union(cu(P), cu(Q), cu(gen.cost_table(N)), cu(ids), 128, n_nodes=cu(n))
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in g.items()}
    o = oracle.select(P, Q, gen.cost_table(N), n_nodes=n)
    res, msgs = compare_select(o, g, n_nodes=n)
    keep = downstream_keep(o, g)
    mu = compare_union(oracle.expert_union(keep, ids, 128, n_nodes=n), {k: v for k, v in g.items() if k in ("union_count", "union_total")})
    mb = compare_build(oracle.build_verify_tree(P, keep, n_nodes=n), {k: v for k, v in g.items() if k != "status"})
    print("PARITY", B, N, res, msgs[:2], mu[:2], mb[:2], flush=True)
    print("LAT", bench.latency(ev, torch, gen, B=B, N=N, steps=s, topk=t), flush=True)
