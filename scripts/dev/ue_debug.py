"""Run the throughput fused call once on a small C2-shaped batch (new union/emit kernel)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import gen  # noqa: E402
import paper_2605_00342_b200 as ev  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
c = gen.CONFIGS["c2"]
N, L, E, K = c["N"], c["L"], c["E"], c["K"]
P, Q, n = gen.trees(1, B, N, c["steps"], c["topk"])
ids = gen.routing(1, B, N, L, E, K)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
g = ev.evict_select_build_union(T(P), T(Q), T(gen.cost_table(N)), T(ids), E, n_nodes=T(n), with_stats=True)
torch.cuda.synchronize()
print("ok", g["k_star"].float().mean().item(), g["union_count"].float().mean().item())
