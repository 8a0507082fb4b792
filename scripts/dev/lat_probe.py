"""Serving-batch calls for an ncu launch list: select and fused at B = 64 and B = 1 (C2 trees)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import gen  # noqa: E402
import paper_2605_00342_b200 as ev  # noqa: E402

for B in (64, 1):
    P, Q, n = gen.trees(4, B, 60, 6, 10)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    tP, tQ, tn, tc = cu(P), cu(Q), cu(n), cu(gen.cost_table(60))
    ids = gen.routing_cuda(4, B, 60, 48, 128, 8)
    fc = ev.FusedCall(tP, tQ, tc, ids, 128, n_nodes=tn)
    for _ in range(10):
        ev.evict_select(tP, tQ, tc, n_nodes=tn)
        fc()
    torch.cuda.synchronize()
print("ok")
