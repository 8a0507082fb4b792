"""Router A8 probe: C2 / C4 / Ling shapes, 20 plain calls each (for an ncu launch list), then the
cold-L2 graph-replay timing the bench reports."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import gen  # noqa: E402
import paper_2605_00342_b200 as ev  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
shapes = {"c2": (1, 60, 6, 10, 48, 2048, 128), "c4": (64, 128, 8, 10, 48, 2048, 128),
          "c3": (16, 60, 6, 10, 94, 4096, 128), "ling1": (1, 60, 6, 10, 32, 4096, 256)}
B, Nn, steps, topk, L, d, E = shapes[which]
P, Q, n = gen.trees(3, B, Nn, steps, topk)
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
sel = ev.evict_select(cu(P), cu(Q), cu(gen.cost_table(Nn)), n_nodes=cu(n))
b = ev.evict_build_verify_tree(cu(P), sel["keep_bits"], n_nodes=cu(n))
h = gen.hidden_cuda(11, B, Nn, L, d, mode=1)
w = gen.wgate_cuda(12, L, E, d, mode=1, scale_log2=-5)
T = int(b["verify_offsets"][-1])
rc = ev.RouterCall(b["verify_offsets"], b["retrieve_index"], h, w, 8, B, Nn, max_rows=T)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(20):
    flush.fill_(1)
    rc()
torch.cuda.synchronize()
print(which, "rows", T)
