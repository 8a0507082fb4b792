"""Cold-L2 per-CTA timeline of the C2 router call (CTA (0, 0)): globaltimer marks relative to the
CTA's first instruction."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import gen  # noqa: E402
import paper_2605_00342_b200 as ev  # noqa: E402

cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
B, N, L, d, K, E = 1, 60, 48, 2048, 8, 128
P, Q, n = gen.trees(3, B, N, 6, 10)
sel = ev.evict_select(cu(P), cu(Q), cu(gen.cost_table(N)), n_nodes=cu(n))
b = ev.evict_build_verify_tree(cu(P), sel["keep_bits"], n_nodes=cu(n))
h = gen.hidden_cuda(11, B, N, L, d, mode=1)
w = gen.wgate_cuda(12, L, E, d, mode=1, scale_log2=-5)
tr = ev._Trees(B, N, None, None, None)
T_rows = int(b["verify_offsets"][-1])
rt = ev._Router(L, E, K, d, ev._p(h), ev._p(w), T_rows)
uc = torch.empty((B, L), dtype=torch.int32, device="cuda")
ut = torch.empty(B, dtype=torch.int32, device="cuda")
ub = torch.empty((B, L, 2), dtype=torch.int64, device="cuda")
trace = torch.zeros(256, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
f = ev.lib().evict_router_union_debug
f.argtypes = [ctypes.c_void_p] * 11
f.restype = ctypes.c_int
runs = []
for it in range(30):
    flush.fill_(1)
    trace.zero_()
    torch.cuda.synchronize()
    f(ctypes.byref(tr), ev._p(b["verify_offsets"]), ev._p(b["retrieve_index"]), ctypes.byref(rt), ev._p(uc),
      ev._p(ut), ev._p(ub), None, None, ev._p(trace), ev._stream())
    torch.cuda.synchronize()
    runs.append(trace.cpu().numpy().copy())
t = np.median(np.stack(runs[5:]), axis=0)
t0 = t[250]
rel = lambda x: round((x - t0) / 1e3, 2) if x > 0 else None  # noqa: E731
print("splits", int(t[251]))
print("mma full-wait passed (us):", [rel(x) for x in t[0:32] if x > 0])
print("tma issue (us, i >= first):", [rel(x) for x in t[64:96] if x > 0])
print("epi start / tfull / staged / sync(all) / after-sync / topk-done:",
      [rel(t[192]), rel(t[193]), rel(t[196]), rel(t[194]), rel(t[195]), rel(t[197])])
