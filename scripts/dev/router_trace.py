import sys, ctypes, numpy as np, torch
sys.path.insert(0, '.')
import gen
import paper_2605_00342_b200 as ev
def cu(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
B, N, L, d, K, E = 1, 60, 48, 2048, 8, 128
P, Q, n = gen.trees(3, B, N, 6, 10)
sel = ev.evict_select(cu(P), cu(Q), cu(gen.cost_table(N)), n_nodes=cu(n))
b = ev.evict_build_verify_tree(cu(P), sel["keep_bits"], n_nodes=cu(n))
h = gen.hidden_cuda(11, B, N, L, d, mode=1); w = gen.wgate_cuda(12, L, E, d, mode=1, scale_log2=-5)
tr = ev._Trees(B, N, None, None, None); T_rows = int(b["verify_offsets"][-1]); rt = ev._Router(L, E, K, d, ev._p(h), ev._p(w), T_rows)
uc = torch.empty((B, L), dtype=torch.int32, device="cuda"); ut = torch.empty(B, dtype=torch.int32, device="cuda")
ub = torch.empty((B, L, 2), dtype=torch.int64, device="cuda")
trace = torch.zeros(256, dtype=torch.int64, device="cuda")
f = ev.lib().evict_router_union_debug; f.argtypes = [ctypes.c_void_p] * 11; f.restype = ctypes.c_int
for it in range(2000):
    trace.zero_()
    rc = f(ctypes.byref(tr), ev._p(b["verify_offsets"]), ev._p(b["retrieve_index"]), ctypes.byref(rt), ev._p(uc), ev._p(ut), ev._p(ub), None, None, ev._p(trace), ev._stream())
    torch.cuda.synchronize()
t = trace.cpu().numpy(); t0 = t[250]
print("rc", rc)
print("mma full-wait passed (us):", [round((x - t0) / 1e3, 2) for x in t[0:32]])
print("tma issue (us):", [round((x - t0) / 1e3, 2) for x in t[64:96]])
print("producer stage start (us):", [round((x - t0) / 1e3, 2) for x in t[128:160]])
print("epi start/tfull/end/sync/staged/topk/prepass/scan:", [round((x - t0) / 1e3, 2) for x in t[192:200]], "inserts", t[200], "scan cycles", t[201])
print("splits", int(t[251]))
