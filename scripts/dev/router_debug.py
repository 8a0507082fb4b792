# Dump router rows that differ from the oracle (integer inputs, C2 shape)
import sys, numpy as np, torch
sys.path.insert(0, '.')
import gen, oracle
import paper_2605_00342_b200 as ev
def cu(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
B, N, L, d, K, E = 1, 60, 48, 2048, 8, 128
P, Q, n = gen.trees(21, B, N, 6, 10)
sel = ev.evict_select(cu(P), cu(Q), cu(gen.cost_table(N)), n_nodes=cu(n))
b = ev.evict_build_verify_tree(cu(P), sel["keep_bits"], n_nodes=cu(n))
h = gen.hidden(31, B, N, L, d, mode=0); w = gen.wgate(32, L, E, d, mode=0)
g = ev.evict_router_union(b["verify_offsets"], b["retrieve_index"], cu(h.view(np.int16)).view(torch.bfloat16),
                          cu(w.view(np.int16)).view(torch.bfloat16), K, B, N, with_topk=True)
T = int(b["verify_offsets"][-1]); ridx = b["retrieve_index"].cpu().numpy()
tk = g["topk_ids"].cpu().numpy()
bad = 0
for l in range(L):
    for r in range(T):
        ids, lg, nt = oracle.router_topk(h[l, ridx[r]], w[l], K)
        if tk[l, r].tolist() != ids.tolist():
            bad += 1
            order = np.argsort(-lg, kind='stable')
            print('layer', l, 'row', r, 'gpu', tk[l, r].tolist(), 'oracle', ids.tolist(), 'near_tie', nt)
            print('   top logits', [(int(e), lg[e]) for e in order[:10]])
            print('   gpu logits', [(int(e), lg[e]) for e in tk[l, r]])
print('bad rows', bad, 'of', L * T)
# raw logits from TMEM
import ctypes
lg = torch.zeros((L, B * N, 128), dtype=torch.float32, device="cuda")
tr = ev._Trees(B, N, None, None, None)
hh = cu(h.view(np.int16)).view(torch.bfloat16); ww = cu(w.view(np.int16)).view(torch.bfloat16)
rt = ev._Router(L, E, K, d, ev._p(hh), ev._p(ww), 0)
uc = torch.empty((B, L), dtype=torch.int32, device="cuda"); ut = torch.empty(B, dtype=torch.int32, device="cuda")
ub = torch.empty((B, L, 2), dtype=torch.int64, device="cuda"); tk2 = torch.empty((L, B * N, K), dtype=torch.int32, device="cuda")
lib = ev.lib(); f = lib.evict_router_union_debug; f.argtypes = [ctypes.c_void_p] * 10; f.restype = ctypes.c_int
rc = f(ctypes.byref(tr), ev._p(b["verify_offsets"]), ev._p(b["retrieve_index"]), ctypes.byref(rt), ev._p(uc), ev._p(ut), ev._p(ub), ev._p(tk2), ev._p(lg), ev._stream())
torch.cuda.synchronize(); print('rc', rc)
lgn = lg.cpu().numpy(); nbad = 0; nrev = 0
for l in range(L):
    for r in range(T):
        ref = (w[l].view(np.int16).astype(np.int32) << 16).view(np.float32).astype(np.float64) @ ((h[l, ridx[r]].astype(np.int32) << 16).view(np.float32).astype(np.float64))
        if not np.array_equal(lgn[l, r], ref.astype(np.float32)):
            nbad += 1
            if nbad < 4:
                d_ = np.nonzero(lgn[l, r] != ref.astype(np.float32))[0]
                print('logit mismatch layer', l, 'row', r, [(int(e), float(lgn[l, r, e]), float(ref[e])) for e in d_[:6]])
        desc = sorted(range(128), key=lambda e: (-lgn[l, r, e], -e))[:K]
        if tk2[l, r].tolist() == desc and desc != sorted(range(128), key=lambda e: (-lgn[l, r, e], e))[:K]: nrev += 1
print('rows with logit mismatch', nbad, 'rows explained by index-desc tie order', nrev)
