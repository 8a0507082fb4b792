"""Small invocations of every kernel of libevict.so, for compute-sanitizer (memcheck / racecheck)."""
import sys

import numpy as np
import torch

import gen
import paper_2605_00342_b200 as ev
from gen import verify as gv
from gen.draft import drafter_tables

which = sys.argv[1] if len(sys.argv) > 1 else "all"
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
B, N, L, E, K = 40, 60, 48, 128, 8
P, Q, n = gen.trees(2, B, N, 6, 10)
ids = gen.routing(2, B, N, L, E, K)
cost = cu(gen.cost_table(N))
if which in ("all", "fused"):
    g = ev.evict_select_build_union(cu(P), cu(Q), cost, cu(ids), E, n_nodes=cu(n))
    g = ev.evict_select_build_union(cu(P), cu(Q), cost, cu(ids), E, n_nodes=cu(n), with_bits=True, with_order=True)
    s = ev.evict_select(cu(P), cu(Q), cost, n_nodes=cu(n), with_order=True)
    ev.evict_union_curve(s["order"], cu(ids), E, n_nodes=cu(n), per_layer=True)
    b = ev.evict_build_verify_tree(cu(P), s["keep_bits"], n_nodes=cu(n))
    ev.evict_expert_union(s["keep_bits"], cu(ids), E, n_nodes=cu(n))
if which in ("all", "fusedbig"):
    # the throughput path (select launch + offset scan + union/emit, folded A9) and pinned host ids
    Bb = 2600
    Pb, Qb, nb = gen.trees(3, Bb, N, 6, 10)
    idsb = gen.routing(3, Bb, N, L, E, K)
    ev.evict_select_build_union(cu(Pb), cu(Qb), cost, cu(idsb), E, n_nodes=cu(nb), with_stats=True)
    ev.evict_select_build_union(cu(Pb), cu(Qb), cost, torch.from_numpy(idsb).pin_memory(), E, n_nodes=cu(nb))
    ev.evict_select_build_union(cu(P), cu(Q), cost, cu(ids), E, n_nodes=cu(n), with_stats=True)
if which in ("all", "router"):
    s = ev.evict_select(cu(P), cu(Q), cost, n_nodes=cu(n))
    b = ev.evict_build_verify_tree(cu(P), s["keep_bits"], n_nodes=cu(n))
    for Ex in (8, 100, 128, 200, 256):
        h = gen.hidden_cuda(3, B, N, 4, 256, mode=1)
        w = gen.wgate_cuda(4, 4, Ex, 256, mode=1)
        ev.evict_router_union(b["verify_offsets"], b["retrieve_index"], h, w, 8, B, N)
if which in ("all", "verify"):
    V = 3000
    s = ev.evict_select(cu(P), cu(Q), cost, n_nodes=cu(n))
    b = ev.evict_build_verify_tree(cu(P), s["keep_bits"], n_nodes=cu(n))
    tok = gv.draft_tokens(5, P, V, n_nodes=n)
    probs = torch.rand((B * N, V), device="cuda")
    probs = probs / probs.sum(1, keepdim=True)
    ua, ub = gv.uniforms(5, B, N)
    for greedy, exact in ((False, False), (False, True), (True, False)):
        ev.evict_verify_sample(b["verify_offsets"], b["next_token"], b["next_sibling"], b["retrieve_index"], cu(tok),
                               probs, u_accept=cu(ua.view(np.int32)), u_bonus=cu(ub.view(np.int32)),
                               greedy=greedy, exact=exact)
if which in ("all", "draft"):
    for Bx, steps, topk, Nx in ((40, 6, 10, 60), (700, 4, 8, 32), (8, 9, 15, 128)):
        t, p = drafter_tables(7, Bx, steps, topk)
        ev.evict_build_draft_tree(cu(t), cu(p), Nx)
torch.cuda.synchronize()
print("sanitize driver ok:", which)
