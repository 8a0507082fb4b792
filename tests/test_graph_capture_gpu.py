"""Every call of the path is stream-ordered and CUDA-graph capturable (the
EVICT ops run inside the captured draft graph): one graph holds draft-tree build → fused
select/build/union → the target's (stand-in) row gather → Eq. 3 tree sampling, and replaying
it on fresh inputs reproduces eager execution bit for bit."""
import numpy as np
import pytest

import gen
from gen import verify as gv
from gen.draft import drafter_tables

pytestmark = pytest.mark.gpu


def _step(ev, torch, bufs, s):
    """One decoding step on static buffers (no host reads, no allocation in the path calls)."""
    d = ev.evict_build_draft_tree(bufs["ctok"], bufs["cprob"], bufs["N"], out=bufs["tree"], stream=s)
    f = ev.evict_select_build_union(d["parent"], d["q"], bufs["cost"], bufs["ids"], bufs["E"],
                                    n_nodes=d["n_nodes"], buffers=bufs["fused"], stream=s)
    # stand-in for the target's verify pass: its next-token rows in packed verify order (rows past
    # the step's T = verify_offsets[B] are capacity, not written by the library: clamp their index)
    ri = f["retrieve_index"].clamp(0, bufs["node_probs"].shape[0] - 1).long()
    torch.index_select(bufs["node_probs"], 0, ri, out=bufs["probs"])
    return ev.evict_verify_sample(f["verify_offsets"], f["next_token"], f["next_sibling"], f["retrieve_index"],
                                  d["tokens"], bufs["probs"], u_accept=bufs["ua"], u_bonus=bufs["ub"],
                                  out=bufs["vout"], stream=s)


def test_full_step_in_one_graph():
    import torch
    import paper_2605_00342_b200 as ev
    B, steps, topk, N, L, E, K, V = 32, 6, 10, 60, 48, 128, 8, 4096
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731

    def inputs(seed):
        tok, pr = drafter_tables(seed, B, steps, topk, V=V)
        ids = gen.routing(seed, B, N, L, E, K)
        rng = np.random.default_rng(seed)
        node_probs = rng.dirichlet(np.ones(V) * 0.05, size=B * N).astype(np.float32)
        ua, ub = gv.uniforms(seed, B, N)
        return dict(ctok=tok, cprob=pr, ids=ids, node_probs=node_probs, ua=ua.view(np.int32), ub=ub.view(np.int32))

    first = inputs(1)
    bufs = {k: cu(v) for k, v in first.items()}
    bufs.update(N=N, E=E, cost=cu(gen.cost_table(N)), probs=torch.empty((B * N, V), device="cuda"),
                fused=ev.FusedBuffers(B, N, L, E, "cuda"),
                tree=dict(parent=torch.empty((B, N), dtype=torch.int32, device="cuda"),
                          q=torch.empty((B, N), dtype=torch.float32, device="cuda"),
                          tokens=torch.empty((B, N), dtype=torch.int32, device="cuda"),
                          n_nodes=torch.empty(B, dtype=torch.int32, device="cuda"),
                          status=torch.empty(B, dtype=torch.int32, device="cuda")),
                vout=dict(accept_len=torch.empty(B, dtype=torch.int32, device="cuda"),
                          accepted_slots=torch.empty((B, N), dtype=torch.int32, device="cuda"),
                          bonus_token=torch.empty(B, dtype=torch.int32, device="cuda"),
                          status=torch.empty(B, dtype=torch.int32, device="cuda")))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        _step(ev, torch, bufs, s)                      # warm-up (eager)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            _step(ev, torch, bufs, s)
    keys = ("k_star", "keep_bits", "union_total", "verify_offsets")
    for seed in (2, 3):
        new = inputs(seed)
        for k, v in new.items():
            bufs[k].copy_(cu(v))
        with torch.cuda.stream(s):
            g.replay()
            s.synchronize()
            got = {k: v.clone() for k, v in bufs["vout"].items()}
            got.update({k: bufs["fused"].t[k].clone() for k in keys})
            _step(ev, torch, bufs, s)                  # eager on the same inputs
            s.synchronize()
        for k in ("accept_len", "accepted_slots", "bonus_token", "status"):
            assert torch.equal(got[k], bufs["vout"][k]), k
        for k in keys:
            assert torch.equal(got[k], bufs["fused"].t[k]), k
        assert int((bufs["vout"]["status"] != 0).sum()) == 0 and int(bufs["vout"]["accept_len"].min()) >= 1
