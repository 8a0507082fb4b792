"""Cold-L2 graph-replay timing of evict_router_union per split override, vs torch.bmm (cuBLAS)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import gen  # noqa: E402
import paper_2605_00342_b200 as ev  # noqa: E402

shapes = {"c2": (1, 60, 6, 10, 48, 2048, 128), "c4": (64, 128, 8, 10, 48, 2048, 128),
          "c3": (16, 60, 6, 10, 94, 4096, 128), "ling1": (1, 60, 6, 10, 32, 4096, 256)}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def cold(fn, reps=50):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            fn()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        for a, b in evs:
            flush.fill_(1)
            a.record(s)
            g.replay()
            b.record(s)
    s.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in evs])) * 1e3


for name in sys.argv[1:]:
    B, Nn, steps, topk, L, d, E = shapes[name]
    P, Q, n = gen.trees(3, B, Nn, steps, topk)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    sel = ev.evict_select(cu(P), cu(Q), cu(gen.cost_table(Nn)), n_nodes=cu(n))
    b = ev.evict_build_verify_tree(cu(P), sel["keep_bits"], n_nodes=cu(n))
    h = gen.hidden_cuda(11, B, Nn, L, d, mode=1)
    w = gen.wgate_cuda(12, L, E, d, mode=1, scale_log2=-5)
    T = int(b["verify_offsets"][-1])
    byt = L * (T * d + E * d) * 2
    for S in ("auto", "1", "2", "3", "4"):
        if S == "auto":
            os.environ.pop("EVICT_ROUTER_SPLITS", None)
        else:
            os.environ["EVICT_ROUTER_SPLITS"] = S
        rc = ev.RouterCall(b["verify_offsets"], b["retrieve_index"], h, w, 8, B, Nn, max_rows=T)
        us = cold(lambda: rc())
        print(f"{name} S={S:4s} {us:7.1f} us  {byt / us / 1e3:7.0f} GB/s")
    os.environ.pop("EVICT_ROUTER_SPLITS", None)
    ridx = b["retrieve_index"][:T].long()
    x = h[:, ridx]                     # [L][T][d] kept rows (gathered outside the timed call)
    wt = w.transpose(1, 2)
    us = cold(lambda: torch.bmm(x, wt))
    print(f"{name} torch.bmm (cuBLAS, rows pre-gathered) {us:7.1f} us  {byt / us / 1e3:7.0f} GB/s")
    us = cold(lambda: w.clone())
    print(f"{name} W_g copy (read+write {2 * w.numel() * 2 / 1e6:.0f} MB) {us:7.1f} us")
