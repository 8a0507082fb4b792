"""NEXT-4: on-device verify-graph dispatch — the verify graph matching the
selected length is chosen and run inside one CUDA graph, with no host round trip."""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu


def _capture(fn, stream):
    import torch
    g = torch.cuda.CUDAGraph(keep_graph=True)
    with torch.cuda.graph(g, stream=stream):
        fn()
    return g


def test_switch_runs_the_body_of_the_smallest_length_that_fits():
    import torch
    import paper_2605_00342_b200 as ev
    s = torch.cuda.Stream()
    lengths = [4, 8, 16, 32, 64]
    marker = torch.zeros(1, dtype=torch.int32, device="cuda")
    rows = torch.zeros(1, dtype=torch.int32, device="cuda")
    chosen = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    with torch.cuda.stream(s):
        bodies = [_capture(lambda i=i: marker.fill_(100 + i), s) for i in range(len(lengths))]
    d = ev.VerifyDispatch(lengths, bodies, rows, chosen)
    for T in (0, 1, 4, 5, 8, 9, 31, 32, 33, 64, 65, 1000):
        marker.fill_(-1)
        rows.fill_(T)
        d.launch(s)
        s.synchronize()
        want = next((i for i, L in enumerate(lengths) if L >= T), -1)
        assert int(chosen.item()) == want, T
        assert int(marker.item()) == (100 + want if want >= 0 else -1), T
    d.close()


def test_pre_graph_selection_and_verify_in_one_launch():
    """pre = the captured EVICT step (fused select → build → union) on a batch of trees; the
    dispatch then reads verify_offsets[B] on the device and runs the matching verify body."""
    import torch
    import paper_2605_00342_b200 as ev
    B, N, L, E, K = 4, 60, 48, 128, 8
    P, Q, n = gen.trees(2, B, N, 6, 10)
    ids = gen.routing(2, B, N, L, E, K)
    cost = gen.cost_table(N)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    s = torch.cuda.Stream()
    lengths = [8, 16, 24, 32, 48, 64, 96, 128, 192, 240]
    marker = torch.zeros(1, dtype=torch.int32, device="cuda")
    chosen = torch.zeros(1, dtype=torch.int32, device="cuda")
    with torch.cuda.stream(s):
        call = ev.FusedCall(cu(P), cu(Q), cu(cost), cu(ids), E, n_nodes=cu(n))
        call(s)                                   # warm-up outside capture
        pre = _capture(lambda: call(s), s)
        rows = call.buffers.t["verify_offsets"][B:]
        bodies = [_capture(lambda i=i: marker.fill_(i), s) for i in range(len(lengths))]
    d = ev.VerifyDispatch(lengths, bodies, rows, chosen, pre=pre)
    marker.fill_(-1)
    d.launch(s)
    s.synchronize()
    T = int(oracle.select(P, Q, cost, n_nodes=n)["k_star"].sum())   # the oracle's verify rows
    want = next(i for i, Lx in enumerate(lengths) if Lx >= T)
    assert int(rows.item()) == T and int(chosen.item()) == want and int(marker.item()) == want


def test_dispatch_rejects_bad_arguments():
    import torch
    import paper_2605_00342_b200 as ev
    s = torch.cuda.Stream()
    rows = torch.zeros(1, dtype=torch.int32, device="cuda")
    with torch.cuda.stream(s):
        g = _capture(lambda: rows.add_(0), s)
    with pytest.raises(ev.EvictError):
        ev.VerifyDispatch([8, 8], [g, g], rows)       # lengths not strictly ascending
