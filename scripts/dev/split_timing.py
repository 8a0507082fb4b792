"""Time the three separate calls (select, build, union) on the C5 sweep vs the fused launch."""
import sys

import torch

sys.path.insert(0, ".")
import gen  # noqa: E402
import paper_2605_00342_b200 as ev  # noqa: E402

M = 1_000_000
P, Q, n = gen.trees_cuda(5, M, 60, 6, 10)
ids = gen.routing_cuda(5, M, 60, 48, 128, 8)
cost = torch.from_numpy(gen.cost_table(60)).cuda()


def t(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


sel = ev.evict_select(P, Q, cost, n_nodes=n)
keep = sel["keep_bits"]
print("select  ms", t(lambda: ev.evict_select(P, Q, cost, n_nodes=n)))
print("build   ms", t(lambda: ev.evict_build_verify_tree(P, keep, n_nodes=n)))
print("union   ms", t(lambda: ev.evict_expert_union(keep, ids, 128, n_nodes=n)))
call = ev.FusedCall(P, Q, cost, ids, 128, n_nodes=n)
print("fused   ms", t(lambda: call()))
