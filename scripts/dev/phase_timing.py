"""k_fused phase breakdown (EVICT_LIB_VARIANT=pt, built with -DEVICT_PHASE_TIMING): warp-cycles
per tree spent in select / publish+early look-back / union / late look-back / emit."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import gen  # noqa: E402
import paper_2605_00342_b200 as ev  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
P, Q, n = gen.trees_cuda(5, M, 60, 6, 10)
ids = gen.routing_cuda(5, M, 60, 48, 128, 8)
cost = torch.from_numpy(gen.cost_table(60)).cuda()
call = ev.FusedCall(P, Q, cost, ids, 128, n_nodes=n)
f = ev.lib().evict_debug_phase_cycles
f.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 8)()
for _ in range(3):
    call()
torch.cuda.synchronize()
f(buf)
reps = 5
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    call()
e1.record()
torch.cuda.synchronize()
f(buf)
ms = e0.elapsed_time(e1) / reps
names = ["select", "publish+early lookback", "union", "late lookback", "emit"]
tot = sum(buf[i] for i in range(5))
print(f"M={M} k_fused {ms:.3f} ms (instrumented)")
for i, nm in enumerate(names):
    print(f"{nm:24s} {buf[i] / reps / M:9.1f} warp-cycles/tree  {100 * buf[i] / tot:5.1f}%")
