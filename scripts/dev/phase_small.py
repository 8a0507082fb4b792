"""Phase breakdown of the serving-batch fused call (EVICT_LIB_VARIANT=pt): warp-cycles per tree."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import gen  # noqa: E402
import paper_2605_00342_b200 as ev  # noqa: E402

for B in (64, 1):
    P, Q, n = gen.trees_cuda(4, B, 60, 6, 10)
    ids = gen.routing_cuda(4, B, 60, 48, 128, 8)
    cost = torch.from_numpy(gen.cost_table(60)).cuda()
    call = ev.FusedCall(P, Q, cost, ids, 128, n_nodes=n)
    f = ev.lib().evict_debug_phase_cycles
    f.argtypes = [ctypes.c_void_p]
    buf = (ctypes.c_ulonglong * 8)()
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    f(buf)
    reps = 50
    for _ in range(reps):
        call()
    torch.cuda.synchronize()
    f(buf)
    names = ["select", "publish+early lookback", "union", "late lookback", "emit"]
    print(f"B={B}: " + ", ".join(f"{nm} {buf[i] / reps / B / 1965:.2f} us" for i, nm in enumerate(names)))
