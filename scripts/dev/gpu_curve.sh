# NEXT-1 union curve: GPU parity + timing on a 400K-tree C5 shard + ncu of k_union_curve
set -x
timeout 600 python -m pytest tests/test_curve.py tests/test_gpu_parity.py tests/test_full_size.py -x -q 2>&1 | tail -5
cat > /tmp/cbench.py <<'PY'
import json, sys, torch, numpy as np, bench, gen
import paper_2605_00342_b200 as ev
M = int(sys.argv[1]) if len(sys.argv) > 1 else 400000
P, Q, n = gen.trees_cuda(5, M, 60, 6, 10)
ids = gen.routing_cuda(5, M, 60, 48, 128, 8)
cost = torch.from_numpy(gen.cost_table(60)).cuda()
s = torch.cuda.current_stream()
print(json.dumps(bench.union_curve_bench(ev, torch, P, Q, n, cost, ids, M, s)))
PY
PYTHONPATH=$PWD timeout 600 python /tmp/cbench.py 400000 2>&1 | tail -2
PYTHONPATH=$PWD timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_union_curve -s 2 -c 1 -o gpurun_out/prof_curve python /tmp/cbench.py 100000 > gpurun_out/ncu_curve.log 2>&1; tail -2 gpurun_out/ncu_curve.log
