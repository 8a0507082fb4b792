set -x
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -6
cat > /tmp/lb.py <<'PY'
import json, torch, bench, gen
import paper_2605_00342_b200 as ev
M = 1000000
P, Q, n = gen.trees_cuda(5, M, 60, 6, 10)
cost = torch.from_numpy(gen.cost_table(60)).cuda()
print(json.dumps(bench.ling_variant(ev, gen, torch, P, Q, n, cost, M, torch.cuda.current_stream(), 10)))
PY
PYTHONPATH=$PWD timeout 600 python /tmp/lb.py 2>&1 | tail -2
PYTHONPATH=$PWD timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_ling python /tmp/lb.py > gpurun_out/ncu_ling.log 2>&1; tail -1 gpurun_out/ncu_ling.log
