set -x
timeout 900 python -m pytest tests/test_router.py -m gpu -q -x 2>&1 | tail -3
timeout 300 python scripts/dev/router_trace.py 2>&1 | tail -3 | cut -c1-400
for s in c2 c4 ling1; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/dev/router_probe.py $s > gpurun_out/router_$s.csv 2>/dev/null; done
timeout 600 python -c "
import bench, json, torch, gen
import paper_2605_00342_b200 as ev
r = bench.router_bench(ev, gen, torch, torch.cuda.current_stream())
print('ROUTER', {k: (round(v['us'], 1), round(v['hbm_frac'], 3)) for k, v in r.items()})
"
