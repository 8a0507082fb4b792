set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stats or pinned or lean" 2>&1 | tail -2
timeout 600 python bench.py --no-extras --steps 10 --warmup 3 --e2e-steps 1 --cpu-seconds 1 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err
python -c "import json;d=json.load(open('gpurun_out/bench_h.json'));r=d['roofline'];print('HEADLINE', r['kernel_ms'], r['frac'], d['ms_per_step'], d['value']); print('E2E', d['e2e'])"
timeout 300 python scripts/dev/router_trace.py 2>&1 | tail -7
for s in c2 c4 ling1; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/dev/router_probe.py $s > gpurun_out/router_$s.csv 2>/dev/null; done
timeout 600 python -c "
import bench, json, torch, gen
import paper_2605_00342_b200 as ev
print('ROUTER', json.dumps(bench.router_bench(ev, gen, torch, torch.cuda.current_stream())))
"
