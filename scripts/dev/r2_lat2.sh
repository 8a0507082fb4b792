# serving-batch kernel with the column union: parity + graph-capture tests, latency lines, headline
set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_graph_capture_gpu.py -m gpu -q -x --tb=short 2>&1 | grep -E "Error|assert|differs|passed|failed" | head -10
timeout 300 python -c "
import bench, json, torch, gen
import paper_2605_00342_b200 as ev
out = {}
for B, N, s, t in ((64, 60, 6, 10), (1, 60, 6, 10), (64, 128, 8, 10)):
    out.update(bench.latency(ev, torch, gen, B=B, N=N, steps=s, topk=t))
print('LATENCY', json.dumps(out))
"
timeout 600 python bench.py --no-extras --steps 10 --warmup 3 --e2e-steps 1 --cpu-seconds 1 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err
python -c "import json;d=json.load(open('gpurun_out/bench_h.json'));r=d['roofline'];print('HEADLINE', r['kernel_ms'], r['frac'], d['ms_per_step'], d['value'])"
