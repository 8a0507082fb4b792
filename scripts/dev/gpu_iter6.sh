set -x
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -8
python scripts/router_trace.py 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value', d['value'], 'kernel_ms', d['roofline']['kernel_ms'], 'frac', d['roofline']['frac'], 'step_ms', d['ms_per_step'])
print('mask', d.get('variants')); print('router', json.dumps(d.get('router'))); print('lat', d.get('latency')); print('e2e', d['e2e']['value'], 'cpu', d['cpu_baseline']['value'], 'clocks', d.get('clocks'))"
