set -x
timeout 600 python -m pytest tests/test_router.py tests/test_gpu_parity.py -q 2>&1 | tail -5
timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import json, torch, bench, gen, paper_2605_00342_b200 as ev
print(json.dumps(bench.router_bench(ev, gen, torch, torch.cuda.current_stream()), indent=0))
print(bench.latency_b64(ev, torch, gen))
"
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -k "toy or c2 or adversarial" 2>&1 | tail -4
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -k "fused_equals_oracle and c2" 2>&1 | tail -4
