set -x
timeout 900 python -m pytest tests/test_router.py "tests/test_gpu_parity.py::test_fused_equals_oracle" -x -q 2>&1 | tail -15
cat > /tmp/rb.py <<'PY'
import json, torch, bench, gen
import paper_2605_00342_b200 as ev
print(json.dumps(bench.router_bench(ev, gen, torch, torch.cuda.current_stream())))
PY
PYTHONPATH=$PWD timeout 600 python /tmp/rb.py 2>&1 | tail -3
