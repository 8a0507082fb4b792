set -x
timeout 900 python -m pytest tests/test_draft_gpu.py tests/test_abi.py -x -q 2>&1 | tail -15
cat > /tmp/db.py <<'PY'
import json, torch, bench
import paper_2605_00342_b200 as ev
print(json.dumps(bench.draft_bench(ev, torch, torch.cuda.current_stream())))
PY
PYTHONPATH=$PWD timeout 600 python /tmp/db.py 2>&1 | tail -3
PYTHONPATH=$PWD timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_draft -s 25 -c 1 -o gpurun_out/prof_draft python /tmp/db.py > gpurun_out/ncu_draft.log 2>&1; tail -2 gpurun_out/ncu_draft.log
