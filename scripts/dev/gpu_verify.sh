# NEXT-3 verify sampling: GPU parity + the verify sub-benchmark + ncu of k_verify
set -x
timeout 600 python -m pytest tests/test_verify_gpu.py -x -q 2>&1 | tail -15
PYTHONPATH=$PWD timeout 600 python - <<'PY' > gpurun_out/verify_bench.json 2> gpurun_out/verify_bench.err
import json, torch, bench, gen
import paper_2605_00342_b200 as ev
s = torch.cuda.current_stream()
print(json.dumps(bench.verify_bench(ev, gen, torch, s)))
PY
tail -3 gpurun_out/verify_bench.err; cat gpurun_out/verify_bench.json
cat > /tmp/vprof.py <<'PY'
import torch, bench, gen
import paper_2605_00342_b200 as ev
bench.verify_bench(ev, gen, torch, torch.cuda.current_stream())
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_verify -s 5 -c 1 -o gpurun_out/prof_verify env PYTHONPATH=$PWD python /tmp/vprof.py > gpurun_out/ncu_verify.log 2>&1; tail -3 gpurun_out/ncu_verify.log
