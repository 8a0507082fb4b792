set -x
EVICT_LIB_VARIANT=pt timeout 300 python scripts/dev/phase_timing.py 2>&1 | tail -7
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lean" 2>&1 | tail -2
timeout 300 python -c "
import bench, json, torch, gen
import paper_2605_00342_b200 as ev
out = {}
for B, N, s, t in ((64, 60, 6, 10), (1, 60, 6, 10), (1024, 60, 6, 10)):
    out.update(bench.latency(ev, torch, gen, B=B, N=N, steps=s, topk=t))
print('LATENCY', json.dumps(out))
"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
