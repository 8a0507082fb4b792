set -x
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_router -s 6 -c 1 -o gpurun_out/prof_router python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, gen, paper_2605_00342_b200 as ev
print(bench.router_bench(ev, gen, torch, torch.cuda.current_stream()))
" > gpurun_out/ncu_router.log 2>&1; tail -2 gpurun_out/ncu_router.log
