# quick iteration: GPU tests, full bench, ncu --set full of the fused kernel
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25
timeout 900 python bench.py --cpu-seconds 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
