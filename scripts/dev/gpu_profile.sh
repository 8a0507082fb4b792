# tests + full-size bench + ncu launch list + ncu --set full of the fused kernel
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|ncclDevKernel" --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > /dev/null 2>&1; tail -8 gpurun_out/launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
