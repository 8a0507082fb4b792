set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_pre python bench.py --steps 1 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ncu_pre.log 2>&1; tail -1 gpurun_out/ncu_pre.log
ls -la gpurun_out
