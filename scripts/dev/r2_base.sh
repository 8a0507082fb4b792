# round 2 baseline on a fresh box: GPU tests, smoke, short headline bench, ncu source-level capture of k_fused
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --no-extras --steps 10 --warmup 3 --e2e-steps 1 --cpu-seconds 2 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err; tail -2 gpurun_out/bench_h.err; cut -c1-1200 gpurun_out/bench_h.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
