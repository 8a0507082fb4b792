# headline k_fused: lean-path parity, a short bench (no extras), ncu full of one k_fused launch
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -x -q 2>&1 | tail -4
timeout 900 python bench.py --no-extras --steps 10 --warmup 3 --e2e-steps 1 --cpu-seconds 2 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err; tail -2 gpurun_out/bench_h.err; cut -c1-1500 gpurun_out/bench_h.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
