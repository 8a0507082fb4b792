# iterate: targeted GPU tests, short headline bench, ncu source-level capture of k_fused
set -x
timeout 1200 python -m pytest tests/test_router.py tests/test_gpu_parity.py tests/test_verify_gpu.py tests/test_full_size.py -m gpu -q -x 2>&1 | tail -8
timeout 900 python bench.py --no-extras --steps 10 --warmup 3 --e2e-steps 1 --cpu-seconds 2 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err; tail -2 gpurun_out/bench_h.err; cut -c1-1500 gpurun_out/bench_h.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
