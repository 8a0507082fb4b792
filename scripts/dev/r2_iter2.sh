# parity of the throughput path (select + union/emit), full-size, headline bench, ncu of both kernels
set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --tb=short  2>&1 | grep -E "Error|assert|differs|passed|failed" | head -20
timeout 900 python -m pytest tests/test_full_size.py tests/test_shards_gpu.py -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --no-extras --steps 10 --warmup 3 --e2e-steps 1 --cpu-seconds 1 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err
python -c "import json;d=json.load(open('gpurun_out/bench_h.json'));r=d['roofline'];print('HEADLINE', r['kernel_ms'], r['frac'], d['ms_per_step'], d['value'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_select_g|k_fused" -s 2 -c 2 -o gpurun_out/prof_it python bench.py --steps 1 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ncu_it.log 2>&1; tail -1 gpurun_out/ncu_it.log
