set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_shards_gpu.py tests/test_full_size.py -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --no-extras --steps 10 --warmup 3 --e2e-steps 1 --cpu-seconds 1 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err
python -c "import json;d=json.load(open('gpurun_out/bench_h.json'));r=d['roofline'];print('HEADLINE', r['kernel_ms'], r['frac'], d['ms_per_step'], d['value'], d['stats_allreduced_trees'], d['k_star_mean'])"
tail -3 gpurun_out/bench_h.err
