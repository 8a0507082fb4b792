set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py tests/test_shards_gpu.py -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --no-extras --steps 10 --warmup 3 --e2e-steps 1 --cpu-seconds 1 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err
python -c "import json;d=json.load(open('gpurun_out/bench_h.json'));r=d['roofline'];print('HEADLINE', r['kernel_ms'], r['frac'], d['ms_per_step'], d['value'])"
tail -2 gpurun_out/bench_h.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 6 --csv --log-file gpurun_out/pre_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > /dev/null 2>&1; grep -c k_ gpurun_out/pre_launches.csv
