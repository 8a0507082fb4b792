# ncu source-level captures of the two throughput kernels (select, union/emit) at the headline shape
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --no-extras --steps 10 --warmup 3 --e2e-steps 1 --cpu-seconds 1 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err
python -c "import json;d=json.load(open('gpurun_out/bench_h.json'));r=d['roofline'];print('HEADLINE', r['kernel_ms'], r['frac'], d['ms_per_step'], d['value'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_select_g|k_fused" -s 6 -c 3 -o gpurun_out/prof_sel python bench.py --steps 1 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ncu_sel.log 2>&1; tail -3 gpurun_out/ncu_sel.log
