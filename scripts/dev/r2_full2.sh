# round-2 evidence (lane-owned-column union): all GPU tests, smoke, the default bench line (all
# extras), ncu launch list, ncu --set full of the union/emit kernel and the select kernel
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -3 gpurun_out/bench_full.err
cut -c1-800 gpurun_out/bench_full.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 60 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 3 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > /dev/null 2>&1; wc -l gpurun_out/launches_r02.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_select_g|k_fused" -s 2 -c 2 -o gpurun_out/prof_r02 python bench.py --steps 1 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ncu_r02.log 2>&1; tail -1 gpurun_out/ncu_r02.log
