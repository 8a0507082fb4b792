# round-2 evidence: all GPU tests, smoke, the default bench line (all extras), ncu launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -3 gpurun_out/bench_full.err
cut -c1-600 gpurun_out/bench_full.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 60 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 3 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > /dev/null 2>&1; wc -l gpurun_out/launches_r02.csv
