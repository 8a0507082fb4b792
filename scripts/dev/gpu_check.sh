set -x
free -g | head -2; nproc; nvidia-smi -L; nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py --trees 200000 --steps 5 --warmup 3 --e2e-steps 1 --cpu-seconds 4 2>&1 | tail -5
