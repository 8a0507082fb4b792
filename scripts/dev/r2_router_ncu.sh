# ncu --set full of the router (A8) launches at the bench's C2 / C3 / C4 shapes (first 3 k_router launches)
set -x
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_router" -c 3 -o gpurun_out/prof_router python bench.py --steps 1 --warmup 3 --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ncu_router.log 2>&1; tail -2 gpurun_out/ncu_router.log
