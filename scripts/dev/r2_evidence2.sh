set -x
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -s 12 -c 6 --csv --log-file gpurun_out/dram_r02.csv python bench.py --steps 2 --warmup 3 --no-extras --e2e-steps 1 --cpu-seconds 1 > /dev/null 2>&1; wc -l gpurun_out/dram_r02.csv
bash scripts/dev/r2_sanitize.sh 2>&1 | grep -v "^+" 
