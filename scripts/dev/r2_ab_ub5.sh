# A/B: union load batch 4 (default) vs 5 (libevict_ub5.so)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --tb=short -k "throughput or lean or stats or fused" 2>&1 | grep -E "Error|assert|passed|failed" | head -5
timeout 900 python -m pytest tests/test_full_size.py -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do
for v in "" ub5; do
EVICT_LIB_VARIANT=$v timeout 600 python bench.py --no-extras --steps 10 --warmup 3 --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ab_$v$i.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/ab_$v$i.json'));r=d['roofline'];print('AB', '$v', r['kernel_ms'], r['frac'])"
done; done
