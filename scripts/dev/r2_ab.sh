# A/B of kernel variants: headline bench per library (libevict.so and libevict_<v>.so), quick parity of each
set -x
for v in "" $VARIANTS; do
  export EVICT_LIB_VARIANT=$v
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fused" 2>&1 | tail -2
  timeout 600 python bench.py --no-extras --steps 10 --warmup 3 --e2e-steps 1 --cpu-seconds 1 > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));r=d['roofline'];print('VARIANT [$v]', r['kernel_ms'], r['frac'], d['ms_per_step'])"
done
