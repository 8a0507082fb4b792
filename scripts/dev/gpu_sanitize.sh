# compute-sanitizer memcheck + racecheck over small invocations of every kernel; the end-to-end graph test
set -x
timeout 600 python -m pytest tests/test_graph_capture_gpu.py -x -q 2>&1 | tail -5
for part in fused router verify draft; do
  PYTHONPATH=$PWD timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_driver.py $part > gpurun_out/memcheck_$part.log 2>&1; tail -3 gpurun_out/memcheck_$part.log
done
for part in fused verify draft; do
  PYTHONPATH=$PWD timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_driver.py $part > gpurun_out/racecheck_$part.log 2>&1; tail -3 gpurun_out/racecheck_$part.log
done
