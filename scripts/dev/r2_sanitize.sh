# compute-sanitizer memcheck + racecheck over small invocations of every kernel (round 2 paths included)
set -x
for part in fused fusedbig router verify draft; do
  PYTHONPATH=$PWD timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/dev/sanitize_driver.py $part > gpurun_out/memcheck_$part.log 2>&1; tail -3 gpurun_out/memcheck_$part.log
done
for part in fused fusedbig verify draft; do
  PYTHONPATH=$PWD timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/dev/sanitize_driver.py $part > gpurun_out/racecheck_$part.log 2>&1; tail -3 gpurun_out/racecheck_$part.log
done
