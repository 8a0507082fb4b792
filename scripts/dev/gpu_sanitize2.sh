set -x
for part in router verify draft; do
  CUDA_MODULE_LOADING=EAGER PYTHONPATH=$PWD timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_driver.py $part > gpurun_out/memcheck_eager_$part.log 2>&1; tail -2 gpurun_out/memcheck_eager_$part.log
  PYTHONPATH=$PWD timeout 900 compute-sanitizer --tool memcheck --report-api-errors no --print-limit 20 python scripts/sanitize_driver.py $part > gpurun_out/memcheck_dev_$part.log 2>&1; tail -2 gpurun_out/memcheck_dev_$part.log
done
PYTHONPATH=$PWD timeout 900 compute-sanitizer --tool initcheck --report-api-errors no --print-limit 20 python scripts/sanitize_driver.py verify > gpurun_out/initcheck_verify.log 2>&1; tail -2 gpurun_out/initcheck_verify.log
PYTHONPATH=$PWD timeout 900 compute-sanitizer --tool synccheck --report-api-errors no --print-limit 20 python scripts/sanitize_driver.py verify > gpurun_out/synccheck_verify.log 2>&1; tail -2 gpurun_out/synccheck_verify.log
