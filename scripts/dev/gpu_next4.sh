set -x
timeout 600 python -m pytest tests/test_dispatch_gpu.py tests/test_curve.py tests/test_abi.py -x -q 2>&1 | tail -15
