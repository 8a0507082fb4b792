set -x
timeout 900 python -m pytest tests/test_router.py -m gpu -q -x 2>&1 | tail -2
timeout 600 python scripts/dev/router_sweep.py c2 c4 ling1 c3 2>&1 | grep -v Warn
