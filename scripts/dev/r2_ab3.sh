set -x
VARIANTS=wsv bash scripts/dev/r2_ab.sh 2>&1 | grep "VARIANT\|passed\|failed\|Error"
EVICT_LIB_VARIANT=wsv timeout 900 python -m pytest tests/test_full_size.py -m gpu -q -x 2>&1 | tail -3
