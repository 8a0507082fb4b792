set -x
timeout 300 python scripts/dev/split_timing.py 2>&1 | tail -4
EVICT_LIB_VARIANT=tlpt timeout 300 python scripts/dev/phase_timing.py 2>&1 | tail -6
EVICT_LIB_VARIANT=pt timeout 300 python scripts/dev/phase_timing.py 2>&1 | tail -6
VARIANTS=tl bash scripts/dev/r2_ab.sh 2>&1 | grep VARIANT
