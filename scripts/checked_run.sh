#!/bin/bash
# The GPU test suite and every launch mode's small cases against the checked build
# (libpcdn_checked.so: device-side bounds / protocol checks, -DPCDN_CHECKS=1) -- the substitute for
# compute-sanitizer, which is closed on this pool.  Logs to gpurun_out/<tag>/checked_*.log.
TAG=${1:-r2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PCDN_SYNTH_CACHE=/tmp/pcdn_synth
python -c "
import sys; sys.path.insert(0, '.')
from paper_1306_4080_b200 import build as b
print(b.build(checks=True))" || exit 1
export PCDN_LIB=$PWD/paper_1306_4080_b200/libpcdn_checked.so
timeout 900 python scripts/checked_cases.py > $OUT/checked_cases.log 2>&1; echo "cases rc=$?"; tail -2 $OUT/checked_cases.log
timeout 2400 python -m pytest tests -m gpu -q > $OUT/checked_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|PCDN_CHECK" $OUT/checked_pytest.log | tail -5
