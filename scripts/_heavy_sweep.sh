#!/bin/bash
# config 5 step time vs the HBM-state kernel's split length (grid mode)
for h in 128 1024 2048 4096 8192 16384; do
  timeout 300 python scripts/probe_config.py 5 --modes 2 --outer 1 --heavy $h 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'step_us' in d: print('heavy', $h, 'step_us', round(d['step_us'],2))"
done
