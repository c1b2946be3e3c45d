#!/bin/bash
# quick iteration pass: GPU parity tests, then device-timed bench lines of the given configs
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt.log
grep -E "FAILED|Error" gpurun_out/pt.log | head -5
for c in ${@:-1 2 3}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/q$c.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('cfg$c', 'ms/solve', round(d['ms_per_step'],3), 'frac', round(r['frac'],4), 'launch_ms', round(r['launch_ms'],4), d.get('outer_iters'))" || tail -3 gpurun_out/q$c.err
done
