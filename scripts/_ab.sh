#!/bin/bash
# A/B of prebuilt library variants (_variants/*.so) on one config, interleaved repetitions
cfg=${1:-2}; reps=${2:-3}; shift 2; vs=${@:-v0 v1}
mkdir -p gpurun_out
cp paper_1306_4080_b200/libpcdn.so /tmp/libpcdn_keep.so
for r in $(seq $reps); do
  for v in $vs; do
    cp _variants/$v.so paper_1306_4080_b200/libpcdn.so
    timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$v rep$r cfg$cfg', round(d['ms_per_step'],4), round(r['launch_ms'],4))"
  done
done
cp /tmp/libpcdn_keep.so paper_1306_4080_b200/libpcdn.so
