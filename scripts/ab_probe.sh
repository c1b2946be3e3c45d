#!/bin/bash
# A/B timing of library variants on the GPU box: bash scripts/ab_probe.sh TAG "probe_config args" VARIANT...
# VARIANT 'cur' = the in-tree libpcdn.so, any other name = scratch/libpcdn_NAME.so (built by
# scripts/ab_build.sh).  One scripts/probe_config.py run per variant (PCDN_LIB), output in
# gpurun_out/TAG/VARIANT.jsonl, one summary line per (config, P) printed.
TAG=$1; ARGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PCDN_SYNTH_CACHE=/tmp/pcdn_synth
for v in "$@"; do
  if [ "$v" = cur ]; then L=paper_1306_4080_b200/libpcdn.so; else L=scratch/libpcdn_$v.so; fi
  PCDN_LIB=$L timeout 600 python scripts/probe_config.py $ARGS > $OUT/$v.jsonl 2>&1
  python -c "
import json,sys
for l in open('$OUT/$v.jsonl'):
    try: r=json.loads(l)
    except Exception: continue
    if 'step_us' in r: print('$v', r['cfg'], r['P'], r['mode_used'], 'step_us %.2f'%r['step_us'], 'F %.9f'%r['F'])
"
done
