# usage: bash scripts/_ab.sh TAG "probe args" variant...   (variant 'cur' = the in-tree library)
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
    if 'step_us' in r: print('$v', r['cfg'], r['P'], r.get('debug',0), 'step_us %.2f'%r['step_us'], 'F %.9f'%r['F'])
"
done
