timeout 300 python scripts/probe_config.py ${1:-4} --modes 4 --outer 1 --profile > gpurun_out/profd.jsonl 2>&1
python -c "
import json
N=['prefetch issue', 'B1', 'D finish', 'B2', 'X dx', 'LS+spec', 'G', '-', 'tile wait', 'decide prev']
for l in open('gpurun_out/profd.jsonl'):
    d=json.loads(l)
    if 'phase_cycles' not in d: print(l.strip()[:200]); continue
    print(d['P'], d['mode_used'], round(d['step_us'],2), ' '.join('%s=%.2f' % (n, c/1965.0) for n,c in zip(N, d['phase_cycles'])))
"
