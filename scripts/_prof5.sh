timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python scripts/probe_config.py ${1:-5} --P ${2:-4096} --modes ${3:-1,2} --outer 1 --profile > gpurun_out/prof5.jsonl 2>&1
python -c "
import json
N=['A rest', 'sync1', 'C1', 'C2', 'C3', 'win', 'commit', 'sync3', 'A light', 'Ap search', 'Ap rounds', 'Ap gridsync']
for l in open('gpurun_out/prof5.jsonl'):
    d=json.loads(l)
    if 'phase_cycles' not in d: print(l.strip()[:300]); continue
    print(d['P'], d['mode_used'], round(d['step_us'],2), ' '.join('%s=%.2f' % (n, c/1965.0) for n,c in zip(N, d['phase_cycles'])))
"
