#!/bin/bash
# phase profile of the grid step kernel on config 5 at the given bundle sizes (no tests)
for P in "$@"; do
timeout 300 python scripts/probe_config.py 5 --P $P --modes 2 --outer 1 --profile 2>/dev/null | python -c "
import json,sys
N=['A rest', 'sync1', 'C1', 'C2', 'C3', 'win', 'commit', 'sync3', 'A light+mid', 'Ap search', 'Ap rounds', 'Ap gridsync']
for l in sys.stdin:
    d=json.loads(l)
    if 'phase_cycles' not in d: continue
    print(d['P'], round(d['step_us'],2), 'GB/s %.0f' % d['kernel_alg_GBs'], ' '.join('%s=%.2f' % (n, c/1965.0) for n,c in zip(N, d['phase_cycles']) if c))"
done
