#!/bin/bash
# persisting-L2 window on/off for the HBM-state kernel on config 5 (both losses), step time and DRAM bytes
for l2 in 0 1; do
  for P in 4096 100000; do
    timeout 300 python scripts/probe_config.py 5 --P $P --modes 2 --outer 1 --l2 $l2 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'step_us' in d: print('l2', $l2, 'P', d['P'], 'step_us', round(d['step_us'],2), 'GB/s', round(d['kernel_alg_GBs'],1))"
  done
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:k_step -s 1 -c 1 --csv python scripts/probe_config.py 5 --modes 2 --outer 1 --l2 $l2 2>/dev/null | grep -E '"(dram|lts|gpu)__' | awk -F'","' -v l2=$l2 '{print "ncu l2=" l2, $(NF-2), $(NF-1), $NF}'
done
