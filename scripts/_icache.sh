#!/bin/bash
# instruction-cache hit/miss counters of the top step kernel (ncu, one launch)
M=sm__icc_requests.sum,sm__icc_requests_lookup_hit.sum,sm__icc_requests_lookup_miss.sum,gcc__cache_requests_type_instruction_lookup_hit.sum,gcc__cache_requests_type_instruction_lookup_miss.sum,gpu__time_duration.sum,smsp__inst_executed.sum
for spec in "2 k_step_res" "4 k_step_dense" "3 k_step_res"; do
  set -- $spec
  timeout 600 ncu --metrics $M --clock-control none -k regex:$2 -s 5 -c 1 --csv python bench.py --config $1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"(sm__|gcc__|gpu__|smsp__)' | awk -F'","' -v cfg=$1 '{print "cfg" cfg, $(NF-2), $NF}'
done
