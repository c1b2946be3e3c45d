#!/bin/bash
# ncu --set full of one real (not a queued no-op) k_step_res launch of the default bench run:
# a solve is 6 step launches + 1 queued no-op; skip 15 = the second launch of the third solve
TAG=${1:-r23}; OUT=gpurun_out/$TAG; mkdir -p $OUT
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_res -s 15 -c 1 \
    -o $OUT/prof_kstep python bench.py $ARGS > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
