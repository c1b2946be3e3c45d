#!/bin/bash
# ncu --set full of one launch of the top step kernel on the default bench workload.
# usage: bash scripts/gpu_ncu_top.sh <tag> <kernel regex> [bench args...]
TAG=$1; KRE=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e $*"
timeout 300 python bench.py $ARGS > $OUT/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 20 -c 1 \
    -o $OUT/prof_kstep python bench.py $ARGS > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -2 $OUT/ncu_full.log
