#!/bin/bash
# ncu --set full of one grid step-kernel launch on config 5 at a large bundle size
P=${1:-1000000}
OUT=gpurun_out/cfg5p; mkdir -p $OUT
timeout 300 python scripts/probe_config.py 5 --P $P --modes 2 --outer 1 > $OUT/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 1 -c 1 \
    -o $OUT/prof_p$P python scripts/probe_config.py 5 --P $P --modes 2 --outer 1 > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
