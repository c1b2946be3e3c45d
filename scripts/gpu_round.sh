#!/bin/bash
# One GPU pass: parity tests, bench line, ncu launch list, one ncu --set full of k_step.
# Usage (from the repo root, on the B200 box): bash scripts/gpu_round.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -c 2500 $OUT/bench.json
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 python bench.py $ARGS > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py $ARGS > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 20 -c 1 \
    -o $OUT/prof_kstep python bench.py $ARGS > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 $OUT/ncu_full.log
