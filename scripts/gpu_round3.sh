#!/bin/bash
# Evidence pass: GPU tests, the default bench line (config 2, CPU baseline + e2e), the reference
# arm, bench lines of configs 1, 3, 4, 5 (LR) and 5 (SVM), ncu launch list of the default run and
# ncu --set full of the cluster-resident (config 2) and dense (config 4) step kernels.
TAG=${1:-r19}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
for c in 1 3 4 5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; echo "cfg$c rc=$?"
done
timeout 900 python bench.py --config 5 --loss 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_cfg5_svm.json 2> $OUT/bench_cfg5_svm.err; echo "cfg5 svm rc=$?"
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 python bench.py $ARGS > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py $ARGS > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python bench.py --config 4 $ARGS > $OUT/plain4.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg4.csv \
    python bench.py --config 4 $ARGS > $OUT/ncu_launch4.log 2>&1; echo "ncu launches cfg4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_res -s 20 -c 1 \
    -o $OUT/prof_kstep python bench.py $ARGS > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_dense -s 2 -c 1 \
    -o $OUT/prof_dense python bench.py --config 4 $ARGS > $OUT/ncu_dense.log 2>&1; echo "ncu dense rc=$?"
