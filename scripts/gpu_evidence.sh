#!/bin/bash
# Evidence pass on one B200 (scripts/gpu_evidence.sh <tag>): compute-sanitizer over every launch
# mode, the ncu launch list of the default bench command, the DRAM traffic of the step kernel
# (profiles/traffic.json), and one `ncu --set full` capture of the step kernel (config 5).
TAG=${1:-r2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PCDN_SYNTH_CACHE=/tmp/pcdn_synth
python -c "import __graft_entry__ as g; g.build()" > /dev/null
if [ "${SAN:-1}" = 1 ]; then
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 100 --kernel-name-exclude regex:at::|vectorized|elementwise|reduce_kernel \
      python scripts/sanitize_cases.py --quick > $OUT/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 $OUT/sanitizer_$tool.log
done
fi
ARGS="--steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 600 python bench.py $ARGS > $OUT/plain.json 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py $ARGS > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_step_sparse --csv --log-file $OUT/traffic.csv python bench.py $ARGS > $OUT/ncu_traffic.log 2>&1
echo "ncu traffic rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_step_sparse --launch-skip 2 --launch-count 1 \
    -o $OUT/prof_kstep -f python bench.py $ARGS > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
