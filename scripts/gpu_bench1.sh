set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -c 3000 gpurun_out/bench.log
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_step -s 20 -c 1 -o gpurun_out/prof_kstep python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
tail -5 gpurun_out/ncu_full.log
