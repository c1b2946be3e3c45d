ARGS="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o gpurun_out/prof_cluster python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
python scripts/phase_profile.py --ctas 0 --modes 1 2>&1 | grep -v "^{"
