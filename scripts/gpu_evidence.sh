#!/bin/bash
# Evidence pass of a round on one B200 (scripts/gpu_evidence.sh <tag>): the GPU tests, smoke, the
# default bench line and the reference arm, bench lines of configs 1-4, the step-kernel floors,
# config 5's P extension, config 3's P sweep with the CPU oracle at P = 1, the ncu launch list of
# the default bench command, the step kernel's DRAM traffic (profiles/traffic.json) and one
# `ncu --set full` capture of it.  Everything lands in gpurun_out/<tag>/.
TAG=${1:-r2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PCDN_SYNTH_CACHE=/tmp/pcdn_synth
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" $OUT/pytest_gpu.log | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; echo "cfg$c rc=$?"
done
timeout 600 python bench.py --config 5 --loss 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_cfg5_svm.json 2> $OUT/bench_cfg5_svm.err; echo "cfg5 svm rc=$?"
timeout 900 python scripts/step_floor.py > $OUT/step_floor.jsonl 2>&1; echo "floor rc=$?"
timeout 900 python scripts/probe_config.py 5 --P 4096,29500,100000,1000000 --modes 2,5 --outer 1 > $OUT/pext_cfg5.jsonl 2>&1; echo "pext rc=$?"
timeout 900 python scripts/probe_config.py 5 --loss 1 --P 4096,100000,1000000 --modes 2 --outer 1 > $OUT/pext_cfg5_svm.jsonl 2>&1
timeout 1200 python scripts/p_sweep_cfg3.py 1,64,1024,8192 --oracle-p1 > $OUT/psweep_cfg3.jsonl 2>&1; echo "cfg3 sweep rc=$?"
PCDN_LIB=paper_1306_4080_b200/libpcdn_prof.so timeout 900 python scripts/probe_config.py 5 --P 4096,100000 --modes 2 --outer 1 --profile > $OUT/phases_cfg5.jsonl 2>&1
PCDN_LIB=paper_1306_4080_b200/libpcdn_prof.so timeout 600 python scripts/cta_profile.py 5 > $OUT/cta_cfg5.json 2>/dev/null
ARGS="--steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 600 python bench.py $ARGS > $OUT/plain.json 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py $ARGS > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_step_sparse --csv --log-file $OUT/traffic.csv python bench.py $ARGS > $OUT/ncu_traffic.log 2>&1
echo "ncu traffic rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_step_sparse --launch-skip 2 --launch-count 1 \
    -o $OUT/prof_kstep -f python bench.py $ARGS > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
