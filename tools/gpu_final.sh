#!/bin/bash
# Full check of the current build: smoke, GPU suite, 2^26 sweeps, bench (default + reference
# arm + --gpus 1 one-process path), launch list, ncu --set full of one c2 call -> summary.
set -u
T=${1:-final}
OUT=gpurun_out/$T; mkdir -p $OUT
{ nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv; } > $OUT/env.txt 2>&1
python __graft_entry__.py > $OUT/smoke.log 2>&1; echo "smoke=$?" >> $OUT/rc.txt
SD_PARITY_STATS=$OUT/parity timeout 1500 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench=$?" >> $OUT/rc.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "bench_ref=$?" >> $OUT/rc.txt
CMD="python bench.py --config c2 --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu"
$CMD > $OUT/plain.json 2> $OUT/plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2.csv $CMD > $OUT/ncu_launch.log 2>&1; echo "ncu_launch=$?" >> $OUT/rc.txt
ncu --set full --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum --clock-control none --import-source on -k regex:eig3 -s 15 -c 5 -o $OUT/prof_c2 $CMD > $OUT/ncu_full.log 2>&1; echo "ncu_full=$?" >> $OUT/rc.txt
python tools/ncu_summary.py $OUT/prof_c2.ncu-rep --config c2 --n 16777216 --out $OUT/ncu_summary.json --source "ncu --set full + sass thread-inst metrics of one sd_eig3_f64 call (5 kernels) of: $CMD" > $OUT/ncu_summary.log 2>&1; echo "summary=$?" >> $OUT/rc.txt
timeout 900 python bench.py --steps 3 --warmup 3 --sweep --no-extra --no-e2e --no-cpu > $OUT/bench_sweep.json 2> $OUT/bench_sweep.err; echo "bench_sweep=$?" >> $OUT/rc.txt
for c in c3 c4; do
C="python bench.py --config $c --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv $C > $OUT/ncu_launch_$c.log 2>&1; echo "ncu_launch_$c=$?" >> $OUT/rc.txt
done
if [ "${SWEEP:-1}" = "1" ]; then
SD_SWEEP_ROWS=16777216 SD_SWEEP_CHUNKS=4 SD_PARITY_STATS=$OUT/sweep timeout 2400 python -m pytest tests/test_gpu_parity_sweep.py -q -rA > $OUT/sweep.log 2>&1; echo "sweep=$?" >> $OUT/rc.txt
fi
