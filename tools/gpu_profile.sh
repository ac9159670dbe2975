#!/bin/bash
# One gpurun call: plain bench run, then (only if it exited 0) the ncu launch
# list and one `--set full` capture of the eig3 kernels of one step.
#   gpurun --timeout 1800 -- bash tools/gpu_profile.sh <tag> [config] [n]
set -u
TAG=${1:-prof}; CFG=${2:-c2}; N=${3:-2097152}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --n $N --no-extra --no-e2e --no-cpu"
$CMD > "$OUT/plain.json" 2> "$OUT/plain.err" && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" $CMD > "$OUT/ncu_launch.log" 2>&1; echo "ncu_launch=$?" >> "$OUT/rc.txt"
ncu --set full --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum --clock-control none --import-source on -k regex:eig[23] -s ${SKIP:-9} -c ${COUNT:-3} -o "$OUT/prof" $CMD > "$OUT/ncu_full.log" 2>&1; echo "ncu_full=$?" >> "$OUT/rc.txt"
