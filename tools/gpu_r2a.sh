#!/bin/bash
# round-2 check: smoke, GPU tests, bench (N=1), bench --gpus 1 path sanity, profile c2
set -u
OUT=gpurun_out/r2a; mkdir -p $OUT
bash tools/gpu_check.sh r2a
SKIP=4 COUNT=4 bash tools/gpu_profile.sh r2a_prof c2 16777216
python tools/ncu_summary.py gpurun_out/r2a_prof/prof.ncu-rep --config c2 --n 16777216 --out gpurun_out/r2a_prof/ncu_summary.json --source "ncu --set full + sass thread-inst metrics, one sd_eig3 call (4 kernels) of bench.py --config c2 --n 16777216" > gpurun_out/r2a_prof/summary.log 2>&1
echo done
