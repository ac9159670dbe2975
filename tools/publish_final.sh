#!/bin/bash
# Copy the artifacts of a tools/gpu_final.sh run (gpurun_out/<tag>) into profiles/r2
set -eu
R=gpurun_out/$1; P=profiles/r2
cp $R/bench.json $P/bench_c2.json
cp $R/bench_sweep.json $P/bench_c2_sweep.json
cp $R/bench_reference.json $P/bench_reference.json
cp $R/launches_c2.csv $R/launches_c3.csv $R/launches_c4.csv $P/
cp $R/pytest_gpu.log $R/smoke.log $R/env.txt $P/
python - <<PY
import json
new = json.load(open('$R/ncu_summary.json'))
try:
    old = json.load(open('profiles/ncu_summary.json'))
except (OSError, ValueError):
    old = {}
old.update(new)  # keeps the other configs' captures (c3: profiles/r2/ncu_summary_c3.json)
json.dump(old, open('profiles/ncu_summary.json', 'w'), indent=1)
PY
rm -rf $P/parity $P/parity_sweep
cp -r $R/parity $P/parity
mkdir -p $P/parity_sweep
cp $R/sweep/* $P/parity_sweep/
cp $R/sweep.log $P/parity_sweep/sweep.log
python - <<PY
import json
d = json.load(open('profiles/ncu_summary.json'))
with open('$P/ncu_c2_kernels.jsonl', 'w') as f:
    for k in d['c2']['kernels']:
        f.write(json.dumps(k) + '\n')
PY
python tools/ncu_functions.py $R/prof_c2.ncu-rep eig3_fast eig3_fast_kernelIdLb1 > $P/fast_kernel_functions.txt
