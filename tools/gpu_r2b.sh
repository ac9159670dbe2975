#!/bin/bash
# tests + 2^26 parity sweep + bench of the current build
set -u
T=${1:-r2b}
OUT=gpurun_out/$T; mkdir -p $OUT
python __graft_entry__.py > $OUT/smoke.log 2>&1; echo "smoke=$?" >> $OUT/rc.txt
SD_PARITY_STATS=$OUT/parity timeout 1500 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
SD_SWEEP_ROWS=16777216 SD_SWEEP_CHUNKS=4 SD_PARITY_STATS=$OUT/sweep timeout 1500 python -m pytest tests/test_gpu_parity_sweep.py -q -rA > $OUT/sweep.log 2>&1; echo "sweep=$?" >> $OUT/rc.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench=$?" >> $OUT/rc.txt
