#!/bin/bash
# quick check: defer census, c2/c3/c4 timing, parity sweep at 2^24 rows per config
set -u
T=${1:-quick}
OUT=gpurun_out/$T; mkdir -p $OUT
python tools/defer_census.py > $OUT/census.json 2>&1; echo "census=$?" >> $OUT/rc.txt
for c in c2 c3 c4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-extra --no-e2e --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench_$c=$?" >> $OUT/rc.txt; done
if [ "${SWEEP:-1}" = "1" ]; then
SD_SWEEP_ROWS=${SWEEP_ROWS:-16777216} SD_SWEEP_CHUNKS=1 SD_PARITY_STATS=$OUT/sweep timeout 1500 python -m pytest tests/test_gpu_parity_sweep.py -q -rA -k "3x3" > $OUT/sweep.log 2>&1; echo "sweep=$?" >> $OUT/rc.txt
fi
