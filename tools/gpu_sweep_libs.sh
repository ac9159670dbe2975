#!/bin/bash
# A/B timing of variant libs + 2^24-row sweeps run through each variant (SD_LIB_PATH)
set -u
T=${1:-sw}
OUT=gpurun_out/$T; mkdir -p $OUT
V=paper_1306_6291_b200/lib/variants
LIBS="$LIBS" bash tools/gpu_ab.sh $T
for L in $SWEEP_LIBS; do
  nm=$(basename $L .so)
  SD_LIB_PATH=$L SD_SWEEP_ROWS=16777216 SD_SWEEP_CHUNKS=1 SD_PARITY_STATS=$OUT/sweep_$nm timeout 1200 python -m pytest tests/test_gpu_parity_sweep.py -q -rA -k "${SWEEPK:-3x3}" > $OUT/sweep_$nm.log 2>&1; echo "sweep_$nm=$?" >> $OUT/rc.txt
done
