#!/bin/bash
set -u
T=${1:-it3}
OUT=gpurun_out/$T; mkdir -p $OUT
V=paper_1306_6291_b200/lib/variants
LIBS="$V/lib_r2a.so $V/lib_v3.so $V/lib_v3pl.so" bash tools/gpu_ab.sh $T
SD_PARITY_STATS=$OUT/parity timeout 900 python -m pytest tests -m gpu -q -rA -k "sign_stage or polish or golden" > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
for v in v3 v3pl; do
SD_LIB_PATH=$V/lib_$v.so SD_SWEEP_ROWS=16777216 SD_SWEEP_CHUNKS=1 SD_PARITY_STATS=$OUT/sweep_$v timeout 1200 python -m pytest tests/test_gpu_parity_sweep.py -q -rA -k "3x3 and (c3 or c4)" > $OUT/sweep_$v.log 2>&1; echo "sweep_$v=$?" >> $OUT/rc.txt
done
LIBS="$V/lib_r2a.so $V/lib_v3.so" bash tools/gpu_prof_ab.sh ${T}_prof c3
