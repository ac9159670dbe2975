#!/bin/bash
set -u
T=${1:-it4}
OUT=gpurun_out/$T; mkdir -p $OUT
V=paper_1306_6291_b200/lib/variants
LIBS="${LIBS:-$V/lib_r2a.so $V/lib_v3.so $V/lib_v4.so}" bash tools/gpu_ab.sh $T
[ -n "${CEN:-}" ] && python tools/defer_census.py $CEN > $OUT/census.jsonl 2>&1
SD_PARITY_STATS=$OUT/parity timeout 900 python -m pytest tests -m gpu -q -rA -k "${TESTK:-sign_stage or golden or fast_path or large_prefix or adversarial or f32}" > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
SD_SWEEP_ROWS=16777216 SD_SWEEP_CHUNKS=1 SD_PARITY_STATS=$OUT/sweep timeout 1200 python -m pytest tests/test_gpu_parity_sweep.py -q -rA -k "${SWEEPK:-3x3}" > $OUT/sweep.log 2>&1; echo "sweep=$?" >> $OUT/rc.txt
