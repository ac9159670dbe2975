#!/bin/bash
# iteration check: A/B of variant libs, selected GPU tests, 2^24-row sweeps (main lib)
set -u
T=${1:-iter}; shift || true
OUT=gpurun_out/$T; mkdir -p $OUT
V=paper_1306_6291_b200/lib/variants
if [ -n "${LIBS:-}" ]; then
timeout 900 python tools/ab_libs.py $LIBS > $OUT/ab.jsonl 2> $OUT/ab.err; echo "ab=$?" >> $OUT/rc.txt
fi
if [ -n "${TESTK:-}" ]; then
SD_PARITY_STATS=$OUT/parity timeout 1200 python -m pytest tests -m gpu -q -rA -k "$TESTK" > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
fi
if [ -n "${SWEEP:-}" ]; then
SD_SWEEP_ROWS=${SWEEP_ROWS:-16777216} SD_SWEEP_CHUNKS=${SWEEP_CHUNKS:-1} SD_PARITY_STATS=$OUT/sweep timeout 1800 python -m pytest tests/test_gpu_parity_sweep.py -q -rA -k "$SWEEP" > $OUT/sweep.log 2>&1; echo "sweep=$?" >> $OUT/rc.txt
fi
