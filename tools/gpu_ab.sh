#!/bin/bash
# A/B of library builds under paper_1306_6291_b200/lib/variants + launch lists
set -u
T=${1:-ab}; shift || true
OUT=gpurun_out/$T; mkdir -p $OUT
V=paper_1306_6291_b200/lib/variants
LIBS=${LIBS:-"$V/lib_r2a.so $V/lib_abcd.so $V/lib_head.so"}
timeout 900 python tools/ab_libs.py $LIBS > $OUT/ab.jsonl 2> $OUT/ab.err; echo "ab=$?" >> $OUT/rc.txt
for c in c2 c3; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv python tools/ab_libs.py --reps 1 --configs $c $LIBS > $OUT/ncu_$c.log 2>&1; echo "ncu_$c=$?" >> $OUT/rc.txt
done
if [ -n "${TESTS:-}" ]; then
SD_PARITY_STATS=$OUT/parity timeout 900 python -m pytest $TESTS -q -rA -x > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
fi
