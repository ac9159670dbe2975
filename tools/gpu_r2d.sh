#!/bin/bash
# A/B of the variants under lib/variants: deferral census, timing, launch lists
set -u
T=${1:-r2d}
OUT=gpurun_out/$T; mkdir -p $OUT
V=paper_1306_6291_b200/lib/variants
LIBS=${LIBS:-$(ls $V/lib_*.so | tr '\n' ' ')}
timeout 600 python tools/defer_census.py $LIBS > $OUT/census.jsonl 2> $OUT/census.err; echo "census=$?" >> $OUT/rc.txt
timeout 900 python tools/ab_libs.py $LIBS > $OUT/ab.jsonl 2> $OUT/ab.err; echo "ab=$?" >> $OUT/rc.txt
for c in ${NCU_CFGS:-c2 c3 c4}; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv python tools/ab_libs.py --reps 1 --configs $c $LIBS > $OUT/ncu_$c.log 2>&1; echo "ncu_$c=$?" >> $OUT/rc.txt
done
if [ -n "${TESTS:-}" ]; then
SD_PARITY_STATS=$OUT/parity timeout 900 python -m pytest $TESTS -q -rA -x > $OUT/pytest.log 2>&1; echo "pytest=$?" >> $OUT/rc.txt
fi
