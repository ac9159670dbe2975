#!/bin/bash
# ncu --set full of the fast kernel for two library builds (first call of each, after warm-up)
set -u
T=${1:-profab}; CFG=${2:-c2}; shift 2 || true
OUT=gpurun_out/$T; mkdir -p $OUT
V=paper_1306_6291_b200/lib/variants
LIBS=${LIBS:-"$V/lib_r2a.so $V/lib_head.so"}
NL=$(echo $LIBS | wc -w)
python tools/ab_libs.py --reps 1 --configs $CFG --n ${N:-4194304} $LIBS > $OUT/plain.jsonl 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:eig3_fast -s $((3*NL)) -c $NL -o $OUT/prof python tools/ab_libs.py --reps 1 --configs $CFG --n ${N:-4194304} $LIBS > $OUT/ncu.log 2>&1; echo "ncu=$?" >> $OUT/rc.txt
