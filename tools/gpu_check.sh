#!/bin/bash
# One gpurun call: smoke, GPU parity suite, bench.  Outputs under gpurun_out/<tag>/.
#   gpurun --timeout 2400 -- bash tools/gpu_check.sh <tag> [bench args...]
set -u
TAG=${1:-run}; shift || true
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
{ nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv; } > "$OUT/env.txt" 2>&1
python __graft_entry__.py > "$OUT/smoke.log" 2>&1; echo "smoke=$?" >> "$OUT/rc.txt"
SD_PARITY_STATS=$OUT/parity timeout 1800 python -m pytest tests -m gpu -q -rA > "$OUT/pytest_gpu.log" 2>&1; echo "pytest=$?" >> "$OUT/rc.txt"
timeout 900 python bench.py --steps 10 --warmup 3 "$@" > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench=$?" >> "$OUT/rc.txt"
