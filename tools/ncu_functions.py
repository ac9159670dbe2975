#!/usr/bin/env python3
"""Per-function instruction shares of one kernel from an ncu report.

    python tools/ncu_functions.py <report.ncu-rep> <kernel-regex> <mangled-substring>

Runs tools/ncu_lines.py (per-source-line warp instructions, active threads
per instruction, stall samples; the in-tree .so must be the profiled build)
and sums its lines per device function of sd_fast3.cuh / per file.
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rep, kre, sub = sys.argv[1:4]
out = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_lines.py"), rep, kre, sub, "5000"],
                     capture_output=True, text=True).stdout
src = (ROOT / "paper_1306_6291_b200" / "csrc" / "sd_fast3.cuh").read_text().splitlines()
starts = []
for i, l in enumerate(src, 1):
    m = re.match(r"(?:SD_FM|template <[^>]*>\s*)?(?:__device__ __forceinline__|__device__ __noinline__|SD_FM)"
                 r"\s+[\w:<>\*& ]+?\s+(\w+)\(", l)
    if m:
        starts.append((i, m.group(1)))


def fn(line):
    name = "?"
    for i, n in starts:
        if i <= line:
            name = n
        else:
            break
    return name


agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for l in out.splitlines():
    p = l.split()
    if len(p) < 4 or ":" not in p[0]:
        continue
    f, ln = p[0].rsplit(":", 1)
    try:
        inst, thr, st = float(p[1]), float(p[2]), float(p[3])
    except ValueError:
        continue
    key = (f, fn(int(ln))) if f == "sd_fast3.cuh" else (f, "")
    a = agg[key]
    a[0] += inst
    a[1] += inst * thr
    a[2] += st
print(f"{'file':22s} {'function':18s} {'inst%':>6s} {'thr/inst':>8s} {'stall%':>6s}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    if a[0] < 0.05:
        continue
    print(f"{k[0]:22s} {k[1]:18s} {a[0]:6.2f} {a[1] / a[0]:8.1f} {a[2]:6.2f}")
