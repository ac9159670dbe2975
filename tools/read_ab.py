#!/usr/bin/env python3
"""Print the A/B timings and per-call kernel durations of a tools/gpu_r2d.sh run.

    python tools/read_ab.py gpurun_out/<tag>
"""
import csv
import json
import sys
from pathlib import Path

d = Path(sys.argv[1])
libs = []
for l in open(d / "ab.jsonl"):
    r = json.loads(l)
    if r["lib"] not in libs:
        libs.append(r["lib"])
    print(r["config"], r["lib"], round(r["ms_median"], 4), "status_diff", r["status_diff_vs_first"])
for c in ("c2", "c3", "c4"):
    f = d / f"launches_{c}.csv"
    if not f.exists():
        continue
    rows = list(csv.reader(open(f)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    kn, mv = h.index("Kernel Name"), h.index("Metric Value")
    seq = [float(r[mv].replace(",", "")) / 1000 for r in rows[hi + 1:] if len(r) > mv and "eig3" in r[kn]]
    calls = [seq[i:i + 5] for i in range(0, len(seq), 5)]
    print(c, "(fast, pass, exact, polish, literal) us, last call of each library")
    for name, cl in zip(libs, calls[-len(libs):]):
        print("  ", name, [round(v, 1) for v in cl], "tail", round(sum(cl[1:]), 1))
