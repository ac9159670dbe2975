#!/usr/bin/env python3
"""Dynamic SASS opcode mix of one kernel from an ncu report.

    python tools/ncu_ops.py <report.ncu-rep> <kernel-regex> [rows]

Sums ncu's per-address "Instructions Executed" (warp level) and "Thread
Instructions Executed" by opcode; with `rows` also prints per-row counts
(warp instructions x 32 / rows = issue slots per row at full warps).
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys


def main():
    rep, kre = sys.argv[1:3]
    rows_n = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    launches = 0
    for r in rows[hi + 1:]:
        if len(r) != len(hdr):
            if r and r[0] == "Address":
                launches += 1
            continue
        if r == hdr:
            launches += 1
            continue
        d = dict(zip(hdr, r))
        src = d["Source"].strip()
        if not src:
            continue
        toks = src.split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        a = agg[op]
        a[0] += float(d["Instructions Executed"] or 0)
        a[1] += float(d["Thread Instructions Executed"] or 0)
    tot = sum(v[0] for v in agg.values()) or 1
    print(f"{'op':10s} {'warp-inst%':>10s} {'thr/inst':>8s}" + ("  per-row" if rows_n else ""))
    for op, (ni, nt) in sorted(agg.items(), key=lambda x: -x[1][0]):
        if ni / tot < 0.002:
            continue
        extra = f"  {ni * 32 / rows_n:8.1f}" if rows_n else ""
        print(f"{op:10s} {100 * ni / tot:10.2f} {nt / ni:8.1f}{extra}")
    print(f"total warp inst {tot:.4g}" + (f"  per row (x32) {tot * 32 / rows_n:.1f}" if rows_n else ""))


if __name__ == "__main__":
    main()
