#!/usr/bin/env python3
"""Per-source-line hot spots of one kernel from an ncu report.

    python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> <mangled-name-substring> [top] [file:line]

Joins ncu's per-SASS-address metrics (source page, SASS view) with the line
table nvdisasm -g prints for the same cubin (extracted from the in-tree
.so, which must be the build that was profiled).  Prints, per CUDA source
line, warp instructions executed, the average active threads per executed
instruction (divergence), and warp-stall samples.
"""

from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path

import os
LIB = Path(os.environ.get("SD_LIB", Path(__file__).resolve().parents[1] / "paper_1306_6291_b200"
                         / "lib" / "libsymdiag_b200.so"))


def line_table(fun_sub: str):
    tmp = Path(tempfile.mkdtemp())
    subprocess.run(["cuobjdump", "-xelf", "all", str(LIB)], cwd=tmp, capture_output=True)
    table = {}
    for cub in tmp.glob("*.cubin"):
        out = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True,
                             text=True).stdout
        cur_fun, cur_line = None, None
        for ln in out.splitlines():
            m = re.match(r"\.text\.(\S+):", ln)
            if m:
                cur_fun = m.group(1)
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur_line = f"{Path(m.group(1)).name}:{m.group(2)}"
                continue
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
            if m and cur_fun and fun_sub in cur_fun:
                table[int(m.group(1), 16)] = cur_line
        if table:
            break
    return table


def main():
    rep, kre, fun_sub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    dump = sys.argv[5] if len(sys.argv) > 5 else None  # print this line's SASS
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    table = line_table(fun_sub)
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, ""])
    base = None
    for r in rows[hi + 1:]:
        if len(r) != len(hdr):
            break
        d = dict(zip(hdr, r))
        try:
            addr = int(d["Address"], 16)
        except ValueError:
            continue
        if base is None:
            base = addr  # ncu prints absolute addresses; nvdisasm function offsets
        addr -= base
        line = table.get(addr, "?")
        a = agg[line]
        if dump and line == dump:
            print(f"{addr:6x} {d['Instructions Executed']:>10s} {d['Thread Instructions Executed']:>12s}  {d['Source']}")
        a[0] += float(d["Instructions Executed"] or 0)
        a[1] += float(d["Thread Instructions Executed"] or 0)
        a[2] += float(d["Warp Stall Sampling (All Samples)"] or 0)
        if not a[3]:
            a[3] = d["Source"][:50]
    tot_i = sum(v[0] for v in agg.values()) or 1
    tot_s = sum(v[2] for v in agg.values()) or 1
    print(f"{'line':32s} {'inst%':>6s} {'thr/inst':>8s} {'stall%':>6s}  first SASS")
    for line, (ni, nt, ns, src) in sorted(agg.items(), key=lambda x: -x[1][2])[:top]:
        print(f"{line:32s} {100 * ni / tot_i:6.2f} {nt / ni if ni else 0:8.1f} {100 * ns / tot_s:6.2f}  {src}")


if __name__ == "__main__":
    main()
