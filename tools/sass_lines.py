#!/usr/bin/env python3
"""Executed instructions per source line of one kernel in an ncu report.

    python tools/sass_lines.py REPORT.ncu-rep LIB.so KERNEL_SUBSTR [--id N] [--top 40]

ncu's source page (--print-source=sass) gives per-SASS-instruction counts
(instructions executed, warp-stall samples); `nvdisasm -g` of the library's
cubin maps each SASS offset to the (inlined) CUDA file:line.  The two are
joined by offset from the function start and aggregated per line and per
file.  Needs the library the report was captured with (same build).
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def line_map(lib: str, kernel: str):
    tmp = Path(tempfile.mkdtemp())
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(lib).resolve())], cwd=tmp,
                   check=True, capture_output=True)
    for cub in sorted(tmp.glob("*.cubin")):
        out = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True,
                             text=True).stdout
        m = None
        cur = None
        offs = {}
        inside = False
        for ln in out.splitlines():
            if ln.startswith("//----") and ".text." in ln:
                name = ln.split(".text.")[1].split()[0]
                inside = kernel in name and (m is None or m == name)
                if inside:
                    m = name
                continue
            if not inside:
                continue
            fm = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
            if fm:
                cur = (Path(fm.group(1)).name, int(fm.group(2)))
                continue
            im = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", ln)
            if im:
                offs[int(im.group(1), 16)] = (cur, im.group(2))
        if offs:
            return m, offs
    raise SystemExit(f"kernel {kernel} not found in {lib}")


def ncu_rows(rep: str, kid: int):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'(?m)^"Kernel Name",', txt)[1:]
    blk = blocks[kid]
    lines = blk.splitlines()[1:]
    rd = csv.DictReader(io.StringIO("\n".join(lines)))
    rows = [r for r in rd if r.get("Address", "").startswith("0x")]
    base = int(rows[0]["Address"], 16)
    return [(int(r["Address"], 16) - base, r) for r in rows]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("lib")
    ap.add_argument("kernel")
    ap.add_argument("--id", type=int, default=0)
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    name, offs = line_map(a.lib, a.kernel)
    rows = ncu_rows(a.report, a.id)
    per_line = collections.Counter()
    per_file = collections.Counter()
    stall = collections.Counter()
    total = 0
    miss = 0
    for off, r in rows:
        n = int(float(r["Instructions Executed"] or 0))
        s = int(float(r.get("Warp Stall Sampling (All Samples)", 0) or 0))
        total += n
        if off not in offs:
            miss += n
            continue
        src, _ = offs[off]
        per_line[src] += n
        stall[src] += s
        per_file[src[0] if src else None] += n
    print(f"{name}: {total} warp instructions executed ({miss} unmapped)")
    for f, n in per_file.most_common():
        print(f"  {str(f):24s} {n:14d} {100.0 * n / total:6.2f}%")
    print("top lines:")
    tot_s = sum(stall.values()) or 1
    for src, n in per_line.most_common(a.top):
        print(f"  {str(src):36s} {n:14d} {100.0 * n / total:6.2f}%  stall {100.0 * stall[src] / tot_s:5.2f}%")


if __name__ == "__main__":
    sys.exit(main())
