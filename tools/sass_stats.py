#!/usr/bin/env python3
"""Static SASS statistics per kernel of the built library.

    python tools/sass_stats.py [--lib path] [--filter substr]

Counts instructions and the FP64 / MUFU / call mnemonics per function from
`cuobjdump -sass` (static counts: code size and op mix, not dynamic work).
"""

from __future__ import annotations

import argparse
import collections
import re
import subprocess
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_1306_6291_b200" / "lib" / "libsymdiag_b200.so"
OPS = ("DFMA", "DMUL", "DADD", "DSETP", "MUFU", "CALL", "BRA", "LDG", "STG", "LDS", "STS", "BSSY")


def stats(lib: Path):
    out = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True,
                         check=True).stdout
    cur, res = None, {}
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            res[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m:
            op = m.group(2)
            res[cur]["total"] += 1
            for o in OPS:
                if op.startswith(o):
                    res[cur][o] += 1
    return res


def short(name: str) -> str:
    m = re.search(r"(\d+)([a-z_0-9]+kernel)", name)
    return (m.group(2) if m else name[:40]) + ("<" + name.split("kernel", 1)[1][:12] + ">" if "kernel" in name else "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=str(LIB))
    ap.add_argument("--filter", default="")
    a = ap.parse_args()
    for name, c in sorted(stats(Path(a.lib)).items(), key=lambda x: -x[1]["total"]):
        if a.filter and a.filter not in name:
            continue
        ops = " ".join(f"{o}={c[o]}" for o in OPS if c[o])
        print(f"{c['total']:6d}  {short(name):45s} {ops}")


if __name__ == "__main__":
    main()
