#!/usr/bin/env python3
"""Markdown rows of DESIGN.md's parity tables from a SD_PARITY_STATS directory.

    python tools/parity_table.py gpurun_out/<tag>/parity [gpurun_out/<tag>/sweep]
"""
import json
import sys
from pathlib import Path


def g(x):
    return "—" if x is None else (f"{x:.1e}" if isinstance(x, float) else str(x))


def row(name, f):
    if not f.exists():
        return
    s = json.loads(f.read_text())
    print(f"| {name} ({s.get('n')}) | {s.get('code_mismatch')} / {s.get('sign_mismatch')} | "
          f"{g(s.get('lam_max_err'))} | {g(s.get('strict_ang_max'))} ({s.get('strict_ang_fail')}) | "
          f"{g(s.get('edge_ang_max'))} | {g(s.get('polished_ang_max'))} | "
          f"{100 * s.get('lam_bit_equal_frac', 0):.0f}% / {100 * s.get('ang_bit_equal_frac', 0):.0f}% | "
          f"flagged {s.get('flagged')} unexplained {s.get('unexplained')} recon_worse {s.get('recon_worse')} |")


d = Path(sys.argv[1])
print("| set (rows) | code / sign | max dlam | strict ang max (fails) | edge max | polished max | bit-equal lam/ang | notes |")
for name in ("golden_c2", "golden_c3", "golden_c4", "golden_edge", "golden_u11", "golden_adv",
             "golden_lastbit", "lastbit_family", "oracle_c2_262144", "oracle_c3_262144",
             "oracle_c4_131072", "oracle_adversarial", "oracle_rotated_scalar",
             "fast_vs_literal_c2", "fast_vs_literal_c3", "fast_vs_literal_c4"):
    row(name, d / f"{name}.json")
if len(sys.argv) > 2:
    for c in ("c2", "c3", "c4"):
        row(f"sweep {c}", Path(sys.argv[2]) / f"sweep_{c}.json")
