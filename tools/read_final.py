#!/usr/bin/env python3
"""Summarise a tools/gpu_final.sh run: bench lines, sweeps, launch lists, ncu summary.

    python tools/read_final.py gpurun_out/<tag>
"""
import csv
import glob
import json
import sys
from pathlib import Path

d = Path(sys.argv[1])
b = json.loads((d / "bench.json").read_text().strip().splitlines()[-1])
print("c2", b["value"], b["ms_per_step"], "frac", b["roofline"]["frac"], "thr/inst",
      b["roofline"].get("ncu_threads_per_inst"), "e2e", b["e2e"]["value"], b["clocks"])
for k, v in b["configs_extra"].items():
    print(k, v.get("value"), v.get("ms_per_step"), "hbm", v.get("hbm_roofline_frac"),
          "fp64", v.get("fp64_executed_frac"))
print("cpu", b["cpu_baseline"])
for f in sorted(glob.glob(str(d / "sweep" / "*.json"))):
    s = json.load(open(f))
    keys = ["n", "code_mismatch", "sign_mismatch", "lam_fail", "lam_max_err", "strict_ang_fail",
            "strict_ang_max", "edge_ang_max", "polished_ang_max", "unexplained", "recon_worse",
            "status_mismatch", "lam_bit_equal", "phi_max"]
    print(Path(f).name, {k: s.get(k) for k in keys if k in s})
for c in ("c2", "c3", "c4"):
    rows = list(csv.reader(open(d / f"launches_{c}.csv")))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    kn, mv = h.index("Kernel Name"), h.index("Metric Value")
    seq = [float(r[mv].replace(",", "")) / 1000 for r in rows[hi + 1:] if len(r) > mv and "eig3" in r[kn]]
    print(c, "last call (fast, pass, exact, polish, literal) us", [round(v, 1) for v in seq[-5:]])
n = json.load(open(d / "ncu_summary.json"))["c2"]
k = n["kernels"][0]
print("ncu fast kernel", {x: k[x] for x in ("duration_ns", "fp64_pipe_pct", "issue_active_pct",
                                            "threads_per_inst", "occupancy_pct", "registers",
                                            "stall_share")})
print("fp64_thread_inst_per_row", n["fp64_thread_inst_per_row"], "dram", n["dram_bytes_per_launch"])
