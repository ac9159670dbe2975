#!/usr/bin/env python3
"""Summarise an ncu --set full report: one block of key metrics per kernel.

    python tools/ncu_summary.py gpurun_out/<tag>/prof.ncu-rep [--json out.json]
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc_per_sm",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
    "smsp__inst_executed.sum": "warp_inst",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma_thread_inst",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul_thread_inst",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd_thread_inst",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def summarise(rep: str):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = {"kernel": d.get("Kernel Name", "")[:80]}
        for m, name in KEYS.items():
            if m in d and d[m] not in ("", "n/a"):
                v = d[m].replace(",", "")
                try:
                    k[name] = float(v)
                except ValueError:
                    k[name] = v
            if m in d:
                u = units[hdr.index(m)]
                if u == "Mbyte" and name.endswith("bytes"):
                    k[name] = k[name] * 1e6
                elif u == "Gbyte" and name.endswith("bytes"):
                    k[name] = k[name] * 1e9
                elif u == "Kbyte" and name.endswith("bytes"):
                    k[name] = k[name] * 1e3
                elif u in ("usecond", "us") and name == "duration_ns":
                    k[name] = k[name] * 1e3
                elif u in ("msecond", "ms") and name == "duration_ns":
                    k[name] = k[name] * 1e6
        stalls = {h[len(STALLS):]: float(d[h]) for h in hdr
                  if h.startswith(STALLS) and not h.endswith("not_issued") and d[h] not in ("", "0")}
        tot = sum(stalls.values()) or 1.0
        k["stall_share"] = {s: round(v / tot, 3) for s, v in
                            sorted(stalls.items(), key=lambda x: -x[1])[:6]}
        out.append(k)
    return out


def update_profile_summary(rep: str, config: str, n: int, path: str, source: str,
                           bytes_per_row: int):
    """Write profiles/ncu_summary.json[config] from the kernels of ONE call
    (the captured launches of one sd_eig3 / sd_eig2 call, in launch order):
    per-kernel metrics, DRAM bytes per call and the executed FP64
    thread-instructions per row that bench.py's roofline uses."""
    import os
    ks = summarise(rep)
    doc = json.load(open(path)) if os.path.exists(path) else {}
    dram = sum(k.get("dram_read_bytes", 0) + k.get("dram_write_bytes", 0) for k in ks)
    fp64 = sum(k.get("dfma_thread_inst", 0) + k.get("dmul_thread_inst", 0)
               + k.get("dadd_thread_inst", 0) for k in ks)
    doc[config] = {"n": n, "dram_bytes_per_launch": dram,
                   "algorithmic_bytes_per_launch": bytes_per_row * n,
                   "fp64_thread_inst_per_row": fp64 / n, "kernels": ks, "source": source}
    json.dump(doc, open(path, "w"), indent=1)
    return doc[config]


if __name__ == "__main__":
    if "--config" in sys.argv:
        a = sys.argv
        cfg = a[a.index("--config") + 1]
        n = int(a[a.index("--n") + 1])
        out = a[a.index("--out") + 1] if "--out" in a else "profiles/ncu_summary.json"
        src = a[a.index("--source") + 1] if "--source" in a else a[1]
        bpr = int(a[a.index("--bytes-per-row") + 1]) if "--bytes-per-row" in a else 96
        r = update_profile_summary(a[1], cfg, n, out, src, bpr)
        print(json.dumps({k: v for k, v in r.items() if k != "kernels"}))
        sys.exit(0)
    res = summarise(sys.argv[1])
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
    for k in res:
        print(json.dumps(k))
