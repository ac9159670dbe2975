#!/usr/bin/env python3
"""Sweep the host-plan chunk size for the e2e path (GPU box)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1306_6291_b200 as sd
from paper_1306_6291_b200 import workloads
n = 1 << 24
A = torch.empty((n, 6), dtype=torch.float64, pin_memory=True)
A.copy_(workloads.generate_torch("c2", n, torch.device("cuda", 0)))
lam = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
ang = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
st = torch.empty((n,), dtype=torch.uint8, pin_memory=True)
for chunk in (1 << 17, 1 << 18, 1 << 19, 1 << 20, 1 << 21, 1 << 22):
    plan = sd.HostPlan(0, chunk=chunk)
    plan.eig3(A, lam, ang, st)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter(); plan.eig3(A, lam, ang, st); ts.append(time.perf_counter() - t0)
    plan.close()
    t = min(ts)
    print(json.dumps({"chunk": chunk, "ms": t * 1e3, "G_per_s": n / t / 1e9,
                      "GBps_each_way": n * 48 / t / 1e9}), flush=True)
# raw copy bandwidth for reference
d = torch.empty((n, 6), dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(A, non_blocking=True); torch.cuda.synchronize()
h2d = time.perf_counter() - t0
t0 = time.perf_counter(); A.copy_(d, non_blocking=True); torch.cuda.synchronize()
d2h = time.perf_counter() - t0
print(json.dumps({"raw_h2d_GBps": n * 48 / h2d / 1e9, "raw_d2h_GBps": n * 48 / d2h / 1e9}))
# concurrent H2D + D2H (the e2e pipeline's ceiling), whole buffers and chunked
B = torch.empty((n, 6), dtype=torch.float64, pin_memory=True)
d2 = torch.empty((n, 6), dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for chunks in (1, 16, 64):
    m = n // chunks
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for c in range(chunks):
            sl = slice(c * m, (c + 1) * m)
            with torch.cuda.stream(s1):
                d[sl].copy_(A[sl], non_blocking=True)
            with torch.cuda.stream(s2):
                B[sl].copy_(d2[sl], non_blocking=True)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    print(json.dumps({"bidir_chunks": chunks, "GBps_each_way": n * 48 / best / 1e9}))
