#!/usr/bin/env python3
"""Throughput of the SURVEY §8f "next" rows on the GPU box.

    python tools/bench_next.py   -> one JSON line per measurement

Jacobi referee, residuals and cubic roots on config-2 rows (device-resident,
CUDA events), and the JSON-lines front end (cmd_solve, host parse + GPU
solve + format) on 2^17 records.
"""

from __future__ import annotations

import io
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def timed(fn, reps=5):
    import torch
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


def main():
    import torch
    import paper_1306_6291_b200 as sd
    from paper_1306_6291_b200 import cli, workloads

    dev = torch.device("cuda", 0)
    n = 1 << 22
    A = workloads.generate_torch("c2", n, dev)
    t = timed(lambda: sd.jacobi_batched(A, dim=3))
    print(json.dumps({"what": "jacobi_batched 3x3 c2", "rows": n, "matrices_per_s": n / t}))
    r = sd.diagonalize3_batched(A, report=True, with_d=True)
    d = r.d.view(-1, 3, 3)
    t = timed(lambda: sd.residuals_batched(A, r.lam, d))
    print(json.dumps({"what": "residuals_batched 3x3 c2", "rows": n, "matrices_per_s": n / t}))
    t = timed(lambda: sd.diagonalize3_batched(A, report=True, with_d=True))
    print(json.dumps({"what": "diagonalize3 report+D (literal) c2", "rows": n,
                      "matrices_per_s": n / t}))
    bcd, _ = sd.char_coeffs_batched(A)
    t = timed(lambda: sd.cubic_roots_batched(bcd))
    print(json.dumps({"what": "cubic_roots_batched c2", "rows": n, "matrices_per_s": n / t}))
    A2 = workloads.generate_torch("c1", n, dev)
    t = timed(lambda: sd.jacobi_batched(A2, dim=2))
    print(json.dumps({"what": "jacobi_batched 2x2 c1", "rows": n, "matrices_per_s": n / t}))
    rows = workloads.generate("c2", 1 << 17)
    text = "\n".join(json.dumps({"id": str(i), "a11": r[0], "a12": r[1], "a13": r[2],
                                 "a22": r[3], "a23": r[4], "a33": r[5]})
                     for i, r in enumerate(rows.tolist())) + "\n"
    cli.cmd_solve(io.StringIO(text[:100000]), io.StringIO())
    t0 = time.perf_counter()
    out = io.StringIO()
    cli.cmd_solve(io.StringIO(text), out)
    dt = time.perf_counter() - t0
    print(json.dumps({"what": "cli solve (host JSON + GPU)", "records": len(rows),
                      "records_per_s": len(rows) / dt}))


if __name__ == "__main__":
    main()
