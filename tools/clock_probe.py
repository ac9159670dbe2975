#!/usr/bin/env python3
"""Burst vs sustained throughput and SM clocks (GPU box).

    python tools/clock_probe.py

1. DFMA probe (sd_probe_dfma): one burst launch, then back-to-back launches
   for ~3 s; TFLOP/s (2 FLOP per DFMA) and the SM clock seen.
2. sd_eig3_f64 on c2 (2^24) and sd_eig3_f32 on c4 (2^26): a few steps, then
   ~3 s back to back; matrices/s and clocks.
One JSON line per measurement.
"""

from __future__ import annotations

import ctypes
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import ClockSampler  # noqa: E402


def timed(fn, seconds):
    import torch
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    t0 = time.time()
    s.record()
    while time.time() - t0 < seconds:
        fn()
        n += 1
        if n % 8 == 0:
            torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    return n, s.elapsed_time(e) * 1e-3


def main():
    import torch
    import paper_1306_6291_b200 as sd
    from paper_1306_6291_b200 import workloads

    dev = torch.device("cuda", 0)
    L = sd._lib.load()
    stream = torch.cuda.current_stream().cuda_stream
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks, iters = nsm * 8, 4096
    sink = torch.empty(blocks * 256, dtype=torch.float64, device=dev)
    tot = ctypes.c_double()
    probe = lambda: L.sd_probe_dfma(blocks, iters, sink.data_ptr(), ctypes.byref(tot), stream)  # noqa: E731
    probe()
    torch.cuda.synchronize()
    n, dt = timed(probe, 0.05)
    print(json.dumps({"what": "dfma_burst", "tflops": 2 * tot.value * n / dt / 1e12, "launches": n}))
    with ClockSampler(0) as c:
        n, dt = timed(probe, 3.0)
    print(json.dumps({"what": "dfma_sustained_3s", "tflops": 2 * tot.value * n / dt / 1e12,
                      "launches": n, "clocks": c.summary()}))
    for cfg, nrows in (("c2", 1 << 24), ("c4", 1 << 26), ("c3", 1 << 24)):
        A = workloads.generate_torch(cfg, nrows, dev)
        f = lambda: sd.diagonalize3_batched(A)  # noqa: E731
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        n, dt = timed(f, 0.05)
        burst = nrows * n / dt
        with ClockSampler(0) as c:
            n, dt = timed(f, 3.0)
        print(json.dumps({"what": f"eig3_{cfg}", "rows": nrows, "burst_mps": burst / 1e9,
                          "sustained_mps": nrows * n / dt / 1e9, "clocks": c.summary()}))
        del A
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
