#!/usr/bin/env python3
"""A/B timing of several builds of the library on the same data (GPU box).

    python tools/ab_libs.py [--n 16777216] [--reps 10] lib_a.so lib_b.so ...

For each config (c2, c3 fp64; c4 fp32) the numpy-seeded batch is generated
once (workloads.generate, cached), copied to HBM, and every library's
sd_eig3_f64 / sd_eig3_f32 is timed with CUDA events (3 warm-up calls,
`reps` timed calls, interleaved round-robin over the libraries so clock or
thermal drift hits all builds alike).  Outputs of each build are compared
with the first one (status bytes; eigenvalue/angle maxima).  One JSON line
per (config, library).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]


def main():
    import numpy as np
    import torch
    from paper_1306_6291_b200 import workloads

    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--configs", default="c2,c3,c4")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream().cuda_stream
    libs = []
    for p in a.libs:
        L = ctypes.CDLL(str(Path(p).resolve()))
        for f in ("sd_eig3_f64", "sd_eig3_f32"):
            getattr(L, f).argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 4
        libs.append((Path(p).stem, L))
    for cfg in a.configs.split(","):
        A = workloads.generate(cfg, a.n)
        dt = torch.float32 if A.dtype == np.float32 else torch.float64
        At = torch.as_tensor(A).to(dev)
        n = At.shape[0]
        fn = "sd_eig3_f32" if dt == torch.float32 else "sd_eig3_f64"
        outs = []
        for _ in libs:
            outs.append((torch.empty((n, 3), dtype=dt, device=dev),
                         torch.empty((n, 3), dtype=dt, device=dev),
                         torch.empty((n,), dtype=torch.uint8, device=dev)))

        def call(i):
            lam, ang, st = outs[i]
            rc = getattr(libs[i][1], fn)(At.data_ptr(), n, lam.data_ptr(), ang.data_ptr(),
                                         st.data_ptr(), stream)
            assert rc == 0, rc

        for i in range(len(libs)):
            for _ in range(3):
                call(i)
        times = [[] for _ in libs]
        for _ in range(a.reps):
            for i in range(len(libs)):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                call(i)
                e1.record()
                torch.cuda.synchronize()
                times[i].append(e0.elapsed_time(e1))
        base = [t.double().cpu() for t in outs[0]]
        for i, (name, _) in enumerate(libs):
            o = [t.double().cpu() for t in outs[i]]
            st_diff = int((o[2] != base[2]).sum())
            lam_d = float(torch.nan_to_num((o[0] - base[0]).abs()).max())
            ang_d = float(torch.nan_to_num((o[1] - base[1]).abs()).max())
            t = sorted(times[i])
            print(json.dumps({"config": cfg, "lib": name, "n": n,
                              "ms_median": t[len(t) // 2], "ms_min": t[0],
                              "status_diff_vs_first": st_diff, "lam_maxdiff": lam_d,
                              "ang_maxdiff": ang_d}), flush=True)
        del At, outs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
