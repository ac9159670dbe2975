#!/usr/bin/env python3
"""Build and time 2x2 kernel variants (config c1) against the literal path.

    python tools/eig2_variants.py build          # here: nvcc each variant
    python tools/eig2_variants.py run            # on the GPU box

Each variant is the library compiled with SD_EIG2_* switches
(symdiag_b200.cu / sd_eig2.cuh).  `run` times sd_eig2_f64 on the c1 batch
(2^20 rows, a 512 MB buffer overwritten between calls so every call starts
from HBM, CUDA events on the launching stream), and compares every variant's
output with the literal variant (SD_EIG2_LITERAL=1) and the CPU oracle on
the same rows.  One JSON line per variant.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
OUT = ROOT / "paper_1306_6291_b200" / "lib" / "variants2"

VARIANTS = {
    "literal_r1_t128": {"SD_EIG2_LITERAL": 1, "SD_EIG2_MODE": 0, "SD_EIG2_ROWS": 1,
                        "SD_EIG2_THREADS": 128},
    "tile_r2_t128": {"SD_EIG2_MODE": 0, "SD_EIG2_ROWS": 2, "SD_EIG2_THREADS": 128},
    "tile_r2_t128_mb10": {"SD_EIG2_MIN_BLOCKS": 10},
    "tile_r2_t128_mb12": {"SD_EIG2_MIN_BLOCKS": 12},
    "tile_r2_t128_mb14": {"SD_EIG2_MIN_BLOCKS": 14},
    "tile_r1_t128_mb12": {"SD_EIG2_ROWS": 1, "SD_EIG2_MIN_BLOCKS": 12},
    "tile_r1_t128_mb16": {"SD_EIG2_ROWS": 1, "SD_EIG2_MIN_BLOCKS": 16},
}


def build(only=None):
    from concurrent.futures import ThreadPoolExecutor

    from paper_1306_6291_b200 import build_ext
    OUT.mkdir(parents=True, exist_ok=True)
    for old in OUT.glob("lib_*.so"):
        if old.stem[4:] not in VARIANTS:
            old.unlink()
    todo = {k: v for k, v in VARIANTS.items() if not only or k in only}

    def one(item):
        name, defs = item
        flags = [f for f in build_ext.NVCC_FLAGS if f not in ("-Xptxas", "-v")]
        cmd = [build_ext.nvcc(), *flags, *[f"-D{k}={v}" for k, v in defs.items()],
               "-o", str(OUT / f"lib_{name}.so"),
               *[str(build_ext.CSRC / s) for s in build_ext.SOURCES]]
        return name, build_ext.run_nvcc(cmd)

    with ThreadPoolExecutor(min(8, len(todo))) as ex:
        for name, res in ex.map(one, todo.items()):
            if res.returncode:
                raise SystemExit(f"{name} failed:\n{(res.stdout + res.stderr)[-3000:]}")
            print("built", name, flush=True)


def run(steps: int):
    import numpy as np
    import torch

    from oracle import oracle as O
    from paper_1306_6291_b200 import workloads

    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    n = workloads.CONFIGS["c1"]["n"]
    A_np = workloads.generate("c1", n)
    A = torch.as_tensor(A_np).to(dev)
    ref = O.eig2(A_np)
    lam = torch.empty((n, 2), dtype=torch.float64, device=dev)
    phi = torch.empty((n,), dtype=torch.float64, device=dev)
    st = torch.empty((n,), dtype=torch.uint8, device=dev)
    flush = torch.empty((1 << 29,), dtype=torch.uint8, device=dev)
    rflush = torch.ones((1 << 27,), dtype=torch.float32, device=dev)  # 512 MB, read-only pass
    acc = torch.empty((), dtype=torch.float32, device=dev)

    def do_flush(mode):
        flush.fill_(1)  # writes 512 MB: L2 full of dirty lines of another buffer
        if mode == "write+read":
            acc.copy_(rflush.sum())  # reads 512 MB: evicts them (write-back outside the timing)

    def timed(call, mode):
        ts = []
        for _ in range(steps):
            do_flush(mode)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            call()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts), min(ts)

    def timed1(call):
        do_flush("write+read")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        call()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    # floor: a device copy of the same byte counts (25.2 MB read, 25.2 MB written)
    src = A.view(-1)
    dst = torch.empty_like(src)
    for mode in ("write", "write+read"):
        ms, mn = timed(lambda: dst.copy_(src), mode)
        print(json.dumps({"variant": "torch_copy_floor", "flush": mode, "ms": ms, "ms_min": mn,
                          "ms_mean_clean_l2": statistics.mean(timed1(lambda: dst.copy_(src))
                                                              for _ in range(50)),
                          "bytes": 2 * src.numel() * 8}), flush=True)
    base = None
    for name in VARIANTS:
        L = ctypes.CDLL(str(OUT / f"lib_{name}.so"))
        f = L.sd_eig2_f64
        f.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 4
        call = lambda: f(A.data_ptr(), n, lam.data_ptr(), phi.data_ptr(), st.data_ptr(), sp)  # noqa
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        got = dict(lam=lam.cpu().numpy().copy(), phi=phi.cpu().numpy().copy(),
                   status=st.cpu().numpy().copy())
        if base is None:
            base = got
        ms, ms_min = timed(call, "write")
        ms_r, ms_rmin = timed(call, "write+read")
        # mean over many calls (event timestamps are quantised to ~1 us here)
        ms_mean = statistics.mean([timed(call, "write+read")[0] for _ in range(1)] +
                                  [timed1(call) for _ in range(50)])
        dl = np.abs(got["lam"] - ref["lam"]).max(axis=1) / np.maximum(1.0, np.abs(ref["lam"]).max(axis=1))
        print(json.dumps({
            "variant": name, "defs": VARIANTS[name], "n": n, "ms": ms, "ms_min": ms_min,
            "ms_clean_l2": ms_r, "ms_clean_l2_min": ms_rmin, "ms_mean_clean_l2": ms_mean,
            "matrices_per_s": n / (ms * 1e-3),
            "hbm_frac": 48 * n / (ms * 1e-3) / 6455.9e9,
            "status_mismatch_vs_oracle": int(np.count_nonzero(got["status"] != ref["status"])),
            "lam_bit_equal_vs_oracle": float(np.mean(np.all(got["lam"] == ref["lam"], axis=1))),
            "lam_max_rel_vs_oracle": float(dl.max()),
            "phi_max_abs_vs_oracle": float(np.abs(got["phi"] - ref["phi"]).max()),
            "phi_bit_equal_vs_oracle": float(np.mean(got["phi"] == ref["phi"])),
            "phi_max_abs_vs_literal": float(np.abs(got["phi"] - base["phi"]).max()),
        }), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["build", "run"])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--only", nargs="*")
    a = ap.parse_args()
    build(a.only) if a.cmd == "build" else run(a.steps)
