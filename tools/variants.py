#!/usr/bin/env python3
"""Build and evaluate fast-path variants (accuracy vs time trade-offs).

    python tools/variants.py build            # here: nvcc each variant
    python tools/variants.py run [--n 262144] # on the GPU box

Each variant is the library compiled with some SD_FAST_* switches of
sd_fast3.cuh set; `run` times sd_eig3_f64 for every variant on c2/c4 and
compares its output with the literal path (sd_eig3_literal_f64) using the
parity comparator of tests/parity.py.  Prints one JSON line per variant.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
OUT = ROOT / "paper_1306_6291_b200" / "lib" / "variants"

VARIANTS = {
    "base": {},
    "pass4": {"SD_PASS_MIN_BLOCKS": 4},
    "pass2": {"SD_PASS_MIN_BLOCKS": 2},
    "fix6": {"SD_FIX_MIN_BLOCKS": 6, "SD_LIT_MIN_BLOCKS": 4},
    "fix3": {"SD_FIX_MIN_BLOCKS": 3, "SD_LIT_MIN_BLOCKS": 4},
}


def build():
    from paper_1306_6291_b200 import build_ext
    OUT.mkdir(parents=True, exist_ok=True)
    for old in OUT.glob("lib_*.so"):  # stale variants would bloat the gpurun snapshot
        if old.stem[4:] not in VARIANTS:
            old.unlink()
    from concurrent.futures import ThreadPoolExecutor

    def one(item):
        name, defs = item
        defs = dict(defs)
        pool = bool(defs.pop("PTX_POOL", 1))
        flags = [f for f in build_ext.NVCC_FLAGS if f not in ("-Xptxas", "-v")]
        cmd = [build_ext.nvcc(), *flags, *[f"-D{k}={v}" for k, v in defs.items()],
               "-o", str(OUT / f"lib_{name}.so"),
               *[str(build_ext.CSRC / s) for s in build_ext.SOURCES]]
        return name, build_ext.run_nvcc(cmd, ptx_pass=pool)

    with ThreadPoolExecutor(len(VARIANTS)) as ex:
        for name, res in ex.map(one, VARIANTS.items()):
            if res.returncode:
                raise SystemExit(f"{name} failed:\n{(res.stdout + res.stderr)[-3000:]}")
            print("built", name)


def run(n: int):
    import numpy as np
    import torch
    from paper_1306_6291_b200 import workloads, _lib
    from parity import compare3

    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream().cuda_stream
    for cfg in ("c2", "c4", "c3"):
        A = torch.as_tensor(workloads.generate(cfg, n).astype(np.float64)).to(dev)
        Abig = workloads.generate_torch(cfg, 1 << 24, dev).double()
        lam = torch.empty((n, 3), dtype=torch.float64, device=dev)
        ang = torch.empty_like(lam)
        st = torch.empty((n,), dtype=torch.uint8, device=dev)
        L0 = _lib.load()
        L0.sd_eig3_literal_f64(A.data_ptr(), n, lam.data_ptr(), ang.data_ptr(), st.data_ptr(),
                               stream)
        torch.cuda.synchronize()
        lit = dict(lam=lam.cpu().numpy(), ang=ang.cpu().numpy(), status=st.cpu().numpy())
        for name in VARIANTS:
            L = ctypes.CDLL(str(OUT / f"lib_{name}.so"))
            L.sd_eig3_f64.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 4
            L.sd_eig3_f64(A.data_ptr(), n, lam.data_ptr(), ang.data_ptr(), st.data_ptr(), stream)
            torch.cuda.synchronize()
            got = dict(lam=lam.cpu().numpy(), ang=ang.cpu().numpy(), status=st.cpu().numpy())
            s = compare3(lit, got, A=A.cpu().numpy())
            nb = Abig.shape[0]
            bl = torch.empty((nb, 3), dtype=torch.float64, device=dev)
            ba = torch.empty_like(bl)
            bs = torch.empty((nb,), dtype=torch.uint8, device=dev)
            for _ in range(3):
                L.sd_eig3_f64(Abig.data_ptr(), nb, bl.data_ptr(), ba.data_ptr(), bs.data_ptr(), stream)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            for _ in range(5):
                L.sd_eig3_f64(Abig.data_ptr(), nb, bl.data_ptr(), ba.data_ptr(), bs.data_ptr(), stream)
            ev1.record()
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1) / 5
            keys = ["code_mismatch", "sign_mismatch", "lam_max_err", "strict_ang_max",
                    "strict_ang_fail", "edge_ang_max", "polished_ang_max"]
            print(json.dumps({"config": cfg, "variant": name, "ms_2^24": ms,
                              **{k: s[k] for k in keys}}), flush=True)
            del bl, ba, bs


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["build", "run"])
    ap.add_argument("--n", type=int, default=1 << 18)
    a = ap.parse_args()
    build() if a.cmd == "build" else run(a.n)
