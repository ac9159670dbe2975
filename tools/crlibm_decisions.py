#!/usr/bin/env python3
"""How far does a correctly rounded libm get from glibc's decisions?

Runs the CPU oracle twice on the same seeded rows -- once with glibc
(the reference's libm) and once built with sd_crlibm.h's correctly rounded
sin/cos/acos/asin/atan2/hypot (oracle/build/libsymdiag_oracle_cr.so) -- and
counts status-code / sign disagreements and bit-equal eigenvalues/angles.
This is what the device's literal solver can reach at best with that libm.

    python tools/crlibm_decisions.py [--n 4194304] [--configs c2,c3,c4]
Also re-checks the rows flagged by the round-2 2^26 sweeps.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def run(lib, A, out):
    code = f"""
import sys, numpy as np
sys.path.insert(0, {str(ROOT)!r})
from oracle import oracle as O
A = np.load({A!r})
r = O.eig3(A, nthreads=O.default_threads())
np.savez({out!r}, status=r['status'], lam=r['lam'], ang=r['ang'])
"""
    env = dict(os.environ)
    if lib:
        env["SD_ORACLE_LIB"] = lib
    subprocess.run([sys.executable, "-c", code], check=True, env=env)
    return np.load(out)


def compare(A, tag):
    np.save("/tmp/crd_A.npy", A)
    g = run(None, "/tmp/crd_A.npy", "/tmp/crd_g.npz")
    c = run(str(ROOT / "oracle/build/libsymdiag_oracle_cr.so"), "/tmp/crd_A.npy", "/tmp/crd_c.npz")
    st_g, st_c = g["status"], c["status"]
    rec = {"set": tag, "n": int(len(A)),
           "code_mismatch": int(((st_g ^ st_c) & 0x0F != 0).sum()),
           "sign_mismatch": int((((st_g ^ st_c) & 0x30 != 0) & ((st_g ^ st_c) & 0x0F == 0)).sum()),
           "polished_mismatch": int(((st_g ^ st_c) & 0x80 != 0).sum()),
           "lam_bit_equal_frac": float((g["lam"] == c["lam"]).all(axis=1).mean()),
           "ang_bit_equal_frac": float((g["ang"] == c["ang"]).all(axis=1).mean())}
    bad = np.nonzero((st_g ^ st_c) & 0x3F)[0]
    rec["mismatch_rows"] = [int(i) for i in bad[:10]]
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 22)
    ap.add_argument("--configs", default="c2,c3,c4")
    args = ap.parse_args()
    sys.path.insert(0, str(ROOT))
    from paper_1306_6291_b200 import workloads
    for cfg in args.configs.split(","):
        A = workloads.generate(cfg, args.n)
        if A.dtype != np.float64:
            A = A.astype(np.float64)
        print(json.dumps(compare(A, cfg)), flush=True)
    for cfg in ("c3", "c4"):
        f = ROOT / f"profiles/r2/parity_sweep/sweep_{cfg}_flagged.npz"
        if f.exists():
            d = np.load(f)
            A = d["A"]
            np.save("/tmp/crd_A.npy", A)
            c = run(str(ROOT / "oracle/build/libsymdiag_oracle_cr.so"), "/tmp/crd_A.npy", "/tmp/crd_c.npz")
            same = (c["status"] & 0x3F) == (d["ref_status"] & 0x3F)
            print(json.dumps({"set": f"{cfg}_sweep_flagged", "n": int(len(A)),
                              "cr_status_equals_reference": int(same.sum()),
                              "gpu_status_equals_reference": int(((d["status"] ^ d["ref_status"]) & 0x3F == 0).sum()),
                              "cr_lam_bit_equal": int((c["lam"] == d["ref_lam"]).all(axis=1).sum())}))


if __name__ == "__main__":
    main()
