#!/usr/bin/env python3
"""Run sd_eig3_f64 of one variant library (tools/variants.py build) on a
config, a few times — a target for `ncu` comparisons of variants.

    python tools/variant_run.py <variant> [config] [n]
"""
import ctypes
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1306_6291_b200 import workloads  # noqa: E402

name = sys.argv[1]
cfg = sys.argv[2] if len(sys.argv) > 2 else "c2"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 24
L = ctypes.CDLL(str(ROOT / "paper_1306_6291_b200" / "lib" / "variants" / f"lib_{name}.so"))
L.sd_eig3_f64.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 4
dev = torch.device("cuda", 0)
A = workloads.generate_torch(cfg, n, dev).double()
lam = torch.empty((n, 3), dtype=torch.float64, device=dev)
ang = torch.empty_like(lam)
st = torch.empty((n,), dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    assert L.sd_eig3_f64(A.data_ptr(), n, lam.data_ptr(), ang.data_ptr(), st.data_ptr(), s) == 0
torch.cuda.synchronize()
print("ok", name, cfg, n)
