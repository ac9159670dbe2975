#!/usr/bin/env python3
"""Time sd_eig3_f32 vs sd_eig3_f64 on the same c4 rows (GPU box)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1306_6291_b200 as sd
from paper_1306_6291_b200 import workloads
dev = torch.device("cuda", 0)
for cfg in ("c4", "c2"):
    A32 = workloads.generate_torch("c4" if cfg == "c4" else "c2", 1 << 24, dev).float()
    A64 = A32.double()
    for name, A in (("f32", A32), ("f64", A64)):
        for _ in range(3):
            sd.diagonalize3_batched(A)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            sd.diagonalize3_batched(A)
        e.record()
        torch.cuda.synchronize()
        print(json.dumps({"data": cfg, "io": name, "ms": s.elapsed_time(e) / 10}))
