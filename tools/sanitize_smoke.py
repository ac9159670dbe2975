#!/usr/bin/env python3
"""Small calls of every device entry point, for compute-sanitizer
(memcheck / racecheck / synccheck) on the GPU box:

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1306_6291_b200 as sd  # noqa: E402
from paper_1306_6291_b200 import workloads  # noqa: E402

dev = torch.device("cuda", 0)
for cfg in ("c2", "c3", "c4"):
    for n in (1, 31, 257, 3000):
        A = torch.as_tensor(workloads.generate(cfg, n).astype(np.float64)).to(dev)
        sd.diagonalize3_batched(A)
        sd.diagonalize3_batched(A.float())
        sd.diagonalize3_batched(A, report=True, with_d=True)
        big = torch.zeros((n + 1, 6), dtype=torch.float64, device=dev)
        big[1:] = A
        sd.diagonalize3_batched(big.view(-1)[6:].view(n, 6))   # offset (8-byte aligned) rows
A1 = torch.as_tensor(workloads.generate("c1", 3000)).to(dev)
sd.diagonalize2_batched(A1)
sd.diagonalize2_batched(A1, with_d=True)
A = torch.as_tensor(workloads.generate("c2", 2000)).to(dev)
r = sd.diagonalize3_batched(A)
sd.jacobi_batched(A)
sd.jacobi_batched(A1, dim=2)
d = sd.compose_rotation_batched(r.ang)
sd.residuals_batched(A, r.lam, d)
bcd, _ = sd.char_coeffs_batched(A)
sd.cubic_roots_batched(bcd)
pqd, _ = sd.compute_pq_batched(bcd)
sd.eigenvalues3_batched(bcd, pqd)
sd.pq_expanded_batched(A)
v, _ = sd.compute_v_batched(A, r.lam)
sd.compute_w_batched(A, r.lam, v)
sd.f_vectors_batched(A)
plan = sd.HostPlan(0, chunk=1 << 10)
h = workloads.generate("c2", 5000)
lam, ang, st = np.empty((5000, 3)), np.empty((5000, 3)), np.empty(5000, np.uint8)
plan.eig3(h, lam, ang, st)
plan.close()
sd.diagonalize3(sd.SymMat3(1.0, 2.0, 3.0, 0.1, 0.2, 0.3))
sd.diagonalize2(sd.SymMat2(1.0, 2.0, 0.3))
torch.cuda.synchronize()
print("sanitize smoke done")
