#!/usr/bin/env python3
"""Rows still pending after the first k passes of sd_eig3_f64 / sd_eig3_f32 (GPU box).

    SD_DEBUG_PASSES=3 python tools/pass_census.py [n]

(fast, compaction, exact, polish, literal): with k = 3 the histogram shows
what the polish pass (codes 5-7) and the literal pass (code 4, by reason)
receive.  The library reads SD_DEBUG_PASSES once, so one process per k.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1306_6291_b200 import workloads, _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
dev = torch.device('cuda', 0)
for cfg in ('c2', 'c3', 'c4'):
    A = workloads.generate(cfg, n)
    f32 = A.dtype == np.float32
    At = torch.as_tensor(A).to(dev)
    dt = torch.float32 if f32 else torch.float64
    lam = torch.empty((n, 3), dtype=dt, device=dev)
    ang = torch.empty_like(lam)
    st = torch.empty((n,), dtype=torch.uint8, device=dev)
    _lib.call("sd_eig3_f32" if f32 else "sd_eig3_f64", At.data_ptr(), n, lam.data_ptr(),
              ang.data_ptr(), st.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    s = st.cpu().numpy()
    code = s & 15
    lit = {int(r): int(((code == 4) & ((s >> 4) == r)).sum()) for r in range(16)
           if ((code == 4) & ((s >> 4) == r)).any()}
    print(json.dumps({"cfg": cfg, "n": n, "passes": os.environ.get("SD_DEBUG_PASSES"),
                      "code4_by_reason": lit,
                      "polish_pending": {int(c): int((code == c).sum()) for c in (5, 6, 7)},
                      "errors": int((code >= 8).sum())}), flush=True)
