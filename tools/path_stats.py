#!/usr/bin/env python3
"""Which path does each row of a workload take?  (GPU box)

    python tools/path_stats.py [--n 2097152] [--configs c2,c3,c4]

Runs only the first pass (sd_eig3_classify_f64) and histograms the status
codes it leaves: finished on the fast path (by branch), polish pending, or
deferred to the literal solver (by reason, see sd_fast3.cuh).  Then runs the
full sd_eig3_f64 and histograms the final branch mix.  One JSON line per
config.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

REASONS = {1: "nonfinite_or_huge", 2: "p_negative", 3: "triple_near_gate", 4: "acos_slack",
           5: "eigen_gap", 6: "vw_excursion", 7: "f_norm_zero", 8: "zero_g_or_z",
           9: "selection_margin", 10: "phi1_route_range", 11: "residual_near_gate",
           12: "not_double_root", 13: "double_pending_pass", 14: "double_f_norm_zero",
           15: "double_zero_g_or_z", 0: "generic_pending_pass"}


def main():
    import numpy as np
    import torch
    import paper_1306_6291_b200 as sd
    from paper_1306_6291_b200 import workloads

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 21)
    ap.add_argument("--configs", default="c2,c3,c4")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    for cfg in a.configs.split(","):
        A = torch.as_tensor(workloads.generate(cfg, a.n).astype(np.float64)).to(dev)
        n = A.shape[0]
        lam = torch.empty((n, 3), dtype=torch.float64, device=dev)
        ang = torch.empty_like(lam)
        st = torch.empty((n,), dtype=torch.uint8, device=dev)
        sd._lib.call("sd_eig3_classify_f64", A.data_ptr(), n, lam.data_ptr(), ang.data_ptr(),
                     st.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        s = st.cpu().numpy()
        code = s & 0x0F
        out = {"config": cfg, "n": n,
               "fast_done": {k: int((code == v).sum()) for k, v in
                             (("generic", 0), ("double_root", 2), ("triple_root", 3))},
               "polish_pending": {k: int((code == v).sum()) for k, v in
                                  (("generic", 5), ("double_root", 6), ("triple_root", 7))},
               "deferred": {REASONS[r]: int(((code == 4) & ((s >> 4) == r)).sum())
                            for r in range(16) if ((code == 4) & ((s >> 4) == r)).any()}}
        full = sd.diagonalize3_batched(A)
        torch.cuda.synchronize()
        fc = full.status.cpu().numpy()
        out["final"] = {"generic": int(((fc & 15) == 0).sum()),
                        "already_diagonal_2d": int(((fc & 15) == 1).sum()),
                        "double_root": int(((fc & 15) == 2).sum()),
                        "triple_root": int(((fc & 15) == 3).sum()),
                        "errors": int(((fc & 15) >= 8).sum()),
                        "polished": int(((fc & 0x80) != 0).sum())}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
