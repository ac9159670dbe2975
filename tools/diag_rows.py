#!/usr/bin/env python3
"""Dump the rows of a golden set where the GPU disagrees with the reference
(GPU box).  For each: input, reference status/lam/ang, fast-path and
literal-path (sd_eig3_literal_f64) results, and the path the fast kernel took
(sd_eig3_classify_f64 status).

    python tools/diag_rows.py eig3_adv [max_rows]
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests"), str(ROOT / "tests" / "golden")]


def main():
    import numpy as np
    import torch
    import paper_1306_6291_b200 as sd
    from conftest import load_golden
    from parity import wrapped_diff

    name = sys.argv[1]
    lim = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    g = load_golden(name)
    dev = torch.device("cuda", 0)
    A = torch.as_tensor(g["A"]).to(dev)
    n = A.shape[0]
    fast = sd.diagonalize3_batched(A)
    outs = {}
    for fn in ("sd_eig3_literal_f64", "sd_eig3_classify_f64"):
        lam = torch.empty((n, 3), dtype=torch.float64, device=dev)
        ang = torch.empty_like(lam)
        st = torch.empty((n,), dtype=torch.uint8, device=dev)
        sd._lib.call(fn, A.data_ptr(), n, lam.data_ptr(), ang.data_ptr(), st.data_ptr(),
                     torch.cuda.current_stream().cuda_stream)
        outs[fn] = (lam.cpu().numpy(), ang.cpu().numpy(), st.cpu().numpy())
    torch.cuda.synchronize()
    fl, fa, fs = fast.lam.cpu().numpy(), fast.ang.cpu().numpy(), fast.status.cpu().numpy()
    rs = g["status"]
    sign_bad = ((rs ^ fs) & 0x30) != 0
    code_bad = ((rs ^ fs) & 0x0F) != 0
    ok = (rs & 0x0F) < 8
    ang_bad = np.zeros(n, bool)
    ang_bad[ok] = np.nanmax(wrapped_diff(g["ang"][ok], fa[ok]), axis=1) > 1e-8
    bad = np.nonzero(ok & (sign_bad | code_bad | ang_bad))[0]
    print(json.dumps({"set": name, "rows": n, "bad": len(bad),
                      "sign_bad": int((ok & sign_bad).sum()), "code_bad": int((ok & code_bad).sum()),
                      "ang_bad": int(ang_bad.sum())}))
    ll, la, ls = outs["sd_eig3_literal_f64"]
    cl, ca, cs = outs["sd_eig3_classify_f64"]
    for i in bad[:lim]:
        print(json.dumps({
            "row": int(i), "A": g["A"][i].tolist(),
            "ref": {"st": int(rs[i]), "lam": g["lam"][i].tolist(), "ang": g["ang"][i].tolist(),
                    "report": g["report"][i].tolist()},
            "fast": {"st": int(fs[i]), "lam": fl[i].tolist(), "ang": fa[i].tolist()},
            "literal": {"st": int(ls[i]), "lam": ll[i].tolist(), "ang": la[i].tolist()},
            "classify_st": int(cs[i]),
        }))


if __name__ == "__main__":
    main()
