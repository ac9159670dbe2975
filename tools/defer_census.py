"""Census of rows the fast kernel leaves for the polish / literal passes (GPU box).

    python tools/defer_census.py
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_1306_6291_b200 as sd
from paper_1306_6291_b200 import workloads
dev = torch.device('cuda', 0)
for cfg, n in (('c2', 1 << 22), ('c3', 1 << 22), ('c4', 1 << 22)):
    A = torch.as_tensor(workloads.generate(cfg, n)).to(dev).double()
    lam = torch.empty((n, 3), dtype=torch.float64, device=dev); ang = torch.empty_like(lam)
    st = torch.empty((n,), dtype=torch.uint8, device=dev)
    sd._lib.call("sd_eig3_classify_f64", A.data_ptr(), n, lam.data_ptr(), ang.data_ptr(), st.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    s = st.cpu().numpy(); code = s & 15
    d = {int(r): int(((code == 4) & ((s >> 4) == r)).sum()) for r in range(16) if ((code == 4) & ((s >> 4) == r)).any()}
    print(json.dumps({"cfg": cfg, "deferred_by_reason": d, "errors": {int(c): int((code == c).sum()) for c in range(8, 16) if (code == c).any()},
                      "polish": {int(c): int((code == c).sum()) for c in (5, 6, 7)}}))
