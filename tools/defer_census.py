"""Census of rows the fast kernel leaves for the polish / literal passes (GPU box).

    python tools/defer_census.py [lib.so ...]

With a library built with -DSD_CLS_CENSUS=1 the rows classify3 cannot
certify show up as deferred with the check that fired as the reason
(sd_fast3.cuh SD_CLS_AMB ids: 9 p sign, 10 triple threshold, 11 discriminant
thresholds, 12 sign of q, 14 arccos clamp/slack, 15 / 3 eigenvalue bounds).
"""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1306_6291_b200 import workloads, _lib

dev = torch.device('cuda', 0)
libs = sys.argv[1:] or [str(_lib.LIB_PATH)]
for cfg, n in (('c2', 1 << 22), ('c3', 1 << 22), ('c4', 1 << 22)):
    A = torch.as_tensor(workloads.generate(cfg, n)).to(dev).double()
    for path in libs:
        L = ctypes.CDLL(path)
        L.sd_eig3_classify_f64.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 4
        lam = torch.empty((n, 3), dtype=torch.float64, device=dev); ang = torch.empty_like(lam)
        st = torch.empty((n,), dtype=torch.uint8, device=dev)
        L.sd_eig3_classify_f64(A.data_ptr(), n, lam.data_ptr(), ang.data_ptr(), st.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        s = st.cpu().numpy(); code = s & 15
        d = {int(r): int(((code == 4) & ((s >> 4) == r)).sum()) for r in range(16) if ((code == 4) & ((s >> 4) == r)).any()}
        warps = ((code == 4) & ((s >> 4) != 0) & ((s >> 4) != 13)).reshape(-1, 32).any(axis=1).mean()
        print(json.dumps({"cfg": cfg, "lib": path.split('/')[-1], "deferred_by_reason": d,
                          "warps_with_deferral": float(warps),
                          "errors": {int(c): int((code == c).sum()) for c in range(8, 16) if (code == c).any()},
                          "polish": {int(c): int((code == c).sum()) for c in (5, 6, 7)}}), flush=True)
