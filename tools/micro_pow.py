"""Throughput of the device glibc pow and the literal solver (GPU box)."""
import sys, json
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1306_6291_b200 as sd
from paper_1306_6291_b200 import workloads, _lib
dev = torch.device('cuda', 0)
n = 1 << 24
x = torch.randn(n, dtype=torch.float64, device=dev)
for k in (2.0, 3.0):
    for _ in range(2):
        sd.glibc_pow_batched(x, k)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); r = sd.glibc_pow_batched(x, k); e1.record(); torch.cuda.synchronize()
    print(json.dumps({"what": f"glibc_pow k={k}", "n": n, "ms": e0.elapsed_time(e1)}))
for cfg in ("c2", "c3"):
    A = torch.as_tensor(workloads.generate(cfg, 1 << 20)).to(dev)
    m = A.shape[0]
    lam = torch.empty((m, 3), dtype=torch.float64, device=dev); ang = torch.empty_like(lam)
    st = torch.empty((m,), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        _lib.call("sd_eig3_literal_f64", A.data_ptr(), m, lam.data_ptr(), ang.data_ptr(), st.data_ptr(), s)
    e0.record()
    _lib.call("sd_eig3_literal_f64", A.data_ptr(), m, lam.data_ptr(), ang.data_ptr(), st.data_ptr(), s)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"what": f"literal {cfg}", "n": m, "ms": e0.elapsed_time(e1)}))
