import ctypes, json, sys, statistics
from pathlib import Path
import torch
sys.path.insert(0, '.')
from paper_1306_6291_b200 import workloads
dev = torch.device('cuda', 0)
n = 1 << 24
A = torch.as_tensor(workloads.generate('c1', n)).to(dev)
lam = torch.empty((n, 2), dtype=torch.float64, device=dev); phi = torch.empty(n, dtype=torch.float64, device=dev); st = torch.empty(n, dtype=torch.uint8, device=dev)
sp = torch.cuda.current_stream().cuda_stream
for lib in sorted(Path('paper_1306_6291_b200/lib/variants2').glob('lib_tile*.so')):
    L = ctypes.CDLL(str(lib)); f = L.sd_eig2_f64; f.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 4
    for _ in range(3): f(A.data_ptr(), n, lam.data_ptr(), phi.data_ptr(), st.data_ptr(), sp)
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(A.data_ptr(), n, lam.data_ptr(), phi.data_ptr(), st.data_ptr(), sp); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"lib": lib.stem, "n": n, "ms": statistics.median(ts), "G_per_s": n / statistics.median(ts) / 1e6}))
