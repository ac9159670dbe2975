#!/usr/bin/env python3
"""Event timing of one c1 (2x2, 2^20 rows) call with the bench flush, through
the Python API vs the raw C-ABI call, with and without a synchronize after
each timed call (outside the events).  Shows whether host enqueue lag lands
inside the device-timed region.    python tools/c1_timing_probe.py   (GPU)
"""
import sys, statistics, json, ctypes
sys.path.insert(0, '.')
import torch
import paper_1306_6291_b200 as sd
from paper_1306_6291_b200 import workloads, _lib
dev = torch.device('cuda', 0)
n = 1 << 20
A = workloads.generate_torch('c1', n, dev)
out = dict(lam=torch.empty((n, 2), dtype=torch.float64, device=dev),
           phi=torch.empty((n,), dtype=torch.float64, device=dev),
           status=torch.empty((n,), dtype=torch.uint8, device=dev))
flush = torch.empty((1 << 29,), dtype=torch.uint8, device=dev)
rflush = torch.ones((1 << 27,), dtype=torch.float32, device=dev)
stream = torch.cuda.current_stream()
L = _lib.load()
raw = lambda: L.sd_eig2_f64(A.data_ptr(), n, out['lam'].data_ptr(), out['phi'].data_ptr(), out['status'].data_ptr(), stream.cuda_stream)
api = lambda: sd.diagonalize2_batched(A, out=out)
def t(fn, sync, steps=60):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s, e in ev:
        flush.fill_(1); rflush.sum()
        s.record(stream); fn(); e.record(stream)
        if sync: torch.cuda.synchronize()
    torch.cuda.synchronize()
    return statistics.mean(s.elapsed_time(e) for s, e in ev) * 1e3
for name, fn in (('api', api), ('raw', raw)):
    for sync in (False, True):
        print(json.dumps({'call': name, 'sync_each': sync, 'us_mean': t(fn, sync)}))
