#!/usr/bin/env python3
"""Benchmark: batched closed-form 3x3 / 2x2 symmetric diagonalization on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
                    [--impl ours|reference] [--no-extra]

One step = one pass of the hot path (sd_eig3_f64 through the C ABI) over one
resident batch of the BASELINE.json configuration.  Default workload is
config 2 (3x3 fp64 iid N(0,1), 2^24 matrices; inputs 805 MB > 126 MB L2, so
every step reads from HBM).  N > 1 (torchrun, one rank per GPU): every rank
processes its own full-size batch, no collective on the data path
(weak scaling); timing = max over ranks of the device-event time.

Prints ONE JSON line (rank 0).  `value` is matrices/s over all ranks with
inputs resident in HBM; `e2e` is the same metric through the host-buffer
C-ABI path (pinned host in/out, H2D + kernel + D2H in the timed region).
`--impl reference` times the reference algorithm on the host CPU cores: the
C restatement in oracle/ (the reference itself is Python and not present on
the GPU box), with all host threads.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

# Frozen cost model: algorithmic FP64-pipe
# instruction-equivalents W and HBM bytes per matrix (in + out; Euler angles
# alias phi; status byte excluded).  1 instr-eq = 1 DFMA = 2 FLOP.
COST = {
    "c1": dict(W=105, bytes=48, metric_dim=2),
    "c2": dict(W=2370, bytes=96, metric_dim=3),
    "c3": dict(W=1500, bytes=96, metric_dim=3),
    "c4": dict(W=2370, bytes=48, metric_dim=3),
    "c5": dict(W=2370, bytes=96, metric_dim=3),
}
L2_BYTES = 126 * 1024 * 1024  # B200 L2
METRIC = "matrices/sec (3x3 fp64 and fp32) at 1/2/4/8 B200; % of roofline"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = {}
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        p = json.loads(f.read_text())
    return p


class NvmlClockSampler:
    """SM clock and clock-event reasons polled through NVML every ~1 ms on a
    background thread while the timed region runs (nvidia-smi's 20 ms loop
    yields only one or two samples in a ~20 ms region)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, cuda_index: int):
        import pynvml
        import torch
        self.nv = pynvml
        pynvml.nvmlInit()
        try:
            pr = torch.cuda.get_device_properties(cuda_index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:  # noqa: BLE001 — older torch / driver: fall back to the index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(cuda_index)
        self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        self.samples, self.masks = [], 0
        self.run = False

    def _poll(self):
        nv = self.nv
        while self.run:
            self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
            self.masks |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            time.sleep(0.001)

    def __enter__(self):
        self.run = True
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()
        t0 = time.time()
        while not self.samples and time.time() - t0 < 1.0:
            time.sleep(0.0005)
        return self

    def __exit__(self, *exc):
        self.run = False
        self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        reasons = [n for n, attr in self.REASONS if self.masks & getattr(self.nv, attr)]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml, ~1 ms"}


def clock_sampler(cuda_index: int):
    try:
        return NvmlClockSampler(cuda_index)
    except Exception:  # noqa: BLE001 — no NVML bindings: nvidia-smi loop
        return ClockSampler(cuda_index)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()  # wait for the first sample so the timed region is covered
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.lines.clear()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for name, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_inputs(config, n, dev, seed_offset):
    import torch
    from paper_1306_6291_b200 import workloads
    t0 = time.time()
    A = workloads.generate_torch(config, n, dev, seed_offset=seed_offset)
    torch.cuda.synchronize()
    log(f"[bench] generated {config} n={n} on {dev} in {time.time() - t0:.2f}s")
    return A


def run_hot(sd, A, steps, warmup, config):
    """Device-resident timing of the fused kernel on the current stream."""
    import torch
    n = A.shape[0]
    dim = COST[config]["metric_dim"]
    if dim == 2:
        out = dict(lam=torch.empty((n, 2), dtype=torch.float64, device=A.device),
                   phi=torch.empty((n,), dtype=torch.float64, device=A.device),
                   status=torch.empty((n,), dtype=torch.uint8, device=A.device))
        fn = lambda: sd.diagonalize2_batched(A, out=out)  # noqa: E731
    else:
        out = dict(lam=torch.empty((n, 3), dtype=A.dtype, device=A.device),
                   ang=torch.empty((n, 3), dtype=A.dtype, device=A.device),
                   status=torch.empty((n,), dtype=torch.uint8, device=A.device))
        fn = lambda: sd.diagonalize3_batched(A, out=out)  # noqa: E731
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    # working sets under 4x L2 (126 MB): between timed calls (outside the
    # events) overwrite a 512 MB buffer, then read another 512 MB one, so
    # every call starts from HBM with a clean L2 (the flush's own dirty lines
    # are written back during the read, not inside the next timed call)
    moved = sum(t.numel() * t.element_size() for t in [A, *out.values()])
    small = moved < 4 * L2_BYTES
    flush = torch.empty((1 << 29,), dtype=torch.uint8, device=A.device) if small else None
    rflush = torch.ones((1 << 27,), dtype=torch.float32, device=A.device) if small else None
    l0 = sd._lib.launch_count()
    for s, e in ev:
        if flush is not None:
            flush.fill_(1)
            rflush.sum()
        s.record(stream)
        fn()
        e.record(stream)
        if flush is not None:
            # microsecond-scale calls: wait here (outside the events) so the
            # next iteration's flush is on the GPU while the host enqueues the
            # timed call; otherwise the host's enqueue lag for the Python call
            # can land between the start event and the kernel
            # (tools/c1_timing_probe.py: 15.0 vs 14.1 us per c1 call)
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    launches = sd._lib.launch_count() - l0
    per = [s.elapsed_time(e) for s, e in ev]
    return per, launches, out


def iq_mean(xs):
    """Mean of the middle half of the samples."""
    xs = sorted(xs)
    k = len(xs) // 4
    return statistics.mean(xs[k:len(xs) - k])


def copy_floor(A, steps):
    """Mean event-timed ms of a device copy of A (same flush as run_hot)."""
    import torch
    src = A.reshape(-1)
    dst = torch.empty_like(src)
    flush = torch.empty((1 << 29,), dtype=torch.uint8, device=A.device)
    rflush = torch.ones((1 << 27,), dtype=torch.float32, device=A.device)
    stream = torch.cuda.current_stream()
    for _ in range(3):
        dst.copy_(src)
    ts = []
    for _ in range(steps):
        flush.fill_(1)
        rflush.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        dst.copy_(src)
        e.record(stream)
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return iq_mean(ts)


def run_sweep(sd, dev, steps=3):
    """sd_eig3 on N(0,1) rows at 2^20, 2^24, 2^28 and N_max
    (HBM-filling) in fp64 and fp32 storage, device-resident."""
    import torch
    from paper_1306_6291_b200 import workloads
    rows = []
    for dt, esz, tag in ((torch.float64, 8, "f64"), (torch.float32, 4, "f32")):
        torch.cuda.empty_cache()
        free, _ = torch.cuda.mem_get_info(dev)
        resident = 12 * esz + 1  # A + lam + ang + status
        nmax = int(0.9 * free / resident) // 4096 * 4096
        for n in (1 << 20, 1 << 24, 1 << 28, nmax):
            t0 = time.time()
            A = workloads.generate_torch("c5", n, dev, dtype=dt)
            torch.cuda.synchronize()
            gen_s = time.time() - t0
            per, launches, out = run_hot(sd, A, steps, 2, "c5")
            kt = statistics.median(per) * 1e-3
            st = out["status"]
            bad = sum(int(torch.count_nonzero((st[k:k + (1 << 26)] & 0x0F) >= 4))
                      for k in range(0, n, 1 << 26))  # internal/deferred codes never escape
            rows.append({"dtype": tag, "n": n, "n_is_max": n == nmax, "ms": kt * 1e3,
                         "value": n / kt, "unit": "matrices/s",
                         "fp64_frac": 2.0 * COST["c5"]["W"] * n / kt / 1e12,
                         "hbm_gbs": resident * n / kt / 1e9, "gen_s": gen_s,
                         "launches_per_call": launches / steps, "bad_status": bad})
            log(f"[bench] sweep {tag} n={n}: {kt * 1e3:.3f} ms")
            del A, out, st
            torch.cuda.empty_cache()
    return rows


def run_e2e(sd, config, n, steps, warmup, dev_index):
    """Host-buffer path: pinned host in/out through the C-ABI plan."""
    import torch
    from paper_1306_6291_b200 import workloads
    dim = COST[config]["metric_dim"]
    dtype = torch.float32 if config == "c4" else torch.float64
    width = 3 if dim == 2 else 6
    A_dev = workloads.generate_torch(config, n, torch.device("cuda", dev_index))
    A = torch.empty((n, width), dtype=dtype, pin_memory=True)
    A.copy_(A_dev.to(dtype))
    del A_dev
    ow = 2 if dim == 2 else 3
    lam = torch.empty((n, ow), dtype=dtype, pin_memory=True)
    ang = torch.empty((n,) if dim == 2 else (n, 3), dtype=dtype, pin_memory=True)
    st = torch.empty((n,), dtype=torch.uint8, pin_memory=True)
    plan = sd.HostPlan(dev_index, chunk=1 << 20)  # best of a 2^17..2^22 sweep (tools/exp_e2e.py)
    call = (lambda: plan.eig2(A, lam, ang, st)) if dim == 2 else \
        (lambda: plan.eig3(A, lam, ang, st))
    for _ in range(warmup):
        call()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call()  # returns after all D2H copies completed
        times.append(time.perf_counter() - t0)
    plan.close()
    esz = A.element_size()
    h2d = n * width * esz
    d2h = n * (ow + (1 if dim == 2 else 3)) * esz + n
    return times, h2d, d2h


def fp64_peak(sd, dev):
    """Measured DFMA throughput (TFLOP/s, 2 FLOP per DFMA) on this GPU."""
    import ctypes
    import torch
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks = nsm * 8
    sink = torch.empty(blocks * 256, dtype=torch.float64, device=dev)
    tot = ctypes.c_double()
    iters = 4096
    L = sd._lib.load()
    for _ in range(2):
        L.sd_probe_dfma(blocks, iters, sink.data_ptr(), ctypes.byref(tot),
                        torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        L.sd_probe_dfma(blocks, iters, sink.data_ptr(), ctypes.byref(tot),
                        torch.cuda.current_stream().cuda_stream)
        e.record()
        torch.cuda.synchronize()
        best = max(best, tot.value / (s.elapsed_time(e) * 1e-3))
    return 2.0 * best / 1e12


def cpu_baseline(config, seconds=12.0):
    """The reference algorithm (oracle C restatement) on all host cores."""
    from oracle import oracle as O
    from paper_1306_6291_b200 import workloads
    threads = O.default_threads()
    dim = COST[config]["metric_dim"]
    n = 1 << 16
    A = workloads.generate(config, n)
    fn = (lambda x: O.eig2(x, nthreads=threads)) if dim == 2 else (
        (lambda x: O.eig3_f32(x, nthreads=threads)) if config == "c4"
        else (lambda x: O.eig3(x, nthreads=threads)))
    fn(A[:4096])
    t0 = time.perf_counter()
    fn(A)
    dt = time.perf_counter() - t0
    reps = max(1, int(seconds / max(dt, 1e-6)))
    t0 = time.perf_counter()
    for _ in range(reps):
        fn(A)
    dt = time.perf_counter() - t0
    return dict(value=n * reps / dt, unit="matrices/s", cores=threads, kind="port",
                sample=f"first {n} rows of {config} x {reps} passes ({dt:.1f} s), "
                       f"oracle/symdiag_oracle.c (C restatement of the reference, "
                       f"OpenMP {threads} threads)")


def ncu_traffic(config):
    f = ROOT / "profiles" / "ncu_summary.json"
    if f.exists():
        try:
            return json.loads(f.read_text()).get(config, {}).get("dram_bytes_per_launch")
        except (ValueError, AttributeError):
            return None
    return None


def ncu_fp64_pipe(config):
    """FP64-pipe active fraction of the top kernel from the committed ncu
    capture (profiles/ncu_summary.json), or None."""
    f = ROOT / "profiles" / "ncu_summary.json"
    try:
        ks = json.loads(f.read_text()).get(config, {}).get("kernels", [])
        return ks[0]["fp64_pipe_pct"] / 100.0 if ks else None
    except (OSError, ValueError, KeyError, AttributeError):
        return None


def reference_arm(args, rank, world):
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_1306_6291_b200 import workloads
    cfg = args.config
    threads = O.default_threads()
    dim = COST[cfg]["metric_dim"]
    n = args.ref_rows
    A = workloads.generate(cfg, n)
    fn = (lambda x: O.eig2(x, nthreads=threads)) if dim == 2 else (
        (lambda x: O.eig3_f32(x, nthreads=threads)) if cfg == "c4"
        else (lambda x: O.eig3(x, nthreads=threads)))
    for _ in range(args.warmup):
        fn(A)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fn(A)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.median(times)
    value = n / (ms * 1e-3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "matrices/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64" if cfg != "c4" else "f32-io/f64",
        "data": "synthetic (seeded numpy PCG64, BASELINE.json config generator)",
        "config": {"workload": workloads.CONFIGS[cfg]["desc"], "rows_per_step": n,
                   "parallelism": "host threads (OpenMP)"},
        "cpu_baseline": {"value": value, "unit": "matrices/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{n} rows of {cfg} per step; oracle/symdiag_oracle.c "
                                   f"(C restatement of the reference, bit-pinned)"},
        "e2e": {"value": value, "unit": "matrices/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(COST))
    ap.add_argument("--n", type=int, default=0, help="override batch size")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-rows", type=int, default=1 << 16)
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sweep", action="store_true",
                    help="also run the C5 size sweep (2^20 .. N_max, fp64 and fp32)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    import paper_1306_6291_b200 as sd
    from paper_1306_6291_b200 import workloads

    sd._lib.require_cuda()
    # one rank per GPU; modulo only matters when a test runs more ranks than GPUs
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        # Control plane only (barriers, max-over-ranks of a scalar time): the
        # data path has no collective, so a CPU (gloo) group is enough and
        # keeps the run independent of NCCL topology.
        import torch.distributed as dist
        dist.init_process_group("gloo")

    cfg = args.config
    n = args.n or workloads.CONFIGS[cfg]["n"]
    A = make_inputs(cfg, n, dev, seed_offset=rank)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    with clock_sampler(dev.index) as clk:
        barrier()
        per, launches, out = run_hot(sd, A, args.steps, args.warmup, cfg)
        barrier()
    total_ms = sum(per)
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / args.steps
    value = n * world / (ms_step * 1e-3)

    result = None
    if rank == 0:
        cost = COST[cfg]
        fp64 = fp64_peak(sd, dev)
        kernel_s = statistics.median(per) * 1e-3
        fp64_achieved = 2.0 * cost["W"] * n / kernel_s / 1e12
        hbm_peak = peaks().get("hbm_gbs", 6650.0)
        hbm_achieved = cost["bytes"] * n / kernel_s / 1e9
        st = out["status"].cpu().numpy()
        mix = np.bincount(st & 0x0F, minlength=16)
        result = {
            "metric": METRIC, "value": value, "unit": "matrices/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64" if cfg != "c4" else "f32-io/f64",
            "data": "synthetic (seeded torch generator on device; BASELINE.json config "
                    "distribution; parity checked on numpy-seeded prefixes in tests/)",
            "config": {"workload": workloads.CONFIGS[cfg]["desc"], "config_id": cfg,
                       "batch_per_gpu": n, "global_batch": n * world,
                       "parallelism": f"dp{world} contiguous shards, no collective",
                       "l2": "inputs > L2 (126 MB): every step streams from HBM"},
            "gpu_launches": launches,
            "roofline": {
                "bound": "fp64", "achieved": fp64_achieved, "peak": fp64,
                "unit": "TFLOP/s", "frac": fp64_achieved / fp64,
                "traffic": ncu_traffic(cfg),
                "kernel": ("sd_eig3 call = eig3_fast_kernel + polish and literal fix-up "
                           "kernels (the fast kernel is ~98% of the step, profiles/)")
                if cost["metric_dim"] == 3 else "eig2_kernel",
                "timing": "CUDA events around each sd_eig3 call on its stream; median",
                "work_per_matrix": f"{cost['W']} FP64 instr-eq (BASELINE.md §4 cost model)",
                "peak_source": "measured: sd_probe_dfma DFMA-chain microbenchmark, this run",
                "ncu_fp64_pipe_active": ncu_fp64_pipe(cfg),
                "note": ("achieved counts the reference algorithm's FP64 work W per matrix; "
                         "the fast path executes fewer FP64 instructions than W, so frac can "
                         "exceed 1 while the pipe itself is ncu_fp64_pipe_active busy"),
            },
            "roofline_hbm": {"bound": "hbm", "achieved": hbm_achieved, "peak": hbm_peak,
                             "unit": "GB/s", "frac": hbm_achieved / hbm_peak,
                             "bytes_per_matrix": cost["bytes"],
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
            "branch_mix": {"generic": int(mix[0]), "already_diagonal_2d": int(mix[1]),
                           "double_root": int(mix[2]), "triple_root": int(mix[3]),
                           "errors": int(mix[8:].sum())},
            "clocks": clk.summary(),
        }
    del out
    if not args.no_e2e:
        # e2e through the public host-buffer C-ABI path (every rank)
        barrier()
        times, h2d, d2h = run_e2e(sd, cfg, n, max(5, args.steps // 2), 2, dev.index)
        tmax = statistics.median(times)
        if dist is not None:
            t = torch.tensor([tmax], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tmax = float(t.item())
        if result is not None:
            result["e2e"] = {"value": n * world / tmax, "unit": "matrices/s",
                             "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                             "ms_per_step": tmax * 1e3,
                             "path": "sd_eig3_f64_host: pinned host in/out, 3-stream "
                                     "chunked H2D/kernel/D2H pipeline"}
    # extras and the CPU baseline: rank 0 of a 1-GPU run only (the scaling
    # runs report the headline metric)
    if rank == 0 and world == 1 and not args.no_extra and args.n == 0:
        extra = {}
        for c in ("c1", "c3", "c4"):
            if c == cfg:
                continue
            nc = workloads.CONFIGS[c]["n"]
            Ac = make_inputs(c, nc, dev, 0)
            small = COST[c]["bytes"] * nc < 4 * L2_BYTES
            pc, _, oc = run_hot(sd, Ac, 30 if small else 5, 3, c)
            # event timestamps are quantised (~1 us) on this part: for the
            # microsecond-scale c1 call the interquartile mean of 30 calls
            # (fine-grained like a mean, robust to a stray slow call like a median)
            kt = (iq_mean(pc) if small else statistics.median(pc)) * 1e-3
            cc = COST[c]
            ach = 2.0 * cc["W"] * nc / kt / 1e12
            extra[c] = {"workload": workloads.CONFIGS[c]["desc"], "n": nc,
                        "value": nc / kt, "unit": "matrices/s", "ms_per_step": kt * 1e3,
                        "fp64_roofline_frac": ach / result["roofline"]["peak"],
                        "hbm_roofline_frac": cc["bytes"] * nc / kt / 1e9
                        / result["roofline_hbm"]["peak"],
                        "l2": ("working set < 4x L2: 512 MB buffer written, another 512 MB "
                               "read between timed calls" if small else "inputs > L2")}
            if small:
                # same-byte device copy under the same flush and timing: the
                # practical floor of one launch moving these bytes
                fl = copy_floor(Ac, 30)
                extra[c]["copy_floor"] = {
                    "ms": fl, "what": "torch copy_ of the input (same bytes read + written), "
                                      "same flush, interquartile mean of 30 event-timed "
                                      "calls",
                    "kernel_over_copy": kt * 1e3 / fl}
            del Ac, oc
            torch.cuda.empty_cache()
        result["configs_extra"] = extra
    if rank == 0 and args.sweep:
        fp = result["roofline"]["peak"]
        sweep = run_sweep(sd, dev)
        for r in sweep:
            r["fp64_frac"] /= fp
        result["sweep_c5"] = sweep
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(cfg)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
