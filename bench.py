#!/usr/bin/env python3
"""Benchmark: batched closed-form 3x3 / 2x2 symmetric diagonalization on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
                    [--impl ours|reference] [--no-extra]

One step = one pass of the hot path (sd_eig3_f64 through the C ABI) over one
resident batch of the BASELINE.json configuration.  Default workload is
config 2 (3x3 fp64 iid N(0,1), 2^24 matrices; inputs 805 MB > 126 MB L2, so
every step reads from HBM).  The timed rows are the numpy-seeded batch the
parity tests check.  N > 1: the config's batch is cut into N
contiguous shards, one per GPU, no collective on the data path (strong
scaling) — either in ONE process (`--gpus N` without torchrun: one stream
per device, asynchronous launches, then every device is synchronised) or
one rank per GPU under torchrun.  Timing = per step, CUDA events on every
device, max over devices and ranks.  `--scaling weak` gives every GPU a
full batch of its own instead.

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


def make_inputs(config, n, dev, start=0, seeded=True, seed_offset=0):
    """Rows [start, start+n) of the BASELINE.json config on `dev`.

    seeded=True (default): the numpy-seeded batch of workloads.generate —
    the very rows the parity tests and golden fixtures check (generated on
    host threads, copied once from pinned memory; outside the timed region).
    seeded=False: the same distribution drawn by torch on the device (the
    C5 sweep's HBM-filling batches, weak-scaling replicas)."""
    import torch
    from paper_1306_6291_b200 import workloads
    t0 = time.time()
    if seeded:
        A = torch.from_numpy(workloads.generate(config, n, start=start)).pin_memory()
        A = A.to(dev, non_blocking=True)
    else:
        A = workloads.generate_torch(config, n, dev, seed_offset=seed_offset)
    torch.cuda.synchronize(dev)
    log(f"[bench] {'seeded' if seeded else 'torch'} {config} rows [{start}, {start + n}) "
        f"on {dev} in {time.time() - t0:.2f}s")
    return A


def _solver(sd, A, out, dim):
    if dim == 2:
        return lambda: sd.diagonalize2_batched(A, out=out)  # noqa: E731
    return lambda: sd.diagonalize3_batched(A, out=out)  # noqa: E731


def _outputs(A, dim):
    import torch
    n = A.shape[0]
    if dim == 2:
        return dict(lam=torch.empty((n, 2), dtype=torch.float64, device=A.device),
                    phi=torch.empty((n,), dtype=torch.float64, device=A.device),
                    status=torch.empty((n,), dtype=torch.uint8, device=A.device))
    return dict(lam=torch.empty((n, 3), dtype=A.dtype, device=A.device),
                ang=torch.empty((n, 3), dtype=A.dtype, device=A.device),
                status=torch.empty((n,), dtype=torch.uint8, device=A.device))


def run_hot(sd, A, steps, warmup, config):
    """Device-resident timing of one call per step on the current stream."""
    per, launches, outs, _ = run_hot_multi(sd, [A], steps, warmup, config)
    return [p[0] for p in per], launches, outs[0]


def run_hot_multi(sd, shards, steps, warmup, config):
    """Device-resident timing over several GPUs of ONE process:
    shard i lives on its own device and runs on that device's current
    stream; every step launches all shards asynchronously, then waits for
    all of them.  Returns per-step per-device event times (ms), the launch
    count, the outputs and the per-step host wall times (first launch to
    last completion)."""
    import torch
    dim = COST[config]["metric_dim"]
    outs, fns, streams = [], [], []
    for A in shards:
        with torch.cuda.device(A.device):
            out = _outputs(A, dim)
            outs.append(out)
            fns.append(_solver(sd, A, out, dim))
            streams.append(torch.cuda.current_stream(A.device))

    def sync_all():
        for A in shards:
            torch.cuda.synchronize(A.device)

    for _ in range(warmup):
        for A, fn in zip(shards, fns):
            with torch.cuda.device(A.device):
                fn()
    sync_all()
    # working sets under 4x L2 (126 MB): between timed calls (outside the
    # events) overwrite a 512 MB buffer, then read another 512 MB one, so
    # every call starts from HBM with a clean L2 (the flush's own dirty lines
    # are written back during the read, not inside the next timed call)
    flushes = []
    for A, out in zip(shards, outs):
        moved = sum(t.numel() * t.element_size() for t in [A, *out.values()])
        small = moved < 4 * L2_BYTES
        with torch.cuda.device(A.device):
            flushes.append((torch.empty((1 << 29,), dtype=torch.uint8, device=A.device),
                            torch.ones((1 << 27,), dtype=torch.float32, device=A.device))
                           if small else None)
    any_small = any(f is not None for f in flushes)
    l0 = sd._lib.launch_count()
    ev = []
    walls = []
    for _ in range(steps):
        if any_small:
            for A, f in zip(shards, flushes):
                if f is not None:
                    with torch.cuda.device(A.device):
                        f[0].fill_(1)
                        f[1].sum()
        row = []
        t0 = time.perf_counter()
        for A, fn, st in zip(shards, fns, streams):
            with torch.cuda.device(A.device):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(st)
                fn()
                e.record(st)
                row.append((s, e))
        if any_small or len(shards) > 1:
            # microsecond-scale calls: wait here (outside the events) so the
            # next step's flush is on the GPU while the host enqueues the
            # timed call; otherwise the host's enqueue lag for the Python call
            # lands between the start event and the kernel
            # (tools/c1_timing_probe.py: 15.0 vs 14.1 us per c1 call)
            sync_all()
            walls.append(time.perf_counter() - t0)
        ev.append(row)
    sync_all()
    launches = sd._lib.launch_count() - l0
    per = [[s.elapsed_time(e) for s, e in row] for row in ev]
    return per, launches, outs, walls


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


def run_e2e(sd, config, n_global, steps, warmup, devices, start=0):
    """Host-buffer path through the public API: pinned host in/out, H2D +
    kernel + D2H inside the timed region.  One device: HostPlan (C-ABI
    3-stream chunked pipeline).  Several devices of one process:
    diagonalize3_host_multi (contiguous shards, one HostPlan and host thread
    per GPU).  Rows [start, start + n_global) of the seeded batch."""
    import torch
    from paper_1306_6291_b200 import workloads
    dim = COST[config]["metric_dim"]
    dtype = torch.float32 if config == "c4" else torch.float64
    width = 3 if dim == 2 else 6
    n = n_global
    A = torch.from_numpy(workloads.generate(config, n, start=start)).pin_memory()
    ow = 2 if dim == 2 else 3
    lam = torch.empty((n, ow), dtype=dtype, pin_memory=True)
    ang = torch.empty((n,) if dim == 2 else (n, 3), dtype=dtype, pin_memory=True)
    st = torch.empty((n,), dtype=torch.uint8, pin_memory=True)
    plan = None
    if len(devices) == 1:
        plan = sd.HostPlan(devices[0], chunk=1 << 20)  # best of a 2^17..2^22 sweep (tools/exp_e2e.py)
        call = (lambda: plan.eig2(A, lam, ang, st)) if dim == 2 else \
            (lambda: plan.eig3(A, lam, ang, st))
    else:
        if dim == 2:
            raise SystemExit("multi-device e2e is 3x3 only")
        call = lambda: sd.diagonalize3_host_multi(A, lam, ang, st, devices=devices)  # noqa: E731
    for _ in range(warmup):
        call()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call()  # returns after all D2H copies completed
        times.append(time.perf_counter() - t0)
    if plan is not None:
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


def _oracle_fn(config, threads):
    from oracle import oracle as O
    dim = COST[config]["metric_dim"]
    if dim == 2:
        return lambda x: O.eig2(x, nthreads=threads)  # noqa: E731
    if config == "c4":
        return lambda x: O.eig3_f32(x, nthreads=threads)  # noqa: E731
    return lambda x: O.eig3(x, nthreads=threads)  # noqa: E731


def cpu_baseline(config, seconds=12.0):
    """The reference algorithm (oracle C restatement) on all host cores.
    Also returns the oracle's branch mix on that prefix (the timed batch's
    first rows), for comparison with the GPU's mix over the whole batch."""
    from oracle import oracle as O
    from paper_1306_6291_b200 import workloads
    threads = O.default_threads()
    n = 1 << 16
    A = workloads.generate(config, n)
    fn = _oracle_fn(config, threads)
    fn(A[:4096])
    t0 = time.perf_counter()
    r = fn(A)
    dt = time.perf_counter() - t0
    reps = max(1, int(seconds / max(dt, 1e-6)))
    t0 = time.perf_counter()
    for _ in range(reps):
        fn(A)
    dt = time.perf_counter() - t0
    base = dict(value=n * reps / dt, unit="matrices/s", cores=threads, kind="port",
                sample=f"first {n} rows of {config} x {reps} passes ({dt:.1f} s), "
                       f"oracle/symdiag_oracle.c (C restatement of the reference, "
                       f"OpenMP {threads} threads)")
    return base, (r["status"], n)


def _mix(codes):
    mix = np.bincount(np.asarray(codes) & 0x0F, minlength=16)
    return {"generic": int(mix[0]), "already_diagonal_2d": int(mix[1]),
            "double_root": int(mix[2]), "triple_root": int(mix[3]),
            "errors": int(mix[8:].sum())}


def ncu_summary(config):
    f = ROOT / "profiles" / "ncu_summary.json"
    try:
        return json.loads(f.read_text()).get(config, {})
    except (OSError, ValueError, AttributeError):
        return {}


def executed_fp64_per_row(config):
    """FP64-pipe thread-instructions (DFMA + DMUL + DADD, predicated on)
    executed per row by one sd_eig3 / sd_eig2 call, summed over its
    kernels, from the committed ncu capture (profiles/ncu_summary.json,
    tools/ncu_summary.py), or None."""
    s = ncu_summary(config)
    ks, n = s.get("kernels", []), s.get("n")
    try:
        tot = sum(k["dfma_thread_inst"] + k["dmul_thread_inst"] + k["dadd_thread_inst"]
                  for k in ks)
    except (KeyError, TypeError):
        return None
    return tot / n if ks and n else None


def reference_arm(args, rank, world):
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_1306_6291_b200 import workloads
    cfg = args.config
    threads = O.default_threads()
    n = args.ref_rows
    A = workloads.generate(cfg, n)
    fn = _oracle_fn(cfg, threads)
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
        "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
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
    ap.add_argument("--n", type=int, default=0, help="override the global batch size")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong (default, SURVEY 8e): contiguous shards of the config's "
                         "global batch; weak: every GPU gets a full batch of its own")
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
    from paper_1306_6291_b200.shard import shard_range

    sd._lib.require_cuda()
    ndev = torch.cuda.device_count()
    dist = None
    if world > 1:
        # torchrun: one rank (process) per GPU.  Control plane only (barriers,
        # max-over-ranks of a scalar time): the data path has no collective,
        # so a CPU (gloo) group is enough.
        import torch.distributed as dist
        dist.init_process_group("gloo")
        devices = [local % ndev]  # modulo only matters when a test runs more ranks than GPUs
        n_units = world
        my_units = [rank]
    else:
        # one process driving --gpus devices: one stream per device,
        # asynchronous launches, then every device is synchronised
        if args.gpus > ndev:
            raise SystemExit(f"--gpus {args.gpus} requested but only {ndev} CUDA devices "
                             f"are visible")
        devices = list(range(args.gpus))
        n_units = args.gpus
        my_units = list(range(args.gpus))
    torch.cuda.set_device(devices[0])

    cfg = args.config
    n_global = args.n or workloads.CONFIGS[cfg]["n"]
    if args.scaling == "weak":
        ranges = [(0, n_global) for _ in my_units]
        total_rows = n_global * n_units
    else:
        ranges = [shard_range(n_global, u, n_units) for u in my_units]
        total_rows = n_global
    shards = [make_inputs(cfg, b - a, torch.device("cuda", d), start=a)
              for d, (a, b) in zip(devices, ranges)]

    def barrier():
        if dist is not None:
            dist.barrier()
        for d in devices:
            torch.cuda.synchronize(d)

    barrier()
    with clock_sampler(devices[0]) as clk:
        barrier()
        per, launches, outs, walls = run_hot_multi(sd, shards, args.steps, args.warmup, cfg)
        barrier()
    # per step: the slowest device of this process, then the slowest rank
    step_ms = [max(row) for row in per]
    total_ms = sum(step_ms)
    if dist is not None:
        t = torch.tensor([total_ms, float(launches)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t[0].item())
        launches = int(t[1].item()) * world
    ms_step = total_ms / args.steps
    value = total_rows / (ms_step * 1e-3)

    result = None
    if rank == 0:
        cost = COST[cfg]
        dev0 = torch.device("cuda", devices[0])
        dfma_tf = fp64_peak(sd, dev0)                      # TFLOP/s = 2 x DFMA/s
        kernel_s = statistics.median(step_ms) * 1e-3
        rows_per_dev = ranges[0][1] - ranges[0][0]
        # executed-work roofline: FP64-pipe thread-instructions
        # this call executes (ncu, per row) over the measured DFMA rate
        ex = executed_fp64_per_row(cfg)
        dev_rate = rows_per_dev / kernel_s               # rows/s of the slowest device
        alg_tf = 2.0 * cost["W"] * dev_rate / 1e12
        achieved = 2.0 * ex * dev_rate / 1e12 if ex else None
        nsum = ncu_summary(cfg)
        top = (nsum.get("kernels") or [{}])[0]
        hbm_peak = peaks().get("hbm_gbs", 6650.0)
        hbm_achieved = cost["bytes"] * dev_rate / 1e9
        st = torch.cat([o["status"].cpu() for o in outs]).numpy()
        scale_desc = (f"dp{n_units} contiguous shards of the {n_global}-row batch, "
                      f"no collective" if args.scaling == "strong"
                      else f"dp{n_units}, a full {n_global}-row batch per GPU, no collective")
        result = {
            "metric": METRIC, "value": value, "unit": "matrices/s", "n_gpus": n_units,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64" if cfg != "c4" else "f32-io/f64",
            "data": "synthetic: the numpy-seeded BASELINE.json batch of workloads.generate "
                    "(the rows the parity tests check), copied to HBM before timing",
            "config": {"workload": workloads.CONFIGS[cfg]["desc"], "config_id": cfg,
                       "global_batch": total_rows,
                       "shard_rows": [b - a for a, b in ranges],
                       "launch": "torchrun, one rank per GPU" if dist is not None
                       else f"one process, {len(devices)} device(s), one stream each",
                       "parallelism": scale_desc,
                       "timing": "per step: CUDA events per device, max over devices "
                                 "and ranks",
                       "l2": ("inputs > L2 (126 MB): every step streams from HBM"
                              if cost["bytes"] * rows_per_dev >= 4 * L2_BYTES else
                              "512 MB written + 512 MB read between timed calls")},
            "gpu_launches": launches,
            "roofline": {
                "bound": "fp64", "achieved": achieved, "peak": dfma_tf,
                "unit": "TFLOP/s", "frac": achieved / dfma_tf if achieved else None,
                "traffic": nsum.get("dram_bytes_per_launch"),
                "kernel": ("sd_eig3 call = eig3_fast_kernel + compaction pass + fix-up "
                           "kernels (the fast kernel is ~98% of the call, profiles/)")
                if cost["metric_dim"] == 3 else "eig2_kernel",
                "definition": "executed FP64-pipe thread-instructions (DFMA+DMUL+DADD, "
                              "ncu smsp__sass_thread_inst_executed_op_*_pred_on.sum, per "
                              "row, profiles/ncu_summary.json) x rows/s of one device, "
                              "each counted as the 2 FLOP a DFMA slot does; peak = measured "
                              "DFMA rate x 2 (sd_probe_dfma, this run); frac <= 1 by "
                              "construction",
                "fp64_thread_inst_per_row": ex,
                "ncu_fp64_pipe_active": (top.get("fp64_pipe_pct") or 0) / 100.0 or None,
                "ncu_threads_per_inst": top.get("threads_per_inst"),
                "algorithm_equivalent": {
                    "achieved": alg_tf, "frac": alg_tf / dfma_tf,
                    "work_per_matrix": f"{cost['W']} FP64 instr-eq of the reference "
                                       f"algorithm (BASELINE.md §4 cost model)",
                    "note": "reference-work-equivalent throughput, not a utilisation: "
                            "the fast path executes fewer FP64 instructions than W"},
            },
            "roofline_hbm": {"bound": "hbm", "achieved": hbm_achieved, "peak": hbm_peak,
                             "unit": "GB/s", "frac": hbm_achieved / hbm_peak,
                             "bytes_per_matrix": cost["bytes"],
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
            "branch_mix": _mix(st),
            "clocks": clk.summary(),
        }
        if walls:
            result["config"]["host_wall_ms_per_step"] = 1e3 * statistics.median(walls)
    for o in outs:
        o.clear()
    if not args.no_e2e:
        # e2e through the public host-buffer API: this process's rows, pinned
        # host in/out, copies inside the timed region
        barrier()
        a0, b0 = ranges[0][0], ranges[-1][1]
        if args.scaling == "weak":
            times, h2d, d2h = run_e2e(sd, cfg, n_global * len(devices), max(5, args.steps // 2),
                                      2, devices) if len(devices) > 1 else \
                run_e2e(sd, cfg, n_global, max(5, args.steps // 2), 2, devices)
        else:
            times, h2d, d2h = run_e2e(sd, cfg, b0 - a0, max(5, args.steps // 2), 2, devices,
                                      start=a0)
        tmax = statistics.median(times)
        if dist is not None:
            t = torch.tensor([tmax, float(h2d), float(d2h)], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tmax = float(t[0].item())
            h2d, d2h = int(t[1].item()) * world, int(t[2].item()) * world
        if result is not None:
            result["e2e"] = {"value": total_rows / tmax, "unit": "matrices/s",
                             "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                             "ms_per_step": tmax * 1e3,
                             "path": ("HostPlan / sd_eig3_f64_host: pinned host in/out, "
                                      "3-stream chunked H2D/kernel/D2H pipeline")
                             if len(devices) == 1 else
                             "diagonalize3_host_multi: one HostPlan + host thread per GPU"}
    # extras and the CPU baseline: rank 0 of a 1-GPU run only (the scaling
    # runs report the headline metric)
    single = world == 1 and len(devices) == 1
    if rank == 0 and single and not args.no_extra and args.n == 0:
        dev = torch.device("cuda", devices[0])
        extra = {}
        for c in ("c1", "c3", "c4"):
            if c == cfg:
                continue
            nc = workloads.CONFIGS[c]["n"]
            Ac = make_inputs(c, nc, dev)
            small = COST[c]["bytes"] * nc < 4 * L2_BYTES
            pc, _, oc = run_hot(sd, Ac, 30 if small else 5, 3, c)
            # event timestamps are quantised (~1 us) on this part: for the
            # microsecond-scale c1 call the interquartile mean of 30 calls
            # (fine-grained like a mean, robust to a stray slow call like a median)
            kt = (iq_mean(pc) if small else statistics.median(pc)) * 1e-3
            cc = COST[c]
            exc = executed_fp64_per_row(c)
            extra[c] = {"workload": workloads.CONFIGS[c]["desc"], "n": nc,
                        "value": nc / kt, "unit": "matrices/s", "ms_per_step": kt * 1e3,
                        "fp64_executed_frac": (exc * nc / kt / (dfma_tf * 0.5e12)
                                               if exc else None),
                        "fp64_algorithm_equivalent_frac": 2.0 * cc["W"] * nc / kt / 1e12
                        / dfma_tf,
                        "hbm_roofline_frac": cc["bytes"] * nc / kt / 1e9
                        / result["roofline_hbm"]["peak"],
                        "branch_mix": _mix(oc["status"].cpu().numpy()),
                        "data": "numpy-seeded BASELINE.json batch",
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
                # the same kernel on a batch large enough to amortise the
                # fixed ~8 us of one launch: 2^24 rows of the same generator
                nb = 1 << 24
                Ab = make_inputs(c, nb, dev)
                pb, _, ob = run_hot(sd, Ab, 5, 3, c)
                kb = statistics.median(pb) * 1e-3
                extra[c]["same_kernel_2p24_rows"] = {
                    "n": nb, "value": nb / kb, "unit": "matrices/s", "ms_per_step": kb * 1e3,
                    "hbm_roofline_frac": cc["bytes"] * nb / kb / 1e9
                    / result["roofline_hbm"]["peak"], "l2": "inputs > L2"}
                del Ab, ob
            del Ac, oc
            torch.cuda.empty_cache()
        result["configs_extra"] = extra
    if rank == 0 and args.sweep:
        sweep = run_sweep(sd, torch.device("cuda", devices[0]))
        for r in sweep:
            r["fp64_frac"] /= result["roofline"]["peak"]
        result["sweep_c5"] = sweep
    if rank == 0 and single and not args.no_cpu:
        base, (ost, on) = cpu_baseline(cfg)
        result["cpu_baseline"] = base
        result["branch_mix_oracle_prefix"] = dict(_mix(ost), rows=on)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
