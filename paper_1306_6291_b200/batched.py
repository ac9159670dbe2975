"""Batched tensor API: the B200 hot path.

Every function takes CUDA tensors in the packed layouts of
include/symdiag_b200.h and launches one kernel of libsymdiag_b200.so on the
current torch stream.  Outputs are freshly allocated (or caller-provided via
`out=`) CUDA tensors; per-matrix outcomes are in the uint8 `status` tensor
(see status.py), never raised.

Reference functions replaced (/root/reference/pkg/src/symdiag):
  diagonalize3_batched  <- diagonalize3 + euler_angles   eig3.py:509-576
  diagonalize2_batched  <- diagonalize2                  eig2.py:44-48
  char_coeffs_batched   <- char_coeffs                   eig3.py:102-109
  compute_pq_batched    <- compute_pq                    eig3.py:129-156
  eigenvalues3_batched  <- eigenvalues3                  eig3.py:159-174
  pq_expanded_batched   <- pq_expanded                   eig3.py:112-126
  compute_v_batched / compute_w_batched <- compute_v/w   eig3.py:183-206
  resolve_signs_batched <- resolve_signs                 eig3.py:269-386
  degenerate_double_batched <- degenerate_double         eig3.py:389-454
  f_vectors_batched / g_vectors_batched                  eig3.py:209-225
  compose_rotation_batched <- compose_rotation           core.py:229-235
"""

from __future__ import annotations

from typing import NamedTuple, Optional

import torch

from . import _lib

REPORT_STRIDE = _lib.REPORT_STRIDE


class Eig3Batch(NamedTuple):
    lam: torch.Tensor        # [n,3] solver order
    ang: torch.Tensor        # [n,3] (phi1, phi2, phi3) = Euler angles
    status: torch.Tensor     # [n] uint8
    report: Optional[torch.Tensor] = None  # [n,24] fp64 SolveReport rows
    d: Optional[torch.Tensor] = None       # [n,9] fp64 eigenvector matrix

    @property
    def euler(self) -> torch.Tensor:
        """euler_angles (eig3.py:568-576): the same triple, no extra storage."""
        return self.ang


class Eig2Batch(NamedTuple):
    lam: torch.Tensor        # [n,2]
    phi: torch.Tensor        # [n]
    status: torch.Tensor     # [n] uint8
    d: Optional[torch.Tensor] = None       # [n,4] fp64 rot2(phi)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _stream(stream=None, tensors=()) -> int:
    """Raw handle of the launch stream.  With an explicit `stream` other than
    the current one, the launch first waits for the current stream (where
    the inputs, any contiguous copies of them and the freshly allocated
    outputs were produced) and every tensor the kernel reads or writes is
    recorded on `stream`, so the caching allocator cannot hand its memory to
    current-stream work before the kernel is done with it."""
    cur = torch.cuda.current_stream()
    if stream is None or stream == cur:
        return cur.cuda_stream
    stream.wait_stream(cur)
    for t in tensors:
        if t is not None:
            t.record_stream(stream)
    return stream.cuda_stream


def _check_input(A: torch.Tensor, width: int, dtypes=(torch.float64,)) -> torch.Tensor:
    if not isinstance(A, torch.Tensor):
        raise TypeError("expected a torch.Tensor")
    if not A.is_cuda:
        _lib.require_cuda()
        raise _lib.CudaUnavailable("input must be a CUDA tensor (no CPU path)")
    if A.dtype not in dtypes:
        raise TypeError(f"dtype {A.dtype} not in {dtypes}")
    if A.dim() == 1:
        A = A.view(-1, width)
    if A.dim() != 2 or A.shape[1] != width:
        raise ValueError(f"expected shape [n, {width}], got {tuple(A.shape)}")
    return A.contiguous()


def _same_rows(n: int, dev, *ts: torch.Tensor) -> None:
    """Secondary inputs must match the primary one row for row and device."""
    for t in ts:
        if t.shape[0] != n:
            raise ValueError(f"row count mismatch: {t.shape[0]} != {n}")
        if t.device != dev:
            raise ValueError(f"inputs on different devices: {t.device} != {dev}")


def _alloc(out, key, shape, dtype, device):
    if out is not None and key in out and out[key] is not None:
        t = out[key]
        if (tuple(t.shape) != tuple(shape) or t.dtype != dtype or not t.is_contiguous()
                or t.device != device):
            raise ValueError(f"out[{key!r}] must be a contiguous {dtype} {tuple(shape)} "
                             f"tensor on {device}")
        return t
    return torch.empty(shape, dtype=dtype, device=device)


def diagonalize3_batched(A: torch.Tensor, *, report: bool = False, with_d: bool = False,
                         out: Optional[dict] = None, stream=None) -> Eig3Batch:
    """Batched diagonalize3 over packed A[n,6] (fp64, or fp32 with fp64
    internals).  `report`/`with_d` (fp64 only) add SolveReport rows and D."""
    A = _check_input(A, 6, (torch.float64, torch.float32))
    n, dev, dt = A.shape[0], A.device, A.dtype
    with torch.cuda.device(dev):
        lam = _alloc(out, "lam", (n, 3), dt, dev)
        ang = _alloc(out, "ang", (n, 3), dt, dev)
        st = _alloc(out, "status", (n,), torch.uint8, dev)
        rep = d = None
        if report or with_d:
            if dt != torch.float64:
                raise TypeError("report/with_d need fp64 input")
            rep = _alloc(out, "report", (n, REPORT_STRIDE), torch.float64, dev) if report else None
            d = _alloc(out, "d", (n, 9), torch.float64, dev) if with_d else None
            _lib.call("sd_eig3_report_f64", A.data_ptr(), n, lam.data_ptr(), ang.data_ptr(),
                      st.data_ptr(), _ptr(rep), _ptr(d),
                      _stream(stream, (A, lam, ang, st, rep, d)))
        elif dt == torch.float64:
            _lib.call("sd_eig3_f64", A.data_ptr(), n, lam.data_ptr(), ang.data_ptr(),
                      st.data_ptr(), _stream(stream, (A, lam, ang, st)))
        else:
            _lib.call("sd_eig3_f32", A.data_ptr(), n, lam.data_ptr(), ang.data_ptr(),
                      st.data_ptr(), _stream(stream, (A, lam, ang, st)))
    return Eig3Batch(lam, ang, st, rep, d)


def diagonalize2_batched(A: torch.Tensor, *, with_d: bool = False,
                         out: Optional[dict] = None, stream=None) -> Eig2Batch:
    """Batched diagonalize2 over packed A[n,3] = (a11, a12, a22)."""
    A = _check_input(A, 3)
    n, dev = A.shape[0], A.device
    with torch.cuda.device(dev):
        lam = _alloc(out, "lam", (n, 2), torch.float64, dev)
        phi = _alloc(out, "phi", (n,), torch.float64, dev)
        st = _alloc(out, "status", (n,), torch.uint8, dev)
        d = None
        if with_d:
            d = _alloc(out, "d", (n, 4), torch.float64, dev)
            _lib.call("sd_eig2_report_f64", A.data_ptr(), n, lam.data_ptr(), phi.data_ptr(),
                      st.data_ptr(), d.data_ptr(), _stream(stream, (A, lam, phi, st, d)))
        else:
            _lib.call("sd_eig2_f64", A.data_ptr(), n, lam.data_ptr(), phi.data_ptr(),
                      st.data_ptr(), _stream(stream, (A, lam, phi, st)))
    return Eig2Batch(lam, phi, st, d)


def shard_to_devices(A, devices, pin: bool = True) -> list:
    """Contiguous shards of host rows A[n, w] (numpy or CPU tensor), one per
    entry of `devices` (shard_range: sizes differ by at most one row), each
    copied to its device (from pinned memory, asynchronously on that
    device's current stream).  Returns the list of device tensors."""
    from .shard import shard_range
    _lib.require_cuda()
    if not isinstance(A, torch.Tensor):
        A = torch.from_numpy(A)
    if A.is_cuda:
        raise ValueError("shard_to_devices takes host rows")
    n, world = A.shape[0], len(devices)
    ndev = torch.cuda.device_count()
    for d in devices:
        if not 0 <= int(d) < ndev:
            raise _lib.CudaUnavailable(f"device {d} requested, {ndev} visible")
    out = []
    for r, d in enumerate(devices):
        a, b = shard_range(n, r, world)
        part = A[a:b]
        if pin:
            part = part.pin_memory()
        with torch.cuda.device(int(d)):
            out.append(part.to(torch.device("cuda", int(d)), non_blocking=pin))
    return out


def diagonalize3_batched_multi(shards: list, *, outs: Optional[list] = None,
                               streams: Optional[list] = None) -> list:
    """One process, several GPUs: `shards[i]` is a packed [n_i, 6]
    CUDA tensor on its own device (e.g. from `shard_to_devices`).  Every
    shard is launched asynchronously on its device's current stream (or
    `streams[i]`), with no collective and no synchronisation: each GPU's
    outputs stay on that GPU.  Returns one Eig3Batch per shard; row order
    within a shard is the input order, so the concatenation over shards is
    the single-call result for the concatenated input bit for bit."""
    res = []
    for i, A in enumerate(shards):
        if not isinstance(A, torch.Tensor) or not A.is_cuda:
            raise TypeError("diagonalize3_batched_multi takes CUDA tensors")
        with torch.cuda.device(A.device):
            res.append(diagonalize3_batched(
                A, out=None if outs is None else outs[i],
                stream=None if streams is None else streams[i]))
    return res


def _empty(n, w, dev, dtype=torch.float64):
    return torch.empty((n, w) if w else (n,), dtype=dtype, device=dev)


def char_coeffs_batched(A):
    A = _check_input(A, 6)
    n, dev = A.shape[0], A.device
    bcd, st = _empty(n, 3, dev), _empty(n, 0, dev, torch.uint8)
    with torch.cuda.device(dev):
        _lib.call("sd_char_coeffs_f64", A.data_ptr(), n, bcd.data_ptr(), st.data_ptr(), _stream())
    return bcd, st


def compute_pq_batched(bcd):
    bcd = _check_input(bcd, 3)
    n, dev = bcd.shape[0], bcd.device
    pqd, st = _empty(n, 3, dev), _empty(n, 0, dev, torch.uint8)
    with torch.cuda.device(dev):
        _lib.call("sd_compute_pq_f64", bcd.data_ptr(), n, pqd.data_ptr(), st.data_ptr(), _stream())
    return pqd, st


def eigenvalues3_batched(bcd, pqd):
    bcd, pqd = _check_input(bcd, 3), _check_input(pqd, 3)
    n, dev = bcd.shape[0], bcd.device
    _same_rows(n, dev, pqd)
    lam = _empty(n, 3, dev)
    with torch.cuda.device(dev):
        _lib.call("sd_eigenvalues3_f64", bcd.data_ptr(), pqd.data_ptr(), n, lam.data_ptr(),
                  _stream())
    return lam


def pq_expanded_batched(A):
    A = _check_input(A, 6)
    n, dev = A.shape[0], A.device
    pq, st = _empty(n, 2, dev), _empty(n, 0, dev, torch.uint8)
    with torch.cuda.device(dev):
        _lib.call("sd_pq_expanded_f64", A.data_ptr(), n, pq.data_ptr(), st.data_ptr(), _stream())
    return pq, st


def compute_v_batched(A, lam):
    A, lam = _check_input(A, 6), _check_input(lam, 3)
    n, dev = A.shape[0], A.device
    _same_rows(n, dev, lam)
    v, st = _empty(n, 0, dev), _empty(n, 0, dev, torch.uint8)
    with torch.cuda.device(dev):
        _lib.call("sd_compute_v_f64", A.data_ptr(), lam.data_ptr(), n, v.data_ptr(),
                  st.data_ptr(), _stream())
    return v, st


def compute_w_batched(A, lam, v):
    A, lam = _check_input(A, 6), _check_input(lam, 3)
    v = _check_input(v.reshape(-1, 1), 1)
    n, dev = A.shape[0], A.device
    _same_rows(n, dev, lam, v)
    w, st = _empty(n, 0, dev), _empty(n, 0, dev, torch.uint8)
    with torch.cuda.device(dev):
        _lib.call("sd_compute_w_f64", A.data_ptr(), lam.data_ptr(), v.data_ptr(), n,
                  w.data_ptr(), st.data_ptr(), _stream())
    return w, st


def resolve_signs_batched(A, lam, vw):
    A, lam, vw = _check_input(A, 6), _check_input(lam, 3), _check_input(vw, 2)
    n, dev = A.shape[0], A.device
    _same_rows(n, dev, lam, vw)
    ang, st, rep = _empty(n, 3, dev), _empty(n, 0, dev, torch.uint8), _empty(n, REPORT_STRIDE, dev)
    with torch.cuda.device(dev):
        _lib.call("sd_resolve_signs_f64", A.data_ptr(), lam.data_ptr(), vw.data_ptr(), n,
                  ang.data_ptr(), st.data_ptr(), rep.data_ptr(), _stream())
    return ang, st, rep


def degenerate_double_batched(A, lam2):
    A, lam2 = _check_input(A, 6), _check_input(lam2, 2)
    n, dev = A.shape[0], A.device
    _same_rows(n, dev, lam2)
    ang, st, rep = _empty(n, 3, dev), _empty(n, 0, dev, torch.uint8), _empty(n, REPORT_STRIDE, dev)
    with torch.cuda.device(dev):
        _lib.call("sd_degenerate_double_f64", A.data_ptr(), lam2.data_ptr(), n, ang.data_ptr(),
                  st.data_ptr(), rep.data_ptr(), _stream())
    return ang, st, rep


def f_vectors_batched(A):
    A = _check_input(A, 6)
    n, dev = A.shape[0], A.device
    f = _empty(n, 4, dev)
    with torch.cuda.device(dev):
        _lib.call("sd_f_vectors_f64", A.data_ptr(), n, f.data_ptr(), _stream())
    return f


def g_vectors_batched(inp):
    """inp[n,7] = (l1, l2, l3, phi2, phi3, v, w) -> g[n,4] = (g1x, g1y, g2x, g2y)."""
    inp = _check_input(inp, 7)
    n, dev = inp.shape[0], inp.device
    g = _empty(n, 4, dev)
    with torch.cuda.device(dev):
        _lib.call("sd_g_vectors_f64", inp.data_ptr(), n, g.data_ptr(), _stream())
    return g


def compose_rotation_batched(ang):
    ang = _check_input(ang, 3)
    n, dev = ang.shape[0], ang.device
    d = _empty(n, 9, dev)
    with torch.cuda.device(dev):
        _lib.call("sd_compose_rotation_f64", ang.data_ptr(), n, d.data_ptr(), _stream())
    return d


class JacobiBatch(NamedTuple):
    evals: torch.Tensor      # [n, dim] final diagonal (Jacobi order, unsorted)
    evecs: torch.Tensor      # [n, dim, dim] columns are eigenvectors
    sweeps: torch.Tensor     # [n] int32
    offdiag: torch.Tensor    # [n]
    status: torch.Tensor     # [n] uint8: 0, 1 NoConvergence, 8 NonFiniteInput


def jacobi_batched(A: torch.Tensor, dim: int = 3, tol: float = 1e-13) -> JacobiBatch:
    """Batched jacobi_eigen (oracle.py:45-84), an independent referee."""
    if tol <= 0.0:
        raise ValueError("tol must be positive")
    A = _check_input(A, 3 if dim == 2 else 6)
    n, dev = A.shape[0], A.device
    ev = _empty(n, dim, dev)
    vec = _empty(n, dim * dim, dev)
    sw = torch.empty((n,), dtype=torch.int32, device=dev)
    od = _empty(n, 0, dev)
    st = _empty(n, 0, dev, torch.uint8)
    with torch.cuda.device(dev):
        _lib.call("sd_jacobi_f64", dim, A.data_ptr(), n, float(tol), ev.data_ptr(),
                  vec.data_ptr(), sw.data_ptr(), od.data_ptr(), st.data_ptr(), _stream())
    return JacobiBatch(ev, vec.view(n, dim, dim), sw, od, st)


def residuals_batched(A: torch.Tensor, lam: torch.Tensor, d: torch.Tensor,
                      dim: int = 3) -> torch.Tensor:
    """Batched residuals (oracle.py:144-161): [n, dim+2] = (recon_rel, ortho,
    eigvec_res...) for decompositions (lam [n,dim], d [n,dim,dim])."""
    A = _check_input(A, 3 if dim == 2 else 6)
    lam = _check_input(lam.reshape(-1, dim), dim)
    d = _check_input(d.reshape(-1, dim * dim), dim * dim)
    n, dev = A.shape[0], A.device
    _same_rows(n, dev, lam, d)
    out = _empty(n, dim + 2, dev)
    with torch.cuda.device(dev):
        _lib.call("sd_residuals_f64", dim, A.data_ptr(), lam.data_ptr(), d.data_ptr(), n,
                  out.data_ptr(), _stream())
    return out


def cubic_roots_batched(bcd: torch.Tensor):
    """Batched cubic_roots_reference (oracle.py:87-133): roots [n,3] and
    status [n] (0, or 1 = ComplexRootsDetected)."""
    bcd = _check_input(bcd, 3)
    n, dev = bcd.shape[0], bcd.device
    roots, st = _empty(n, 3, dev), _empty(n, 0, dev, torch.uint8)
    with torch.cuda.device(dev):
        _lib.call("sd_cubic_roots_f64", bcd.data_ptr(), n, roots.data_ptr(), st.data_ptr(),
                  _stream())
    return roots, st


def glibc_pow_batched(x: torch.Tensor, y) -> torch.Tensor:
    """x ** y elementwise with the reference's pow (glibc 2.39 restated,
    csrc/sd_glibc_pow.h): bit-identical to CPython's float ** on the
    reference's host; y a scalar or tensor of integer-valued exponents."""
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float64:
        raise TypeError("x must be a CUDA float64 tensor")
    x = x.contiguous().view(-1)
    y = (torch.full_like(x, float(y)) if not isinstance(y, torch.Tensor)
         else y.to(device=x.device, dtype=torch.float64).contiguous().view(-1))
    _same_rows(x.shape[0], x.device, y)
    out = torch.empty_like(x)
    with torch.cuda.device(x.device):
        _lib.call("sd_glibc_pow_f64", x.data_ptr(), y.data_ptr(), x.shape[0], out.data_ptr(),
                  _stream())
    return out


_CR_FN = {"sin": 0, "cos": 1, "acos": 2, "asin": 3, "atan2": 4, "hypot": 5}


def crlibm_batched(fn: str, x: torch.Tensor, y: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The literal solver's correctly rounded libm, elementwise (csrc/sd_crlibm.h):
    fn in sin, cos, acos, asin, atan2(x, y), hypot(x, y)."""
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float64:
        raise TypeError("x must be a CUDA float64 tensor")
    code = _CR_FN[fn]
    x = x.contiguous().view(-1)
    if code >= 4:
        if y is None:
            raise ValueError(f"{fn} takes two arguments")
        y = y.to(device=x.device, dtype=torch.float64).contiguous().view(-1)
        _same_rows(x.shape[0], x.device, y)
    out = torch.empty_like(x)
    with torch.cuda.device(x.device):
        _lib.call("sd_crlibm_f64", code, x.data_ptr(), _ptr(y) if code >= 4 else None,
                  x.shape[0], out.data_ptr(), _stream())
    return out


class HostPlan:
    """End-to-end path over HOST buffers (numpy or pinned torch CPU tensors):
    chunked H2D -> kernel -> D2H, pipelined over three streams in C++
    (sd_host.cu).  Use pinned memory for full copy/compute overlap."""

    def __init__(self, device: int = 0, chunk: int = 1 << 22):
        import ctypes
        _lib.require_cuda()
        self._h = ctypes.c_void_p()
        _lib.call("sd_plan_create", device, chunk, ctypes.byref(self._h))
        self.device, self.chunk = device, chunk

    def close(self):
        if self._h:
            _lib.load().sd_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 — interpreter shutdown
            pass

    @staticmethod
    def _hp(x, n, width, kinds):
        """Pointer of a contiguous host buffer holding n*width elements of
        one of `kinds` ("f64" / "f32" / "u8"), or ValueError."""
        if isinstance(x, torch.Tensor):
            if x.is_cuda or not x.is_contiguous():
                raise ValueError("host buffers must be contiguous CPU tensors")
            kind = {torch.float64: "f64", torch.float32: "f32", torch.uint8: "u8"}.get(x.dtype)
            ptr, count = x.data_ptr(), x.numel()
        else:
            if not x.flags["C_CONTIGUOUS"]:
                raise ValueError("host buffers must be C-contiguous")
            kind = {"float64": "f64", "float32": "f32", "uint8": "u8"}.get(str(x.dtype))
            ptr, count = x.ctypes.data, x.size
        if kind not in kinds:
            raise TypeError(f"host buffer dtype {x.dtype} not in {kinds}")
        if count != n * width:
            raise ValueError(f"host buffer has {count} elements, expected {n} x {width}")
        return ptr

    def eig3(self, A, lam, ang, status):
        n = A.shape[0]
        f32 = str(A.dtype) in ("torch.float32", "float32")
        fk = ("f32",) if f32 else ("f64",)
        name = "sd_eig3_f32_host" if f32 else "sd_eig3_f64_host"
        _lib.call(name, self._h, self._hp(A, n, 6, fk), n, self._hp(lam, n, 3, fk),
                  self._hp(ang, n, 3, fk), self._hp(status, n, 1, ("u8",)))

    def eig2(self, A, lam, phi, status):
        n = A.shape[0]
        _lib.call("sd_eig2_f64_host", self._h, self._hp(A, n, 3, ("f64",)), n,
                  self._hp(lam, n, 2, ("f64",)), self._hp(phi, n, 1, ("f64",)),
                  self._hp(status, n, 1, ("u8",)))


# ---- low-latency path of the reference-style scalar calls -----------------
_scalar_plans: dict = {}
_scalar_lock = __import__("threading").Lock()


def _scalar_plan():
    """One small HostPlan per device (lazily), shared by scalar calls under a
    lock (the reference's values are safe to use from several threads)."""
    _lib.require_cuda()
    dev = torch.cuda.current_device()
    plan = _scalar_plans.get(dev)
    if plan is None:
        plan = _scalar_plans[dev] = HostPlan(dev, chunk=1024)
    return plan


class _ScalarScratch(__import__("threading").local):
    """Per-thread staging for the n = 1 drop-in calls: one float64 buffer
    (inputs and every output of one row) and one status byte, allocated once
    with their addresses cached — the scalar calls then cost one C call plus
    a tolist(), not five numpy allocations and ctypes pointer objects."""

    def __init__(self):
        import numpy as np
        self.buf = np.zeros(64)          # A[0:6] lam[6:9] ang[9:12] rep[12:36] d[36:45]
        self.st = np.zeros(8, np.uint8)
        self.p = self.buf.ctypes.data
        self.ps = self.st.ctypes.data
        self.fn3 = self.fn2 = None


_scratch = _ScalarScratch()


def eig3_report_scalar(packed):
    """One 3x3 matrix (a11, a12, a13, a22, a23, a33) through
    sd_eig3_report_f64_host -> (status, lam[3], ang[3], rep[24], d[9]) as
    Python scalars / lists."""
    sc = _scratch
    if sc.fn3 is None:
        sc.fn3 = _lib.load().sd_eig3_report_f64_host
    sc.buf[0:6] = packed
    p = sc.p
    with _scalar_lock:
        plan = _scalar_plan()
        rc = sc.fn3(plan._h, p, 1, p + 48, p + 72, sc.ps, p + 96, p + 288)
    if rc != _lib.SD_OK:
        _lib.call("sd_eig3_report_f64_host", plan._h, p, 1, p + 48, p + 72, sc.ps, p + 96, p + 288)
    v = sc.buf[6:45].tolist()
    return int(sc.st[0]), v[0:3], v[3:6], v[6:30], v[30:39]


def eig2_report_scalar(packed):
    """One 2x2 matrix (a11, a12, a22) through sd_eig2_report_f64_host ->
    (status, lam[2], phi, d[4]) as Python scalars / lists."""
    sc = _scratch
    if sc.fn2 is None:
        sc.fn2 = _lib.load().sd_eig2_report_f64_host
    sc.buf[0:3] = packed
    p = sc.p
    with _scalar_lock:
        plan = _scalar_plan()
        rc = sc.fn2(plan._h, p, 1, p + 48, p + 72, sc.ps, p + 288)
    if rc != _lib.SD_OK:
        _lib.call("sd_eig2_report_f64_host", plan._h, p, 1, p + 48, p + 72, sc.ps, p + 288)
    v = sc.buf[6:40].tolist()
    return int(sc.st[0]), v[0:2], v[3], v[30:34]


def eig3_report_host(A, report: bool = True, with_d: bool = True):
    """sd_eig3_report_f64_host on host rows A[n,6] -> numpy (lam, ang,
    status, report | None, d | None); one synchronous C call."""
    import numpy as np
    A = np.ascontiguousarray(A, np.float64).reshape(-1, 6)
    n = A.shape[0]
    lam, ang = np.empty((n, 3)), np.empty((n, 3))
    st = np.empty(n, np.uint8)
    rep = np.empty((n, REPORT_STRIDE)) if report else None
    d = np.empty((n, 9)) if with_d else None
    with _scalar_lock:
        plan = _scalar_plan()
        _lib.call("sd_eig3_report_f64_host", plan._h, A.ctypes.data, n, lam.ctypes.data,
                  ang.ctypes.data, st.ctypes.data, None if rep is None else rep.ctypes.data,
                  None if d is None else d.ctypes.data)
    return lam, ang, st, rep, d


def eig2_report_host(A, with_d: bool = True):
    """sd_eig2_report_f64_host on host rows A[n,3] = (a11, a12, a22)."""
    import numpy as np
    A = np.ascontiguousarray(A, np.float64).reshape(-1, 3)
    n = A.shape[0]
    lam, phi, st = np.empty((n, 2)), np.empty(n), np.empty(n, np.uint8)
    d = np.empty((n, 4)) if with_d else None
    with _scalar_lock:
        plan = _scalar_plan()
        _lib.call("sd_eig2_report_f64_host", plan._h, A.ctypes.data, n, lam.ctypes.data,
                  phi.ctypes.data, st.ctypes.data, None if d is None else d.ctypes.data)
    return lam, phi, st, d


def diagonalize3_host_multi(A, lam, ang, status, devices=None, chunk: int = 1 << 20):
    """One process, several GPUs: host rows A[n,6] (fp64 or
    fp32) are cut into contiguous shards, one per entry of `devices`
    (default: every visible GPU), and each shard runs through its own
    HostPlan (3-stream copy/compute pipeline) on its own host thread; the
    ctypes calls release the GIL, so the shards' PCIe links and GPUs work
    concurrently.  No collective: outputs land in the caller's host buffers."""
    import threading
    from .shard import shard_range
    _lib.require_cuda()
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    n, world = A.shape[0], len(devices)
    plans = [HostPlan(dev, chunk=chunk) for dev in devices]
    errors = []

    def work(r):
        a, b = shard_range(n, r, world)
        try:
            if b > a:
                plans[r].eig3(A[a:b], lam[a:b], ang[a:b], status[a:b])
        except Exception as e:  # noqa: BLE001 — re-raised below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for p in plans:
        p.close()
    if errors:
        raise errors[0]
