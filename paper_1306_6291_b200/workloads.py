"""Seeded synthetic workloads for the five BASELINE.json configurations.

No public dataset is involved: BASELINE.json's configs define the inputs, and
these generators produce them (seeded numpy PCG64, the generator family the
reference's own bench uses, cli.py:176-181).  Generation runs in fixed chunks
of CHUNK matrices, each with its own `default_rng([seed, chunk_index])`, so any
prefix of a large batch is identical to a smaller batch — the parity tests and
golden fixtures therefore check exactly the first rows of the benchmarked
data.

Packed layouts (include/symdiag_b200.h):
  2x2: (a11, a12, a22);  3x3: (a11, a12, a13, a22, a23, a33).

Config table (BASELINE.json "configs"):
  c1  2x2 fp64, 2^20, iid U[-1,1], seed 0
  c2  3x3 fp64, 2^24, iid N(0,1), seed 1
  c3  3x3 fp64, 2^24, degenerate stress (R diag(l) R^T, 1/3 distinct /
      two-equal / all-equal eigenvalue classes, 1% exactly diagonal), seed 2
  c4  3x3 fp32, 2^28, SPD R diag(exp(N(0,1.5^2))) R^T, seed 3
  c5  3x3 iid N(0,1) sweep, seed 4
"""

from __future__ import annotations

import numpy as np

CHUNK = 1 << 16

CONFIGS = {
    "c1": dict(dim=2, n=1 << 20, dtype="float64", seed=0,
               desc="2x2 fp64 iid U[-1,1] (a11,a12,a22), seed 0"),
    "c2": dict(dim=3, n=1 << 24, dtype="float64", seed=1,
               desc="3x3 fp64 iid N(0,1) packed upper triangle, seed 1"),
    "c3": dict(dim=3, n=1 << 24, dtype="float64", seed=2,
               desc="3x3 fp64 degenerate stress R diag(l) R^T, seed 2"),
    "c4": dict(dim=3, n=1 << 28, dtype="float32", seed=3,
               desc="3x3 fp32 SPD structure tensors l=exp(N(0,1.5^2)), seed 3"),
    "c5": dict(dim=3, n=1 << 24, dtype="float64", seed=4,
               desc="3x3 iid N(0,1) sweep (2^20, 2^24, 2^28, N_max), seed 4"),
}


def _rng(seed: int, chunk: int) -> np.random.Generator:
    return np.random.default_rng([seed, chunk])


def _quat_rotations(q: np.ndarray) -> np.ndarray:
    """Unit quaternions (from normalised 4-D Gaussians) -> R[n,3,3]."""
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    r = np.empty((q.shape[0], 3, 3))
    r[:, 0, 0] = 1.0 - 2.0 * (y * y + z * z)
    r[:, 0, 1] = 2.0 * (x * y - w * z)
    r[:, 0, 2] = 2.0 * (x * z + w * y)
    r[:, 1, 0] = 2.0 * (x * y + w * z)
    r[:, 1, 1] = 1.0 - 2.0 * (x * x + z * z)
    r[:, 1, 2] = 2.0 * (y * z - w * x)
    r[:, 2, 0] = 2.0 * (x * z - w * y)
    r[:, 2, 1] = 2.0 * (y * z + w * x)
    r[:, 2, 2] = 1.0 - 2.0 * (x * x + y * y)
    return r


_UPPER = ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))


def _conjugate_packed(r: np.ndarray, lam: np.ndarray) -> np.ndarray:
    """Packed upper triangle of R diag(lam) R^T, summed in a fixed order."""
    out = np.empty((r.shape[0], 6))
    for col, (i, j) in enumerate(_UPPER):
        out[:, col] = ((r[:, i, 0] * lam[:, 0]) * r[:, j, 0]
                       + (r[:, i, 1] * lam[:, 1]) * r[:, j, 1]
                       + (r[:, i, 2] * lam[:, 2]) * r[:, j, 2])
    return out


def _chunk_c1(seed, k, m):
    return _rng(seed, k).uniform(-1.0, 1.0, (m, 3))


def _chunk_normal6(seed, k, m):
    return _rng(seed, k).standard_normal((m, 6))


def _chunk_c3(seed, k, m):
    rng = _rng(seed, k)
    r = _quat_rotations(rng.standard_normal((m, 4)))
    cls = rng.integers(0, 3, m)
    u = rng.uniform(-10.0, 10.0, (m, 3))
    lam = u.copy()
    two = cls == 1
    lam[two, 1] = lam[two, 0]            # exactly two equal: (x, x, y)
    three = cls == 2
    lam[three, 1] = lam[three, 0]        # all three equal: (x, x, x)
    lam[three, 2] = lam[three, 0]
    a = _conjugate_packed(r, lam)
    diag = rng.uniform(0.0, 1.0, m) < 0.01   # 1% exactly diagonal diag(lam)
    a[diag] = 0.0
    a[diag, 0] = lam[diag, 0]
    a[diag, 3] = lam[diag, 1]
    a[diag, 5] = lam[diag, 2]
    return a


def _chunk_c4(seed, k, m):
    rng = _rng(seed, k)
    r = _quat_rotations(rng.standard_normal((m, 4)))
    lam = np.exp(1.5 * rng.standard_normal((m, 3)))
    return _conjugate_packed(r, lam)


_CHUNKERS = {"c1": _chunk_c1, "c2": _chunk_normal6, "c3": _chunk_c3,
             "c4": _chunk_c4, "c5": _chunk_normal6}


def generate(config: str, n: int | None = None, start: int = 0) -> np.ndarray:
    """Rows [start, start+n) of config `config` as a packed numpy array.

    fp32 configs are generated in fp64 and rounded once at the end.
    """
    spec = CONFIGS[config]
    if n is None:
        n = spec["n"] - start
    width = 3 if spec["dim"] == 2 else 6
    out = np.empty((n, width), dtype=spec["dtype"])
    pieces = []
    pos = 0
    while pos < n:
        k, off = divmod(start + pos, CHUNK)
        take = min(CHUNK - off, n - pos)
        pieces.append((pos, k, off, take))
        pos += take

    def fill(piece):
        p, k, off, take = piece
        block = _CHUNKERS[config](spec["seed"], k, CHUNK)
        out[p:p + take] = block[off:off + take]

    if len(pieces) <= 2:
        for piece in pieces:
            fill(piece)
        return out
    # chunks are independent (own generator each): fill them on host
    # threads (numpy's generators and ufuncs release the GIL); the values do
    # not depend on the thread count
    import os
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(fill, pieces))
    return out


def generate_torch(config: str, n: int, device, seed_offset: int = 0, dtype=None):
    """Same distribution as `generate`, produced on the device by torch.

    Used by bench.py only for batches too large to build on the host in a
    few seconds (c4 at 2^28, c5 at N_max); the values are NOT identical to
    `generate` (different generator), the distribution is.  `dtype`
    overrides the config's storage type (c5 is swept in fp64 and fp32);
    values are always drawn in fp64 and cast once.
    """
    import torch

    spec = CONFIGS[config]
    g = torch.Generator(device=device)
    g.manual_seed(spec["seed"] * 1_000_003 + seed_offset)
    f64 = torch.float64
    if config == "c1":
        return (torch.rand((n, 3), generator=g, device=device, dtype=f64)
                * 2.0 - 1.0)
    odt = dtype if dtype is not None else getattr(torch, spec["dtype"])
    if config in ("c2", "c5"):
        if odt == f64 and n <= (1 << 28):
            return torch.randn((n, 6), generator=g, device=device, dtype=f64)
        out = torch.empty((n, 6), device=device, dtype=odt)  # chunked: N_max fills HBM
        step = 1 << 24
        for s in range(0, n, step):
            m = min(step, n - s)
            out[s:s + m] = torch.randn((m, 6), generator=g, device=device, dtype=f64)
        return out
    out = torch.empty((n, 6), device=device, dtype=odt)
    step = 1 << 24
    for s in range(0, n, step):
        m = min(step, n - s)
        q = torch.randn((m, 4), generator=g, device=device, dtype=f64)
        q = q / q.norm(dim=1, keepdim=True)
        w, x, y, z = q.unbind(1)
        r = torch.stack([
            1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
            2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
            2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y),
        ], dim=1).view(m, 3, 3)
        if config == "c4":
            lam = torch.exp(1.5 * torch.randn((m, 3), generator=g,
                                              device=device, dtype=f64))
        else:  # c3
            cls = torch.randint(0, 3, (m,), generator=g, device=device)
            lam = torch.rand((m, 3), generator=g, device=device,
                             dtype=f64) * 20.0 - 10.0
            lam[:, 1] = torch.where(cls >= 1, lam[:, 0], lam[:, 1])
            lam[:, 2] = torch.where(cls == 2, lam[:, 0], lam[:, 2])
        cols = []
        for i, j in _UPPER:
            cols.append((r[:, i, 0] * lam[:, 0]) * r[:, j, 0]
                        + (r[:, i, 1] * lam[:, 1]) * r[:, j, 1]
                        + (r[:, i, 2] * lam[:, 2]) * r[:, j, 2])
        a = torch.stack(cols, dim=1)
        if config == "c3":
            diag = torch.rand((m,), generator=g, device=device) < 0.01
            d = torch.zeros_like(a)
            d[:, 0], d[:, 3], d[:, 5] = lam[:, 0], lam[:, 1], lam[:, 2]
            a = torch.where(diag[:, None], d, a)
        out[s:s + m] = a.to(out.dtype)
    return out
