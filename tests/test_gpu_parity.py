"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (golden fixtures) and the CPU oracle, on a B200.

Tolerances (BASELINE.json north_star; tests/parity.py states them as code):
fp64 eigenvalues 1e-12 normwise, angles 1e-10 absolute away from
degeneracies, identical branch and sign choices; fp32 1e-5 relative.
"""

from __future__ import annotations

import io
import json
import math
import os

import numpy as np
import pytest

from conftest import load_golden
from parity import assert_parity, compare3, wrapped_diff

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1306_6291_b200 as sd  # noqa: E402
from paper_1306_6291_b200 import workloads  # noqa: E402
from oracle import oracle as O  # noqa: E402

DEV = torch.device("cuda", 0)
STATS_DIR = os.environ.get("SD_PARITY_STATS", "")


def residual_rows(A: torch.Tensor, lam: torch.Tensor, ang: torch.Tensor) -> torch.Tensor:
    """||D diag(lam) D^T - A||_F / SymMat3.scale() per row, D from the GPU's
    own compose_rotation kernel (eig3.py:504-506)."""
    A, lam, ang = A.double(), lam.double(), ang.double()
    d = sd.compose_rotation_batched(ang.contiguous()).view(-1, 3, 3)
    rec = (d * lam[:, None, :]) @ d.transpose(1, 2)
    full = torch.stack([A[:, 0], A[:, 1], A[:, 2], A[:, 1], A[:, 3], A[:, 4],
                        A[:, 2], A[:, 4], A[:, 5]], 1).view(-1, 3, 3)
    w = torch.tensor([1.0, 2.0, 2.0, 1.0, 2.0, 1.0], device=A.device, dtype=torch.float64)
    s = torch.clamp(torch.sqrt((A * A * w).sum(1)), min=1.0)
    return torch.linalg.matrix_norm(rec - full) / s


def gpu3(A, report=False, with_d=False, dtype=torch.float64):
    """The product hot path (fast kernel + deferred literal rows) unless
    `report`, which runs the SolveReport kernel.  Adds a residual column
    (report[:, 2]) either way so polished-bit differences can be gated."""
    t = torch.as_tensor(np.ascontiguousarray(A), dtype=dtype).to(DEV)
    r = sd.diagonalize3_batched(t, report=report and dtype == torch.float64,
                                with_d=with_d and dtype == torch.float64)
    torch.cuda.synchronize()
    out = dict(lam=r.lam.double().cpu().numpy(), ang=r.ang.double().cpu().numpy(),
               status=r.status.cpu().numpy())
    if r.report is not None:
        out["report"] = r.report.cpu().numpy()
    if r.d is not None:
        out["d"] = r.d.cpu().numpy()
    return out


def dump(name, stats):
    if STATS_DIR:
        os.makedirs(STATS_DIR, exist_ok=True)
        with open(os.path.join(STATS_DIR, f"{name}.json"), "w") as f:
            json.dump(stats, f, indent=1)


@pytest.mark.parametrize("name", ["edge", "c2", "c3", "c4", "u11", "adv"])
def test_eig3_matches_reference_golden(name):
    g = load_golden(f"eig3_{name}")
    got = gpu3(g["A"])
    # the adversarial set sits on decision boundaries by construction: every
    # disagreement there must be explained (tests/parity.py)
    stats = compare3(g, got, A=g["A"], explain=(name == "adv"))
    dump(f"golden_{name}", stats)
    assert_parity(stats)


@pytest.mark.parametrize("name", ["edge", "c2", "c3", "c4", "u11"])
def test_report_kernel_matches_reference_golden(name):
    """sd_eig3_report_f64: the literal path with SolveReport rows."""
    g = load_golden(f"eig3_{name}")
    got = gpu3(g["A"], report=True)
    stats = compare3(g, got, A=g["A"])
    dump(f"golden_report_{name}", stats)
    assert_parity(stats)
    ok = ((g["status"] & 0x0F) == (got["status"] & 0x0F)) & ((g["status"] & 0x0F) < 8)
    rr, gr = g["report"][ok], got["report"][ok]
    assert np.array_equal(rr[:, 3], gr[:, 3])                      # candidate count
    sc = np.maximum(1.0, np.abs(g["A"][ok]).max(axis=1))
    assert np.all(np.abs(rr[:, :2] - gr[:, :2]) <= 1e-15 * sc[:, None])  # f-norms
    for k in range(4):                                              # candidate signs
        m = rr[:, 3] > k
        assert np.array_equal(rr[m, 4 + 5 * k: 6 + 5 * k], gr[m, 4 + 5 * k: 6 + 5 * k])


def test_eig3_edge_d_matrix_matches_reference():
    g = load_golden("eig3_edge")
    got = gpu3(g["A"], with_d=True)
    ok = (g["status"] & 0x0F) < 2
    pol = ((g["status"] | got["status"]) & 0x80) != 0
    m = ok & ~pol
    assert np.nanmax(np.abs(g["d"][m] - got["d"][m])) <= 1e-10


@pytest.mark.parametrize("config,n", [("c2", 1 << 18), ("c3", 1 << 18), ("c4", 1 << 17)])
def test_eig3_matches_oracle_large_prefix(config, n):
    A = workloads.generate(config, n).astype(np.float64)
    ref = O.eig3(A, report=True, nthreads=O.default_threads())
    got = gpu3(A)
    stats = compare3(ref, got, A=A, explain=True)
    dump(f"oracle_{config}_{n}", stats)
    # every disagreement must be one the reference itself makes under 1-ulp
    # libm perturbations (tests/parity.py), none unexplained
    assert_parity(stats)


def test_rotated_scalar_rows_decide_like_glibc_pow():
    """R diag(l, l, l) R^T in floating point: p = b^2 - 3c and q are pure
    rounding noise, and the sign of q (the double-root endpoint, a ~sqrt(p)
    eigenvalue split, eig3.py:147-150) is decided by the last bit of glibc's
    pow(b, 3).  Round 1 exempted such rows as "q-noise"; with the device
    restatement of glibc's pow (classify3 gates, classify3_exact) branch,
    signs and eigenvalues must match the oracle on every row."""
    from paper_1306_6291_b200.workloads import _quat_rotations
    rng = np.random.default_rng(4242)
    n = 1 << 17
    R = _quat_rotations(rng.standard_normal((n, 4)))
    lam = rng.uniform(-10.0, 10.0, n)
    M = np.einsum("nij,nkj->nik", R * lam[:, None, None], R)
    A = np.stack([M[:, 0, 0], M[:, 0, 1], M[:, 0, 2], M[:, 1, 1], M[:, 1, 2], M[:, 2, 2]], 1)
    ref = O.eig3(A, report=True, nthreads=O.default_threads())
    got = gpu3(A)
    stats = compare3(ref, got, A=A, explain=True)
    dump("oracle_rotated_scalar", stats)
    assert (ref["status"] & 0x0F == 2).sum() > n // 20  # the q-noise population is there
    assert stats["code_mismatch"] == 0 and stats["sign_mismatch"] == 0, stats
    assert stats["lam_fail"] == 0, stats
    assert_parity(stats)


def test_adversarial_rows_match_oracle():
    """2^17 seeded rows on the decision boundaries (cases.adversarial_3x3):
    the fast path's guards must hand every ambiguous row to the literal path."""
    from cases import adversarial_3x3
    A = adversarial_3x3(1 << 17, seed=7200)
    ref = O.eig3(A, report=True, nthreads=O.default_threads())
    got = gpu3(A)
    stats = compare3(ref, got, A=A, explain=True)
    dump("oracle_adversarial", stats)
    assert_parity(stats)


def test_lastbit_rows_decide_like_the_reference():
    """Rows whose reference decisions hinge on glibc's last bits
    (tests/golden/eig3_lastbit: diagonal matrices with close entries,
    |phi2|/|phi3| within 1e-9..1e-6 of 0 or pi/2, gaps 1e-8..1e-5, plus the
    rows the round-2 2^26 sweeps flagged, incl. the two c3 DoubleRoot-vs-
    Generic rows and the c4 phi3-sign row).  The fast path must defer every
    such decision and the literal solver, with its correctly rounded libm
    (sd_crlibm.h), must then take the reference's: branch, signs, near_tie
    identical on every row, eigenvalues within 1e-12.  The sweep-flagged
    rows are in the set because their angles are ill conditioned (strict
    angles up to 5e-10 from the reference's): angle differences must be
    ones the reference itself makes under 1-ulp libm perturbations."""
    g = load_golden("eig3_lastbit")
    got = gpu3(g["A"])
    stats = compare3(g, got, A=g["A"], explain=True)
    dump("golden_lastbit", stats)
    bad = np.nonzero((got["status"] ^ g["status"]) & 0x7F)[0]
    assert len(bad) == 0, [(int(i), hex(g["status"][i]), hex(got["status"][i])) for i in bad[:8]]
    assert stats["lam_fail"] == 0, stats
    assert_parity(stats)


def test_lastbit_family_matches_cr_oracle_decisions():
    """2^17 fresh last-bit rows (cases.lastbit_3x3, another seed): the GPU's
    decisions equal, row for row, those of the oracle built with the same
    correctly rounded libm (O.eig3(cr=True)) -- the fast path defers what it
    cannot certify, the literal solver computes what the oracle computes --
    and differ from the glibc oracle's only on rows where the two oracles
    differ (a misrounded glibc call, ~2e-5 of this adversarial family)."""
    from cases import lastbit_3x3
    A = lastbit_3x3(1 << 17, seed=7301)
    ref = O.eig3(A, nthreads=O.default_threads())
    crr = O.eig3(A, nthreads=O.default_threads(), cr=True)
    got = gpu3(A)
    d_cr = np.nonzero((got["status"] ^ crr["status"]) & 0x7F)[0]
    assert len(d_cr) == 0, [(int(i), hex(crr["status"][i]), hex(got["status"][i])) for i in d_cr[:8]]
    d_ref = ((got["status"] ^ ref["status"]) & 0x7F) != 0
    oracles_differ = ((crr["status"] ^ ref["status"]) & 0x7F) != 0
    assert not (d_ref & ~oracles_differ).any()
    dump("lastbit_family", {"n": int(len(A)), "gpu_vs_glibc_decisions": int(d_ref.sum()),
                            "oracles_differ": int(oracles_differ.sum()),
                            "gpu_vs_cr_decisions": int(len(d_cr)),
                            "lam_bit_equal_vs_cr": float((got["lam"] == crr["lam"]).all(1).mean()),
                            "lam_bit_equal_vs_glibc": float((got["lam"] == ref["lam"]).all(1).mean())})


@pytest.mark.parametrize("config", ["c2", "c3", "c4"])
def test_fast_path_matches_literal_path(config):
    """sd_eig3_f64 (fast path + deferred literal rows) vs sd_eig3_literal_f64
    (reference evaluation order for every row): same branch/sign decisions,
    values within the parity tolerance, residual-gated polished bits."""
    A = torch.as_tensor(workloads.generate(config, 1 << 18).astype(np.float64)).to(DEV)
    n = A.shape[0]
    fast = sd.diagonalize3_batched(A)
    lam = torch.empty((n, 3), dtype=torch.float64, device=DEV)
    ang = torch.empty((n, 3), dtype=torch.float64, device=DEV)
    st = torch.empty((n,), dtype=torch.uint8, device=DEV)
    sd._lib.call("sd_eig3_literal_f64", A.data_ptr(), n, lam.data_ptr(), ang.data_ptr(),
                 st.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    lit = dict(lam=lam.cpu().numpy(), ang=ang.cpu().numpy(), status=st.cpu().numpy())
    got = dict(lam=fast.lam.cpu().numpy(), ang=fast.ang.cpu().numpy(),
               status=fast.status.cpu().numpy())
    assert not np.any((got["status"] & 0x0F) == 4), "deferred marker leaked"
    stats = compare3(lit, got, A=A.cpu().numpy(), explain=True)
    dump(f"fast_vs_literal_{config}", stats)
    assert_parity(stats)


def test_eig3_f32_matches_reference_within_1e5():
    g = load_golden("eig3_c4")
    got = gpu3(g["A32"], report=False, dtype=torch.float32)
    # branch codes and selected signs (fp32 storage, fp64 internals)
    assert np.array_equal(got["status"] & 0x3F, g["status"] & 0x3F)
    lam_r = g["lam"]
    rel = np.abs(got["lam"] - lam_r) / np.abs(lam_r)
    assert rel.max() <= 1e-5
    ok = ((g["status"] & 0x0F) < 2) & (((g["status"] | got["status"]) & 0x80) == 0)
    assert wrapped_diff(g["ang"][ok], got["ang"][ok]).max() <= 1e-5


def test_eig3_f32_large_matches_oracle():
    A32 = workloads.generate("c4", 1 << 17)
    ref = O.eig3_f32(A32, nthreads=O.default_threads())
    got = gpu3(A32, report=False, dtype=torch.float32)
    dec_mis = ((ref["status"] ^ got["status"]) & 0x3F) != 0  # branch code and signs
    assert dec_mis.sum() == 0, np.nonzero(dec_mis)[0][:10]
    ok = (ref["status"] & 0x0F) < 8
    rel = np.abs(got["lam"][ok].astype(np.float64) - ref["lam"][ok]) / np.abs(ref["lam"][ok])
    assert rel.max() <= 1e-5


def test_eig2_matches_reference_golden():
    g = load_golden("eig2_c1")
    t = torch.as_tensor(g["A"]).to(DEV)
    r = sd.diagonalize2_batched(t, with_d=True)
    torch.cuda.synchronize()
    st = r.status.cpu().numpy()
    assert np.array_equal(st, g["status"])
    ok = st == 0
    lam = r.lam.cpu().numpy()
    # eigenvalues2 uses only +, *, and math.hypot (restated exactly): bit-exact
    assert np.array_equal(lam[ok], g["lam"][ok])
    assert np.all(np.isnan(lam[~ok]))
    phi = r.phi.cpu().numpy()
    assert np.abs(phi[ok] - g["phi"][ok]).max() <= 1e-15
    d = r.d.cpu().numpy()
    assert np.abs(d[ok] - g["d"][ok]).max() <= 1e-15


def test_eig2_full_config_matches_oracle():
    A = workloads.generate("c1")  # the whole 2^20 benchmark batch
    ref = O.eig2(A, nthreads=O.default_threads())
    r = sd.diagonalize2_batched(torch.as_tensor(A).to(DEV))
    torch.cuda.synchronize()
    assert np.array_equal(r.status.cpu().numpy(), ref["status"])
    assert np.array_equal(r.lam.cpu().numpy(), ref["lam"])
    assert np.abs(r.phi.cpu().numpy() - ref["phi"]).max() <= 1e-15


def eig2_boundary_rows(seed=7):
    """Rows on and around every gate of the fast 2x2 path (sd_eig2.cuh
    diagonalize2_fast): the 2^500 input bound and the x**2 overflow, hypot's
    2^-1021 operand bound and subnormals, the phi = 0 gate of eig2.py:37-39
    (m near 1e-14 max(1, ||A||_F) at several scales), the octant boundary
    |2 a12| = |a11 - a22|, signed zeros, and wide-range random rows."""
    rng = np.random.default_rng(seed)
    rows = []
    big = [2.0 ** 499.9, 2.0 ** 500, np.nextafter(2.0 ** 500, 0), np.nextafter(2.0 ** 500, 1e308),
           2.0 ** 510, 1.3e154, 1.35e154, 1e300, np.inf, -np.inf, np.nan]
    for b in big:
        rows += [(b, 0.5, 0.25), (0.5, b, 0.25), (0.25, 0.5, b), (b, b, b), (b, -b, b / 3)]
    tiny = [2.0 ** -1021, np.nextafter(2.0 ** -1021, 0), 2.0 ** -1022, 2.0 ** -1023, 5e-324, 0.0]
    for t in tiny:
        rows += [(t, 0.0, 0.0), (0.0, t, 0.0), (0.0, t / 2, 0.0), (t, t, 0.0), (3 * t, t, t),
                 (1.0, t, 1.0), (t, 0.0, -t)]
    for scale in (1.0, 1e3, 1e-3, 1e10, 1e-10, 3.7):
        for d in (0.0, 0.5e-14, 0.99e-14, 1e-14, 1.01e-14, 2e-14, 2.0 ** -44, 2.0 ** -45,
                  3e-14, 1e-13, 1e-12):
            for off in (0.0, d, -d, d / 2):
                a22 = scale * rng.uniform(-1, 1)
                rows += [(a22 + scale * d, scale * off, a22), (a22, scale * off, a22 + scale * d)]
    for v in (1.0, -1.0, 3.0, 1e-300, 1e300, 2.5e-310):
        rows += [(v, v / 2, 0.0), (0.0, v / 2, v), (v, -v / 2, 0.0), (v, v / 2, -v), (v, 0.0, v),
                 (v, -0.0, v), (-0.0, v, 0.0), (0.0, -0.0, -0.0), (-0.0, 0.0, 0.0)]
    e = rng.uniform(-600, 600, (4096, 3))
    r = rng.uniform(-1, 1, (4096, 3)) * 10.0 ** rng.uniform(-3, 3, (4096, 1)) * 2.0 ** e.round()
    return np.vstack([np.array(rows, dtype=np.float64), r])


def test_eig2_fast_path_boundaries_match_oracle():
    A = eig2_boundary_rows()
    ref = O.eig2(A, d=True)
    r = sd.diagonalize2_batched(torch.as_tensor(A).to(DEV), with_d=True)
    torch.cuda.synchronize()
    st = r.status.cpu().numpy()
    assert np.array_equal(st, ref["status"])
    ok = st == 0
    lam = r.lam.cpu().numpy()
    assert np.array_equal(lam[ok], ref["lam"][ok])
    assert np.all(np.isnan(lam[~ok]))
    phi = r.phi.cpu().numpy()
    assert np.abs(phi[ok] - ref["phi"][ok]).max() <= 1e-15
    assert np.array_equal(np.signbit(phi[ok]), np.signbit(ref["phi"][ok]))


@pytest.mark.parametrize("name", ["edge", "c3"])
def test_stage_kernels_match_reference(name):
    g = load_golden(f"stages_{name}")
    A = torch.as_tensor(g["A"]).to(DEV)
    s = np.maximum(1.0, np.abs(g["A"]).max(axis=1))
    bcd, st = sd.char_coeffs_batched(A)
    st = st.cpu().numpy()
    assert np.array_equal(st, g["cc_status"])
    ok = st == 0
    bcd = bcd.cpu().numpy()
    tol = np.stack([s, s * s, s ** 3], axis=1) * 1e-14
    assert np.all(np.abs(bcd[ok] - g["bcd"][ok]) <= tol[ok])
    pqe, st = sd.pq_expanded_batched(A)
    assert np.array_equal(st.cpu().numpy(), g["pqe_status"])
    pq_ok = g["pqe_status"] == 0
    pqe = pqe.cpu().numpy()
    tol2 = np.stack([s * s, s ** 3], axis=1) * 1e-13
    assert np.all(np.abs(pqe[pq_ok] - g["pqe"][pq_ok]) <= tol2[pq_ok])
    # compute_pq on the reference's own (b, c, d): same branch decisions
    pqd, st = sd.compute_pq_batched(torch.as_tensor(g["bcd"][ok]).to(DEV))
    st = st.cpu().numpy()
    assert np.array_equal(st, g["pq_status"][ok])
    pqd = pqd.cpu().numpy()
    ref = g["pqd"][ok]
    assert np.array_equal(np.isnan(pqd[:, 2]), np.isnan(ref[:, 2]))
    assert np.array_equal(pqd[:, 0], ref[:, 0], equal_nan=True)  # p = b*b - 3c: exact
    # q uses b**3: glibc pow vs a correctly rounded cube may differ by 1 ulp
    b, c, d = (g["bcd"][ok][:, k] for k in range(3))
    qn = np.abs(2 * b ** 3) + np.abs(9 * b * c) + np.abs(27 * d)
    okq = st == 0
    assert np.all(np.abs(pqd[okq, 1] - ref[okq, 1]) <= 4e-16 * qn[okq])
    dm = ~np.isnan(ref[:, 2])
    assert np.abs(pqd[dm, 2] - ref[dm, 2]).max(initial=0) <= 1e-9
    ok2 = ok & (g["pq_status"] == 0)
    lam = sd.eigenvalues3_batched(torch.as_tensor(g["bcd"][ok2]).to(DEV),
                                  torch.as_tensor(g["pqd"][ok2]).to(DEV)).cpu().numpy()
    sc = np.maximum(1.0, np.abs(g["lam"][ok2]).max(axis=1, keepdims=True))
    assert np.all(np.abs(lam - g["lam"][ok2]) <= 1e-14 * sc)
    v, st = sd.compute_v_batched(torch.as_tensor(g["A"][ok2]).to(DEV),
                                 torch.as_tensor(g["lam"][ok2]).to(DEV))
    st = st.cpu().numpy()
    vst = g["vw_status"][ok2]
    assert np.array_equal(st[st != 0], vst[st != 0])
    # compute_w (eig3.py:198-206) on the reference's own v
    okv = np.isfinite(g["vw"][ok2][:, 0])
    vref = g["vw"][ok2][okv]
    w, st = sd.compute_w_batched(torch.as_tensor(g["A"][ok2][okv]).to(DEV),
                                 torch.as_tensor(g["lam"][ok2][okv]).to(DEV),
                                 torch.as_tensor(vref[:, 0].copy()).to(DEV))
    assert np.array_equal(st.cpu().numpy(), np.zeros(okv.sum(), np.uint8))
    assert np.array_equal(w.cpu().numpy(), vref[:, 1])


def _edge_window(ang):
    """|phi2| or |phi3| within 1e-2 of 0 or pi/2: arccos(sqrt(.)) amplifies
    1-ulp libm differences there."""
    m = np.abs(ang[:, 1:3])
    return ((m < 1e-2) | (np.abs(m - np.pi / 2) < 1e-2)).any(axis=1)


@pytest.mark.parametrize("name", ["edge", "c2", "c3", "adv"])
def test_sign_stage_kernels_match_reference_golden(name):
    """resolve_signs (eig3.py:269-386) and degenerate_double (eig3.py:389-454)
    as stage kernels, fed the reference's own (lam, v, w) / (lam, lam3):
    identical status bytes (selected signs, near_tie, exception codes),
    bit-identical f-norms (CPython hypot restated), identical candidate
    availability, angles and candidates within 1e-10 mod pi (1e-7 in the
    edge window)."""
    g = load_golden(f"signs_{name}")
    for tag, fn, args in (("rs", sd.resolve_signs_batched, ("lam", "vw")),
                          ("dd", sd.degenerate_double_batched, ("lam2",))):
        rows = np.nonzero(g[f"{tag}_status"] != 255)[0]
        ins = [torch.as_tensor(np.ascontiguousarray(g[k][rows])).to(DEV) for k in ("A",) + args]
        ang, st, rep = (x.cpu().numpy() for x in fn(*ins))
        want = g[f"{tag}_status"][rows]
        mis = st != want
        if name == "adv":
            # the adversarial set puts phi1 exactly on the +-pi/2 wrap where
            # _assemble_angles flips both signs (eig3.py:262-263): the last
            # bit of atan2 picks one of two equivalent decompositions there.
            # Only those rows may differ, and only in the sign flags.
            ra = g[f"{tag}_ang"][rows]
            boundary = np.abs(np.abs(ra[:, 0]) - np.pi / 2) < 1e-12
            assert np.all(boundary[mis]), (tag, np.nonzero(mis & ~boundary)[0][:10])
            assert np.all(((st ^ want)[mis] & 0x0F) == 0)
            mis_rows = np.nonzero(mis)[0]
        else:
            assert not mis.any(), (tag, np.nonzero(mis)[0][:10])
            mis_rows = np.zeros(0, int)
        ok = (want < 8) & ~mis
        ra, gr = g[f"{tag}_ang"][rows][ok], g[f"{tag}_report"][rows][ok]
        ang, rep = ang[ok], rep[ok]
        assert np.array_equal(rep[:, :2].view(np.uint64), gr[:, :2].view(np.uint64)), tag
        assert np.array_equal(rep[:, 3], gr[:, 3]), tag
        cand = np.arange(4, 24).reshape(4, 5)
        assert np.array_equal(np.isnan(rep[:, 4:24]), np.isnan(gr[:, 4:24])), tag
        assert np.array_equal(rep[:, cand[:, :2]], gr[:, cand[:, :2]], equal_nan=True), tag
        edge = _edge_window(ra)
        tol = np.where(edge, 1e-7, 1e-10)
        err = np.nan_to_num(wrapped_diff(ang, ra)).max(axis=1)
        assert np.all(err <= tol), (tag, float(err.max()), np.nonzero(err > tol)[0][:10])
        cerr = np.nan_to_num(wrapped_diff(rep[:, cand[:, 2:4]], gr[:, cand[:, 2:4]]))
        cerr = cerr.reshape(len(cerr), -1).max(axis=1)
        assert np.all(cerr <= tol), (tag, float(cerr.max()))
        dump(f"signs_{name}_{tag}", dict(rows=int(rows.size), wrap_flip_rows=int(mis_rows.size),
                                           ang_max=float(err.max(initial=0)),
                                           cand_max=float(cerr.max(initial=0)),
                                           ang_bit_equal=float(np.mean(np.all(ang == ra, axis=1)))))


def test_device_glibc_pow_bit_exact():
    """The device's pow (csrc/sd_glibc_pow.h, every `**` of the literal path)
    against the host's libm pow — CPython's `x ** k` — bit for bit, for the
    reference's exponents 2, 3, 6 over normal, tiny, huge, negative,
    subnormal and overflowing bases."""
    rng = np.random.default_rng(11)
    parts = [rng.standard_normal(200_000),
             rng.standard_normal(100_000) * 10.0 ** rng.integers(-160, 160, 100_000),
             rng.uniform(-10, 10, 100_000),
             np.ldexp(rng.uniform(1, 2, 20_000), rng.integers(-1074, -1000, 20_000)),
             np.array([0.0, -0.0, 1.0, -1.0, 1e154, 1.4e154, 5.7e102, 1e-160, 1e-320,
                       2.2250738585072014e-308, 3.0, -7.0])]
    x = np.concatenate(parts)
    for k in (2.0, 3.0, 6.0):
        exp = []
        for v in x.tolist():
            try:
                exp.append(v ** k)
            except OverflowError:
                exp.append(math.inf if (v > 0 or k % 2 == 0) else -math.inf)
        exp = np.array(exp)
        got = sd.glibc_pow_batched(torch.as_tensor(x).to(DEV), k).cpu().numpy()
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64)), \
            (k, int((got.view(np.uint64) != exp.view(np.uint64)).sum()))


def test_device_crlibm_equals_host_build():
    """The literal solver's libm on the device (csrc/sd_crlibm.h: quick
    double-double phase, rounding test, accurate phase) against the same
    source compiled for the host (oracle/glibc_check, which
    tests/test_crlibm.py holds to mpmath): bit for bit."""
    import ctypes
    from test_crlibm import CHECK, ev
    if not CHECK.exists():
        O.build(force=True)
    host = ctypes.CDLL(str(CHECK))
    rng = np.random.default_rng(14)
    n = 400_000
    j = np.arange(-30, 31) / 32.0
    ang = np.concatenate([j, np.nextafter(j, 5), rng.uniform(-7, 7, n),
                          10 ** rng.uniform(-12, 0, n // 4), rng.uniform(-1e5, 1e5, n // 8),
                          [0.0, -0.0, 1e-300, math.pi / 2, math.pi, -math.pi]])
    unit = np.concatenate([rng.uniform(-1, 1, n),
                           (1 - 10 ** rng.uniform(-16, -0.3, n // 2)) * rng.choice([-1, 1], n // 2),
                           10 ** rng.uniform(-9, 0, n // 4), [1.0, -1.0, 0.5, -0.5, 0.0, -0.0]])
    ya = rng.standard_normal(n) * 10 ** rng.uniform(-8, 8, n)
    xa = rng.standard_normal(n) * 10 ** rng.uniform(-8, 8, n)
    ya[:4], xa[:4] = [0.0, -0.0, 1.0, -1.0], [-1.0, -1.0, 0.0, -0.0]
    for k, (name, a, b) in enumerate([("sin", ang, None), ("cos", ang, None), ("acos", unit, None),
                                      ("asin", unit, None), ("atan2", ya, xa), ("hypot", ya, xa)]):
        got = sd.crlibm_batched(name, torch.as_tensor(a).to(DEV),
                                None if b is None else torch.as_tensor(b).to(DEV)).cpu().numpy()
        exp = ev(host, k, 0, a, b)
        bad = got.view(np.uint64) != exp.view(np.uint64)
        assert not bad.any(), (name, int(bad.sum()), a[bad][:4], got[bad][:4], exp[bad][:4])


def test_error_rows_are_nan_and_coded():
    A = np.array([[np.nan, 0, 0, 1, 0, 1], [1, np.inf, 0, 1, 0, 1],
                  [1e200, 0, 0, 1, 0, 1], [1.0, 0.0, 0.0, 2.0, 0.0, 3.0]])
    got = gpu3(A)
    assert list(got["status"][:3] & 0x0F) == [8, 8, 15]
    assert np.isnan(got["lam"][:3]).all() and np.isnan(got["ang"][:3]).all()
    assert (got["status"][3] & 0x0F) == 1


def test_deterministic_and_shard_invariant():
    A = torch.as_tensor(workloads.generate("c3", 1 << 16)).to(DEV)
    r1 = sd.diagonalize3_batched(A)
    r2 = sd.diagonalize3_batched(A)
    h = A.shape[0] // 3
    parts = [sd.diagonalize3_batched(A[:h]), sd.diagonalize3_batched(A[h:])]
    torch.cuda.synchronize()
    for k in ("lam", "ang", "status"):
        a = getattr(r1, k)
        assert torch.equal(a.view(torch.uint8) if a.dtype != torch.uint8 else a,
                           getattr(r2, k).view(torch.uint8) if a.dtype != torch.uint8
                           else getattr(r2, k))
        cat = torch.cat([getattr(parts[0], k), getattr(parts[1], k)])
        assert torch.equal(torch.nan_to_num(a.double(), nan=7.0),
                           torch.nan_to_num(cat.double(), nan=7.0))


def test_unaligned_input_path():
    A = workloads.generate("c2", 4097)
    buf = torch.empty(A.size + 1, dtype=torch.float64, device=DEV)
    buf[1:] = torch.as_tensor(A.reshape(-1)).to(DEV)
    t = buf[1:].view(-1, 6)  # 8-byte aligned only: scalar staging path
    r = sd.diagonalize3_batched(t)
    ref = sd.diagonalize3_batched(torch.as_tensor(A).to(DEV))
    torch.cuda.synchronize()
    assert torch.equal(r.lam, ref.lam) and torch.equal(r.status, ref.status)


def test_explicit_stream_and_argument_checks():
    """stream= runs on the given stream after the producer's work (a
    non-contiguous input is copied on the current stream first); mismatched
    secondary inputs are rejected before launch."""
    A = torch.as_tensor(workloads.generate("c2", 50_000)).to(DEV)
    ref = sd.diagonalize3_batched(A)
    At = A.t().contiguous().t()  # same values, column-major: forces a copy
    s = torch.cuda.Stream()
    r = sd.diagonalize3_batched(At, stream=s)
    s.synchronize()
    assert torch.equal(r.lam, ref.lam) and torch.equal(r.ang, ref.ang)
    with pytest.raises(ValueError):
        sd.compute_v_batched(A, ref.lam[:-1])
    with pytest.raises(ValueError):
        sd.diagonalize3_batched(A, out={"lam": torch.empty((50_000, 3), dtype=torch.float64)})


def test_host_plan_matches_device_path():
    A = workloads.generate("c2", 300_001)
    plan = sd.HostPlan(0, chunk=1 << 16)
    lam = np.empty((A.shape[0], 3))
    ang = np.empty((A.shape[0], 3))
    st = np.empty(A.shape[0], np.uint8)
    plan.eig3(A, lam, ang, st)
    ref = sd.diagonalize3_batched(torch.as_tensor(A).to(DEV))
    torch.cuda.synchronize()
    assert np.array_equal(lam, ref.lam.cpu().numpy())
    assert np.array_equal(ang, ref.ang.cpu().numpy())
    assert np.array_equal(st, ref.status.cpu().numpy())
    A2 = workloads.generate("c1", 70_000)
    l2, p2, s2 = np.empty((70_000, 2)), np.empty(70_000), np.empty(70_000, np.uint8)
    plan.eig2(A2, l2, p2, s2)
    r2 = sd.diagonalize2_batched(torch.as_tensor(A2).to(DEV))
    torch.cuda.synchronize()
    assert np.array_equal(l2, r2.lam.cpu().numpy())
    plan.close()


def test_full_size_properties_c2():
    """BASELINE config 2 at full size (2^24): size-independent properties."""
    A = workloads.generate_torch("c2", 1 << 24, DEV)
    r = sd.diagonalize3_batched(A)
    code = (r.status & 0x0F)
    assert int((code >= 8).sum()) == 0
    b = A[:, 0] + A[:, 3] + A[:, 5]
    w = torch.tensor([1.0, 2.0, 2.0, 1.0, 2.0, 1.0], device=DEV, dtype=torch.float64)
    s = torch.clamp(torch.sqrt((A * A * w).sum(1)), min=1.0)  # SymMat3.scale()
    assert float(((r.lam.sum(1) - b).abs() / s).max()) <= 1e-12
    d = sd.compose_rotation_batched(r.ang).view(-1, 3, 3)
    rec = (d * r.lam[:, None, :]) @ d.transpose(1, 2)
    full = torch.stack([A[:, 0], A[:, 1], A[:, 2], A[:, 1], A[:, 3], A[:, 4],
                        A[:, 2], A[:, 4], A[:, 5]], 1).view(-1, 3, 3)
    res = torch.linalg.matrix_norm(rec - full) / s
    assert float(res.max()) <= 1e-10


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_c5_hbm_filling_batch(dtype):
    """SURVEY 8(d) C5 at N_max: one sd_eig3 call over a batch that fills
    ~85% of HBM (> 2^31 rows in fp32).  Sampled rows (head, tail, seeded
    random) against the oracle on the same values; no internal code leaks."""
    torch.cuda.empty_cache()
    esz = 8 if dtype == torch.float64 else 4
    free, _ = torch.cuda.mem_get_info(DEV)
    n = int(0.85 * free / (12 * esz + 1)) // 4096 * 4096
    A = workloads.generate_torch("c5", n, DEV, dtype=dtype)
    r = sd.diagonalize3_batched(A)
    for k in range(0, n, 1 << 26):  # chunked: reductions materialise int64 temporaries
        code = r.status[k:k + (1 << 26)] & 0x0F
        assert int(torch.count_nonzero((code >= 4) & (code < 8))) == 0
    rng = np.random.default_rng(55)
    idx = np.unique(np.concatenate([np.arange(4096), np.arange(n - 4096, n),
                                    rng.integers(0, n, 8192)]))
    ti = torch.as_tensor(idx, device=DEV)
    As = A[ti].cpu().numpy()
    got = dict(lam=r.lam[ti].double().cpu().numpy(), ang=r.ang[ti].double().cpu().numpy(),
               status=r.status[ti].cpu().numpy())
    del A, r
    torch.cuda.empty_cache()
    if dtype == torch.float64:
        ref = O.eig3(As, report=True, nthreads=O.default_threads())
        stats = compare3(ref, got, A=As, explain=True)
        assert_parity(stats)
    else:
        ref = O.eig3_f32(As, nthreads=O.default_threads())
        dec_mis = ((ref["status"] ^ got["status"]) & 0x3F) != 0  # branch code and signs
        assert dec_mis.sum() <= 2
        ok = ~dec_mis & ((ref["status"] & 0x0F) < 8)
        lr = ref["lam"][ok].astype(np.float64)
        norm = np.maximum(1.0, np.abs(lr).max(axis=1, keepdims=True))  # normwise
        assert (np.abs(got["lam"][ok] - lr) / norm).max() <= 1e-5


# ---- referees: GPU Jacobi, residuals, cubic roots ------------
@pytest.mark.parametrize("dim", [3, 2])
def test_jacobi_matches_reference_golden(dim):
    """Jacobi has no transcendental calls: with numpy's FMA orders, CPython's
    hypot and IEEE division it is expected to match the reference bit for
    bit; the only difference allowed is x*x for numpy's pow(x, 2) in the
    convergence test (one sweep more or less, values then within 1e-15)."""
    g = load_golden(f"referee{dim}")
    r = sd.jacobi_batched(torch.as_tensor(g["A"]).to(DEV), dim=dim)
    torch.cuda.synchronize()
    st = r.status.cpu().numpy()
    assert np.array_equal(st, g["jstatus"])
    ok = st == 0
    ev, vec = r.evals.cpu().numpy()[ok], r.evecs.cpu().numpy().reshape(len(st), -1)[ok]
    same = np.all(ev == g["evals"][ok], axis=1) & np.all(vec == g["evecs"][ok], axis=1)
    assert same.mean() >= 0.999, same.mean()
    sc = np.maximum(1.0, np.abs(g["evals"][ok]).max(axis=1))
    assert np.all(np.abs(ev - g["evals"][ok]).max(axis=1) <= 1e-15 * sc)


def test_jacobi_large_matches_oracle():
    A = workloads.generate("c2", 1 << 16)
    ref = O.jacobi(A, dim=3, nthreads=O.default_threads())
    r = sd.jacobi_batched(torch.as_tensor(A).to(DEV), dim=3)
    torch.cuda.synchronize()
    assert np.array_equal(r.status.cpu().numpy(), ref["status"])
    ev = r.evals.cpu().numpy()
    exact = np.all(ev == ref["evals"], axis=1)
    assert exact.mean() >= 0.999
    assert np.abs(ev - ref["evals"]).max() <= 1e-13
    assert np.mean(r.sweeps.cpu().numpy() == ref["sweeps"]) >= 0.999


@pytest.mark.parametrize("dim", [3, 2])
def test_residuals_match_reference_golden(dim):
    g = load_golden(f"referee{dim}")
    ok = ~np.isnan(g["resid"][:, 0])
    A = g["A"][ok]
    dec = O.eig3(A, d=True) if dim == 3 else O.eig2(A, d=True)
    good = (dec["status"] & 0x80) == 0  # polished D is not pinned
    out = sd.residuals_batched(torch.as_tensor(A).to(DEV), torch.as_tensor(dec["lam"]).to(DEV),
                               torch.as_tensor(dec["d"]).to(DEV), dim=dim).cpu().numpy()
    assert np.all(np.abs(out[good] - g["resid"][ok][good]) <= 1e-15)


def test_cubic_roots_match_reference_golden():
    g = load_golden("referee3")
    bcd, st = O.char_coeffs(g["A"])
    use = (st == 0) & (g["rstatus"] != 2)
    roots, rst = sd.cubic_roots_batched(torch.as_tensor(bcd[use]).to(DEV))
    rst = rst.cpu().numpy()
    assert np.array_equal(rst, g["rstatus"][use])
    okr = rst == 0
    ref = g["roots"][use][okr]
    got = roots.cpu().numpy()[okr]
    sc = np.maximum(1.0, np.abs(ref).max(axis=1, keepdims=True))
    # brentq (xtol 1e-15, rtol 4 eps) vs bisection to adjacent doubles: equal
    # to 1e-13 where the root is well conditioned; near a multiple root the
    # polynomial is flat inside its rounding noise and any point there is a
    # root, so the GPU root must then be as good a root as the reference's
    b, c, d = (bcd[use][okr][:, k:k + 1] for k in range(3))
    poly = lambda x: ((x - b) * x + c) * x + d  # noqa: E731
    noise = 8 * np.finfo(float).eps * (np.abs(got) ** 3 + np.abs(b) * got ** 2
                                       + np.abs(c) * np.abs(got) + np.abs(d))
    close = np.abs(got - ref) <= 1e-13 * sc
    flat = np.abs(poly(got)) <= np.maximum(noise, np.abs(poly(ref)))
    assert np.all(close | flat)
    assert close.mean() >= 0.99


def test_referee_scalar_api():
    a = sd.SymMat3(2.0, 1.0, 3.0, 0.5, -0.25, 0.125)
    jr = sd.jacobi_eigen(a)
    dec = sd.diagonalize3(a)
    assert np.allclose(np.sort(jr.eigenvalues), np.sort(dec.lambdas), atol=1e-12)
    recon, ortho, ev = sd.residuals(a, dec)
    assert recon <= 1e-14 and ortho <= 1e-14 and max(ev) <= 1e-14
    roots = sd.cubic_roots_reference(sd.char_coeffs(a))
    assert np.allclose(sorted(roots), sorted(dec.lambdas), atol=1e-12)
    with pytest.raises(ValueError):
        sd.jacobi_eigen(a, tol=0.0)
    r2 = sd.jacobi_eigen(sd.SymMat2(1.0, 0.0, 2.0))  # (a11, a22, a12): (1 +- sqrt 17) / 2
    assert np.allclose(np.sort(r2.eigenvalues), [(1 - 17 ** 0.5) / 2, (1 + 17 ** 0.5) / 2],
                       atol=1e-13)


def test_scalar_api_matches_batched_and_raises_like_reference():
    """The reference-style scalar calls (one synchronous host-buffer call
    each) return exactly the report kernel's rows, and raise the reference's
    exceptions on error rows."""
    g = load_golden("eig3_edge")
    A = g["A"]
    batch = sd.diagonalize3_batched(torch.as_tensor(A).to(DEV), report=True, with_d=True)
    torch.cuda.synchronize()
    lam, ang, st = batch.lam.cpu().numpy(), batch.ang.cpu().numpy(), batch.status.cpu().numpy()
    d = batch.d.cpu().numpy()
    for k, row in enumerate(A):
        if (st[k] & 0x0F) >= 8:
            with pytest.raises(Exception):  # at SymMat3 construction or in the solve
                sd.diagonalize3(sd.SymMat3(row[0], row[3], row[5], row[1], row[2], row[4]))
            continue
        m = sd.SymMat3(row[0], row[3], row[5], row[1], row[2], row[4])
        dec = sd.diagonalize3(m)
        assert list(dec.lambdas) == lam[k].tolist()
        assert [dec.angles.phi1, dec.angles.phi2, dec.angles.phi3] == ang[k].tolist()
        assert np.array_equal(dec.d.reshape(-1), d[k])
    g2 = load_golden("eig2_c1")
    A2 = g2["A"][:300]
    b2 = sd.diagonalize2_batched(torch.as_tensor(A2).to(DEV), with_d=True)
    torch.cuda.synchronize()
    st2 = b2.status.cpu().numpy()
    for k, (a11, a12, a22) in enumerate(A2):
        if (st2[k] & 0x0F) >= 8:
            with pytest.raises(Exception):
                sd.diagonalize2(sd.SymMat2(a11, a22, a12))
            continue
        dec = sd.diagonalize2(sd.SymMat2(a11, a22, a12))
        assert [dec.lambda1, dec.lambda2] == b2.lam[k].tolist()
        assert dec.phi == b2.phi[k].item()
        assert np.array_equal(dec.d.reshape(-1), b2.d[k].cpu().numpy())


def test_single_process_multi_device_host_path():
    """diagonalize3_host_multi: contiguous shards on concurrent host threads,
    one HostPlan each (two on the same GPU here; one per GPU on a node),
    equal to the single-call result bit for bit."""
    A = workloads.generate("c2", 300_001)
    ref = sd.diagonalize3_batched(torch.as_tensor(A).to(DEV))
    torch.cuda.synchronize()
    lam, ang = np.empty((A.shape[0], 3)), np.empty((A.shape[0], 3))
    st = np.empty(A.shape[0], np.uint8)
    sd.diagonalize3_host_multi(A, lam, ang, st, devices=[0, 0, 0], chunk=1 << 16)
    assert np.array_equal(lam, ref.lam.cpu().numpy())
    assert np.array_equal(ang, ref.ang.cpu().numpy())
    assert np.array_equal(st, ref.status.cpu().numpy())


def test_device_resident_multi_shards_equal_single_call():
    """diagonalize3_batched_multi over shard_to_devices (contiguous shards,
    two on the same GPU here; one per GPU on a node): the concatenated
    outputs equal one call over the whole batch bit for bit."""
    A = workloads.generate("c3", 200_003)
    ref = sd.diagonalize3_batched(torch.as_tensor(A).to(DEV))
    shards = sd.shard_to_devices(A, [0, 0])
    assert [s.shape[0] for s in shards] == [100_002, 100_001]
    res = sd.diagonalize3_batched_multi(shards)
    torch.cuda.synchronize()
    for k in ("lam", "ang", "status"):
        got = torch.cat([getattr(r, k) for r in res])
        assert torch.equal(torch.nan_to_num(got, nan=7.0) if got.is_floating_point() else got,
                           torch.nan_to_num(getattr(ref, k), nan=7.0)
                           if got.is_floating_point() else getattr(ref, k)), k
    with pytest.raises(sd.CudaUnavailable):
        sd.shard_to_devices(A, [0, torch.cuda.device_count()])


@pytest.mark.parametrize("n", [1, 31, 257, 4099])
def test_no_writes_outside_outputs(n):
    """Out-of-bounds write check (compute-sanitizer is not available on the
    pool): every output is a window of a larger buffer whose guard bands hold
    a sentinel; after each entry point the guards must be untouched."""
    G = 4096  # guard elements on each side
    A = torch.as_tensor(workloads.generate("c3", n).astype(np.float64)).to(DEV)

    def window(shape, dtype):
        numel = int(np.prod(shape))
        buf = torch.full((numel + 2 * G,), 0x5A if dtype == torch.uint8 else -7.25e30,
                         dtype=dtype, device=DEV)
        return buf, buf[G:G + numel].view(*shape)

    def check(buf, dtype):
        s = 0x5A if dtype == torch.uint8 else -7.25e30
        assert bool((buf[:G] == s).all()) and bool((buf[-G:] == s).all())

    for dt in (torch.float64, torch.float32):
        bl, lam = window((n, 3), dt)
        ba, ang = window((n, 3), dt)
        bs, st = window((n,), torch.uint8)
        sd.diagonalize3_batched(A.to(dt), out={"lam": lam, "ang": ang, "status": st})
        torch.cuda.synchronize()
        for b, t in ((bl, dt), (ba, dt), (bs, torch.uint8)):
            check(b, t)
    bl, lam = window((n, 3), torch.float64)
    ba, ang = window((n, 3), torch.float64)
    bs, st = window((n,), torch.uint8)
    br, rep = window((n, 24), torch.float64)
    bd, dm = window((n, 9), torch.float64)
    sd.diagonalize3_batched(A, report=True, with_d=True,
                            out={"lam": lam, "ang": ang, "status": st, "report": rep, "d": dm})
    torch.cuda.synchronize()
    for b, t in ((bl, torch.float64), (ba, torch.float64), (bs, torch.uint8),
                 (br, torch.float64), (bd, torch.float64)):
        check(b, t)
    A2 = torch.as_tensor(workloads.generate("c1", n)).to(DEV)
    bl, lam = window((n, 2), torch.float64)
    bp, phi = window((n,), torch.float64)
    bs, st = window((n,), torch.uint8)
    bd, dm = window((n, 4), torch.float64)
    sd.diagonalize2_batched(A2, with_d=True, out={"lam": lam, "phi": phi, "status": st, "d": dm})
    torch.cuda.synchronize()
    for b, t in ((bl, torch.float64), (bp, torch.float64), (bs, torch.uint8),
                 (bd, torch.float64)):
        check(b, t)


def test_empty_batches():
    """n = 0 through every batched entry point and the host paths: empty
    outputs, no launch error."""
    e6 = torch.empty((0, 6), dtype=torch.float64, device=DEV)
    e3 = torch.empty((0, 3), dtype=torch.float64, device=DEV)
    for r in (sd.diagonalize3_batched(e6), sd.diagonalize3_batched(e6.float()),
              sd.diagonalize3_batched(e6, report=True, with_d=True)):
        assert r.lam.shape == (0, 3) and r.status.shape == (0,)
    r2 = sd.diagonalize2_batched(e3, with_d=True)
    assert r2.lam.shape == (0, 2) and r2.phi.shape == (0,)
    assert sd.jacobi_batched(e6).evals.shape == (0, 3)
    assert sd.compose_rotation_batched(e3).shape == (0, 9)
    plan = sd.HostPlan(0, chunk=1 << 10)
    z = np.empty((0, 6))
    plan.eig3(z, np.empty((0, 3)), np.empty((0, 3)), np.empty(0, np.uint8))
    plan.close()
    from paper_1306_6291_b200 import cli
    out = io.StringIO()
    assert cli.cmd_solve_native(io.StringIO(""), out) == 0 and out.getvalue() == ""
    torch.cuda.synchronize()


def test_unaligned_outputs_take_the_scalar_scan_paths():
    """status / lam / ang at odd offsets (no 8/16-byte vector scans in the
    compaction pass and fix-ups, no vector stores): results equal the
    aligned call bit for bit on a mixed batch that exercises every pass."""
    n = 70_001
    A = torch.as_tensor(workloads.generate("c3", n).astype(np.float64)).to(DEV)
    ref = sd.diagonalize3_batched(A)
    buf_s = torch.zeros(n + 3, dtype=torch.uint8, device=DEV)
    buf_l = torch.zeros(3 * n + 1, dtype=torch.float64, device=DEV)
    buf_a = torch.zeros(3 * n + 1, dtype=torch.float64, device=DEV)
    st, lam, ang = buf_s[3:], buf_l[1:].view(n, 3), buf_a[1:].view(n, 3)
    sd.diagonalize3_batched(A, out={"lam": lam, "ang": ang, "status": st})
    torch.cuda.synchronize()
    same = lambda x, y: bool(((x == y) | (torch.isnan(x) & torch.isnan(y))).all())  # noqa: E731
    assert torch.equal(st, ref.status)
    assert same(lam, ref.lam) and same(ang, ref.ang)


def test_fp32_mixed_batch_through_the_compaction_pass():
    """fp32 storage on the degenerate-stress mix: most Generic rows are handed
    to the compaction pass, their fp64 eigenvalues stashed across the fp32
    lam + ang slots meanwhile.  Same status as the oracle's fp32 entry,
    eigenvalues within 1e-5 normwise."""
    A32 = workloads.generate("c3", 1 << 17).astype(np.float32)
    ref = O.eig3_f32(A32, nthreads=O.default_threads())
    got = gpu3(A32, dtype=torch.float32)
    dec_mis = ((ref["status"] ^ got["status"]) & 0x3F) != 0  # branch code and signs
    assert dec_mis.sum() == 0, np.nonzero(dec_mis)[0][:10]
    ok = (ref["status"] & 0x0F) < 8
    lr = ref["lam"][ok].astype(np.float64)
    norm = np.maximum(1.0, np.abs(lr).max(axis=1, keepdims=True))
    assert (np.abs(got["lam"][ok] - lr) / norm).max() <= 1e-5
    gen = ok & ((ref["status"] & 0x0F) == 0) & (((ref["status"] | got["status"]) & 0x80) == 0)
    assert wrapped_diff(got["ang"][gen], ref["ang"][gen]).max() <= 1e-5
