"""Pin the CPU oracle (oracle/symdiag_oracle.c) to the reference.

Bit-for-bit on every status byte, every eigenvalue, every angle (polished
rows included) and every SolveReport field.
Fixtures come from the reference itself (tests/golden/make_golden.py); the
`live` tests re-run the reference on fresh seeded samples when
/root/reference is present (build container only).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import bits_equal, load_golden, wrapped_diff
from oracle import oracle as O

POLISHED = 0x80
SETS3 = ["edge", "c2", "c3", "c4", "u11", "adv", "lastbit"]


def check_eig3_against(ref, got, A=None):
    """Bit for bit: status bytes (branch, signs, near_tie, polished), every
    eigenvalue, every angle — polished rows included: the Gauss-Newton
    polish's numpy/OpenBLAS operation orders (j.T @ j, j.T @ r, dgesv) are
    restated exactly (oracle/symdiag_oracle.c solve3 / jt_resid) — and every
    SolveReport field (f-norms, candidate tuples, near_tie, residual)."""
    st_ok = ref["status"] == got["status"]
    assert st_ok.all(), np.nonzero(~st_ok)[0][:10]
    assert bits_equal(ref["lam"], got["lam"]).all()
    ang_ok = bits_equal(ref["ang"], got["ang"]).all(axis=1)
    assert ang_ok.all(), np.nonzero(~ang_ok)[0][:10]
    rep_ok = bits_equal(ref["report"], got["report"]).all(axis=1)
    assert rep_ok.all(), np.nonzero(~rep_ok)[0][:10]


@pytest.mark.parametrize("name", SETS3)
def test_oracle_eig3_matches_golden(name):
    g = load_golden(f"eig3_{name}")
    got = O.eig3(g["A"], report=True, d=("d" in g), nthreads=2)
    check_eig3_against(g, got)
    if "d" in g:
        assert bits_equal(g["d"], got["d"]).all()


def test_oracle_f32_path_matches_upcast_golden():
    g = load_golden("eig3_c4")
    got = O.eig3_f32(g["A32"])
    assert np.array_equal(got["status"], g["status"])
    assert np.array_equal(got["lam"], g["lam"].astype(np.float32))
    assert np.array_equal(got["ang"], g["ang"].astype(np.float32))


def test_oracle_eig2_matches_golden():
    g = load_golden("eig2_c1")
    got = O.eig2(g["A"], d=True)
    assert np.array_equal(got["status"], g["status"])
    assert bits_equal(got["lam"], g["lam"]).all()
    assert bits_equal(got["phi"], g["phi"]).all()
    assert bits_equal(got["d"], g["d"]).all()


@pytest.mark.parametrize("name", ["edge", "c3"])
def test_oracle_stages_match_golden(name):
    g = load_golden(f"stages_{name}")
    A = g["A"]
    bcd, st = O.char_coeffs(A)
    assert np.array_equal(st, g["cc_status"])
    assert bits_equal(bcd, g["bcd"]).all()
    pqe, st = O.pq_expanded(A)
    assert np.array_equal(st, g["pqe_status"])
    assert bits_equal(pqe, g["pqe"]).all()
    ok = g["cc_status"] == 0
    pqd, st = O.compute_pq(bcd[ok])
    assert np.array_equal(st, g["pq_status"][ok])
    assert bits_equal(pqd, g["pqd"][ok]).all()
    ok2 = ok & (g["pq_status"] == 0)
    lam = O.eigenvalues3(g["bcd"][ok2], g["pqd"][ok2])
    assert bits_equal(lam, g["lam"][ok2]).all()
    vw, st = O.compute_vw(A[ok2], g["lam"][ok2])
    assert np.array_equal(st, g["vw_status"][ok2])
    assert bits_equal(vw, g["vw"][ok2]).all()


SIGN_SETS = ["edge", "c2", "c3", "adv"]


def check_sign_stage(g, tag, ang, st, rep, rows):
    """Status byte (sign / near-tie flags or exception code), the three
    angles and every report field the stage fills (f-norms, the candidate
    tuples), bit for bit on `rows`."""
    want_st = g[f"{tag}_status"][rows]
    assert np.array_equal(st, want_st), np.nonzero(st != want_st)[0][:10]
    ok = want_st < 8
    assert bits_equal(ang[ok], g[f"{tag}_ang"][rows][ok]).all()
    keep = np.r_[0, 1, 3:24]
    assert bits_equal(rep[ok][:, keep], g[f"{tag}_report"][rows][ok][:, keep]).all()


@pytest.mark.parametrize("name", SIGN_SETS)
def test_oracle_sign_stages_match_golden(name):
    """resolve_signs (eig3.py:269-386) and degenerate_double (eig3.py:389-454)
    called directly with the reference's own stage inputs."""
    g = load_golden(f"signs_{name}")
    rs = np.nonzero(g["rs_status"] != 255)[0]
    assert rs.size > 0
    ang, st, rep = O.resolve_signs(g["A"][rs], g["lam"][rs], g["vw"][rs])
    check_sign_stage(g, "rs", ang, st, rep, rs)
    dd = np.nonzero(g["dd_status"] != 255)[0]
    assert dd.size > 0
    ang, st, rep = O.degenerate_double(g["A"][dd], g["lam2"][dd])
    check_sign_stage(g, "dd", ang, st, rep, dd)


def test_py_hypot_is_cpython_hypot():
    rng = np.random.default_rng(11)
    for scale in (1.0, 1e-300, 1e300, 1e-160):
        x = rng.standard_normal(20000) * scale
        y = rng.standard_normal(20000) * scale * rng.uniform(0, 1, 20000) ** 4
        for a, b in zip(x.tolist(), y.tolist()):
            assert O.py_hypot(a, b) == math.hypot(a, b)
    assert O.py_hypot(0.0, 0.0) == 0.0
    assert O.py_hypot(5e-324, 5e-324) == math.hypot(5e-324, 5e-324)
    assert math.isinf(O.py_hypot(math.inf, math.nan))


def test_oracle_threads_do_not_change_results():
    g = load_golden("eig3_c3")
    a = O.eig3(g["A"], nthreads=1)
    b = O.eig3(g["A"], nthreads=4)
    for k in ("lam", "ang"):
        assert bits_equal(a[k], b[k]).all()
    assert np.array_equal(a["status"], b["status"])


# ---- live leg: re-run the reference itself on fresh samples -------------
refrun = pytest.importorskip("refrun")
live = pytest.mark.skipif(not refrun.available(),
                          reason="/root/reference not present (GPU box)")


@live
@pytest.mark.parametrize("config,n,start", [("c2", 3000, 70000), ("c3", 6000, 200000),
                                            ("c4", 3000, 5000)])
def test_oracle_matches_live_reference(config, n, start):
    from paper_1306_6291_b200 import workloads
    A = workloads.generate(config, n, start=start).astype(np.float64)
    ref = refrun.run_eig3(A)
    got = O.eig3(A, report=True)
    check_eig3_against(ref, got)


@live
def test_oracle_matches_live_reference_2x2():
    from paper_1306_6291_b200 import workloads
    A = workloads.generate("c1", 20000, start=100000)
    ref = refrun.run_eig2(A, with_d=True)
    got = O.eig2(A, d=True)
    assert np.array_equal(ref["status"], got["status"])
    assert bits_equal(ref["lam"], got["lam"]).all()
    assert bits_equal(ref["phi"], got["phi"]).all()
    assert bits_equal(ref["d"], got["d"]).all()


# ---- oracle.py referees: Jacobi bit-exact, residuals at noise
@pytest.mark.parametrize("dim", [3, 2])
def test_oracle_jacobi_matches_reference_golden(dim):
    g = load_golden(f"referee{dim}")
    o = O.jacobi(g["A"], dim=dim, nthreads=2)
    assert np.array_equal(o["status"], g["jstatus"])
    ok = g["jstatus"] == 0
    for k, gk in (("evals", "evals"), ("evecs", "evecs"), ("offdiag", "offdiag")):
        assert bits_equal(o[k][ok], g[gk][ok]).all(), k
    assert np.array_equal(o["sweeps"][ok], g["sweeps"][ok])


@pytest.mark.parametrize("dim", [3, 2])
def test_oracle_residuals_match_reference_golden(dim):
    """residuals (oracle.py:144-161) bit for bit, polished rows included:
    numpy's matmul / dgemv / norm orders restated (OpenBLAS 0.3.30)."""
    g = load_golden(f"referee{dim}")
    ok = ~np.isnan(g["resid"][:, 0])
    dec = O.eig3(g["A"][ok], d=True) if dim == 3 else O.eig2(g["A"][ok], d=True)
    res = O.residuals(g["A"][ok], dec["lam"], dec["d"], dim=dim)
    good = ~np.isnan(res[:, 0])
    assert good.sum() > 0.9 * ok.sum()
    assert bits_equal(res[good], g["resid"][ok][good]).all()


def test_numpy_small_linalg_orders_restated():
    """The operation orders the oracle restates for numpy's j.T @ j,
    j.T @ r, m @ v and np.linalg.solve (OpenBLAS 0.3.30 here) still match
    numpy bit for bit (tools/polish_orders.py)."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    import polish_orders
    ok = polish_orders.main(n=1500, seed=7)
    assert all(v == 1500 for v in ok.values()), ok
