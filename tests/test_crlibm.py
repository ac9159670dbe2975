"""The literal solver's libm (paper_1306_6291_b200/csrc/sd_crlibm.h):
correctly rounded sin, cos, acos, asin, atan2 and hypot, compiled here as
plain C (oracle/glibc_check/crlibm_check.c) -- the same source the device
compiles.

* its constants equal their generator (tools/gen_crlibm_consts.py);
* every result equals the correctly rounded value (400-bit mpmath) on
  seeded random and edge arguments;
* it agrees with glibc (the reference's libm) wherever glibc rounds
  correctly, i.e. on >= 99.5% of arguments;
* the oracle built with it (oracle/cr_variant.c: what the device's literal
  solver computes) takes the reference's decisions -- branch, signs, flags
  -- on every row of the golden sets, including eig3_lastbit, the rows
  whose decisions hinge on libm's last bits.
The GPU legs are test_gpu_parity.py::test_lastbit_*.
"""

from __future__ import annotations

import ctypes
import math
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O

ROOT = Path(__file__).resolve().parents[1]
CHECK = ROOT / "oracle" / "build" / "libcrlibm_check.so"
P = ctypes.POINTER(ctypes.c_double)


@pytest.fixture(scope="module")
def cr():
    if not CHECK.exists():
        O.build(force=True)
    return ctypes.CDLL(str(CHECK))


def ev(lib, fn, which, x, y=None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = x if y is None else np.ascontiguousarray(y, dtype=np.float64)
    out = np.empty_like(x)
    lib.cr_eval(fn, which, x.ctypes.data_as(P), y.ctypes.data_as(P), out.ctypes.data_as(P),
                ctypes.c_long(len(x)))
    return out


def test_constants_match_generator():
    pytest.importorskip("mpmath")
    sys.path.insert(0, str(ROOT / "tools"))
    import gen_crlibm_consts as g
    assert g.render() == g.OUT.read_text()


def _args(rng, fn, n):
    tiny = np.array([0.0, -0.0, 5e-324, 1e-300, 2.0 ** -27, 2.0 ** -26, 1e-9, 0.5, 1.0])
    if fn in (0, 1):  # sin, cos: every angle the solver takes, plus reduction edges
        k = np.arange(-8, 9)
        pio2 = np.array([math.pi / 2, 0.5 * math.pi])
        edges = np.concatenate([k * math.pi / 2, np.nextafter(k * math.pi / 2, 10),
                                np.nextafter(k * math.pi / 2, -10), tiny, -tiny, pio2])
        return np.concatenate([edges, rng.uniform(-7, 7, n), rng.uniform(-1e5, 1e5, n // 8)])
    if fn in (2, 3):  # acos, asin on [-1, 1], dense near +-1 and +-0.5
        near = 1 - 10 ** rng.uniform(-16, -0.3, n // 2)
        edges = np.array([1.0, -1.0, 0.5, -0.5, np.nextafter(0.5, 1), np.nextafter(-0.5, -1),
                          np.nextafter(1, 0), np.nextafter(-1, 0), 0.0, -0.0, 1e-300, 2 ** -26])
        return np.concatenate([edges, rng.uniform(-1, 1, n), near * rng.choice([-1, 1], n // 2)])
    return None


def test_exactly_rounded_against_mpmath(cr):
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.prec = 200
    rng = np.random.default_rng(11)
    F = {0: mpmath.sin, 1: mpmath.cos, 2: mpmath.acos, 3: mpmath.asin}
    for fn in range(4):
        x = _args(rng, fn, 3000)
        got = ev(cr, fn, 0, x)
        ref = np.array([float(F[fn](mpmath.mpf(v))) for v in x])
        # signed zeros: sin/asin keep the argument's
        assert np.array_equal(got, ref), (fn, x[got != ref][:5])
        z = ref == 0
        assert np.array_equal(np.signbit(got[z]), np.signbit(ref[z]) | (np.signbit(x[z]) & (fn in (0, 3))))
    # atan2 and hypot: mixed magnitudes and quadrants
    y = rng.standard_normal(3000) * 10 ** rng.uniform(-8, 8, 3000)
    x = rng.standard_normal(3000) * 10 ** rng.uniform(-8, 8, 3000)
    y[:4], x[:4] = [0.0, -0.0, 1.0, -1.0], [-1.0, -1.0, 0.0, -0.0]
    got = ev(cr, 4, 0, y, x)
    ref = np.array([float(mpmath.atan2(mpmath.mpf(a), mpmath.mpf(b))) for a, b in zip(y, x)])
    ref = np.where(y == 0, np.copysign(ref, y), ref)   # C99: atan2(-0, x<0) = -pi
    assert np.array_equal(got, ref)
    got = ev(cr, 5, 0, y, x)
    ref = np.array([float(mpmath.sqrt(mpmath.mpf(a) ** 2 + mpmath.mpf(b) ** 2)) for a, b in zip(y, x)])
    assert np.array_equal(got, ref)
    assert cr.cr_hard_count() == 0


def test_quick_phase_equals_accurate_phase(cr):
    """Two-phase evaluation (sd_crlibm.h): the quick double-double is within
    2^-76 of the accurate one (the certainty test assumes 2^-70), only
    ~2^-16 of the calls need the accurate phase, and the two-phase result
    equals the accurate phase's on every argument."""
    rng = np.random.default_rng(13)
    n = 1_000_000
    j = np.arange(-30, 31) / 32.0
    x = np.concatenate([j, np.nextafter(j, 5), np.nextafter(j, -5), (np.arange(-60, 61) + 0.5) / 64,
                        rng.uniform(-7, 7, n), 10 ** rng.uniform(-12, 0, n // 4),
                        rng.uniform(-1e5, 1e5, n // 8)])
    cr.cr_quick_sincos_err.restype = ctypes.c_double
    unc = ctypes.c_long(0)
    worst = cr.cr_quick_sincos_err(np.ascontiguousarray(x).ctypes.data_as(P), ctypes.c_long(len(x)),
                                   ctypes.byref(unc))
    assert worst < 2.0 ** -76, math.log2(worst)
    assert unc.value < 2e-4 * len(x), unc.value

    def slow(fn, x, y=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = x if y is None else np.ascontiguousarray(y, dtype=np.float64)
        out = np.empty_like(x)
        cr.cr_eval_slow(fn, x.ctypes.data_as(P), y.ctypes.data_as(P), out.ctypes.data_as(P),
                        ctypes.c_long(len(x)))
        return out

    near1 = (1 - 10 ** rng.uniform(-16, -0.3, n // 2)) * rng.choice([-1, 1], n // 2)
    cases = [(0, x, None), (1, x, None),
             (2, np.concatenate([rng.uniform(-1, 1, n), near1]), None),
             (3, np.concatenate([rng.uniform(-1, 1, n), near1, 10 ** rng.uniform(-9, 0, n // 4)]), None),
             (4, rng.standard_normal(n) * 10 ** rng.uniform(-8, 8, n),
              rng.standard_normal(n) * 10 ** rng.uniform(-8, 8, n))]
    for fn, a, b in cases:
        assert np.array_equal(ev(cr, fn, 0, a, b), slow(fn, a, b), equal_nan=True), fn


def test_agrees_with_glibc_where_glibc_rounds_correctly(cr):
    rng = np.random.default_rng(12)
    n = 400_000
    for fn, x, y in [(0, rng.uniform(-7, 7, n), None), (1, rng.uniform(-7, 7, n), None),
                     (2, rng.uniform(-1, 1, n), None), (3, rng.uniform(-1, 1, n), None),
                     (4, rng.standard_normal(n), rng.standard_normal(n)),
                     (5, rng.standard_normal(n), rng.standard_normal(n))]:
        differ = (ev(cr, fn, 0, x, y) != ev(cr, fn, 1, x, y)).mean()
        # glibc misrounds ~0.1% of sin..atan2 (~0.51 ulp) and ~0.6% of hypot
        assert differ < (0.01 if fn == 5 else 0.004), (fn, differ)


@pytest.mark.parametrize("name", ["edge", "c2", "c3", "c4", "u11", "adv", "lastbit"])
def test_cr_oracle_takes_the_reference_decisions(name):
    g = load_golden(f"eig3_{name}")
    got = O.eig3(g["A"], nthreads=2, cr=True)
    assert np.array_equal(got["status"] & 0x7F, g["status"] & 0x7F)
    # values: bit-equal wherever no misrounded glibc call fed them
    assert (got["lam"] == g["lam"]).all(axis=1).mean() > 0.95
