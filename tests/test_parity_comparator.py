"""Negative and positive controls for the parity comparator (tests/parity.py).

The GPU parity suite is only as strict as `compare3`: these CPU tests feed
it the reference's own golden outputs, once untouched (nothing may be
flagged) and once with deliberate corruptions of the size the contract
forbids (angles moved by 1e-9, a selected sign flipped, eigenvalues scaled
by 1 + 1e-11, a branch code changed) — every corrupted row must come out
flagged AND unexplained, i.e. neither the 1-ulp libm perturbation tier nor
the valid-alternative tier may excuse it.
"""

from __future__ import annotations

import numpy as np

from conftest import load_golden
from parity import S2, compare3, edge_window


def _robust_generic_rows(g, k):
    st = g["status"]
    ok = ((st & 0x0F) == 0) & ((st & 0x80) == 0) & ~edge_window(g["ang"])
    rows = np.nonzero(ok)[0]
    assert len(rows) >= k
    return rows[np.linspace(0, len(rows) - 1, k).astype(int)]


def test_comparator_passes_the_reference_against_itself():
    g = load_golden("eig3_c2")
    got = {k: g[k].copy() for k in ("lam", "ang", "status")}
    s = compare3(g, got, A=g["A"], explain=True)
    assert s["flagged"] == 0 and s["unexplained"] == 0
    assert s["lam_bit_equal_frac"] == 1.0 and s["ang_bit_equal_frac"] == 1.0


def test_comparator_flags_every_corruption_as_unexplained():
    g = load_golden("eig3_c2")
    got = {k: g[k].copy() for k in ("lam", "ang", "status")}
    rows = _robust_generic_rows(g, 24)
    nudge, flip, scale, code = rows[:6], rows[6:12], rows[12:18], rows[18:]
    got["ang"][nudge, 0] += 1e-9                    # phi1 off by 10x the angle tolerance
    got["ang"][flip, 1] *= -1.0                     # phi2 sign flipped with its flag
    got["status"][flip] ^= S2
    got["lam"][scale] *= 1.0 + 1e-11                # eigenvalues off by 10x the tolerance
    got["status"][code] = (got["status"][code] & 0xF0) | 2   # branch -> DoubleRoot
    s = compare3(g, got, A=g["A"], explain=True)
    assert s["strict_ang_fail"] >= len(nudge)
    assert s["sign_mismatch"] == len(flip)
    assert s["lam_fail"] == len(scale)
    assert s["code_mismatch"] == len(code)
    assert s["flagged"] == len(rows), s
    assert s["unexplained"] == len(rows), s
    assert s["explained_by_ulp"] == 0 and s["valid_alternative"] == 0
