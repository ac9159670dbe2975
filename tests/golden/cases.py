"""Hand-built edge-case inputs (packed layouts), mirroring what the
reference's own tests exercise:

- the 12-record golden corpus (tests/data/golden_input.jsonl, 9 3x3 + 3 2x2);
- scalar matrices (test_acceptance.py:118-121), diag(3,2,1) and its
  permutations (test_eig3_angles.py:29, 183-200);
- separated double roots and near-boundary gaps 1e-3/1e-6/1e-9 built from QR
  factors (test_acceptance.py:105-132, test_eig3_angles.py:165-218);
- conjugation round trips with solver-order eigenvalues (conftest.py:42-50);
- zero f-vector patterns, signed zeros, tiny / subnormal / huge magnitudes
  (overflow in `**`), NaN / inf entries.
All generated deterministically from fixed seeds; no reference code needed.
"""

from __future__ import annotations

import math

import numpy as np

_UP = ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))


def _pack(m):
    m = np.asarray(m, dtype=float)
    s = 0.5 * (m + m.T)
    return [m[0, 0], s[0, 1], s[0, 2], m[1, 1], s[1, 2], m[2, 2]]


def _rot(p1, p2, p3):
    c1, s1 = math.cos(p1), math.sin(p1)
    c2, s2 = math.cos(p2), math.sin(p2)
    c3, s3 = math.cos(p3), math.sin(p3)
    rx = np.array([[1, 0, 0], [0, c1, -s1], [0, s1, c1]])
    ry = np.array([[c2, 0, s2], [0, 1, 0], [-s2, 0, c2]])
    rz = np.array([[c3, -s3, 0], [s3, c3, 0], [0, 0, 1]])
    return rx @ ry @ rz


def _conj(phis, lams):
    d = _rot(*phis)
    return _pack((d * np.asarray(lams, dtype=float)) @ d.T)


def edge_cases_3x3() -> np.ndarray:
    rows = []
    # golden corpus 3x3 records, packed (a11,a12,a13,a22,a23,a33)
    rows += [
        [1, 0, 0, 1, 0, 1],
        [2.5, 0, 0, 2.5, 0, 2.5],
        [3, 0, 0, 2, 0, 1],
        [0, 1, 1, 0, 1, 0],
        [1.6811788772383369, 0, -0.4660195429836132, 2, 0, 1.3188211227616633],
        [5, 0, 0, 1, -2.1285471334023225e-17, 1],
        [1.8250200448230833, 0.78821148340683078, 0.34388344776385738,
         2.4664238340913922, -0.3064514246013107, 1.7085561210855242],
        [0.25, 0.125, -0.375, -0.5, 0.625, 0.75],
        [3, 1e-08, 0, 2, -1e-08, 1],
    ]
    for c in (-7.0, -1.0, 0.0, 0.25, 1.0, 3.5):
        rows.append([c, 0, 0, c, 0, c])
    for d in ((3, 2, 1), (1, 2, 3), (2, 3, 1), (2, 1, 3), (3, 1, 2), (1, 3, 2),
              (2, 2, 1), (1, 2, 2), (2, 1, 2), (5, 1, 1), (1, 1, 5), (-1, 0, 1)):
        rows.append([d[0], 0, 0, d[1], 0, d[2]])
    # one nonzero off-diagonal entry (f1 = 0 or f2 = 0 patterns)
    rows += [[1, 0.5, 0, 2, 0, 3], [1, 0, 0.5, 2, 0, 3], [1, 0, 0, 2, 0.5, 3],
             [2, 0, 0, 2, 0.5, 2], [1, 0.3, 0, 1, 0, 4], [0, 0, 1, 0, 0, 0],
             [1, 0, 0, 1, 0, 2], [1, 0, 0, 3, 0, 3], [0, 1, 0, 0, 0, 0],
             [1, 0, 0, 2, 0, 2], [2, 0, 0, 1, 1e-20, 1]]
    # signed zeros
    rows += [[-0.0, -0.0, -0.0, -0.0, -0.0, -0.0], [1, -0.0, 0.0, 2, -0.0, 3],
             [0.0, 1.0, -0.0, 0.0, -0.0, 0.0]]
    # conjugated round trips at the constructing (largest, smallest, middle)
    rng = np.random.default_rng(7001)
    for _ in range(60):
        phis = rng.uniform(-math.pi / 2 + 0.05, math.pi / 2 - 0.05, 3)
        lams = np.sort(rng.uniform(-4.0, 4.0, 3))
        rows.append(_conj(phis, (lams[2], lams[0], lams[1])))
    # angles at / near 0, pi/4, pi/2 (refinement windows)
    for p in (0.0, 1e-9, 1e-5, 0.1, math.pi / 8, math.pi / 4, 3 * math.pi / 8,
              math.pi / 2 - 1e-5, math.pi / 2):
        rows.append(_conj((0.3, p, 0.7), (3.0, 1.0, 2.0)))
        rows.append(_conj((0.3, 0.7, p), (3.0, 1.0, 2.0)))
        rows.append(_conj((p, 0.4, 0.9), (3.0, 1.0, 2.0)))
    # separated double roots (test_acceptance.py:105-117 construction)
    rng = np.random.default_rng(7002)
    for _ in range(40):
        lam = rng.uniform(-3.0, 3.0)
        lam3 = lam + math.copysign(rng.uniform(0.5, 3.0), rng.uniform(-1, 1))
        q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        rows.append(_pack((q * np.array([lam, lam, lam3])) @ q.T))
    # near-boundary gaps (test_acceptance.py:124-131)
    for gap in (1e-3, 1e-6, 1e-9, 1e-12):
        for _ in range(15):
            lam = rng.uniform(-3.0, 3.0)
            q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
            rows.append(_pack((q * np.array([lam, lam + gap, lam + 2.0])) @ q.T))
    # conjugated double roots about single axes (test_eig3_angles.py:150-170)
    rows.append(_conj((0.0, 0.6, 0.0), (2.0, 2.0, 1.0)))
    rows.append(_conj((0.4, 0.0, 0.0), (5.0, 1.0, 1.0)))
    # magnitudes: tiny, subnormal, large, overflowing `**`
    base = np.array([0.25, 0.125, -0.375, -0.5, 0.625, 0.75])
    for s in (1e-300, 1e-200, 1e-160, 1e-100, 1e-20, 1e20, 1e40, 1e50, 1e52,
              1e60, 1e100, 1e155, 1e200):
        rows.append(list(base * s))
    rows.append([5e-324, 0, 0, 1e-323, 0, 0])
    # non-finite inputs
    rows += [[math.nan, 0, 0, 1, 0, 1], [1, math.inf, 0, 1, 0, 1],
             [1, 0, 0, 1, 0, -math.inf]]
    return np.array(rows, dtype=np.float64)


def adversarial_3x3(n: int, seed: int = 7100) -> np.ndarray:
    """Seeded stress rows for the fast path's guards: every row family below
    sits on or near a decision boundary of the reference algorithm.
      - random rotations of diag(l) with two / three eigenvalues equal up to
        relative gaps 0, 1e-15 .. 1e-3 (double/triple-root thresholds,
        DegenerateEigenvalues, the q-sign noise)
      - angles at and near 0, pi/8, pi/4, 3pi/8, pi/2 (refinement windows,
        edge window, the wrap at +-pi/2)
      - magnitudes 2^-200 .. 2^200 (fast-path guard at 2^160, tolerances
        that scale with max(1, |A|))
      - integer-valued and exactly diagonal / block-diagonal matrices (zero
        f-vectors, AlreadyDiagonal2D, exact ties)
    """
    rng = np.random.default_rng(seed)
    rows = np.empty((n, 6))
    fam = rng.integers(0, 5, n)
    for i in range(n):
        f = fam[i]
        if f == 0:  # near-repeated eigenvalues under a random rotation
            base = rng.uniform(-5, 5)
            gap = rng.choice([0.0, 1e-15, 1e-13, 1e-11, 1e-9, 1e-6, 1e-3])
            k = rng.integers(0, 2)
            lam = [base, base + gap, base + rng.uniform(0.5, 3) * (1 if k else gap * 1e3)]
            q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
            rows[i] = _pack((q * np.asarray(lam)) @ q.T)
        elif f == 1:  # angles at the refinement / wrap boundaries
            special = [0.0, 1e-12, 1e-8, math.pi / 8, math.pi / 4, 3 * math.pi / 8,
                       math.pi / 2 - 1e-8, math.pi / 2]
            phis = [rng.choice(special) * rng.choice([-1, 1]) + rng.normal(0, 1e-10) * rng.integers(0, 2)
                    for _ in range(3)]
            lam = np.sort(rng.uniform(-4, 4, 3))
            rows[i] = _conj(phis, (lam[2], lam[0], lam[1]))
        elif f == 2:  # magnitudes across the fast-path guard
            rows[i] = rng.standard_normal(6) * 2.0 ** rng.integers(-200, 200)
        elif f == 3:  # integer matrices (exact ties, zero f-vectors)
            rows[i] = rng.integers(-3, 4, 6).astype(float)
        else:  # diagonal / block-diagonal with repeated entries
            d = rng.integers(-2, 3, 3).astype(float)
            r = np.zeros(6)
            r[[0, 3, 5]] = d
            if rng.random() < 0.5:
                r[rng.choice([1, 2, 4])] = rng.choice([1e-300, 1e-16, 0.5])
            rows[i] = r
    return rows


def edge_cases_2x2() -> np.ndarray:
    rows = [[1, 0, 1], [2, 1, 2], [1, 2, 0], [3, 0, 1], [1, 0, 3], [0, 0, 0],
            [-0.0, -0.0, -0.0], [0, 1, 0], [0, -1, 0], [1, 1e-15, 1],
            [1, 1e-13, 1], [1 + 1e-15, 0, 1], [2, -1, 2], [-1, 0, 1],
            [1e-300, 1e-300, 0], [1e200, 1e200, -1e200], [1e160, 1, 0],
            [5e-324, 5e-324, 0], [math.nan, 0, 1], [1, math.inf, 1]]
    rng = np.random.default_rng(7003)
    for _ in range(40):
        a11, a12, a22 = rng.uniform(-1, 1, 3)
        rows.append([a11, a12, a22])
        rows.append([a22, a12, a11])       # swap symmetry pair
    return np.array(rows, dtype=np.float64)


def lastbit_3x3(n: int, seed: int = 7300) -> np.ndarray:
    """Seeded rows whose reference decisions hinge on the last bits of
    glibc's acos / cos / sin (round-2 sweeps: the two c3 DoubleRoot-vs-
    Generic rows and the c4 phi3 sign row were all of these kinds):
      - diagonal matrices with two entries at relative gaps 1e-4 .. 1e-1
        (v is rounding noise of the eigenvalues: the V_ZERO_EPS test and
        the w clamp decide DoubleRoot vs Generic, eig3.py:183-206, 547)
      - the same with one tiny off-diagonal a23 (f1 = 0 route)
      - random rotations with |phi3| or |phi2| at 1e-9 .. 1e-6 of 0 or
        pi/2 (w, v within an ulp of 0 / 1: the sign selection of
        eig3.py:302-326 on noise-sized magnitudes)
      - random rotations of eigenvalues with relative gaps 1e-8 .. 1e-5
        (conditioning: angles carry the eigenvalues' last-bit noise)
    """
    rng = np.random.default_rng(seed)
    rows = np.empty((n, 6))
    fam = rng.integers(0, 4, n)
    for i in range(n):
        f = fam[i]
        if f in (0, 1):
            x = rng.uniform(-5, 5)
            d = [x, x * (1 + 10 ** rng.uniform(-4, -1) * rng.choice([-1, 1])), rng.uniform(-5, 5)]
            rng.shuffle(d)
            r = np.zeros(6)
            r[[0, 3, 5]] = d
            if f == 1:
                r[4] = 10 ** rng.uniform(-12, -6) * rng.choice([-1, 1])
            rows[i] = r
        elif f == 2:
            phis = list(rng.uniform(-math.pi / 2, math.pi / 2, 3))
            k = rng.integers(1, 3)
            t = 10 ** rng.uniform(-9, -6)
            phis[k] = (t if rng.random() < 0.5 else math.pi / 2 - t) * rng.choice([-1, 1])
            rows[i] = _conj(phis, rng.uniform(-4, 4, 3))
        else:
            base = rng.uniform(-5, 5)
            lam = [base, base * (1 + 10 ** rng.uniform(-8, -5)), rng.uniform(-5, 5)]
            q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
            rows[i] = _pack((q * np.asarray(lam)) @ q.T)
    return rows
