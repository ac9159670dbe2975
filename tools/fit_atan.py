#!/usr/bin/env python3
"""Minimax polynomial for the 2x2 fast path's arctangent (build-time tool).

    python tools/fit_atan.py [--deg 11]

atan(w) = w + w*s*P(s), s = w^2, on w in [0, tan(pi/8)] (the fast 2x2 path
reduces atan2 to that interval, see sd_eig2.cuh).  P is fitted by a Remez
exchange on the absolute error of P in 80-digit arithmetic (mpmath), its
coefficients rounded to double, and the rounded polynomial checked by
evaluating the device's exact Horner/FMA sequence in double (numpy) against
mpmath's atan on 2e6 points: prints the coefficients as C literals and the
max error in ulps of the result.
"""

from __future__ import annotations

import argparse

import mpmath as mp
import numpy as np

mp.mp.dps = 80
T = mp.tan(mp.pi / 8)
S_MAX = T * T


def f(s):
    s = mp.mpf(s)
    if s == 0:
        return mp.mpf(-1) / 3
    w = mp.sqrt(s)
    return (mp.atan(w) - w) / (w * s)


def remez(deg: int, iters: int = 30):
    n = deg + 2
    # Chebyshev extrema as the starting reference
    xs = [S_MAX * (1 - mp.cos(mp.pi * k / (n - 1))) / 2 for k in range(n)]
    coef = None
    for _ in range(iters):
        A = mp.matrix(n, n)
        b = mp.matrix(n, 1)
        for i, x in enumerate(xs):
            for j in range(deg + 1):
                A[i, j] = x ** j
            A[i, deg + 1] = (-1) ** i
            b[i] = f(x)
        sol = mp.lu_solve(A, b)
        coef = [sol[j] for j in range(deg + 1)]
        # locate the extrema of the error on a fine grid, then refine
        grid = [S_MAX * k / 4000 for k in range(4001)]
        err = [mp.polyval(coef[::-1], x) - f(x) for x in grid]
        ext = []
        for k in range(len(grid)):
            left = err[k - 1] if k > 0 else None
            right = err[k + 1] if k + 1 < len(grid) else None
            e = err[k]
            if (left is None or abs(e) >= abs(left)) and (right is None or abs(e) >= abs(right)):
                ext.append((grid[k], e))
        # keep alternating extrema, n of them with the largest magnitudes
        alt = []
        for x, e in ext:
            if alt and mp.sign(alt[-1][1]) == mp.sign(e):
                if abs(e) > abs(alt[-1][1]):
                    alt[-1] = (x, e)
            else:
                alt.append((x, e))
        while len(alt) > n:
            if abs(alt[0][1]) < abs(alt[-1][1]):
                alt.pop(0)
            else:
                alt.pop()
        if len(alt) < n:
            break
        xs = [x for x, _ in alt]
    return coef


def check(c, npts=2_000_000, seed=0):
    rng = np.random.default_rng(seed)
    w = np.concatenate([rng.uniform(0, float(T), npts),
                        np.linspace(0, float(T), 20001),
                        np.float64(float(T)) * (1 - rng.uniform(0, 1e-6, 1000))])
    s = w * w
    p = np.full_like(s, c[-1])
    for k in range(len(c) - 2, -1, -1):
        p = p * s + c[k]  # numpy: rounded multiply + add; device uses fma (better)
    ws = w * s
    r = ws * p + w
    worst = 0.0
    idx = np.argsort(-np.abs(r))[:0]
    sample = rng.choice(len(w), 20000, replace=False)
    for i in list(sample) + list(range(len(w) - 1000, len(w))) + list(idx):
        ref = mp.atan(mp.mpf(float(w[i])))
        if ref == 0:
            continue
        ulp = np.spacing(np.float64(float(ref)))
        worst = max(worst, float(abs(mp.mpf(float(r[i])) - ref)) / ulp)
    return worst


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--deg", type=int, default=11)
    a = ap.parse_args()
    coef = remez(a.deg)
    maxerr = max(abs(mp.polyval(coef[::-1], S_MAX * k / 20000) - f(S_MAX * k / 20000))
                 for k in range(20001))
    c = [float(x) for x in coef]
    print(f"// degree {a.deg} in s = w^2, minimax |P - f| = {mp.nstr(maxerr, 5)}")
    for k, x in enumerate(c):
        print(f"  {x!r},  // s^{k}")
    print(f"// max error of atan(w) (double Horner, no fma) = {check(c):.3f} ulp")


if __name__ == "__main__":
    main()
