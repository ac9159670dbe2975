"""Shared fixtures for the parity suite.

Markers: `gpu` — needs a B200 (run with `-m gpu`); everything else runs on
CPU.  Golden fixtures live in tests/golden/*.npz (made by the reference
itself, tests/golden/make_golden.py).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
for p in (str(ROOT), str(GOLDEN)):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long CPU-only check")


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden():
    return load_golden


def bits_equal(x, y):
    """Elementwise bit equality treating NaN == NaN (signed zeros differ)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return (x.view(np.uint64) == y.view(np.uint64)) | (np.isnan(x) & np.isnan(y))


def wrapped_diff(a, b):
    """|remainder(a - b, pi)| elementwise (core.py:49-51), NaN-propagating."""
    return np.abs(np.remainder(np.asarray(a) - np.asarray(b) + np.pi / 2, np.pi)
                  - np.pi / 2)
