"""The reference's `**` is CPython float_pow -> libm pow (glibc 2.39 here).
The device restates that pow bit for bit (csrc/sd_glibc_pow.h).  These CPU
tests pin the restatement:

* its lookup tables, regenerated from their published construction by
  tools/gen_glibc_tables.py, equal the committed header and the bytes of the
  installed libm.so.6 (when it is the Ubuntu GLIBC 2.39 build the golden
  fixtures came from);
* the same C++ source compiled for the host (oracle/glibc_check/pow_check.cpp)
  returns libm's pow bit for bit on edge cases and millions of random
  bases for the exponents the reference uses;
* CPython's own `x ** k` agrees with libm pow (so the oracle's pow and the
  reference's `**` are the same function).
The GPU leg (test_gpu_parity.py::test_device_glibc_pow_bit_exact) runs the
device build of the same source against host libm values.
"""

from __future__ import annotations

import ctypes
import math
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))


def _gen():
    import gen_glibc_tables
    return gen_glibc_tables


def test_generated_tables_match_committed_header():
    pytest.importorskip("mpmath")
    g = _gen()
    assert g.render() == g.OUT.read_text()


def test_tables_and_constants_match_installed_libm():
    pytest.importorskip("mpmath")
    g = _gen()
    lib = g.libm_tables()
    if lib is None:
        pytest.skip("libm.so.6 is not the Ubuntu GLIBC 2.39-0ubuntu8.5 build")
    rows, words, consts = lib
    assert rows == g.pow_log_table()
    assert words == g.exp_table()
    # the published constants restated in sd_glibc_pow.h
    head = consts["pow_log_head"]
    assert head[0] == float.fromhex("0x1.62e42fefa3800p-1")
    assert head[1] == float.fromhex("0x1.ef35793c76730p-45")
    assert head[2:] == (-0.5, float.fromhex("0x1.555555555556p-2") * -2,
                        float.fromhex("-0x1.0000000000006p-2") * -2,
                        float.fromhex("0x1.999999959554ep-3") * 4,
                        float.fromhex("-0x1.555555529a47ap-3") * 4,
                        float.fromhex("0x1.2495b9b4845e9p-3") * -8,
                        float.fromhex("-0x1.0002b8b263fc3p-3") * -8)
    e = consts["exp_head"]
    assert e == (float.fromhex("0x1.71547652b82fep0") * 128, float.fromhex("0x1.8p52"),
                 float.fromhex("-0x1.62e42fefa0000p-8"), float.fromhex("-0x1.cf79abc9e3b3ap-47"),
                 float.fromhex("0x1.ffffffffffdbdp-2"), float.fromhex("0x1.555555555543cp-3"),
                 float.fromhex("0x1.55555cf172b91p-5"), float.fromhex("0x1.1111167a4d017p-7"))


@pytest.fixture(scope="module")
def pow_check(tmp_path_factory):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not available")
    exe = tmp_path_factory.mktemp("powcheck") / "pow_check"
    src = ROOT / "oracle" / "glibc_check" / "pow_check.cpp"
    subprocess.run([gxx, "-O2", "-ffp-contract=off", "-std=c++17", "-o", str(exe), str(src),
                    "-lm"], check=True, capture_output=True)
    return exe


@pytest.mark.parametrize("seed", [1, 2])
def test_host_build_of_device_pow_is_libm_bit_for_bit(pow_check, seed):
    r = subprocess.run([str(pow_check), "3000000", str(seed)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "mismatches 0" in r.stdout


def test_python_pow_is_libm_pow():
    """CPython float ** float calls libm pow (float_pow), so the oracle's
    pow() and the reference's ** are the same function."""
    libm = ctypes.CDLL("libm.so.6")
    libm.pow.restype = ctypes.c_double
    libm.pow.argtypes = [ctypes.c_double, ctypes.c_double]
    rng = np.random.default_rng(3)
    xs = np.concatenate([rng.standard_normal(20000) * 10.0 ** rng.integers(-30, 30, 20000),
                         rng.uniform(-10, 10, 20000)])
    diff = 0
    for x in xs.tolist():
        for k in (2.0, 3.0, 6.0):
            if x ** k != libm.pow(x, k):
                diff += 1
    assert diff == 0
    # and glibc's pow is not the correctly rounded power: x*x differs
    assert any(x * x != libm.pow(x, 2.0) for x in xs.tolist())
    assert math.isinf(libm.pow(1e200, 2.0))
