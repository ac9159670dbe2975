"""JSON-lines front end against the reference's own
cmd_solve output on a corpus built by tests/golden/make_golden.py."""

from __future__ import annotations

import io
import json
import math
from pathlib import Path

import numpy as np
import pytest

from paper_1306_6291_b200 import cli

GOLDEN = Path(__file__).resolve().parent / "golden"


def expected_lines():
    return (GOLDEN / "cli_solve_expected.jsonl").read_text().splitlines()


def test_parse_errors_match_reference_messages():
    """Every malformed line gets the reference's inline error text."""
    inp = (GOLDEN / "cli_solve_input.jsonl").read_text().splitlines()
    exp = [json.loads(x) for x in expected_lines()]
    errs = [e["error"] for e in exp if "error" in e]
    got = []
    for line in inp:
        if not line.strip():
            continue
        try:
            cli.parse_record(line)
        except cli.ParseError as e:
            got.append(str(e))
    assert got == errs


def test_dumps_formatting_matches_reference_style():
    obj = {"id": "x", "dim": 3, "v": [1.0, 0.1, -0.0, 1e-300, 2.5e16], "b": None, "t": True,
           "r": {"a": 1.0000000000000002}}
    s = cli.dumps(obj)
    assert s == ('{"id": "x", "dim": 3, "v": [1, 0.10000000000000001, -0, 1e-300, '
                 '25000000000000000], "b": null, "t": true, "r": {"a": 1.0000000000000002}}')
    refrun = pytest.importorskip("refrun")
    if refrun.available():
        refrun._import()
        from symdiag import cli as RC
        assert s == RC._dumps(obj)


def test_fast_result_formatter_equals_generic_dumps():
    rng = np.random.default_rng(5)
    for dim in (2, 3):
        for _ in range(200):
            lam = rng.standard_normal(dim) * 10.0 ** rng.integers(-300, 300)
            d = rng.standard_normal((dim, dim))
            res = np.abs(rng.standard_normal(dim + 2)) * 1e-16
            rec = cli.result_record(str(rng.integers(1e9)) if rng.random() < 0.8 else None, dim,
                                    rng.integers(0, 4), lam, rng.standard_normal(dim if dim == 3
                                                                                else 1), d, res)
            assert cli.dumps_result(rec) == cli.dumps(rec)


def test_random_stream_matches_reference_generator():
    rows = cli.random_symmetric_rows(50, 42)
    rng = np.random.default_rng(42)
    for r in rows:
        a11, a22, a33, a12, a13, a23 = rng.uniform(-1.0, 1.0, 6)
        assert list(r) == [a11, a12, a13, a22, a23, a33]


torch = pytest.importorskip("torch")
gpu = pytest.mark.gpu


def _solve(text, **kw):
    out = io.StringIO()
    rc = cli.cmd_solve(io.StringIO(text), out, **kw)
    return rc, out.getvalue().splitlines()


@gpu
def test_cli_solve_matches_reference_output():
    rc, got = _solve((GOLDEN / "cli_solve_input.jsonl").read_text())
    exp = expected_lines()
    assert rc == 0 and len(got) == len(exp)
    # rows the reference polished (Gauss-Newton, not bit-pinned): angle-exempt
    with np.load(GOLDEN / "eig3_edge.npz") as z:
        polished = {f"e3-{i}" for i in np.nonzero(z["status"] & 0x80)[0]}
    identical = 0
    for g_line, e_line in zip(got, exp):
        identical += g_line == e_line
        g, e = json.loads(g_line), json.loads(e_line)
        if "error" in e:
            assert g == e
            continue
        assert g["id"] == e["id"] and g["dim"] == e["dim"] and g["branch"] == e["branch"]
        sc = max(1.0, max(abs(x) for x in e["eigenvalues"]))
        assert max(abs(a - b) for a, b in zip(g["eigenvalues"], e["eigenvalues"])) <= 1e-12 * sc
        assert g["eigenvalues_sorted"] == sorted(g["eigenvalues"], reverse=True)
        assert g["euler_angles"] == g["angles"]
        assert set(g["residuals"]) == set(e["residuals"])
        if e["branch"] in ("Generic", "AlreadyDiagonal2D", None) and e["id"] not in polished:
            for a, b in zip(g["angles"], e["angles"]):
                d = abs(math.remainder(a - b, math.pi))
                edge = min(abs(b), abs(abs(b) - math.pi / 2)) < 1e-2
                assert d <= (1e-7 if edge else 1e-10), (g["id"], a, b)
            assert g["residuals"]["recon_rel"] <= max(4 * e["residuals"]["recon_rel"], 1e-12)
    # byte-identical wherever the GPU's libm agrees with glibc to the last bit
    # (all error lines, triple roots, diagonal cases; 104 of 340 on B200)
    assert identical >= 100, identical


@gpu
def test_cli_solver_exception_aborts_or_inlines():
    text = ('{"id": "ok", "a11": 1, "a22": 2, "a33": 3, "a12": 0.1, "a13": 0.2, "a23": 0.3}\n'
            '{"id": "big", "a11": 1e200, "a22": 2, "a33": 3, "a12": 0, "a13": 0, "a23": 0}\n')
    with pytest.raises(OverflowError):
        _solve(text)
    rc, lines = _solve(text, inline_errors=True)
    assert rc == 0 and json.loads(lines[1]) == {"id": "big",
                                                "error": json.loads(lines[1])["error"]}
    assert json.loads(lines[1])["error"].startswith("OverflowError")


@gpu
def test_cli_verify_and_corrupt_hook():
    from paper_1306_6291_b200 import workloads
    rows = workloads.generate("c2", 2000)
    good = "\n".join(json.dumps({"id": str(i), "a11": r[0], "a12": r[1], "a13": r[2],
                                 "a22": r[3], "a23": r[4], "a33": r[5]})
                     for i, r in enumerate(rows.tolist()))
    out = io.StringIO()
    assert cli.cmd_verify(io.StringIO(good), out, 1e-6) == 0
    s = json.loads(out.getvalue())
    assert s["fail"] == 0 and s["records"] == len(good.splitlines())
    out = io.StringIO()
    assert cli.cmd_verify(io.StringIO(good), out, 1e-6, corrupt=True) == 1
    assert json.loads(out.getvalue())["fail"] > 0


@gpu
def test_cli_bench_reports_ratio():
    out = io.StringIO()
    assert cli.cmd_bench(out, 100_000, 42) == 0
    r = json.loads(out.getvalue())
    assert r["n"] == 100_000 and r["throughput_ratio_closed_over_jacobi"] > 0


def _both(text, **kw):
    """(rc, output, exception type) of the Python front end and the native
    codec on the same input."""
    res = []
    for fn in (cli.cmd_solve, cli.cmd_solve_native):
        out = io.StringIO()
        try:
            rc, exc = fn(io.StringIO(text), out, **kw), None
        except Exception as e:  # noqa: BLE001 — compared below
            rc, exc = None, type(e)
        res.append((rc, out.getvalue(), exc))
    return res


def _mixed_corpus(n=3000, seed=5):
    rng = np.random.default_rng(seed)
    lines = []
    for k in range(n):
        r = rng.random()
        if r < 0.6:
            v = rng.standard_normal(6)
            lines.append(json.dumps({"id": f"m{k}", "a11": v[0], "a22": v[1], "a33": v[2],
                                     "a12": v[3], "a13": v[4], "a23": v[5]}))
        elif r < 0.8:
            v = rng.uniform(-1, 1, 3)
            lines.append(json.dumps({"a11": v[0], "a22": v[1], "a12": v[2]}))
        elif r < 0.85:
            lines.append(json.dumps({"id": "é\n", "a11": 1.0, "a22": 2.0, "a12": 0.5}))
        elif r < 0.9:
            lines.append(["{bad", "{}", '{"a11": NaN, "a22": 1, "a12": 0}', "", "  "][k % 5])
        else:  # rotated degenerate / diagonal / integer matrices
            lines.append('{"id": "d%d", "a11": 2, "a22": 2, "a33": 2, "a12": 0, "a13": 0, '
                         '"a23": 0}' % k)
    return "\n".join(lines) + "\n"


@gpu
def test_native_codec_solve_is_byte_identical():
    """cmd_solve_native (C++ codec) writes exactly what cmd_solve writes: the
    golden corpus, a mixed stream with parse errors, blank lines, escaped
    ids and 2x2/3x3 records, with and without --inline-errors."""
    for text in ((GOLDEN / "cli_solve_input.jsonl").read_text(), _mixed_corpus()):
        for kw in ({}, {"inline_errors": True}, {"batch": 257}):
            (rc_p, out_p, ex_p), (rc_n, out_n, ex_n) = _both(text, **kw)
            assert (rc_p, ex_p) == (rc_n, ex_n)
            assert out_p == out_n


@gpu
def test_native_codec_solver_exception_prefix():
    text = ('{"id": "ok", "a11": 1, "a22": 2, "a33": 3, "a12": 0.1, "a13": 0.2, "a23": 0.3}\n'
            '{"bad json\n'
            '{"id": "big", "a11": 1e200, "a22": 2, "a33": 3, "a12": 0, "a13": 0, "a23": 0}\n'
            '{"id": "after", "a11": 1, "a22": 2, "a12": 0.5}\n')
    (rc_p, out_p, ex_p), (rc_n, out_n, ex_n) = _both(text)
    assert ex_p is ex_n is OverflowError and out_p == out_n and len(out_n.splitlines()) == 2


@gpu
def test_native_verify_matches_python_verify():
    from paper_1306_6291_b200 import workloads
    rows = workloads.generate("c2", 3000)
    recs = [json.dumps({"id": f"v{k}", "a11": r[0], "a22": r[3], "a33": r[5], "a12": r[1],
                        "a13": r[2], "a23": r[4]}) for k, r in enumerate(rows)]
    recs += [json.dumps({"a11": 0.5, "a22": -1.0, "a12": 0.25})] * 5
    text = "\n".join(recs) + "\n"
    for corrupt in (False, True):
        outs = []
        for fn in (cli.cmd_verify, cli.cmd_verify_native):
            out = io.StringIO()
            rc = fn(io.StringIO(text), out, 1e-9, corrupt=corrupt)
            outs.append((rc, out.getvalue()))
        assert outs[0] == outs[1]
    bad = text + "{oops\n"
    for fn in (cli.cmd_verify, cli.cmd_verify_native):
        with pytest.raises(cli.ParseError):
            fn(io.StringIO(bad), io.StringIO(), 1e-9)


def test_whole_line_chunks_cut_only_at_newlines():
    """The chunk reader never splits a line, also with a tiny chunk size,
    and applies universal newlines to raw bytes."""
    text = "".join(f'{{"id": {k}, "a11": 1, "a22": 2, "a12": 0.{k}}}\n' for k in range(50))
    got = list(cli._whole_line_chunks(io.StringIO(text + "tail"), chunk=7))
    assert "".join(got) == text + "tail"
    assert all(c.endswith("\n") for c in got[:-1]) and got[-1].endswith("tail")
    raw = io.TextIOWrapper(io.BytesIO(text.replace("\n", "\r\n").encode()))
    assert "".join(cli._whole_line_chunks(raw, chunk=11)) == text


@gpu
@pytest.mark.parametrize("codec", [[], ["--python-codec"]])
def test_solve_streams_one_answer_per_line_over_a_pipe(codec):
    """A pipe client sends one record and waits: the answer must arrive while
    stdin is still open (the reference writes each result as its line
    arrives, cli.py:117-137)."""
    import os
    import select
    import subprocess
    import sys
    root = Path(__file__).resolve().parents[1]
    p = subprocess.Popen([sys.executable, "-m", "paper_1306_6291_b200.cli", "solve", *codec],
                         cwd=root, stdin=subprocess.PIPE, stdout=subprocess.PIPE,
                         stderr=subprocess.PIPE)
    try:
        for k in range(2):
            p.stdin.write(b'{"id": "r%d", "a11": 1, "a22": 2, "a33": 3, "a12": 0.5, '
                          b'"a13": 0.25, "a23": 0.125}\n' % k)
            p.stdin.flush()
            ready, _, _ = select.select([p.stdout], [], [], 180)
            assert ready, "no answer while stdin is open"
            rec = json.loads(p.stdout.readline())
            assert rec["id"] == f"r{k}" and rec["dim"] == 3, rec
        p.stdin.close()
        assert p.wait(timeout=60) == 0
        assert p.stdout.read() == b""
    finally:
        if p.poll() is None:
            os.kill(p.pid, 9)
