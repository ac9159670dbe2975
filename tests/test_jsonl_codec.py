"""The native JSON-lines codec (csrc/sd_jsonl.cpp) against the Python
front end it replaces (cli.parse_record / cli.dumps_result, which mirror the
reference's cli.py:33-114).  Host-only: runs without a GPU."""

from __future__ import annotations

import json
import math
import struct

import numpy as np
import pytest

from paper_1306_6291_b200 import cli


def _bits(x: float) -> bytes:
    return struct.pack("<d", x)


def _num(rng, style: int) -> str:
    """A JSON number in one of several spellings."""
    if style == 0:
        return repr(float(rng.standard_normal()))
    if style == 1:
        return str(int(rng.integers(-10**6, 10**6)))
    if style == 2:
        return f"{rng.standard_normal() * 10.0 ** rng.integers(-300, 300):.17e}"
    if style == 3:
        return format(float(rng.uniform(-1, 1)), ".3g").replace("e", "E")
    if style == 4:
        return "-0.0" if rng.random() < 0.5 else "0"
    if style == 5:
        return str(int(rng.integers(1, 9))) + "0" * int(rng.integers(15, 25))  # big ints
    return f"{rng.uniform(-1, 1):.25f}"  # more digits than a double holds


def _record(rng) -> str:
    dim = 3 if rng.random() < 0.7 else 2
    keys = ["a11", "a22", "a33", "a12", "a13", "a23"] if dim == 3 else ["a11", "a22", "a12"]
    items = [(k, _num(rng, int(rng.integers(0, 7)))) for k in keys]
    r = rng.random()
    if r < 0.5:
        items.append(("id", json.dumps(f"rec-{int(rng.integers(0, 10**9))}")))
    elif r < 0.6:
        items.append(("id", "null"))
    elif r < 0.7:
        items.append(("id", json.dumps("café \"quoted\"")))  # escaped: Python path
    rng.shuffle(items)
    sep = [", ", ",", " ,  ", ",\t"][int(rng.integers(0, 4))]
    colon = [": ", ":", " : "][int(rng.integers(0, 3))]
    body = sep.join(f'"{k}"{colon}{v}' for k, v in items)
    pad = [" ", "", "\t", "  "][int(rng.integers(0, 4))]
    return pad + "{" + body + "}" + pad


BAD_LINES = [
    "{", "[]", "{}", '{"a11": 1}', '{"a11": 1, "a22": 2, "a12": true}',
    '{"a11": 1, "a22": 2, "a12": null}', '{"a11": 1, "a22": 2, "a12": "3"}',
    '{"a11": NaN, "a22": 2, "a12": 3}', '{"a11": 1e999, "a22": 2, "a12": 3}',
    '{"a11": -Infinity, "a22": 2, "a12": 3}', '{"a11": 01, "a22": 2, "a12": 3}',
    '{"a11": 1, "a22": 2, "a12": 3, "a12": 4}', '{"a11": 1, "a22": 2, "a12": 3, "x": 4}',
    '{"a11": 1, "a22": 2, "a12": 3, "id": 7}', '{"a11": 1, "a22": 2, "a12": 3} x',
    '{"a11": 1., "a22": 2, "a12": 3}', '{"a11": .5, "a22": 2, "a12": 3}',
    '{"a11": +1, "a22": 2, "a12": 3}', '{"a11": 1e-400, "a22": 2, "a12": 3}',
    '{"a\\u0031\\u0031": 1, "a22": 2, "a12": 3}', "not json at all",
]


def _python_parse(line: str):
    try:
        return cli.parse_record(line.strip())
    except cli.ParseError:
        return "error"
    except (OverflowError, ValueError):
        return "error"


def test_native_parse_matches_python_parser():
    rng = np.random.default_rng(2024)
    lines = [_record(rng) for _ in range(20000)] + BAD_LINES + ["", "   ", "\t"]
    rng.shuffle(lines)
    buf = ("\n".join(lines) + "\n").encode()
    kind, rows, span, consumed = cli.native_parse(buf, nthreads=4)
    assert consumed == len(buf)
    nonblank = [ln for ln in lines if ln.strip()]
    assert len(kind) == len(nonblank)
    native = 0
    for k, line in enumerate(nonblank):
        assert buf[span[k, 0]:span[k, 1]].decode() == line.strip()
        ref = _python_parse(line)
        if kind[k] == 0:
            continue  # the Python parser decides (error message or escaped id)
        native += 1
        assert ref != "error", line
        rec_id, dim, row = ref
        assert dim == kind[k]
        assert all(_bits(a) == _bits(b) for a, b in zip(row, rows[k, :len(row)])), line
        tok = None if span[k, 2] < 0 else json.loads(buf[span[k, 2]:span[k, 3]])
        assert tok == rec_id
    assert native > 15000  # the common spellings take the native path
    # every malformed line is left to Python (which raises the reference's message)
    for line in BAD_LINES:
        k = nonblank.index(line)
        assert kind[k] == 0


def test_native_format_matches_python_formatter():
    rng = np.random.default_rng(7)
    n = 9001  # > the codec's 4096-record threading threshold: exercises the compaction
    dims = rng.choice([2, 3], n).astype(np.int8)
    scale = 10.0 ** rng.integers(-320, 300, (n, 1))
    lam = rng.standard_normal((n, 3)) * scale
    lam[::7, 1] = lam[::7, 0]          # ties: stable reverse sort
    lam[::11, 2] = -0.0
    ang = rng.uniform(-math.pi / 2, math.pi / 2, (n, 3))
    d = rng.standard_normal((n, 9))
    res = np.abs(rng.standard_normal((n, 5))) * 1e-16
    res[::5, 3] = res[::5, 2]           # equal maxima: first one
    st = rng.integers(0, 4, n).astype(np.uint8) | (rng.integers(0, 16, n).astype(np.uint8) << 4)
    ids = [f"r{k}" if k % 3 else None for k in range(n)]
    idbuf = "".join(json.dumps(i) if i else "" for i in ids).encode()
    spans, pos = np.full((n, 2), -1, np.int64), 0
    for k, i in enumerate(ids):
        if i:
            t = len(json.dumps(i))
            spans[k] = (pos, pos + t)
            pos += t
    dims[::13] = 0                     # skipped records
    out, offsets = cli.native_format(dims, idbuf, spans, lam, ang, d, res, st, nthreads=3)
    out = bytes(out)
    for k in range(n):
        got = out[offsets[k]:offsets[k + 1]].decode()
        if dims[k] == 0:
            assert got == ""
            continue
        dim = int(dims[k])
        rec = cli.result_record(ids[k], dim, st[k], lam[k, :dim], ang[k, :3 if dim == 3 else 1],
                                d[k, :dim * dim].reshape(dim, dim), res[k, :dim + 2])
        assert got == cli.dumps_result(rec) + "\n", k


@pytest.mark.parametrize("x", [0.1, 1e-5, 1e-4, 1e16, 1e17, 123456789012345678.0, 5e-324,
                               1.7976931348623157e308, -0.0, 0.0, 2.0 ** -1074, 1 / 3])
def test_float_spelling(x):
    dims = np.array([2], np.int8)
    lam = np.array([[x, x, 0.0]])
    out, _ = cli.native_format(dims, b"", np.full((1, 2), -1, np.int64), lam, np.zeros((1, 3)),
                               np.zeros((1, 9)), np.zeros((1, 5)), np.zeros(1, np.uint8))
    assert bytes(out).decode().startswith('{"id": null, "dim": 2, "eigenvalues": [' +
                                         format(x, ".17g") + ", " + format(x, ".17g") + "]")
