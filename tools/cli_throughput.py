#!/usr/bin/env python3
"""Records/s of the `solve` front end (GPU box): native codec vs the Python
codec, on N seeded 3x3 MatrixRecords read from and written to files in a
temporary directory (as `symdiag-b200 solve --input F --output G` does).

    python tools/cli_throughput.py [--n 1000000] [--python-n 100000]
"""
import argparse
import io
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1306_6291_b200 import cli  # noqa: E402


def corpus(n, seed=11):
    v = np.random.default_rng(seed).standard_normal((n, 6))
    return "".join('{"id": "r%d", "a11": %r, "a22": %r, "a33": %r, "a12": %r, "a13": %r, '
                   '"a23": %r}\n' % (k, *map(float, v[k])) for k in range(n))


def run(fn, text, reps):
    import tempfile
    best = 1e9
    with tempfile.TemporaryDirectory() as tmp:
        fin, fout = Path(tmp) / "in.jsonl", Path(tmp) / "out.jsonl"
        fin.write_text(text)
        for _ in range(reps):
            t0 = time.perf_counter()
            with open(fin) as fi, open(fout, "w") as fo:
                fn(fi, fo)
            best = min(best, time.perf_counter() - t0)
        out = fout.read_text()
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--python-n", type=int, default=100_000)
    a = ap.parse_args()
    text = corpus(a.n)
    cli.cmd_solve_native(io.StringIO(text[:10000]), io.StringIO())  # warm up (GPU, lib)
    t_nat, out_nat = run(cli.cmd_solve_native, text, 3)
    sub = "".join(text.splitlines(keepends=True)[:a.python_n])
    t_py, out_py = run(cli.cmd_solve, sub, 1)
    same = out_py == "".join(out_nat.splitlines(keepends=True)[:a.python_n])
    print(json.dumps({"records": a.n, "native_records_per_s": a.n / t_nat,
                      "native_s": t_nat, "python_records": a.python_n,
                      "python_records_per_s": a.python_n / t_py,
                      "outputs_identical_on_python_subset": same,
                      "threads": cli._threads(),
                      "bytes_in": len(text), "bytes_out": len(out_nat)}))


if __name__ == "__main__":
    main()
