"""Freeze golden fixtures from the UNMODIFIED reference implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `symdiag` in place from /root/reference/pkg/src (read-only,
PYTHONDONTWRITEBYTECODE), runs diagonalize3 / diagonalize2 and the stage
functions row by row over seeded inputs, and writes compressed .npz files
next to this script.  The GPU box never needs the reference: the tests read
only these files.

Sets (prefixes of the benchmark configs are exact, see workloads.py):
  eig3_edge  hand-built edge cases (cases.py)
  eig3_c2    first 2048 rows of config 2 (N(0,1), seed 1)
  eig3_c3    first 4096 rows of config 3 (degenerate stress, seed 2)
  eig3_c4    first 2048 rows of config 4 (SPD fp32, seed 3; upcast exactly)
  eig3_u11   2048 U[-1,1] rows, seed 101 (acceptance criterion 1 style)
  eig2_c1    2x2 edge cases + first 4096 rows of config 1 (seed 0)
  stages_*   char_coeffs / compute_pq / eigenvalues3 / pq_expanded /
             compute_v / compute_w on the edge + c3 sets
  signs_*    resolve_signs on the reference's own (lam, v, w) and
             degenerate_double on its _double_root_lambdas, edge / c2 / c3 /
             adversarial sets (`python make_golden.py signs` writes only these)
  eig3_lastbit  rows whose decisions hinge on glibc's last bits:
             cases.lastbit_3x3(4096) plus the rows the round-2 2^26 sweeps
             flagged (profiles/r2/parity_sweep/*_flagged.npz: seeded c2/c3/c4
             rows), `python make_golden.py lastbit` writes only this
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parents[1]))

import cases  # noqa: E402
import refrun  # noqa: E402
from paper_1306_6291_b200 import workloads  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz", {k: v.shape for k, v in arrays.items()})


def sets3_inputs():
    return {
        "edge": cases.edge_cases_3x3(),
        "c2": workloads.generate("c2", 2048),
        "c3": workloads.generate("c3", 4096),
        "c4": workloads.generate("c4", 2048),
        "u11": np.random.default_rng(101).uniform(-1.0, 1.0, (2048, 6)),
        "adv": cases.adversarial_3x3(4096),
    }


def sign_stages(sets3):
    for name in ("edge", "c2", "c3", "adv"):
        A = np.asarray(sets3[name], dtype=np.float64)
        s = refrun.run_stages(A)
        out = refrun.run_sign_stages(A, s["lam"], s["vw"])
        save(f"signs_{name}", A=A, lam=s["lam"], vw=s["vw"], **out)


def lastbit():
    rows = [cases.lastbit_3x3(4096)]
    for c in ("c2", "c3", "c4"):
        f = HERE.parents[1] / "profiles" / "r2" / "parity_sweep" / f"sweep_{c}_flagged.npz"
        rows.append(np.load(f)["A"])
    A = np.concatenate(rows).astype(np.float64)
    r = refrun.run_eig3(A)
    save("eig3_lastbit", A=A, lam=r["lam"], ang=r["ang"], status=r["status"],
         report=r["report"])


def main(only=None):
    if not refrun.available():
        raise SystemExit("reference not available at " + refrun.REF_SRC)
    if only == "lastbit":
        lastbit()
        return
    sets3 = sets3_inputs()
    if only == "signs":
        sign_stages(sets3)
        return
    for name, A in sets3.items():
        A32 = A if A.dtype == np.float32 else None
        A64 = np.asarray(A, dtype=np.float64)
        r = refrun.run_eig3(A64, with_d=(name == "edge"))
        extra = dict(A32=A32) if A32 is not None else {}
        if name == "edge":
            extra["d"] = r["d"]
        save(f"eig3_{name}", A=A64, lam=r["lam"], ang=r["ang"],
             status=r["status"], report=r["report"], **extra)
    A2 = np.concatenate([cases.edge_cases_2x2(), workloads.generate("c1", 4096)])
    r = refrun.run_eig2(A2, with_d=True)
    save("eig2_c1", A=A2, lam=r["lam"], phi=r["phi"], status=r["status"], d=r["d"])
    for name in ("edge", "c3"):
        A = sets3[name]
        s = refrun.run_stages(A)
        save(f"stages_{name}", A=A, **s)
    sign_stages(sets3)
    lastbit()
    # oracle.py referees: Jacobi, cubic roots, residuals
    ref3 = np.concatenate([cases.edge_cases_3x3(), workloads.generate("c2", 1024),
                           workloads.generate("c3", 1024)])
    save("referee3", A=ref3, **refrun.run_referees(ref3, 3))
    ref2 = np.concatenate([cases.edge_cases_2x2(), workloads.generate("c1", 1024)])
    save("referee2", A=ref2, **refrun.run_referees(ref2, 2))
    # JSON-lines front end: the reference's cmd_solve on a corpus built here
    # (edge rows it accepts + malformed lines), expected output kept verbatim
    import io
    symdiag, eig3, core = refrun._import()
    from symdiag import cli as RC
    lines = []
    r3 = refrun.run_eig3(sets3["edge"])
    for i, row in enumerate(sets3["edge"]):
        if (r3["status"][i] & 0x0F) < 8:
            a11, a12, a13, a22, a23, a33 = (float(x) for x in row)
            lines.append(json.dumps({"id": f"e3-{i}", "a11": a11, "a22": a22, "a33": a33,
                                     "a12": a12, "a13": a13, "a23": a23}))
    r2 = refrun.run_eig2(cases.edge_cases_2x2())
    for i, row in enumerate(cases.edge_cases_2x2()):
        if r2["status"][i] < 8:
            lines.append(json.dumps({"id": f"e2-{i}", "a11": float(row[0]),
                                     "a22": float(row[2]), "a12": float(row[1])}))
    lines[3:3] = ['{"a11": 1, "a22": 2}', "not json", '{"id": 5, "a11": 1, "a22": 2, "a12": 0}',
                  '{"a11": true, "a22": 2, "a12": 0}', "[1, 2, 3]", ""]
    text = "\n".join(lines) + "\n"
    out = io.StringIO()
    rc = RC.cmd_solve(io.StringIO(text), out)
    (HERE / "cli_solve_input.jsonl").write_text(text)
    (HERE / "cli_solve_expected.jsonl").write_text(out.getvalue())
    print("wrote cli_solve_{input,expected}.jsonl", len(lines), "lines, rc", rc)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
