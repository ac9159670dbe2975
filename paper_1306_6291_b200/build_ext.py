"""Build the in-tree CUDA library paper_1306_6291_b200/lib/libsymdiag_b200.so.

Plain nvcc, sm_100a only, no torch in the ABI:
    python -m paper_1306_6291_b200.build_ext
The .so is git-ignored but travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import re
import shlex
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libsymdiag_b200.so"
SOURCES = ["symdiag_b200.cu", "sd_host.cu", "sd_jsonl.cpp"]
# PTX pass between cicc and ptxas (ptx_constpool.py); SD_PTX_POOL=0 disables
PTX_POOL = os.environ.get("SD_PTX_POOL", "1") != "0"
HEADERS = ["sd_math.cuh", "sd_eig3.cuh", "sd_eig2.cuh", "sd_fast3.cuh", "sd_jacobi.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo",
    "-fmad=false",            # CPython never contracts a*b+c
    "-std=c++17",
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-fvisibility=default",
    "--shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def run_nvcc(cmd: list[str], ptx_pass: bool = PTX_POOL) -> subprocess.CompletedProcess:
    """Run an nvcc command; with `ptx_pass`, replay nvcc's own compilation
    trajectory (`-dryrun -keep`) and rewrite every .ptx with ptx_constpool
    just before ptxas assembles it."""
    if not ptx_pass:
        return subprocess.run(cmd, capture_output=True, text=True)
    from paper_1306_6291_b200 import ptx_constpool
    keep = Path(tempfile.mkdtemp(prefix="sd_nvcc_"))
    dry = subprocess.run([cmd[0], "-dryrun", "-keep", "-keep-dir", str(keep), *cmd[1:]],
                         capture_output=True, text=True)
    if dry.returncode != 0:
        return dry
    env = dict(os.environ)
    log = []
    try:
        for line in dry.stderr.splitlines():
            if not line.startswith("#$ "):
                continue
            c = line[3:].strip()
            m = re.match(r"^([A-Za-z_][A-Za-z0-9_]*)=(.*)$", c)
            if m:  # environment assignment of the trajectory
                val = re.sub(r"\$(\w+)", lambda v: env.get(v.group(1), ""), m.group(2).strip())
                env[m.group(1)] = " ".join(shlex.split(val)) if val else ""
                continue
            if c.startswith("ptxas "):
                for tok in shlex.split(c):
                    if tok.endswith(".ptx"):
                        text, n = ptx_constpool.rewrite(Path(tok).read_text())
                        Path(tok).write_text(text)
                        log.append(f"ptx_constpool: {tok}: {n} pooled f64 constants\n")
            r = subprocess.run(["bash", "-c", c], env=env, capture_output=True, text=True)
            log.append(r.stdout + r.stderr)
            if r.returncode != 0 and not c.startswith("rm "):
                return subprocess.CompletedProcess(cmd, r.returncode, "".join(log), "")
        return subprocess.CompletedProcess(cmd, 0, "".join(log), "")
    finally:
        shutil.rmtree(keep, ignore_errors=True)


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "symdiag_b200.h",
                                                     PKG / "ptx_constpool.py"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(tmp), *[str(CSRC / s) for s in SOURCES]]
    res = run_nvcc(cmd)
    log = res.stdout + res.stderr
    (LIB_DIR / "build.log").write_text(" ".join(cmd) + "\n" + log)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + log[-4000:])
    os.replace(tmp, LIB)
    if verbose:
        print(log)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
