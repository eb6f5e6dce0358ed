"""Build libbmv.so (sm_100a) in-tree with nvcc, and the host plan builder
libbmvplan.so (g++ -fopenmp, no CUDA).

`python -m paper_1907_01005_b200.build` or `__graft_entry__.build()`.
The shared library lands next to this file so it travels with the repo
snapshot to the GPU box (a JIT cache under ~/.cache would not).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libbmv.so"
PLAN_LIB = PKG / "libbmvplan.so"
PLAN_SOURCES = ["bmv_plan.cpp"]
SOURCES = ["bmv_util.cu", "bmv_misc.cu", "bmv_k1.cu", "bmv_spmm.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    home = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cand = Path(home) / "bin" / "nvcc"
    return str(cand) if cand.exists() else "nvcc"


def needs_rebuild() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "bmv.h"]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def _cxx() -> str:
    # /usr/bin/g++ ships libgomp; a wrapper earlier on PATH may not
    return "/usr/bin/g++" if Path("/usr/bin/g++").exists() else "g++"


def build_plan(force: bool = False) -> Path:
    """g++ -O3 -fopenmp -> libbmvplan.so (include/bmv_plan.h).  -ffp-contract=off keeps
    the hashed fill bit-identical to numpy."""
    deps = [CSRC / s for s in PLAN_SOURCES] + [ROOT / "include" / "bmv_plan.h"]
    if not force and PLAN_LIB.exists() and all(p.stat().st_mtime <= PLAN_LIB.stat().st_mtime
                                               for p in deps):
        return PLAN_LIB
    cmd = [_cxx(), "-O3", "-std=c++17", "-fopenmp", "-ffp-contract=off",
           "-shared", "-fPIC", "-I", str(ROOT / "include"),
           *[str(CSRC / s) for s in PLAN_SOURCES], "-o", str(PLAN_LIB) + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("g++ failed building libbmvplan.so")
    os.replace(str(PLAN_LIB) + ".tmp", PLAN_LIB)
    return PLAN_LIB


def build(force: bool = False, verbose: bool = False) -> Path:
    build_plan(force)
    if not force and not needs_rebuild():
        return LIB
    cmd = [
        nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "--shared", "-Xcompiler", "-fPIC",
        "-I", str(ROOT / "include"), "-I", str(CSRC),
        *[str(CSRC / s) for s in SOURCES], "-o", str(LIB) + ".tmp",
    ]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libbmv.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
