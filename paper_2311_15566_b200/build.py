"""In-tree build of libspotkm.so for sm_100a (run: python -m paper_2311_15566_b200.build).

Compiled with nvcc directly (no JIT cache), so the .so travels with the repo
snapshot to the GPU box.  -fmad=false and no fast-math: the matcher must
replay the reference's IEEE double arithmetic exactly.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import sysconfig
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SRC = [PKG / "csrc" / "spotkm.cu", PKG / "csrc" / "planner.cpp", PKG / "csrc" / "reshard.cu",
       PKG / "csrc" / "estimator.cu"]
OUT = PKG / "_lib" / "libspotkm.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared",
    f"-I{ROOT / 'include'}",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


HOSTPACK_SRC = PKG / "csrc" / "hostpack.cpp"
HOSTPACK_OUT = PKG / f"_hostpack{sysconfig.get_config_var('EXT_SUFFIX')}"


def build_hostpack(force: bool = False) -> Path:
    """The CPython extension that flattens the caller's inventories (g++)."""
    if not force and HOSTPACK_OUT.exists() and HOSTPACK_OUT.stat().st_mtime >= HOSTPACK_SRC.stat().st_mtime:
        return HOSTPACK_OUT
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", f"-I{sysconfig.get_paths()['include']}",
           "-o", str(HOSTPACK_OUT), str(HOSTPACK_SRC)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"g++ failed ({res.returncode}):\n{res.stderr}")
    return HOSTPACK_OUT


def build(force: bool = False, verbose: bool = False) -> Path:
    build_hostpack(force)
    OUT.parent.mkdir(parents=True, exist_ok=True)
    newest = max(p.stat().st_mtime for p in SRC + [ROOT / "include" / "spotkm.h", PKG / "csrc" / "exact.cuh"])
    if not force and OUT.exists() and OUT.stat().st_mtime >= newest:
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), "-o", str(OUT),
           *map(str, SRC)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr}")
    if verbose:
        print(res.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
