"""TEST INFRASTRUCTURE ONLY: build + ctypes loader for oracle/spotkm_oracle.c.

Compiled with gcc (-O2, no fast-math, -ffp-contract=off so the double
operation order of the reference is kept) into oracle/_build/liboracle.so.
Used by tests/ (parity checker) and bench.py (cpu_baseline); never by the
product package.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "spotkm_oracle.c"
OUT = HERE / "_build" / "liboracle.so"

_lib = None


def build(force: bool = False) -> Path:
    OUT.parent.mkdir(parents=True, exist_ok=True)
    if not force and OUT.exists() and OUT.stat().st_mtime >= SRC.stat().st_mtime:
        return OUT
    cmd = ["gcc", "-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC",
           "-shared", "-o", str(OUT), str(SRC), "-lm"]
    subprocess.run(cmd, check=True)
    return OUT


def load():
    global _lib
    if _lib is None:
        if not OUT.exists():
            build()
        lib = ctypes.CDLL(str(OUT))
        vp, i32 = ctypes.c_void_p, ctypes.c_int
        lib.oc_map_sweep.argtypes = [vp, i32, vp, vp, vp, vp, vp, i32]
        lib.oc_map_sweep.restype = i32
        lib.oc_hungarian.argtypes = [vp, i32, vp]
        lib.oc_hungarian.restype = i32
        _lib = lib
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def map_sweep(desc, plans, alive, tok, n_threads: int | None = None):
    """Solve every sweep plan on the CPU.  Returns (assign int32[sum R], totals[Q])."""
    lib = load()
    n_threads = n_threads or os.cpu_count() or 1
    rows = int(plans["rows"].sum())
    assign = np.full(max(rows, 1), -2, dtype=np.int32)
    totals = np.zeros(len(plans), dtype=np.float64)
    desc = np.ascontiguousarray(desc)
    plans = np.ascontiguousarray(plans)
    alive = np.ascontiguousarray(alive, dtype=np.uint32)
    tok = np.ascontiguousarray(tok, dtype=np.int64)
    lib.oc_map_sweep(_p(desc), len(desc), _p(plans), _p(alive), _p(tok), _p(assign), _p(totals),
                     n_threads)
    return assign[:rows], totals


def hungarian(w: np.ndarray) -> list[int]:
    w = np.ascontiguousarray(w, dtype=np.float64)
    n = w.shape[0]
    out = np.zeros(max(n, 1), dtype=np.int32)
    load().oc_hungarian(_p(w), n, _p(out))
    return out[:n].tolist()
