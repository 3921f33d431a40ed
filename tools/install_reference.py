#!/usr/bin/env python
"""Install the UNMODIFIED reference (`spotsim`, pure Python) into baseline/_ref.

    python tools/install_reference.py

Runs the task's offline install recipe from a scratch copy (the reference
checkout is read-only):

    pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
        --target baseline/_ref <copy of /root/reference/pkg> --no-deps

and copies the reference's own test files to baseline/_ref/spotsim_tests, so
both travel to the GPU box with the repo snapshot (baseline/_ref is
git-ignored, not gpurun-ignored).  The GPU-side tests
(tests/test_reference_suite.py) and bench.py's reference arm import spotsim
from there; nothing on the box reads /root/reference.
"""

from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg")
DEST = ROOT / "baseline" / "_ref"


def main() -> int:
    if not (REF / "src" / "spotsim").exists():
        print(f"{REF} not present", file=sys.stderr)
        return 1
    with tempfile.TemporaryDirectory() as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(REF, src, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--find-links", "/opt/wheelhouse", "--target", str(DEST), "--upgrade", "--no-deps",
               str(src)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        print(res.stdout[-800:], res.stderr[-800:])
        if res.returncode:
            return res.returncode
    tests = DEST / "spotsim_tests"
    if tests.exists():
        shutil.rmtree(tests)
    shutil.copytree(REF / "tests", tests, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    print(f"installed spotsim into {DEST}; tests in {tests}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
