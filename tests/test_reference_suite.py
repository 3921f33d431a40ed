"""Run the REFERENCE's own test files with this implementation installed in
place of the reference's planner and estimator (CPU; needs the read-only
reference checkout, present only in the build container -- skipped
elsewhere).  The mapper parts of those files keep the reference mapper
because they need no GPU here; the device mapper is covered bit-for-bit by
the golden tests."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg")
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not (REF / "src" / "spotsim").exists(), reason="reference not present")
@pytest.mark.parametrize("target", [
    "tests/test_migration.py",
    "tests/test_costmodel.py::TestMigrationCost",
    "tests/test_acceptance.py::test_criterion_03_migration_plan_soundness",
    "tests/test_acceptance.py::test_criterion_06_case_study",
    "tests/test_simulator.py",
])
def test_reference_tests_pass_with_dropin(target, tmp_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF / "src"), str(ROOT), str(ROOT / "tests" / "plugins"),
                                         str(REF / "tests")])
    env["SPOTKM_INSTALL_PARTS"] = "planner,estimator"
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                          "-p", "spotsim_dropin", "--rootdir", str(tmp_path), str(REF / target)],
                         cwd=tmp_path, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
    assert " passed" in res.stdout
