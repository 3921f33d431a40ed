"""Run the REFERENCE's own test files with this implementation installed in
place of the reference's hot path (`install.install(spotsim)`).

The reference (`spotsim`, unmodified) and its test files come from
baseline/_ref (tools/install_reference.py; it travels to the GPU box with the
snapshot), else from the read-only checkout in the build container.

* CPU (no GPU): the native planner and estimator replace the reference's.
* GPU: everything, INCLUDING the device mapper (build_graph / km_match /
  map_devices on the sm_100a kernels): the reference's test_mapping.py,
  acceptance criteria 01 (KM optimality), 02 (two-step reduction), 03 (plan
  soundness), 06 (case study), the migration / cost-model / simulator suites.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _locate():
    local = ROOT / "baseline" / "_ref"
    if (local / "spotsim").exists() and (local / "spotsim_tests").exists():
        return local, local / "spotsim_tests"
    ref = Path("/root/reference/pkg")
    if (ref / "src" / "spotsim").exists():
        return ref / "src", ref / "tests"
    return None, None


SRC, TESTS = _locate()
needs_ref = pytest.mark.skipif(SRC is None, reason="reference (baseline/_ref) not present")


def _run(target, parts, tmp_path, timeout=1200):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(SRC), str(ROOT), str(ROOT / "tests" / "plugins"),
                                         str(TESTS)])
    env["SPOTKM_INSTALL_PARTS"] = parts
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                          "-p", "spotsim_dropin", "--rootdir", str(tmp_path), str(TESTS / target)],
                         cwd=tmp_path, env=env, capture_output=True, text=True, timeout=timeout)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
    assert " passed" in res.stdout
    return res.stdout


@needs_ref
@pytest.mark.parametrize("target", [
    "test_migration.py",
    "test_costmodel.py::TestMigrationCost",
    "test_acceptance.py::test_criterion_03_migration_plan_soundness",
    "test_acceptance.py::test_criterion_06_case_study",
    "test_simulator.py",
])
def test_reference_tests_pass_with_native_planner(target, tmp_path):
    _run(target, "planner,estimator", tmp_path)


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("target", [
    "test_mapping.py",
    "test_acceptance.py::test_criterion_01_km_optimality",
    "test_acceptance.py::test_criterion_02_two_step_reduction",
    "test_acceptance.py::test_criterion_03_migration_plan_soundness",
    "test_acceptance.py::test_criterion_06_case_study",
    "test_migration.py",
    "test_costmodel.py::TestMigrationCost",
    "test_simulator.py",
])
def test_reference_tests_pass_with_full_dropin(target, tmp_path):
    """Mapper included: every map_devices / km_match / build_graph call of
    these reference tests runs on the GPU through libspotkm.so."""
    out = _run(target, "mapper,planner,estimator", tmp_path)
    assert "passed" in out
