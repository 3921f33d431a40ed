"""pytest plugin: install the native planner/estimator into the reference
package before its test modules are imported (used by
tests/test_reference_suite.py to run the reference's OWN migration and
cost-model tests against this implementation)."""

import os

import spotsim  # noqa: F401  (the reference package, from PYTHONPATH)
import spotsim.costmodel  # noqa: F401
import spotsim.mapping  # noqa: F401
import spotsim.migration  # noqa: F401
import spotsim.simulator  # noqa: F401

from paper_2311_15566_b200.install import install

PARTS = tuple(os.environ.get("SPOTKM_INSTALL_PARTS", "planner,estimator").split(","))
REPLACED = install(spotsim, parts=PARTS)
assert REPLACED, "nothing was rebound"

if "mapper" in PARTS:
    # the device mapper has no CPU fallback: make sure the CUDA library is the
    # thing these tests exercise
    import torch

    from paper_2311_15566_b200 import _native

    assert torch.cuda.is_available(), "mapper drop-in needs a GPU"
    _native.load()
