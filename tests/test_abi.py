"""CPU-side checks of the C ABI boundary: the in-tree library loads and
exports every symbol include/spotkm.h declares; the numpy struct mirrors
match the header's sizes.  No compute calls (no GPU here)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2311_15566_b200 import _native as nat

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "spotkm.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*|void|double)\s+(sk_\w+)\s*\(",
                                 text, re.M)))


def test_header_declares_expected_symbols():
    syms = header_symbols()
    assert set(syms) == set(nat.EXPORTS) | {"sk_rat_to_double"}


def test_library_loads_and_exports_all_symbols():
    from paper_2311_15566_b200.build import build

    build()
    lib = ctypes.CDLL(str(nat.LIB_PATH))
    for s in header_symbols():
        assert hasattr(lib, s), s
    loaded = nat.load()
    assert loaded.sk_abi_version() == nat.ABI_VERSION


def test_struct_sizes_match_header():
    text = (ROOT / "include" / "spotkm.h").read_text()
    assert "} sk_segment; /* 32 bytes */" in text and nat.SEGMENT.itemsize == 32
    assert "} sk_plan; /* 64 bytes */" in text and nat.PLAN.itemsize == 64
    assert "} sk_sweep_desc; /* 48 bytes */" in text and nat.SWEEP_DESC.itemsize == 48


def test_compute_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2311_15566_b200 as sk

    g = sk.BipartiteGraph(gpus=[("i-0", 0)], slots=[sk.TopologyPosition(1, 1, 1)], weights=[[1.0]])
    with pytest.raises(RuntimeError):
        sk.km_match(g)
