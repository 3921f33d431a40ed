"""ctypes binding of the C ABI in include/spotkm.h (libspotkm.so, built in-tree).

There is no fallback: if the shared library is missing, importing any
compute entry point raises.  Build it with `python -m paper_2311_15566_b200.build`
(or `__graft_entry__.build()`).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_DIR = Path(__file__).resolve().parent / "_lib"
LIB_PATH = LIB_DIR / "libspotkm.so"

SK_OK, SK_EINVAL, SK_EGROUP, SK_ERANGE, SK_ENOSOURCE, SK_ECUDA, SK_ENOPEER = range(7)
SK_PLAN_FUSED_SUM = 1
SK_PLAN_DENSE = 2
SK_PLAN_GENERIC = 4
ABI_VERSION = 3
MAX_GENERIC_GROUP = 32   # k_fuse_generic: one warp per fused pair

# numpy mirrors of the C structs (field order and sizes must match spotkm.h)
SEGMENT = np.dtype([("l0", "<i4"), ("l1", "<i4"), ("a", "<i4"), ("b", "<i4"), ("pipe", "<i4"),
                    ("reserved", "<i4"), ("unit", "<i8")], align=True)
SEGMENT_WIDE = np.dtype([("l0", "<i4"), ("l1", "<i4"), ("pipe", "<i4"), ("reserved", "<i4"),
                         ("a", "<i8"), ("b", "<i8"), ("unit", "<i8"), ("reserved2", "<i8", (3,))],
                        align=True)
PLAN = np.dtype([("rows", "<i4"), ("D", "<i4"), ("P", "<i4"), ("M", "<i4"), ("L", "<i4"),
                 ("K", "<i4"), ("group", "<i4"), ("flags", "<i4"), ("row_base", "<i4"),
                 ("reserved", "<i4"), ("f_off", "<i8"), ("out_off", "<i8"), ("Kw", "<i8")],
                align=True)
SWEEP_DESC = np.dtype([("oD", "<i4"), ("oP", "<i4"), ("oM", "<i4"), ("G", "<i4"), ("n_inst", "<i4"),
                       ("alive_off", "<i4"), ("tok_off", "<i4"), ("plan", "<i4"), ("bpl", "<i8"),
                       ("kv", "<i8")], align=True)
COPY = np.dtype([("src", "<u8"), ("dst", "<u8"), ("bytes", "<u8")], align=True)
REGION = np.dtype([("ptr", "<u8"), ("bytes", "<u8"), ("key", "<u8"), ("base", "<u8")])
TL_PLAN = np.dtype([("act_begin", "<i4"), ("act_end", "<i4"), ("inst_base", "<i4"), ("n_inst", "<i4"),
                    ("start", "<f8"), ("step", "<f8"), ("progressive", "<i4"), ("reserved", "<i4")])
assert SEGMENT_WIDE.itemsize == 64
assert SEGMENT.itemsize == 32 and PLAN.itemsize == 64 and SWEEP_DESC.itemsize == 48 and COPY.itemsize == 24

EXPORTS = (
    "sk_abi_version", "sk_last_error", "sk_build_weights", "sk_map_batched", "sk_map_fuse",
    "sk_map_outer", "sk_map_outer_codes", "sk_outer_codes_bytes", "sk_km_dense",
    "sk_precoded_bytes", "sk_map_fuse_coded", "sk_map_outer_coded",
    "sk_sweep_expand", "sk_copy_batched", "sk_enable_peer_access",
    "sk_plan_migration", "sk_mig_counts", "sk_mig_export", "sk_mig_free", "sk_planner_error",
    "sk_plan_timeline", "sk_memopt_order", "sk_dev_alloc", "sk_dev_free", "sk_ipc_get_handle",
    "sk_ipc_open_handle", "sk_ipc_close_handle", "sk_fill_regions", "sk_verify_regions",
    "sk_reshard_error", "sk_migration_cost_batched", "sk_migration_cost",
    "sk_simulate_buffer_usage", "sk_fused_elems", "sk_exec_ctl_bytes", "sk_exec_plan", "sk_exec_reset", "sk_host_register",
    "sk_host_unregister",
    "sk_memcpy_batched", "sk_d2h", "sk_wait_flag", "sk_stream_wait_flag", "sk_score_configs", "sk_select_configs",
    "sk_estimator_error", "sk_plan_migration_many",
)


class NativeError(RuntimeError):
    """A CUDA-side failure (SK_ECUDA / SK_ENOPEER)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"spotkm error {code}: {msg}")
        self.code = code


_lib = None


def load():
    """Load libspotkm.so (once).  Raises if it is absent -- no CPU fallback."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("SPOTKM_LIB", LIB_PATH))
    if not path.exists():
        raise RuntimeError(
            f"{path} not found: the CUDA library is not built.  Run "
            "`python -m paper_2311_15566_b200.build` (there is no CPU fallback).")
    lib = ctypes.CDLL(str(path))
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    sig = {
        "sk_abi_version": ([], i32),
        "sk_last_error": ([], ctypes.c_char_p),
        "sk_build_weights": ([vp, i32, vp, vp, vp, i32, i32, vp], i32),
        "sk_map_batched": ([vp, i32, vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, i64, vp], i32),
        "sk_map_fuse": ([vp, i32, vp, vp, vp, vp, i32, i32, i32, i64, i64, vp], i32),
        "sk_map_outer": ([vp, i32, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp], i32),
        "sk_map_outer_codes": ([vp, i32, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp, i64, vp], i32),
        "sk_outer_codes_bytes": ([i32, i32, i32], i64),
        "sk_precoded_bytes": ([i32, i32, ctypes.POINTER(i64)], i64),
        "sk_map_fuse_coded": ([vp, i32, vp, vp, vp, vp, i32, i32, i32, vp, i64, vp, i64, vp], i32),
        "sk_map_outer_coded": ([vp, i32, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp, i64, vp, vp], i32),
        "sk_km_dense": ([vp, i32, vp, vp, vp, i32, i32, vp], i32),
        "sk_fused_elems": ([i32, i32, i32, i32], i64),
        "sk_sweep_expand": ([vp, i32, vp, vp, vp, vp, vp, i32, vp], i32),
        "sk_copy_batched": ([vp, i32, i32, vp], i32),
        "sk_enable_peer_access": ([i32, vp, i32], i32),
        "sk_dev_alloc": ([ctypes.c_uint64, ctypes.POINTER(vp)], i32),
        "sk_dev_free": ([vp], i32),
        "sk_ipc_get_handle": ([vp, vp], i32),
        "sk_ipc_open_handle": ([vp, ctypes.POINTER(vp)], i32),
        "sk_ipc_close_handle": ([vp], i32),
        "sk_fill_regions": ([vp, i32, vp], i32),
        "sk_verify_regions": ([vp, i32, vp, vp], i32),
        "sk_reshard_error": ([], ctypes.c_char_p),
        "sk_migration_cost_batched": ([vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_double,
                                       ctypes.c_double, vp, vp], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.sk_abi_version() != ABI_VERSION:
        raise RuntimeError(f"libspotkm ABI {lib.sk_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


def last_error() -> str:
    return load().sk_last_error().decode(errors="replace")


def check(rc: int, mapping_error=ValueError, migration_error=ValueError):
    """Translate an sk_status into the caller's (reference) exception class."""
    if rc == SK_OK:
        return
    msg = last_error()
    if rc in (SK_EINVAL, SK_EGROUP, SK_ERANGE):
        raise mapping_error(msg)
    if rc == SK_ENOSOURCE:
        raise migration_error(msg)
    raise NativeError(rc, msg)
