"""Batch assembly and the device calls behind the drop-in API.

One `MapBatch` gathers any number of mapping problems (one per
build_graph / map_devices call or per sweep plan), ships all host inputs in
ONE host->device copy (plans | row_ptr | segments), runs the C-ABI kernels on
the current torch stream, and returns all results in ONE device->host copy.
PyTorch provides device memory and the stream; all compute is libspotkm.so.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _native as nat


def _align(n: int, a: int = 64) -> int:
    return (n + a - 1) // a * a


def fused_elems(nA: int, nB: int, g: int, flags: int) -> int:
    """Fused-buffer elements of one plan (include/spotkm.h sk_fused_elems)."""
    pairs = nA * nB
    if not flags & nat.SK_PLAN_GENERIC:
        return pairs
    return pairs * (1 + g) + (pairs * g + 7) // 8


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2311_15566_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


class MapBatch:
    """Accumulates mapping problems in the sk_plan / sk_segment layout."""

    def __init__(self):
        self.plans: list[tuple] = []   # (rows, D, P, M, L, K, group, flags)
        self.row_ptrs: list[np.ndarray] = []
        self.segs: list[np.ndarray] = []

    def add(self, rows, D, P, M, L, K, group, flags, row_ptr, segs) -> int:
        self.plans.append((rows, D, P, M, L, K, group, flags))
        self.row_ptrs.append(row_ptr)
        self.segs.append(segs)
        return len(self.plans) - 1

    # -- layout ---------------------------------------------------------------
    def _layout(self, dense_cols: bool, order=None):
        """Plans in `order` (default: insertion order); returns arrays in that
        order plus summary sizes."""
        Q = len(self.plans)
        order = list(range(Q)) if order is None else list(order)
        plans = np.zeros(Q, dtype=nat.PLAN)
        seg_base = row_base = f_off = out_off = 0
        rp_parts = []
        max_pairs = max_n = max_rows = max_cols = max_na = max_nb = 0
        gmask = 0
        seg_parts = []
        for slot, q in enumerate(order):
            R, D, P, M, L, K, g, flags = self.plans[q]
            C = D * P * M
            nA, nB = R // g, C // g
            pairs = R * C if dense_cols else fused_elems(nA, nB, g, flags)
            generic = bool(flags & nat.SK_PLAN_GENERIC)
            # general-range plans carry K in Kw (sk_plan.K = 0)
            plans[slot] = (R, D, P, M, L, 0 if generic else K, g, flags, row_base, 0, f_off, out_off,
                           K if generic else 0)
            rp_parts.append(self.row_ptrs[q][:-1].astype(np.int64) + seg_base)
            seg_parts.append(self.segs[q])
            seg_base += len(self.segs[q])
            row_base += R
            f_off += pairs
            out_off += R
            max_pairs = max(max_pairs, nA * nB)
            max_n = max(max_n, nA, nB)
            max_na = max(max_na, nA)
            max_nb = max(max_nb, nB)
            max_rows = max(max_rows, R)
            max_cols = max(max_cols, C)
            gmask |= 1 if generic else 1 << g
        rp_parts.append(np.array([seg_base], dtype=np.int64))
        row_ptr = np.concatenate(rp_parts).astype(np.int32)
        segs = np.concatenate(seg_parts) if seg_parts else np.zeros(0, dtype=nat.SEGMENT)
        info = dict(Q=Q, rows=row_base, pairs=f_off, max_pairs=max_pairs, max_n=max_n,
                    max_na=max_na, max_nb=max_nb,
                    max_rows=max_rows, max_cols=max_cols, gmask=gmask)
        return plans, row_ptr, segs, info

    @staticmethod
    def _upload(*arrays):
        """One H2D copy of several arrays; returns (device tensor, [device ptrs])."""
        offs, total = [], 0
        for a in arrays:
            offs.append(total)
            total = _align(total + a.nbytes)
        host = np.zeros(max(total, 64), dtype=np.uint8)
        for a, o in zip(arrays, offs):
            if a.nbytes:
                host[o:o + a.nbytes] = np.frombuffer(a.tobytes(), dtype=np.uint8)
        dev = torch.from_numpy(host).to(_device(), non_blocking=False)
        base = dev.data_ptr()
        return dev, [base + o for o in offs]

    # -- K2: map_devices ----------------------------------------------------------
    def run_map(self, mapping_error=ValueError):
        """-> (assign int32 [sum R] (col or -1), totals float64 [Q], out_off per plan),
        all indexed by insertion order."""
        from .sweep import outer_classes

        lib = nat.load()
        n_of = []
        for (R, D, P, M, L, K, g, flags) in self.plans:
            n_of.append(max(R // g, (D * P * M) // g))
        order = sorted(range(len(self.plans)), key=lambda q: (-n_of[q], q))
        plans, row_ptr, segs, info = self._layout(dense_cols=False, order=order)
        dev_in, (p_plans, p_rp, p_segs) = self._upload(plans, row_ptr, segs)
        dev = _device()
        Q, rows = info["Q"], info["rows"]
        fused = torch.empty(max(info["pairs"], 1), dtype=torch.float64, device=dev)
        perm = torch.empty(max(info["pairs"], 1), dtype=torch.int32, device=dev)
        out = torch.empty(_align(8 * Q + 4 * rows) // 8 + 1, dtype=torch.float64, device=dev)
        p_total = out.data_ptr()
        p_assign = p_total + 8 * Q
        st = _stream_ptr()
        ns = np.array([n_of[q] for q in order], dtype=np.int64)
        if os.environ.get("SK_PRECODED", "0") == "1":
            # the sweep's coded K2 per size class (opt-in for the drop-in: its
            # calls are small, where the double matrix measured faster)
            g = plans["group"].astype(np.int64)
            na = plans["rows"].astype(np.int64) // g
            nb = (plans["D"] * plans["P"] * plans["M"]).astype(np.int64) // g
            gbit = np.where(plans["flags"] & nat.SK_PLAN_GENERIC, 1, np.left_shift(1, g))
            keep = []
            for a, b, mn in outer_classes(ns):
                mr = int(plans["rows"][a:b].max())
                d = ctypes.c_int64(0)
                cb = int(lib.sk_precoded_bytes(b - a, mn, ctypes.byref(d)))
                cmask = int(np.bitwise_or.reduce(gbit[a:b]))
                if cb > 0:
                    codes = torch.empty(cb, dtype=torch.uint8, device=dev)
                    dct = torch.empty((int(d.value) + 7) // 8, dtype=torch.int64, device=dev)
                    keep += [codes, dct]
                    rc = lib.sk_map_fuse_coded(p_plans + 64 * a, b - a, p_rp, p_segs, fused.data_ptr(),
                                               perm.data_ptr(), int(na[a:b].max()), int(nb[a:b].max()),
                                               cmask, codes.data_ptr(), cb, dct.data_ptr(), int(d.value), st)
                    nat.check(rc, mapping_error)
                    rc = lib.sk_map_outer_coded(p_plans + 64 * a, b - a, p_rp, p_segs, fused.data_ptr(),
                                                perm.data_ptr(), p_assign, p_total + 8 * a, 0, mn, mr,
                                                codes.data_ptr(), cb, dct.data_ptr(), st)
                else:
                    rc = lib.sk_map_fuse(p_plans + 64 * a, b - a, p_rp, p_segs, fused.data_ptr(),
                                         perm.data_ptr(), int(na[a:b].max()), int(nb[a:b].max()), cmask,
                                         0, 0, st)
                    nat.check(rc, mapping_error)
                    rc = lib.sk_map_outer(p_plans + 64 * a, b - a, p_rp, p_segs, fused.data_ptr(),
                                          perm.data_ptr(), p_assign, p_total + 8 * a, 0, mn, mr, st)
                nat.check(rc, mapping_error)
        else:
            rc = lib.sk_map_fuse(p_plans, Q, p_rp, p_segs, fused.data_ptr(), perm.data_ptr(),
                                 info["max_na"], info["max_nb"], info["gmask"], 0, 0, st)
            nat.check(rc, mapping_error)
            for a, b, mn in outer_classes(ns):
                mr = int(plans["rows"][a:b].max())
                rc = lib.sk_map_outer(p_plans + 64 * a, b - a, p_rp, p_segs, fused.data_ptr(),
                                      perm.data_ptr(), p_assign, p_total + 8 * a, 0, mn, mr, st)
                nat.check(rc, mapping_error)
        host = out.cpu().numpy().view(np.uint8)
        del dev_in
        totals_sorted = host[:8 * Q].view(np.float64)
        assign = host[8 * Q:8 * Q + 4 * rows].view(np.int32).copy()
        totals = np.empty(Q, dtype=np.float64)
        out_off = np.empty(Q, dtype=np.int64)
        for slot, q in enumerate(order):
            totals[q] = totals_sorted[slot]
            out_off[q] = plans["out_off"][slot]
        return assign, totals, out_off

    # -- K1: build_graph -----------------------------------------------------------
    def run_weights(self, mapping_error=ValueError):
        """-> list of float64 W matrices (R x C), one per plan."""
        lib = nat.load()
        plans, row_ptr, segs, info = self._layout(dense_cols=True)
        dev_in, (p_plans, p_rp, p_segs) = self._upload(plans, row_ptr, segs)
        W = torch.empty(max(info["pairs"], 1), dtype=torch.float64, device=_device())
        rc = lib.sk_build_weights(p_plans, info["Q"], p_rp, p_segs, W.data_ptr(), info["max_rows"],
                                  info["max_cols"], _stream_ptr())
        nat.check(rc, mapping_error)
        host = W.cpu().numpy()
        del dev_in
        out = []
        for q, (R, D, P, M, *_rest) in enumerate(self.plans):
            C = D * P * M
            o = int(plans["f_off"][q])
            out.append(host[o:o + R * C].reshape(R, C))
        return out


def km_dense(weights: np.ndarray, mapping_error=ValueError):
    """km_match on one dense float64 matrix -> (assign int32[R], total)."""
    lib = nat.load()
    R, C = weights.shape
    plans = np.zeros(1, dtype=nat.PLAN)
    plans[0] = (R, 1, 1, C, 1, 1, 1, nat.SK_PLAN_DENSE, 0, 0, 0, 0, 0)
    W = np.ascontiguousarray(weights, dtype=np.float64)
    dev_in, (p_plans, p_w) = MapBatch._upload(plans, W)
    out = torch.empty(_align(8 + 4 * R) // 8 + 1, dtype=torch.float64, device=_device())
    rc = lib.sk_km_dense(p_plans, 1, p_w, out.data_ptr() + 8, out.data_ptr(), max(R, C), R,
                         _stream_ptr())
    nat.check(rc, mapping_error)
    host = out.cpu().numpy().view(np.uint8)
    del dev_in
    return host[8:8 + 4 * R].view(np.int32).copy(), float(host[:8].view(np.float64)[0])
