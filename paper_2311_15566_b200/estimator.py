"""Batched candidate scoring on the device.

* `exec_latency_many` / `throughput_many` -- the reference's exec_latency and
  throughput (costmodel.py:144-183, with the prefill interpolation of
  costmodel.py:121-137) for many (config, workload) queries in one launch
  (`sk_score_configs`), bit-identical to the reference.
* `optimize_config_many` -- the controller's choice (controller.py:79-117)
  for many (n_available, rate, cloud_limit) scenarios over one candidate set:
  the candidates are scored once, then one device thread per scenario replays
  the reference's selection, ties included (`sk_select_configs`).
* `exec_latency`, `throughput`, `optimize_config` -- single-call drop-ins with
  the reference signatures (they run the same kernels on a batch of one).

The profile object is the caller's (reference `PerfProfile` or any object
with the same fields); a query whose (P,M,B) shape is not profiled raises the
caller's ProfileMissError, as the reference does (costmodel.py:104-118).
"""

from __future__ import annotations

import ctypes
import sys

import numpy as np

from . import _native as nat

EST_QUERY = np.dtype([("shape", "<i4"), ("D", "<i4"), ("P", "<i4"), ("B", "<i4"), ("s_in", "<i8"),
                      ("s_out", "<i8")])
assert EST_QUERY.itemsize == 32
LATENCY_SIMILARITY = 0.01   # controller.py:19


class ProfileMissError(ValueError):
    """(reference: costmodel.py:30-31; the caller's class is raised when known)"""


def _lib():
    lib = nat.load()
    if not getattr(lib, "_est_sigs", False):
        vp, i32 = ctypes.c_void_p, ctypes.c_int32
        lib.sk_score_configs.argtypes = [vp, i32, vp, vp, vp, vp, ctypes.c_double, vp, vp, vp]
        lib.sk_score_configs.restype = i32
        lib.sk_select_configs.argtypes = [vp, vp, vp, i32, vp, vp, vp, i32, ctypes.c_double, vp, vp]
        lib.sk_select_configs.restype = i32
        lib._est_sigs = True
    return lib


def _miss_error(profile):
    mod = sys.modules.get(type(profile).__module__)
    return getattr(mod, "ProfileMissError", ProfileMissError)


class _Tables:
    """A profile's decode / prefill tables as device arrays (one H2D)."""

    def __init__(self, profile):
        import torch

        from .device import _device

        self.shapes = sorted(set(profile.decode_table) | set(profile.prefill_table))
        self.index = {s: i for i, s in enumerate(self.shapes)}
        self.has_decode = [s in profile.decode_table for s in self.shapes]
        ptr, xs, ys = [0], [], []
        for s in self.shapes:
            pts = sorted(profile.prefill_table.get(s, {}).items())
            xs += [int(x) for x, _ in pts]
            ys += [float(y) for _, y in pts]
            ptr.append(len(xs))
        self.has_prefill = [ptr[i + 1] > ptr[i] for i in range(len(self.shapes))]
        dev = _device()
        self.decode = torch.tensor([float(profile.decode_table.get(s, 0.0)) for s in self.shapes] or [0.0],
                                   dtype=torch.float64, device=dev)
        self.ptr = torch.tensor(ptr, dtype=torch.int32, device=dev)
        self.xs = torch.tensor(xs or [0], dtype=torch.int64, device=dev)
        self.ys = torch.tensor(ys or [0.0], dtype=torch.float64, device=dev)
        self.eta = float(profile.pipeline_efficiency)


def _score(profile, rows, want_phi: bool, tables=None):
    """rows: [(D, P, M, B, s_in, s_out)] -> (latency[], phi[] or None)."""
    import torch

    from .device import _device, _stream_ptr

    T = tables or _Tables(profile)
    q = np.zeros(len(rows), dtype=EST_QUERY)
    for i, (D, P, M, B, s_in, s_out) in enumerate(rows):
        # the reference's order of checks (costmodel.py:146-152)
        if s_in < 0 or s_out < 0:
            mod = sys.modules.get(type(profile).__module__)
            raise getattr(mod, "CostModelError", ValueError)("sequence lengths must be >= 0")
        k = T.index.get((P, M, B))
        if k is None or not T.has_prefill[k]:
            raise _miss_error(profile)(f"no prefill entry for (P,M,B)={(P, M, B)}")
        if s_out > 0 and not T.has_decode[k]:
            raise _miss_error(profile)(f"no decode entry for (P,M,B)={(P, M, B)}")
        q[i] = (k, D, P, B, s_in, s_out)
    dev = _device()
    dq = torch.from_numpy(q.view(np.uint8)).to(dev)
    lat = torch.empty(max(len(rows), 1), dtype=torch.float64, device=dev)
    phi = torch.empty(max(len(rows), 1), dtype=torch.float64, device=dev) if want_phi else None
    nat.check(_lib().sk_score_configs(dq.data_ptr(), len(rows), T.decode.data_ptr(), T.ptr.data_ptr(),
                                      T.xs.data_ptr(), T.ys.data_ptr(), T.eta, lat.data_ptr(),
                                      phi.data_ptr() if phi is not None else 0, _stream_ptr()))
    lat_h = lat.cpu().numpy()[:len(rows)]
    return lat_h, (phi.cpu().numpy()[:len(rows)] if phi is not None else None)


def exec_latency_many(profile, queries) -> list:
    """queries: [(config, s_in, s_out[, batch_size])] -> exec_latency of each
    (costmodel.py:144-152)."""
    rows = []
    for qq in queries:
        cfg, s_in, s_out = qq[:3]
        b = qq[3] if len(qq) > 3 and qq[3] is not None else cfg.batch_limit
        rows.append((cfg.data_parallel, cfg.pipeline_stages, cfg.tensor_shards, b, int(s_in), int(s_out)))
    return _score(profile, rows, False)[0].tolist()


def throughput_many(profile, configs, s_in=None, s_out=None) -> list:
    """phi(C) for each config at the nominal (or given) workload
    (costmodel.py:170-183)."""
    s_in = profile.nominal_s_in if s_in is None else s_in
    s_out = profile.nominal_s_out if s_out is None else s_out
    rows = [(c.data_parallel, c.pipeline_stages, c.tensor_shards, c.batch_limit, int(s_in), int(s_out))
            for c in configs]
    return _score(profile, rows, True)[1].tolist()


def exec_latency(profile, config, s_in, s_out, batch_size=None) -> float:
    """(reference: costmodel.py:144-152)"""
    return exec_latency_many(profile, [(config, s_in, s_out, batch_size)])[0]


def throughput(profile, config, s_in=None, s_out=None) -> float:
    """(reference: costmodel.py:170-183)"""
    return throughput_many(profile, [config], s_in, s_out)[0]


class CandidateScores:
    """A candidate set scored once (nominal workload) and resident on the
    device, for many optimize_config decisions."""

    def __init__(self, profile, candidates, gpus_per_instance: int = 1):
        import torch

        from .device import _device

        if not candidates:
            mod = sys.modules.get(type(profile).__module__.replace("costmodel", "controller"))
            raise getattr(mod, "ControllerError", ValueError)("empty candidate set")
        self.cands = sorted(candidates)
        rows = [(c.data_parallel, c.pipeline_stages, c.tensor_shards, c.batch_limit,
                 int(profile.nominal_s_in), int(profile.nominal_s_out)) for c in self.cands]
        lat, phi = _score(profile, rows, True)
        dev = _device()
        self.n_inst = np.array([c.instances(gpus_per_instance) for c in self.cands], dtype=np.int32)
        self.d_inst = torch.from_numpy(self.n_inst).to(dev)
        self.d_phi = torch.from_numpy(phi).to(dev)
        self.d_lat = torch.from_numpy(lat).to(dev)
        self.latency, self.phi = lat, phi

    def choose(self, scenarios) -> list:
        """scenarios: [(n_available, rate[, cloud_limit])] -> chosen config or None."""
        import torch

        from .device import _device, _stream_ptr

        n = len(scenarios)
        if n == 0:
            return []
        avail = np.array([int(s[0]) for s in scenarios], dtype=np.int32)
        obt = np.array([int(s[2]) if len(s) > 2 and s[2] is not None else int(s[0]) for s in scenarios],
                       dtype=np.int32)
        rate = np.array([float(s[1]) for s in scenarios], dtype=np.float64)
        dev = _device()
        da, do, dr = (torch.from_numpy(x).to(dev) for x in (avail, obt, rate))
        out = torch.empty(n, dtype=torch.int32, device=dev)
        nat.check(_lib().sk_select_configs(self.d_inst.data_ptr(), self.d_phi.data_ptr(), self.d_lat.data_ptr(),
                                           len(self.cands), da.data_ptr(), do.data_ptr(), dr.data_ptr(), n,
                                           1 + LATENCY_SIMILARITY, out.data_ptr(), _stream_ptr()))
        return [None if k < 0 else self.cands[k] for k in out.cpu().tolist()]


def optimize_config_many(scenarios, profile, candidates, gpus_per_instance: int = 1) -> list:
    """optimize_config (controller.py:79-117) for many scenarios
    (n_available, rate[, cloud_limit]) over one candidate set."""
    return CandidateScores(profile, candidates, gpus_per_instance).choose(scenarios)


def optimize_config(n_available, current, rate, profile, candidates, gpus_per_instance: int = 1,
                    cloud_limit=None):
    """(reference: controller.py:79-117); `current` is unused there too."""
    return optimize_config_many([(n_available, rate, cloud_limit)], profile, candidates, gpus_per_instance)[0]
