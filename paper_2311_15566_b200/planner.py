"""Drop-in migration planner and T_mig estimator, computed natively.

`plan_migration`, `derive_transfers` and `memopt_layer_order` (reference:
migration.py:89-384) and `plan_timeline` / `migration_cost` (costmodel.py:189-260)
with the reference signatures and results, backed by the bit-exact C++
planner in libspotkm.so (csrc/planner.cpp; include/spotkm.h `sk_plan_migration`,
`sk_memopt_order`, `sk_plan_timeline`).  This module only flattens the caller's
objects into integer arrays and builds the caller's result objects back.

The plan produced here is the input of the migration executor (reshard.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _native as nat
from ._types import result_types
from .domain import natural_key


# ---------------------------------------------------------------------------
# ctypes mirrors of the planner structs (include/spotkm.h)

class _MigInput(ctypes.Structure):
    _fields_ = [("n_inst", ctypes.c_int32), ("n_gpus", ctypes.c_int32),
                ("inst_natrank", ctypes.c_void_p), ("inst_strrank", ctypes.c_void_p),
                ("inst_departing", ctypes.c_void_p), ("gpu_inst", ctypes.c_void_p),
                ("gpu_local", ctypes.c_void_p), ("gpu_pos", ctypes.c_void_p),
                ("model_ptr", ctypes.c_void_p), ("model_shards", ctypes.c_void_p),
                ("cache_ptr", ctypes.c_void_p), ("cache_shards", ctypes.c_void_p),
                ("D", ctypes.c_int32), ("P", ctypes.c_int32), ("M", ctypes.c_int32),
                ("L", ctypes.c_int32), ("bpl", ctypes.c_int64), ("kv", ctypes.c_int64),
                ("K", ctypes.c_int64), ("inh_ptr", ctypes.c_void_p), ("inh_items", ctypes.c_void_p),
                ("has_umax", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("u_max", ctypes.c_double)]


class _TimelineInput(ctypes.Structure):
    _fields_ = [("n_inst", ctypes.c_int32), ("n_actions", ctypes.c_int32),
                ("action_ptr", ctypes.c_void_p), ("src_inst", ctypes.c_void_p),
                ("dst_inst", ctypes.c_void_p), ("bytes", ctypes.c_void_p),
                ("bandwidth", ctypes.c_double), ("latency", ctypes.c_double),
                ("start", ctypes.c_double), ("has_release", ctypes.c_void_p),
                ("release", ctypes.c_void_p)]


TRANSFER = np.dtype([("kind", "<i4"), ("layer", "<i4"), ("lo", "<i8"), ("hi", "<i8"),
                     ("src", "<i4"), ("dst", "<i4"), ("bytes", "<f8"), ("rid", "<i8"),
                     ("tokens", "<i8")], align=True)
ACTION = np.dtype([("kind", "<i4"), ("layer", "<i4"), ("stage", "<i4"), ("tr_begin", "<i4"),
                   ("tr_end", "<i4"), ("rel_begin", "<i4"), ("rel_end", "<i4"),
                   ("reserved", "<i4")])
RELEASE = np.dtype([("inst", "<i4"), ("layer", "<i4"), ("bytes", "<f8")])
assert TRANSFER.itemsize == 56 and ACTION.itemsize == 32 and RELEASE.itemsize == 16

_ACTION_KINDS = ("migrate_cache", "migrate_layer", "start_stage")
_TRANSFER_KINDS = ("model", "cache")


def _lib():
    lib = nat.load()
    if not getattr(lib, "_planner_sigs", False):
        vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        lib.sk_plan_migration.argtypes = [vp, i32, ctypes.POINTER(vp)]
        lib.sk_plan_migration.restype = i32
        lib.sk_mig_counts.argtypes = [vp, vp]
        lib.sk_mig_counts.restype = i32
        lib.sk_mig_export.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        lib.sk_mig_export.restype = i32
        lib.sk_mig_free.argtypes = [vp]
        lib.sk_mig_free.restype = None
        lib.sk_planner_error.argtypes = []
        lib.sk_planner_error.restype = ctypes.c_char_p
        lib.sk_plan_timeline.argtypes = [vp, vp]
        lib.sk_plan_timeline.restype = i32
        lib.sk_memopt_order.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp, i32, dbl, vp]
        lib.sk_memopt_order.restype = i32
        lib.sk_migration_cost.argtypes = [vp, vp, dbl, i32, vp]
        lib.sk_migration_cost.restype = i32
        lib.sk_simulate_buffer_usage.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        lib.sk_simulate_buffer_usage.restype = i32
        lib.sk_plan_migration_many.argtypes = [vp, i32, i32, i32, vp, vp, vp]
        lib.sk_plan_migration_many.restype = i32
        lib.sk_rat_to_double.argtypes = [i64, ctypes.c_uint64, i64]
        lib.sk_rat_to_double.restype = dbl
        lib._planner_sigs = True
    return lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


@dataclass
class LayerTraffic:
    """(reference: migration.py:78-83)"""

    incoming: dict = field(default_factory=dict)
    freed: dict = field(default_factory=dict)


# ---------------------------------------------------------------------------
# flattening

class _Flat:
    """The caller's mapping + old layout as integer arrays over one K."""

    def __init__(self, mapping, old_layout, model, inherited_by_pipeline, departing):
        target = mapping.config
        self.gpus = sorted(old_layout, key=lambda g: (natural_key(g[0]), g[1]))
        self.insts = list(dict.fromkeys(g[0] for g in old_layout))  # old_layout first-seen order
        self.inst_idx = {name: i for i, name in enumerate(self.insts)}
        nat_keys = sorted({natural_key(n) for n in self.insts})
        nat_rank = {k: i for i, k in enumerate(nat_keys)}
        str_rank = {n: i for i, n in enumerate(sorted(self.insts))}
        self.natrank = np.array([nat_rank[natural_key(n)] for n in self.insts], dtype=np.int32)
        self.strrank = np.array([str_rank[n] for n in self.insts], dtype=np.int32)
        self.departing = np.array([1 if n in departing else 0 for n in self.insts], dtype=np.uint8)
        D, P, M = target.data_parallel, target.pipeline_stages, target.tensor_shards
        self.D, self.P, self.M = D, P, M
        # common denominator (native)
        from .pack import common_denominator

        invs = [old_layout[g] for g in self.gpus]
        K = self.K = common_denominator(invs, M)
        self.rids: dict = {}
        self.rid_names: list = []
        rids = self.rids

        def rid(name):
            r = rids.get(name)
            if r is None:
                r = rids[name] = len(self.rid_names)
                self.rid_names.append(name)
            return r

        self.gpu_inst = np.array([self.inst_idx[g[0]] for g in self.gpus], dtype=np.int32)
        self.gpu_local = np.array([g[1] for g in self.gpus], dtype=np.int32)
        pos = []
        for g in self.gpus:
            p = mapping.assignment.get(g)
            pos.append(-1 if p is None else ((p.pipeline - 1) * P + (p.stage - 1)) * M + (p.shard - 1))
        self.gpu_pos = np.array(pos, dtype=np.int32)
        from .pack import _native

        mp, ms, cp, cs = _native().flatten(invs, K, self.rids, self.rid_names)
        self.model_ptr = np.frombuffer(mp, dtype=np.int32).copy()
        self.model_shards = np.frombuffer(ms, dtype=np.int64).reshape(-1, 3).copy()
        self.cache_ptr = np.frombuffer(cp, dtype=np.int32).copy()
        self.cache_shards = np.frombuffer(cs, dtype=np.int64).reshape(-1, 5).copy()
        self.inh_ptr = None
        self.inh_items = None
        if inherited_by_pipeline:
            ptr, items = [0, 0], []
            for d in range(1, D + 1):
                for r_, tok in inherited_by_pipeline.get(d) or ():
                    items.append((rid(r_), tok))
                ptr.append(len(items))
            self.inh_ptr = np.array(ptr, dtype=np.int32)
            self.inh_items = np.array(items, dtype=np.int64).reshape(-1, 2) if items else np.zeros((0, 2), np.int64)
        self.model = model

    def struct(self, u_max):
        m = self.model
        s = _MigInput()
        s.n_inst, s.n_gpus = len(self.insts), len(self.gpus)
        s.inst_natrank, s.inst_strrank = _p(self.natrank), _p(self.strrank)
        s.inst_departing = _p(self.departing)
        s.gpu_inst, s.gpu_local, s.gpu_pos = _p(self.gpu_inst), _p(self.gpu_local), _p(self.gpu_pos)
        s.model_ptr, s.model_shards = _p(self.model_ptr), _p(self.model_shards)
        s.cache_ptr, s.cache_shards = _p(self.cache_ptr), _p(self.cache_shards)
        s.D, s.P, s.M, s.L = self.D, self.P, self.M, m.num_layers
        s.bpl, s.kv, s.K = m.bytes_per_layer, m.kv_bytes_per_token_per_layer, self.K
        if self.inh_ptr is not None:
            s.inh_ptr, s.inh_items = _p(self.inh_ptr), _p(self.inh_items)
        s.has_umax = 0 if u_max is None else 1
        s.u_max = 0.0 if u_max is None else float(u_max)
        return s


def _raise(flat, rc, T, lo=None, hi=None):
    lib = _lib()
    if rc == nat.SK_ENOSOURCE:
        if lo is None:
            lo, hi = (int(x) for x in lib.sk_planner_error().decode().split())
        raise T.MigrationError(
            f"no source holds required shard [{Fraction(lo, flat.K)},{Fraction(hi, flat.K)}): "
            "layout inconsistent with mapping")
    raise T.MigrationError(lib.sk_planner_error().decode())


def _export(res):
    """Copy a native sk_mig_result into numpy arrays, then free it."""
    lib = _lib()
    try:
        counts = np.zeros(7, dtype=np.int64)
        lib.sk_mig_counts(res, _p(counts))
        tr = np.zeros(max(int(counts[0]), 1), dtype=TRANSFER)
        ac = np.zeros(max(int(counts[1]), 1), dtype=ACTION)
        at = np.zeros(max(int(counts[2]), 1), dtype=np.int32)
        rl = np.zeros(max(int(counts[3]), 1), dtype=RELEASE)
        pk = np.zeros(max(int(counts[4]), 1), dtype=np.float64)
        lr = np.zeros(max(int(counts[5]), 1), dtype=RELEASE)
        lib.sk_mig_export(res, _p(tr), _p(ac), _p(at), _p(rl), _p(pk), _p(lr))
    finally:
        lib.sk_mig_free(res)
    return counts, tr, ac, at, rl, pk, lr


def _run(flat, u_max, derive_only, T):
    lib = _lib()
    s = flat.struct(u_max)
    res = ctypes.c_void_p()
    rc = lib.sk_plan_migration(ctypes.byref(s), 1 if derive_only else 0, ctypes.byref(res))
    if rc != nat.SK_OK:
        _raise(flat, rc, T)
    return _export(res)


def _transfers(flat, tr, n, T):
    K, gpus, names = flat.K, flat.gpus, flat.rid_names
    fracs: dict = {}

    def frac(v):  # memoised Fraction(v, K): few distinct endpoints
        f = fracs.get(v)
        if f is None:
            f = Fraction(v, K)
            fracs[v] = f
        return f

    make, kinds = T.Transfer, _TRANSFER_KINDS
    return [make(kind=kinds[kind], layer=layer, lo=frac(lo), hi=frac(hi), src=gpus[src],
                 dst=gpus[dst], bytes=b, request=None if rid < 0 else names[rid], tokens=tok)
            for kind, layer, lo, hi, src, dst, b, rid, tok in tr[:n].tolist()]


# ---------------------------------------------------------------------------
# public API

def derive_transfers(mapping, old_layout, model, inherited_by_pipeline=None, departing=frozenset()):
    """(reference: migration.py:201-305) -> (model_transfers{layer: [Transfer]},
    cache_transfers, layer_releases{layer: {inst: bytes}}, cache_releases{inst: bytes})."""
    T = result_types(mapping)
    if mapping.config is None:
        raise T.MigrationError("mapping carries no target config")
    flat = _Flat(mapping, old_layout, model, inherited_by_pipeline, departing)
    counts, tr, _, _, rl, _, lr = _run(flat, None, True, T)
    n_model = int(counts[6])
    allt = _transfers(flat, tr, int(counts[0]), T)
    model_transfers: dict = {}
    for t in allt[:n_model]:
        model_transfers.setdefault(t.layer, []).append(t)
    cache_transfers = allt[n_model:]
    layer_releases: dict = {}
    for inst, layer, b in lr[:int(counts[5])].tolist():
        layer_releases.setdefault(layer, {})[flat.insts[inst]] = b
    cache_releases = {flat.insts[inst]: b for inst, _, b in rl[:int(counts[3])].tolist()}
    return model_transfers, cache_transfers, layer_releases, cache_releases


def plan_migration(mapping, old_layout, model, u_max=None, inherited_by_pipeline=None,
                   departing=frozenset()):
    """(reference: migration.py:311-384)"""
    T = result_types(mapping)
    if mapping.config is None:
        raise T.MigrationError("mapping carries no target config")
    flat = _Flat(mapping, old_layout, model, inherited_by_pipeline, departing)
    return _build_plan(flat, _run(flat, u_max, False, T), u_max, T)


def _build_plan(flat, exported, u_max, T):
    counts, tr, ac, at, rl, pk, _ = exported
    allt = _transfers(flat, tr, int(counts[0]), T)
    at = at[:int(counts[2])].tolist()
    rel = [(flat.insts[i], b) for i, _, b in rl[:int(counts[3])].tolist()]
    actions = []
    for kind, layer, stage, t0, t1, r0, r1, _ in ac[:int(counts[1])].tolist():
        actions.append(T.MigrationAction(
            kind=_ACTION_KINDS[kind], transfers=tuple(allt[i] for i in at[t0:t1]),
            releases=tuple(rel[r0:r1]), layer=None if layer < 0 else layer,
            stage=None if stage < 0 else stage))
    plan = T.MigrationPlan(actions=actions, u_max=u_max)
    plan.peak_usage = {name: float(pk[i]) for i, name in enumerate(flat.insts)}
    return plan


def plan_migration_many(problems, threads: int = 0) -> list:
    """`plan_migration` for many independent problems (host,
    one thread per plan): each problem is the argument tuple
    (mapping, old_layout, model[, u_max[, inherited_by_pipeline[, departing]]]).
    The caller's objects are flattened here; the planning itself runs in ONE
    native call on a pool of `threads` host threads (0 = all cores, GIL
    released).  Returns one MigrationPlan per problem, or the exception the
    single call would raise, in place (not raised)."""
    flats, structs, Ts, umax = [], [], [], []
    for args in problems:
        mapping, old_layout, model = args[:3]
        u_max = args[3] if len(args) > 3 else None
        inh = args[4] if len(args) > 4 else None
        dep = args[5] if len(args) > 5 else frozenset()
        T = result_types(mapping)
        if mapping.config is None:
            flats.append(T.MigrationError("mapping carries no target config"))
            structs.append(None)
        else:
            f = _Flat(mapping, old_layout, model, inh, dep)
            flats.append(f)
            structs.append(f.struct(u_max))
        Ts.append(T)
        umax.append(u_max)
    idx = [i for i, st in enumerate(structs) if st is not None]
    n = len(idx)
    arr = (_MigInput * max(n, 1))(*[structs[i] for i in idx])
    outs = (ctypes.c_void_p * max(n, 1))()
    status = np.zeros(max(n, 1), dtype=np.int32)
    err = np.zeros(2 * max(n, 1), dtype=np.int64)
    if n:
        _lib().sk_plan_migration_many(ctypes.cast(arr, ctypes.c_void_p), n, 0, int(threads),
                                      ctypes.cast(outs, ctypes.c_void_p), _p(status), _p(err))
    results = list(flats)
    for k, i in enumerate(idx):
        f, T = flats[i], Ts[i]
        if status[k] != nat.SK_OK:
            if outs[k]:
                _lib().sk_mig_free(outs[k])
            try:
                _raise(f, int(status[k]), T, int(err[2 * k]), int(err[2 * k + 1]))
            except Exception as e:  # noqa: BLE001
                results[i] = e
            continue
        results[i] = _build_plan(f, _export(outs[k]), umax[i], T)
    return results


def memopt_layer_order(traffic_by_layer, u_max):
    """(reference: migration.py:114-143) -- native greedy over the caller's
    per-layer LayerTraffic."""
    layers = sorted(traffic_by_layer)
    insts: dict = {}
    ip, ii, ib, fp, fi, fb = [0], [], [], [0], [], []
    for layer in layers:
        t = traffic_by_layer[layer]
        for name, b in t.incoming.items():
            ii.append(insts.setdefault(name, len(insts)))
            ib.append(float(b))
        ip.append(len(ii))
        for name, b in t.freed.items():
            fi.append(insts.setdefault(name, len(insts)))
            fb.append(float(b))
        fp.append(len(fi))
    arr = [np.array(x, dtype=dt) for x, dt in ((ip, np.int32), (ii, np.int32), (ib, np.float64),
                                              (fp, np.int32), (fi, np.int32), (fb, np.float64))]
    arr = [a if a.size else np.zeros(1, a.dtype) for a in arr]
    order = np.zeros(max(len(layers), 1), dtype=np.int32)
    _lib().sk_memopt_order(len(layers), max(len(insts), 1), *(_p(a) for a in arr),
                           0 if u_max is None else 1, 0.0 if u_max is None else float(u_max),
                           _p(order))
    return [layers[i] for i in order[:len(layers)].tolist()]


def simulate_buffer_usage(plan, old_layout) -> dict:
    """(reference: migration.py:387-401): replay receives and end-of-round
    releases; per-instance peak -- computed by sk_simulate_buffer_usage."""
    names: dict = {}
    for gpu in old_layout:
        names.setdefault(gpu[0], len(names))
    n_seed = len(names)
    tr_ptr, tr_dst, tr_b, rel_ptr, rel_i, rel_b = [0], [], [], [0], [], []
    for action in plan.actions:
        for tr in action.transfers:
            tr_dst.append(names.setdefault(tr.dst[0], len(names)))
            tr_b.append(tr.bytes)
        for inst, b in action.releases:
            rel_i.append(names.setdefault(inst, len(names)))
            rel_b.append(b)
        tr_ptr.append(len(tr_dst))
        rel_ptr.append(len(rel_i))
    n = max(len(names), 1)
    by_name = sorted(names, key=lambda x: x)
    rank = np.zeros(n, dtype=np.int32)
    for r, name in enumerate(by_name):
        rank[names[name]] = r
    arrs = [np.array(tr_ptr, np.int32), np.array(tr_dst or [0], np.int32),
            np.array(tr_b or [0.0], np.float64), np.array(rel_ptr, np.int32),
            np.array(rel_i or [0], np.int32), np.array(rel_b or [0.0], np.float64)]
    peaks = np.zeros(n, dtype=np.float64)
    order = np.zeros(n, dtype=np.int32)
    n_order = ctypes.c_int32(0)
    _lib().sk_simulate_buffer_usage(len(names), n_seed, len(plan.actions), *(_p(a) for a in arrs),
                                    _p(rank), _p(peaks), _p(order), ctypes.addressof(n_order))
    inv = {i: name for name, i in names.items()}
    return {inv[int(i)]: float(peaks[int(i)]) for i in order[:n_order.value]}


def _timeline_input(plan, profile, release, start):
    """Flatten a plan for sk_plan_timeline / sk_migration_cost.  Returns the
    struct and the arrays it points into (kept alive by the caller)."""
    release = release or {}
    names: dict = {}
    ptr, src, dst, byt = [0], [], [], []
    for action in plan.actions:
        for tr in action.transfers:
            src.append(names.setdefault(tr.src[0], len(names)))
            dst.append(names.setdefault(tr.dst[0], len(names)))
            byt.append(float(tr.bytes))
        ptr.append(len(src))
    for name in release:
        names.setdefault(name, len(names))
    n = max(len(names), 1)
    has_rel = np.zeros(n, dtype=np.uint8)
    rel = np.zeros(n, dtype=np.float64)
    for name, t in release.items():
        has_rel[names[name]] = 1
        rel[names[name]] = float(t)
    arrs = [np.array(ptr, np.int32), np.array(src or [0], np.int32), np.array(dst or [0], np.int32),
            np.array(byt or [0.0], np.float64), has_rel, rel]
    ti = _TimelineInput()
    ti.n_inst, ti.n_actions = n, len(plan.actions)
    ti.action_ptr, ti.src_inst, ti.dst_inst, ti.bytes = (_p(a) for a in arrs[:4])
    ti.bandwidth, ti.latency, ti.start = float(profile.bandwidth), float(profile.transfer_latency), float(start)
    ti.has_release, ti.release = _p(has_rel), _p(rel)
    return ti, arrs


def plan_timeline(plan, profile, release=None, start=0.0) -> list:
    """(reference: costmodel.py:189-228), computed by sk_plan_timeline."""
    ti, _keep = _timeline_input(plan, profile, release, start)
    ends = np.zeros(max(len(plan.actions), 1), dtype=np.float64)
    _lib().sk_plan_timeline(ctypes.byref(ti), _p(ends))
    return ends[:len(plan.actions)].tolist()


def migration_cost(plan, profile, config=None, progressive=False, release=None, start=0.0) -> float:
    """(reference: costmodel.py:231-260): full T_mig, or with progressive start
    the worst stage-ready constraint -- computed by sk_migration_cost."""
    ti, _keep = _timeline_input(plan, profile, release, start)
    stages = np.array([a.stage if a.kind == "start_stage" else -1 for a in plan.actions] or [-1],
                      dtype=np.int32)
    step = 0.0
    if progressive and config is not None:
        step = profile.decode_seconds(config) / config.pipeline_stages
    out = np.zeros(1, dtype=np.float64)
    _lib().sk_migration_cost(ctypes.byref(ti), _p(stages), float(step), 1 if progressive else 0, _p(out))
    return float(out[0])


def plan_to_dict(plan) -> dict:
    """JSON wire format, Fractions as [num, den] (reference: migration.py:407-431)."""
    actions = []
    for a in plan.actions:
        doc = {"kind": a.kind}
        if a.layer is not None:
            doc["layer"] = a.layer
        if a.stage is not None:
            doc["stage"] = a.stage
        if a.transfers:
            docs = []
            for t in a.transfers:
                td = {"kind": t.kind, "layer": t.layer, "lo": [t.lo.numerator, t.lo.denominator],
                      "hi": [t.hi.numerator, t.hi.denominator], "src": [t.src[0], t.src[1]],
                      "dst": [t.dst[0], t.dst[1]], "bytes": t.bytes}
                if t.request:
                    td["request"] = t.request
                    td["tokens"] = t.tokens
                docs.append(td)
            doc["transfers"] = docs
        if a.releases:
            doc["releases"] = [[inst, b] for inst, b in a.releases]
        actions.append(doc)
    return {"u_max": plan.u_max, "actions": actions,
            "peak_usage": dict(sorted(plan.peak_usage.items()))}


def plan_from_dict(doc: dict, types=None):
    """(reference: migration.py:434-453)"""
    from . import migration as own

    T = types or own
    actions = []
    for a in doc["actions"]:
        trs = tuple(T.Transfer(kind=t["kind"], layer=t["layer"], lo=Fraction(*t["lo"]),
                               hi=Fraction(*t["hi"]), src=(t["src"][0], t["src"][1]),
                               dst=(t["dst"][0], t["dst"][1]), bytes=t["bytes"],
                               request=t.get("request"), tokens=t.get("tokens", 0))
                    for t in a.get("transfers", ()))
        rels = tuple((inst, b) for inst, b in a.get("releases", ()))
        actions.append(T.MigrationAction(kind=a["kind"], transfers=trs, releases=rels,
                                         layer=a.get("layer"), stage=a.get("stage")))
    plan = T.MigrationPlan(actions=actions, u_max=doc.get("u_max"))
    plan.peak_usage = dict(doc.get("peak_usage", {}))
    return plan


def migration_cost_many(plans, profile, configs=None, progressive=False, releases=None,
                        starts=None) -> list:
    """Batched `migration_cost` (costmodel.py:231-260) for many candidate plans
    on the GPU, one thread per plan (`sk_migration_cost_batched`); the result
    of each entry is bit-identical to `migration_cost` with the same
    arguments.  `configs`, `releases`, `starts` are per-plan sequences (or None)."""
    import torch

    from .device import _device, _stream_ptr

    Q = len(plans)
    if Q == 0:
        return []
    configs = configs or [None] * Q
    releases = releases or [None] * Q
    starts = starts or [0.0] * Q
    tl = np.zeros(Q, dtype=nat.TL_PLAN)
    act_ptr, act_stage, src, dst, byt = [0], [], [], [], []
    has_rel, rel = [], []
    inst_base = 0
    n_act = 0
    for q, plan in enumerate(plans):
        names: dict = {}
        for action in plan.actions:
            for tr in action.transfers:
                src.append(names.setdefault(tr.src[0], len(names)))
                dst.append(names.setdefault(tr.dst[0], len(names)))
                byt.append(float(tr.bytes))
            act_ptr.append(len(src))
            act_stage.append(action.stage if action.kind == "start_stage" else -1)
        r = releases[q] or {}
        for name in r:
            names.setdefault(name, len(names))
        flags = [0] * len(names)
        vals = [0.0] * len(names)
        for name, t in r.items():
            flags[names[name]] = 1
            vals[names[name]] = float(t)
        has_rel += flags
        rel += vals
        cfg = configs[q]
        step = profile.decode_seconds(cfg) / cfg.pipeline_stages if (progressive and cfg is not None) else 0.0
        tl[q] = (n_act, n_act + len(plan.actions), inst_base, len(names), float(starts[q]), step,
                 1 if progressive else 0, 0)
        n_act += len(plan.actions)
        inst_base += len(names)
    arrs = [np.array(act_ptr, np.int32), np.array(act_stage or [0], np.int32),
            np.array(src or [0], np.int32), np.array(dst or [0], np.int32),
            np.array(byt or [0.0], np.float64), np.array(has_rel or [0], np.uint8),
            np.array(rel or [0.0], np.float64)]
    dev = _device()
    d = [torch.from_numpy(a).to(dev) for a in arrs]
    d_tl = torch.from_numpy(tl.view(np.uint8)).to(dev)
    scratch = torch.empty(max(2 * inst_base, 1), dtype=torch.float64, device=dev)
    flags_d = torch.empty(max(2 * inst_base, 1), dtype=torch.uint8, device=dev)
    cost = torch.empty(Q, dtype=torch.float64, device=dev)
    rc = nat.load().sk_migration_cost_batched(
        d_tl.data_ptr(), Q, *(x.data_ptr() for x in d), scratch.data_ptr(), flags_d.data_ptr(),
        float(profile.bandwidth), float(profile.transfer_latency), cost.data_ptr(), _stream_ptr())
    nat.check(rc)
    return cost.cpu().tolist()
