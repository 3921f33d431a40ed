"""Drop-in device mapper: `build_graph`, `km_match`, `map_devices` with the
reference signatures and results (reference: mapping.py:35-283), computed by
the sm_100a kernels K1 (weights) and K2 (inner KM + outer KM) through the C ABI.

Host work is limited to validation, the row/column order, and re-encoding
inventories as exact integer segments (pack.py).  Every edge weight, match,
assignment and total_weight comes from the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from ._types import result_types
from .device import MapBatch, km_dense
from .domain import natural_key, shard_interval, stage_layers
from .pack import PackError, common_denominator, inherited_by_new, need_tokens, pack_rows


class MappingError(ValueError):
    """(reference: mapping.py:31-32)"""


@dataclass
class BipartiteGraph:
    """(reference: mapping.py:35-50)"""

    gpus: list
    slots: list
    weights: list

    def __post_init__(self):
        if len(self.weights) != len(self.gpus):
            raise MappingError("weight rows must match gpu count")
        for row in self.weights:
            if len(row) != len(self.slots):
                raise MappingError("weight cols must match slot count")
            if any(w < 0 for w in row):
                raise MappingError("weights must be >= 0")


@dataclass
class DeviceMapping:
    """(reference: mapping.py:53-65)"""

    assignment: dict
    total_weight: float
    config: object = None

    def position_of(self, gpu):
        return self.assignment.get(gpu)

    def gpu_for(self) -> dict:
        return {pos: gpu for gpu, pos in self.assignment.items()}


def default_inheritance(d_old: int, d_new: int) -> dict[int, int]:
    """Identity on min(D_old, D_new) (reference: mapping.py:172-174)."""
    return {d: d for d in range(1, min(d_old, d_new) + 1)}


def sorted_gpu_refs(instances) -> list:
    """(reference: mapping.py:177-181)"""
    refs = []
    for inst in sorted(instances, key=lambda i: natural_key(i.id)):
        refs.extend(inst.gpu_refs())
    return refs


def required_context_with_cache(config, pos, model, inherited, inventory_cls=None):
    """Position needs: model block x shard, plus cache of inherited requests
    with tokens > 0 (reference: mapping.py:155-169).  Host-side helper for the
    planner; the device evaluates the same thing in closed form."""
    if inventory_cls is None:
        inventory_cls = result_types(config).ContextInventory
    lo, hi = shard_interval(config.tensor_shards, pos.shard)
    block = stage_layers(model.num_layers, config.pipeline_stages, pos.stage)
    shards = tuple((layer, lo, hi) for layer in block)
    if not inherited:
        return inventory_cls(model_shards=shards)
    cache = tuple((rid, layer, lo, hi, tok) for rid, tok in inherited for layer in block if tok > 0)
    return inventory_cls(model_shards=shards, cache_shards=cache)


# ---------------------------------------------------------------------------
# problem packing

class _Problem:
    __slots__ = ("refs", "rows", "D", "P", "M", "L", "K", "row_ptr", "segs", "wide")


def _pack_problem(instances, target, model, inheritance, requests_by_old_pipeline, err,
                  force_wide=False):
    prob = _Problem()
    refs, invs = [], []
    for inst in sorted(instances, key=lambda i: natural_key(i.id)):
        for g in range(inst.gpus):
            refs.append((inst.id, g))
            invs.append(inst.gpu_inventories[g])
    prob.refs = refs
    prob.rows = len(refs)
    prob.D, prob.P, prob.M = target.data_parallel, target.pipeline_stages, target.tensor_shards
    prob.L = model.num_layers
    need = need_tokens(inherited_by_new(inheritance, requests_by_old_pipeline), prob.D)
    try:
        prob.K = common_denominator(invs, prob.M)
        prob.row_ptr, prob.segs, prob.wide = pack_rows(invs, prob.K, model.bytes_per_layer,
                                                       model.kv_bytes_per_token_per_layer, need,
                                                       force_wide)
    except PackError as e:
        raise err(str(e)) from None
    return prob


def _slots(target, T):
    D, P, M = target.data_parallel, target.pipeline_stages, target.tensor_shards
    return [T.TopologyPosition(d, p, m) for d in range(1, D + 1) for p in range(1, P + 1)
            for m in range(1, M + 1)]


# ---------------------------------------------------------------------------
# public API

def build_graph(instances, target, model, inheritance=None, requests_by_old_pipeline=None):
    """Reusable-bytes matrix W[gpu][position] (reference: mapping.py:184-216),
    built by kernel K1."""
    T = result_types(target)
    prob = _pack_problem(instances, target, model, inheritance, requests_by_old_pipeline,
                         T.MappingError)
    slots = _slots(target, T)
    if prob.rows == 0:
        return T.BipartiteGraph(gpus=[], slots=slots, weights=[])
    batch = MapBatch()
    batch.add(prob.rows, prob.D, prob.P, prob.M, prob.L, prob.K, 1,
              nat.SK_PLAN_GENERIC if prob.wide else 0, prob.row_ptr, prob.segs)
    (W,) = batch.run_weights(T.MappingError)
    return T.BipartiteGraph(gpus=prob.refs, slots=slots, weights=W.tolist())


def km_match(graph):
    """Maximum-weight assignment on a given graph (reference: mapping.py:125-149),
    replayed exactly by the device KM."""
    T = result_types(graph)
    n_l, n_r = len(graph.gpus), len(graph.slots)
    if n_l == 0 or n_r == 0:
        return T.DeviceMapping(assignment={}, total_weight=0.0)
    W = np.array(graph.weights, dtype=np.float64).reshape(n_l, n_r)
    assign, total = km_dense(W, T.MappingError)
    mapping = {}
    for i in range(n_l):
        j = int(assign[i])
        if j >= 0:
            mapping[graph.gpus[i]] = graph.slots[j]
    return T.DeviceMapping(assignment=mapping, total_weight=total)


def _validate(instances, target, gpus_per_instance, fused_weight, T):
    for inst in instances:
        if inst.gpus != gpus_per_instance:
            raise T.MappingError(
                f"instance {inst.id} has {inst.gpus} GPUs, expected {gpus_per_instance}")
    if fused_weight not in ("max", "sum"):
        raise T.MappingError("fused_weight must be 'max' or 'sum'")
    group = min(gpus_per_instance, target.tensor_shards)
    if not (group == 1 and gpus_per_instance == 1):
        if gpus_per_instance % group or target.tensor_shards % group:
            raise T.MappingError(
                f"group size {group} must divide both G={gpus_per_instance} "
                f"and M={target.tensor_shards}")
    if group > nat.MAX_GENERIC_GROUP:
        raise T.MappingError(f"fused group {group} > {nat.MAX_GENERIC_GROUP} GPUs is not supported "
                             "by the device matcher")
    return group


def map_devices(instances, target, model, gpus_per_instance, inheritance=None,
                requests_by_old_pipeline=None, fused_weight="max"):
    """Two-step KM device mapping (reference: mapping.py:222-283): NodeFusion,
    inner KM per fused pair, max|sum fused edge, outer KM, expansion -- all on
    the device (K2)."""
    return map_devices_many([(instances, target, model, gpus_per_instance, inheritance,
                              requests_by_old_pipeline, fused_weight)])[0]


def map_devices_many(problems):
    """Batched map_devices: a list of argument tuples
    (instances, target, model, G[, inheritance[, requests[, fused_weight]]])
    solved in one device batch.  Returns one DeviceMapping per problem."""
    batch = MapBatch()
    metas = []
    for args in problems:
        instances, target, model, G = args[:4]
        inheritance = args[4] if len(args) > 4 else None
        reqs = args[5] if len(args) > 5 else None
        fused_weight = args[6] if len(args) > 6 else "max"
        T = result_types(target)
        group = _validate(instances, target, G, fused_weight, T)
        # fused groups > 8 take the general-range kernels (so do numerators
        # >= 2^53 and denominators > 2^31 - 1, detected by the packer)
        prob = _pack_problem(instances, target, model, inheritance, reqs, T.MappingError,
                             force_wide=group > 8)
        flags = nat.SK_PLAN_FUSED_SUM if fused_weight == "sum" else 0
        if prob.wide:
            flags |= nat.SK_PLAN_GENERIC
        idx = None
        if prob.rows:
            idx = batch.add(prob.rows, prob.D, prob.P, prob.M, prob.L, prob.K, group, flags,
                            prob.row_ptr, prob.segs)
        metas.append((T, target, prob, idx))
    if batch.plans:
        assign, totals, out_off = batch.run_map(metas[0][0].MappingError)
    results = []
    for T, target, prob, idx in metas:
        if idx is None:
            results.append(T.DeviceMapping(assignment={}, total_weight=0.0, config=target))
            continue
        slots = _slots(target, T)
        o = int(out_off[idx])
        cols = assign[o:o + prob.rows]
        mapping = {prob.refs[r]: slots[c] for r, c in enumerate(cols.tolist()) if c >= 0}
        results.append(T.DeviceMapping(assignment=mapping, total_weight=float(totals[idx]),
                                       config=target))
    return results
