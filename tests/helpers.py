"""Test helpers: golden cases -> this package's own domain objects."""

from __future__ import annotations

from cases import decode_map_case

import paper_2311_15566_b200 as sk
from paper_2311_15566_b200.domain import natural_key


def own_problem(case):
    model, target, G, instances, inh, reqs, fw = decode_map_case(case)
    mspec = sk.ModelSpec(name="m", num_layers=model[0], bytes_per_layer=model[1],
                         kv_bytes_per_token_per_layer=model[2])
    cfg = sk.ParallelConfig(*target, 1)
    insts = []
    for iid, invs in instances:
        insts.append(sk.InstanceState(
            id=iid, kind="spot", gpus=len(invs),
            gpu_inventories=[sk.ContextInventory(model_shards=inv.model, cache_shards=inv.cache)
                             for inv in invs]))
    rq = None
    if reqs is not None:
        rq = {d: [sk.RequestSpec(id=rid, arrival_time=0.0, s_in=tok, s_out=max(tok, 1))
                  for rid, tok in lst] for d, lst in reqs.items()}
    return mspec, cfg, G, insts, inh, rq, fw


def assignment_cols(mapping, instances, cfg):
    slots = sk.positions(cfg)
    col = {s: j for j, s in enumerate(slots)}
    out = []
    for inst in sorted(instances, key=lambda i: natural_key(i.id)):
        for g in range(inst.gpus):
            pos = mapping.assignment.get((inst.id, g))
            out.append(-1 if pos is None else col[pos])
    return out


def own_from_port(instances, new, G, inh, reqs, model_geom):
    """oracle-port plain values (oracle.sweep_inputs.plan_to_port) -> this
    package's own domain objects, for the drop-in map_devices."""
    L, bpl, kv = model_geom
    mspec = sk.ModelSpec(name="m", num_layers=L, bytes_per_layer=bpl, kv_bytes_per_token_per_layer=kv)
    insts = [sk.InstanceState(id=iid, kind="spot", gpus=G,
                              gpu_inventories=[sk.ContextInventory(model_shards=tuple(i.model),
                                                                   cache_shards=tuple(i.cache))
                                               for i in invs])
             for iid, invs in instances]
    rq = {d: [sk.RequestSpec(id=rid, arrival_time=0.0, s_in=tok, s_out=max(tok, 1)) for rid, tok in lst]
          for d, lst in reqs.items()}
    return mspec, sk.ParallelConfig(*new, 1), insts, rq


def port_mapper(instances, target, model, G, inheritance=None, requests_by_old_pipeline=None,
                fused_weight="max"):
    """map_devices computed by the CPU oracle (tests only: lets host-side
    executor logic be tested without a GPU)."""
    from oracle import port

    insts = sorted(instances, key=lambda i: natural_key(i.id))
    pinst = [(i.id, [port.Inv(tuple(v.model_shards), tuple(v.cache_shards)) for v in i.gpu_inventories])
             for i in insts]
    reqs = None
    if requests_by_old_pipeline is not None:
        reqs = {d: [(r.id, r.s_in + r.tokens_generated) for r in rs]
                for d, rs in requests_by_old_pipeline.items()}
    tgt = (target.data_parallel, target.pipeline_stages, target.tensor_shards)
    refs, slots, W, assign, total = port.map_devices(pinst, tgt, (model.num_layers, model.bytes_per_layer,
                                                                  model.kv_bytes_per_token_per_layer),
                                                     G, inheritance, reqs, fused_weight)
    pos = sk.positions(target)
    mapping = {refs[r]: pos[c] for r, c in enumerate(assign) if c >= 0}
    return sk.DeviceMapping(assignment=mapping, total_weight=total, config=target)
