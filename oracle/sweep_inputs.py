"""TEST INFRASTRUCTURE ONLY: sweep plan -> oracle-port inputs.

Decodes the compact sweep descriptors (paper_2311_15566_b200/sweep.py)
independently of the device expansion kernel into the plain-value inputs of
oracle/port.py: instances with positional old inventories and per-request KV
cache shards.  Each old pipeline's token sum is split over `n_requests`
requests (sum preserved, so the weights are identical) so the CPU baseline
does the same per-shard work as the reference would."""

from __future__ import annotations

from oracle import port


def plan_to_port(batch, q, model, n_requests: int = 1):
    d = batch.desc[q]
    p = batch.plans[q]
    oD, oP, oM, G, n_inst = int(d["oD"]), int(d["oP"]), int(d["oM"]), int(d["G"]), int(d["n_inst"])
    words = batch.alive[int(d["alive_off"]):int(d["alive_off"]) + (n_inst + 31) // 32]
    alive = [(int(words[k >> 5]) >> (k & 31)) & 1 for k in range(n_inst)]
    toks = batch.tok[int(d["tok_off"]):int(d["tok_off"]) + oD]
    old = (oD, oP, oM)
    slots = port.positions(old)
    reqs = {}
    for dd in range(oD):
        tot = int(toks[dd])
        parts = [tot // n_requests] * n_requests
        parts[0] += tot - sum(parts)
        reqs[dd + 1] = [(f"r{dd + 1}-{j:02d}", t) for j, t in enumerate(parts)]
    instances = []
    for k in range(n_inst):
        if not alive[k]:
            continue
        invs = []
        for g in range(G):
            qq = k * G + g
            if qq < len(slots):
                inv = port.required(old, slots[qq], model)
                cache = tuple((rid, layer, lo, hi, t) for rid, t in reqs[slots[qq][0]]
                              for layer, lo, hi in inv.model)
                invs.append(port.Inv(inv.model, cache))
            else:
                invs.append(port.Inv())
        instances.append((f"i-{k}", invs))
    new = (int(p["D"]), int(p["P"]), int(p["M"]))
    inh = {dd: dd for dd in range(1, min(oD, new[0]) + 1)}
    fw = "sum" if int(p["flags"]) & 1 else "max"
    return instances, new, G, inh, reqs, fw


def plan_to_spotsim(batch, q, model_geom, spotsim, n_requests: int = 4):
    """One sweep plan -> the REAL reference's objects (spotsim.domain), so the
    reference's own map_devices can run on exactly the plan the GPU solves.
    Returns the map_devices arguments (instances, target, model, G,
    inheritance, requests_by_old_pipeline, fused_weight)."""
    dm = spotsim.domain
    instances, new, G, inh, reqs, fw = plan_to_port(batch, q, model_geom, n_requests=n_requests)
    L, bpl, kv = model_geom
    model = dm.ModelSpec(name="sweep", num_layers=L, bytes_per_layer=bpl, kv_bytes_per_token_per_layer=kv)
    insts = []
    for iid, invs in instances:
        inst = dm.InstanceState(id=iid, kind="spot", gpus=G)
        inst.gpu_inventories = [dm.ContextInventory(model_shards=tuple(i.model), cache_shards=tuple(i.cache))
                                for i in invs]
        insts.append(inst)
    rq = {d: [dm.RequestSpec(id=rid, arrival_time=0.0, s_in=tok, s_out=max(tok, 1)) for rid, tok in lst]
          for d, lst in reqs.items()}
    return insts, dm.ParallelConfig(*new, 1), model, G, inh, rq, fw


def mapping_cols(mapping, instances, target, spotsim):
    """A DeviceMapping as assigned column per GPU row (reference row order)."""
    slots = spotsim.domain.positions(target)
    col = {s: j for j, s in enumerate(slots)}
    out = []
    for inst in sorted(instances, key=lambda i: spotsim.domain.natural_key(i.id)):
        for g in range(inst.gpus):
            pos = mapping.assignment.get((inst.id, g))
            out.append(-1 if pos is None else col[pos])
    return out
