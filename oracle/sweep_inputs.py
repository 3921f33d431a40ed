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
