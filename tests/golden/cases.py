"""Decode golden mapping cases into the oracle's plain-value form."""

from __future__ import annotations

import hashlib

import numpy as np

from fmt import dec_inv, unhx

from oracle.port import Inv


def decode_map_case(case):
    model = tuple(case["model"])
    target = tuple(case["target"])
    instances = [(iid, [Inv(*dec_inv(inv)) for inv in invs]) for iid, invs in case["instances"]]
    inheritance = None
    if case["inheritance"] is not None:
        inheritance = {int(k): v for k, v in case["inheritance"].items()}
    reqs = None
    if case["reqs"] is not None:
        reqs = {int(d): [(rid, tok) for rid, tok in lst] for d, lst in case["reqs"].items()}
    return model, target, case["G"], instances, inheritance, reqs, case["fused_weight"]


def golden_w(case):
    return [[unhx(x) for x in row] for row in case["W"]]


def plan_digest(batch, q) -> str:
    """Digest of one sweep plan's compact inputs (pins the regenerated plan)."""
    d = batch.desc[q]
    p = batch.plans[q]
    n_inst, oD = int(d["oD"]), int(d["oD"])
    n_inst = int(d["n_inst"])
    words = batch.alive[int(d["alive_off"]):int(d["alive_off"]) + (n_inst + 31) // 32]
    toks = batch.tok[int(d["tok_off"]):int(d["tok_off"]) + oD]
    h = hashlib.sha256()
    for x in (d["oD"], d["oP"], d["oM"], d["G"], d["n_inst"], d["bpl"], d["kv"], p["rows"], p["D"], p["P"],
              p["M"], p["L"], p["K"], p["group"], p["flags"]):
        h.update(int(x).to_bytes(8, "little", signed=True))
    h.update(np.ascontiguousarray(words).tobytes())
    h.update(np.ascontiguousarray(toks).tobytes())
    return h.hexdigest()[:32]
