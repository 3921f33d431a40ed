"""Decode golden mapping cases into the oracle's plain-value form."""

from __future__ import annotations

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
