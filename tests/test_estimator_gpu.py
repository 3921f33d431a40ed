"""Batched T_mig estimator on the GPU (sk_migration_cost_batched) vs the
reference's own migration_cost values (golden scenario calls) and the host
estimator -- bit-exact."""

from types import SimpleNamespace

import pytest

from fmt import unhx

import paper_2311_15566_b200 as sk
from paper_2311_15566_b200 import planner

pytestmark = pytest.mark.gpu


def test_batched_costs_match_reference_scenario(golden):
    docs = golden("scenario")["costs"]
    by_key = {}
    for doc in docs:
        by_key.setdefault((doc["bandwidth"], doc["latency"], doc["t_dec"], doc["progressive"]), []).append(doc)
    n = 0
    for (bw, lat, t_dec, prog), group in by_key.items():
        prof = SimpleNamespace(bandwidth=bw, transfer_latency=lat, decode_seconds=lambda cfg, _t=t_dec: _t)
        plans = [planner.plan_from_dict(d["plan"]) for d in group]
        cfgs = [sk.ParallelConfig(*d["config"]) if d["config"] else None for d in group]
        rels = [None if d["release"] is None else {k: unhx(v) for k, v in d["release"].items()}
                for d in group]
        starts = [unhx(d["start"]) for d in group]
        got = planner.migration_cost_many(plans, prof, cfgs, prog, rels, starts)
        for g, d in zip(got, group):
            assert g.hex() == d["value"]
            n += 1
    assert n == len(docs)


def test_batched_costs_match_host_on_synthetic_plans(golden):
    prof = SimpleNamespace(bandwidth=1e9, transfer_latency=0.005, decode_seconds=lambda cfg: 0.1)
    plans = [planner.plan_from_dict(d["plan"]) for d in golden("plans")["cases"] if not d["error"]]
    got = planner.migration_cost_many(plans, prof)
    exp = [planner.migration_cost(p, prof) for p in plans]
    assert [x.hex() for x in got] == [x.hex() for x in exp]
    cfg = sk.ParallelConfig(1, 2, 1, 1)
    got = planner.migration_cost_many(plans, prof, [cfg] * len(plans), True, None, [1.5] * len(plans))
    exp = [planner.migration_cost(p, prof, config=cfg, progressive=True, start=1.5) for p in plans]
    assert [x.hex() for x in got] == [x.hex() for x in exp]
