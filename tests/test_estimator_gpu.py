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


# ---------------------------------------------------------------------------
# candidate scoring (estimator.py): exec_latency / throughput / optimize_config
# vs the reference's own values (tests/golden/gen_golden_r2.py, all three
# bundled profiles, every candidate config up to 64 GPUs)

def _profile(t):
    from fmt import unhx as u

    return SimpleNamespace(
        decode_table={(P, M, B): u(v) for P, M, B, v in t["decode"]},
        prefill_table={k: d for k, d in _prefill(t["prefill"]).items()},
        pipeline_efficiency=u(t["eta"]), nominal_s_in=t["nominal"][0], nominal_s_out=t["nominal"][1])


def _prefill(rows):
    out = {}
    for P, M, B, s, v in rows:
        out.setdefault((P, M, B), {})[s] = unhx(v)
    return out


@pytest.mark.parametrize("prof", ["gpt-20b", "opt-6.7b", "llama-30b"])
def test_exec_latency_and_throughput_bit_exact(golden, prof):
    from paper_2311_15566_b200 import estimator

    doc = golden("estimator")["profiles"][prof]
    p = _profile(doc["profile"])
    rows = [(sk.ParallelConfig(*c), s_in, s_out) for c, s_in, s_out, v in doc["latency"] if v is not None]
    got = estimator.exec_latency_many(p, rows)
    exp = [v for *_, v in doc["latency"] if v is not None]
    assert [g.hex() for g in got] == exp
    phi = estimator.throughput_many(p, [sk.ParallelConfig(*c) for c, _ in doc["throughput"]])
    assert [x.hex() for x in phi] == [v for _, v in doc["throughput"]]
    # single-call drop-ins
    c0, s0, o0, v0 = doc["latency"][3]
    assert estimator.exec_latency(p, sk.ParallelConfig(*c0), s0, o0).hex() == v0


@pytest.mark.parametrize("prof", ["gpt-20b", "opt-6.7b", "llama-30b"])
def test_optimize_config_decisions_match_reference(golden, prof):
    from paper_2311_15566_b200 import estimator

    doc = golden("estimator")["profiles"][prof]
    p = _profile(doc["profile"])
    cands = [sk.ParallelConfig(*c) for c, _ in doc["throughput"]]
    for G in (1, 4):
        dec = [d for d in doc["decisions"] if d[0] == G]
        scores = estimator.CandidateScores(p, cands, G)
        got = scores.choose([(n, r, lim) for _, n, r, lim, _ in dec])
        exp = [None if d[-1] is None else sk.ParallelConfig(*d[-1]) for d in dec]
        assert got == exp
    one = dec[len(dec) // 2]
    assert estimator.optimize_config(one[1], None, one[2], p, cands, G, one[3]) == exp[len(dec) // 2]
