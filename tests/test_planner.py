"""Native migration planner + T_mig estimator vs the reference's own outputs.

The planner is host C++ inside libspotkm.so (no GPU needed), so these run in
the CPU suite.  Golden plans come from running the real reference
(tests/golden/gen_golden.py): 60 synthetic transitions (acceptance-03 style,
with KV cache, departing instances, U_max caps, missing-source errors) and
every plan_migration / migration_cost call of the B_S scenario.  Comparison is
plan_to_dict equality (Fractions as [num, den], floats exact)."""

from fractions import Fraction
from types import SimpleNamespace

import pytest

from fmt import dec_inv, unhx

import paper_2311_15566_b200 as sk
from paper_2311_15566_b200 import planner
from paper_2311_15566_b200.migration import MigrationAction, MigrationPlan, Transfer


def rebuild(doc):
    model = sk.ModelSpec("m", *doc["model"])
    target = sk.ParallelConfig(*doc["target"], 1) if doc["target"] else None
    assignment = {(g, i): sk.TopologyPosition(d, p, m) for g, i, d, p, m in doc["assignment"]}
    mapping = sk.DeviceMapping(assignment=assignment, total_weight=0.0, config=target)
    layout = {}
    for iid, g, inv in doc["old_layout"]:
        m_, c_ = dec_inv(inv)
        layout[(iid, g)] = sk.ContextInventory(model_shards=m_, cache_shards=c_)
    inherited = None
    if doc["inherited"] is not None:
        inherited = {int(d): [(r, t) for r, t in lst] for d, lst in doc["inherited"].items()}
    return model, mapping, layout, inherited, frozenset(doc["departing"])


def _check_cases(cases):
    n = 0
    for doc in cases:
        model, mapping, layout, inh, dep = rebuild(doc)
        if doc["error"]:
            with pytest.raises(sk.MigrationError) as ei:
                planner.plan_migration(mapping, layout, model, u_max=doc["u_max"],
                                       inherited_by_pipeline=inh, departing=dep)
            if "message" in doc:
                assert str(ei.value) == doc["message"]
            continue
        plan = planner.plan_migration(mapping, layout, model, u_max=doc["u_max"],
                                      inherited_by_pipeline=inh, departing=dep)
        assert planner.plan_to_dict(plan) == doc["plan"]
        assert plan.peak_usage == planner.simulate_buffer_usage(plan, layout)
        n += 1
    return n


def test_plans_match_reference_synthetic(golden):
    cases = golden("plans")["cases"]
    assert _check_cases(cases) >= 40
    assert any(c["error"] for c in cases)


def test_plans_match_reference_scenario(golden):
    assert _check_cases(golden("scenario")["plans"]) >= 5


def test_cost_full_matches_reference(golden):
    prof = SimpleNamespace(bandwidth=1e9, transfer_latency=0.005)
    n = 0
    for doc in golden("plans")["cases"]:
        if doc["error"]:
            continue
        plan = planner.plan_from_dict(doc["plan"])
        assert planner.migration_cost(plan, prof).hex() == doc["cost_full"]
        n += 1
    assert n > 20


def test_scenario_costs_match_reference(golden):
    for doc in golden("scenario")["costs"]:
        plan = planner.plan_from_dict(doc["plan"])
        t_dec = doc["t_dec"]
        prof = SimpleNamespace(bandwidth=doc["bandwidth"], transfer_latency=doc["latency"],
                               decode_seconds=lambda cfg, _t=t_dec: _t)
        cfg = sk.ParallelConfig(*doc["config"]) if doc["config"] else None
        rel = None if doc["release"] is None else {k: unhx(v) for k, v in doc["release"].items()}
        got = planner.migration_cost(plan, prof, config=cfg, progressive=doc["progressive"],
                                     release=rel, start=unhx(doc["start"]))
        assert got.hex() == doc["value"]


def test_derive_transfers_consistent_with_plan(golden):
    for doc in golden("plans")["cases"][:30]:
        if doc["error"]:
            continue
        model, mapping, layout, inh, dep = rebuild(doc)
        mt, ct, lr, cr = planner.derive_transfers(mapping, layout, model, inh, dep)
        plan = planner.plan_migration(mapping, layout, model, u_max=None,
                                      inherited_by_pipeline=inh, departing=dep)
        moved = [t for a in plan.actions for t in a.transfers]
        assert sorted(moved, key=repr) == sorted([t for v in mt.values() for t in v] + list(ct), key=repr)


# reference unit known-answers (tests/test_migration.py:98-118, 249-281)
def _traffic(inc, freed=None):
    freed = freed or {}
    return {l: planner.LayerTraffic(incoming=dict(v), freed=dict(freed.get(l, {}))) for l, v in inc.items()}


def test_memopt_known_answers():
    t = _traffic({i: {"a": 10.0} for i in range(5)}, {i: {"a": 10.0} for i in range(5)})
    assert planner.memopt_layer_order(t, u_max=100.0) == [0, 1, 2, 3, 4]
    t = _traffic({0: {"a": 10}, 1: {"a": 10}, 2: {"a": 200}, 3: {"a": 10}},
                 {0: {"a": 10}, 1: {"a": 10}, 2: {"a": 200}, 3: {"a": 10}})
    assert planner.memopt_layer_order(t, u_max=50.0) == [0, 1, 3, 2]
    t = _traffic({i: {"a": float(i + 1)} for i in range(6)})
    assert planner.memopt_layer_order(t, u_max=None) == list(range(6))
    t = _traffic({0: {"a": 100}, 1: {"a": 100}, 2: {"a": 100}})
    assert planner.memopt_layer_order(t, u_max=10.0) == [0, 1, 2]


def test_buffer_usage_hand_replay():
    def tr(src, dst, nbytes):
        return Transfer(kind="model", layer=0, lo=Fraction(0), hi=Fraction(1), src=(src, 0),
                        dst=(dst, 0), bytes=float(nbytes))

    plan = MigrationPlan(actions=[
        MigrationAction(kind="migrate_layer", layer=0, transfers=(tr("a", "b", 60), tr("b", "c", 40)),
                        releases=(("a", 60.0), ("b", 40.0))),
        MigrationAction(kind="migrate_layer", layer=1, transfers=(tr("c", "a", 30),),
                        releases=(("c", 30.0),)),
    ])
    inv = {(x, 0): sk.ContextInventory() for x in "abc"}
    assert planner.simulate_buffer_usage(plan, inv) == {"a": 0.0, "b": 60.0, "c": 40.0}


def test_costmodel_known_answers():
    prof = SimpleNamespace(bandwidth=1e9, transfer_latency=0.0)

    def ft(src, dst, nbytes):
        return Transfer(kind="model", layer=0, lo=Fraction(0), hi=Fraction(1), src=src, dst=dst,
                        bytes=float(nbytes))

    one = MigrationPlan(actions=[MigrationAction(kind="migrate_layer", layer=0,
                                                 transfers=(ft(("a", 0), ("b", 0), 1e9),))])
    assert planner.migration_cost(one, prof) == pytest.approx(1.0)
    assert planner.migration_cost(MigrationPlan(actions=[]), prof) == 0.0
    shared = MigrationPlan(actions=[MigrationAction(kind="migrate_layer", layer=0, transfers=(
        ft(("a", 0), ("b", 0), 1e9), ft(("a", 1), ("c", 0), 1e9)))])
    assert planner.migration_cost(shared, prof) == pytest.approx(2.0)
    local = MigrationPlan(actions=[MigrationAction(kind="migrate_layer", layer=0,
                                                   transfers=(ft(("a", 0), ("a", 1), 5e9),))])
    assert planner.migration_cost(local, prof) == 0.0
    assert planner.migration_cost(one, prof, release={"a": 5.0}, start=2.0) == pytest.approx(4.0)


def test_rat_to_double_correctly_rounded():
    import random

    lib = planner._lib()
    rng = random.Random(3)
    for _ in range(3000):
        num = rng.getrandbits(rng.choice([10, 53, 60, 64, 90, 120]))
        den = rng.randrange(1, 1 << rng.choice([3, 20, 31, 40]))
        got = lib.sk_rat_to_double(num >> 64, num & ((1 << 64) - 1), den)
        assert got == float(Fraction(num, den)), (num, den)


def test_plan_migration_many_equals_single_calls(golden):
    """The threaded batch (one native call, a pool of host threads) returns
    exactly the single-call plans, errors in place."""
    docs = golden("plans")["cases"] + golden("scenario")["plans"]
    probs = []
    for doc in docs:
        model, mapping, layout, inh, dep = rebuild(doc)
        probs.append((mapping, layout, model, doc["u_max"], inh, dep))
    for threads in (1, 4, 0):
        got = planner.plan_migration_many(probs, threads=threads)
        assert len(got) == len(docs)
        for g, doc in zip(got, docs):
            if doc["error"]:
                assert isinstance(g, sk.MigrationError)
                if "message" in doc:
                    assert str(g) == doc["message"]
            else:
                assert planner.plan_to_dict(g) == doc["plan"]
