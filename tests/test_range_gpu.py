"""GPU parity beyond the regular encoding and at the headline sizes, against
vectors produced by the REAL reference (tests/golden/gen_golden_r2.py):

* fused groups > 8 (G = M = 10, 12, 16 and M = 32), edge-weight numerators
  >= 2^53, interval denominators > 2^31 - 1, inheritance maps naming
  pipelines outside 1..D -- the general-range kernels (SK_PLAN_GENERIC);
* flat km_match on huge / subnormal weights and at n = 5,000 (> 4,095: the
  k_outer_huge path), the latter against the C oracle;
* plans of the headline sweep at 64 / 128 / 256 / 512 / 1,024 positions
  solved by the reference's own map_devices, through both the batched sweep
  path (SweepRunner) and the drop-in map_devices on caller objects;
* the OPT-6.7B and LLaMA-30B B_S scenario replans (BASELINE.json configs[1]).
All comparisons are bit-exact (float hex)."""

import numpy as np
import pytest

from cases import plan_digest
from fmt import unhx
from helpers import assignment_cols, own_from_port, own_problem
from oracle import cport
from oracle.sweep_inputs import plan_to_port

import paper_2311_15566_b200 as sk
from paper_2311_15566_b200 import sweep

pytestmark = pytest.mark.gpu


def graph_of(weights):
    gpus = [(f"i-{k}", 0) for k in range(len(weights))]
    slots = [sk.TopologyPosition(1, 1, m + 1) for m in range(len(weights[0]))]
    return sk.BipartiteGraph(gpus=gpus, slots=slots, weights=[list(r) for r in weights])


def cols_of(got, n_rows):
    cols = [-1] * n_rows
    for (iid, _), pos in got.assignment.items():
        cols[int(iid.split("-")[1])] = pos.shard - 1
    return cols


@pytest.mark.parametrize("name", ["edge", "models_bs"])
def test_map_devices_golden_r2(golden, name):
    doc = golden(name)
    cases = doc["cases"] if name == "edge" else doc["maps"]
    n = 0
    for case in cases:
        model, cfg, G, insts, inh, rq, fw = own_problem(case)
        if "W" in case:
            g = sk.build_graph(insts, cfg, model, inh, rq)
            assert [[x.hex() for x in row] for row in g.weights] == case["W"]
        got = sk.map_devices(insts, cfg, model, G, inh, rq, fw)
        assert assignment_cols(got, insts, cfg) == case["assign"]
        assert got.total_weight.hex() == case["total"]
        n += 1
    assert n >= 30


@pytest.mark.parametrize("coded", ["0", "1"])
def test_generic_plans_batched_with_regular_ones(golden, monkeypatch, coded):
    """general-range and regular plans in ONE device batch (coded = 1: the
    coded K2 entry points, general-range plans keeping their double matrix)"""
    monkeypatch.setenv("SK_PRECODED", coded)
    cases = golden("edge")["cases"] + golden("mapping")["cases"][:40]
    cases = [c for c in cases if not c["error"]]
    probs = [own_problem(c) for c in cases]
    many = sk.map_devices_many([(i, c, m, G, inh, rq, fw) for m, c, G, i, inh, rq, fw in probs])
    for (m, c, G, i, inh, rq, fw), got, case in zip(probs, many, cases):
        assert assignment_cols(got, i, c) == case["assign"]
        assert got.total_weight.hex() == case["total"]


def test_km_wide_golden(golden):
    for case in golden("edge")["km"]:
        W = [[unhx(x) for x in row] for row in case["W"]]
        got = sk.km_match(graph_of(W))
        assert cols_of(got, len(W)) == case["assign"]
        assert got.total_weight.hex() == case["total"]


def test_km_match_n5000_vs_c_oracle():
    n = 5000
    rng = np.random.default_rng(n)
    w = np.zeros((n, n))
    idx = np.arange(n)
    w[idx, (idx * 7) % n] = rng.integers(1, 100, size=n)
    w += (rng.random((n, n)) < 0.002) * rng.integers(1, 100, size=(n, n))
    exp = cport.hungarian(w)
    got = sk.km_match(graph_of(w.tolist()))
    assert cols_of(got, n) == exp
    total = 0.0
    for i, j in enumerate(exp):
        total += w[i, j]
    assert got.total_weight == total


def test_sweep_beyond_4095_outer_vs_c_oracle():
    """G = 1 sweep at 4,800 positions: outer n ~ 4,800 -> k_outer_huge"""
    b = sweep.make_sweep(4800, 1, seed=3, G=1, shapes=((2, 8), (4, 4)))
    assert int(b.stats()["n"].max()) > 4095
    assign, totals = sweep.SweepRunner(b).run()
    exp_assign, exp_totals = cport.map_sweep(b.desc, b.plans, b.alive, b.tok)
    assert np.array_equal(assign, exp_assign)
    assert [t.hex() for t in totals] == [t.hex() for t in exp_totals]


@pytest.mark.parametrize("coded", ["auto", "1"])
def test_headline_sweep_plans_vs_reference(golden, monkeypatch, coded):
    monkeypatch.setenv("SK_PRECODED", coded)
    cases = golden("sweep_ref")["cases"]
    by_n = {}
    for c in cases:
        by_n.setdefault(c["N"], []).append(c)
    assert set(by_n) == {64, 128, 256, 512, 1024}
    for N, cs in sorted(by_n.items()):
        b = sweep.make_sweep(N, cs[0]["sets"], seed=cs[0]["seed"])
        assign, totals = sweep.SweepRunner(b).run()
        for c in cs:
            q = c["q"]
            assert plan_digest(b, q) == c["digest"]
            o, R = int(b.plans["out_off"][q]), int(b.plans["rows"][q])
            assert assign[o:o + R].tolist() == c["assign"], (N, q)
            assert totals[q].hex() == c["total"], (N, q)
            # the drop-in on caller objects gives the same plan
            inst, new, G, inh, reqs, fw = plan_to_port(b, q, sweep.GPT20B, n_requests=4)
            model, cfg, insts, rq = own_from_port(inst, new, G, inh, reqs, sweep.GPT20B)
            got = sk.map_devices(insts, cfg, model, G, inh, rq, fw)
            assert assignment_cols(got, insts, cfg) == c["assign"], (N, q)
            assert got.total_weight.hex() == c["total"], (N, q)
