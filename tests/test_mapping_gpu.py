"""GPU parity: the CUDA path (through the C ABI) vs the reference's golden
outputs and the CPU oracle.  Bit-exact: W entries, assignments and
total_weight compare as float hex."""

import numpy as np
import pytest

from fmt import unhx
from helpers import assignment_cols, own_problem
from oracle import port

import paper_2311_15566_b200 as sk

pytestmark = pytest.mark.gpu


def graph_of(weights):
    gpus = [(f"i-{k}", 0) for k in range(len(weights))]
    slots = [sk.TopologyPosition(1, 1, m + 1) for m in range(len(weights[0]))]
    return sk.BipartiteGraph(gpus=gpus, slots=slots, weights=[list(r) for r in weights])


def test_km_match_golden(golden):
    for case in golden("km")["cases"]:
        W = [[unhx(x) for x in row] for row in case["W"]]
        got = sk.km_match(graph_of(W))
        cols = [-1] * len(W)
        for (iid, _), pos in got.assignment.items():
            cols[int(iid.split("-")[1])] = pos.shard - 1
        assert cols == case["assign"]
        assert got.total_weight.hex() == case["total"]


@pytest.mark.parametrize("name", ["mapping", "scenario"])
def test_build_graph_and_map_devices_golden(golden, name):
    doc = golden(name)
    cases = doc["cases"] if name == "mapping" else doc["maps"]
    for case in cases:
        model, cfg, G, insts, inh, rq, fw = own_problem(case)
        if "W" in case:
            g = sk.build_graph(insts, cfg, model, inh, rq)
            assert [[x.hex() for x in row] for row in g.weights] == case["W"]
        if case["error"]:
            with pytest.raises(sk.MappingError):
                sk.map_devices(insts, cfg, model, G, inh, rq, fw)
            continue
        got = sk.map_devices(insts, cfg, model, G, inh, rq, fw)
        assert assignment_cols(got, insts, cfg) == case["assign"]
        assert got.total_weight.hex() == case["total"]


def test_batched_equals_single(golden):
    cases = [c for c in golden("mapping")["cases"] if not c["error"]][:40]
    probs = [own_problem(c) for c in cases]
    many = sk.map_devices_many([(i, c, m, G, inh, rq, fw) for m, c, G, i, inh, rq, fw in probs])
    for (m, c, G, i, inh, rq, fw), got, case in zip(probs, many, cases):
        assert assignment_cols(got, i, c) == case["assign"]
        assert got.total_weight.hex() == case["total"]


def test_km_random_tie_heavy_vs_oracle():
    rng = np.random.default_rng(5)
    for n in (3, 17, 33, 64, 130, 257, 300):
        for kind in ("tie", "int"):
            w = (rng.integers(0, 3, size=(n, n)) if kind == "tie"
                 else rng.integers(0, 10**6, size=(n, n))).astype(float).tolist()
            exp_assign, exp_total = port.km_flat(w, n, n)
            got = sk.km_match(graph_of(w))
            cols = [-1] * n
            for (iid, _), pos in got.assignment.items():
                cols[int(iid.split("-")[1])] = pos.shard - 1
            assert cols == exp_assign, (n, kind)
            assert got.total_weight == exp_total
