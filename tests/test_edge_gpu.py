"""Edge cases and maximum sizes on the GPU vs the CPU oracles: empty and
rectangular graphs, the largest outer KM sizes (multi-warp path), non-dyadic
(M = 3, 6) sweeps where weights need a rounded division, and the compensated
builtin-sum fused weight at scale."""

import numpy as np
import pytest

from oracle import cport, port

import paper_2311_15566_b200 as sk
from paper_2311_15566_b200 import sweep

pytestmark = pytest.mark.gpu


def graph_of(weights):
    gpus = [(f"i-{k}", 0) for k in range(len(weights))]
    slots = [sk.TopologyPosition(1, 1, m + 1) for m in range(len(weights[0]))] if weights else []
    return sk.BipartiteGraph(gpus=gpus, slots=slots, weights=[list(r) for r in weights])


def cols_of(got, n_rows):
    cols = [-1] * n_rows
    for (iid, _), pos in got.assignment.items():
        cols[int(iid.split("-")[1])] = pos.shard - 1
    return cols


def test_empty_and_degenerate():
    got = sk.km_match(sk.BipartiteGraph(gpus=[], slots=[], weights=[]))
    assert got.assignment == {} and got.total_weight == 0.0
    got = sk.km_match(graph_of([[0.0], [9.0], [1.0]]))
    assert got.total_weight == 9.0 and list(got.assignment) == [("i-1", 0)]
    w = [[float(x) for x in range(300)]]
    exp_assign, exp_total = port.km_flat(w, 1, 300)
    got = sk.km_match(graph_of(w))
    assert cols_of(got, 1) == exp_assign and got.total_weight == exp_total
    w = [[float(i % 3)] for i in range(300)]
    exp_assign, exp_total = port.km_flat(w, 300, 1)
    got = sk.km_match(graph_of(w))
    assert cols_of(got, 300) == exp_assign and got.total_weight == exp_total


@pytest.mark.parametrize("n,kind", [(257, "tie"), (600, "tie"), (1100, "tie"), (1500, "int"),
                                    (2600, "tie")])
def test_large_outer_km_vs_c_oracle(n, kind):
    rng = np.random.default_rng(n)
    w = (rng.integers(0, 3, size=(n, n)) if kind == "tie"
         else rng.integers(0, 10**6, size=(n, n))).astype(np.float64)
    exp = cport.hungarian(w)
    got = sk.km_match(graph_of(w.tolist()))
    assert cols_of(got, n) == exp
    total = 0.0
    for i, j in enumerate(exp):
        total += w[i, j]
    assert got.total_weight == total


@pytest.mark.parametrize("shapes,G,n_pos", [(((2, 3), (4, 3), (1, 6)), 3, 48),
                                            (((2, 3), (2, 6), (3, 2)), 1, 24)])
def test_non_dyadic_sweep_vs_c_oracle(shapes, G, n_pos):
    b = sweep.make_sweep(n_pos, 3, seed=11, G=G, shapes=shapes)
    assert (b.plans["K"] % 3 == 0).any()
    assign, totals = sweep.SweepRunner(b).run()
    exp_assign, exp_totals = cport.map_sweep(b.desc, b.plans, b.alive, b.tok)
    assert np.array_equal(assign, exp_assign)
    assert [t.hex() for t in totals] == [t.hex() for t in exp_totals]


def test_fused_sum_sweep_at_256_vs_c_oracle():
    b = sweep.make_sweep(256, 2, seed=13, fused_sum=True)
    assign, totals = sweep.SweepRunner(b).run()
    exp_assign, exp_totals = cport.map_sweep(b.desc, b.plans, b.alive, b.tok)
    assert np.array_equal(assign, exp_assign)
    assert [t.hex() for t in totals] == [t.hex() for t in exp_totals]
