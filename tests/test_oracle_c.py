"""Pin the C oracle (oracle/spotkm_oracle.c) to the Python port (itself
pinned to the reference goldens) on sweep plans, bit for bit.  CPU only."""

import numpy as np
import pytest

from oracle import cport, port
from oracle.sweep_inputs import plan_to_port

from paper_2311_15566_b200 import sweep


@pytest.mark.parametrize("n_pos,fused_sum,shapes,G", [
    (16, False, sweep.GPT20B_SHAPES, 4), (32, False, sweep.GPT20B_SHAPES, 4),
    (24, True, sweep.GPT20B_SHAPES, 4), (48, False, ((2, 3), (4, 3), (1, 6)), 3),
    (24, True, ((2, 3), (2, 6), (3, 2)), 1)])
def test_c_oracle_matches_port_on_sweep(n_pos, fused_sum, shapes, G):
    cport.build()
    b = sweep.make_sweep(n_pos, 2, seed=n_pos, fused_sum=fused_sum, shapes=shapes, G=G)
    assign, totals = cport.map_sweep(b.desc, b.plans, b.alive, b.tok, n_threads=4)
    for q in range(b.n_plans):
        inst, new, G, inh, reqs, fw = plan_to_port(b, q, sweep.GPT20B, n_requests=1 + q % 3)
        _, _, _, exp_assign, exp_total = port.map_devices(inst, new, sweep.GPT20B, G, inh, reqs, fw)
        o = int(b.plans["out_off"][q])
        R = int(b.plans["rows"][q])
        assert assign[o:o + R].tolist() == exp_assign, q
        assert totals[q].hex() == exp_total.hex(), q


def test_c_hungarian_matches_port():
    rng = np.random.default_rng(1)
    for n in (1, 2, 5, 9, 40):
        w = rng.integers(0, 3, size=(n, n)).astype(float)
        assert cport.hungarian(w) == port.hungarian_max(w.tolist())
