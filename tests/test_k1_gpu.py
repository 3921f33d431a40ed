"""K1 (k_weights, the dense build_graph weights) on headline sweep plans vs an
exact numpy restatement of the closed form (pack.py docstring; overlap_bytes
domain.py:299-320) over the same device-expanded segments: bit-exact.  The
drop-in build_graph itself is pinned to the reference's W in
test_mapping_gpu.py / test_range_gpu.py."""

from fractions import Fraction

import numpy as np
import pytest
import torch

from paper_2311_15566_b200 import _native as nat
from paper_2311_15566_b200 import sweep

pytestmark = pytest.mark.gpu


def exact_w(plan, rp, segs):
    D, P, M, L, K = (int(plan[k]) for k in ("D", "P", "M", "L", "K"))
    C = D * P * M
    c = np.arange(C)
    m, t = c % M, c // M
    st, d = t % P, t // P + 1
    q, r = divmod(L, P)
    s0 = st * q + np.minimum(st, r)
    s1 = s0 + q + (st < r)
    w = K // M
    i0, i1 = m * w, m * w + w
    R = len(rp) - 1
    out = np.zeros((R, C), dtype=object)
    for row in range(R):
        acc = np.zeros(C, dtype=object)
        for sg in segs[rp[row]:rp[row + 1]]:
            ol = np.minimum(int(sg["l1"]), s1) - np.maximum(int(sg["l0"]), s0)
            oi = np.minimum(int(sg["b"]), i1) - np.maximum(int(sg["a"]), i0)
            ok = (ol > 0) & (oi > 0) & ((int(sg["pipe"]) == 0) | (int(sg["pipe"]) == d))
            acc = acc + np.where(ok, ol.astype(object) * oi.astype(object) * int(sg["unit"]), 0)
        out[row] = [float(Fraction(int(x), K)) for x in acc]
    return out.astype(np.float64)


@pytest.mark.parametrize("n_pos,sets", [(64, 2), (256, 1), (1024, 1)])
def test_k1_matches_exact_closed_form(n_pos, sets):
    b = sweep.make_sweep(n_pos, sets, seed=31)
    r = sweep.SweepRunner(b)
    r.run()
    st = b.stats()
    RC = (st["rows"] * st["cols"]).astype(np.int64)
    plans = b.plans.copy()
    plans["f_off"] = np.concatenate([[0], np.cumsum(RC)[:-1]])
    d_plans = torch.from_numpy(plans.view(np.uint8)).cuda()
    W = torch.full((int(RC.sum()),), -1.0, dtype=torch.float64, device="cuda")
    nat.check(nat.load().sk_build_weights(d_plans.data_ptr(), b.n_plans, r.row_ptr.data_ptr(),
                                          r.segs.data_ptr(), W.data_ptr(), int(st["rows"].max()),
                                          int(st["cols"].max()), torch.cuda.current_stream().cuda_stream))
    Wh = W.cpu().numpy()
    rp_all = r.row_ptr.cpu().numpy()
    seg_all = r.segs.cpu().numpy().view(nat.SEGMENT)
    # every 6th plan plus the first plan of each (D, P, M) shape: shard counts
    # that are and are not multiples of 4 take different column loops in k_weights
    qs = set(range(0, b.n_plans, max(1, b.n_plans // 6)))
    shapes = np.stack([plans["D"], plans["P"], plans["M"]], axis=1)
    qs |= set(np.unique(shapes, axis=0, return_index=True)[1].tolist())
    assert {2, 4} <= set(plans["M"].tolist())
    for q in sorted(qs):
        R, C = int(st["rows"][q]), int(st["cols"][q])
        base = int(plans["row_base"][q])
        rp = rp_all[base:base + R + 1]
        exp = exact_w(plans[q], rp - 0, seg_all)
        got = Wh[int(plans["f_off"][q]):int(plans["f_off"][q]) + R * C].reshape(R, C)
        assert np.array_equal(got.view(np.int64), exp.view(np.int64)), q
