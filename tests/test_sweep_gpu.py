"""GPU parity at BASELINE.json's sweep sizes (64..1024 positions): the device
(sk_sweep_expand + sk_map_fuse + sk_map_outer) vs the C oracle (itself pinned
to the Python port and the reference goldens) -- bit-exact assignments and
total_weight for every plan of every (old, new) config pair."""

import numpy as np
import pytest

from oracle import cport

from paper_2311_15566_b200 import sweep

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_pos,sets,fused_sum,model", [
    (64, 4, False, "gpt-20b"), (128, 2, False, "gpt-20b"), (256, 2, False, "gpt-20b"),
    (512, 1, False, "gpt-20b"), (1024, 1, False, "gpt-20b"), (128, 2, True, "gpt-20b"),
    (256, 1, False, "llama-30b"), (64, 2, False, "opt-6.7b"), (256, 1, True, "gpt-20b"),
    (256, 1, False, "opt-6.7b"),
])
def test_sweep_matches_c_oracle(n_pos, sets, fused_sum, model):
    geom, shapes = sweep.MODELS[model]
    b = sweep.make_sweep(n_pos, sets, seed=7 + n_pos, model=geom, shapes=shapes,
                         fused_sum=fused_sum)
    r = sweep.SweepRunner(b)
    assign, totals = r.run()
    exp_assign, exp_totals = cport.map_sweep(b.desc, b.plans, b.alive, b.tok)
    assert np.array_equal(assign, exp_assign)
    assert [t.hex() for t in totals] == [t.hex() for t in exp_totals]
    # every target position is covered exactly once when enough GPUs are alive
    for q in range(b.n_plans):
        o, R = int(b.plans["out_off"][q]), int(b.plans["rows"][q])
        C = int(b.plans["D"][q] * b.plans["P"][q] * b.plans["M"][q])
        cols = assign[o:o + R]
        got = np.sort(cols[cols >= 0])
        assert np.array_equal(got, np.arange(C)), q


def test_steps_counter_and_repeatability():
    import torch

    b = sweep.make_sweep(128, 2, seed=3)
    r = sweep.SweepRunner(b)
    a1, t1 = r.run()
    steps = torch.zeros(2 * b.n_plans, dtype=torch.int64, device="cuda")
    # k_fuse writes every fused element itself: stale scratch must not matter
    r.fused.fill_(float("nan"))
    r.perm.fill_(-1)
    r.upload()
    r.solve(steps=steps)
    r.download()
    torch.cuda.synchronize()
    a2, t2 = r.results()
    assert np.array_equal(a1, a2) and np.array_equal(t1, t2)
    s = steps.cpu().numpy().reshape(-1, 2)
    n = b.stats()["n"]
    assert (s[:, 0] >= n).all()            # at least one Dijkstra step per row


def test_chunks_sharing_scratch_match_c_oracle():
    """A sweep run as consecutive chunks on one device scratch (bench.py's
    all-sizes mode): every chunk still equals the oracle, run interleaved."""
    import torch

    bs = [sweep.make_sweep(256, 1 + c, seed=40 + c) for c in range(3)]
    cap = (max(b.rows for b in bs), max(int(b.stats()["pairs"].sum()) for b in bs))
    runs = []
    for b in bs:
        runs.append(sweep.SweepRunner(b, scratch=runs[0] if runs else None, reserve=cap))
    assert all(r.fused is runs[0].fused and r.segs is runs[0].segs for r in runs)
    for r in runs:
        r.upload()
    for r in runs:
        r.solve()
    for r in runs:
        r.download()
    torch.cuda.synchronize()
    for r, b in zip(runs, bs):
        assign, totals = r.results()
        exp_assign, exp_totals = cport.map_sweep(b.desc, b.plans, b.alive, b.tok)
        assert np.array_equal(assign, exp_assign)
        assert [t.hex() for t in totals] == [t.hex() for t in exp_totals]


def test_global_code_mode_matches_c_oracle():
    """A size class big enough (n ~ 130, > 2 waves) that the outer KM keeps its
    dictionary codes in the global scratch instead of shared memory."""
    b = sweep.make_sweep(256, 2600, seed=21, shapes=((6, 2), (2, 8)))
    r = sweep.SweepRunner(b)
    assert any(x > 0 for x in r.codes_need)
    assign, totals = r.run()
    exp_assign, exp_totals = cport.map_sweep(b.desc, b.plans, b.alive, b.tok)
    assert np.array_equal(assign, exp_assign)
    assert [t.hex() for t in totals] == [t.hex() for t in exp_totals]


@pytest.mark.parametrize("n_pos", [128, 512])
def test_forced_global_codes_all_shapes_match_c_oracle(n_pos):
    """Every size class (1-, 2- and 4-warp shapes) in the global-code mode,
    forced with SK_OUTER_FORCE_GLOBAL in a subprocess (the mode is chosen per
    launch from the class size, so small test batches would not reach it)."""
    import os
    import subprocess
    import sys

    code = (
        "import numpy as np\n"
        "from oracle import cport\n"
        "from paper_2311_15566_b200 import sweep\n"
        f"b = sweep.make_sweep({n_pos}, 2, seed=41)\n"
        "r = sweep.SweepRunner(b)\n"
        "assert all(x > 0 for x in r.codes_need), r.codes_need\n"
        "assign, totals = r.run()\n"
        "ea, et = cport.map_sweep(b.desc, b.plans, b.alive, b.tok)\n"
        "assert np.array_equal(assign, ea)\n"
        "assert [t.hex() for t in totals] == [t.hex() for t in et]\n"
        "print('ok', b.n_plans)\n")
    env = dict(os.environ, SK_OUTER_FORCE_GLOBAL="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                         text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    assert res.stdout.startswith("ok")


def test_coded_fuse_overflow_and_stale_scratch():
    """k_fuse codes the fused matrix itself (sk_map_fuse_coded): plans with
    more than 255 distinct fused values overflow their dictionary and take the
    double-matrix path; stale code / dictionary scratch must not matter."""
    import torch

    b = sweep.make_sweep(1024, 1, seed=5)   # plan 0 has ~400 distinct fused values
    r = sweep.SweepRunner(b)
    assert all(r.class_coded)
    a1, t1 = r.run()
    exp_assign, exp_totals = cport.map_sweep(b.desc, b.plans, b.alive, b.tok)
    assert np.array_equal(a1, exp_assign)
    assert [t.hex() for t in t1] == [t.hex() for t in exp_totals]
    d = r.dict.cpu().numpy()
    flags = np.concatenate([d[r.dict_off[c] // 8:r.dict_off[c] // 8 + 256 * (hi - lo):256]
                            for c, (lo, hi, _) in enumerate(r.classes)])
    assert len(flags) == b.n_plans
    assert (flags != -1).sum() >= 1          # some plan overflowed ...
    assert (flags == -1).sum() >= 1          # ... and some stayed coded
    r.codes.fill_(0x5A)
    r.dict.fill_(123)
    r.fused.fill_(float("nan"))
    r.perm.fill_(-1)
    r.upload()
    r.solve(download=True)
    torch.cuda.synchronize()
    a2, t2 = r.results()
    assert np.array_equal(a1, a2) and [t.hex() for t in t1] == [t.hex() for t in t2]


@pytest.mark.parametrize("n_pos,fused_sum", [(64, False), (128, False), (128, True)])
def test_coded_path_forced_at_small_sizes(monkeypatch, n_pos, fused_sum):
    """The coded K2 runs by default from n >= 96; forced on, the small sweeps
    must give the same bits as the C oracle too."""
    monkeypatch.setenv("SK_PRECODED", "1")
    b = sweep.make_sweep(n_pos, 2, seed=11 + n_pos, fused_sum=fused_sum)
    r = sweep.SweepRunner(b)
    assert all(r.class_coded)
    assign, totals = r.run()
    exp_assign, exp_totals = cport.map_sweep(b.desc, b.plans, b.alive, b.tok)
    assert np.array_equal(assign, exp_assign)
    assert [t.hex() for t in totals] == [t.hex() for t in exp_totals]
