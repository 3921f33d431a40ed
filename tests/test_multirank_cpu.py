"""N>1 host logic on CPU with world_size-2 gloo process groups:
* reshard issue lists: every copy issued exactly once across ranks, by the
  destination (pull) or the source (push), local copies by the owner;
* the bench's weak-scaling reductions (max of times, sum of plans) and
  per-rank sweep sharding (distinct plan batches per rank)."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_15566_b200 import reshard

SMALL = ("toy-bf16", 8, 8 * 1024 * 64, 1024)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2311_15566_b200 import sweep

        res = {}
        # weak-scaling reductions (gloo, CPU tensors)
        import torch

        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res["max"] = float(t.item())
        t2 = torch.tensor([10.0 * (rank + 1)])
        dist.all_reduce(t2, op=dist.ReduceOp.SUM)
        res["sum"] = float(t2.item())
        b = sweep.make_sweep(16, 1, seed=1000 + rank)
        got = [None] * world
        dist.all_gather_object(got, b.alive.tolist())
        res["distinct"] = got[0] != got[1]
        _ = bench
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_gloo_weak_scaling_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0]["max"] == out[1]["max"] == 2.0
    assert out[0]["sum"] == 30.0
    assert out[0]["distinct"]


def test_issue_lists_partition_every_copy_once():
    """plan -> copies -> issuer partition, pure host logic (no device memory)."""
    from fractions import Fraction

    import paper_2311_15566_b200 as sk
    from paper_2311_15566_b200 import domain as dm

    # a 4-GPU (1,2,2)->(1,1,4) plan built from the oracle-free host pieces:
    model = dm.ModelSpec("toy", 8, 8 * 1024 * 64, 1024)
    old = dm.ParallelConfig(1, 2, 2, 1)
    new = dm.ParallelConfig(1, 1, 4, 1)
    layout = {}
    for k, pos in enumerate(dm.positions(old)):
        layout[(f"i-{k}", 0)] = dm.required_context(old, pos, model)
    assignment = {(f"i-{k}", 0): pos for k, pos in enumerate(dm.positions(new))}
    mapping = sk.DeviceMapping(assignment=assignment, total_weight=0.0, config=new)
    plan = sk.plan_migration(mapping, layout, model)
    need = reshard.required_layout(mapping, model, None, dm.ContextInventory)
    _, _, copies = reshard.plan_copies(plan, layout, need, model)
    owner = {g: i for i, g in enumerate(sorted(layout))}
    for mode in ("pull", "push"):
        lists = reshard.issue_lists(copies, owner, mode)
        flat = sorted(c for lst in lists.values() for c in lst)
        expect = sorted((src, dst, so, do, n) for dst, lst in copies.items() for src, so, do, n in lst)
        assert flat == expect
        for rank, lst in lists.items():
            for src, dst, *_ in lst:
                who = dst if (mode == "pull" or src == dst) else src
                assert owner[who] == rank
    bin_, bout = reshard.traffic(plan)
    assert sum(bin_.values()) == sum(bout.values()) > 0
    assert all(isinstance(t.lo, Fraction) for t in plan.transfers())
