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


def _reshard_worker(rank, world, port, q):
    """One rank of the executor's host protocol with MOCKED device memory:
    slab offsets, the all-gathered (handle, arena offsets) exchange and the
    peer mapping (opener decodes a fake 'handle' into a fake base address),
    then this rank's pull / push issue lists and send/recv ops."""
    import sys

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path[:0] = [os.path.join(os.path.dirname(__file__)), os.path.join(os.path.dirname(__file__), "golden")]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from helpers import port_mapper

        plan, layout, need, model, refs = reshard.make_reshard_problem(SMALL, (1, 2, 2), (1, 1, 4), 3, 64,
                                                                       u_max=2.0e5, mapper=port_mapper)
        L = reshard.ArenaLayout(plan, layout, need, model)
        owner = {g: i * world // len(refs) for i, g in enumerate(refs)}
        ref_off, size = reshard.slab_offsets(L, owner, rank, 4096)
        fake = (rank + 1) << 40                       # this rank's mocked slab address
        handle = fake.to_bytes(8, "little") + bytes(56)  # a 64-byte mocked IPC handle
        base, ctl, opened = reshard.exchange_slabs(rank, world, fake, handle, ref_off,
                                                   lambda h: int.from_bytes(h[:8], "little"))

        def where(ptr):   # (owning rank, offset) of an address
            return (ptr >> 40) - 1, ptr & ((1 << 40) - 1)

        res = {"size": size, "opened": len(opened), "ctl": sorted(ctl),
               "own": {str(g): o for g, o in ref_off.items()}}
        for mode in ("pull", "push"):
            lst = reshard.issue_list(L, owner, rank, mode, base)
            res[mode] = [(ri, where(s), where(d), n, w, str(t.src), str(t.dst)) for ri, s, d, n, w, t in lst]
        ops = reshard.p2p_ops(L, owner, rank, {g: fake + o for g, o in ref_off.items()})
        res["ops"] = [(k, peer, n) for k, peer, ptr, n in ops]
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_gloo_executor_protocol_two_ranks():
    """Two real processes run the executor's host protocol (handle exchange,
    peer mapping, issue partition, send/recv pairing) with mocked handles:
    every transfer extent is issued exactly once, by its destination's rank
    (pull) or its source's (push), the addresses resolve into the right
    rank's slab at the right arena offset, and every send has its recv."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_reshard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        assert out[r]["opened"] == 1 and out[r]["ctl"] == [0, 1]
    for mode in ("pull", "push"):
        both = out[0][mode] + out[1][mode]
        # a transfer extent is identified by (round, src address, dst address)
        keys = [(ri, s, d) for ri, s, d, *_ in both]
        assert len(keys) == len(set(keys)) > 0
        for r in (0, 1):
            for ri, (sr, so), (dr, do), n, w, src, dst in out[r][mode]:
                assert (dr if mode == "pull" else sr) == r
                assert so >= out[sr]["own"][src] and do >= out[dr]["own"][dst]
        # both ranks issue the same plan, split
        assert sorted(keys) == sorted({k for k in keys})
    pull = sorted((ri, s, d, n) for ri, s, d, n, *_ in out[0]["pull"] + out[1]["pull"])
    push = sorted((ri, s, d, n) for ri, s, d, n, *_ in out[0]["push"] + out[1]["push"])
    assert pull == push                        # the same copies, issued from the other side
    sends = [(n,) for k, peer, n in out[0]["ops"] if k == "send" and peer == 1]
    recvs = [(n,) for k, peer, n in out[1]["ops"] if k == "recv" and peer == 0]
    assert sends == recvs and sends           # pairwise in order and size
    sends = [(n,) for k, peer, n in out[1]["ops"] if k == "send" and peer == 0]
    recvs = [(n,) for k, peer, n in out[0]["ops"] if k == "recv" and peer == 1]
    assert sends == recvs
