"""Tune the executor's copy geometry on real GPUs (torchrun, one process per GPU):
chunk size x CTAs per launch, push and pull, on the bench's reshard case."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_15566_b200 import reshard  # noqa: E402


def main():
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    geom = reshard.LLAMA30B_BF16 if world <= 4 else reshard.GPT20B_BF16
    old, new = {2: ((1, 2, 1), (2, 1, 1)), 4: ((1, 2, 2), (1, 1, 4))}.get(world, ((1, 2, 4), (2, 1, 4)))
    plan, layout, need, model, refs = reshard.make_reshard_problem(geom, old, new, 8, 2048)
    owner = {g: i for i, g in enumerate(refs)}
    bin_, bout = reshard.traffic(plan)
    peak = max(max(bin_.values()), max(bout.values()))
    res = []
    for mode in ("push", "pull"):
        ex = reshard.ReshardExecutor(plan, layout, need, model, owner, rank, world, mode=mode)
        ex.fill_old()
        for chunk in (1 << 18, 1 << 20, 1 << 22):
            ex.set_chunk(chunk)
            for ctas in (148, 296, 592, 1184):
                ts = []
                for it in range(4):
                    dist.barrier()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    ex.run(ctas)
                    e1.record()
                    e1.synchronize()
                    t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    if it:
                        ts.append(float(t.item()))
                ms = min(ts)
                res.append({"mode": mode, "chunk": chunk, "ctas": ctas, "ms": ms,
                            "gbs": peak / ms / 1e6})
        ex.close()
    if rank == 0:
        for r in sorted(res, key=lambda r: r["ms"]):
            print(json.dumps(r))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
