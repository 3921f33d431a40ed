"""Multi-GPU reshard correctness check (one process per GPU under torchrun):
plan a transition with this package's mapper + planner, execute it across the
ranks' GPUs over NVLink (pull and push, one persistent k_exec launch per rank)
and verify every new shard is byte-identical to the regenerated pattern.
Exit code 0 = all identical and every run completed its rounds.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
      tools/reshard_check.py
"""

import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2311_15566_b200 import reshard  # noqa: E402

SMALL = ("toy-bf16", 8, 8 * 1024 * 64, 1024)
CASES = {2: [((1, 2, 1), (2, 1, 1)), ((2, 1, 1), (1, 2, 1))],
         4: [((1, 2, 2), (1, 1, 4)), ((1, 4, 1), (2, 1, 2))],
         8: [((1, 2, 4), (2, 1, 4)), ((1, 4, 2), (1, 2, 4))]}


def main():
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    bad_total = 0
    cases = list(CASES.get(world, CASES[2]))
    if world in (2, 4):
        cases += CASES[8]  # 8 GPU refs hosted 2 or 4 per rank: the 8-GPU transitions
    for old, new in cases:
        for u_max in (None, 2.0e5):
            plan, layout, need, model, refs = reshard.make_reshard_problem(SMALL, old, new, 3, 64, u_max=u_max)
            owner = {g: i * world // len(refs) for i, g in enumerate(refs)}
            for mode in ("pull", "push"):
                ex = reshard.ReshardExecutor(plan, layout, need, model, owner, rank, world, mode=mode)
                ex.fill_old()
                torch.cuda.synchronize()
                dist.barrier()
                ex.run()
                torch.cuda.synchronize()
                dist.barrier()
                ctl = ex.control()
                bad = torch.tensor([float(ex.verify()), float(ctl["error"] != 0)], device="cuda")
                dist.all_reduce(bad)
                bad_total += int(bad[0].item()) + int(bad[1].item())
                if rank == 0:
                    print(f"{old}->{new} u_max={u_max} {mode}: mismatched words {int(bad[0].item())}, "
                          f"errors {int(bad[1].item())}", flush=True)
                ex.close()
    dist.destroy_process_group()
    sys.exit(1 if bad_total else 0)


if __name__ == "__main__":
    main()
