"""Migration executor (K3) on one GPU: every GPU of the plan emulated on the
local device (same plan -> copy-list -> k_copy -> verify path as the
multi-GPU run; peers are local pointers).  Resharded bytes must be identical
to the regenerated pattern of the new layout."""

import pytest
import torch

from paper_2311_15566_b200 import reshard

pytestmark = pytest.mark.gpu

SMALL = ("toy-bf16", 8, 8 * 1024 * 64, 1024)


@pytest.mark.parametrize("mode", ["pull", "push"])
@pytest.mark.parametrize("old,new", [((1, 2, 2), (1, 1, 4)), ((1, 2, 4), (2, 1, 4)),
                                     ((1, 4, 2), (1, 2, 4)), ((2, 2, 1), (1, 2, 2)),
                                     ((1, 2, 1), (2, 1, 1))])
def test_reshard_byte_identical(old, new, mode):
    plan, layout, need, model, refs = reshard.make_reshard_problem(SMALL, old, new, batch=3, seq=64)
    owner = {g: 0 for g in set(layout) | set(need)}
    ex = reshard.ReshardExecutor(plan, layout, need, model, owner, mode=mode)
    try:
        ex.fill_old()
        assert ex.verify() > 0 or ex.remote_bytes == 0   # new slabs start empty
        ex.run()
        assert ex.verify() == 0
        bin_, bout = reshard.traffic(plan)
        assert ex.remote_bytes == sum(bin_.values())
    finally:
        ex.close()


def test_progressive_rounds_and_stage_events():
    plan, layout, need, model, refs = reshard.make_reshard_problem(SMALL, (1, 4, 2), (1, 2, 4),
                                                                   batch=2, seq=64)
    owner = {g: 0 for g in set(layout) | set(need)}
    ex = reshard.ReshardExecutor(plan, layout, need, model, owner)
    try:
        ex.fill_old()
        ready = ex.run_progressive()
        torch.cuda.synchronize()
        stages = {a.stage for a in plan.actions if a.kind == "start_stage"}
        assert set(ready) == stages
        times = {s: ex.progress_begin.elapsed_time(ev) for s, ev in ready.items()}
        assert all(t >= 0 for t in times.values())
        assert ex.verify() == 0
    finally:
        ex.close()


def test_executor_ingests_the_json_wire_plan():
    """The paper ships plans as JSON over TCP; the executor
    runs a plan that went through plan_to_dict -> json -> plan_from_dict."""
    import json

    from paper_2311_15566_b200 import planner

    plan, layout, need, model, refs = reshard.make_reshard_problem(SMALL, (1, 2, 4), (2, 1, 4),
                                                                   batch=2, seq=64)
    wire = json.loads(json.dumps(planner.plan_to_dict(plan)))
    back = planner.plan_from_dict(wire)
    assert planner.plan_to_dict(back) == planner.plan_to_dict(plan)
    owner = {g: 0 for g in set(layout) | set(need)}
    ex = reshard.ReshardExecutor(back, layout, need, model, owner, mode="push")
    try:
        ex.fill_old()
        ex.run()
        assert ex.verify() == 0
    finally:
        ex.close()
