"""Migration executor (K3) on one GPU: every GPU of the plan emulated on the
local device (same plan -> copy-list -> k_copy -> verify path as the
multi-GPU run; peers are local pointers).  Resharded bytes must be identical
to the regenerated pattern of the new layout."""

import pytest

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
