"""Host side of the plan-ordered executor (reshard.ArenaLayout): where every
byte of the old and new contexts lives, which arena space each received
transfer recycles, and the memory high-water mark -- checked on the
BASELINE.json reshard geometries (GPT-20B / LLaMA-30B bf16, KV batch 8 x seq
2048) without a GPU (the mapping comes from the CPU oracle, the plan from the
native planner).  The arena must free exactly the plan's `releases`
(migration.py:283-305), never hand out live bytes, and peak at the plan's
`peak_usage` (simulate_buffer_usage, migration.py:387-401) above the old
footprint."""

from fractions import Fraction

import pytest

from helpers import port_mapper

from paper_2311_15566_b200 import reshard
from paper_2311_15566_b200.reshard import ALIGN, Arena

SMALL = ("toy-bf16", 8, 8 * 1024 * 64, 1024)
CASES = [(reshard.GPT20B_BF16, (1, 2, 4), (2, 1, 4)), (reshard.GPT20B_BF16, (1, 4, 2), (1, 2, 4)),
         (reshard.LLAMA30B_BF16, (1, 4, 2), (1, 2, 4)), (reshard.LLAMA30B_BF16, (1, 2, 1), (2, 1, 1)),
         (reshard.LLAMA30B_BF16, (1, 2, 2), (1, 1, 4)), (SMALL, (2, 2, 1), (1, 2, 2)),
         (SMALL, (1, 2, 2), (1, 1, 4))]


def test_arena_first_fit_scatter_and_wait_rounds():
    a = Arena()
    x = a.alloc_top(1000)
    y = a.alloc_top(5000)
    z = a.alloc_top(3000)
    assert (x, y, z) == (0, 1024, 6144) and a.high == 9144
    a.release(y, 5000, 3)
    # fits in the hole: one extent, recycles round 3
    assert a.alloc(4096) == [(1024, 4096, 3)]
    # too big for any hole: fresh space at the top, no wait
    ext = a.alloc(200 << 10)
    assert len(ext) == 1 and ext[0][2] == -1 and ext[0][0] >= 9144
    # two holes from different rounds, neither big enough alone: scattered
    b = Arena()
    offs = [b.alloc_top(128 << 10) for _ in range(4)]
    b.release(offs[0], 128 << 10, 1)
    b.release(offs[2], 128 << 10, 5)
    ext = b.alloc(200 << 10)
    assert sum(n for _, n, _ in ext) == 200 << 10 and len(ext) == 2
    assert {w for _, _, w in ext} == {1, 5} and b.high == 4 * (128 << 10)


def _replay(L):
    """independent replay: live byte ranges per GPU never overlap, releases
    free live bytes only, and recycled space is waited for"""
    for g, gl in L.gpus.items():
        live = []   # (start, end, round freed or None)
        for reg in gl.old:
            live.append([reg.off, reg.off + reg.byte_range(reg.lo, reg.hi)[1]])
        freed = []  # (start, end, round)
        for ri, action in enumerate(L.rounds):
            for t in action.transfers:
                if t.dst != g:
                    continue
                for off, n, w in gl.incoming[id(t)]:
                    assert off % ALIGN == 0
                    for s, e in live:
                        assert off + n <= s or off >= e, (g, ri, "overlaps live bytes")
                    need = max((r for s, e, r in freed if off < e and s < off + n), default=-1)
                    assert w >= need, (g, ri, w, need)
                    live.append([off, off + n])
            for reg in gl.old:
                for rr, lo, hi in reg.released:
                    if rr != ri:
                        continue
                    s, n = reg.byte_range(lo, hi)
                    # carve [s, s+n) out of the live set
                    nxt = []
                    hit = 0
                    for a, b in live:
                        if b <= s or a >= s + n:
                            nxt.append([a, b])
                            continue
                        hit += min(b, s + n) - max(a, s)
                        if a < s:
                            nxt.append([a, s])
                        if b > s + n:
                            nxt.append([s + n, b])
                    assert hit == n, "released bytes were not live"
                    live = nxt
                    freed.append((s, s + n, ri))


@pytest.mark.parametrize("geom,old,new", CASES)
def test_arena_layout_follows_the_plan(geom, old, new):
    plan, layout, need, model, refs = reshard.make_reshard_problem(geom, old, new, 8, 2048,
                                                                   mapper=port_mapper)
    L = reshard.ArenaLayout(plan, layout, need, model)
    L.check_releases()          # frees exactly the plan's releases, round by round
    _replay(L)
    rep = L.memory_report()
    for inst, d in rep.items():
        # high-water == old context + the plan's peak migration buffers
        # (alignment only: 256 B per piece)
        bound = d["plan_bound_bytes"]
        assert d["arena_bytes"] >= bound - 1
        assert d["arena_bytes"] <= bound * 1.001 + 4096 * ALIGN, (inst, d)
    # every required shard is covered: kept pieces stay where they were
    for g, gl in L.gpus.items():
        kept = [p for p in gl.pieces if any(p[5] >= r.off and p[0] == r.key for r in gl.old)]
        assert all(isinstance(p[1], Fraction) for p in gl.pieces)
        assert len(kept) <= len(gl.pieces)


def test_memopt_order_changes_the_arena_peak():
    """U_max reorders the layer rounds (memopt_layer_order, migration.py:114-143):
    the arena peak follows whichever order the plan ships."""
    geom, old, new = reshard.GPT20B_BF16, (1, 2, 4), (2, 1, 4)
    peaks = {}
    for u in (None, 4e9, 1e9):
        plan, layout, need, model, refs = reshard.make_reshard_problem(geom, old, new, 8, 2048, u_max=u,
                                                                       mapper=port_mapper)
        L = reshard.ArenaLayout(plan, layout, need, model)
        rep = L.memory_report()
        peaks[u] = max(d["arena_bytes"] - d["old_bytes"] for d in rep.values())
        assert abs(peaks[u] - max(plan.peak_usage.values())) <= 0.001 * peaks[u] + 4096 * ALIGN
    assert peaks[4e9] <= peaks[None]


def test_daemon_wire_format_roundtrip():
    """The context daemon's request (plan_to_dict + layouts + mapping, JSON)
    decodes to the same plan and inventories (paper_2311_15566_b200/daemon.py)."""
    import json

    from paper_2311_15566_b200 import daemon, planner

    plan, layout, need, model, refs, mapping = reshard.make_reshard_problem(
        SMALL, (1, 2, 2), (1, 1, 4), 3, 64, mapper=port_mapper, with_mapping=True)
    req = json.loads(json.dumps(daemon.migrate_request(plan, layout, need, model, mapping.assignment)))
    assert planner.plan_to_dict(planner.plan_from_dict(req["plan"])) == planner.plan_to_dict(plan)
    assert {(i, g): daemon.dec_inv(v) for i, g, v in req["old"]} == layout
    assert {(i, g): daemon.dec_inv(v) for i, g, v in req["new"]} == need
    assert len(req["assignment"]) == len(mapping.assignment)
