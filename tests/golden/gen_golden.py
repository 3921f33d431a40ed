"""Generate golden vectors by running the REAL reference (`spotsim`).

Run in the build container only (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

Writes `tests/golden/{km,mapping,scenario,plans}.json.gz`.  Every case stores
its inputs in plain JSON (rationals as [num, den]) and the reference outputs
with floats as `float.hex()`, so the oracle and the CUDA path are pinned
bit-for-bit.  `meta.python` records the interpreter that produced them
(builtin `sum` is compensated from Python 3.12 on; see SURVEY.md finding 6).
"""

from __future__ import annotations

import itertools
import sys
from dataclasses import replace
from fractions import Fraction
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
from fmt import enc_inv, hx, save  # noqa: E402

import spotsim  # noqa: E402
from spotsim import costmodel as ref_cost  # noqa: E402
from spotsim import mapping as ref_map  # noqa: E402
from spotsim import migration as ref_mig  # noqa: E402
from spotsim import simulator as ref_sim  # noqa: E402
from spotsim.data import bundled_path  # noqa: E402
from spotsim.domain import (  # noqa: E402
    ContextInventory,
    InstanceState,
    ModelSpec,
    ParallelConfig,
    RequestSpec,
    TopologyPosition,
    positions,
    required_context,
)
from spotsim.simconfig import load_simconfig  # noqa: E402

META = {"python": sys.version, "spotsim": spotsim.__version__}


# ---------------------------------------------------------------------------
# helpers

def graph_of(weights):
    gpus = [(f"i-{k}", 0) for k in range(len(weights))]
    slots = [TopologyPosition(1, 1, m + 1) for m in range(len(weights[0]))] if weights else []
    return ref_map.BipartiteGraph(gpus=gpus, slots=slots, weights=[list(r) for r in weights])


def enc_instances(instances):
    return [[inst.id, [enc_inv(inv.model_shards, inv.cache_shards) for inv in inst.gpu_inventories]]
            for inst in instances]


def enc_mapping_result(graph_gpus, slots, mapping):
    col = {s: j for j, s in enumerate(slots)}
    return [col[mapping.assignment[g]] if g in mapping.assignment else -1 for g in graph_gpus]


def reqs_of(tokens_by_pipe):
    """{d_old: [(rid, tokens)]} -> RequestSpec lists (tokens = s_in + generated)."""
    out = {}
    for d, lst in tokens_by_pipe.items():
        out[d] = [RequestSpec(id=rid, arrival_time=0.0, s_in=tok, s_out=max(tok, 1),
                              tokens_generated=0) for rid, tok in lst]
    return out


def run_map_case(model, target, G, instances, inheritance, tokens_by_pipe, fused_weight="max",
                 want_w=True):
    reqs = reqs_of(tokens_by_pipe) if tokens_by_pipe is not None else None
    case = {
        "model": [model.num_layers, model.bytes_per_layer, model.kv_bytes_per_token_per_layer],
        "target": list(target.shape()),
        "G": G,
        "fused_weight": fused_weight,
        "instances": enc_instances(instances),
        "inheritance": None if inheritance is None else {str(k): v for k, v in inheritance.items()},
        "reqs": None if tokens_by_pipe is None else
        {str(d): [[rid, tok] for rid, tok in lst] for d, lst in tokens_by_pipe.items()},
    }
    graph = ref_map.build_graph(instances, target, model, inheritance, reqs)
    if want_w:
        case["W"] = [[hx(w) for w in row] for row in graph.weights]
    try:
        m = ref_map.map_devices(instances, target, model, G, inheritance=inheritance,
                                requests_by_old_pipeline=reqs, fused_weight=fused_weight)
    except ref_map.MappingError as e:
        case["error"] = "MappingError"
        case["message"] = str(e)
        return case
    case["error"] = None
    case["assign"] = enc_mapping_result(graph.gpus, graph.slots, m)
    case["total"] = hx(m.total_weight)
    return case


# ---------------------------------------------------------------------------
# 1. flat KM (km_match)

def gen_km(rng):
    cases = []
    kinds = ["int", "tie3", "tie6", "dyadic", "float"]
    for t in range(400):
        kind = kinds[t % len(kinds)]
        n_l = int(rng.integers(1, 11))
        n_r = int(rng.integers(1, 11))
        if kind == "int":
            w = rng.integers(0, 10**6, size=(n_l, n_r)).astype(float)
        elif kind == "tie3":
            w = rng.integers(0, 3, size=(n_l, n_r)).astype(float)
        elif kind == "tie6":
            w = rng.integers(0, 6, size=(n_l, n_r)).astype(float)
        elif kind == "dyadic":
            w = rng.integers(0, 9, size=(n_l, n_r)) * (1693181818 / 8.0)
        else:
            w = rng.random((n_l, n_r)) * 1e9
        cases.append(w.tolist())
    for n, kind in [(32, "tie3"), (64, "int"), (64, "tie3"), (100, "dyadic"), (128, "tie6"),
                    (40, "float"), (7, "tie3"), (150, "tie3")]:
        if kind == "int":
            w = rng.integers(0, 10**6, size=(n, n)).astype(float)
        elif kind == "tie3":
            w = rng.integers(0, 3, size=(n, n)).astype(float)
        elif kind == "tie6":
            w = rng.integers(0, 6, size=(n, n)).astype(float)
        elif kind == "dyadic":
            w = rng.integers(0, 9, size=(n, n)) * (1693181818 / 8.0)
        else:
            w = rng.random((n, n)) * 1e9
        cases.append(w.tolist())
    # the SURVEY finding-4 counter-example (tie-break is not lexicographic)
    cases.append([[0.0, 0.0, 2.0, 0.0], [1.0, 0.0, 1.0, 1.0], [0.0, 0.0, 2.0, 0.0], [0.0, 0.0, 0.0, 1.0]])
    out = []
    for w in cases:
        g = graph_of(w)
        m = ref_map.km_match(g)
        assign = enc_mapping_result(g.gpus, g.slots, m)
        out.append({"W": [[hx(x) for x in row] for row in w], "assign": assign,
                    "total": hx(m.total_weight),
                    "perm": ref_map._hungarian_max(ref_map._pad_square(w))})
    return out


# ---------------------------------------------------------------------------
# 2. random (unstructured) inventories -- test_mapping / acceptance 02 style

def random_inventory(rng, model, denoms=(2,), p_model=0.5, cache_reqs=()):
    shards = []
    for lyr in range(model.num_layers):
        if rng.random() < p_model:
            den = int(rng.choice(denoms))
            k = int(rng.integers(0, den))
            width = int(rng.integers(1, den - k + 1))
            shards.append((lyr, Fraction(k, den), Fraction(k + width, den)))
    cache = []
    for rid, tok in cache_reqs:
        for lyr, lo, hi in shards:
            if rng.random() < 0.7:
                cache.append((rid, lyr, lo, hi, max(0, int(tok + rng.integers(-3, 4)))))
    return ContextInventory(model_shards=tuple(shards), cache_shards=tuple(cache))


def gen_random_inventories(rng):
    out = []
    for t in range(160):
        L = int(rng.integers(2, 9))
        model = ModelSpec(name="r", num_layers=L, bytes_per_layer=int(rng.integers(100, 5000)),
                          kv_bytes_per_token_per_layer=int(rng.integers(4, 64)))
        G = int(rng.choice([1, 1, 2, 2, 4]))
        M = int(rng.choice([1, 2, 4]))
        if t % 16 == 15:
            M = 3
            G = int(rng.choice([1, 3]))
        P = int(rng.integers(1, min(L, 4) + 1))
        D = int(rng.integers(1, 3))
        target = ParallelConfig(D, P, M, 1)
        n_inst = max(1, (target.gpus + G - 1) // G + int(rng.integers(-1, 3)))
        denoms = (2,) if t % 3 else (1, 2, 4, 3, 8)
        use_cache = rng.random() < 0.5
        tokens_by_pipe = None
        inheritance = None
        req_pool = []
        if use_cache:
            d_old = int(rng.integers(1, 3))
            tokens_by_pipe = {}
            for d in range(1, d_old + 1):
                tokens_by_pipe[d] = [(f"r-{d}-{j}", int(rng.integers(0, 40)))
                                     for j in range(int(rng.integers(1, 4)))]
                req_pool.extend(tokens_by_pipe[d])
            inheritance = {d: d for d in range(1, min(d_old, D) + 1)}
            if rng.random() < 0.3 and D >= 2 and d_old >= 1:
                inheritance = {1: D}
        instances = []
        for k in range(n_inst):
            inst = InstanceState(id=f"i-{k}", kind="spot", gpus=G)
            inst.gpu_inventories = [
                random_inventory(rng, model, denoms, 0.5,
                                 cache_reqs=[req_pool[int(rng.integers(0, len(req_pool)))]]
                                 if req_pool and rng.random() < 0.6 else ())
                for _ in range(G)]
            instances.append(inst)
        # shuffle ids to exercise natural-key row order
        if t % 4 == 0:
            ids = [f"i-{k}" for k in rng.permutation(n_inst * 3)[:n_inst]]
            for inst, iid in zip(instances, ids):
                inst.id = iid
        fw = "sum" if t % 7 == 3 else "max"
        out.append(run_map_case(model, target, G, instances, inheritance, tokens_by_pipe, fw))
    return out


# ---------------------------------------------------------------------------
# 3. structured layouts (simulator-like): positional old config on G-GPU
#    instances, some instances preempted, per-pipeline cached requests

def structured_case(rng, model, old, new, G, n_inst, n_drop, batch, fused="max", spare_first=False):
    ids = [f"i-{k}" for k in range(n_inst)]
    refs = [(iid, g) for iid in ids for g in range(G)]
    slots = positions(old)
    tokens_by_pipe = {d: [(f"r{d}-{j:02d}", int(512 + rng.integers(0, 129))) for j in range(batch)]
                      for d in range(1, old.data_parallel + 1)} if batch else None
    layout = {}
    start = G if spare_first else 0
    for k, ref in enumerate(refs):
        pos_idx = k - start
        if 0 <= pos_idx < len(slots):
            pos = slots[pos_idx]
            inv = required_context(old, pos, model)
            cache = ()
            if tokens_by_pipe:
                cache = tuple((rid, lyr, lo, hi, tok) for rid, tok in tokens_by_pipe[pos.pipeline]
                              for lyr, lo, hi in inv.model_shards)
            layout[ref] = ContextInventory(inv.model_shards, cache)
        else:
            layout[ref] = ContextInventory.empty()
    dropped = set(rng.choice(n_inst, size=n_drop, replace=False).tolist()) if n_drop else set()
    instances = []
    for k, iid in enumerate(ids):
        if k in dropped:
            continue
        inst = InstanceState(id=iid, kind="spot", gpus=G)
        inst.gpu_inventories = [layout[(iid, g)] for g in range(G)]
        instances.append(inst)
    inheritance = ref_map.default_inheritance(old.data_parallel, new.data_parallel) if batch else None
    return run_map_case(model, new, G, instances, inheritance, tokens_by_pipe, fused)


def gen_structured(rng):
    out = []
    gpt = ModelSpec("gpt-20b", 44, 1693181818, 24576)
    llama = ModelSpec("llama-30b", 60, 1070071808, 26624)
    toy = ModelSpec("toy", 6, 600, 64)
    combos = [
        (gpt, (2, 2, 8), (1, 2, 8), 4), (gpt, (1, 2, 8), (2, 3, 4), 4), (gpt, (2, 3, 4), (2, 2, 8), 4),
        (gpt, (2, 2, 8), (2, 3, 4), 4), (gpt, (1, 4, 4), (1, 6, 2), 4), (gpt, (1, 6, 2), (2, 4, 4), 4),
        (llama, (1, 2, 4), (2, 1, 4), 4), (llama, (1, 4, 2), (1, 2, 4), 2), (llama, (2, 3, 4), (1, 4, 8), 4),
        (toy, (2, 2, 2), (2, 3, 1), 1), (toy, (1, 2, 2), (1, 3, 2), 2), (toy, (2, 2, 1), (1, 2, 2), 2),
        (toy, (1, 3, 2), (1, 2, 3), 1), (toy, (1, 2, 3), (2, 1, 3), 3), (toy, (2, 1, 6), (1, 2, 6), 3),
        (gpt, (2, 2, 8), (1, 3, 3), 1), (gpt, (2, 3, 4), (1, 2, 6), 1), (toy, (1, 2, 4), (1, 2, 3), 4),
    ]
    for idx, (model, o, n, G) in enumerate(combos):
        old = ParallelConfig(*o, 2)
        new = ParallelConfig(*n, 2)
        need = max(old.gpus, new.gpus)
        for rep in range(3):
            n_inst = (need + G - 1) // G + 2 + rep
            n_drop = int(rng.integers(0, 3))
            while (n_inst - n_drop) * G < new.gpus:
                n_drop -= 1
            batch = [0, 3, 8][rep]
            fused = "sum" if (idx + rep) % 5 == 4 else "max"
            out.append(structured_case(rng, model, old, new, G, n_inst, n_drop, batch, fused,
                                       spare_first=(rep == 1)))
    # error paths
    inst = InstanceState(id="i-0", kind="spot", gpus=2)
    out.append(run_map_case(toy, ParallelConfig(1, 2, 2, 1), 4, [inst], None, None, "max"))
    out.append(run_map_case(toy, ParallelConfig(1, 2, 2, 1), 2, [inst], None, None, "median"))
    return out


# ---------------------------------------------------------------------------
# 4. the B_S scenario: record every map_devices / plan_migration / migration_cost
#    call the simulator makes (configs[0] and configs[1] of BASELINE.json)

def gen_scenario():
    maps, plans, costs = [], [], []
    orig_map, orig_plan, orig_cost = ref_sim.map_devices, ref_sim.plan_migration, ref_sim.migration_cost
    profile_ref = {}

    def rec_map(instances, target, model, G, inheritance=None, requests_by_old_pipeline=None,
                fused_weight="max"):
        tokens = None
        if requests_by_old_pipeline is not None:
            tokens = {d: [(r.id, r.s_in + r.tokens_generated) for r in rs]
                      for d, rs in requests_by_old_pipeline.items()}
        case = run_map_case(model, target, G, instances, inheritance, tokens, fused_weight,
                            want_w=len(maps) < 12)
        case["config_batch"] = target.batch_limit
        maps.append(case)
        return orig_map(instances, target, model, G, inheritance=inheritance,
                        requests_by_old_pipeline=requests_by_old_pipeline, fused_weight=fused_weight)

    def rec_plan(mapping, old_layout, model, u_max=None, inherited_by_pipeline=None,
                 departing=frozenset()):
        doc = {
            "model": [model.num_layers, model.bytes_per_layer, model.kv_bytes_per_token_per_layer],
            "target": list(mapping.config.shape()) if mapping.config else None,
            "assignment": [[g[0], g[1], p.pipeline, p.stage, p.shard]
                           for g, p in mapping.assignment.items()],
            "old_layout": [[g[0], g[1], enc_inv(inv.model_shards, inv.cache_shards)]
                           for g, inv in old_layout.items()],
            "u_max": u_max,
            "inherited": None if inherited_by_pipeline is None else
            {str(d): [[rid, tok] for rid, tok in lst] for d, lst in inherited_by_pipeline.items()},
            "departing": sorted(departing),
        }
        try:
            plan = orig_plan(mapping, old_layout, model, u_max=u_max,
                             inherited_by_pipeline=inherited_by_pipeline, departing=departing)
        except ref_mig.MigrationError:
            doc["error"] = "MigrationError"
            plans.append(doc)
            raise
        doc["error"] = None
        doc["plan"] = ref_mig.plan_to_dict(plan)
        plans.append(doc)
        return plan

    def rec_cost(plan, profile, config=None, progressive=False, release=None, start=0.0):
        val = orig_cost(plan, profile, config=config, progressive=progressive, release=release,
                        start=start)
        profile_ref["bw"] = profile.bandwidth
        costs.append({
            "plan": ref_mig.plan_to_dict(plan),
            "bandwidth": profile.bandwidth, "latency": profile.transfer_latency,
            "config": None if config is None else list(config.as_tuple()),
            "t_dec": None if config is None else profile.decode_seconds(config),
            "progressive": progressive,
            "release": None if release is None else {k: hx(v) for k, v in release.items()},
            "start": hx(start), "value": hx(val)})
        return val

    ref_sim.map_devices, ref_sim.plan_migration, ref_sim.migration_cost = rec_map, rec_plan, rec_cost
    try:
        base = load_simconfig(bundled_path("scenario_bs.json"))
        for rate in (0.25, 0.35, 0.55):
            cfg = replace(base, workload=replace(base.workload, rate=rate))
            ref_sim.run(cfg)
    finally:
        ref_sim.map_devices, ref_sim.plan_migration, ref_sim.migration_cost = orig_map, orig_plan, orig_cost
    return maps, plans, costs


# ---------------------------------------------------------------------------
# 5. synthetic migration plans (acceptance 03 style), for the planner rows

def gen_plans(rng):
    out = []
    for t in range(60):
        layers = int(rng.integers(2, 13))
        model = ModelSpec(name="t", num_layers=layers, bytes_per_layer=int(rng.integers(200, 2000)),
                          kv_bytes_per_token_per_layer=int(rng.integers(4, 64)))

        def rand_cfg(max_gpus):
            while True:
                p = int(rng.integers(1, 5))
                m = int(rng.choice([1, 2, 4]))
                if p > layers:
                    continue
                cap = max_gpus // (p * m)
                if cap < 1:
                    continue
                return ParallelConfig(int(rng.integers(1, cap + 1)), p, m, int(rng.choice([1, 2, 4])))

        old, new = rand_cfg(12), rand_cfg(12)
        n_inst = max(old.gpus, new.gpus) + int(rng.integers(0, 3))
        instances = [InstanceState(id=f"i-{k}", kind="spot", gpus=1) for k in range(n_inst)]
        layout = {}
        slots = positions(old)
        for inst, pos in itertools.zip_longest(instances, slots):
            if inst is None:
                break
            ref = (inst.id, 0)
            layout[ref] = ContextInventory.empty() if pos is None else required_context(old, pos, model)
        inherited = None
        if rng.random() < 0.5:
            inherited = {}
            for d in range(1, min(old.data_parallel, new.data_parallel) + 1):
                inherited[d] = [(f"r-{d}-{j}", int(rng.integers(8, 200)))
                                for j in range(int(rng.integers(1, new.batch_limit + 1)))]
            for ref, pos in zip([(i.id, 0) for i in instances], slots):
                if pos.pipeline in inherited:
                    inv = layout[ref]
                    cache = tuple((rid, lyr, lo, hi, tok) for rid, tok in inherited[pos.pipeline]
                                  for lyr, lo, hi in inv.model_shards)
                    layout[ref] = ContextInventory(inv.model_shards, cache)
        for inst in instances:
            inst.gpu_inventories = [layout[(inst.id, 0)]]
        mapping = ref_map.map_devices(instances, new, model, 1)
        u_max = None if t % 4 == 0 else float(model.bytes_per_layer) * float(rng.uniform(0.5, 3.0))
        departing = frozenset({instances[int(rng.integers(0, n_inst))].id}) if t % 5 == 2 else frozenset()
        doc = {
            "model": [model.num_layers, model.bytes_per_layer, model.kv_bytes_per_token_per_layer],
            "target": list(new.shape()),
            "assignment": [[g[0], g[1], p.pipeline, p.stage, p.shard] for g, p in mapping.assignment.items()],
            "old_layout": [[g[0], g[1], enc_inv(inv.model_shards, inv.cache_shards)] for g, inv in layout.items()],
            "u_max": u_max,
            "inherited": None if inherited is None else
            {str(d): [[rid, tok] for rid, tok in lst] for d, lst in inherited.items()},
            "departing": sorted(departing),
        }
        try:
            plan = ref_mig.plan_migration(mapping, layout, model, u_max=u_max,
                                          inherited_by_pipeline=inherited, departing=departing)
            doc["error"] = None
            doc["plan"] = ref_mig.plan_to_dict(plan)
            doc["cost_full"] = hx(ref_cost.migration_cost(plan, _toy_profile(model)))
        except ref_mig.MigrationError:
            doc["error"] = "MigrationError"
        out.append(doc)
    # missing-source error paths (test_migration.py:222-233 style): wipe every
    # copy of one layer before planning
    for t, (o, n) in enumerate([((1, 2, 2), (1, 2, 2)), ((1, 2, 4), (2, 1, 2)), ((2, 2, 1), (1, 4, 1))]):
        model = ModelSpec(name="e", num_layers=8, bytes_per_layer=1000, kv_bytes_per_token_per_layer=16)
        old, new = ParallelConfig(*o, 1), ParallelConfig(*n, 1)
        n_inst = max(old.gpus, new.gpus)
        instances = [InstanceState(id=f"i-{k}", kind="spot", gpus=1) for k in range(n_inst)]
        layout = {}
        for inst, pos in itertools.zip_longest(instances, positions(old)):
            ref = (inst.id, 0)
            inv = ContextInventory.empty() if pos is None else required_context(old, pos, model)
            layout[ref] = ContextInventory(tuple(s for s in inv.model_shards if s[0] != t))
            inst.gpu_inventories = [layout[ref]]
        mapping = ref_map.map_devices(instances, new, model, 1)
        doc = {
            "model": [model.num_layers, model.bytes_per_layer, model.kv_bytes_per_token_per_layer],
            "target": list(new.shape()),
            "assignment": [[g[0], g[1], p.pipeline, p.stage, p.shard] for g, p in mapping.assignment.items()],
            "old_layout": [[g[0], g[1], enc_inv(inv.model_shards, inv.cache_shards)] for g, inv in layout.items()],
            "u_max": None, "inherited": None, "departing": [],
        }
        try:
            plan = ref_mig.plan_migration(mapping, layout, model)
            doc["error"] = None
            doc["plan"] = ref_mig.plan_to_dict(plan)
            doc["cost_full"] = hx(ref_cost.migration_cost(plan, _toy_profile(model)))
        except ref_mig.MigrationError as e:
            doc["error"] = "MigrationError"
            doc["message"] = str(e)
        out.append(doc)
    return out


def _toy_profile(model):
    return ref_cost.PerfProfile(model=model, decode_table={(1, 1, 1): 0.1},
                                prefill_table={(1, 1, 1): {512: 1.0}}, pipeline_efficiency=1.0,
                                bandwidth=1e9, transfer_latency=0.005,
                                prices=ref_cost.PriceSheet(1.0, 2.0))


def main():
    rng = np.random.default_rng(20261018)
    km = gen_km(rng)
    save("km", {"meta": META, "cases": km})
    mapping = gen_random_inventories(rng) + gen_structured(rng)
    save("mapping", {"meta": META, "cases": mapping})
    maps, plans, costs = gen_scenario()
    save("scenario", {"meta": META, "maps": maps, "plans": plans, "costs": costs})
    save("plans", {"meta": META, "cases": gen_plans(rng)})
    print(f"km={len(km)} mapping={len(mapping)} scenario maps={len(maps)} plans={len(plans)} "
          f"costs={len(costs)}")


if __name__ == "__main__":
    main()
