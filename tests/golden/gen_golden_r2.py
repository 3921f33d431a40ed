"""Round-2 golden vectors, produced by running the REAL reference (`spotsim`).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=baseline/_ref python tests/golden/gen_golden_r2.py

Writes
* `edge.json.gz`   -- map_devices / build_graph cases at the limits of the
  exact device encoding: fused groups > 8 (G = M = 12, 16), edge-weight
  numerators >= 2^53, interval denominators > 2^31 - 1, inheritance maps
  that name pipelines outside 1..D (ignored by build_graph, mapping.py:210),
  and flat km_match on huge weights.
* `sweep_ref.json.gz` -- plans of the headline batched sweep
  (paper_2311_15566_b200.sweep.make_sweep, BASELINE.json configs[2]) at 64,
  128, 256, 512 and 1,024 positions, each solved by the reference's
  map_devices on the equivalent spotsim objects (the plan's inputs are
  regenerated from (N, seed) by the tests; a digest pins them).
* `models_bs.json.gz` -- every map_devices call of the B_S scenario with the
  OPT-6.7B and LLaMA-30B profiles at 0.25 / 0.35 / 0.55 req/s (BASELINE.json
  configs[1]), with the plans and T_mig the simulator computes from them.
"""

from __future__ import annotations

import multiprocessing as mp
import sys
import time
from dataclasses import replace
from fractions import Fraction
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
for p in (HERE, ROOT):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

from cases import plan_digest  # noqa: E402
from fmt import enc_inv, hx, save  # noqa: E402
from gen_golden import META, random_inventory, run_map_case  # noqa: E402

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
    positions,
    required_context,
)
from spotsim.simconfig import load_simconfig  # noqa: E402


# ---------------------------------------------------------------------------
# 1. edge cases of the exact encoding

def _instances(rng, model, G, n_inst, denoms, req_pool, p_model=0.5):
    out = []
    for k in range(n_inst):
        inst = InstanceState(id=f"i-{k}", kind="spot", gpus=G)
        inst.gpu_inventories = [
            random_inventory(rng, model, denoms, p_model,
                             cache_reqs=[req_pool[int(rng.integers(0, len(req_pool)))]]
                             if req_pool and rng.random() < 0.6 else ())
            for _ in range(G)]
        out.append(inst)
    return out


def _structured(model, old, G, n_inst, drop, tokens_by_pipe):
    """Positional old layout of `old` on n_inst G-GPU instances, `drop` removed."""
    slots = positions(old)
    insts = []
    for k in range(n_inst):
        invs = []
        for g in range(G):
            q = k * G + g
            if q < len(slots):
                inv = required_context(old, slots[q], model)
                cache = ()
                if tokens_by_pipe:
                    cache = tuple((rid, lyr, lo, hi, tok) for rid, tok in tokens_by_pipe[slots[q].pipeline]
                                  for lyr, lo, hi in inv.model_shards)
                invs.append(ContextInventory(inv.model_shards, cache))
            else:
                invs.append(ContextInventory.empty())
        if k in drop:
            continue
        inst = InstanceState(id=f"i-{k}", kind="spot", gpus=G)
        inst.gpu_inventories = invs
        insts.append(inst)
    return insts


def gen_edge(rng):
    out = []
    # (a) fused groups > 8: G = M = 12 / 16, and G = 16 with M = 32
    for t, (G, tgt, L) in enumerate([(16, (1, 2, 16), 6), (12, (1, 2, 12), 5), (16, (1, 1, 32), 4),
                                     (16, (2, 1, 16), 3), (12, (1, 3, 12), 6), (10, (1, 2, 10), 4)]):
        model = ModelSpec(name="big-g", num_layers=L, bytes_per_layer=int(rng.integers(1000, 50000)),
                          kv_bytes_per_token_per_layer=int(rng.integers(4, 64)))
        target = ParallelConfig(*tgt, 1)
        for rep in range(2):
            if rep == 0:
                old = ParallelConfig(tgt[0], tgt[1], tgt[2], 1) if t % 2 else ParallelConfig(1, 1, tgt[2], 1)
                n_inst = -(-max(old.gpus, target.gpus) // G) + 1
                toks = {d: [(f"r{d}-{j}", int(rng.integers(1, 60))) for j in range(2)]
                        for d in range(1, old.data_parallel + 1)}
                insts = _structured(model, old, G, n_inst, {int(rng.integers(0, n_inst))} if n_inst > 2 else set(),
                                    toks)
                inh = ref_map.default_inheritance(old.data_parallel, target.data_parallel)
                fw = "sum" if t % 3 == 1 else "max"
                out.append(run_map_case(model, target, G, insts, inh, toks, fw))
            else:
                n_inst = -(-target.gpus // G) + 1
                denoms = (2, 4, G) if tgt[2] % 4 == 0 else (2, G)
                insts = _instances(rng, model, G, n_inst, denoms, [], 0.6)
                out.append(run_map_case(model, target, G, insts, None, None, "max" if t % 2 else "sum"))
    # (b) edge-weight numerators >= 2^53 (bytes_per_layer ~ 2^55), dyadic and M = 3
    for t in range(8):
        bpl = int(rng.integers(1 << 53, 1 << 58)) | 1
        kv = int(rng.integers(1 << 40, 1 << 44)) | 1
        model = ModelSpec(name="wide", num_layers=int(rng.integers(3, 9)), bytes_per_layer=bpl,
                          kv_bytes_per_token_per_layer=kv)
        M = (2, 3, 4, 1)[t % 4]
        G = (2, 3, 4, 1)[t % 4]
        target = ParallelConfig(int(rng.integers(1, 3)), int(rng.integers(1, min(model.num_layers, 3) + 1)), M, 1)
        old = ParallelConfig(int(rng.integers(1, 3)), int(rng.integers(1, 3)), (4, 3, 2, 2)[t % 4], 1)
        n_inst = -(-max(old.gpus, target.gpus) // G) + 2
        toks = {d: [(f"r{d}-{j}", int(rng.integers(100, 4000))) for j in range(3)]
                for d in range(1, old.data_parallel + 1)}
        insts = _structured(model, old, G, n_inst, {1} if n_inst > 3 else set(), toks)
        inh = ref_map.default_inheritance(old.data_parallel, target.data_parallel)
        out.append(run_map_case(model, target, G, insts, inh, toks, "sum" if t % 2 else "max"))
    # (c) interval denominators > 2^31 - 1 (lcm of large primes), random inventories
    for t in range(10):
        model = ModelSpec(name="bigk", num_layers=int(rng.integers(2, 6)),
                          bytes_per_layer=int(rng.integers(100, 5000)),
                          kv_bytes_per_token_per_layer=int(rng.integers(4, 64)))
        G = (1, 2, 4, 1, 2)[t % 5]
        M = (1, 2, 4, 2, 4)[t % 5]
        target = ParallelConfig(int(rng.integers(1, 3)), int(rng.integers(1, model.num_layers + 1)), M, 1)
        denoms = (65537, 65539, 2) if t % 2 else (65521, 131071, 4)
        d_old = 2
        toks = {d: [(f"r-{d}-{j}", int(rng.integers(0, 40))) for j in range(2)] for d in range(1, d_old + 1)}
        pool = [x for lst in toks.values() for x in lst]
        n_inst = max(1, -(-target.gpus // G) + 1)
        insts = _instances(rng, model, G, n_inst, denoms, pool)
        inh = {d: d for d in range(1, min(d_old, target.data_parallel) + 1)}
        out.append(run_map_case(model, target, G, insts, inh, toks, "max" if t % 3 else "sum"))
    # (d) both at once: big denominators and huge bytes
    for t in range(4):
        model = ModelSpec(name="bigk-wide", num_layers=3, bytes_per_layer=int(rng.integers(1 << 50, 1 << 54)) | 1,
                          kv_bytes_per_token_per_layer=int(rng.integers(1 << 30, 1 << 34)) | 1)
        G, M = (1, 1), (2, 2)
        G, M = ((1, 1), (2, 2), (2, 4), (1, 3))[t]
        target = ParallelConfig(1, 2, M, 1)
        toks = {1: [("r-1-0", int(rng.integers(1, 40)))]}
        n_inst = -(-target.gpus // G) + 1
        insts = _instances(rng, model, G, n_inst, (65537, 65539, 3), list(toks[1]), 0.7)
        out.append(run_map_case(model, target, G, insts, {1: 1}, toks, "max"))
    # (e) inheritance naming pipelines outside 1..D (ignored by build_graph)
    toy = ModelSpec(name="toy", num_layers=6, bytes_per_layer=600, kv_bytes_per_token_per_layer=64)
    for t, (o, n, G, inh) in enumerate([((2, 2, 2), (2, 2, 2), 2, {1: 3, 2: 2}),
                                        ((2, 2, 2), (2, 2, 2), 2, {1: 0, 2: 1}),
                                        ((3, 1, 2), (2, 1, 2), 2, {1: 1, 2: 2, 3: 3}),
                                        ((2, 2, 2), (1, 2, 2), 1, {2: 1, 1: 2}),
                                        ((3, 2, 2), (2, 2, 2), 4, {1: 7, 2: -1, 3: 2}),
                                        ((2, 2, 1), (2, 3, 1), 1, {1: 2, 2: 9})]):
        old, new = ParallelConfig(*o, 1), ParallelConfig(*n, 1)
        toks = {d: [(f"r{d}-{j}", int(rng.integers(1, 50))) for j in range(3)]
                for d in range(1, old.data_parallel + 1)}
        n_inst = -(-max(old.gpus, new.gpus) // G) + 1
        insts = _structured(toy, old, G, n_inst, set(), toks)
        out.append(run_map_case(toy, new, G, insts, inh, toks, "max" if t % 2 else "sum"))
    return out


def gen_km_wide(rng):
    """flat km_match on huge / tiny / subnormal weights (no encoding limits)."""
    out = []
    for t in range(12):
        n_l, n_r = int(rng.integers(1, 12)), int(rng.integers(1, 12))
        kind = t % 4
        if kind == 0:
            w = rng.integers(1 << 53, 1 << 62, size=(n_l, n_r)).astype(float)
        elif kind == 1:
            w = rng.random((n_l, n_r)) * 1e300
        elif kind == 2:
            w = rng.random((n_l, n_r)) * 1e-310
        else:
            w = rng.integers(0, 3, size=(n_l, n_r)) * 2.0 ** 1000
        gpus = [(f"i-{k}", 0) for k in range(n_l)]
        slots = [ref_map.TopologyPosition(1, 1, m + 1) for m in range(n_r)]
        g = ref_map.BipartiteGraph(gpus=gpus, slots=slots, weights=w.tolist())
        m = ref_map.km_match(g)
        col = {s: j for j, s in enumerate(slots)}
        out.append({"W": [[hx(x) for x in row] for row in w.tolist()],
                    "assign": [col[m.assignment[gp]] if gp in m.assignment else -1 for gp in gpus],
                    "total": hx(m.total_weight)})
    return out


# ---------------------------------------------------------------------------
# 2. headline sweep plans solved by the reference

SWEEP_SEED = 4242
SWEEP_PICK = {64: 6, 128: 6, 256: 5, 512: 4, 1024: 2}


def sweep_to_spotsim(batch, q, model_geom, n_requests=4):
    """One sweep plan -> spotsim objects (the semantics of sweep.py's header)."""
    from oracle.sweep_inputs import plan_to_port

    instances, new, G, inh, reqs, fw = plan_to_port(batch, q, model_geom, n_requests=n_requests)
    L, bpl, kv = model_geom
    model = ModelSpec(name="gpt-20b", num_layers=L, bytes_per_layer=bpl, kv_bytes_per_token_per_layer=kv)
    insts = []
    for iid, invs in instances:
        inst = InstanceState(id=iid, kind="spot", gpus=G)
        inst.gpu_inventories = [ContextInventory(model_shards=tuple(i.model), cache_shards=tuple(i.cache))
                                for i in invs]
        insts.append(inst)
    rq = {d: [RequestSpec(id=rid, arrival_time=0.0, s_in=tok, s_out=max(tok, 1)) for rid, tok in lst]
          for d, lst in reqs.items()}
    return insts, ParallelConfig(*new, 1), model, G, inh, rq, fw


def _solve_sweep(args):
    N, q = args
    from paper_2311_15566_b200 import sweep

    batch = sweep.make_sweep(N, 1, seed=SWEEP_SEED + N)
    insts, target, model, G, inh, rq, fw = sweep_to_spotsim(batch, q, sweep.GPT20B)
    t0 = time.perf_counter()
    m = ref_map.map_devices(insts, target, model, G, inheritance=inh, requests_by_old_pipeline=rq,
                            fused_weight=fw)
    dt = time.perf_counter() - t0
    refs = [(inst.id, g) for inst in insts for g in range(inst.gpus)]  # natural order (i-0..)
    col = {s: j for j, s in enumerate(positions(target))}
    return {"N": N, "seed": SWEEP_SEED + N, "sets": 1, "q": int(q), "digest": plan_digest(batch, q),
            "rows": len(refs), "target": list(target.shape()), "G": G,
            "assign": [col[m.assignment[r]] if r in m.assignment else -1 for r in refs],
            "total": hx(m.total_weight), "ref_seconds": dt}


def gen_sweep():
    from paper_2311_15566_b200 import sweep

    jobs = []
    for N, k in SWEEP_PICK.items():
        batch = sweep.make_sweep(N, 1, seed=SWEEP_SEED + N)
        Q = batch.n_plans
        # spread over the config pairs (plans are sorted by outer size)
        for q in np.linspace(0, Q - 1, k).round().astype(int).tolist():
            jobs.append((N, q))
    with mp.get_context("fork").Pool(min(len(jobs), mp.cpu_count())) as pool:
        out = pool.map(_solve_sweep, sorted(jobs, key=lambda j: -j[0]), chunksize=1)
    return sorted(out, key=lambda c: (c["N"], c["q"]))


# ---------------------------------------------------------------------------
# 3. B_S scenario replans with the OPT-6.7B and LLaMA-30B profiles

def gen_models_bs():
    maps, plans = [], []
    orig_map, orig_plan = ref_sim.map_devices, ref_sim.plan_migration

    def rec_map(instances, target, model, G, inheritance=None, requests_by_old_pipeline=None,
                fused_weight="max"):
        tokens = None
        if requests_by_old_pipeline is not None:
            tokens = {d: [(r.id, r.s_in + r.tokens_generated) for r in rs]
                      for d, rs in requests_by_old_pipeline.items()}
        case = run_map_case(model, target, G, instances, inheritance, tokens, fused_weight, want_w=False)
        case["config_batch"] = target.batch_limit
        case["profile"] = current[0]
        maps.append(case)
        return orig_map(instances, target, model, G, inheritance=inheritance,
                        requests_by_old_pipeline=requests_by_old_pipeline, fused_weight=fused_weight)

    def rec_plan(mapping, old_layout, model, u_max=None, inherited_by_pipeline=None, departing=frozenset()):
        doc = {
            "model": [model.num_layers, model.bytes_per_layer, model.kv_bytes_per_token_per_layer],
            "target": list(mapping.config.shape()) if mapping.config else None,
            "assignment": [[g[0], g[1], p.pipeline, p.stage, p.shard] for g, p in mapping.assignment.items()],
            "old_layout": [[g[0], g[1], enc_inv(inv.model_shards, inv.cache_shards)]
                           for g, inv in old_layout.items()],
            "u_max": u_max,
            "inherited": None if inherited_by_pipeline is None else
            {str(d): [[rid, tok] for rid, tok in lst] for d, lst in inherited_by_pipeline.items()},
            "departing": sorted(departing), "profile": current[0],
        }
        plan = orig_plan(mapping, old_layout, model, u_max=u_max, inherited_by_pipeline=inherited_by_pipeline,
                         departing=departing)
        doc["error"] = None
        doc["plan"] = ref_mig.plan_to_dict(plan)
        plans.append(doc)
        return plan

    current = [None]
    ref_sim.map_devices, ref_sim.plan_migration = rec_map, rec_plan
    try:
        base = load_simconfig(bundled_path("scenario_bs.json"))
        for prof in ("profile_opt67b.json", "profile_llama30b.json"):
            for rate in (0.25, 0.35, 0.55):
                current[0] = f"{prof}@{rate}"
                cfg = replace(base, profile_path=bundled_path(prof), workload=replace(base.workload, rate=rate))
                ref_sim.run(cfg)
    finally:
        ref_sim.map_devices, ref_sim.plan_migration = orig_map, orig_plan
    return maps, plans


# ---------------------------------------------------------------------------
# 4. candidate scoring: exec_latency / throughput / optimize_config

def gen_estimator():
    from spotsim import controller as ref_ctl
    from spotsim import costmodel as ref_cost

    out = {}
    for prof in ("gpt-20b", "opt-6.7b", "llama-30b"):
        profile = ref_cost.load_profile(bundled_path(prof))
        cands = ref_ctl.candidate_configs(profile, max_gpus=64)
        lat = []
        for cfg in cands:
            for s_in, s_out in ((512, 128), (128, 0), (1000, 64), (2048, 512), (1, 1), (700, 3), (96, 7),
                                (4096, 1)):
                try:
                    v = ref_cost.exec_latency(profile, cfg, s_in, s_out)
                    lat.append([list(cfg.as_tuple()), s_in, s_out, hx(v)])
                except ref_cost.ProfileMissError:
                    lat.append([list(cfg.as_tuple()), s_in, s_out, None])
        phi = [[list(c.as_tuple()), hx(ref_cost.throughput(profile, c))] for c in cands]
        dec = []
        for G in (1, 4):
            for n_av in range(0, 22):
                for rate in (0.0, 0.1, 0.25, 0.35, 0.55, 1.0, 2.0, 3.5, 5.0, 10.0, 40.0):
                    for lim in (None, n_av + 2, max(n_av - 1, 0)):
                        c = ref_ctl.optimize_config(n_av, None, rate, profile, cands, gpus_per_instance=G,
                                                    cloud_limit=lim)
                        dec.append([G, n_av, rate, lim, None if c is None else list(c.as_tuple())])
        tables = {"decode": [[*k, hx(v)] for k, v in sorted(profile.decode_table.items())],
                  "prefill": [[*k, s_, hx(v)] for k, d in sorted(profile.prefill_table.items())
                              for s_, v in sorted(d.items())],
                  "eta": hx(profile.pipeline_efficiency),
                  "nominal": [profile.nominal_s_in, profile.nominal_s_out]}
        out[prof] = {"latency": lat, "throughput": phi, "decisions": dec, "profile": tables}
    return out


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "estimator":
        save("estimator", {"meta": META, "profiles": gen_estimator()})
        return
    rng = np.random.default_rng(20261019)
    edge = gen_edge(rng)
    kmw = gen_km_wide(rng)
    save("edge", {"meta": META, "cases": edge, "km": kmw})
    save("estimator", {"meta": META, "profiles": gen_estimator()})
    maps, plans = gen_models_bs()
    save("models_bs", {"meta": META, "maps": maps, "plans": plans})
    t0 = time.perf_counter()
    sw = gen_sweep()
    save("sweep_ref", {"meta": META, "cases": sw})
    print(f"edge={len(edge)} ({sum(1 for c in edge if c['error'])} errors) km_wide={len(kmw)} "
          f"models maps={len(maps)} plans={len(plans)} sweep={len(sw)} ({time.perf_counter() - t0:.0f}s; "
          f"per-plan reference seconds max {max(c['ref_seconds'] for c in sw):.1f})")


if __name__ == "__main__":
    main()
