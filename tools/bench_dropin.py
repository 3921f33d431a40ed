"""bench.py helpers: the CPU reference legs and the drop-in (reference-facing
API) block.  Test/bench tooling: the reference (`spotsim` from baseline/_ref)
and the oracle are only timed baselines and checkers here.

* `load_spotsim()`        the UNMODIFIED reference installed by
                          tools/install_reference.py, or None
* `cpu_reference_rate()`  the reference's map_devices on sampled sweep plans,
                          all host cores, a pool created OUTSIDE the timed
                          window and fed continuously (no lock-step chunks);
                          returns every sampled plan's answer so the caller can
                          check the GPU's results for exactly those plans
* `dropin_block()`        reference-facing calls with caller objects in and
                          DeviceMapping / MigrationPlan out: the 15 B_S scenario
                          map_devices calls, the configs[0] replans
                          (2,2,8)->(1,2,8)->(2,3,4) on 12 four-GPU instances,
                          map_devices_many throughput and plan_migration --
                          each beside the reference on the same inputs
"""

from __future__ import annotations

import os
import statistics
import sys
import time
from concurrent.futures import FIRST_COMPLETED, ProcessPoolExecutor, wait
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "tests", ROOT / "tests" / "golden"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def load_spotsim():
    """The reference package from baseline/_ref (or the build container's
    checkout); None when neither is present."""
    for cand in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (cand / "spotsim").exists():
            if str(cand) not in sys.path:
                sys.path.append(str(cand))
            try:
                import spotsim
                import spotsim.controller  # noqa: F401
                import spotsim.costmodel  # noqa: F401
                import spotsim.data  # noqa: F401
                import spotsim.domain  # noqa: F401
                import spotsim.mapping  # noqa: F401
                import spotsim.migration  # noqa: F401
                return spotsim
            except ImportError:
                return None
    return None


# ---------------------------------------------------------------------------
# the reference on sampled sweep plans, all cores

_W = {}


def _ref_plan(q):
    from oracle.sweep_inputs import mapping_cols, plan_to_spotsim, plan_to_port

    b, model, spot = _W["batch"], _W["model"], _W["spot"]
    t0 = time.perf_counter()
    if spot is not None:
        args = plan_to_spotsim(b, q, model, spot, n_requests=4)
        m = spot.mapping.map_devices(*args[:4], inheritance=args[4], requests_by_old_pipeline=args[5],
                                     fused_weight=args[6])
        cols, total = mapping_cols(m, args[0], args[1], spot), m.total_weight
    else:
        from oracle import port

        inst, new, G, inh, reqs, fw = plan_to_port(b, q, model, n_requests=4)
        _, _, _, cols, total = port.map_devices(inst, new, model, G, inh, reqs, fw)
    return q, cols, total.hex(), time.perf_counter() - t0


def _warm(_):
    import oracle.sweep_inputs  # noqa: F401

    return os.getpid()


def sample_order(n_plans: int, n_pairs: int = 36):
    """Plans round-robin over the config pairs (the batch is sorted by outer
    size, so consecutive indices are one size class)."""
    S = max(1, n_plans // n_pairs)
    order = [p * S + s for s in range(S) for p in range(min(n_pairs, n_plans))]
    return [q for q in order if q < n_plans]


def cpu_reference_rate(batch, model, seconds: float, cores: int, spot, order=None):
    """-> dict(rate, done, seconds, kind, answers {q: (cols, total hex)}).
    The pool is forked before the clock starts; `cores` plans are kept in
    flight and refilled as each finishes until `seconds` have passed; the
    window closes when the last in-flight plan returns."""
    import multiprocessing as mp

    order = sample_order(batch.n_plans) if order is None else order
    _W.update(batch=batch, model=model, spot=spot)
    ctx = mp.get_context("fork")
    answers = {}
    with ProcessPoolExecutor(max_workers=cores, mp_context=ctx) as ex:
        # warm the workers (imports, first-call costs) outside the window
        list(ex.map(_warm, range(cores)))
        it = iter(order)
        t0 = time.perf_counter()
        running = set()
        for _ in range(cores):
            q = next(it, None)
            if q is None:
                break
            running.add(ex.submit(_ref_plan, q))
        while running:
            done, running = wait(running, return_when=FIRST_COMPLETED)
            for f in done:
                q, cols, tot, _ = f.result()
                answers[q] = (cols, tot)
                if time.perf_counter() - t0 < seconds:
                    nq = next(it, None)
                    if nq is not None:
                        running.add(ex.submit(_ref_plan, nq))
        dt = time.perf_counter() - t0
    return {"rate": len(answers) / dt, "done": len(answers), "seconds": dt,
            "kind": "reference" if spot is not None else "port", "answers": answers}


def check_answers(answers, assign, totals, plans):
    """GPU results of the sampled plans vs the reference's answers."""
    ok = 0
    for q, (cols, tot) in answers.items():
        o, R = int(plans["out_off"][q]), int(plans["rows"][q])
        ok += assign[o:o + R].tolist() == cols and totals[q].hex() == tot
    return ok


# ---------------------------------------------------------------------------
# drop-in block

def _spot_problem(case, spot):
    from cases import decode_map_case

    dm = spot.domain
    model, target, G, instances, inh, reqs, fw = decode_map_case(case)
    mspec = dm.ModelSpec(name="m", num_layers=model[0], bytes_per_layer=model[1],
                         kv_bytes_per_token_per_layer=model[2])
    insts = []
    for iid, invs in instances:
        inst = dm.InstanceState(id=iid, kind="spot", gpus=len(invs))
        inst.gpu_inventories = [dm.ContextInventory(model_shards=i.model, cache_shards=i.cache) for i in invs]
        insts.append(inst)
    rq = None
    if reqs is not None:
        rq = {d: [dm.RequestSpec(id=rid, arrival_time=0.0, s_in=tok, s_out=max(tok, 1)) for rid, tok in lst]
              for d, lst in reqs.items()}
    return mspec, dm.ParallelConfig(*target, 1), G, insts, inh, rq, fw


def _spot_plan_inputs(doc, spot):
    from fmt import dec_inv

    dm = spot.domain
    model = dm.ModelSpec("m", *doc["model"])
    target = dm.ParallelConfig(*doc["target"], 1) if doc["target"] else None
    assignment = {(g, i): dm.TopologyPosition(d, p, m) for g, i, d, p, m in doc["assignment"]}
    mapping = spot.mapping.DeviceMapping(assignment=assignment, total_weight=0.0, config=target)
    layout = {}
    for iid, g, inv in doc["old_layout"]:
        m_, c_ = dec_inv(inv)
        layout[(iid, g)] = dm.ContextInventory(model_shards=m_, cache_shards=c_)
    inherited = None
    if doc["inherited"] is not None:
        inherited = {int(d): [(r, t) for r, t in lst] for d, lst in doc["inherited"].items()}
    return model, mapping, layout, inherited, frozenset(doc["departing"])


def config1_problems(ns, map_devices, required_context_with_cache):
    """BASELINE.json configs[0]: GPT-20B (2,2,8) on 12 four-GPU instances
    (positional on i-0..i-7, 8 cached requests of 512 + 64 tokens per
    pipeline), replanned to (1,2,8) and then to (2,3,4).  `ns` is the domain
    namespace (the reference's or this package's); returns the two
    map_devices argument tuples (the second one's layout is the first
    mapping's required context)."""
    model = ns.ModelSpec("gpt-20b", 44, 1693181818, 24576)
    old = ns.ParallelConfig(2, 2, 8, 8)
    G, n_inst = 4, 12
    reqs = {d: [ns.RequestSpec(id=f"r{d}-{j}", arrival_time=0.0, s_in=512, s_out=128, tokens_generated=64)
                for j in range(8)] for d in (1, 2)}
    slots = ns.positions(old)
    insts = []
    for k in range(n_inst):
        invs = []
        for g in range(G):
            q = k * G + g
            if q < len(slots):
                base = ns.required_context(old, slots[q], model)
                cache = tuple((r.id, lyr, lo, hi, r.s_in + r.tokens_generated) for r in reqs[slots[q].pipeline]
                              for lyr, lo, hi in base.model_shards)
                invs.append(ns.ContextInventory(base.model_shards, cache))
            else:
                invs.append(ns.ContextInventory())
        insts.append(ns.InstanceState(id=f"i-{k}", kind="spot", gpus=G, gpu_inventories=invs))
    t1 = ns.ParallelConfig(1, 2, 8, 8)
    inh1 = {1: 1}
    first = (insts, t1, model, G, inh1, reqs, "max")
    m1 = map_devices(insts, t1, model, G, inheritance=inh1, requests_by_old_pipeline=reqs)
    inherited = [(r.id, r.s_in + r.tokens_generated) for r in reqs[1]]
    insts2 = []
    for inst in insts:
        invs = []
        for g in range(G):
            pos = m1.assignment.get((inst.id, g))
            invs.append(ns.ContextInventory() if pos is None
                        else required_context_with_cache(t1, pos, model, inherited))
        insts2.append(ns.InstanceState(id=inst.id, kind="spot", gpus=G, gpu_inventories=invs))
    t2 = ns.ParallelConfig(2, 3, 4, 8)
    reqs2 = {1: reqs[1]}
    second = (insts2, t2, model, G, {1: 1}, reqs2, "max")
    return [first, second]


def _time(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def dropin_block(spot, ref_reps: int = 1):
    """Reference-facing calls, ours vs the reference on identical inputs."""
    import torch

    from fmt import load
    from helpers import assignment_cols, own_problem
    from test_planner import rebuild

    import paper_2311_15566_b200 as sk
    from paper_2311_15566_b200 import planner
    from paper_2311_15566_b200.mapping import required_context_with_cache as own_rcwc

    def sync_time(fn, reps=5):
        def run():
            fn()
            torch.cuda.synchronize()
        return _time(run, reps)

    doc = load("scenario")
    out = {"reference": "spotsim (baseline/_ref)" if spot else "unavailable (oracle port not used here)"}
    rows = []
    problems = []
    for case in doc["maps"]:
        model, cfg, G, insts, inh, rq, fw = own_problem(case)
        problems.append((insts, cfg, model, G, inh, rq, fw))
        got = sk.map_devices(insts, cfg, model, G, inh, rq, fw)
        exact = assignment_cols(got, insts, cfg) == case["assign"] and got.total_weight.hex() == case["total"]
        r = {"rows": sum(i.gpus for i in insts), "cols": cfg.gpus, "exact_vs_reference_golden": exact,
             "ms_ours": 1e3 * sync_time(lambda: sk.map_devices(insts, cfg, model, G, inh, rq, fw))}
        if spot:
            sm, sc, sG, si, sinh, srq, sfw = _spot_problem(case, spot)
            r["ms_reference"] = 1e3 * _time(lambda: spot.mapping.map_devices(
                si, sc, sm, sG, inheritance=sinh, requests_by_old_pipeline=srq, fused_weight=sfw), ref_reps)
        rows.append(r)
    out["bs_map_devices"] = _summary(rows)
    # configs[0]: (2,2,8) -> (1,2,8) -> (2,3,4) on 12 four-GPU instances
    ours_c1 = config1_problems(sk, sk.map_devices, own_rcwc)
    c1 = []
    ref_c1 = config1_problems(spot.domain, spot.mapping.map_devices,
                              spot.mapping.required_context_with_cache) if spot else None
    for k, args in enumerate(ours_c1):
        insts, cfg, model, G, inh, rq, fw = args
        got = sk.map_devices(*args)
        r = {"transition": ["(2,2,8)->(1,2,8)", "(1,2,8)->(2,3,4)"][k], "rows": 48, "cols": cfg.gpus,
             "ms_ours": 1e3 * sync_time(lambda: sk.map_devices(*args))}
        if spot:
            sa = ref_c1[k]
            m = spot.mapping.map_devices(*sa[:4], inheritance=sa[4], requests_by_old_pipeline=sa[5],
                                         fused_weight=sa[6])
            from oracle.sweep_inputs import mapping_cols

            r["exact_vs_reference"] = (assignment_cols(got, insts, cfg) == mapping_cols(m, sa[0], sa[1], spot)
                                       and got.total_weight.hex() == m.total_weight.hex())
            r["ms_reference"] = 1e3 * _time(lambda: spot.mapping.map_devices(
                *sa[:4], inheritance=sa[4], requests_by_old_pipeline=sa[5], fused_weight=sa[6]), ref_reps)
        c1.append(r)
    out["config1_map_devices"] = _summary(c1)
    # map_devices_many: every scenario call x 32 in one batched call
    batch = problems * 32
    sk.map_devices_many(batch)
    t = sync_time(lambda: sk.map_devices_many(batch), 3)
    out["map_devices_many"] = {"calls": len(batch), "ms": 1e3 * t, "calls_per_s": len(batch) / t}
    if spot:
        out["map_devices_many"]["reference_calls_per_s"] = len(rows) / (sum(r["ms_reference"] for r in rows) / 1e3)
    # plan_migration (native C++) on the scenario's recorded plans
    prow = []
    for d in doc["plans"]:
        if d["error"]:
            continue
        model, mapping, layout, inh_, dep = rebuild(d)
        plan = planner.plan_migration(mapping, layout, model, u_max=d["u_max"], inherited_by_pipeline=inh_,
                                      departing=dep)
        r = {"transfers": sum(len(a.get("transfers", ())) for a in d["plan"]["actions"]),
             "exact_vs_reference_golden": planner.plan_to_dict(plan) == d["plan"],
             "ms_ours": 1e3 * _time(lambda: planner.plan_migration(mapping, layout, model, u_max=d["u_max"],
                                                                   inherited_by_pipeline=inh_, departing=dep), 3)}
        if spot:
            sm, smap, slay, sinh, sdep = _spot_plan_inputs(d, spot)
            r["ms_reference"] = 1e3 * _time(lambda: spot.migration.plan_migration(
                smap, slay, sm, u_max=d["u_max"], inherited_by_pipeline=sinh, departing=sdep), ref_reps)
        prow.append(r)
    out["plan_migration"] = _summary(prow)
    # plan_migration_many: the scenario's plans x 8 on all host threads, vs
    # the same plans one call at a time
    probs = []
    for d in doc["plans"]:
        if not d["error"]:
            model, mapping, layout, inh_, dep = rebuild(d)
            probs.append((mapping, layout, model, d["u_max"], inh_, dep))
    batch = probs * 8
    t_many = _time(lambda: planner.plan_migration_many(batch, threads=0), 2)
    t_one = _time(lambda: [planner.plan_migration(*p[:3], u_max=p[3], inherited_by_pipeline=p[4],
                                                  departing=p[5]) for p in batch], 1)
    out["plan_migration_many"] = {"plans": len(batch), "threads": os.cpu_count(), "ms": 1e3 * t_many,
                                  "ms_sequential": 1e3 * t_one, "speedup_vs_sequential": t_one / t_many}
    out["optimize_config_many"] = _guarded(lambda: controller_leg(spot))
    return out


def _guarded(fn):
    try:
        return fn()
    except Exception as e:  # noqa: BLE001
        return {"error": f"{type(e).__name__}: {e}"}


def controller_leg(spot, n_scen: int = 20000):
    """optimize_config (controller.py:79-117) for many (n_available, rate,
    cloud_limit) scenarios: one device batch vs the reference one call at a
    time (a timed sample), on the GPT-20B profile's candidates up to 64 GPUs;
    the sampled reference decisions are checked against the batch's."""
    import random
    from types import SimpleNamespace

    import torch

    from fmt import load, unhx

    import paper_2311_15566_b200 as sk
    from paper_2311_15566_b200 import estimator

    t = load("estimator")["profiles"]["gpt-20b"]["profile"]
    pre = {}
    for P, M, B, s_, v in t["prefill"]:
        pre.setdefault((P, M, B), {})[s_] = unhx(v)
    prof = SimpleNamespace(decode_table={(P, M, B): unhx(v) for P, M, B, v in t["decode"]}, prefill_table=pre,
                           pipeline_efficiency=unhx(t["eta"]), nominal_s_in=t["nominal"][0],
                           nominal_s_out=t["nominal"][1])
    cands = [sk.ParallelConfig(*c) for c, _ in load("estimator")["profiles"]["gpt-20b"]["throughput"]]
    rng = random.Random(5)
    scen = [(rng.randint(0, 24), rng.choice([0.1, 0.25, 0.35, 0.55, 1.0, 2.0, 5.0]) * rng.uniform(0.5, 1.5),
             rng.choice([None, rng.randint(0, 30)])) for _ in range(n_scen)]

    def ours():
        r = estimator.optimize_config_many(scen, prof, cands, 4)
        torch.cuda.synchronize()
        return r

    got = ours()
    t_ours = _time(ours, 3)
    out = {"scenarios": n_scen, "candidates": len(cands), "ms": 1e3 * t_ours,
           "decisions_per_s": n_scen / t_ours}
    if spot:
        from spotsim import controller as rc
        from spotsim import costmodel as rcost

        rprof = rcost.load_profile(spot.data.bundled_path("gpt-20b"))
        rc_cands = [spot.domain.ParallelConfig(*c.as_tuple()) for c in cands]
        k = 500
        t0 = time.perf_counter()
        ref = [rc.optimize_config(n, None, r, rprof, rc_cands, gpus_per_instance=4, cloud_limit=lim)
               for n, r, lim in scen[:k]]
        dt = time.perf_counter() - t0
        same = sum((a is None and b is None) or (a is not None and b is not None and a.as_tuple() == b.as_tuple())
                   for a, b in zip(got[:k], ref))
        out.update({"reference_decisions_per_s": k / dt, "speedup": (n_scen / t_ours) / (k / dt),
                    "checked_vs_reference": f"{same}/{k}"})
    return out


def _summary(rows):
    s = {"calls": len(rows), "ms_ours_median": statistics.median(r["ms_ours"] for r in rows),
         "ms_ours_max": max(r["ms_ours"] for r in rows)}
    ex = [v for r in rows for k, v in r.items() if k.startswith("exact")]
    if ex:
        s["all_exact"] = all(ex)
    if all("ms_reference" in r for r in rows):
        s["ms_reference_median"] = statistics.median(r["ms_reference"] for r in rows)
        s["speedup_median"] = statistics.median(r["ms_reference"] / r["ms_ours"] for r in rows)
        s["speedup_total"] = sum(r["ms_reference"] for r in rows) / sum(r["ms_ours"] for r in rows)
    s["per_call"] = rows
    return s
