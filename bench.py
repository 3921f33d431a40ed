#!/usr/bin/env python
"""Benchmark: batched device-mapping sweep (BASELINE.json configs[2]).

One "step" = one pass of the hot path (sk_sweep_expand -> per size class
sk_map_fuse_coded -> sk_map_outer_coded; the double-matrix sk_map_fuse ->
sk_map_outer for sweeps with outer n < 96) over one batch of synthetic sweep
plans: every (old, new) GPT-20B candidate config pair at N target positions x
S preemption sets.

  value  plans/s with inputs resident in HBM (device-timed, CUDA events on
         the launching stream, L2 flushed between steps), max over ranks
  e2e    same metric through the public batched API (SweepRunner): pinned
         H2D of the compact plan descriptors + kernels + D2H of assignments
         and total weights, every step
  --impl reference   the unmodified reference (spotsim.map_devices from
         baseline/_ref; oracle/port.py only if that install is absent) on all
         host cores, rank 0 only

Multi-GPU (torchrun): plans are independent, so each rank solves its own
batch (no data-path collective; weak scaling); times are maxed over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "device-mapping plans/sec (batched KM, 64-1024 positions)"
UNIT = "plans/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--positions", type=int, default=256)
    ap.add_argument("--sets", type=int, default=4096,
                    help="preemption sets per config pair per step (BASELINE configs[2]: 4096)")
    ap.add_argument("--model", default="gpt-20b")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--all-sizes", action=argparse.BooleanOptionalAction, default=True,
                    help="also report 64..1024 positions (default on)")
    ap.add_argument("--no-reshard", action="store_true", help="skip the N>1 context reshard")
    ap.add_argument("--no-dropin", action="store_true", help="skip the drop-in API block")
    ap.add_argument("--no-k1", action="store_true", help="skip the K1 (build_graph) leg")
    return ap.parse_args()


def workload_name(args, n_plans):
    return (f"batched mapping sweep, {args.model}, {args.positions} positions, all candidate "
            f"(D,P,M) pairs x {args.sets} preemption sets ({n_plans} plans/step), G=4")


# ---------------------------------------------------------------------------
# clocks during the timed region

class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[4 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------

def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0}, "fallback"


def ncu_traffic(kernel: str, workload_key: str):
    """dram bytes per launch from a committed `ncu --set full` summary, if any."""
    try:
        doc = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
        return doc.get(workload_key, {}).get(kernel)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# CPU legs (the oracle is used only here and in tests)

def _tools():
    sys.path.insert(0, str(ROOT / "tools"))
    import bench_dropin

    return bench_dropin


def _guard(fn):
    """A side leg that fails reports its error instead of losing the line."""
    try:
        return fn()
    except Exception as e:  # noqa: BLE001
        import traceback

        traceback.print_exc()
        return {"error": f"{type(e).__name__}: {e}"}


def cpu_reference(batch, model, seconds: float, cores: int):
    """The REFERENCE (spotsim map_devices from baseline/_ref; the oracle port
    only if the reference is absent) on a bounded sample of this workload's
    plans, all host cores (tools/bench_dropin.cpu_reference_rate)."""
    bd = _tools()
    return bd.cpu_reference_rate(batch, model, seconds, cores, bd.load_spotsim())


def cpu_c_rate(batch, cores: int, seconds: float):
    """C restatement of the same algorithm (oracle/spotkm_oracle.c), OpenMP on all cores."""
    from oracle import cport

    cport.build()
    Q = batch.n_plans
    n = Q
    cport.map_sweep(batch.desc[:1], batch.plans, batch.alive, batch.tok, cores)  # load / warm
    probe = np.arange(0, Q, max(1, Q // (4 * cores)))[:4 * cores]
    t0 = time.perf_counter()
    cport.map_sweep(batch.desc[probe], batch.plans, batch.alive, batch.tok, cores)
    one = (time.perf_counter() - t0) * cores / len(probe)  # single-core seconds per plan
    if one * Q / cores > seconds:
        n = max(cores, int(seconds * cores / max(one, 1e-6)))
    step = max(1, Q // n)
    sel = np.arange(0, Q, step)[:n]
    t0 = time.perf_counter()
    cport.map_sweep(batch.desc[sel], batch.plans, batch.alive, batch.tok, cores)
    dt = time.perf_counter() - t0
    return len(sel) / dt, len(sel), dt


# ---------------------------------------------------------------------------

def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2311_15566_b200 import sweep

    geom, shapes = sweep.MODELS[args.model]
    cores = os.cpu_count() or 1
    batch = sweep.make_sweep(args.positions, args.sets, seed=1000, model=geom, shapes=shapes)
    per_step = max(1.0, 60.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        cpu_reference(batch, geom, 0.0, cores)
    total_plans, total_s, kind = 0, 0.0, "port"
    for _ in range(args.steps):
        r = cpu_reference(batch, geom, per_step, cores)
        total_plans += r["done"]
        total_s += r["seconds"]
        kind = r["kind"]
    rate = total_plans / total_s
    what = ("spotsim.mapping.map_devices (the unmodified reference, baseline/_ref)" if kind == "reference"
            else "oracle/port.py (reference absent)")
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_name(args, batch.n_plans), "positions": args.positions,
                   "sets_per_pair": args.sets},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{total_plans} plans of the workload, round-robin over config "
                                   f"pairs, each step ~{per_step:.0f}s on {cores} processes: {what}"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# seconds of reference work per sweep size (the window closes when the
# in-flight plans finish: ~25 s at 1,024 positions, where one plan takes ~20 s)
SIZE_CPU_SECONDS = 6.0


def k1_leg(geom, shapes, flush, hbm, reps=5):
    """K1 (build_graph's dense W, k_weights via sk_build_weights) on sweep
    plans at 256 and 1,024 positions: the weight builder's own HBM rate.
    Algorithmic bytes per plan = 8*R*C (the float64 W written once) + the
    rows' segments read (64 B per row)."""
    import torch

    from paper_2311_15566_b200 import _native as nat
    from paper_2311_15566_b200 import sweep

    out = {}
    for n_pos, sets in ((256, 96), (1024, 8)):
        b = sweep.make_sweep(n_pos, sets, seed=77, model=geom, shapes=shapes)
        r = sweep.SweepRunner(b)
        r.run()                                   # expands rows/segments on the device
        st = b.stats()
        RC = (st["rows"] * st["cols"]).astype(np.int64)
        plans = b.plans.copy()
        plans["f_off"] = np.concatenate([[0], np.cumsum(RC)[:-1]])
        d_plans = torch.from_numpy(plans.view(np.uint8)).cuda()
        W = torch.empty(int(RC.sum()), dtype=torch.float64, device="cuda")
        lib = nat.load()
        s = torch.cuda.current_stream().cuda_stream

        def launch():
            nat.check(lib.sk_build_weights(d_plans.data_ptr(), b.n_plans, r.row_ptr.data_ptr(),
                                           r.segs.data_ptr(), W.data_ptr(), int(st["rows"].max()),
                                           int(st["cols"].max()), s))

        launch()
        ts = []
        for k in range(reps):
            flush.fill_(k & 0xff)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            launch()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        alg = float(8 * RC.sum() + 64 * st["rows"].sum())
        out[str(n_pos)] = {"plans": b.n_plans, "W_bytes": int(8 * RC.sum()), "ms": ms,
                           "achieved_gbs": alg / (ms / 1e3) / 1e9, "peak_gbs": hbm,
                           "frac": alg / (ms / 1e3) / 1e9 / hbm,
                           "traffic": ncu_traffic("k_weights", f"k1-N{n_pos}")}
        del W, d_plans, r
    return out


# preemption sets per chunk for the all-sizes sweep (device scratch <= ~90 GB)
SIZE_CHUNK_SETS = {64: 4096, 128: 4096, 256: 4096, 512: 4096, 1024: 2048}


class Chunked:
    """Consecutive SweepRunners (one sweep split into chunks) as one step."""

    def __init__(self, runs):
        self.runs = runs

    def upload(self):
        for r in self.runs:
            r.upload()

    def solve(self, download=False):
        for r in self.runs:
            r.solve(download=download)

    def download(self):
        for r in self.runs:
            r.download()

    def run(self):
        for r in self.runs:
            r.run()


def measure_ours(runner, K, W, world, rank, local, flush, count_launches):
    """-> (device ms over K steps, e2e ms over K steps, clocks, launches)."""
    import torch

    for _ in range(W):
        runner.run()
    runner.upload()   # the device-resident steps below read inputs already in HBM
    torch.cuda.synchronize()
    barrier(world)
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    dev_ms = 0.0
    launches = 0
    for k in range(K):
        flush.fill_(k & 0xff)                       # evict L2 outside the timed window
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        runner.solve()
        e1.record()
        launches += count_launches
        e1.synchronize()
        dev_ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    barrier(world)
    e2e_ms = 0.0
    for k in range(K):
        flush.fill_(k & 0xff)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        runner.upload()
        runner.solve(download=True)     # per-class D2H overlapped with the other classes
        e1.record()
        launches += count_launches
        e1.synchronize()
        e2e_ms += e0.elapsed_time(e1)
    clk = clocks.stop()
    barrier(world)
    return dev_ms, e2e_ms, clk, launches


def kernel_breakdown(runner, flush, reps=2):
    """Serialised, event-bracketed launches (untimed for `value`): per-kernel
    ms per step plus the outer KM's Dijkstra-step / cost-load counters."""
    import torch

    Q = runner.b.n_plans
    acc: dict[str, float] = {}
    steps = torch.zeros(2 * Q, dtype=torch.int64, device="cuda")
    for r in range(reps):
        flush.fill_(r & 0xff)
        prof = {}
        runner.solve(steps=steps, profile=prof)
        torch.cuda.synchronize()
        for k, v in runner.kernel_ms(prof).items():
            acc[k] = acc.get(k, 0.0) + v / reps
    return acc, steps.cpu().numpy().reshape(-1, 2)


RESHARD_CASES = {
    # SURVEY.md 8(d) / BASELINE.md: [(geometry, old (D,P,M), new (D,P,M))] per GPU count;
    # the first case is the headline, the rest are reported alongside
    2: [("llama-30b", (1, 2, 1), (2, 1, 1))],
    4: [("llama-30b", (1, 2, 2), (1, 1, 4))],
    8: [("gpt-20b", (1, 2, 4), (2, 1, 4)), ("gpt-20b", (1, 4, 2), (1, 2, 4)),
        ("llama-30b", (1, 4, 2), (1, 2, 4))],
}


class _CudaView:
    """Zero-copy uint8 view of a raw device range (for the NCCL baseline)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3}


def run_reshard(world, rank, local, K=3, W=2):
    """Every reshard case for this GPU count, both executor modes (destination
    pull / source push); per case the faster mode is reported, the first case
    is the headline and the others are listed under "other_cases"."""
    cases = RESHARD_CASES.get(world, [("gpt-20b", (1, 2, 1), (2, 1, 1))])
    results = []
    for ci, case in enumerate(cases):
        pull = _reshard_once(world, rank, K, W, "pull", case, comparisons=(ci == 0))
        push = _reshard_once(world, rank, K, W, "push", case, comparisons=False)
        best = pull if pull["ms"] <= push["ms"] else push
        out = dict(best)
        out["modes_ms"] = {"pull": pull["ms"], "push": push["ms"]}
        for k in ("comparisons",):
            if k in pull:
                out[k] = pull[k]
        results.append(out)
    head = results[0]
    if len(results) > 1:
        head["other_cases"] = results[1:]
    return head


def _timed_runs(world, K, W, prep, go):
    """W + K runs, each on a fresh fill (prep), barrier, event-timed go();
    -> min over the K timed runs of the max over ranks (ms)."""
    import torch

    out = []
    for it in range(W + K):
        prep()
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        go()
        e1.record()
        e1.synchronize()
        t = allreduce_max(e0.elapsed_time(e1), world)
        if it >= W:
            out.append(t)
    barrier(world)
    return min(out)


def _reshard_once(world, rank, K, W, mode, case, comparisons):
    """Context reshard of BASELINE.json configs[3]/[4] across the world's GPUs:
    plan from this package's mapper + native planner (memopt order under the
    scenario's U_max), executed by ONE persistent k_exec launch per rank in
    plan order over CUDA-IPC peer mappings, with released old bytes recycled
    for later rounds.  Each timed run starts from a fresh fill of the old
    contexts (a run recycles their released space)."""
    import torch
    import torch.distributed as dist

    from paper_2311_15566_b200 import reshard

    name, old, new = case
    geom = reshard.LLAMA30B_BF16 if name == "llama-30b" else reshard.GPT20B_BF16
    plan, layout, need, model, refs = reshard.make_reshard_problem(geom, old, new, 8, 2048)
    owner = {g: i * world // len(refs) for i, g in enumerate(refs)}
    bin_, bout = reshard.traffic(plan)
    peak_gpu = max(max(bin_.values(), default=0), max(bout.values(), default=0))
    ex = reshard.ReshardExecutor(plan, layout, need, model, owner, rank, world, mode=mode)
    ms = _timed_runs(world, K, W, ex.fill_old, ex.run)
    ctl = ex.control()
    bad = allreduce_sum(float(ex.verify()), world)
    errors = allreduce_sum(float(ctl["error"] != 0), world)
    stage_ready = {str(s): allreduce_max(v, world) for s, v in sorted(ctl["stage_ready_ms"].items())}
    rep = ex.layout.memory_report()
    mine = {g[0] for g in ex.mine}
    mem = {"arena_over_plan_max": max(d["arena_over_plan"] for i, d in rep.items()),
           "per_instance_rank0": {i: {k: d[k] for k in ("old_bytes", "arena_bytes", "plan_peak_usage")}
                                  for i, d in sorted(rep.items()) if i in mine}}
    waits = sum(1 for gl in ex.layout.gpus.values() for e in gl.incoming.values() for _, _, w in e if w >= 0)
    ex.close()
    t = ms / 1e3
    out = {
        "case": f"{name} bf16 {old}->{new}, KV batch 8 x seq 2048, {world} GPUs, u_max 4e9",
        "bytes_total": int(sum(bin_.values())), "bytes_max_gpu": int(peak_gpu),
        "ms": ms, "gbs_per_gpu": peak_gpu / t / 1e9,
        "roofline": {"bound": "nvlink", "peak_nominal_gbs": 900.0, "peak_measured_gbs": 770.0,
                     "frac_nominal": (peak_gpu / 900e9) / t, "frac_measured": (peak_gpu / 770e9) / t},
        "byte_identical": bad == 0, "mismatched_words": int(bad), "run_errors": int(errors),
        "transfers": len(plan.transfers()), "rounds": len(ex.layout.rounds),
        "recycled_extents": waits, "stage_ready_ms": stage_ready, "memory": mem,
        "method": f"k_exec {mode}: one persistent launch per rank, plan (round) order, released bytes "
                  f"recycled with cross-rank waits, device stage-ready flags; 1 MiB chunks over CUDA-IPC",
    }
    if comparisons:
        out["comparisons"] = _reshard_comparisons(world, rank, K, W, plan, layout, need, model, owner, peak_gpu)
    return out


def _reshard_comparisons(world, rank, K, W, plan, layout, need, model, owner, peak_gpu):
    """The same bytes moved three other ways, on a layout that recycles
    nothing (arena = old + every received byte, so order does not matter):
    one unordered k_copy launch, one cudaMemcpyAsync per transfer (copy
    engines), and grouped NCCL send/recv (the paper's mechanism)."""
    import torch
    import torch.distributed as dist

    from paper_2311_15566_b200 import reshard

    ex = reshard.ReshardExecutor(plan, layout, need, model, owner, rank, world, mode="pull", recycle=False)
    res = {}
    for name, fn in (("k_copy_unordered", ex.run_unordered), ("memcpy_per_transfer", ex.run_memcpy)):
        ms = _timed_runs(world, K, W, ex.fill_old, fn)
        bad = allreduce_sum(float(ex.verify()), world)
        res[name] = {"ms": ms, "gbs_per_gpu": peak_gpu / (ms / 1e3) / 1e9, "byte_identical": bad == 0}
    ops = ex.p2p_ops()

    def nccl():
        p2p = []
        for kind, peer, ptr, n in ops:
            if kind == "local":
                nat_copy = torch.as_tensor(_CudaView(ptr[1], n), device="cuda")
                nat_copy.copy_(torch.as_tensor(_CudaView(ptr[0], n), device="cuda"))
                continue
            buf = torch.as_tensor(_CudaView(ptr, n), device="cuda")
            p2p.append(dist.P2POp(dist.isend if kind == "send" else dist.irecv, buf, peer))
        if p2p:
            for r in dist.batch_isend_irecv(p2p):
                r.wait()

    if world > 1:
        ms = _timed_runs(world, K, W, ex.fill_old, nccl)
        bad = allreduce_sum(float(ex.verify()), world)
        res["nccl_grouped_sendrecv"] = {"ms": ms, "gbs_per_gpu": peak_gpu / (ms / 1e3) / 1e9,
                                        "byte_identical": bad == 0}
    ex.close()
    return res


def run_ours(args):
    import torch

    world, rank, local = dist_setup()
    from paper_2311_15566_b200 import sweep

    geom, shapes = sweep.MODELS[args.model]
    batch = sweep.make_sweep(args.positions, args.sets, seed=1000 + rank, model=geom, shapes=shapes)
    runner = sweep.SweepRunner(batch)
    per_step_launches = runner.launches_per_solve
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    K, W = args.steps, args.warmup
    dev_ms, e2e_ms, clk, launches = measure_ours(runner, K, W, world, rank, local, flush,
                                                 per_step_launches)
    dev_ms_max = allreduce_max(dev_ms, world)
    e2e_ms_max = allreduce_max(e2e_ms, world)
    plans_all = allreduce_sum(float(batch.n_plans * K), world)
    value = plans_all / (dev_ms_max / 1e3)
    e2e_value = plans_all / (e2e_ms_max / 1e3)

    kms, st = kernel_breakdown(runner, flush)
    stats = batch.stats()
    nA, nB = stats["nA"], stats["nB"]
    # algorithmic HBM bytes per launch-set (per step):
    #   k_sweep_expand: writes 2 segments (64 B) + row_ptr (4 B) per row, reads descriptors
    #   k_fuse: reads 2 segments per row once + writes the fused weight (8 B; coded: a 1 B
    #     code per padded n x n entry + the 2 KB dictionary) + perm (4 B) per pair
    #   k_outer: reads the fused matrix once (8 B per pair; coded: 1 B per padded entry +
    #     the dictionary), the epilogue's segments (64 B per row), writes assign + total
    pairs = float(stats["pairs"].sum())
    if runner.precoded:
        padded = float((stats["n"].astype(np.float64) ** 2).sum())
        fuse_b = padded + 4 * pairs + 64 * batch.rows + 2048 * batch.n_plans
        outer_b = padded + 2048 * batch.n_plans + 68 * batch.rows + 8 * batch.n_plans
    else:
        fuse_b = 12 * pairs + 64 * batch.rows
        outer_b = 8 * pairs + 68 * batch.rows + 8 * batch.n_plans
    kernels = {
        "k_sweep_expand": {"ms": kms.get("k_sweep_expand", 0.0),
                           "bytes": int(68 * batch.rows + 112 * batch.n_plans)},
        "k_fuse": {"ms": kms.get("k_fuse", 0.0), "bytes": int(fuse_b)},
        "k_outer": {"ms": kms.get("k_outer", 0.0), "bytes": int(outer_b)},
    }
    dom = max(kernels, key=lambda k: kernels[k]["ms"])
    pk, src = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    wl_key = f"{args.model}-N{args.positions}-S{args.sets}"
    # algorithmic bytes per plan = 16*R*C (an int64 W written
    # once by the builder and read once by the matcher).  The fused pipeline
    # never materialises W, so the honest HBM figure is the WHOLE STEP's: 16RC
    # bytes of all plans / device time per step (the ceiling the SURVEY
    # defines, plans/s <= peak / 16RC).  The kernels themselves are bound by
    # instruction issue / latency, measured with ncu (`kernels[*].issue`).
    survey_bytes = 16.0 * float((stats["rows"] * stats["cols"]).sum())
    step_s = dev_ms_max / K / 1e3
    ach = survey_bytes / step_s / 1e9
    traffic_step = None
    kern = {}
    tot_ms = sum(v["ms"] for v in kernels.values()) or 1.0
    for name, v in kernels.items():
        dram = ncu_traffic(name, wl_key)
        issue = ncu_traffic(name + "_issue", wl_key)
        kern[name] = {"ms_serialized": v["ms"], "share": v["ms"] / tot_ms,
                      "design_bytes": v["bytes"], "dram_bytes_ncu": dram,
                      "hbm_frac_measured": (dram / (v["ms"] / 1e3) / 1e9 / hbm) if dram else None,
                      "issue": None if not issue else dict(issue, peak_ipc=4.0,
                                                            frac=issue["ipc"] / 4.0)}
        if dram:
            traffic_step = (traffic_step or 0) + dram
    roofline = {"bound": "hbm", "kernel": "pipeline (k_sweep_expand + k_fuse + k_outer, one step)",
                "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": traffic_step, "peak_source": src,
                "algorithmic_bytes_per_launch": survey_bytes,
                "per_unit": "16*R*C bytes per plan (SURVEY.md 8d) x plans per step, over the "
                            "device time of the whole step",
                "dominant_kernel": dom, "kernels": kern,
                "note": "W is never materialised, so measured DRAM traffic (`traffic`, ncu, per "
                        "step) is below the 16RC figure; k_outer and k_fuse are bound by "
                        "instruction issue / latency (`kernels[*].issue`: ncu IPC of 4)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": dev_ms_max / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args, batch.n_plans), "positions": args.positions,
                   "sets_per_pair": args.sets, "plans_per_step_per_gpu": batch.n_plans,
                   "rows_per_plan_mean": float(stats["rows"].mean()),
                   "outer_n_max": int(stats["n"].max()),
                   "l2": "flushed between timed steps (512 MiB device write, outside the events)",
                   "parallelism": f"plan-sharded x{world} (no collective)"},
        "roofline": roofline,
        "kernels_ms_per_step_serialized": {k: v["ms"] for k, v in kernels.items()},
        "outer_km": {"dijkstra_steps_per_plan": float(st[:, 0].mean()),
                     "steps_per_s": float(st[:, 0].sum()) / (kernels["k_outer"]["ms"] / 1e3)},
        "pipeline_roofline": {"bytes_per_plan_16RC": survey_bytes / batch.n_plans,
                              "ceiling_plans_per_s": hbm * 1e9 * batch.n_plans / survey_bytes,
                              "frac": value / world / (hbm * 1e9 * batch.n_plans / survey_bytes)},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": runner.h2d_bytes,
                "d2h_bytes_per_step": runner.d2h_bytes},
        "gpu_launches": int(allreduce_sum(float(launches), world)),
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        ref = cpu_reference(batch, geom, args.cpu_seconds, cores)
        assign, totals = runner.run()
        ok = _tools().check_answers(ref["answers"], assign, totals, batch.plans)
        line["cpu_baseline"] = {
            "value": ref["rate"], "unit": UNIT, "cores": cores, "kind": ref["kind"],
            "sample": f"{ref['done']} plans of this workload (round-robin over config pairs) in "
                      f"{ref['seconds']:.1f}s on {cores} processes (pool forked before the clock, "
                      f"plans fed continuously): "
                      + ("spotsim.mapping.map_devices, the unmodified reference from baseline/_ref"
                         if ref["kind"] == "reference" else "oracle/port.py (reference absent)"),
            "gpu_results_bit_exact": f"{ok}/{ref['done']}"}
        crate, cdone, cdt = cpu_c_rate(batch, cores, args.cpu_seconds / 2)
        line["cpu_baseline_c"] = {
            "value": crate, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{cdone} plans in {cdt:.1f}s; oracle/spotkm_oracle.c (same algorithm in C, "
                      f"OpenMP)"}
    if world > 1 and not args.no_reshard:
        line["reshard"] = run_reshard(world, rank, local)
    if args.all_sizes:
        del runner
        sizes = {}
        for n_pos in (64, 128, 256, 512, 1024):
            # the full sweep (every config pair x args.sets preemption sets); at the
            # large sizes it runs as consecutive chunks sharing one device scratch
            chunk = min(args.sets, SIZE_CHUNK_SETS[n_pos])
            bs = [sweep.make_sweep(n_pos, min(chunk, args.sets - c * chunk),
                                   seed=2000 + 64 * rank + c, model=geom, shapes=shapes)
                  for c in range(-(-args.sets // chunk))]
            cap = (max(b.rows for b in bs), max(int(b.stats()["pairs"].sum()) for b in bs))
            runs = []
            for b in bs:
                runs.append(sweep.SweepRunner(b, scratch=runs[0] if runs else None, reserve=cap))
            chunked = Chunked(runs)
            k2 = max(2, K // 2) if len(runs) == 1 else 2
            d_ms, x_ms, _, _ = measure_ours(chunked, k2, 2, world, rank, local, flush, 0)
            km = {}
            for r in runs:
                for k, v in kernel_breakdown(r, flush, 1)[0].items():
                    km[k] = km.get(k, 0.0) + v
            q = sum(r.b.n_plans for r in runs)
            rate, e2e_rate = q * k2 / (d_ms / 1e3), q * k2 / (x_ms / 1e3)
            rc = sum(float((r.b.stats()["rows"] * r.b.stats()["cols"]).sum()) for r in runs)
            ceiling = hbm * 1e9 / (16.0 * rc / q)
            entry = {"plans_per_step": q, "chunks": len(runs), "plans_per_s": rate,
                     "e2e_plans_per_s": e2e_rate, "kernels_ms_serialized": km,
                     "pipeline_roofline": {"ceiling_plans_per_s_16RC": ceiling, "frac": rate / ceiling}}
            if rank == 0 and world == 1 and not args.no_cpu_baseline:
                # the reference on a sample of this size's plans, beside the GPU
                ref = cpu_reference(runs[0].b, geom, SIZE_CPU_SECONDS, os.cpu_count() or 1)
                a0, t0 = runs[0].run()
                ok = _tools().check_answers(ref["answers"], a0, t0, runs[0].b.plans)
                entry["cpu_reference"] = {
                    "plans_per_s": ref["rate"], "plans": ref["done"], "seconds": ref["seconds"],
                    "cores": os.cpu_count() or 1, "kind": ref["kind"],
                    "gpu_results_bit_exact": f"{ok}/{ref['done']}",
                    "speedup_device": rate / ref["rate"], "speedup_e2e": e2e_rate / ref["rate"]}
            sizes[str(n_pos)] = entry
            del runs, chunked
        line["sweep_sizes"] = sizes
    if rank == 0 and world == 1 and not args.no_dropin:
        line["dropin"] = _guard(lambda: _tools().dropin_block(_tools().load_spotsim()))
    if rank == 0 and world == 1 and not args.no_k1:
        line["k1_build_weights"] = _guard(lambda: k1_leg(geom, shapes, flush, hbm))
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
