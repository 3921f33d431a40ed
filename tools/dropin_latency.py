"""Latency of the reference-facing drop-in calls on the B_S scenario replans.

Times this package's `map_devices` / `build_graph` (device) and
`plan_migration` (native) on every recorded scenario call
(tests/golden/scenario.json.gz, produced by the real reference), next to the
CPU oracle port (oracle/port.py, a restatement of the reference measured within
~10% of its speed) on the same inputs, and checks bit-exactness.  Prints one
JSON line.  Test/bench tooling: the oracle is only the timed baseline here.
"""

import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests"), str(ROOT / "tests" / "golden")]

import torch  # noqa: E402

from cases import decode_map_case  # noqa: E402
from fmt import load  # noqa: E402
from helpers import assignment_cols, own_problem  # noqa: E402
from oracle import port  # noqa: E402

import paper_2311_15566_b200 as sk  # noqa: E402
from paper_2311_15566_b200 import planner  # noqa: E402
from test_planner import rebuild  # noqa: E402


def best_of(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def main():
    doc = load("scenario")
    rows = []
    for case in doc["maps"]:
        model, cfg, G, insts, inh, rq, fw = own_problem(case)
        got = sk.map_devices(insts, cfg, model, G, inh, rq, fw)
        exact = (assignment_cols(got, insts, cfg) == case["assign"]
                 and got.total_weight.hex() == case["total"])
        t_dev = best_of(lambda: sk.map_devices(insts, cfg, model, G, inh, rq, fw))
        pm, pt, pG, pinst, pinh, preq, pfw = decode_map_case(case)
        t_cpu = best_of(lambda: port.map_devices(pinst, pt, pm, pG, pinh, preq, pfw), reps=2)
        rows.append({"rows": sum(i.gpus for i in insts), "cols": cfg.gpus, "exact": exact,
                     "ms_device": 1e3 * t_dev, "ms_reference_port": 1e3 * t_cpu})
    plans = []
    for d in doc["plans"]:
        if d["error"]:
            continue
        model, mapping, layout, inh_, dep = rebuild(d)
        t = best_of(lambda: planner.plan_migration(mapping, layout, model, u_max=d["u_max"],
                                                   inherited_by_pipeline=inh_, departing=dep))
        plans.append({"transfers": sum(len(a.get("transfers", ())) for a in d["plan"]["actions"]),
                      "ms_native": 1e3 * t})
    out = {"map_devices": rows, "plan_migration": plans,
           "all_exact": all(r["exact"] for r in rows)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
