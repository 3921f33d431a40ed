"""Fold one `ncu --set full` report of a bench pass into profiles/ncu_traffic.json:
per kernel (all launches of the pass summed) DRAM bytes, and duration-weighted
IPC / issue-slot utilisation (the issue roofline of the latency/issue-bound KM
kernels).  usage: python tools/ncu_to_json.py REPORT.ncu-rep WORKLOAD_KEY"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

rep, key = sys.argv[1], sys.argv[2]
ROOT = Path(__file__).resolve().parents[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9,
         "us": 1e-6, "ms": 1e-3, "s": 1.0}
metrics = {"dram__bytes_read.sum": "r", "dram__bytes_write.sum": "w",
           "gpu__time_duration.sum": "t", "sm__instruction_throughput.avg.pct_of_peak_sustained_active": "x",
           "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue",
           "sm__inst_executed.avg.per_cycle_active": "ipc"}
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
agg = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0]
    a = agg.setdefault(name, {"bytes": 0.0, "t": 0.0, "ipc_t": 0.0, "issue_t": 0.0, "launches": 0})
    val = {}
    for m, k in metrics.items():
        if m in hdr and d.get(m, "") not in ("", "n/a"):
            u = units[hdr.index(m)]
            val[k] = float(d[m].replace(",", "")) * SCALE.get(u, 1.0)
    t = val.get("t", 0.0)
    a["bytes"] += val.get("r", 0.0) + val.get("w", 0.0)
    a["t"] += t
    a["ipc_t"] += val.get("ipc", 0.0) * t
    a["issue_t"] += val.get("issue", 0.0) * t
    a["launches"] += 1
path = ROOT / "profiles" / "ncu_traffic.json"
doc = json.loads(path.read_text()) if path.exists() else {}
entry = {}
for name, a in agg.items():
    entry[name] = int(a["bytes"])
    if a["t"] > 0:
        entry[name + "_issue"] = {"ipc": round(a["ipc_t"] / a["t"], 3),
                                  "issue_active_pct": round(a["issue_t"] / a["t"], 1),
                                  "launches": a["launches"], "ncu_ms": round(1e3 * a["t"], 3)}
doc[key] = entry
path.write_text(json.dumps(doc, indent=1) + "\n")
print(json.dumps(entry, indent=1))
