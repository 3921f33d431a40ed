"""Summarise an ncu report: key metrics per kernel launch + top stall reasons.

usage: python tools/ncu_summary.py REPORT.ncu-rep [--stalls]
"""
import csv
import io
import subprocess
import sys

KEEP = ["Duration", "Elapsed Cycles", "SM Active Cycles", "Executed Ipc Active", "Issue Slots Busy",
        "Achieved Active Warps Per SM", "Theoretical Active Warps per SM", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "DRAM Throughput", "L2 Hit Rate", "Memory Throughput",
        "Compute (SM) Throughput"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki, ii, mn, mu, mv = (hdr.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Unit",
                                                  "Metric Value"))
    gi = hdr.index("Grid Size")
    by = {}
    for r in rows[1:]:
        if r[mn] in KEEP:
            by.setdefault((r[ii], r[ki].split("(")[0], r[gi]), {})[r[mn]] = f"{r[mv]} {r[mu]}"
    return by


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append((d.get("ID"), d.get("Kernel Name", "").split("(")[0],
                    d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum"),
                    d.get("gpu__time_duration.sum")))
    return rows[1] if len(rows) > 1 else None, res


if __name__ == "__main__":
    rep = sys.argv[1]
    for (i, k, g), m in details(rep).items():
        print(f"[{i}] {k} grid={g}")
        for name in KEEP:
            if name in m:
                print(f"    {name:38s} {m[name]}")
    units, rr = raw(rep)
    print("units:", units and dict(zip(["id", "kernel", "dram_read", "dram_write", "time"],
                                       [units[0], "", units[-3] if len(units) > 3 else "", "", ""])))
    for r in rr:
        print("   ", r)
