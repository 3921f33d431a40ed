"""Per-source-line memory counters of one kernel in an ncu report (needs
-lineinfo and --import-source on): the lines moving the most global sectors.
usage: python tools/ncu_line_mem.py REPORT [kernel-substring] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
for blk in out.split('"File Path"')[1:]:
    rows = list(csv.reader(io.StringIO('"File Path"' + blk)))
    fn = rows[1][1] if len(rows) > 1 else ""
    if ksub and ksub not in fn:
        continue
    hdr = rows[2]
    print("   header:", hdr)
    cols = [i for i, h in enumerate(hdr) if "Sector" in h or "L2" in h or "Global" in h]
    print("==", fn[:100])
    print("   columns:", [hdr[i] for i in cols])
    best = []
    for r in rows[3:]:
        if len(r) <= max(cols, default=0) or not r[0]:
            continue
        vals = []
        for i in cols:
            try:
                vals.append(float(r[i] or 0))
            except ValueError:
                vals.append(0.0)
        best.append((sum(vals), r[0], r[1].strip()[:80], vals))
    for tot, ln, src, vals in sorted(best, key=lambda x: -x[0])[:top]:
        print(f"  {ln:>5} {tot:14.0f}  {src}")
        print("        ", [int(v) for v in vals])
