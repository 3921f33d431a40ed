"""Per-kernel stall-reason breakdown + top stalled SASS lines from an ncu report.

usage: python tools/ncu_stalls.py REPORT.ncu-rep [kernel-substring] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
out = subprocess.run(args, capture_output=True, text=True).stdout
blocks = [b for b in out.split('"Kernel Name"') if b.strip()]
for blk in blocks:
    lines = blk.split("\n")
    name = lines[0]
    if ksub and ksub not in name:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    if not rows:
        continue
    hdr = rows[0]
    names = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    idx = {n: hdr.index(n) for n in names}
    tot = {n: 0 for n in names}
    src = hdr.index("Source")
    samp = hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        for n in names:
            try:
                tot[n] += int(r[idx[n]] or 0)
            except ValueError:
                pass
        try:
            data.append((int(r[samp] or 0), r[0], r[src]))
        except ValueError:
            pass
    s = sum(tot.values()) or 1
    print("==", name[:100])
    print("   " + ", ".join(f"{n[6:]} {100 * v / s:.1f}%" for n, v in
                            sorted(tot.items(), key=lambda x: -x[1]) if v))
    S = sum(d[0] for d in data) or 1
    for d in sorted(data, reverse=True)[:top]:
        print(f"   {100 * d[0] / S:5.1f}%  {d[2][:90]}")
