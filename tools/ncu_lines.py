"""Warp-stall samples aggregated per CUDA source line (needs -lineinfo and
ncu --import-source on).  usage: python tools/ncu_lines.py REPORT [kernel-substring] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
for blk in out.split('"File Path"')[1:]:
    rows = list(csv.reader(io.StringIO('"File Path"' + blk)))
    fn = rows[1][1] if len(rows) > 1 else ""
    if ksub and ksub not in fn:
        continue
    hdr = rows[2]
    samp = hdr.index("Warp Stall Sampling (All Samples)")
    acc, src, cur = {}, {}, None
    for r in rows[3:]:
        if len(r) <= samp:
            continue
        if r[0]:
            cur = int(r[0])
            src[cur] = r[1]
        try:
            acc[cur] = acc.get(cur, 0) + int(r[samp] or 0)
        except ValueError:
            pass
    tot = sum(acc.values()) or 1
    print("==", fn[:110], "samples", tot)
    for ln, v in sorted(acc.items(), key=lambda x: -x[1])[:top]:
        print(f"  {100 * v / tot:5.1f}%  {ln:5d}  {src.get(ln, '').strip()[:90]}")
