"""Hottest SASS instructions by warp-stall samples, per kernel of an ncu report.

    python tools/ncu_hot.py <report.ncu-rep> [kernel-substring] [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kr = sys.argv[2] if len(sys.argv) > 2 else ""
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "hdr": None, "rows": []}
        blocks.append(cur)
    elif cur is not None and r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and cur["hdr"] and len(r) == len(cur["hdr"]):
        cur["rows"].append(r)
for b in blocks:
    if kr and kr not in b["name"]:
        continue
    h = b["hdr"]
    si = h.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[si] or 0) for r in b["rows"]) or 1.0
    print(f"== {b['name'][:100]}  ({tot:.0f} samples)")
    rows = sorted(b["rows"], key=lambda r: -float(r[si] or 0))
    for r in rows[:n]:
        print(f"{100 * float(r[si] or 0) / tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:100]}")
    break
