"""Source lines by warp-stall samples (first kernel matching a substring):  python tools/ncu_lines.py rep [substr] [N]"""
import csv
import io
import subprocess
import sys

rep, kr = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fn, path, rows, take = None, None, [], False
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r and r[0] == "Function Name":
        if rows and r[1] != fn:
            break
        take = kr in r[1]
        if take:
            fn = r[1]
    elif take and len(r) > 5 and r[2] == "-" and r[0].isdigit():
        rows.append((float(r[4] or 0), path, r[0], r[1].strip()))
tot = sum(x[0] for x in rows) or 1
print(f"== {fn[:110]}")
for s, p, ln, src in sorted(rows, key=lambda x: -x[0])[:n]:
    print(f"{100 * s / tot:5.1f}%  {p}:{ln}  {src[:100]}")
