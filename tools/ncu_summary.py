"""Summarise ncu outputs for profiles/: a per-kernel launch list share table and key metrics of --set full reports.

usage: python tools/ncu_summary.py launches <launches.csv>
       python tools/ncu_summary.py report <file.ncu-rep> [more.ncu-rep ...]
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
    for r in data:
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        key = r[ki].split("(")[0]
        agg[key][0] += 1
        agg[key][1] += v
    tot = sum(v[1] for v in agg.values())
    print("| share | launches | mean us | kernel |\n|---:|---:|---:|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {t / tot * 100:.1f}% | {n} | {t / n / 1e3:.1f} | `{k}` |")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"### {d.get('Kernel Name', '?')[:120]}  ({path})")
        for k in KEYS:
            if k in d:
                print(f"- {k}: {d[k]}")
        stalls = {k.split("stalled_")[1]: float(v) for k, v in d.items()
                  if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued") and v.replace(".", "").isdigit()}
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:5]
        print("- top stall samples: " + ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in top))
        print()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        for p in sys.argv[2:]:
            report(p)
