"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV).
Usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
agg = collections.defaultdict(list)
for r in rows[h + 1:]:
    if len(r) > mi and r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0].replace("void ", "").replace("kk::<unnamed>::", "")
        agg[name].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':55s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:55s} {len(v):8d} {sum(v):12.1f} {sum(v) / len(v):10.1f} {sum(v) / tot:6.3f}")
print(f"{'TOTAL':55s} {sum(len(v) for v in agg.values()):8d} {tot:12.1f}")
