"""Group an ncu SASS source page (csv) by execution count: which code blocks
(same count = same basic-block frequency) carry the instructions.
Usage: ncu -i rep --page source --csv --print-source=sass > x.csv; python tools/sass_hot.py x.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie, src = h.index("Instructions Executed"), h.index("Source")
data = []
for r in rows[2:]:
    try:
        n = int(r[ie] or 0)
    except (ValueError, IndexError):
        continue
    data.append((n, r[src].strip()))
tot = sum(n for n, _ in data)
agg, cnt, ex = defaultdict(int), defaultdict(int), defaultdict(list)
for n, s in data:
    agg[n] += n
    cnt[n] += 1
    if len(ex[n]) < 2:
        ex[n].append(s[:40])
for n, v in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
    print(f"count={n:10d} ninstr={cnt[n]:4d} {100 * v / tot:5.1f}%  e.g. {ex[n]}")
