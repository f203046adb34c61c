"""Per-CUDA-source-line totals of an ncu report: thread instructions and warp
instructions per unit (e.g. per site update) and warp-stall samples.
Usage: python tools/ncu_lines.py report.ncu-rep [units] [top_n] [--sort line]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
by_line = "--sort" in sys.argv and sys.argv[-1] == "line"
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
fname, hdr = None, None
agg = defaultdict(lambda: [0, 0, 0, ""])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ti, wi, sm = hdr.index("Thread Instructions Executed"), hdr.index("Instructions Executed"), hdr.index("# Samples")
        continue
    if hdr is None or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    try:
        agg[key][0] += int(r[ti] or 0)
        agg[key][1] += int(r[wi] or 0)
        agg[key][2] += int(r[sm] or 0)
    except (ValueError, IndexError):
        pass
    if not agg[key][3]:
        agg[key][3] = r[1].strip()[:72]
tot_w = sum(v[1] for v in agg.values()) or 1
tot_s = sum(v[2] for v in agg.values()) or 1
print(f"total: thread-inst {sum(v[0] for v in agg.values()) / units:.2f}/unit, warp-inst {tot_w / units:.4f}/unit, "
      f"samples {tot_s}")
items = sorted(agg.items()) if by_line else sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]
for k, v in items:
    if by_line and v[1] / tot_w < 0.002:
        continue
    print(f"{k[0]:>16s}:{k[1]:<5d} thr {v[0] / units:7.3f} warp {v[1] / units:8.4f} ({100 * v[1] / tot_w:4.1f}%) "
          f"samples {100 * v[2] / tot_s:4.1f}%  {v[3]}")
