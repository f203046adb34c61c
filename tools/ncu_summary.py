"""Summarise an ncu --set full report: key counters + SASS opcode mix.
Usage: python tools/ncu_summary.py report.ncu-rep [updates_per_launch]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
upd = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "thread_inst_executed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
out = {}
for i, h in enumerate(hdr):
    if h in want:
        out[h] = (vals[i], units[i])
        print(f"{h:70s} {vals[i]} {units[i]}")
stalls = []
for i, h in enumerate(hdr):
    if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
        try:
            v = float(vals[i])
        except ValueError:
            continue
        if v > 0.05:
            stalls.append((v, h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
print("stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)))
if upd:
    ti = float(out["thread_inst_executed"][0].replace(",", ""))
    print(f"thread-instructions per update: {ti / upd:.2f}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                      capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(sass)))
h2 = srows[1]
ie, src = h2.index("Instructions Executed"), h2.index("Source")
byop = collections.Counter()
tot = 0
for r in srows[2:]:
    try:
        n = int(r[ie] or 0)
    except (ValueError, IndexError):
        continue
    toks = r[src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    byop[op.split(".")[0]] += n
    tot += n
print("opcode mix:", ", ".join(f"{o}={100 * n / tot:.1f}%" for o, n in byop.most_common(14)))
