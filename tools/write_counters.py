"""Write profiles/pass_kernel_counters.json (read by bench.py for the roofline)
from an ncu --set full capture of one bench-lattice pass, stamped with the
launch plan it was captured under (kk_plan_config of the 65536^2 bench lattice
on a 148-SM B200): bench.py refuses the counters if its own plan differs.
Usage: python tools/write_counters.py report.ncu-rep updates_per_launch "tile description" [out.json]"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1309_4349_b200 import kk  # noqa: E402
import bench  # noqa: E402

rep, upd, tile = sys.argv[1], float(sys.argv[2]), sys.argv[3]
out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                         "profiles", "pass_kernel_counters.json")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]


def val(name):
    x = float(v[h.index(name)].replace(",", ""))
    u = units[h.index(name)]
    return x * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}.get(u, 1.0)


name = v[h.index("Kernel Name")]
d = {
    "kernel": name.split("(")[0].replace("void ", "").replace("unnamed>::", ""),
    "T": 8,
    "thread_inst_per_update": val("thread_inst_executed") / upd,
    "dram_bytes_per_update": (val("dram__bytes_read.sum") + val("dram__bytes_write.sum")) / upd,
    "launch_ms_ncu": val("gpu__time_duration.sum"),
    "issue_active_pct": round(val("smsp__issue_active.avg.pct_of_peak_sustained_active"), 2),
    "alu_pipe_pct": round(val("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"), 2),
    "fma_pipe_pct": round(val("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"), 2),
    "fmaheavy_pipe_pct": round(val("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"), 2),
    "source": os.environ.get("KK_COUNTERS_SOURCE", f"ncu --set full --clock-control none of the bench lattice; "
                                                    f"{os.path.basename(rep)}"),
    "tile": tile,
    "source_sha256": bench.pass_source_sha256(kk.plan(65536, 65536, iters_per_pass=8, n_sm=148)["kernel"]),
    "plan": {k: v for k, v in kk.plan(65536, 65536, iters_per_pass=8, n_sm=148).items()
             if k in ("kernel", "iters_per_pass", "tile_words", "tile_rows", "threads", "tma_boxes")},
}
with open(out, "w") as f:
    json.dump(d, f, indent=1)
print(json.dumps(d, indent=1))
