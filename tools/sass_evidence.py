"""Static SASS instruction counts of the sm_100a kernels in libkk.so
(nvdisasm of the extracted cubins: cuobjdump -sass truncates long functions).
Usage: python tools/sass_evidence.py [lib] > profiles/<round>_sass_evidence.txt"""
import collections
import glob
import os
import re
import subprocess
import sys
import tempfile

lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                        "paper_1309_4349_b200", "libkk.so")
WANT = [("planar_pass_kernelILi8ELi768", "planar_pass_kernel<8, 768> (bench kernel)"),
        ("planar_pass_kernelILi8ELi512", "planar_pass_kernel<8, 512> (one-wave mid sizes, 4096^2)"),
        ("pass_kernelILi8ELb1ELi640", "pass_kernel<8, FAST, 640> (row-major tile kernel)"),
        ("cluster_kernelILi256ELi4ELb0", "cluster_kernel<256, 4, DSMEM>"),
        ("ccl_runs_kernel", "ccl_runs_kernel (CCL tile kernel)"),
        ("observe_kernel", "observe_kernel")]
KEYS = ["UTMALDG", "SYNCS", "UCGABAR", "ATOMS", "BAR.SYNC", "IMAD.WIDE.U32", "IMAD.HI", "LOP3.LUT", "PRMT",
        "LDS.128", "ISETP", "SEL", "VIADD", "POPC"]
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, check=True, capture_output=True)
    text = ""
    for cub in sorted(glob.glob(os.path.join(d, "*.cubin"))):
        text += subprocess.run(["nvdisasm", "-c", cub], capture_output=True, text=True).stdout
funcs = {}
cur = None
for ln in text.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", ln)
    if cur and m:
        funcs[cur][m.group(1)] += 1
print("# SASS evidence (static instruction counts, nvdisasm of the sm_100a cubins in libkk.so)")
print("# UTMALDG = TMA tensor load (cp.async.bulk.tensor); SYNCS.* = mbarrier expect-tx / try-wait;")
print("# UCGABAR_* = cluster barrier; ATOMS = shared-memory atomics (XOR flips, CAS unions); IMAD.WIDE.U32 =")
print("# Philox rounds + the 6w split (R6); LOP3.LUT = Philox XORs, bit-plane muxes / full adders;")
print("# ISETP/SEL/VIADD = the acceptance-level compares and bit inserts (R5)")
for key, name in WANT:
    hits = [f for f in funcs if key in f]
    if not hits:
        print(f"{name}: not found")
        continue
    c = funcs[hits[0]]
    parts = [f"{k}={sum(v for op, v in c.items() if op.startswith(k))}" for k in KEYS]
    print(f"{name}: total={sum(c.values())} " + ", ".join(p for p in parts if not p.endswith('=0')))
