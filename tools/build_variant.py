"""Build libkk.so variants with extra -D flags into build/var/libkk_<name>.so
(for A/B rate measurements with KK_LIB=...; not the product build).

  python tools/build_variant.py NAME [-DFOO=1 ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1309_4349_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "build", "var", f"libkk_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
flags = [f for f in B.NVCC_FLAGS if f != "-v" and f != "-Xptxas"]
cmd = ["nvcc", *flags, *defs, "-o", out, *[os.path.join(B.CSRC, s) for s in B.SOURCES]]
r = subprocess.run(cmd, cwd=B.CSRC, capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stdout + r.stderr)
    sys.exit(1)
print(out)
