"""Default plan vs forced CTA sizes on one-wave tile grids.
Usage: python tools/nt_default.py [sizes...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for L_ in [int(a) for a in sys.argv[1:]] or (2560, 3072, 4096, 5120, 6144, 7168):
    line = f"{L_}^2 (default {kk.plan(L_, L_)['threads']}):"
    for nt in ("0", "512", "640"):
        os.environ["KK_PASS_THREADS"] = nt
        L = kk.Lattice(L_, L_, 0.5, 0.6, 3, init=kk.KK_INIT_BLOCK)
        L.sweep(1, s)
        torch.cuda.synchronize()
        n = max(2, int(8e9 / (L_ * L_)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.sweep(n, s)
        e1.record(s)
        torch.cuda.synchronize()
        line += f" {'default' if nt == '0' else nt}: {n * L_ * L_ / e0.elapsed_time(e1) / 1e6:.1f}"
        L.close()
    print(line + " G/s", flush=True)
