"""Cluster kernel (TB=4) vs resident on small single lattices.
Usage: python tools/small_cluster.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for L_ in (64, 128, 192, 256):
    line = f"{L_}^2:"
    for C in (0, 2, 4, 8):
        os.environ["KK_CLUSTER"] = str(C)
        L = kk.Lattice(L_, L_, 0.5, 0.6, 3, init=kk.KK_INIT_BLOCK)
        L.sweep(2, s)
        torch.cuda.synchronize()
        n = max(200, int(2e8 / (L_ * L_)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.sweep(n, s)
        e1.record(s)
        torch.cuda.synchronize()
        line += f" {kk.plan(L_, L_, n_sm=0)['kernel']}(C={C}): {n * L_ * L_ / e0.elapsed_time(e1) / 1e6:.2f}"
        L.close()
    print(line + " G/s", flush=True)
