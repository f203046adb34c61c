"""Cluster kernel: halo exchange every TB iterations (KK_CLUSTER_TB) on
single lattices.  Usage: python tools/cluster_tb.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for (L_, R, C) in ((400, 1, 8), (400, 1, 16), (512, 1, 8), (512, 1, 16), (400, 18, 8), (400, 74, 2)):
    line = f"{R} x {L_}^2 C={C}:"
    for tb in (1, 2, 4, 8):
        os.environ["KK_CLUSTER"] = str(C)
        os.environ["KK_CLUSTER_TB"] = str(tb)
        L = kk.Lattice(L_, L_, 0.5, 0.6, 3, replicas=R, init=kk.KK_INIT_BLOCK)
        L.sweep(2, s)
        torch.cuda.synchronize()
        n = max(20, int(2e9 / (L_ * L_ * R)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.sweep(n, s)
        e1.record(s)
        torch.cuda.synchronize()
        line += f" TB={tb}: {n * L_ * L_ * R / e0.elapsed_time(e1) / 1e6:.2f}"
        L.close()
    print(line + " G/s", flush=True)
