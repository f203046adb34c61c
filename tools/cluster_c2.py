"""Cluster size 2/4/8 vs resident for 400^2 replica batches (KK_CLUSTER forced).
Usage: python tools/cluster_c2.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for R in (1, 37, 74):
    line = f"{R} x 400^2:"
    for C in (0, 2, 4, 8):
        os.environ["KK_CLUSTER"] = str(C)
        L = kk.Lattice(400, 400, 0.5, 0.6, 3, replicas=R, init=kk.KK_INIT_BLOCK)
        L.sweep(2, s)
        torch.cuda.synchronize()
        n = max(20, int(4e9 / (160000 * R)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.sweep(n, s)
        e1.record(s)
        torch.cuda.synchronize()
        line += f" C={C}: {n * 160000 * R / e0.elapsed_time(e1) / 1e6:.1f}"
        L.close()
    print(line + " G/s", flush=True)
