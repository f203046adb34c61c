"""16-CTA (non-portable) vs 8-CTA clusters for single lattices and small
replica batches.  Usage: python tools/cluster16.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for (L_, R) in ((320, 1), (384, 1), (400, 1), (448, 1), (512, 1), (640, 1), (400, 2), (400, 4), (512, 4), (400, 8)):
    line = f"{R} x {L_}^2:"
    for C in (8, 16):
        os.environ["KK_CLUSTER"] = str(C)
        try:
            L = kk.Lattice(L_, L_, 0.5, 0.6, 3, replicas=R, init=kk.KK_INIT_BLOCK)
        except kk.KKError:
            line += f" C={C}: n/a"
            continue
        L.sweep(2, s)
        torch.cuda.synchronize()
        n = max(20, int(4e8 / (L_ * L_ * R)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.sweep(n, s)
        e1.record(s)
        torch.cuda.synchronize()
        line += f" C={C}: {n * L_ * L_ * R / e0.elapsed_time(e1) / 1e6:.2f}"
        L.close()
    print(line + " G/s", flush=True)
