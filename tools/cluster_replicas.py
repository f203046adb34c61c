"""Default plan (cluster kernel when R*8 <= #SMs) vs KK_CLUSTER=0 (resident)
for replica batches of 400^2.  Usage: python tools/cluster_replicas.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for R in (1, 4, 16, 18, 19, 64):
    line = f"{R} x 400^2:"
    for mode in (None, "0"):
        if mode is None:
            os.environ.pop("KK_CLUSTER", None)
        else:
            os.environ["KK_CLUSTER"] = mode
        L = kk.Lattice(400, 400, 0.5, 0.6, 3, replicas=R, init=kk.KK_INIT_BLOCK)
        L.sweep(2, s)
        torch.cuda.synchronize()
        n = max(20, int(4e9 / (160000 * R)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.sweep(n, s)
        e1.record(s)
        torch.cuda.synchronize()
        name = kk.plan(400, 400, replicas=R, n_sm=0)["kernel"] if mode is None else "resident"
        line += f" {name}: {n * 160000 * R / e0.elapsed_time(e1) / 1e6:.1f}"
        L.close()
    print(line + " G/s", flush=True)
