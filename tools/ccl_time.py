"""Device time of kk_cluster_histogram on equilibrating lattices (random
start + S sweeps).  Usage: python tools/ccl_time.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for (Lx, Ly, R, S) in [(65536, 65536, 1, 20), (16384, 16384, 1, 100), (400, 400, 1024, 100), (4096, 4096, 1, 100)]:
    L = kk.Lattice(Lx, Ly, 0.5, 0.6, 5, replicas=R)
    L.sweep(S, s)
    L.cluster_histogram(1, stream=s)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        h = L.cluster_histogram(1, stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{R} x {Lx}x{Ly} after {S} sweeps: cluster histogram {min(ts):.2f} ms "
          f"({sum(c for _, c in h[0])} clusters in replica 0)", flush=True)
    L.close()
