"""Cluster-histogram cost on the replica batch (configs[3]): C call vs the
Python list API.  Usage: python tools/ccl_rep_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
L = kk.Lattice(400, 400, 0.5, 0.6, 5, replicas=1024)
L.sweep(100, s)
L.cluster_histogram(1, stream=s)
torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter()
    raw = L.cluster_histogram_raw(1, stream=s)
    t1 = time.perf_counter()
    h = L.cluster_histogram(1, stream=s)
    t2 = time.perf_counter()
    print(f"raw C call {1e3 * (t1 - t0):.1f} ms ({len(raw)} rows); list API {1e3 * (t2 - t1):.1f} ms", flush=True)
