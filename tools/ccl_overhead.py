"""Where a 65536^2 kk_cluster_histogram call spends its time beyond the CCL
kernels: device-timed (CUDA events) per call through the Python list API, the
raw-rows API, and with the lattice already in the public layout (no planar ->
row-major conversion).  Usage: python tools/ccl_overhead.py [L] [sweeps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
lat = kk.Lattice(L, L, 0.5, 0.6, 5)
lat.sweep(n, s)
lat.cluster_histogram(1, stream=s)
torch.cuda.synchronize()


def timed(fn, sweep_first):
    best, wall = 1e9, 1e9
    for _ in range(3):
        if sweep_first:
            lat.sweep(1, s)  # back to the planar layout
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        wall = min(wall, (time.perf_counter() - t0) * 1e3)
        best = min(best, e0.elapsed_time(e1))
    return best, wall


for name, fn, sw in [("list API after a sweep (planar layout)", lambda: lat.cluster_histogram(1, stream=s), True),
                     ("list API, public layout", lambda: lat.cluster_histogram(1, stream=s), False),
                     ("raw rows API, public layout", lambda: lat.cluster_histogram_raw(1, stream=s), False)]:
    ev, wall = timed(fn, sw)
    print(f"{name:42s} events {ev:7.2f} ms   host wall {wall:7.2f} ms", flush=True)
