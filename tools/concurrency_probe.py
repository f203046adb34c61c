"""Do independent handles on separate streams run concurrently?  Host time of
each kk_sweep call and per-stream end times relative to a common start.
Usage: python tools/concurrency_probe.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
lib = kk.load()
for n_lat, env in ((4, {}), (4, {"KK_RESIDENT": "0"})):
    for k, v in env.items():
        os.environ[k] = v
    streams = [torch.cuda.Stream() for _ in range(n_lat)]
    lats = [kk.Lattice(400, 400, 0.5, 0.6, 1 + i) for i in range(n_lat)]
    for L, s in zip(lats, streams):
        L.sweep(10, s)
    torch.cuda.synchronize()
    calls = []
    t0 = time.perf_counter()
    for L, s in zip(lats, streams):
        a = time.perf_counter()
        rc = lib.kk_sweep(L._h, 1000, ctypes.c_void_p(s.cuda_stream))
        calls.append(1e3 * (time.perf_counter() - a))
    t_enq = time.perf_counter() - t0
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{n_lat} lattices {env}: wall {1e3 * dt:.1f} ms, kk_sweep host times (ms): "
          + " ".join(f"{c:.2f}" for c in calls), flush=True)
    for L in lats:
        L.close()
    for k in env:
        os.environ.pop(k)
