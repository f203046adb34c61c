"""Single small lattices: tile vs resident kernel, and concurrency of several
handles on separate streams (resident: one launch per kk_sweep call).
Usage: python tools/single_small.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
for L_ in (64, 256, 400, 1024):
    for mode in ("0", "2"):
        os.environ["KK_RESIDENT"] = mode
        for n_lat in (1, 18):
            streams = [torch.cuda.Stream() for _ in range(n_lat)]
            lats = [kk.Lattice(L_, L_, 0.5, 0.6, 1 + i) for i in range(n_lat)]
            for L, s in zip(lats, streams):
                L.sweep(10, s)
            torch.cuda.synchronize()
            n = max(20, int(2e8 / (L_ * L_)))
            t0 = time.perf_counter()
            for L, s in zip(lats, streams):
                L.sweep(n, s)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            print(f"{L_}^2 x {n_lat} {'resident' if mode == '2' else 'tile'}: {n} sweeps each, {1e3 * dt:.1f} ms "
                  f"-> {n_lat * n * L_ * L_ / dt / 1e9:.2f} G/s", flush=True)
            for L in lats:
                L.close()
