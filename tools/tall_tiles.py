"""Bench lattice: 2 CTAs/SM x 384 threads (cost-model tiles) vs 1 CTA/SM x 640
threads with tall tiles.  Usage: python tools/tall_tiles.py [L] [sweeps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
L_ = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfgs = [("default", {}), ("KK_TALL=0", {"KK_TALL": "0"})] + [
    (f"640 x {h}", {"KK_PASS_THREADS": "640", "KK_THI": str(h), "KK_TWI": "64"}) for h in (560, 596, 660)]
for rep in range(2):
    for name, env in cfgs:
        for k in ("KK_PASS_THREADS", "KK_THI", "KK_TWI", "KK_TALL"):
            os.environ.pop(k, None)
        os.environ.update(env)
        L = kk.Lattice(L_, L_, 0.5, 0.6, 3, init=kk.KK_INIT_BLOCK)
        L.sweep(1, s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.sweep(n, s)
        e1.record(s)
        torch.cuda.synchronize()
        print(f"{L_}^2 {name}: {n * L_ * L_ / e0.elapsed_time(e1) / 1e6:.1f} G/s", flush=True)
        L.close()
