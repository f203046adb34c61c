"""Band kernel (default 8192^2..12288^2) vs a one-wave tile grid with
640-thread CTAs and PDL.  Usage: python tools/band_vs_wide_tile.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()


def rate(L_, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        L = kk.Lattice(L_, L_, 0.5, 0.6, 3, init=kk.KK_INIT_BLOCK)
        L.sweep(1, s)
        torch.cuda.synchronize()
        n = max(2, int(8e9 / (L_ * L_)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.sweep(n, s)
        e1.record(s)
        torch.cuda.synchronize()
        L.close()
        return n * L_ * L_ / e0.elapsed_time(e1) / 1e6
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


for L_, thi, twi in ((8192, 224, 64), (8192, 112, 128), (10240, 356, 64), (12288, 512, 64), (12288, 256, 128)):
    line = f"{L_}^2: default {rate(L_, {}):.1f}"
    for nt in ("640", "512"):
        line += (f" tile {thi}x{twi} nt={nt} pdl=1: "
                 f"{rate(L_, {'KK_BAND': '0', 'KK_THI': str(thi), 'KK_TWI': str(twi), 'KK_PASS_THREADS': nt, 'KK_PDL': '1'}):.1f}")
    print(line + " G/s", flush=True)
