"""Band kernel vs tile kernel throughput on mid-size lattices.
Usage: python tools/band_vs_tile.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()


def rate(L_, band):
    os.environ["KK_BAND"] = str(band)
    L = kk.Lattice(L_, L_, 0.5, 0.6, 3, init=kk.KK_INIT_BLOCK)
    L.sweep(2, s)
    torch.cuda.synchronize()
    n = max(4, int(4e9 / (L_ * L_)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    L.sweep(n, s)
    e1.record(s)
    torch.cuda.synchronize()
    L.stats()  # raises if the band exchange timed out
    L.close()
    return n * L_ * L_ / e0.elapsed_time(e1) / 1e6


for L_ in (1024, 2048, 4096, 8192, 12288):
    print(f"{L_}^2: tile {rate(L_, 0):.1f} | band {rate(L_, 2):.1f} G site-updates/s", flush=True)
