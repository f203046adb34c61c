"""Band kernel with temporal blocking (KK_BAND=2, KK_BAND_TB) vs the tile
kernel on mid-size lattices.  Usage: python tools/band_tb.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for L_ in (2048, 4096, 8192, 12288):
    line = f"{L_}^2:"
    for band, tb in ((0, 1), (2, 1), (2, 2), (2, 4), (2, 8)):
        os.environ["KK_BAND"] = str(band)
        os.environ["KK_BAND_TB"] = str(tb)
        L = kk.Lattice(L_, L_, 0.5, 0.6, 3, init=kk.KK_INIT_BLOCK)
        L.sweep(2, s)
        torch.cuda.synchronize()
        n = max(4, int(4e9 / (L_ * L_)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.sweep(n, s)
        e1.record(s)
        torch.cuda.synchronize()
        L.stats()
        name = "tile" if band == 0 else f"band TB={tb}"
        line += f" {name}: {n * L_ * L_ / e0.elapsed_time(e1) / 1e6:.1f}"
        L.close()
    print(line + " G/s", flush=True)
