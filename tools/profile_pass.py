"""Small driver for ncu captures of the pass kernel (kept short: ncu replays
each kernel ~40x).  Usage: python tools/profile_pass.py [Lx] [Ly] [sweeps] [T]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

Lx = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
Ly = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
n = int(sys.argv[3]) if len(sys.argv) > 3 else 2
T = int(sys.argv[4]) if len(sys.argv) > 4 else 4
torch.cuda.set_device(0)
L = kk.Lattice(Lx, Ly, 0.5, 0.6, 7, iters_per_pass=T)
L.sweep(n)
torch.cuda.synchronize()
print("ok", L.stats()[0].tolist(), L.energy()[0][0])
