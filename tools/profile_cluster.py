"""ncu driver for the cluster kernel on one 400x400 lattice (BASELINE
configs[1]).  Usage: python tools/profile_cluster.py [sweeps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
torch.cuda.set_device(0)
L = kk.Lattice(400, 400, 0.5, 0.6, 7)
L.sweep(n)
torch.cuda.synchronize()
print("ok", kk.plan(400, 400, n_sm=0)["kernel"], L.stats()[0].tolist())
