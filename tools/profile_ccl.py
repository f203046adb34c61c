"""Driver for ncu captures of the cluster-histogram kernels on an equilibrated
lattice.  Usage: python tools/profile_ccl.py [L] [sweeps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
torch.cuda.set_device(0)
lat = kk.Lattice(L, L, 0.5, 0.6, 7)
lat.sweep(n)
h = lat.cluster_histogram(1)[0]
h = lat.cluster_histogram(1)[0]
torch.cuda.synchronize()
print("clusters", sum(c for _, c in h), "largest", max(s for s, _ in h))
