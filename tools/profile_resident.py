"""ncu driver for the resident kernel on BASELINE configs[3] (1024 replicas
of 400x400).  Usage: python tools/profile_resident.py [replicas] [sweeps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
torch.cuda.set_device(0)
L = kk.Lattice(400, 400, 0.5, 0.6, 7, replicas=R)
L.sweep(n)
torch.cuda.synchronize()
print("ok", L.stats()[0].tolist(), int(L.energy()[0][0]))
