"""TMA staging (KK_TMA=1) against the default LDG staging: same lattice after
a few sweeps?  Usage: KK_TMA=1 python tools/tma_check.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
L = kk.Lattice(4096, 4096, 0.5, 0.6, 11)
L.sweep(3)
a = L.get_packed()
torch.cuda.synchronize()
print("sweeps ok", a.sum())
np.save("gpurun_out/tma_%s.npy" % os.environ.get("KK_TMA", "0"), a)
