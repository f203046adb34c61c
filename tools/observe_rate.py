"""Device time of kk_energy / kk_composition (observe_kernel) and the HBM rate
it reaches (bytes = the lattice once).  Usage: python tools/observe_rate.py [L]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
lat = kk.Lattice(L, L, 0.5, 0.6, 3, init=kk.KK_INIT_BLOCK)
lat.energy(stream=s)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    lat.energy(stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = min(ts)
print(f"{L}^2 kk_energy: {ms:.3f} ms (incl. the host read-back) -> {L * L / 8 / (ms / 1e3) / 1e9:.0f} GB/s of lattice")
