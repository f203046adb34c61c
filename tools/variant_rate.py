"""Pass-kernel rate of the library in KK_LIB on the bench lattice and 4096^2.
Usage: KK_LIB=... python tools/variant_rate.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for L_, n in ((65536, 4), (4096, 100)):
    L = kk.Lattice(L_, L_, 0.5, 0.6, 3, init=kk.KK_INIT_BLOCK)
    L.sweep(1, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    L.sweep(n, s)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"{os.environ.get('KK_LIB', 'default')} {L_}^2: {n * L_ * L_ / e0.elapsed_time(e1) / 1e6:.1f} G/s",
          flush=True)
    L.close()
