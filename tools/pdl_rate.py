"""Pass-kernel rate with programmatic dependent launch of consecutive passes (KK_PDL=1) vs plain stream order (KK_PDL=0).
Usage: python tools/pdl_rate.py [sizes...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for L_ in [int(a) for a in sys.argv[1:]] or (1024, 2048, 4096, 8192, 16384, 65536):
    line = f"{L_}^2:"
    for pdl in ("0", "1", "0", "1"):
        os.environ["KK_PDL"] = pdl
        L = kk.Lattice(L_, L_, 0.5, 0.6, 3, init=kk.KK_INIT_BLOCK)
        L.sweep(1, s)
        torch.cuda.synchronize()
        n = max(2, int(8e9 / (L_ * L_)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.sweep(n, s)
        e1.record(s)
        torch.cuda.synchronize()
        line += f" pdl={pdl}: {n * L_ * L_ / e0.elapsed_time(e1) / 1e6:.1f}"
        L.close()
    print(line + " G/s", flush=True)
