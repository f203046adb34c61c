"""Time the pass kernel for tile/T settings (CUDA events, warm, 1 GPU).
Usage: python tools/tune_pass.py Lx Ly "T,THI,TWI;T,THI,TWI;..." [replicas] """
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

Lx, Ly = int(sys.argv[1]), int(sys.argv[2])
R = int(sys.argv[4]) if len(sys.argv) > 4 else 1
cfgs = [tuple(int(v) for v in c.split(",")) for c in sys.argv[3].split(";")]
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for (T, THI, TWI) in cfgs:
    os.environ["KK_THI"], os.environ["KK_TWI"] = str(THI), str(TWI)
    L = kk.Lattice(Lx, Ly, 0.5, 0.6, 3, iters_per_pass=T, init=kk.KK_INIT_BLOCK, replicas=R)
    L.sweep(2, s)
    torch.cuda.synchronize()
    n = max(1, int(4e9 / (Lx * Ly * R)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    L.sweep(n, s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"T={T} THI={THI} TWI={TWI}: {n} sweeps {ms:.2f} ms -> {n * Lx * Ly * R / ms / 1e6:.1f} G site-updates/s",
          flush=True)
    L.close()
