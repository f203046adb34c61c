"""A/B rates of the default plan on small and mid lattices (site-updates/s),
for comparing two builds: KK_LIB=path/to/libkk.so python tools/ab_rate.py [Lx ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
out = []
for (Lx, Ly, R) in ((64, 64, 1), (256, 256, 1), (400, 400, 1), (512, 512, 1), (1024, 1024, 1),
                    (4096, 4096, 1), (8192, 8192, 1), (12288, 12288, 1), (400, 400, 37), (400, 400, 74), (400, 400, 1024)):
    if len(sys.argv) > 1 and str(Lx) not in sys.argv[1:]:
        continue
    L = kk.Lattice(Lx, Ly, 0.5, 0.6, 3, replicas=R, init=kk.KK_INIT_BLOCK)
    L.sweep(4, s)
    torch.cuda.synchronize()
    n = max(16, int(2e9 / (Lx * Ly * R)) // 16 * 16)
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.sweep(n, s)
        e1.record(s)
        torch.cuda.synchronize()
        best = max(best, n * Lx * Ly * R / e0.elapsed_time(e1) / 1e6)
    out.append(f"{R}x{Lx}x{Ly} {kk.plan(Lx, Ly, replicas=R, n_sm=0)['kernel']}: {best:.2f} G/s")
    L.close()
print(os.environ.get("KK_LIB", "default"), " | ".join(out))
