"""Resident-kernel throughput vs CTA size (KK_RES_THREADS) and replica count.
Usage: python tools/res_threads.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()


def rate(Lx, Ly, R, nt):
    os.environ["KK_RES_THREADS"] = str(nt)
    L = kk.Lattice(Lx, Ly, 0.5, 0.6, 3, replicas=R, init=kk.KK_INIT_BLOCK)
    L.sweep(1, s)
    torch.cuda.synchronize()
    n = max(2, int(2e9 / (Lx * Ly * R)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    L.sweep(n, s)
    e1.record(s)
    torch.cuda.synchronize()
    L.close()
    return n * Lx * Ly * R / e0.elapsed_time(e1) / 1e6


for (Lx, Ly, R) in [(400, 400, 1024), (400, 400, 296), (400, 400, 148), (400, 400, 16), (400, 400, 1),
                    (64, 64, 1), (64, 64, 4096), (1024, 1024, 148)]:
    print(f"{R} x {Lx}x{Ly}: " + " | ".join(f"{nt}: {rate(Lx, Ly, R, nt):.1f}" for nt in (0, 128, 256, 512)),
          flush=True)
