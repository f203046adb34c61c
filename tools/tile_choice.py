"""Pass-kernel throughput with the automatic tile choice vs forced shapes.
Usage: python tools/tile_choice.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()


def rate(Lx, Ly, env):
    for k in ("KK_TWI", "KK_THI", "KK_RESIDENT"):
        os.environ.pop(k, None)
    os.environ["KK_RESIDENT"] = "0"
    for k, v in env.items():
        os.environ[k] = str(v)
    L = kk.Lattice(Lx, Ly, 0.5, 0.6, 3, init=kk.KK_INIT_BLOCK)
    L.sweep(2, s)
    torch.cuda.synchronize()
    n = max(2, int(3e9 / (Lx * Ly)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    L.sweep(n, s)
    e1.record(s)
    torch.cuda.synchronize()
    L.close()
    return n * Lx * Ly / e0.elapsed_time(e1) / 1e6


for (Lx, Ly, alts) in [(1024, 1024, [(8, 28), (8, 64), (32, 32)]),
                       (2048, 2048, [(8, 116), (16, 56), (32, 28)]),
                       (4096, 4096, [(32, 56), (16, 228), (16, 112), (32, 112), (64, 28)]),
                       (8192, 8192, [(32, 224), (64, 112), (64, 320)]),
                       (16384, 16384, [(64, 300), (64, 320), (32, 444)]),
                       (65536, 65536, [(64, 320), (64, 332)])]:
    line = f"{Lx}x{Ly}: auto {rate(Lx, Ly, {}):.1f}"
    for (twi, thi) in alts:
        line += f" | {twi}w x {thi}r {rate(Lx, Ly, {'KK_TWI': twi, 'KK_THI': thi}):.1f}"
    print(line, flush=True)
